// gram_kernel.cuh — the tile engine: K1 (tall-skinny Gram on fp64 tensor cores) and K12 (the
// block update of step k fused in front of the Gram of step k+1).
//
// K1 replaces fused_gram (dist_block.cpp:79-88) + gram_accumulate (dense_kernels.cpp:10-27)
// + the per-rank half of exact_allreduce (communicator.cpp:226-250).  K12 additionally
// replaces the local_axpy_block / scale_right_block / set_block sequence that sits between
// two syncs of onesync_impl (bcgs.cpp:329-331, 346-359) and pipi_impl (bcgs.cpp:196-214):
//
//   A = (srcA - Qp CA) TA^{-1}            e.g. Q_k     = (U_k - Q_{1:k} Y) Y_kk^{-1}
//   B = (srcB - Qp CB - A S2) TB^{-1}     e.g. U_{k+1} = (X_{k+1} - Q_{1:k} Z - Q_k S2) S^{-1}
//   G = [tile]^T [right columns]          the next step's fused Gram, on the updated tile
//
// so each block step streams the Q prefix from HBM once instead of twice.
//
// Accuracy: the reference accumulates every product exactly (2176-bit fixed point).  Here
// each RS-row stage is contracted with DMMA.8x8x4 into a fresh accumulator that is folded
// into a double-double (hi, lo) pair every GRAM_FLUSH stages; CTA partials are summed in a
// fixed order in double-double (gram_reduce) — deterministic, O(RS u) per entry.
//
// Tile geometry.  A stage is RS = 16H rows (H = 2 or 4) x all tile columns, loaded by TMA
// through a 3-D view of the column-major matrix: dims {16, ceil(rows/16), cols}, strides
// {128 B, ld*8 B}, box {16, H, w}, SWIZZLE_128B.  Each column's RS rows are one contiguous
// 16H*8-byte run (>= 256 B: what keeps HBM near 6.9 TB/s; 128-byte pieces cap it at
// ~4.6 TB/s) and each box moves w in {128, 64, 32, 16, 8} columns (TMA costs ~450 cycles per
// box per SM, so spans are cut greedily into the widest boxes; profiles/r01_tma_*.log).
// In shared memory, 128-byte line L = H*c + h holds rows 16h..16h+15 of tile column c, its
// 16-byte chunk j stored at chunk j ^ (L & 7).  Both fragment shapes are conflict-free:
//   Gram (column-major, lane = (col ii, k kk)): two LDS.128 per 4 rows; odd-ii lanes fetch
//     the two chunks in swapped order (then swap back) so a quarter-warp hits 8 chunks;
//   update (row-major, lane = (row ii, col kk)): one LDS.64; with H = 2 the four columns of
//     a k-step sit on lines with distinct (L & 7), so 16 lanes hit 16 distinct slots.
//
// This header holds the kernel template and its dispatch templates: gram.cu instantiates the
// plain instances (CT = false), gram_ct.cu the compensated-tile ones (CT = true: output
// tiles >= p.comp_t0 fold every 4-row k-step into a double-double; BCGSI+1S).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace bgs {
namespace tiled {

// 8 warps = 2 per scheduler (the 64K register file allows 255 registers per thread).
// Warp 7 lane 0 issues the TMA.  K1: warps 0-6 run the Gram, warp 7 only streams.
// K12: warps 0-6 split the update k-steps while warp 7 refills the freed slot (a TMA box
// keeps the issuing thread ~1 cycle per 128-byte line), then all 8 warps run the
// epilogue and the Gram.
constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * kConsumerWarps;
constexpr int kUpdWarps = 7;
constexpr int kProducerWarp = 7;
template <bool UPD>
struct Roles {
  static constexpr int WG = UPD ? 8 : 7;  // Gram warps
};

// Named barrier over the warps that run the stage loop (all 8 in K12, 0-6 in K1).
template <int NWARPS>
BGS_DEV void bar_warps() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NWARPS) : "memory");
}

constexpr int SMAX_E = 8;  // fused epilogue supports s <= 8 (K12 is instantiated for s <= 4)

template <int H, int NT, int MTW, bool COMP, bool UPD, int KW, bool CT>
__global__ void __launch_bounds__(kThreads, 1) tile_kernel(const __grid_constant__ TileParams p) {
  if (p.status && status_bad(p.status)) return;
  constexpr int RS = 16 * H;
  constexpr int W = kConsumerWarps;   // epilogue / barrier width
  constexpr int WG = Roles<UPD>::WG;  // Gram m-tile stride
  constexpr int WU = kUpdWarps;       // update k-step stride
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const int stage_bytes = p.units * 8 * RS * 8;
  double* red = reinterpret_cast<double*>(smem + (size_t)S * stage_bytes);  // [W][8][RS+4]
  uint64_t* full = reinterpret_cast<uint64_t*>(
      reinterpret_cast<unsigned char*>(red) + (UPD ? (size_t)W * 8 * (RS + 4) * sizeof(double) : 0));
  uint64_t* empty = full + S;
  __shared__ double ep_ta[SMAX_E * SMAX_E], ep_tb[SMAX_E * SMAX_E], ep_s2[SMAX_E * SMAX_E];
  __shared__ double ep_tai[SMAX_E * SMAX_E], ep_tbi[SMAX_E * SMAX_E], ep_w[SMAX_E * SMAX_E];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long T = p.total_stages;
  const long st0 = (long)blockIdx.x * T / gridDim.x;
  const long st1 = (long)(blockIdx.x + 1) * T / gridDim.x;
  const int nst = (int)(st1 - st0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WG);  // every warp that consumes the slot releases it
    }
    fence_mbar_init();
  }
  if (UPD) {
    // Epilogue factors, once per CTA: TA^{-1}, TB^{-1} (upper, by back-substitution on the
    // identity, column j by thread j) and W = S2 TB^{-1}; the per-row epilogue then needs
    // only short dot products instead of a serial substitution per row.
    const int s = p.s;
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
      const int i = e % s, j = e / s;
      ep_ta[i + j * SMAX_E] = p.TA ? p.TA[i + j * s] : (i == j ? 1.0 : 0.0);
      ep_tb[i + j * SMAX_E] = p.TB ? p.TB[i + j * s] : (i == j ? 1.0 : 0.0);
      ep_s2[i + j * SMAX_E] = (p.upd_a && p.upd_b) ? p.CB[p.kp + i + (size_t)j * p.ldcb] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 2 * s) {
      const bool isb = threadIdx.x >= s;
      const int j = isb ? threadIdx.x - s : threadIdx.x;
      const double* T = isb ? ep_tb : ep_ta;
      double* Ti = isb ? ep_tbi : ep_tai;
      for (int i = s - 1; i >= 0; --i) {  // column j of T^{-1}: T y = e_j
        double acc = (i == j) ? 1.0 : 0.0;
        for (int l = i + 1; l < s; ++l) acc -= T[i + l * SMAX_E] * Ti[l + j * SMAX_E];
        Ti[i + j * SMAX_E] = acc / T[i + i * SMAX_E];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
      const int m = e % s, j = e / s;
      double acc = 0.0;
      for (int l = 0; l < s; ++l) acc += ep_s2[m + l * SMAX_E] * ep_tbi[l + j * SMAX_E];
      ep_w[m + j * SMAX_E] = acc;
    }
  }
  __syncthreads();

  // ---------------- TMA issue (thread 0): greedy widest boxes per span ----------------
  auto issue_stage = [&](int it) {
    const int slot = it % S;
    mbar_arrive_expect_tx(&full[slot], (uint32_t)stage_bytes);
    unsigned char* dst = smem + (size_t)slot * stage_bytes;
    const int rb = (int)((st0 + it) * H);  // first 16-row block of this stage
    int u = 0;                              // 8-column units issued so far (tile column = 8u)
    for (int sp = 0; sp < 2; ++sp) {
      int left = p.units_span[sp], c = p.col0[sp];
      while (left > 0) {
        int wi;  // width index: 0:128, 1:64, 2:32, 3:16, 4:8 columns
        const CUtensorMap* mp;
        if (sp == 0) {
          wi = left >= 16 ? 0 : left >= 8 ? 1 : left >= 4 ? 2 : left >= 2 ? 3 : 4;
          mp = &p.map0[wi];
        } else {
          wi = left >= 2 ? 3 : 4;
          mp = &p.map1[wi - 3];
        }
        const int wu = 16 >> wi;
        tma_load_3d(dst + (size_t)u * 8 * RS * 8, mp, &full[slot], 0, rb, c);
        u += wu;
        c += 8 * wu;
        left -= wu;
      }
    }
  };
  const bool producer = threadIdx.x == 32 * kProducerWarp;
  if (producer) {
    for (int i = 0; i < 5; ++i) prefetch_tmap(&p.map0[i]);
    for (int i = 0; i < 2; ++i) prefetch_tmap(&p.map1[i]);
    for (int it = 0; it < S && it < nst; ++it) issue_stage(it);
  }
  if (!UPD && warp == kProducerWarp) {
    // K1: dedicated producer warp
    if (producer) {
      for (int it = 0; it + S < nst; ++it) {
        mbar_wait(&empty[it % S], (it / S) & 1);
        issue_stage(it + S);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int cw = warp;
  const int kk = lane & 3, ii = lane >> 2, odd = ii & 1;
  (void)lane;
  int cnt = 0;
  for (int t = cw; t < p.mt_out; t += WG) ++cnt;
  int bcol[NT];
  bool bval[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int col = p.rcol[nt * 8 + ii];
    bval[nt] = col >= 0;
    bcol[nt] = col >= 0 ? col : 0;
  }

  int acol[MTW];
#pragma unroll
  for (int j = 0; j < MTW; ++j) acol[j] = 8 * (j < cnt ? cw + WG * j : 0) + ii;
  // (CT) the compensated tile of this warp (tiles >= p.comp_t0; at most one per warp: the
  // runtime keeps the range <= WG tiles): each 4-row k-step goes straight into (chi, clo)
  int cj = -1, acolc = ii;
  if (CT) {
#pragma unroll
    for (int j = 0; j < MTW; ++j)
      if (j < cnt && cw + WG * j >= p.comp_t0 && cj < 0) {
        cj = j;
        acolc = 8 * (cw + WG * j) + ii;
      }
  }
  double chi[CT ? NT : 1][2], clo[CT ? NT : 1][2];
#pragma unroll
  for (int nt = 0; nt < (CT ? NT : 1); ++nt) chi[nt][0] = chi[nt][1] = clo[nt][0] = clo[nt][1] = 0.0;

  double acc[MTW][NT][2];
  double hi[COMP ? MTW : 1][NT][2];
  double lo[COMP ? MTW : 1][NT][2];
#pragma unroll
  for (int j = 0; j < MTW; ++j)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      acc[j][nt][0] = acc[j][nt][1] = 0.0;
      if (COMP) hi[j][nt][0] = hi[j][nt][1] = lo[j][nt][0] = lo[j][nt][1] = 0.0;
    }

  // Update coefficients as DMMA B fragments held in registers for the whole kernel:
  // this warp owns k-steps g = cw + W*j (columns 4g..4g+3 of the prefix); lane holds
  // C[4g + kk][n = ii] where C = [CA | CB] (kp x 2s, zero padded).
  double bco[UPD ? KW : 1];
  const int s = p.s;
  if (UPD) {
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const int c = cw < WU ? 4 * (cw + WU * j) + kk : p.kp;  // warp 7: no update k-steps
      double v = 0.0;
      if (c < p.kp) {
        if (ii < s && p.upd_a) v = p.CA[c + (size_t)ii * p.ldca];
        else if (ii >= s && ii < 2 * s && p.upd_b) v = p.CB[c + (size_t)(ii - s) * p.ldcb];
      }
      bco[j] = v;
    }
  }

  auto flush = [&]() {
    if (COMP) {
#pragma unroll
      for (int j = 0; j < MTW; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double sm, err;
            two_sum(hi[j][nt][e], acc[j][nt][e], sm, err);
            hi[j][nt][e] = sm;
            lo[j][nt][e] += err;
            acc[j][nt][e] = 0.0;
          }
    }
  };

  const uint32_t sbase = smem_u32(smem);
  int since = 0;
  const bool prof = p.phase && threadIdx.x == 0;
  // wait, update, reduce+bar, epilogue+bar, gram, total, fence+arrive, refill issue, flush
  unsigned long long ph[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long ph_prod = 0;                   // thread 0 waiting to refill a slot
  const unsigned long long t_begin = prof ? clock64() : 0;
  for (int it = 0; it < nst; ++it) {
    const int slot = it % S;
    unsigned long long t0 = prof ? clock64() : 0;
    if (p.dbg & 64) mbar_wait_dbg(&full[slot], (it / S) & 1, 1, it);
    else mbar_wait(&full[slot], (it / S) & 1);
    unsigned long long t1 = prof ? clock64() : 0;
    if (prof) ph[0] += t1 - t0;
    const uint32_t base = sbase + (uint32_t)(slot * stage_bytes);
    const long row0 = (st0 + it) * RS;
    const int vrows = (int)((p.n_rows - row0) < RS ? (p.n_rows - row0) : RS);
    if (vrows < RS) {
      // rows past the shard end inside the last 16-row block are not TMA zero-filled;
      // (only the WG warps of the stage loop run this: K1's producer warp has left)
      const int ncol = p.units * 8;
      for (int e = threadIdx.x; e < ncol * (RS - vrows); e += 32 * WG) {
        const int c = e / (RS - vrows), r = vrows + e % (RS - vrows);
        sts64(base + elem_off<H>(c, r), 0.0);
      }
      bar_warps<WG>();
    }

    if (UPD) {
      // warp 7 refills the slot released at the end of the previous stage while warps
      // 0-6 run the update MMAs (stage it-1+S goes into slot (it-1)%S)
      if (producer && it >= 1 && it - 1 + S < nst) {
        const unsigned long long tw = p.phase ? clock64() : 0;
        if (p.dbg & 64) mbar_wait_dbg(&empty[(it - 1) % S], ((it - 1) / S) & 1, 2, it);
        else mbar_wait(&empty[(it - 1) % S], ((it - 1) / S) & 1);
        if (p.phase) ph_prod += clock64() - tw;
        issue_stage(it - 1 + S);
      }
      // reconverge warp 7 before anything reaches a bar.sync (an aligned barrier)
      if (warp == kProducerWarp) __syncwarp();
      // ---- update MMAs: D[row][n] = sum_c tile[row][c] * C[c][n], k-split over warps ----
      constexpr int MT_U = RS / 8;
      // two accumulator sets (even / odd k-steps) -> 2*MT_U independent DMMA chains;
      // k-steps past kp are predicated to zero instead of branched around.
      double d[2][MT_U][2];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int mt = 0; mt < MT_U; ++mt) d[e][mt][0] = d[e][mt][1] = 0.0;
      if (!(p.dbg & 4) && cw < WU) {
#pragma unroll
        for (int j = 0; j < KW; ++j) {
          const int c = 4 * (cw + WU * j) + kk;
          const bool in = c < p.kp && cw < WU;
          double av[MT_U];
#pragma unroll
          for (int mt = 0; mt < MT_U; ++mt) {
            const double v = lds64(base + elem_off<H>(in ? c : 0, 8 * mt + ii));
            av[mt] = in ? v : 0.0;
          }
#pragma unroll
          for (int mt = 0; mt < MT_U; ++mt) dmma(d[j & 1][mt][0], d[j & 1][mt][1], av[mt], bco[j]);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT_U; ++mt) {
        d[0][mt][0] += d[1][mt][0];
        d[0][mt][1] += d[1][mt][1];
      }
      if (prof) { const unsigned long long t = clock64(); ph[1] += t - t1; t1 = t; }
      // partial sums, transposed with a padded row stride: red[warp][n][RL], RL = RS + 4
      constexpr int RL = RS + 4;
      if (cw < WU) {
#pragma unroll
        for (int mt = 0; mt < MT_U; ++mt) {
          double* rr = red + ((size_t)cw * 8 + 2 * kk) * RL + 8 * mt + ii;
          rr[0] = d[0][mt][0];
          rr[RL] = d[0][mt][1];
        }
      }
      bar_warps<WG>();
      if (prof) { const unsigned long long t = clock64(); ph[2] += t - t1; t1 = t; }
      // ---- epilogue: a quad of lanes per row (lane j of the quad owns column j) ----
      // Sum the W warp partials in order, then back-substitute across the quad with
      // shuffles: A = (srcA - Qp CA) TA^{-1}, B = (srcB - Qp CB - A S2) TB^{-1}.
      const uint32_t red_s = smem_u32(red);
      for (int e0 = 0; e0 < 4 * RS && !(p.dbg & 16); e0 += 32 * W) {
        const int e = e0 + (int)threadIdx.x;
        if (e >= 4 * RS) break;  // whole warps (4 RS and 32 W are multiples of 32)
        const int r = e >> 2, j = e & 3;
        const bool jv = j < s;
        const int quad = (int)(threadIdx.x & 31) & ~3;
        // warp partials, two independent halves per sum
        double pa[2] = {0.0, 0.0}, pb[2] = {0.0, 0.0};
#pragma unroll
        for (int w = 0; w < WU; ++w) {
          pa[w & 1] += lds64(red_s + (uint32_t)((((size_t)w * 8 + j) * RL + r) * 8));
          pb[w & 1] += lds64(red_s + (uint32_t)((((size_t)w * 8 + (jv ? s + j : j)) * RL + r) * 8));
        }
        const double aA = pa[0] + pa[1], aB = pb[0] + pb[1];
        const bool live = r < vrows;
        const long grow = row0 + r;
        const uint32_t offA = base + elem_off<H>(p.colA + (jv ? j : 0), r);
        const uint32_t offB = base + elem_off<H>(p.colB + (jv ? j : 0), r);
        const double uA = p.upd_a ? lds64(offA) : 0.0;
        const double uB = p.upd_b ? lds64(offB) : 0.0;
        // A_j = sum_{l<=j} (srcA - acc)_l TA^{-1}[l][j]
        double dA = jv ? uA - aA : 0.0, q[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) q[l] = __shfl_sync(0xffffffffu, dA, quad | l);
        double x = 0.0;
        if (p.upd_a) {
#pragma unroll
          for (int l = 0; l < 4; ++l)
            if (l <= j && l < s) x += q[l] * ep_tai[l + j * SMAX_E];
#pragma unroll
          for (int l = 0; l < 4; ++l) q[l] = __shfl_sync(0xffffffffu, x, quad | l);
          if (jv) {
            sts64(offA, x);
            if (live && !(p.dbg & 2)) p.dstA[grow + (size_t)j * p.lddA] = x;
          }
        } else {
#pragma unroll
          for (int l = 0; l < 4; ++l) q[l] = 0.0;
        }
        if (p.upd_b) {
          // B_j = sum_{l<=j} (srcB - acc)_l TB^{-1}[l][j] - sum_m A_m (S2 TB^{-1})[m][j]
          const double dB = jv ? uB - aB : 0.0;
          double y = 0.0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const double dl = __shfl_sync(0xffffffffu, dB, quad | l);
            if (l <= j && l < s) y += dl * ep_tbi[l + j * SMAX_E];
            if (l < s && jv) y -= q[l] * ep_w[l + j * SMAX_E];
          }
          if (jv) {
            sts64(offB, y);
            if (live && !(p.dbg & 2)) p.dstB[grow + (size_t)j * p.lddB] = y;
          }
        }
      }
      bar_warps<WG>();
      if (prof) { const unsigned long long t = clock64(); ph[3] += t - t1; t1 = t; }
    }

    // ---- Gram on the (updated) tile ----
    // Every warp runs MTW m-tiles (the tail warps clamp to a valid tile and drop the
    // result), loads all A fragments of a 16-row half first, then issues the DMMAs
    // k-step-major so consecutive DMMAs are independent (MTW*NT chains in flight).
    if (!(p.dbg & 8)) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        double b[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          frag4<H>(base, bcol[nt], h, kk, odd, b[nt]);
          if (!bval[nt]) b[nt][0] = b[nt][1] = b[nt][2] = b[nt][3] = 0.0;
        }
        double a[MTW][4];
#pragma unroll
        for (int j = 0; j < MTW; ++j) frag4<H>(base, acol[j], h, kk, odd, a[j]);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
          for (int j = 0; j < MTW; ++j)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[j][nt][0], acc[j][nt][1], a[j][q4], b[nt][q4]);
        // (CT) this warp's compensated tile again, each 4-row k-step straight into
        // (chi, clo): outside the loop above, which stays branch-free (a flag tested at
        // every DMMA split it into basic blocks: BCGSI+1S at s = 8 / 16 57 / 60 ms against
        // 40 / 39 for P-1S); the plain sums of that tile are dropped at the end
        if (CT && cj >= 0) {
          double ac[4];
          frag4<H>(base, acolc, h, kk, odd, ac);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              double c0 = 0.0, c1 = 0.0, sm, err;
              dmma(c0, c1, ac[q4], b[nt][q4]);
              two_sum(chi[CT ? nt : 0][0], c0, sm, err);
              chi[CT ? nt : 0][0] = sm;
              clo[CT ? nt : 0][0] += err;
              two_sum(chi[CT ? nt : 0][1], c1, sm, err);
              chi[CT ? nt : 0][1] = sm;
              clo[CT ? nt : 0][1] += err;
            }
        }
      }
    }
    if (prof) { const unsigned long long t = clock64(); ph[4] += t - t1; t1 = t; }
    if (UPD && !(p.dbg & 1)) fence_proxy_async();  // generic smem writes before TMA reuses the slot
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (prof) { const unsigned long long t = clock64(); ph[6] += t - t1; t1 = t; }

    if (prof) { const unsigned long long t = clock64(); ph[7] += t - t1; t1 = t; }
    if (++since == GRAM_FLUSH) {
      flush();
      since = 0;
    }
    if (prof) ph[8] += clock64() - t1;
  }
  flush();
  if (prof) {
    ph[5] = clock64() - t_begin;
    for (int i = 0; i < 9; ++i) atomicAdd(&p.phase[blockIdx.x * 16 + i], ph[i]);
    atomicAdd(&p.phase[blockIdx.x * 16 + 9], (unsigned long long)nst);
    atomicAdd(&p.phase[blockIdx.x * 16 + 10], ph_prod);
  }

  // ---------------- per-CTA partial (hi, lo) ----------------
  const int N8 = 8 * NT;
  double2* part = reinterpret_cast<double2*>(p.partial) + (size_t)blockIdx.x * p.mt_out * 8 * N8;
#pragma unroll
  for (int j = 0; j < MTW; ++j) {
    if (j < cnt) {
      const int t = cw + WG * j;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = nt * 8 + 2 * kk + e;
          double hv = COMP ? hi[j][nt][e] : acc[j][nt][e];
          double lv = COMP ? lo[j][nt][e] : 0.0;
          if (CT && j == cj) {
            hv = chi[CT ? nt : 0][e];
            lv = clo[CT ? nt : 0][e];
          }
          part[((size_t)t * 8 + ii) * N8 + n] = make_double2(hv, lv);
        }
    }
  }
}

template <int H, int NT, int MTW, bool COMP, bool UPD, int KW, bool CT>
static cudaError_t launch_t(const TileParams& p, int grid, cudaStream_t st) {
  auto k = tile_kernel<H, NT, MTW, COMP, UPD, KW, CT>;
  const size_t smem = tile_smem_bytes(H, p.stages, p.units, UPD);
  cudaError_t e = ensure_smem(k, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

// The tile loops run exactly MTW m-tiles and KW k-steps per warp (predicated, no
// branches), so instantiations are dense where the block steps live.
template <int H, int NT, bool CT>
static cudaError_t dispatch_gram(const TileParams& p, int mtw, int grid, cudaStream_t st) {
  constexpr bool CO = NT <= 2;  // double-double folding when the registers allow it
  switch (mtw) {
    case 1: return launch_t<H, NT, 1, true, false, 1, CT>(p, grid, st);
    case 2: return launch_t<H, NT, 2, true, false, 1, CT>(p, grid, st);
    case 3: return launch_t<H, NT, 3, true, false, 1, CT>(p, grid, st);
    case 4: return launch_t<H, NT, 4, CO, false, 1, CT>(p, grid, st);
    case 5: return launch_t<H, NT, 5, CO, false, 1, CT>(p, grid, st);
    case 6: return launch_t<H, NT, 6, NT == 1, false, 1, CT>(p, grid, st);
    case 7: return launch_t<H, NT, 7, NT == 1, false, 1, CT>(p, grid, st);
    case 8: return launch_t<H, NT, 8, NT == 1, false, 1, CT>(p, grid, st);
    default: break;
  }
  if (mtw <= 15) return launch_t<H, NT, 15, false, false, 1, CT>(p, grid, st);
  return cudaErrorInvalidValue;
}

template <int H, int MTW, bool CT>
static cudaError_t fused_kw(const TileParams& p, int kw, int grid, cudaStream_t st) {
  constexpr int K1 = 2 * MTW - 1 > 0 ? 2 * MTW - 1 : 1, K2 = 2 * MTW;
  if (kw <= K1) return launch_t<H, 1, MTW, true, true, K1, CT>(p, grid, st);
  if (kw <= K2) return launch_t<H, 1, MTW, true, true, K2, CT>(p, grid, st);
  return cudaErrorInvalidValue;
}

template <int H, bool CT>
static cudaError_t dispatch_fused(const TileParams& p, int mtw, int kw, int grid, cudaStream_t st) {
  // k-steps per warp track m-tiles per warp (kw ~ 2 mtw along a sweep); widen the
  // Gram side when the update side needs more.
  if (kw > 2 * mtw) mtw = (kw + 1) / 2;
  switch (mtw) {
    case 1: return fused_kw<H, 1, CT>(p, kw, grid, st);
    case 2: return fused_kw<H, 2, CT>(p, kw, grid, st);
    case 3: return fused_kw<H, 3, CT>(p, kw, grid, st);
    case 4: return fused_kw<H, 4, CT>(p, kw, grid, st);
    case 5: return fused_kw<H, 5, CT>(p, kw, grid, st);
    case 6: return fused_kw<H, 6, CT>(p, kw, grid, st);
    case 7: return fused_kw<H, 7, CT>(p, kw, grid, st);
    case 8: return fused_kw<H, 8, CT>(p, kw, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

// mtw / kw / nt dispatch shared by gram.cu and gram_ct.cu (p.nt, p.total_stages set)
template <bool CT>
static cudaError_t tile_dispatch(const TileParams& p, bool upd, int grid, cudaStream_t st) {
  const int WGv = upd ? Roles<true>::WG : Roles<false>::WG;
  const int mtw = (p.mt_out + WGv - 1) / WGv;
  if (upd) {
    if (p.nt != 1 || p.s > 4) return cudaErrorInvalidValue;
    const int kw = ((p.kp + 3) / 4 + kUpdWarps - 1) / kUpdWarps;
    return p.H == 2 ? dispatch_fused<2, CT>(p, mtw, kw, grid, st)
                    : dispatch_fused<4, CT>(p, mtw, kw, grid, st);
  }
  switch (p.nt) {
    case 1:
      return p.H == 2 ? dispatch_gram<2, 1, CT>(p, mtw, grid, st) : dispatch_gram<4, 1, CT>(p, mtw, grid, st);
    case 2:
      return p.H == 2 ? dispatch_gram<2, 2, CT>(p, mtw, grid, st) : dispatch_gram<4, 2, CT>(p, mtw, grid, st);
    default:
      return p.H == 2 ? dispatch_gram<2, 4, CT>(p, mtw, grid, st) : dispatch_gram<4, 4, CT>(p, mtw, grid, st);
  }
}

}  // namespace tiled
}  // namespace bgs
