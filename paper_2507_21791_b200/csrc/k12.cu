// k12.cu — K12c: the block update of step k fused in front of the Gram of step k+1,
// split over a CTA pair (thread-block cluster of two) with ping-pong consumer groups.
//
// Same algebra and call sites as gram.cu's K12 (onesync_impl bcgs.cpp:329-331, 346-359;
// pipi_impl bcgs.cpp:196-214):
//   A = (srcA - Qp CA) TA^{-1},  B = (srcB - Qp CB - A S2) TB^{-1},  G = [tile]^T [span 1]
// Why a pair: late in a sweep one 32-row stage of the tile is 400+ columns (100+ KB), so
// a single SM holds two stages and computes one while the other loads — the update, its
// cross-warp reduction, the epilogue and the Gram then run back to back with nothing to
// hide their latencies.  Splitting the prefix columns over two SMs halves the stage, so
// each SM keeps 4 stages: two being computed by two consumer groups (4 warps each,
// alternate stages, one warp per scheduler each) and two in flight.
//
//   rank r of the pair loads: its own span-0 units (the prefix half it contracts), the
//   A-block units (rank 0 only; rank 1 owns them), and all of span 1 (the B block and
//   the right-hand columns).  Update: warp w of a group owns rows 8w..8w+7 of the stage
//   and runs all of this rank's k-steps (coefficients in registers as DMMA B fragments),
//   giving a partial D (8 rows x [CA | CB]) per warp.  The partial goes to the same warp
//   of the peer through distributed shared memory (st.async + mbarrier complete_tx);
//   both ranks form D0 + D1 (same operands, same order -> identical bits), run the
//   epilogue in registers (quad shuffles, explicit inverses), write A / B back into their
//   stage, and then contract their own output tiles against span 1.
//
// Output tiles: rank 0 = own span-0 units + the span-1 left units, rank 1 = its own
// span-0 units (which include the A block).  Partials: one slot per (cluster, group),
// every global tile written by exactly one rank -> gram_reduce sums 2 x clusters slots.
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {

constexpr int kGroupWarps = 4;
constexpr int kGroups = 2;
constexpr int kConsWarps = kGroups * kGroupWarps;  // warps 0-7: two consumer groups
constexpr int kProdWarp = kConsWarps;              // warp 8: TMA producer (warps 8-11: its warpgroup)
constexpr int kThreads = 32 * (kConsWarps + 4);
// setmaxnreg: the producer warpgroup gives registers to the two consumer warpgroups
// (4 x 32 x (2 x 232 + 40) = 64512 <= 65536)
constexpr int kProdRegs = 40, kConsRegs = 232;
constexpr int RS = 32;                    // rows per stage (H = 2: 256-byte column runs)
constexpr int kUnitBytes = 8 * RS * 8;    // one 8-column unit of a stage
constexpr int kXchgBytes = kGroups * 2 * kGroupWarps * 32 * 16;  // [group][parity][warp][lane]
constexpr int kRedBytes = kGroups * kGroupWarps * 4 * 32 * 16;  // [group][warp][m-tile][lane]
constexpr int kStaticSmem = 6 * 16 * 8;   // the epilogue factor arrays below
constexpr int kSmemOptin = 232448;        // per-block opt-in maximum (227 KB)
constexpr int kMaxStages = 8;

}  // namespace

size_t k12_smem_bytes(int stages, int slot_units) {
  return 1024 + (size_t)stages * slot_units * kUnitBytes + kRedBytes + kXchgBytes +
         (size_t)(2 * stages + 4) * sizeof(uint64_t);
}

template <int KW, int MTW>
__global__ void __launch_bounds__(kThreads, 1) k12_kernel(const __grid_constant__ SplitParams p) {
  if (p.status && status_bad(p.status)) return;  // both ranks read the same word
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const int slot_bytes = p.slot_units * kUnitBytes;
  unsigned char* redbuf = smem + (size_t)S * slot_bytes;  // [group][warp][m-tile][lane]
  unsigned char* xbuf = redbuf + kRedBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + kXchgBytes);
  uint64_t* empty = full + S;
  uint64_t* xfull = empty + S;  // [group][parity]
  __shared__ double ep_t[2][16], ep_s2[16], ep_ai[16], ep_bi[16], ep_w[16];

  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int own_u0 = p.own_u0[rank], own_n = p.own_n[rank];
  const int ext_u0 = p.ext_u0[rank], ext_n = p.ext_n[rank];
  const int nloc = own_n + ext_n + p.U1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long T = p.total_stages;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const long st0 = (long)cl * T / ncl;
  const int nst = (int)((long)(cl + 1) * T / ncl - st0);
  const int s = p.s;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kGroupWarps);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&xfull[i], 1);
    fence_mbar_init();
  }
  // Epilogue factors padded to 4x4 with identity: TA^{-1}, TB^{-1}, W = S2 TB^{-1}.
  if (threadIdx.x < 16) {
    const int i = threadIdx.x & 3, j = threadIdx.x >> 2;
    const bool in = i < s && j < s;
    const double id = i == j ? 1.0 : 0.0;
    ep_t[0][threadIdx.x] = (in && p.TA) ? p.TA[i + j * s] : id;
    ep_t[1][threadIdx.x] = (in && p.TB) ? p.TB[i + j * s] : id;
    ep_s2[threadIdx.x] = (in && p.upd_a && p.upd_b) ? p.CB[p.kp + i + (size_t)j * p.ldcb] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const int which = threadIdx.x >> 2, j = threadIdx.x & 3;
    const double* Tm = ep_t[which];
    double* Ti = which ? ep_bi : ep_ai;
    for (int i = 3; i >= 0; --i) {  // column j of T^{-1}: T y = e_j
      double acc = (i == j) ? 1.0 : 0.0;
      for (int l = i + 1; l < 4; ++l) acc -= Tm[i + 4 * l] * Ti[l + 4 * j];
      Ti[i + 4 * j] = acc / Tm[i + 4 * i];
    }
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const int m = threadIdx.x & 3, j = threadIdx.x >> 2;
    double acc = 0.0;
    for (int l = 0; l < 4; ++l) acc += ep_s2[m + 4 * l] * ep_bi[l + 4 * j];
    ep_w[m + 4 * j] = acc;
  }
  __syncthreads();
  cluster_sync_all();  // the peer's mbarriers exist before any st.async can reach them

  if (warp >= kProdWarp) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsRegs));
  }
  if (warp >= kProdWarp) {
    // ---------------- producer: one thread streams the stages ----------------
    if (warp == kProdWarp && lane == 0) {
      for (int i = 0; i < 5; ++i) prefetch_tmap(&p.map0[i]);
      for (int i = 0; i < 2; ++i) prefetch_tmap(&p.map1[i]);
      const uint32_t bytes = (uint32_t)nloc * kUnitBytes;
      for (int it = 0; it < nst; ++it) {
        const int slot = it % S;
        if (it >= S) mbar_wait(&empty[slot], ((it / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], bytes);
        unsigned char* dst = smem + (size_t)slot * slot_bytes;
        const int rb = (int)((st0 + it) * 2);  // first 16-row block of the stage
        int u = 0;
        for (int seg = 0; seg < 3; ++seg) {  // own span-0 units, extra units, span 1
          int left = seg == 0 ? own_n : seg == 1 ? ext_n : p.U1;
          int c = seg == 0 ? p.col0[0] + 8 * own_u0 : seg == 1 ? p.col0[0] + 8 * ext_u0 : p.col0[1];
          while (left > 0) {
            int wi;
            const CUtensorMap* mp;
            if (seg < 2) {
              wi = left >= 16 ? 0 : left >= 8 ? 1 : left >= 4 ? 2 : left >= 2 ? 3 : 4;
              mp = &p.map0[wi];
            } else {
              wi = left >= 2 ? 3 : 4;
              mp = &p.map1[wi - 3];
            }
            const int wu = 16 >> wi;
            tma_load_3d(dst + (size_t)u * kUnitBytes, mp, &full[slot], 0, rb, c);
            u += wu;
            c += 8 * wu;
            left -= wu;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- consumers: group g takes stages g, g+2, g+4, ... ----------------
    const int g = warp / kGroupWarps, w = warp % kGroupWarps;
    const int gtid = threadIdx.x - 32 * kGroupWarps * g;
    const int ii = lane >> 2, kk = lane & 3, odd = ii & 1;
    const int gbar = 1 + g;
    // This rank's k-steps are prefix columns [8 own_u0, pc1) (local columns from 0); warp w
    // takes k-steps j = w + 4t.  Lane (ii, kk) holds C[4j + kk][n = ii] of [CA | CB]
    // (CA in n = 0..3, CB in n = 4..7, zero padded) as the DMMA B fragment.
    const int pc1 = min(8 * (own_u0 + own_n), p.kp);
    const int kcols = max(0, pc1 - 8 * own_u0);
    const int ksteps = kcols / 4;  // whole k-steps (k12_plan)
    double bco[KW];
#pragma unroll
    for (int t = 0; t < KW; ++t) {
      const int lc = 4 * (w + kGroupWarps * t) + kk, c = 8 * own_u0 + lc;
      double v = 0.0;
      if (lc < kcols) {
        if (ii < 4) {
          if (ii < s && p.upd_a) v = p.CA[c + (size_t)ii * p.ldca];
        } else if (ii - 4 < s && p.upd_b) {
          v = p.CB[c + (size_t)(ii - 4) * p.ldcb];
        }
      }
      bco[t] = v;
    }
    // Update A fragments: m-tile q is rows {4i + q}, so lane (ii, kk) needs rows
    // 4ii..4ii+3 of tile column 4j + kk: two LDS.128 (frag4 with h = ii/4, kk' = ii%4).
    // Column 4j + kk sits on line 8j + 2kk + ii/4, i.e. at 1024 j past k-step 0.
    uint32_t uoff0, uoff1;
    {
      const int line = 2 * kk + (ii >> 2);
      const int o = (ii & 3) & 1;
      uoff0 = (uint32_t)(line * 128 + ((((ii & 3) * 2 + o) ^ (line & 7)) << 4));
      uoff1 = (uint32_t)(line * 128 + ((((ii & 3) * 2 + 1 - o) ^ (line & 7)) << 4));
    }
    const bool uswap = ((ii & 3) & 1) != 0;
    // local columns of the A block, the B block (= span-1 column 0) and the right operand
    const bool a_own = p.kp >= 8 * own_u0 && p.kp < 8 * (own_u0 + own_n);
    const int colA = a_own ? p.kp - 8 * own_u0 : 8 * own_n + p.kp - 8 * ext_u0;
    const int colB = 8 * (own_n + ext_n);
    const int rc = ii < p.N ? p.rcol1[ii] : -1;
    const bool bval = rc >= 0;
    const int bcol = colB + (bval ? rc : 0);
    // output tiles of this rank: own units, then (rank 0) the span-1 left units
    const int mt_loc = own_n + (rank == 0 ? p.s1_left : 0);
    // epilogue row of this lane: warp w handles rows 8w..8w+7 (coalesced stores)
    const int qsel = lane >> 3, isel = 2 * w + ((lane >> 2) & 1);
    const int erow = 4 * isel + qsel;
    const int quad = lane & ~3;

    double hi[MTW][2], lo[MTW][2];
#pragma unroll
    for (int j = 0; j < MTW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) hi[j][e] = lo[j][e] = 0.0;

    const uint32_t sbase = smem_u32(smem);
    const uint32_t red_w = smem_u32(redbuf) + (uint32_t)(((g * kGroupWarps + w) * 4 * 32 + lane) * 16);
    const uint32_t red_r = smem_u32(redbuf) +
                           (uint32_t)(((g * kGroupWarps * 4 + qsel) * 32 + 4 * isel + kk) * 16);
    const uint32_t xb_local = smem_u32(xbuf);
    const uint32_t xfull_local = smem_u32(xfull);
    const bool prof = p.phase && gtid == 0;
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};  // full wait, update, exchange, epilogue, gram
    const unsigned long long t_begin = prof ? clock64() : 0;
    for (int j = 0;; ++j) {
      const int it = g + kGroups * j;
      if (it >= nst) break;
      const int slot = it % S;
      unsigned long long t0 = prof ? clock64() : 0;
      mbar_wait(&full[slot], (it / S) & 1);
      unsigned long long t1 = prof ? clock64() : 0;
      if (prof) ph[0] += t1 - t0;
      const uint32_t base = sbase + (uint32_t)(slot * slot_bytes);
      const long row0 = (st0 + it) * RS;
      const int vrows = (int)((p.n_rows - row0) < RS ? (p.n_rows - row0) : RS);
      if (vrows < RS) {
        // rows past the shard end inside its last 16-row block are not TMA zero-filled
        const int ncol = nloc * 8, nr = RS - vrows;
        for (int e = gtid; e < ncol * nr; e += 32 * kGroupWarps)
          sts64(base + elem_off<2>(e / nr, vrows + e % nr), 0.0);
        bar_named(gbar, 32 * kGroupWarps);
      }

      // ---- update partial: all 32 rows (4 m-tiles = 4 DMMA chains), k-steps w + 4t ----
      double d[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q][0] = d[q][1] = 0.0;
#pragma unroll
      for (int t = 0; t < KW; ++t) {
        const int jk = w + kGroupWarps * t;
        if (jk < ksteps) {
          const uint32_t a = base + 1024u * (uint32_t)jk;
          const double2 x0 = lds128(a + uoff0), x1 = lds128(a + uoff1);
          const double v0 = uswap ? x1.x : x0.x, v1 = uswap ? x1.y : x0.y;
          const double v2 = uswap ? x0.x : x1.x, v3 = uswap ? x0.y : x1.y;
          dmma(d[0][0], d[0][1], v0, bco[t]);
          dmma(d[1][0], d[1][1], v1, bco[t]);
          dmma(d[2][0], d[2][1], v2, bco[t]);
          dmma(d[3][0], d[3][1], v3, bco[t]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) sts128(red_w + (uint32_t)(q * 32 * 16), d[q][0], d[q][1]);
      bar_named(gbar, 32 * kGroupWarps);
      if (prof) { const unsigned long long t = clock64(); ph[1] += t - t1; t1 = t; }

      // ---- sum the 4 warp partials of this lane's row, exchange with the peer (DSMEM) ----
      double D0 = 0.0, D1 = 0.0;
#pragma unroll
      for (int ws = 0; ws < kGroupWarps; ++ws) {
        const double2 v = lds128(red_r + (uint32_t)(ws * 4 * 32 * 16));
        D0 += v.x;
        D1 += v.y;
      }
      const int xb = g * 2 + (j & 1);
      const uint32_t mine = xb_local + (uint32_t)(((xb * kGroupWarps + w) * 32 + lane) * 16);
      st_async_v2f64(mapa_shared(mine, peer), D0, D1,
                     mapa_shared(xfull_local + (uint32_t)(xb * 8), peer));
      if (w == 0 && lane == 0) mbar_arrive_expect_tx(&xfull[xb], kGroupWarps * 32 * 16);
      mbar_wait_cluster(&xfull[xb], (j >> 1) & 1);
      {
        const double2 o = lds128(mine);
        D0 += o.x;  // IEEE addition commutes: both ranks hold (rank 0) + (rank 1)
        D1 += o.y;
      }
      if (prof) { const unsigned long long t = clock64(); ph[2] += t - t1; t1 = t; }

      // ---- epilogue: every lane of a quad forms the row's A and B; lane kk stores col kk ----
      double Dv[8];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        Dv[2 * l] = __shfl_sync(0xffffffffu, D0, quad | l);
        Dv[2 * l + 1] = __shfl_sync(0xffffffffu, D1, quad | l);
      }
      double A[4] = {0.0, 0.0, 0.0, 0.0}, B[4] = {0.0, 0.0, 0.0, 0.0};
      if (p.upd_a) {
        double x[4];
#pragma unroll
        for (int l = 0; l < 4; ++l)
          x[l] = l < s ? lds64(base + elem_off<2>(colA + l, erow)) - Dv[l] : 0.0;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          double a = 0.0;
#pragma unroll
          for (int l = 0; l <= jj; ++l) a += x[l] * ep_ai[l + 4 * jj];
          A[jj] = a;
        }
      }
      if (p.upd_b) {
        double y[4];
#pragma unroll
        for (int l = 0; l < 4; ++l)
          y[l] = l < s ? lds64(base + elem_off<2>(colB + l, erow)) - Dv[4 + l] : 0.0;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          double b = 0.0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            if (l <= jj) b += y[l] * ep_bi[l + 4 * jj];
            b -= A[l] * ep_w[l + 4 * jj];
          }
          B[jj] = b;
        }
      }
      if (kk < s) {
        const double av = kk == 0 ? A[0] : kk == 1 ? A[1] : kk == 2 ? A[2] : A[3];
        const double bv = kk == 0 ? B[0] : kk == 1 ? B[1] : kk == 2 ? B[2] : B[3];
        const bool live = erow < vrows;
        const long grow = row0 + erow;
        if (p.upd_a) {
          if (rank == 1) sts64(base + elem_off<2>(colA + kk, erow), av);  // rank 1 owns A's rows
          if (rank == 0 && live) p.dstA[grow + (size_t)kk * p.lddA] = av;
        }
        if (p.upd_b) {
          sts64(base + elem_off<2>(colB + kk, erow), bv);
          if (rank == 1 && live) p.dstB[grow + (size_t)kk * p.lddB] = bv;
        }
      }
      bar_named(gbar, 32 * kGroupWarps);
      if (prof) { const unsigned long long t = clock64(); ph[3] += t - t1; t1 = t; }

      // ---- Gram of this rank's output tiles (w + 4 jj) against span 1 ----
      double acc[MTW][2];
#pragma unroll
      for (int jj = 0; jj < MTW; ++jj) acc[jj][0] = acc[jj][1] = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double b[4];
        frag4<2>(base, bcol, h, kk, odd, b);
        if (!bval) b[0] = b[1] = b[2] = b[3] = 0.0;
#pragma unroll
        for (int jp = 0; jp < MTW; jp += 2) {
          const int t0i = w + kGroupWarps * jp, t1i = t0i + kGroupWarps;
          if (t0i < mt_loc) {
            const bool two = jp + 1 < MTW && t1i < mt_loc;
            const int lu0 = t0i < own_n ? t0i : t0i + ext_n;
            const int lu1 = two ? (t1i < own_n ? t1i : t1i + ext_n) : lu0;
            double a0[4], a1[4];
            frag4<2>(base, 8 * lu0 + ii, h, kk, odd, a0);
            frag4<2>(base, 8 * lu1 + ii, h, kk, odd, a1);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              dmma(acc[jp][0], acc[jp][1], a0[q4], b[q4]);
              if (jp + 1 < MTW && two) dmma(acc[jp + 1][0], acc[jp + 1][1], a1[q4], b[q4]);
            }
          }
        }
      }
      fence_proxy_async();  // generic writes of A / B before TMA refills the slot
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
      for (int jj = 0; jj < MTW; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double sm, err;
          two_sum(hi[jj][e], acc[jj][e], sm, err);
          hi[jj][e] = sm;
          lo[jj][e] += err;
        }
      if (prof) { const unsigned long long t = clock64(); ph[4] += t - t1; }
    }
    if (prof) {
      ph[5] = clock64() - t_begin;
      unsigned long long* dst = p.phase + (size_t)blockIdx.x * 16 + 8 * g;
      for (int i = 0; i < 6; ++i) atomicAdd(&dst[i], ph[i]);
      atomicAdd(&dst[6], (unsigned long long)((nst - g + 1) / 2));
    }
    double2* part = reinterpret_cast<double2*>(p.partial) + (size_t)(cl * 2 + g) * p.mt_out * 64;
#pragma unroll
    for (int jj = 0; jj < MTW; ++jj) {
      const int t = w + kGroupWarps * jj;
      if (t < mt_loc) {
        const int tg = t < own_n ? own_u0 + t : p.U0 + (t - own_n);
#pragma unroll
        for (int e = 0; e < 2; ++e)
          part[((size_t)tg * 8 + ii) * 8 + 2 * kk + e] = make_double2(hi[jj][e], lo[jj][e]);
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while its peer may still address its shared memory
}

// ------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------
namespace {
// instances: KW k-steps per warp in {2, 4, ..., 16}, MTW = KW / 2 output tiles per warp
constexpr int kKwStep = 2, kKwMax = 16;
int mtw_for(int kw_t) { return (kw_t + 1) / 2; }
}  // namespace

bool k12_plan(SplitParams& p) {
  if (p.s < 1 || p.s > 4 || p.N < 1 || p.N > 8 || p.U0 < 1 || p.U1 < 1) return false;
  for (int j = 0; j < p.N; ++j)
    if (p.rcol1[j] < 0 || p.rcol1[j] >= 8 * p.U1) return false;
  const int na = p.upd_a ? p.U0 - p.kp / 8 : 0;  // units holding the A block (span-0 tail)
  if (na < 0 || na > p.U0) return false;
  const int uh = (p.U0 - na + 1) / 2;
  p.own_u0[0] = 0;       p.own_n[0] = uh;
  p.ext_u0[0] = p.U0 - na; p.ext_n[0] = na;
  p.own_u0[1] = uh;      p.own_n[1] = p.U0 - uh;
  p.ext_u0[1] = 0;       p.ext_n[1] = 0;
  p.s1_left = (p.lcols1 + 7) / 8;
  p.mt_out = p.U0 + p.s1_left;
  p.slot_units = std::max(uh + na, p.U0 - uh) + p.U1;
  const int c0 = std::min(8 * uh, p.kp), c1 = std::max(0, p.kp - 8 * uh);
  if (c0 % 4 || c1 % 4) return false;  // whole k-steps only (always true for s = 4)
  const int k0 = c0 / 4, k1 = c1 / 4;
  const int kw = (std::max(k0, k1) + kGroupWarps - 1) / kGroupWarps;
  const int mt = std::max(uh + p.s1_left, p.U0 - uh);
  const int mtw = (mt + kGroupWarps - 1) / kGroupWarps;
  int kw_t = std::max(kKwStep, (kw + kKwStep - 1) / kKwStep * kKwStep);
  while (mtw_for(kw_t) < mtw) kw_t += kKwStep;
  if (kw_t > kKwMax) return false;
  p.kw = kw_t;
  p.mtw = mtw_for(kw_t);
  int S = 0;
  for (int st = kMaxStages; st >= 2; --st)
    if (k12_smem_bytes(st, p.slot_units) + kStaticSmem + 256 <= (size_t)kSmemOptin) {
      S = st;
      break;
    }
  if (S < 3) return false;
  p.stages = S;
  return true;
}

template <int KW>
static cudaError_t launch_k12(const SplitParams& p, int grid, cudaStream_t st) {
  constexpr int MTW = (KW + 1) / 2;
  auto k = k12_kernel<KW, MTW>;
  const size_t smem = k12_smem_bytes(p.stages, p.slot_units);
  cudaError_t e = ensure_smem(k, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, p);
}

cudaError_t k12_launch(const SplitParams& p, int grid, cudaStream_t st, int* launches) {
  if (grid < 2 || (grid & 1)) return cudaErrorInvalidValue;
  if (launches) *launches += 1;
  switch (p.kw) {
    case 2: return launch_k12<2>(p, grid, st);
    case 4: return launch_k12<4>(p, grid, st);
    case 6: return launch_k12<6>(p, grid, st);
    case 8: return launch_k12<8>(p, grid, st);
    case 10: return launch_k12<10>(p, grid, st);
    case 12: return launch_k12<12>(p, grid, st);
    case 14: return launch_k12<14>(p, grid, st);
    case 16: return launch_k12<16>(p, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bgs
