// update_tma.cu — K2m: the block update for s = 5..16 with the prefix streamed by TMA.
//
// Same algebra and call sites as K2 (update.cu; local_axpy_block + scale_right_block,
// dist_block.cpp:90-117, bcgs.cpp:329-331, 346-359, 151-160):
//   A = (srcA - Qp CA) TA^{-1},  B = (srcB - Qp CB[0:kp] - A CB[kp:kp+s]) TB^{-1}
// At s >= 8 K2t (update.cu) fetched its DMMA A fragments with per-lane global loads and ran
// latency-bound at 0.3-0.45 of the roofline (profiles/r02_ncu_k2t.md).  Here:
//  * a persistent CTA per SM walks 128-row blocks of its shard; the prefix Q[:, 0:kp] of a
//    block streams through a ring of k-chunk stages: 128 rows x 32 columns as four 32-row
//    quads (3-D TMA boxes {16, 2, w}: 256-byte runs per column, SWIZZLE_128B, K12c's
//    conflict-free fragment layout) FOLLOWED BY THE CHUNK'S COEFFICIENTS, already in
//    DMMA-fragment order (one 1-D bulk copy from a buffer a small pack kernel fills once per
//    launch).  The first K2m kept all kp x 2S coefficients in shared memory (102 KB at
//    kp = 400, s = 16), which left room for neither a wider warp tile nor long prefixes;
//  * 8 DMMA warps, each a 32-row quad x TWO n-tiles of [CA | CB] (8 accumulators: 8 DMMAs
//    per 2 LDS.128 + 2 LDS.64; one n-tile per warp was shared-memory bound at s = 16: ncu
//    79% of the shared pipe, DMMA pipe 48%): warp w = quad w % 4, and w / 4 selects the
//    n-tile pair (s > 8: NT = 4) or the k-part (s <= 8: NT = 2, the k-steps split in two);
//  * the products of a block go to one of two shared scratch buffers (one slice per k-part)
//    and four epilogue warps, one per quad (lane r owns row 32 e + r), apply the block's
//    factors while the DMMA warps run the next block: z = src - D, then A = zA TA^{-1} and
//    B = (zB - A S2) TB^{-1} by back-substitution (the reference's tri_solve_right order).
// Bytes per row: 8 (kp + 2s) read + 8 (2s) written, as K2 (+ the coefficients once per block,
// from L2).  s = 8 is HBM-bound (AI 4), s = 16 fp64-tensor-bound (AI 8).
#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {
constexpr int kUmWarps = 8;                          // DMMA warps
constexpr int kUmEpi = 4;                            // epilogue warps (one per quad)
constexpr int kUmProd = kUmWarps + kUmEpi;           // producer warp index
constexpr int kUmThreads = 32 * (kUmWarps + kUmEpi + 1);
constexpr int kUmQuads = 4;                          // 32-row quads per block
constexpr int kUmRows = 32 * kUmQuads;               // rows per block
constexpr int kUmKC = 32;                            // prefix columns per stage
constexpr int kUmTileBytes = kUmKC * kUmRows * 8;    // 32 KB
constexpr int kUmQuadBytes = kUmKC * 32 * 8;         // 8 KB
constexpr int kUmNTW = 2;                            // n-tiles per DMMA warp
constexpr int kUmStagesMax = 6;
constexpr int kUmBufs = 2;                           // D scratch buffers (alternate blocks)
constexpr int kUmSmemMax = 232448 - 1024;

__host__ __device__ constexpr int um_nt(int S) { return 2 * S / 8; }
// k-parts: the 8 warps are 4 quads x (NT / 2 n-tile pairs) x KS
__host__ __device__ constexpr int um_ks(int S) { return kUmWarps / (kUmQuads * (um_nt(S) / kUmNTW)); }
__host__ __device__ constexpr int um_coef_chunk_bytes(int S) { return (kUmKC / 4) * um_nt(S) * 32 * 8; }
__host__ __device__ constexpr int um_stage_bytes(int S) { return kUmTileBytes + um_coef_chunk_bytes(S); }
// per-block scratch [KS k-parts][128 rows][2S + 1]; the epilogue sums the k-parts in order
__host__ __device__ constexpr int um_scratch_doubles(int S) { return um_ks(S) * kUmRows * (2 * S + 1); }

}  // namespace

size_t update_tma_coef_doubles(int s, int kp) {
  const int S = s <= 8 ? 8 : 16;
  return (size_t)((kp + 3) / 4) * um_nt(S) * 32;
}

size_t update_tma_smem_bytes(int s, int kp, int stages) {
  (void)kp;
  const int S = s <= 8 ? 8 : 16;
  return 1024 + (size_t)stages * um_stage_bytes(S) +
         (size_t)kUmBufs * um_scratch_doubles(S) * sizeof(double) +
         (size_t)3 * S * S * sizeof(double) +
         (2 * kUmStagesMax + 2 * kUmBufs) * sizeof(uint64_t) + 64;
}

static int um_stages(int s, int kp) {
  for (int st = kUmStagesMax; st >= 3; --st)
    if (update_tma_smem_bytes(s, kp, st) <= (size_t)kUmSmemMax) return st;
  return 0;
}

int update_tma_max_kp(int s) {
  return um_stages(s, 8) >= 3 ? 1 << 20 : 0;  // (the coefficients stream: no panel limit)
}

// coefficient fragments: lane (i, kk) of n-tile t, k-step j holds C[4j + kk][8t + i]
template <int S, bool HA, bool HB>
__global__ void um_pack_kernel(const UpdTmaParams p) {
  constexpr int NT = um_nt(S);
  const int total = (p.kp / 4) * NT * 32;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int l = idx & 31, t = (idx >> 5) % NT, j = (idx >> 5) / NT;
    const int c = 4 * j + (l & 3), n = 8 * t + (l >> 2);
    double v = 0.0;
    if (n < S) {
      if (HA && n < p.s) v = p.CA[c + (size_t)n * p.ldca];
    } else if (HB && n - S < p.s) {
      v = p.CB[c + (size_t)(n - S) * p.ldcb];
    }
    p.coef_ws[idx] = v;
  }
}

template <int S, bool HA, bool HB>
__global__ void __launch_bounds__(kUmThreads, 1) update_tma_kernel(const __grid_constant__ UpdTmaParams p) {
  constexpr int NT = um_nt(S), KS = um_ks(S);
  constexpr int LDD = 2 * S + 1;
  constexpr int kStage = um_stage_bytes(S);
  if (p.status && status_bad(p.status)) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kp = p.kp, s = p.s;
  const int ksteps = kp / 4;                       // kp is a multiple of 8 here
  const int nchunk = (kp + kUmKC - 1) / kUmKC;
  const int NS = p.stages;
  double* scr = reinterpret_cast<double*>(smem + (size_t)NS * kStage);  // [kUmBufs][KS][128][LDD]
  double* ta = scr + (size_t)kUmBufs * um_scratch_doubles(S);  // S x S each (col-major)
  double* tb = ta + S * S;
  double* s2 = tb + S * S;                         // CB[kp:kp+s] (B's coupling to A)
  uint64_t* full = reinterpret_cast<uint64_t*>(s2 + S * S);
  uint64_t* empty = full + kUmStagesMax;
  uint64_t* dfull = empty + kUmStagesMax;          // [kUmBufs]
  uint64_t* dempty = dfull + kUmBufs;              // [kUmBufs]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nblk = p.total_blocks;
#ifdef BGS_CHECKED
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    BGS_DCHECK(reinterpret_cast<unsigned char*>(dempty + kUmBufs) - smem_raw <= (long)dyn,
               "k2m: shared-memory layout exceeds the allocation");
    BGS_DCHECK(kp % 8 == 0 && NS >= 3 && NS <= kUmStagesMax, "k2m: kp / ring depth");
  }
#endif
  const long b0 = (long)blockIdx.x * nblk / gridDim.x;
  const long b1 = (long)(blockIdx.x + 1) * nblk / gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kUmWarps);
    }
    for (int i = 0; i < kUmBufs; ++i) {
      mbar_init(&dfull[i], kUmWarps);
      mbar_init(&dempty[i], kUmEpi);
    }
    fence_mbar_init();
  }
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx % S, j = idx / S;
    const bool in = i < s && j < s;
    ta[idx] = (HA && p.TA && in) ? p.TA[i + (size_t)j * s] : (i == j ? 1.0 : 0.0);
    tb[idx] = (HB && p.TB && in) ? p.TB[i + (size_t)j * s] : (i == j ? 1.0 : 0.0);
    s2[idx] = (HA && HB && p.cb_has_a && in) ? p.CB[kp + i + (size_t)j * p.ldcb] : 0.0;
  }
  __syncthreads();
  // The epilogue warps back-substitute with TA / TB themselves (tri_solve_right's order,
  // dense_kernels.cpp:89-110: x_j = (z_j - sum_{l<j} x_l T_lj) / T_jj), one row per lane.
  // They run beside the DMMA warps with a whole block's contraction to hide their serial
  // chains, and an explicit factor matrix [[TA^-1, -TA^-1 S2 TB^-1], [0, TB^-1]] (the first
  // K2m, as K12c's) cost BCGSI+1S orthogonality at s = 8 on ill-conditioned diagonal blocks
  // (fuzz case n = m = 80: LOO 14x the oracle's against 2.7x with substitution).

  if (warp == kUmProd) {
    // ---------------- producer: k-chunk stages (tile quads + coefficients) of every block ----------------
    if (lane == 0) {
      for (int i = 0; i < 5; ++i) prefetch_tmap(&p.map[i]);
      long it = 0;
      for (long b = b0; b < b1; ++b) {
        for (int c = 0; c < nchunk; ++c, ++it) {
          const int slot = (int)(it % NS);
          if (it >= NS) mbar_wait(&empty[slot], (uint32_t)(((it / NS) - 1) & 1));
          const int c0 = c * kUmKC, w = min(kUmKC, kp - c0);
          const uint32_t cbytes = (uint32_t)((w / 4) * NT * 32 * 8);
          mbar_arrive_expect_tx(&full[slot], (uint32_t)(w * kUmRows * 8) + cbytes);
          unsigned char* dst = smem + (size_t)slot * kStage;
          bulk_load_1d(dst + kUmTileBytes, p.coef_ws + (size_t)(c0 / 4) * NT * 32, cbytes, &full[slot]);
          int done = 0;
          while (done < w) {  // greedy boxes {16, 2, 32 / 16 / 8}, one per 32-row quad
            const int left = w - done;
            const int wi = left >= 32 ? 2 : left >= 16 ? 3 : 4;
            BGS_DCHECK(done + (128 >> wi) <= kUmKC, "k2m: TMA box past the stage");
#pragma unroll
            for (int qd = 0; qd < kUmQuads; ++qd)
              tma_load_3d(dst + (size_t)qd * kUmQuadBytes + (size_t)done * 256, &p.map[wi],
                          &full[slot], 0, (int)(2 * kUmQuads * b + 2 * qd), p.col0 + c0 + done);
            done += 128 >> wi;
          }
        }
      }
    }
    return;
  }

  if (warp >= kUmWarps) {
    // ---------------- epilogue warps: warp e takes quad e (row 32 e + lane) of every block ----------------
    const int e = warp - kUmWarps;
    long u = 0;  // blocks so far
    for (long b = b0; b < b1; ++b, ++u) {
      const int buf = (int)(u % kUmBufs);
      double* zb0 = scr + (size_t)buf * um_scratch_doubles(S);
      const long row = b * kUmRows + 32 * e + lane;
      const bool live = row < p.n_rows;
      // the sources of this lane's row do not depend on the contraction: loaded before the wait
      double za[S], zb[S];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        za[j] = (HA && live && j < s) ? p.srcA[row + (size_t)j * p.ld_srcA] : 0.0;
        zb[j] = (HB && live && j < s) ? p.srcB[row + (size_t)j * p.ld_srcB] : 0.0;
      }
      mbar_wait(&dfull[buf], (uint32_t)((u / kUmBufs) & 1));
      // z = src - D, in place in this row of the scratch (odd stride: conflict-free)
      double* zr = zb0 + (size_t)(32 * e + lane) * LDD;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        double da = zr[j], db = zr[S + j];
        if (KS > 1) {
#pragma unroll
          for (int k2 = 1; k2 < KS; ++k2) {  // k-part order
            da += zr[(size_t)k2 * kUmRows * LDD + j];
            db += zr[(size_t)k2 * kUmRows * LDD + S + j];
          }
        }
        if (HA) zr[j] = za[j] - da;
        if (HB) zr[S + j] = zb[j] - db;
      }
      double a[S];
#pragma unroll
      for (int j = 0; j < S; ++j) a[j] = 0.0;
      if (HA) {
#pragma unroll
        for (int j = 0; j < S; ++j) {  // A = zA TA^{-1}
          double acc = zr[j];
#pragma unroll
          for (int l = 0; l < j; ++l) acc -= a[l] * ta[l + j * S];
          a[j] = acc / ta[j + j * S];
        }
        if (live)
#pragma unroll
          for (int j = 0; j < S; ++j)
            if (j < s) p.dstA[row + (size_t)j * p.ld_dstA] = a[j];
      }
      if (HB) {
        double bb[S];
#pragma unroll
        for (int j = 0; j < S; ++j) {  // B = (zB - A S2) TB^{-1}
          double acc = zr[S + j];
          if (HA && p.cb_has_a) {
#pragma unroll
            for (int l = 0; l < S; ++l) acc -= a[l] * s2[l + j * S];
          }
#pragma unroll
          for (int l = 0; l < j; ++l) acc -= bb[l] * tb[l + j * S];
          bb[j] = acc / tb[j + j * S];
        }
        if (live)
#pragma unroll
          for (int j = 0; j < S; ++j)
            if (j < s) p.dstB[row + (size_t)j * p.ld_dstB] = bb[j];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[buf]);  // (all four quads: the scratch is free again)
    }
    return;
  }

  // ---------------- DMMA warps ----------------
  const int qd = warp % kUmQuads, g2 = warp / kUmQuads;
  const int tp = NT > kUmNTW ? g2 : 0;         // n-tile pair of this warp
  const int kpart = NT > kUmNTW ? 0 : g2;      // or its k-part
  const int ii = lane >> 2, kk = lane & 3;
  // m-tile q of the quad, row index i is quad row 4 f(i) + q with f(i) = (i >> 1) + 4 (i & 1):
  // two LDS.128 give lane (i, kk) its 4 rows of k-step column 4j + kk (K12c's conflict-free
  // scheme on the {16, 2, w} quad layout: line 2c + h)
  uint32_t uoff0, uoff1;
  {
    const int line = 2 * kk + (ii & 1);
    const int rc = 2 * (ii >> 1);
    uoff0 = (uint32_t)(line * 128 + ((rc ^ (line & 7)) << 4));
    uoff1 = (uint32_t)(line * 128 + (((rc + 1) ^ (line & 7)) << 4));
  }
  const int f = (ii >> 1) + 4 * (ii & 1);
  const uint32_t sbase = smem_u32(smem);
  // this lane's coefficient of n-tile 2 tp + n2, local k-step jj: chunk + ((jj NT + t) 32 + lane) 8
  const uint32_t cfo = (uint32_t)(kUmTileBytes + ((kUmNTW * tp) * 32 + lane) * 8);
  long it = 0;
  for (long b = b0; b < b1; ++b) {
    double d[4][kUmNTW][2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int n2 = 0; n2 < kUmNTW; ++n2) d[q][n2][0] = d[q][n2][1] = 0.0;
    for (int c = 0; c < nchunk; ++c, ++it) {
      const int slot = (int)(it % NS);
      mbar_wait(&full[slot], (uint32_t)((it / NS) & 1));
      const int j0 = c * (kUmKC / 4), nj = min(kUmKC / 4, ksteps - j0);
      const uint32_t stg = sbase + (uint32_t)(slot * kStage);
      const uint32_t base = stg + (uint32_t)(qd * kUmQuadBytes);
#pragma unroll 2
      for (int jj = kpart; jj < nj; jj += KS) {
        const uint32_t a0 = base + 1024u * (uint32_t)jj;
        const double2 x0 = lds128(a0 + uoff0), x1 = lds128(a0 + uoff1);
        const uint32_t cf = stg + cfo + (uint32_t)(jj * NT * 256);
        const double bv0 = lds64(cf), bv1 = lds64(cf + 256u);
        dmma(d[0][0][0], d[0][0][1], x0.x, bv0);
        dmma(d[1][0][0], d[1][0][1], x0.y, bv0);
        dmma(d[2][0][0], d[2][0][1], x1.x, bv0);
        dmma(d[3][0][0], d[3][0][1], x1.y, bv0);
        dmma(d[0][1][0], d[0][1][1], x0.x, bv1);
        dmma(d[1][1][0], d[1][1][1], x0.y, bv1);
        dmma(d[2][1][0], d[2][1][1], x1.x, bv1);
        dmma(d[3][1][0], d[3][1][1], x1.y, bv1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    // this warp's product -> scratch[(b - b0) % kUmBufs][kpart][row][8 t + 2 kk + e]
    const long ub = b - b0;
    const int e = (int)(ub % kUmBufs);
    if (ub >= kUmBufs) mbar_wait(&dempty[e], (uint32_t)((ub / kUmBufs - 1) & 1));
    double* sl = scr + (size_t)e * um_scratch_doubles(S) + (size_t)kpart * kUmRows * LDD;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int n2 = 0; n2 < kUmNTW; ++n2) {
        double* rp = sl + (size_t)(32 * qd + 4 * f + q) * LDD + 8 * (kUmNTW * tp + n2) + 2 * kk;
        rp[0] = d[q][n2][0];
        rp[1] = d[q][n2][1];
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&dfull[e]);
  }
}

template <int S, bool HA, bool HB>
static cudaError_t launch_um(const UpdTmaParams& p, int grid, cudaStream_t st) {
  const int total = (p.kp / 4) * um_nt(S) * 32;
  um_pack_kernel<S, HA, HB><<<std::max(1, std::min(64, (total + 255) / 256)), 256, 0, st>>>(p);
  auto k = update_tma_kernel<S, HA, HB>;
  const size_t smem = update_tma_smem_bytes(S, p.kp, p.stages);
  cudaError_t e = ensure_smem(k, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, kUmThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t update_tma_launch(UpdTmaParams& p, int num_sms, cudaStream_t st, int* launches) {
  if (p.s < 5 || p.s > 16 || p.kp < 8 || p.kp % 8 || !p.coef_ws) return cudaErrorInvalidValue;
  p.total_blocks = (p.n_rows + kUmRows - 1) / kUmRows;
  p.stages = um_stages(p.s, p.kp);
  if (p.stages < 3) return cudaErrorInvalidValue;
  if (p.total_blocks < 1) return cudaSuccess;
  const int grid = (int)std::min<long>(num_sms, p.total_blocks);
  if (launches) *launches += 2;
  const bool S8 = p.s <= 8;
  if (p.has_a && p.has_b)
    return S8 ? launch_um<8, true, true>(p, grid, st) : launch_um<16, true, true>(p, grid, st);
  if (p.has_a)
    return S8 ? launch_um<8, true, false>(p, grid, st) : launch_um<16, true, false>(p, grid, st);
  if (p.has_b)
    return S8 ? launch_um<8, false, true>(p, grid, st) : launch_um<16, false, true>(p, grid, st);
  return cudaSuccess;
}

}  // namespace bgs
