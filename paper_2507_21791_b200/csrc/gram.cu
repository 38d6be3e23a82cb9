// gram.cu — K1: tall-skinny Gram  G = L^T R  on fp64 tensor cores (DMMA), TMA-fed.
//
// Replaces fused_gram (dist_block.cpp:79-88) + gram_accumulate (dense_kernels.cpp:10-27)
// + the per-rank half of exact_allreduce (communicator.cpp:226-250).  The reference
// accumulates every product exactly in a 2176-bit fixed-point register; here each
// 16-row stage is contracted with DMMA.8x8x4 and the stage sums are folded into a
// double-double (hi, lo) accumulator every FLUSH stages, then CTA partials are summed
// in a fixed order in double-double (gram_reduce) — deterministic, and accurate to
// O(16u) per entry instead of O(n u).
//
// Data layout: the operand columns come from up to two column spans of column-major
// matrices (the Q buffer and X), each addressed by a CUtensorMap.  One pipeline stage =
// 16 rows x (all boxes); a box = 16 rows x 8 columns = 1 KB, SWIZZLE_128B, so a stage of
// a (k+2)s = 408-column operand is 51 KB and the whole operand row-tile streams from HBM
// exactly once.  The right operand R is a set of columns that are already in the tile
// (BlockSpan semantics of the reference: R's columns are a suffix of L's, or of the
// second span), so it costs no extra HBM traffic.
//
// Roles: warp 0 lane 0 = TMA producer; warps 1..W = DMMA consumers.  Consumer warp w owns
// m-tiles (boxes) w, w+W, ... and all n-tiles; per k-step (4 rows) one DMMA per
// (m-tile, n-tile).  Fragment loads are conflict-free LDS.128 thanks to the swizzle.
#include "common.cuh"
#include "kernels.h"

namespace bgs {

template <int NT, int W, int MTW, bool COMP>
__global__ void __launch_bounds__(32 * (W + 1), 1)
    gram_kernel(const __grid_constant__ GramParams p) {
  if (p.status && status_bad(p.status)) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const int stage_bytes = p.nboxes * 1024;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long T = p.total_stages;
  const long st0 = (long)blockIdx.x * T / gridDim.x;
  const long st1 = (long)(blockIdx.x + 1) * T / gridDim.x;
  const int nst = (int)(st1 - st0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], W);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      prefetch_tmap(&p.map[0]);
      if (p.nbox[1] > 0) prefetch_tmap(&p.map[1]);
      for (int it = 0; it < nst; ++it) {
        const int slot = it % S;
        const int round = it / S;
        mbar_wait(&empty[slot], (round & 1) ^ 1);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)stage_bytes);
        unsigned char* dst = smem + (size_t)slot * stage_bytes;
        const int row = (int)((st0 + it) * 16);
        for (int b = 0; b < p.nbox[0]; ++b)
          tma_load_2d(dst + b * 1024, &p.map[0], &full[slot], row, p.col0[0] + 8 * b);
        for (int b = 0; b < p.nbox[1]; ++b)
          tma_load_2d(dst + (p.nbox[0] + b) * 1024, &p.map[1], &full[slot], row,
                      p.col0[1] + 8 * b);
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  const int cw = warp - 1;
  const int kk = lane & 3, ii = lane >> 2;
  int cnt = 0;
  for (int t = cw; t < p.mt_out; t += W) ++cnt;

  uint32_t boff0[NT], boff1[NT];
  bool bval[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int col = p.rcol[nt * 8 + ii];
    bval[nt] = col >= 0;
    const int c = col >= 0 ? col : 0;
    boff0[nt] = swz(c, 2 * kk);
    boff1[nt] = swz(c, 2 * kk + 1);
  }
  uint32_t aoff0[MTW], aoff1[MTW];
#pragma unroll
  for (int j = 0; j < MTW; ++j) {
    const int t = cw + W * (j < cnt ? j : 0);
    const int col = 8 * t + ii;
    aoff0[j] = swz(col, 2 * kk);
    aoff1[j] = swz(col, 2 * kk + 1);
  }

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

  auto flush = [&]() {
    if (COMP) {
#pragma unroll
      for (int j = 0; j < MTW; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double s, err;
            two_sum(hi[j][nt][e], acc[j][nt][e], s, err);
            hi[j][nt][e] = s;
            lo[j][nt][e] += err;
            acc[j][nt][e] = 0.0;
          }
    }
  };

  const uint32_t sbase = smem_u32(smem);
  int since = 0;
  for (int it = 0; it < nst; ++it) {
    const int slot = it % S;
    mbar_wait(&full[slot], (it / S) & 1);
    const uint32_t base = sbase + (uint32_t)(slot * stage_bytes);
    double b[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double2 v0 = lds128(base + boff0[nt]);
      double2 v1 = lds128(base + boff1[nt]);
      b[nt][0] = bval[nt] ? v0.x : 0.0;
      b[nt][1] = bval[nt] ? v0.y : 0.0;
      b[nt][2] = bval[nt] ? v1.x : 0.0;
      b[nt][3] = bval[nt] ? v1.y : 0.0;
    }
#pragma unroll
    for (int j = 0; j < MTW; ++j) {
      if (j < cnt) {
        double2 a0 = lds128(base + aoff0[j]);
        double2 a1 = lds128(base + aoff1[j]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(acc[j][nt][0], acc[j][nt][1], a0.x, b[nt][0]);
          dmma(acc[j][nt][0], acc[j][nt][1], a0.y, b[nt][1]);
          dmma(acc[j][nt][0], acc[j][nt][1], a1.x, b[nt][2]);
          dmma(acc[j][nt][0], acc[j][nt][1], a1.y, b[nt][3]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++since == GRAM_FLUSH) {
      flush();
      since = 0;
    }
  }
  flush();

  // ---------------- per-CTA partial (hi, lo) ----------------
  const int N8 = 8 * NT;
  double2* part = reinterpret_cast<double2*>(p.partial) + (size_t)blockIdx.x * p.mt_out * 8 * N8;
#pragma unroll
  for (int j = 0; j < MTW; ++j) {
    if (j < cnt) {
      const int t = cw + W * j;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = nt * 8 + 2 * kk + e;
          double h = COMP ? hi[j][nt][e] : acc[j][nt][e];
          double l = COMP ? lo[j][nt][e] : 0.0;
          part[((size_t)t * 8 + ii) * N8 + n] = make_double2(h, l);
        }
    }
  }
}

// Deterministic cross-CTA reduction in double-double, rank-local.  One thread per
// output entry; CTA partials are summed in CTA order (fixed, so results are
// reproducible run to run).  Writes the compact M x N column-major Gram.
__global__ void gram_reduce_kernel(const double2* __restrict__ part, int G, int mt_out, int N8,
                                   int N, int nbox0, int lcols0, int lcols1, int M,
                                   double* __restrict__ out, const DevStatus* status) {
  if (status && status_bad(status)) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int per_cta = mt_out * 8 * N8;
  if (idx >= per_cta) return;
  const int n = idx % N8;
  const int i = (idx / N8) % 8;
  const int t = idx / (8 * N8);
  if (n >= N) return;
  int row;
  if (t < nbox0) {
    row = 8 * t + i;
    if (row >= lcols0) return;
  } else {
    const int r = 8 * (t - nbox0) + i;
    if (r >= lcols1) return;
    row = lcols0 + r;
  }
  double s = 0.0, e = 0.0;
  const double2* ptr = part + idx;
#pragma unroll 8
  for (int g = 0; g < G; ++g) {
    const double2 v = ptr[(size_t)g * per_cta];
    double s2, err;
    two_sum(s, v.x, s2, err);
    s = s2;
    e += err + v.y;
  }
  out[row + (size_t)n * M] = s + e;
}

// ------------------------------------------------------------------------------------
// Host launchers
// ------------------------------------------------------------------------------------
template <int NT, int W, int MTW, bool COMP>
static cudaError_t launch_one(const GramParams& p, int grid, size_t smem, cudaStream_t st) {
  auto k = gram_kernel<NT, W, MTW, COMP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, 32 * (W + 1), smem, st>>>(p);
  return cudaGetLastError();
}

template <int NT>
static cudaError_t dispatch_mtw(const GramParams& p, int mtw, int grid, size_t smem,
                                cudaStream_t st) {
  constexpr bool C2 = NT * 2 * 6 <= 96, C4 = NT * 4 * 6 <= 96, C7 = NT * 7 * 6 <= 96,
                 C13 = NT * 13 * 6 <= 96;
  if (mtw <= 2) return launch_one<NT, 8, 2, C2>(p, grid, smem, st);
  if (mtw <= 4) return launch_one<NT, 8, 4, C4>(p, grid, smem, st);
  if (mtw <= 7) return launch_one<NT, 8, 7, C7>(p, grid, smem, st);
  if (mtw <= 13) return launch_one<NT, 8, 13, (NT == 1) && C13>(p, grid, smem, st);
  return cudaErrorInvalidValue;
}

int gram_n_tiles(int N) {
  int nt = (N + 7) / 8;
  return nt == 3 ? 4 : nt;
}

size_t gram_partial_doubles_per_cta(int mt_out, int N) {
  return (size_t)mt_out * 8 * 8 * gram_n_tiles(N) * 2;
}

cudaError_t gram_partials_launch(GramParams& p, int grid, cudaStream_t st, int* launches) {
  const int W = 8;
  if (p.N < 1 || p.N > 32 || p.mt_out < 1 || grid < 1) return cudaErrorInvalidValue;
  p.nt = gram_n_tiles(p.N);
  p.total_stages = (p.n_rows + 15) / 16;
  const int stage_bytes = p.nboxes * 1024;
  int S = (GRAM_SMEM_BUDGET - 2048) / stage_bytes;
  if (S > 16) S = 16;
  if (S < 2) return cudaErrorInvalidValue;
  p.stages = S;
  const size_t smem = (size_t)S * stage_bytes + 1024 + 2 * S * sizeof(uint64_t) + 64;
  const int mtw = (p.mt_out + W - 1) / W;
  if (launches) *launches += 1;
  switch (p.nt) {
    case 1: return dispatch_mtw<1>(p, mtw, grid, smem, st);
    case 2: return dispatch_mtw<2>(p, mtw, grid, smem, st);
    default: return dispatch_mtw<4>(p, mtw, grid, smem, st);
  }
}

cudaError_t gram_reduce_launch(const GramParams& p, int ctas, double* out, cudaStream_t st,
                               int* launches) {
  const int N8 = 8 * gram_n_tiles(p.N);
  const int entries = p.mt_out * 8 * N8;
  const int lc1 = p.mt_out > p.nbox[0] ? p.lcols[1] : 0;
  gram_reduce_kernel<<<(entries + 255) / 256, 256, 0, st>>>(
      reinterpret_cast<const double2*>(p.partial), ctas, p.mt_out, N8, p.N, p.nbox[0],
      p.lcols[0], lc1, p.lcols[0] + lc1, out, p.status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
