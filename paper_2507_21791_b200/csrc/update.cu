// update.cu — K2: fused tall-skinny block update.
//
// Replaces local_axpy_block (dist_block.cpp:90-108) + scale_right_block /
// tri_solve_right (dist_block.cpp:110-117, dense_kernels.cpp:89-110) + the
// extract_block / set_block copies (dist_block.cpp:46-49, 119-125) of one block step of
// bcgs.cpp.  One pass over the Q prefix produces up to two output blocks per row:
//
//   A = (srcA - Qp * CA) * TA^{-1}                       (e.g. Q_k = (U - Q Y) Y_kk^{-1})
//   B = (srcB - Qp * CB[0:kp] - A * CB[kp:kp+s]) * TB^{-1}
//                                   (e.g. U_{k+1} = (X_{k+1} - Q_{1:k+1} [Z; S2]) S^{-1})
//
// Triangular factors are applied by back-substitution (never an explicit inverse,
// SPEC.md:383/415), exactly as tri_solve_right does per row.  Each thread owns RPT
// consecutive rows; the prefix columns are read once, coalesced, with 128-bit loads;
// the (kp x 2s) coefficient panel is staged in shared memory and read as broadcasts.
// HBM traffic per row: 8*(kp + 2s) bytes read + 8*2s written.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace bgs {

template <int S, int RPT, bool HA, bool HB>
__global__ void __launch_bounds__(256) update_kernel(const UpdateParams p) {
  if (p.status && status_bad(p.status)) return;
  extern __shared__ __align__(16) double coef[];  // [kp][2S] interleaved CA | CB rows
  double* ta = coef + (size_t)p.kp * 2 * S;        // S x S (col-major)
  double* tb = ta + S * S;                         // S x S
  double* cbx = tb + S * S;                        // S x S: CB rows kp..kp+S-1
  const int kp = p.kp;
  // Runtime block width s <= S: padded coefficient columns are zero and padded
  // triangular factors are the identity, so padded outputs are exact zeros (not stored).
  const int s = p.s;
  for (int idx = threadIdx.x; idx < kp * S; idx += blockDim.x) {
    const int c = idx / S, j = idx % S;
    coef[c * 2 * S + j] = (HA && j < s) ? p.CA[c + (size_t)j * p.ldca] : 0.0;
    coef[c * 2 * S + S + j] = (HB && j < s) ? p.CB[c + (size_t)j * p.ldcb] : 0.0;
  }
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx % S, j = idx / S;
    const bool in = i < s && j < s;
    ta[idx] = (HA && p.TA && in) ? p.TA[i + (size_t)j * p.ldta] : (i == j ? 1.0 : 0.0);
    tb[idx] = (HB && p.TB && in) ? p.TB[i + (size_t)j * p.ldtb] : (i == j ? 1.0 : 0.0);
    cbx[idx] = (HA && HB && p.cb_has_a && in) ? p.CB[kp + i + (size_t)j * p.ldcb] : 0.0;
  }
  __syncthreads();

  const long nrow_groups = (p.n_rows + RPT - 1) / RPT;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < nrow_groups;
       g += (long)gridDim.x * blockDim.x) {
    const long r0 = g * RPT;
    double accA[RPT][S], accB[RPT][S];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int j = 0; j < S; ++j) accA[r][j] = accB[r][j] = 0.0;

    const double* qcol = p.qp + r0;
    int c = 0;
    // 4-way unrolled stream over the prefix columns (independent loads in flight).
    for (; c + 4 <= kp; c += 4) {
      double v[4][RPT];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* ptr = qcol + (size_t)(c + u) * p.ldq;
        if (RPT == 2) {
          const double2 t = __ldg(reinterpret_cast<const double2*>(ptr));
          v[u][0] = t.x;
          v[u][RPT - 1] = t.y;
        } else {
          v[u][0] = __ldg(ptr);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* cr = coef + (c + u) * 2 * S;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const double ca = cr[j], cb = cr[S + j];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            if (HA) accA[r][j] = fma(v[u][r], ca, accA[r][j]);
            if (HB) accB[r][j] = fma(v[u][r], cb, accB[r][j]);
          }
        }
      }
    }
    for (; c < kp; ++c) {
      double v[RPT];
      const double* ptr = qcol + (size_t)c * p.ldq;
      if (RPT == 2) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(ptr));
        v[0] = t.x;
        v[RPT - 1] = t.y;
      } else {
        v[0] = __ldg(ptr);
      }
      const double* cr = coef + c * 2 * S;
#pragma unroll
      for (int j = 0; j < S; ++j)
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          if (HA) accA[r][j] = fma(v[r], cr[j], accA[r][j]);
          if (HB) accB[r][j] = fma(v[r], cr[S + j], accB[r][j]);
        }
    }

#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const long row = r0 + r;
      if (row >= p.n_rows) break;
      double a[S];
      if (HA) {
        // A = (srcA - acc) * TA^{-1}: back-substitution along the row (tri_solve_right)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          double t = (j < s ? p.srcA[row + (size_t)j * p.ld_srcA] : 0.0) - accA[r][j];
#pragma unroll
          for (int l = 0; l < j; ++l) t -= a[l] * ta[l + j * S];
          a[j] = t / ta[j + j * S];
        }
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j < s) p.dstA[row + (size_t)j * p.ld_dstA] = a[j];
      }
      if (HB) {
        double b[S];
#pragma unroll
        for (int j = 0; j < S; ++j) {
          double t = (j < s ? p.srcB[row + (size_t)j * p.ld_srcB] : 0.0) - accB[r][j];
          if (HA && p.cb_has_a) {
#pragma unroll
            for (int l = 0; l < S; ++l) t -= a[l] * cbx[l + j * S];
          }
#pragma unroll
          for (int l = 0; l < j; ++l) t -= b[l] * tb[l + j * S];
          b[j] = t / tb[j + j * S];
        }
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j < s) p.dstB[row + (size_t)j * p.ld_dstB] = b[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// S = 8 / 16: the same update on the fp64 tensor core.  Per row and prefix column K2 does
// 2S FMAs; at S >= 8 that bounds it on the scalar FP64 pipe (2.5 TB/s at s = 8, 1.5 at
// s = 16).  Here a warp owns 32 rows (4 m-tiles of 8) and walks the prefix in k-steps of
// 4 columns: A fragments straight from global memory (lane (i, kk) loads row 8q + i of
// column 4j + kk: 64-byte runs, each 128-byte line shared by two m-tiles), B fragments
// (the coefficients) from shared memory in fragment order, D = Qp [CA | CB] in
// 4 x (2S / 8) DMMA.8x8x4 accumulators.  The epilogue stages D through shared memory so
// that lane r owns row r and runs the same row-wise back-substitution as K2.
// ---------------------------------------------------------------------------------
namespace {
constexpr int kTcWarps = 8;
constexpr int kPf = 4;  // k-steps of A fragments in flight per warp
}

template <int S, bool HA, bool HB>
__global__ void __launch_bounds__(32 * kTcWarps) update_tc_kernel(const UpdateParams p) {
  if (p.status && status_bad(p.status)) return;
  constexpr int NT = 2 * S / 8;  // n-tiles of [CA | CB]
  extern __shared__ __align__(16) double sm[];
  const int kp = p.kp, s = p.s;
  const int ksteps = (kp + 3) / 4;
  double* coefB = sm;                                   // [kstep][NT][32 lanes]
  double* ta = coefB + (size_t)ksteps * NT * 32;        // S x S
  double* tb = ta + S * S;
  double* cbx = tb + S * S;
  double* rdg = cbx + S * S;                            // 1 / diag(TA), 1 / diag(TB)
  double* dst = rdg + 2 * S;                            // [warp][32 rows][2S + 1]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ii = lane >> 2, kk = lane & 3;
  // coefficient fragments: lane (i, kk) of n-tile t, k-step j holds C[4j + kk][8t + i]
  for (int idx = threadIdx.x; idx < ksteps * NT * 32; idx += blockDim.x) {
    const int l = idx & 31, t = (idx >> 5) % NT, j = (idx >> 5) / NT;
    const int c = 4 * j + (l & 3), n = 8 * t + (l >> 2);
    double v = 0.0;
    if (c < kp) {
      if (n < S) {
        if (HA && n < s) v = p.CA[c + (size_t)n * p.ldca];
      } else if (HB && n - S < s) {
        v = p.CB[c + (size_t)(n - S) * p.ldcb];
      }
    }
    coefB[idx] = v;
  }
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx % S, j = idx / S;
    const bool in = i < s && j < s;
    ta[idx] = (HA && p.TA && in) ? p.TA[i + (size_t)j * p.ldta] : (i == j ? 1.0 : 0.0);
    tb[idx] = (HB && p.TB && in) ? p.TB[i + (size_t)j * p.ldtb] : (i == j ? 1.0 : 0.0);
    cbx[idx] = (HA && HB && p.cb_has_a && in) ? p.CB[kp + i + (size_t)j * p.ldcb] : 0.0;
  }
  __syncthreads();
  // The row epilogue multiplies by reciprocals of the diagonals: S (or 2S) dependent fp64
  // divisions per row would cost as much as the contraction here (K12c likewise applies
  // explicit triangular inverses; both stay within the parity tolerances).
  if (threadIdx.x < 2 * S) {
    const int j = threadIdx.x % S;
    rdg[threadIdx.x] = 1.0 / (threadIdx.x < S ? ta[j + j * S] : tb[j + j * S]);
  }
  __syncthreads();
  double* dw = dst + (size_t)warp * 32 * (2 * S + 1);
  const long nchunks = (p.n_rows + 31) / 32;
  const long last_row = p.n_rows - 1;
  for (long ch = blockIdx.x * (long)kTcWarps + warp; ch < nchunks; ch += (long)gridDim.x * kTcWarps) {
    const long r0 = ch * 32;
    double acc[4][NT][2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < NT; ++t) acc[q][t][0] = acc[q][t][1] = 0.0;
    // lane (ii, kk): rows r0 + 8q + ii (clamped into the shard), column 4j + kk (clamped
    // into the prefix: past kp the coefficients are zero)
    const double* rowp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rowp[q] = p.qp + min(r0 + 8 * q + ii, last_row);
    const double* cf = coefB + lane;
    // A fragments of kPf k-steps in flight per lane (kPf x 1 KB per warp): the loop is
    // bound by HBM latency x bytes in flight, not by the DMMAs
    double a[kPf][4];
    auto load_a = [&](int j, double (&v)[4]) {
      const size_t col = (size_t)min(4 * j + kk, kp - 1) * p.ldq;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldg(rowp[q] + col);
    };
#pragma unroll
    for (int u = 0; u < kPf; ++u)
      if (u < ksteps) load_a(u, a[u]);
    for (int j0 = 0; j0 < ksteps; j0 += kPf) {
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        const int j = j0 + u;
        if (j < ksteps) {  // warp-uniform
          double b[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) b[t] = cf[(j * NT + t) * 32];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma(acc[q][t][0], acc[q][t][1], a[u][q], b[t]);
          if (j + kPf < ksteps) load_a(j + kPf, a[u]);
        }
      }
    }
    // D[8q + ii][8t + 2kk + e] -> row-major scratch; then lane r owns row r0 + r
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) dw[(8 * q + ii) * (2 * S + 1) + 8 * t + 2 * kk + e] = acc[q][t][e];
    __syncwarp();
    const long row = r0 + lane;
    if (row <= last_row) {
      const double* dr = dw + lane * (2 * S + 1);
      double a[S];
      if (HA) {
        // A = (srcA - D_A) * TA^{-1}: back-substitution along the row (tri_solve_right)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          double t = (j < s ? p.srcA[row + (size_t)j * p.ld_srcA] : 0.0) - dr[j];
#pragma unroll
          for (int l = 0; l < j; ++l) t -= a[l] * ta[l + j * S];
          a[j] = t * rdg[j];
        }
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j < s) p.dstA[row + (size_t)j * p.ld_dstA] = a[j];
      }
      if (HB) {
        double b[S];
#pragma unroll
        for (int j = 0; j < S; ++j) {
          double t = (j < s ? p.srcB[row + (size_t)j * p.ld_srcB] : 0.0) - dr[S + j];
          if (HA && p.cb_has_a) {
#pragma unroll
            for (int l = 0; l < S; ++l) t -= a[l] * cbx[l + j * S];
          }
#pragma unroll
          for (int l = 0; l < j; ++l) t -= b[l] * tb[l + j * S];
          b[j] = t * rdg[S + j];
        }
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j < s) p.dstB[row + (size_t)j * p.ld_dstB] = b[j];
      }
    }
  }
}

template <int S>
static size_t tc_smem(int kp) {
  return ((size_t)((kp + 3) / 4) * (2 * S / 8) * 32 + 3 * S * S + 2 * S +
          (size_t)kTcWarps * 32 * (2 * S + 1)) * sizeof(double) + 16;
}

template <int S>
static cudaError_t launch_tc(const UpdateParams& p, int num_sms, cudaStream_t st) {
  const size_t smem = tc_smem<S>(p.kp);
  int per_sm = (int)(220 * 1024 / smem);
  per_sm = per_sm < 1 ? 1 : per_sm > 4 ? 4 : per_sm;
  const long chunks = (p.n_rows + 31) / 32;
  long grid = (chunks + kTcWarps - 1) / kTcWarps;
  if (grid > (long)num_sms * per_sm) grid = (long)num_sms * per_sm;
  if (grid < 1) grid = 1;
  cudaError_t e = cudaSuccess;
  if (p.has_a && p.has_b) {
    auto k = update_tc_kernel<S, true, true>;
    if ((e = ensure_smem(k, smem)) != cudaSuccess) return e;
    k<<<(int)grid, 32 * kTcWarps, smem, st>>>(p);
  } else if (p.has_a) {
    auto k = update_tc_kernel<S, true, false>;
    if ((e = ensure_smem(k, smem)) != cudaSuccess) return e;
    k<<<(int)grid, 32 * kTcWarps, smem, st>>>(p);
  } else if (p.has_b) {
    auto k = update_tc_kernel<S, false, true>;
    if ((e = ensure_smem(k, smem)) != cudaSuccess) return e;
    k<<<(int)grid, 32 * kTcWarps, smem, st>>>(p);
  } else {
    return cudaSuccess;
  }
  return cudaGetLastError();
}

template <int S, int RPT>
static cudaError_t launch_s(const UpdateParams& p, int grid, size_t smem, cudaStream_t st) {
  const bool ha = p.has_a, hb = p.has_b;
  if (ha && hb) {
    auto k = update_kernel<S, RPT, true, true>;
    ensure_smem(k, smem);
    k<<<grid, 256, smem, st>>>(p);
  } else if (ha) {
    auto k = update_kernel<S, RPT, true, false>;
    ensure_smem(k, smem);
    k<<<grid, 256, smem, st>>>(p);
  } else if (hb) {
    auto k = update_kernel<S, RPT, false, true>;
    ensure_smem(k, smem);
    k<<<grid, 256, smem, st>>>(p);
  } else {
    return cudaSuccess;
  }
  return cudaGetLastError();
}

// Longest prefix one launch can take (the coefficient panel lives in shared memory); the
// runtime splits longer prefixes into chained launches (Runner::update).
int update_max_kp(int s) {
  const int S = s <= 1 ? 1 : s <= 2 ? 2 : s <= 4 ? 4 : s <= 8 ? 8 : 16;
  int best = 0;
  for (int kp = 4; kp <= 8192; kp += 4) {
    const bool tc = S >= 8 && (S == 8 ? tc_smem<8>(kp) : tc_smem<16>(kp)) <= 220 * 1024;
    const bool sc = ((size_t)kp * 2 * S + 3 * S * S) * sizeof(double) + 16 <= 200 * 1024;
    if (tc || sc) best = kp;
    else break;
  }
  return best;
}

cudaError_t update_launch(const UpdateParams& p, int num_sms, cudaStream_t st, int* launches) {
  const int s = p.s;
  const int S = s <= 1 ? 1 : s <= 2 ? 2 : s <= 4 ? 4 : s <= 8 ? 8 : 16;
  if (s < 1 || s > 16) return cudaErrorInvalidValue;
  static const bool scalar_only = getenv("BGS_K2_SCALAR") != nullptr;  // A/B experiments
  if (S >= 8 && p.kp >= 1 && !scalar_only) {  // fp64 tensor-core path
    const size_t need = S == 8 ? tc_smem<8>(p.kp) : tc_smem<16>(p.kp);
    if (need <= 220 * 1024) {
      if (launches) *launches += 1;
      return S == 8 ? launch_tc<8>(p, num_sms, st) : launch_tc<16>(p, num_sms, st);
    }
  }
  const size_t smem = ((size_t)p.kp * 2 * S + 3 * S * S) * sizeof(double) + 16;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  const int rpt = S <= 4 ? 2 : 1;
  const long groups = (p.n_rows + rpt - 1) / rpt;
  long grid = (groups + 255) / 256;
  const long cap = (long)num_sms * (smem > 64 * 1024 ? 2 : 4);
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (launches) *launches += 1;
  switch (S) {
    case 1: return launch_s<1, 2>(p, (int)grid, smem, st);
    case 2: return launch_s<2, 2>(p, (int)grid, smem, st);
    case 4: return launch_s<4, 2>(p, (int)grid, smem, st);
    case 8: return launch_s<8, 1>(p, (int)grid, smem, st);
    case 16: return launch_s<16, 1>(p, (int)grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bgs
