// tsqr.cu — K4: communication-avoiding TSQR of a tall n x s block on the device.
//
// Replaces run_tsqr / factor_local_leaves / plan_leaves (intraorth.cpp:27-111),
// householder_qr (dense_kernels.cpp:135-203), combine_leaf_factors / propagate_tree
// (tsqr_tree.cpp:14-78) and the tree half of tsqr_leaf_reduce (communicator.cpp:252-317).
//
//  leaf kernel : one CTA per row leaf (<= 1024 rows); Householder QR in shared memory with
//                the reference's scaled-norm reflector and nonnegative-diagonal sign fix;
//                writes the explicit leaf Q in place and the leaf R (s x s).
//  up kernel   : one CTA per shard tree; levels of pairwise QRs of stacked 2s x s R
//                factors, one warp per pair (lanes = rows); node Q factors kept.
//  cross kernel: the tree over the per-rank roots (after an NCCL allgather on a
//                multi-GPU context); identical inputs -> bitwise identical on every rank.
//  down kernel : pushes the root's M down the tree: M_leaf with Q_global = Q_leaf M_leaf.
//  apply kernel: Q rows of each leaf <- Q rows * M_leaf.
// Every factor is carried as s x s (zero-padded rows for short leaves, which stack as
// no-ops exactly like the reference's trapezoidal factors).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {

constexpr int SMAX = 16;
constexpr int kLeafThreads = 256;

// ---------------------------------------------------------------------------------
// CTA reductions (deterministic order)
// ---------------------------------------------------------------------------------
__device__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sums nv (<= SMAX) per-thread values over the CTA; result broadcast in out[0..nv).
__device__ void cta_sum_multi(double* v, int nv, double* scratch /*[8][SMAX]*/, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 0; i < nv; ++i) {
    const double r = warp_sum(v[i]);
    if (lane == 0) scratch[warp * SMAX + i] = r;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double acc = 0.0;
    for (int w = 0; w < kLeafThreads / 32; ++w) acc += scratch[w * SMAX + threadIdx.x];
    out[threadIdx.x] = acc;
  }
  __syncthreads();
}

__device__ double cta_max(double v, double* scratch, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double r = warp_max(v);
  if (lane == 0) scratch[warp] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < kLeafThreads / 32; ++w) m = fmax(m, scratch[w]);
    out[0] = m;
  }
  __syncthreads();
  return out[0];
}

}  // namespace

// ---------------------------------------------------------------------------------
// Leaf Householder QR
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(kLeafThreads)
    tsqr_leaf_kernel(const double* __restrict__ src, long lds, double* __restrict__ dst,
                     long ldd, const long* __restrict__ leaf_row0, int s,
                     double* __restrict__ rleaf, const DevStatus* status) {
  if (status && status_bad(status)) return;
  extern __shared__ __align__(16) double sm[];
  const int l = blockIdx.x;
  const long g0 = leaf_row0[l];
  const int h = (int)(leaf_row0[l + 1] - g0);
  double* A = sm;                    // h x s (V below the diagonal after the sweep)
  double* Q = A + (size_t)h * s;     // h x s
  __shared__ double scratch[8 * SMAX];
  __shared__ double red[SMAX];
  __shared__ double v0s[SMAX], taus[SMAX], rdiag[SMAX], rup[SMAX * SMAX];
  const int tid = threadIdx.x;
  const int p = h < s ? h : s;

  for (int j = 0; j < s; ++j)
    for (int i = tid; i < h; i += kLeafThreads) A[i + j * h] = src[g0 + i + (size_t)j * lds];
  __syncthreads();

  for (int k = 0; k < p; ++k) {
    double lm = 0.0;
    for (int i = k + tid; i < h; i += kLeafThreads) lm = fmax(lm, fabs(A[i + k * h]));
    const double mx = cta_max(lm, scratch, red);
    if (mx == 0.0) {
      if (tid == 0) { taus[k] = 0.0; v0s[k] = 0.0; rdiag[k] = A[k + k * h]; }
      __syncthreads();
      continue;
    }
    // scaled sum of squares of a(k:h, k) and plain sum of squares of a(k+1:h, k)
    double v2[2] = {0.0, 0.0};
    for (int i = k + tid; i < h; i += kLeafThreads) {
      const double a = A[i + k * h];
      const double t = a / mx;
      v2[0] = fma(t, t, v2[0]);
      if (i > k) v2[1] = fma(a, a, v2[1]);
    }
    cta_sum_multi(v2, 2, scratch, red);
    const double sigma = mx * sqrt(red[0]);
    const double akk = A[k + k * h];
    const double alpha = akk >= 0.0 ? -sigma : sigma;
    const double v0 = akk - alpha;
    const double vtv = v0 * v0 + red[1];
    const double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    // w_j = tau * (v0 a(k,j) + sum_{i>k} v_i a(i,j)),  j > k
    double w[SMAX];
    const int nj = s - k - 1;
    for (int j = 0; j < nj; ++j) w[j] = 0.0;
    for (int i = k + 1 + tid; i < h; i += kLeafThreads) {
      const double vi = A[i + k * h];
      for (int j = 0; j < nj; ++j) w[j] = fma(vi, A[i + (k + 1 + j) * h], w[j]);
    }
    __syncthreads();
    cta_sum_multi(w, nj, scratch, red);
    for (int j = 0; j < nj; ++j) {
      const double wj = tau * fma(v0, A[k + (k + 1 + j) * h], red[j]);
      for (int i = k + 1 + tid; i < h; i += kLeafThreads)
        A[i + (k + 1 + j) * h] -= wj * A[i + k * h];
      w[j] = wj;
    }
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < nj; ++j) A[k + (k + 1 + j) * h] -= w[j] * v0;
      v0s[k] = v0;
      taus[k] = tau;
      rdiag[k] = alpha;
    }
    __syncthreads();
  }
  // R (s x s, zero padded) before the sign fix
  if (tid < s * s) {
    const int i = tid % s, j = tid / s;
    double v = 0.0;
    if (i < p && i <= j) v = (i == j) ? rdiag[i] : A[i + j * h];
    rup[tid] = v;
  }
  // Q = H_0 ... H_{p-1} [I; 0]
  for (int j = 0; j < s; ++j)
    for (int i = tid; i < h; i += kLeafThreads) Q[i + j * h] = (i == j && j < p) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = p - 1; k >= 0; --k) {
    const double tau = taus[k];
    if (tau == 0.0) continue;
    const double v0 = v0s[k];
    double w[SMAX];
    for (int j = 0; j < p; ++j) w[j] = 0.0;
    for (int i = k + 1 + tid; i < h; i += kLeafThreads) {
      const double vi = A[i + k * h];
      for (int j = 0; j < p; ++j) w[j] = fma(vi, Q[i + j * h], w[j]);
    }
    cta_sum_multi(w, p, scratch, red);
    for (int j = 0; j < p; ++j) w[j] = tau * fma(v0, Q[k + j * h], red[j]);
    for (int i = k + 1 + tid; i < h; i += kLeafThreads) {
      const double vi = A[i + k * h];
      for (int j = 0; j < p; ++j) Q[i + j * h] -= w[j] * vi;
    }
    __syncthreads();
    if (tid == 0)
      for (int j = 0; j < p; ++j) Q[k + j * h] -= w[j] * v0;
    __syncthreads();
  }
  // canonical sign: nonnegative diag(R)
  __shared__ double sgn[SMAX];
  if (tid < s) sgn[tid] = (tid < p && rup[tid + tid * s] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  if (tid < s * s) {
    const int i = tid % s;
    rleaf[(size_t)l * s * s + tid] = sgn[i] * rup[tid];
  }
  for (int j = 0; j < s; ++j)
    for (int i = tid; i < h; i += kLeafThreads) dst[g0 + i + (size_t)j * ldd] = sgn[j] * Q[i + j * h];
}

// ---------------------------------------------------------------------------------
// Register-resident leaf Householder QR for s in {1, 2, 4, 8, 16}: thread t owns rows
// t + 256 r (r < RPT) of the leaf; the reflector arithmetic is the generic kernel's
// (scaled norm, alpha = -sign(a_kk) sigma, tau = 2 / v^T v, explicit Q by backward
// accumulation, nonnegative-diagonal sign fix); only the row-to-thread assignment of the
// partial sums differs.
// ---------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void cta_sum_t(double (&v)[NV], double* scratch /*[8][SMAX]*/,
                                          double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double r = warp_sum(v[i]);
    if (lane == 0) scratch[warp * SMAX + i] = r;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double acc = 0.0;
    for (int w = 0; w < kLeafThreads / 32; ++w) acc += scratch[w * SMAX + threadIdx.x];
    out[threadIdx.x] = acc;
  }
  __syncthreads();
}

template <int S, int RPT>
__global__ void __launch_bounds__(kLeafThreads, S <= 8 ? 3 : 2)  // 3 leaves per SM for s <= 8, else 2
    tsqr_leaf_reg_kernel(const double* __restrict__ src, long lds, double* __restrict__ dst,
                         long ldd, const long* __restrict__ leaf_row0,
                         double* __restrict__ rleaf, const DevStatus* status) {
  if (status && status_bad(status)) return;
  __shared__ double scratch[8 * SMAX];
  __shared__ double red[SMAX];
  __shared__ double top[S];  // row k of the working matrix (A during the sweep, Q after)
  __shared__ double v0s[S], taus[S], rdiag[S], rup[S * S];
  const int tid = threadIdx.x;
  const int l = blockIdx.x;
  const long g0 = leaf_row0[l];
  const int h = (int)(leaf_row0[l + 1] - g0);
  const int p = h < S ? h : S;
  double a[RPT][S];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = tid + r * kLeafThreads;
#pragma unroll
    for (int j = 0; j < S; ++j) a[r][j] = i < h ? src[g0 + i + (size_t)j * lds] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < S; ++k) {
    if (k >= p) break;
    // owner of row k publishes it (current values) for the top-row terms
    if ((k & (kLeafThreads - 1)) == tid)
#pragma unroll
      for (int j = 0; j < S; ++j) top[j] = a[k / kLeafThreads][j];
    double lm = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i >= k && i < h) lm = fmax(lm, fabs(a[r][k]));
    }
    const double mx = cta_max(lm, scratch, red);  // (its barriers also publish top[])
    if (mx == 0.0) {
      if (tid == 0) { taus[k] = 0.0; v0s[k] = 0.0; rdiag[k] = top[k]; }
      __syncthreads();
      continue;
    }
    double v2[2] = {0.0, 0.0};
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i >= k && i < h) {
        const double t = a[r][k] / mx;
        v2[0] = fma(t, t, v2[0]);
        if (i > k) v2[1] = fma(a[r][k], a[r][k], v2[1]);
      }
    }
    cta_sum_t<2>(v2, scratch, red);
    const double sigma = mx * sqrt(red[0]);
    const double akk = top[k];
    const double alpha = akk >= 0.0 ? -sigma : sigma;
    const double v0 = akk - alpha;
    const double vtv = v0 * v0 + red[1];
    const double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    __syncthreads();  // red[] is reused below
    // w_j = tau (v0 a(k, j) + sum_{i > k} v_i a(i, j)), j > k
    double w[S];
#pragma unroll
    for (int j = 0; j < S; ++j) w[j] = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i > k && i < h)
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j > k) w[j] = fma(a[r][k], a[r][j], w[j]);
    }
    cta_sum_t<S>(w, scratch, red);
#pragma unroll
    for (int j = 0; j < S; ++j) w[j] = j > k ? tau * fma(v0, top[j], red[j]) : 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i > k && i < h)
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j > k) a[r][j] -= w[j] * a[r][k];
      if (i == k)
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j > k) a[r][j] -= w[j] * v0;
    }
    if (tid == 0) {
      v0s[k] = v0;
      taus[k] = tau;
      rdiag[k] = alpha;
    }
    __syncthreads();
  }
  // R (before the sign fix): rows i < p of the swept matrix, diagonal = alpha
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = tid + r * kLeafThreads;
    if (i < S)
#pragma unroll
      for (int j = 0; j < S; ++j)
        rup[i + j * S] = (i < p && i <= j) ? (i == j ? rdiag[i] : a[r][j]) : 0.0;
  }
  // Q = H_0 ... H_{p-1} [I; 0], accumulated backwards in registers
  double q[RPT][S];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = tid + r * kLeafThreads;
#pragma unroll
    for (int j = 0; j < S; ++j) q[r][j] = (i == j && j < p) ? 1.0 : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = S - 1; k >= 0; --k) {
    if (k >= p) continue;
    const double tau = taus[k];
    if (tau == 0.0) continue;
    const double v0 = v0s[k];
    if ((k & (kLeafThreads - 1)) == tid)
#pragma unroll
      for (int j = 0; j < S; ++j) top[j] = q[k / kLeafThreads][j];
    double w[S];
#pragma unroll
    for (int j = 0; j < S; ++j) w[j] = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i > k && i < h)
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (j < p) w[j] = fma(a[r][k], q[r][j], w[j]);
    }
    cta_sum_t<S>(w, scratch, red);  // (its first barrier also publishes top[])
#pragma unroll
    for (int j = 0; j < S; ++j) w[j] = j < p ? tau * fma(v0, top[j], red[j]) : 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = tid + r * kLeafThreads;
      if (i > k && i < h)
#pragma unroll
        for (int j = 0; j < S; ++j) q[r][j] -= w[j] * a[r][k];
      if (i == k)
#pragma unroll
        for (int j = 0; j < S; ++j) q[r][j] -= w[j] * v0;
    }
    __syncthreads();
  }
  // canonical sign: nonnegative diag(R)
  double sg[S];
#pragma unroll
  for (int j = 0; j < S; ++j) sg[j] = (j < p && rup[j + j * S] < 0.0) ? -1.0 : 1.0;
  if (tid < S * S) rleaf[(size_t)l * S * S + tid] = sg[tid % S] * rup[tid];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = tid + r * kLeafThreads;
    if (i < h)
#pragma unroll
      for (int j = 0; j < S; ++j) dst[g0 + i + (size_t)j * ldd] = sg[j] * q[r][j];
  }
}

// ---------------------------------------------------------------------------------
// Pairwise QR of two stacked s x s factors, one warp: lane i < 2s owns row i.
// q (2s x s, col-major) and r (s x s) written to global/shared.
// ---------------------------------------------------------------------------------
__device__ void warp_pair_qr(const double* top, const double* bot, int s, double* qout,
                             double* rout) {
  const int lane = threadIdx.x & 31;
  const int m = 2 * s;
  double a[SMAX];
  for (int j = 0; j < s; ++j)
    a[j] = lane < s ? top[lane + j * s] : (lane < m ? bot[(lane - s) + j * s] : 0.0);
  double vs[SMAX], taus[SMAX], rd[SMAX];
  for (int k = 0; k < s; ++k) {
    const double mine = (lane >= k && lane < m) ? a[k] : 0.0;
    const double mx = warp_max(fabs(mine));
    if (mx == 0.0) {
      taus[k] = 0.0; vs[k] = 0.0;
      rd[k] = __shfl_sync(0xffffffffu, a[k], k);
      continue;
    }
    const double t = mine / mx;
    const double ssq = warp_sum(t * t);
    const double below = warp_sum(lane > k ? mine * mine : 0.0);
    const double sigma = mx * sqrt(ssq);
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    const double alpha = akk >= 0.0 ? -sigma : sigma;
    const double v0 = akk - alpha;
    const double vtv = v0 * v0 + below;
    const double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    const double vi = lane == k ? v0 : (lane > k && lane < m ? a[k] : 0.0);
    for (int j = k + 1; j < s; ++j) {
      const double wj = tau * warp_sum(vi * a[j]);
      a[j] -= wj * vi;
    }
    vs[k] = vi;
    taus[k] = tau;
    rd[k] = alpha;
  }
  // R rows (lane i < s): a[j] for j > i, rd[i] on the diagonal
  double q[SMAX];
  for (int j = 0; j < s; ++j) q[j] = (lane == j) ? 1.0 : 0.0;
  for (int k = s - 1; k >= 0; --k) {
    if (taus[k] == 0.0) continue;
    for (int j = 0; j < s; ++j) {
      const double wj = taus[k] * warp_sum(vs[k] * q[j]);
      q[j] -= wj * vs[k];
    }
  }
  // sign fix: lane j knows whether R(j,j) < 0
  for (int j = 0; j < s; ++j) {
    const double d = rd[j];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    if (lane < m) qout[lane + j * m] = sg * q[j];
    if (lane == j) {
      for (int jj = 0; jj < s; ++jj) {
        double v = 0.0;
        if (jj == j) v = d;
        else if (jj > j) v = a[jj];
        rout[j + jj * s] = sg * v;
      }
    } else if (lane > j && lane < s) {
      rout[lane + j * s] = 0.0;
    }
  }
}

// The same pair QR with s a template parameter: rows and reflectors in registers, and
// reductions over the 2s active lanes only (log2 steps; the skipped xor steps would add
// exact zeros from the idle lanes, so the results are bit-identical to warp_pair_qr).
template <int S>
BGS_DEV double lane_sum(double v) {
  constexpr int W = 2 * S >= 32 ? 32 : (2 * S >= 16 ? 16 : (2 * S >= 8 ? 8 : (2 * S >= 4 ? 4 : 2)));
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);  // warp-uniform (lanes >= W reduced only zeros)
}
template <int S>
BGS_DEV double lane_max(double v) {
  constexpr int W = 2 * S >= 32 ? 32 : (2 * S >= 16 ? 16 : (2 * S >= 8 ? 8 : (2 * S >= 4 ? 4 : 2)));
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return __shfl_sync(0xffffffffu, v, 0);  // warp-uniform: every lane takes the same branches
}

template <int S>
__device__ void warp_pair_qr_t(const double* top, const double* bot, double* qout, double* rout) {
  const int lane = threadIdx.x & 31;
  constexpr int m = 2 * S;
  double a[S];
#pragma unroll
  for (int j = 0; j < S; ++j)
    a[j] = lane < S ? top[lane + j * S] : (lane < m ? bot[(lane - S) + j * S] : 0.0);
  double vs[S], taus[S], rd[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const double mine = (lane >= k && lane < m) ? a[k] : 0.0;
    const double mx = lane_max<S>(fabs(mine));
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    if (mx == 0.0) {
      taus[k] = 0.0; vs[k] = 0.0;
      rd[k] = akk;
      continue;
    }
    const double t = mine / mx;
    const double ssq = lane_sum<S>(t * t);
    const double below = lane_sum<S>(lane > k ? mine * mine : 0.0);
    const double sigma = mx * sqrt(ssq);
    const double alpha = akk >= 0.0 ? -sigma : sigma;
    const double v0 = akk - alpha;
    const double vtv = v0 * v0 + below;
    const double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    const double vi = lane == k ? v0 : (lane > k && lane < m ? a[k] : 0.0);
#pragma unroll
    for (int j = k + 1; j < S; ++j) {
      const double wj = tau * lane_sum<S>(vi * a[j]);
      a[j] -= wj * vi;
    }
    vs[k] = vi;
    taus[k] = tau;
    rd[k] = alpha;
  }
  double q[S];
#pragma unroll
  for (int j = 0; j < S; ++j) q[j] = (lane == j) ? 1.0 : 0.0;
#pragma unroll
  for (int k = S - 1; k >= 0; --k) {
    if (taus[k] == 0.0) continue;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double wj = taus[k] * lane_sum<S>(vs[k] * q[j]);
      q[j] -= wj * vs[k];
    }
  }
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const double d = rd[j];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    if (lane < m) qout[lane + j * m] = sg * q[j];
    if (lane == j) {
#pragma unroll
      for (int jj = 0; jj < S; ++jj) {
        double v = 0.0;
        if (jj == j) v = d;
        else if (jj > j) v = a[jj];
        rout[j + jj * S] = sg * v;
      }
    } else if (lane > j && lane < S) {
      rout[lane + j * S] = 0.0;
    }
  }
}

// C = A(s x s, lda) * B(s x s); one warp.
__device__ void warp_mm(const double* A, int lda, const double* B, int s, double* C) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < s * s; e += 32) {
    const int i = e % s, j = e / s;
    double acc = 0.0;
    for (int k = 0; k < s; ++k) acc = fma(A[i + k * lda], B[k + j * s], acc);
    C[e] = acc;
  }
}

// Workspace layout per leaf index: [R | Rtmp | M | Mtmp] (s*s each) + nodeQ (2s*s)
struct TreeWs {
  double *R, *Rt, *M, *Mt, *NQ;
};
__device__ TreeWs tree_ws(double* ws, int L, int s) {
  const size_t ss = (size_t)s * s;
  TreeWs t;
  t.R = ws;
  t.Rt = ws + L * ss;
  t.M = ws + 2 * L * ss;
  t.Mt = ws + 3 * L * ss;
  t.NQ = ws + 4 * L * ss;
  return t;
}

// Bottom-up over items [off, off + c) of the workspace; root -> root_out (ld lr).
__device__ void tree_up(TreeWs w, int off, int c, int s, double* root_out, int lr) {
  const size_t ss = (size_t)s * s;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* cur = w.R + off * ss;
  double* nxt = w.Rt + off * ss;
  int node = off;
  int cnt = c;
  while (cnt > 1) {
    const int np = cnt / 2;
    for (int i = warp; i < np; i += nw)
      warp_pair_qr(cur + 2 * i * ss, cur + (2 * i + 1) * ss, s, w.NQ + (size_t)(node + i) * 2 * ss,
                   nxt + i * ss);
    if (cnt & 1)
      for (int e = threadIdx.x; e < (int)ss; e += blockDim.x) nxt[np * ss + e] = cur[(cnt - 1) * ss + e];
    __syncthreads();
    node += np;
    cnt = np + (cnt & 1);
    double* t = cur; cur = nxt; nxt = t;
  }
  for (int e = threadIdx.x; e < (int)ss; e += blockDim.x) root_out[(e % s) + (e / s) * lr] = cur[e];
  __syncthreads();
}

// Top-down: leaf M's into w.M[off .. off+c)
__device__ void tree_down(TreeWs w, int off, int c, int s, const double* mtop) {
  const size_t ss = (size_t)s * s;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int cnts[40], bases[40];
  int nl = 0, cnt = c, node = off;
  while (cnt > 1) {
    cnts[nl] = cnt;
    bases[nl] = node;
    node += cnt / 2;
    cnt = cnt / 2 + (cnt & 1);
    ++nl;
  }
  // the buffer that must end up holding level 0 is w.M; alternate backwards
  double* bufs[2] = {w.M + off * ss, w.Mt + off * ss};
  int top_buf = nl & 1;  // level l lives in bufs[l & 1]; level nl (root) in bufs[nl & 1]
  double* root = bufs[top_buf];
  for (int e = threadIdx.x; e < (int)ss; e += blockDim.x)
    root[e] = mtop ? mtop[e] : ((e % s) == (e / s) ? 1.0 : 0.0);
  __syncthreads();
  for (int lv = nl - 1; lv >= 0; --lv) {
    double* par = bufs[(lv + 1) & 1];
    double* chi = bufs[lv & 1];
    const int cn = cnts[lv], np = cn / 2;
    for (int i = warp; i < np; i += nw) {
      const double* qn = w.NQ + (size_t)(bases[lv] + i) * 2 * ss;
      warp_mm(qn, 2 * s, par + i * ss, s, chi + 2 * i * ss);
      warp_mm(qn + s, 2 * s, par + i * ss, s, chi + (2 * i + 1) * ss);
    }
    if (cn & 1)
      for (int e = threadIdx.x; e < (int)ss; e += blockDim.x) chi[(cn - 1) * ss + e] = par[np * ss + e];
    __syncthreads();
  }
}

__global__ void tsqr_cross_kernel(const double* roots, int n, int s, double* ws2, double* rout,
                                  int ldr, double* mout, const DevStatus* status) {
  if (status && status_bad(status)) return;
  TreeWs w = tree_ws(ws2, n, s);
  const size_t ss = (size_t)s * s;
  for (int e = threadIdx.x; e < (int)(n * ss); e += blockDim.x) w.R[e] = roots[e];
  __syncthreads();
  tree_up(w, 0, n, s, rout, ldr);
  if (mout) {
    tree_down(w, 0, n, s, nullptr);
    for (int e = threadIdx.x; e < (int)(n * ss); e += blockDim.x) mout[e] = w.M[e];
  }
}

__global__ void tsqr_apply_kernel(double* dst, long ldd, const long* leaf_row0, const double* M,
                                  int s, const DevStatus* status) {
  if (status && status_bad(status)) return;
  __shared__ double m[SMAX * SMAX];
  const int l = blockIdx.x;
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) m[e] = M[(size_t)l * s * s + e];
  __syncthreads();
  const long g0 = leaf_row0[l], g1 = leaf_row0[l + 1];
  for (long i = g0 + threadIdx.x; i < g1; i += blockDim.x) {
    double row[SMAX];
    for (int j = 0; j < s; ++j) row[j] = dst[i + (size_t)j * ldd];
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int k = 0; k < s; ++k) acc = fma(row[k], m[k + j * s], acc);
      dst[i + (size_t)j * ldd] = acc;
    }
  }
}

// ---------------------------------------------------------------------------------
// Grouped tree levels.  The tree pairs items level by level (pairs (2i, 2i+1); an odd last
// item passes up), and pair i of level l is node nb[l] + i — the same numbering as
// tree_up / tree_down.  A CTA takes 2^D consecutive items of level l0 and runs D levels in
// shared memory (one warp per pair), so ~1000 leaves need two launches instead of one CTA
// walking ten levels with ~30 serial pair QRs per warp at the bottom.
// ---------------------------------------------------------------------------------
struct TreeGroupArgs {
  const double* in;   // level l0 items (up) / level l0 + D items (down), s x s each
  double* out;        // level l0 + D items (up) / level l0 items (down)
  double* nq;         // node Q factors of this tree (2s x s per node)
  int s, D;
  int cnt[9];         // item counts of levels l0 .. l0 + D
  int nb[8];          // node bases of levels l0 .. l0 + D - 1
  int identity_top;   // down: the top item is the identity (no M from above)
};

template <int S>  // S = 0: runtime s (generic pair QR)
// (S = 16: 256 threads so a warp's pair QR gets the registers it needs; 512 spilled)
__global__ void __launch_bounds__(S >= 16 ? 256 : 512) tsqr_up_group_kernel(const TreeGroupArgs a,
                                                            const DevStatus* status) {
  if (status && status_bad(status)) return;
  extern __shared__ double tsm[];
  const int s = a.s, D = a.D, ss = s * s;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* b0 = tsm;
  double* b1 = tsm + (size_t)(1 << D) * ss;
  const int g = blockIdx.x;
  const int lo = g << D, n0 = min(1 << D, a.cnt[0] - lo);
  for (int e = threadIdx.x; e < n0 * ss; e += blockDim.x) b0[e] = a.in[(size_t)lo * ss + e];
  __syncthreads();
  for (int d = 0; d < D; ++d) {
    const int lod = g << (D - d);
    const int nd = min(1 << (D - d), a.cnt[d] - lod);
    const int np = nd / 2;
    for (int i = warp; i < np; i += nw) {
      double* qo = a.nq + (size_t)(a.nb[d] + (lod >> 1) + i) * 2 * ss;
      if (S > 0)
        warp_pair_qr_t<S ? S : 1>(b0 + (size_t)2 * i * ss, b0 + (size_t)(2 * i + 1) * ss, qo,
                                  b1 + (size_t)i * ss);
      else
        warp_pair_qr(b0 + (size_t)2 * i * ss, b0 + (size_t)(2 * i + 1) * ss, s, qo,
                     b1 + (size_t)i * ss);
    }
    if (nd & 1)
      for (int e = threadIdx.x; e < ss; e += blockDim.x) b1[(size_t)np * ss + e] = b0[(size_t)(nd - 1) * ss + e];
    __syncthreads();
    double* t = b0; b0 = b1; b1 = t;
  }
  for (int e = threadIdx.x; e < ss; e += blockDim.x) a.out[(size_t)g * ss + e] = b0[e];
}

__global__ void __launch_bounds__(512) tsqr_down_group_kernel(const TreeGroupArgs a,
                                                              const DevStatus* status) {
  if (status && status_bad(status)) return;
  extern __shared__ double tsm[];
  const int s = a.s, D = a.D, ss = s * s;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* b0 = tsm;
  double* b1 = tsm + (size_t)(1 << D) * ss;
  const int g = blockIdx.x;
  for (int e = threadIdx.x; e < ss; e += blockDim.x)
    b0[e] = a.identity_top ? ((e % s) == (e / s) ? 1.0 : 0.0) : a.in[(size_t)g * ss + e];
  __syncthreads();
  for (int d = D - 1; d >= 0; --d) {
    const int lod = g << (D - d);
    const int nd = min(1 << (D - d), a.cnt[d] - lod);
    const int np = nd / 2;
    for (int i = warp; i < np; i += nw) {
      const double* qn = a.nq + (size_t)(a.nb[d] + (lod >> 1) + i) * 2 * ss;
      warp_mm(qn, 2 * s, b0 + (size_t)i * ss, s, b1 + (size_t)2 * i * ss);
      warp_mm(qn + s, 2 * s, b0 + (size_t)i * ss, s, b1 + (size_t)(2 * i + 1) * ss);
    }
    if (nd & 1)
      for (int e = threadIdx.x; e < ss; e += blockDim.x) b1[(size_t)(nd - 1) * ss + e] = b0[(size_t)np * ss + e];
    __syncthreads();
    double* t = b0; b0 = b1; b1 = t;
  }
  const int lo = g << D, n0 = min(1 << D, a.cnt[0] - lo);
  for (int e = threadIdx.x; e < n0 * ss; e += blockDim.x) a.out[(size_t)lo * ss + e] = b0[e];
}

namespace {
struct TreePlan {
  int nlev = 0;
  int cnt[40], nb[40];
  std::vector<std::pair<int, int>> launches;  // (l0, D), bottom-up
};
TreePlan tree_plan(int L, int s) {
  TreePlan t;
  int c = L, base = 0;
  while (true) {
    t.cnt[t.nlev] = c;
    t.nb[t.nlev] = base;
    ++t.nlev;
    if (c <= 1) break;
    base += c / 2;
    c = (c + 1) / 2;
  }
  const int dmax = s <= 8 ? 5 : 4;
  for (int l0 = 0; l0 < t.nlev - 1;) {
    const int D = std::min(dmax, t.nlev - 1 - l0);
    t.launches.push_back({l0, D});
    l0 += D;
  }
  return t;
}
TreeGroupArgs group_args(const TreePlan& t, int l0, int D, int s, double* nq) {
  TreeGroupArgs a;
  memset(&a, 0, sizeof a);
  a.s = s;
  a.D = D;
  a.nq = nq;
  for (int d = 0; d <= D; ++d) a.cnt[d] = t.cnt[l0 + d];
  for (int d = 0; d < D; ++d) a.nb[d] = t.nb[l0 + d];
  return a;
}
}  // namespace

// Bottom-up tree of one shard's leaves [leaf_base, leaf_base + Lt) (leaf R's already in
// the workspace); the shard root goes to root_out (s x s, ld s).
cudaError_t tsqr_tree_up_shard(double* ws, int L, int leaf_base, int Lt, int s, double* root_out,
                               const DevStatus* status, cudaStream_t st, int* launches) {
  const size_t ss = (size_t)s * s;
  double* R = ws + (size_t)leaf_base * ss;
  double* Rt = ws + (size_t)L * ss + (size_t)leaf_base * ss;
  double* nq = ws + (size_t)4 * L * ss + (size_t)leaf_base * 2 * ss;
  if (Lt <= 1)
    return cudaMemcpyAsync(root_out, R, ss * sizeof(double), cudaMemcpyDeviceToDevice, st);
  const TreePlan t = tree_plan(Lt, s);
  double* bufs[2] = {R, Rt};
  for (size_t j = 0; j < t.launches.size(); ++j) {
    const int l0 = t.launches[j].first, D = t.launches[j].second;
    TreeGroupArgs a = group_args(t, l0, D, s, nq);
    a.in = bufs[j & 1];
    a.out = j + 1 == t.launches.size() ? root_out : bufs[(j + 1) & 1];
    const int groups = (t.cnt[l0] + (1 << D) - 1) >> D;
    const size_t smem = (size_t)2 * (1 << D) * ss * sizeof(double);
    const int threads = std::min(s >= 16 ? 256 : 512, 32 * std::max(1, (1 << D) / 2));
    cudaError_t e = cudaSuccess;
#define BGS_UP_GROUP(S_)                                                        \
  {                                                                           \
    e = ensure_smem(tsqr_up_group_kernel<S_>, smem);                          \
    if (e != cudaSuccess) return e;                                           \
    tsqr_up_group_kernel<S_><<<groups, threads, smem, st>>>(a, status);       \
  }
    switch (s) {
      case 1: BGS_UP_GROUP(1) break;
      case 2: BGS_UP_GROUP(2) break;
      case 4: BGS_UP_GROUP(4) break;
      case 8: BGS_UP_GROUP(8) break;
      case 16: BGS_UP_GROUP(16) break;
      default: BGS_UP_GROUP(0) break;
    }
#undef BGS_UP_GROUP
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

__global__ void set_identity_kernel(double* M, int s) {
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) M[e] = (e % s == e / s) ? 1.0 : 0.0;
}

// Top-down: the shard root's M (mtop, or identity when null) to the leaf M's in the
// workspace's M region.
cudaError_t tsqr_tree_down_shard(double* ws, int L, int leaf_base, int Lt, int s,
                                 const double* mtop, const DevStatus* status, cudaStream_t st,
                                 int* launches) {
  const size_t ss = (size_t)s * s;
  double* M = ws + (size_t)2 * L * ss + (size_t)leaf_base * ss;
  double* Mt = ws + (size_t)3 * L * ss + (size_t)leaf_base * ss;
  double* nq = ws + (size_t)4 * L * ss + (size_t)leaf_base * 2 * ss;
  if (Lt <= 1) {
    if (mtop) return cudaMemcpyAsync(M, mtop, ss * sizeof(double), cudaMemcpyDeviceToDevice, st);
    // (a kernel, not an H2D copy of a host temporary: when the factorization is captured
    // into a CUDA graph the copy node would keep the pointer of a vector that is gone by
    // the time the graph runs -- wrong Q for every single-leaf shard on this path, i.e.
    // s not in {1, 2, 4, 8, 16}, found by the round-2 fuzz through bgs_factor_device)
    set_identity_kernel<<<1, 256, 0, st>>>(M, s);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const TreePlan t = tree_plan(Lt, s);
  const int K = (int)t.launches.size();
  double* bufs[2] = {M, Mt};  // launch j writes level l0_j into bufs[j & 1] (j = 0 -> M)
  for (int j = K - 1; j >= 0; --j) {
    const int l0 = t.launches[j].first, D = t.launches[j].second;
    TreeGroupArgs a = group_args(t, l0, D, s, nq);
    a.out = bufs[j & 1];
    if (j == K - 1) {
      a.in = mtop;
      a.identity_top = mtop ? 0 : 1;
    } else {
      a.in = bufs[(j + 1) & 1];
    }
    const int groups = (t.cnt[l0] + (1 << D) - 1) >> D;
    const size_t smem = (size_t)2 * (1 << D) * ss * sizeof(double);
    cudaError_t e = ensure_smem(tsqr_down_group_kernel, smem);
    if (e != cudaSuccess) return e;
    tsqr_down_group_kernel<<<groups, 32 * std::max(1, (1 << D) / 2), smem, st>>>(a, status);
    if (launches) *launches += 1;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Apply with the leaf's M computed on the fly (no top-down pass).  Leaf l's item index at
// level k is l >> k; it is a pass-through where it is the odd last item, else it is half
// (l >> k) & 1 of node nb[k] + (l >> (k + 1)).  M_leaf = H_0 H_1 ... H_{top-1} M_top with
// H_k that half of the node's 2s x s Q — the same products, in the same order, as
// tree_down's warp_mm, so the leaf M's are bit-identical to the top-down pass.
// ---------------------------------------------------------------------------------
struct TreePath {
  int nlev;
  int cnt[32];
  int nb[32];
};

template <int S>
__global__ void __launch_bounds__(256)
    tsqr_apply_path_kernel(double* __restrict__ dst, long ldd, const long* __restrict__ leaf_row0,
                           const double* __restrict__ nq, const double* __restrict__ mtop,
                           const TreePath tp, const DevStatus* status) {
  if (status && status_bad(status)) return;
  constexpr int SS = S * S;
  __shared__ double hq[S <= 8 ? 32 : 20][SS];  // (static shared memory <= 48 KB)
  __shared__ __align__(16) double mm[2][SS];
  const int l = blockIdx.x, tid = threadIdx.x;
  const int nh = tp.nlev - 1;  // levels with nodes below the root
  // every path factor at once (independent L2 reads); pass-throughs become identities
  for (int idx = tid; idx < nh * SS; idx += blockDim.x) {
    const int k = idx / SS, e = idx % SS, r = e % S, c = e / S;
    const int ik = l >> k;
    const bool pass = ik == tp.cnt[k] - 1 && (tp.cnt[k] & 1);
    double v;
    if (pass) {
      v = r == c ? 1.0 : 0.0;
    } else {
      const int node = tp.nb[k] + (ik >> 1), half = ik & 1;
      v = nq[(size_t)node * 2 * SS + (half * S + r) + (size_t)c * 2 * S];
    }
    hq[k][e] = v;
  }
  for (int e = tid; e < SS; e += blockDim.x)
    mm[0][e] = mtop ? mtop[e] : ((e % S) == (e / S) ? 1.0 : 0.0);
  __syncthreads();
  int cur = 0;
  if (tid < 32) {
    for (int k = nh - 1; k >= 0; --k) {
      const int ik = l >> k;
      if (ik == tp.cnt[k] - 1 && (tp.cnt[k] & 1)) continue;  // pass-through: M unchanged
      for (int e = tid; e < SS; e += 32) {
        const int i = e % S, j = e / S;
        double acc = 0.0;
        for (int q = 0; q < S; ++q) acc = fma(hq[k][i + q * S], mm[cur][q + j * S], acc);
        mm[cur ^ 1][e] = acc;
      }
      __syncwarp();
      cur ^= 1;
    }
  }
  __syncthreads();
  cur = __shfl_sync(0xffffffffu, cur, 0);  // (warp 0's value; every warp reads the same)
  __shared__ int cur_s;
  if (tid == 0) cur_s = cur;
  __syncthreads();
  const double* m = mm[cur_s];
  const long g0 = leaf_row0[l], g1 = leaf_row0[l + 1];
  if constexpr (S <= 8) {
    double mr[SS];
#pragma unroll
    for (int e = 0; e < SS; ++e) mr[e] = m[e];
    for (long i = g0 + tid; i < g1; i += blockDim.x) {
      double row[S];
#pragma unroll
      for (int j = 0; j < S; ++j) row[j] = dst[i + (size_t)j * ldd];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < S; ++k) acc = fma(row[k], mr[k + j * S], acc);
        dst[i + (size_t)j * ldd] = acc;
      }
    }
  } else {
    // S = 16: M (2 KB) stays in shared memory (broadcast reads, two entries per load); in
    // registers it spilled 1.8 KB per thread.  Same products in the same order.
    for (long i = g0 + tid; i < g1; i += blockDim.x) {
      double row[S];
#pragma unroll
      for (int j = 0; j < S; ++j) row[j] = dst[i + (size_t)j * ldd];
#pragma unroll 4
      for (int j = 0; j < S; ++j) {
        const double2* mc = reinterpret_cast<const double2*>(m + j * S);
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < S; k += 2) {
          const double2 t = mc[k / 2];
          acc = fma(row[k], t.x, acc);
          acc = fma(row[k + 1], t.y, acc);
        }
        dst[i + (size_t)j * ldd] = acc;
      }
    }
  }
}

// Q rows of one shard's leaves <- Q rows * M_leaf, with M_leaf walked down from mtop
// (identity if null); falls back to the top-down pass + apply for other s.
cudaError_t tsqr_apply_path_shard(double* dst, long ldd, const long* d_bounds, double* ws, int L,
                                  int leaf_base, int Lt, int s, const double* mtop,
                                  const DevStatus* status, cudaStream_t st, int* launches) {
  const size_t ss = (size_t)s * s;
  if (Lt <= 0) return cudaSuccess;
  const TreePlan t = tree_plan(Lt, s);
  if (t.nlev > (s <= 8 ? 32 : 20) || !(s == 1 || s == 2 || s == 4 || s == 8 || s == 16)) {
    cudaError_t e = tsqr_tree_down_shard(ws, L, leaf_base, Lt, s, mtop, status, st, launches);
    if (e != cudaSuccess) return e;
    return tsqr_apply_launch(dst, ldd, d_bounds, Lt, s, ws + (size_t)2 * L * ss + (size_t)leaf_base * ss,
                             status, st, launches);
  }
  TreePath tp;
  memset(&tp, 0, sizeof tp);
  tp.nlev = t.nlev;
  for (int k = 0; k < t.nlev; ++k) {
    tp.cnt[k] = t.cnt[k];
    tp.nb[k] = t.nb[k];
  }
  const double* nq = ws + (size_t)4 * L * ss + (size_t)leaf_base * 2 * ss;
#define BGS_APPLY_PATH(S_)                                                                   \
  if (s == S_) tsqr_apply_path_kernel<S_><<<Lt, 256, 0, st>>>(dst, ldd, d_bounds, nq, mtop, tp, status);
  BGS_APPLY_PATH(1)
  BGS_APPLY_PATH(2)
  BGS_APPLY_PATH(4)
  BGS_APPLY_PATH(8)
  BGS_APPLY_PATH(16)
#undef BGS_APPLY_PATH
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------------
size_t tsqr_ws_bytes(int leaves, int s) {
  return (size_t)leaves * s * s * 6 * sizeof(double);
}

cudaError_t tsqr_leaf_launch(const double* src, long lds, double* dst, long ldd,
                             const long* d_bounds, int L, long hmax, int s, double* rleaf,
                             const DevStatus* status, cudaStream_t st, int* launches) {
  static const bool generic = [] {
    const char* e = getenv("BGS_TSQR_GENERIC");
    return e && *e && *e != '0';
  }();
#define BGS_LEAF_REG(S_, RPT_)                                                             \
  if (!generic && s == S_ && hmax <= (long)RPT_ * kLeafThreads) {                                     \
    tsqr_leaf_reg_kernel<S_, RPT_><<<L, kLeafThreads, 0, st>>>(src, lds, dst, ldd, d_bounds, \
                                                              rleaf, status);              \
    if (launches) *launches += 1;                                                          \
    return cudaGetLastError();                                                             \
  }
  BGS_LEAF_REG(1, 4)
  BGS_LEAF_REG(2, 4)
  BGS_LEAF_REG(4, 4)
  BGS_LEAF_REG(8, 2)
  BGS_LEAF_REG(16, 1)
#undef BGS_LEAF_REG
  const size_t smem = (size_t)2 * (hmax > 0 ? hmax : 1) * s * sizeof(double);
  cudaError_t e = ensure_smem(tsqr_leaf_kernel, smem);
  if (e != cudaSuccess) return e;
  tsqr_leaf_kernel<<<L, kLeafThreads, smem, st>>>(src, lds, dst, ldd, d_bounds, s, rleaf, status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t tsqr_apply_launch(double* dst, long ldd, const long* d_bounds, int L, int s,
                              const double* M, const DevStatus* status, cudaStream_t st,
                              int* launches) {
  tsqr_apply_kernel<<<L, 256, 0, st>>>(dst, ldd, d_bounds, M, s, status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t tsqr_cross_launch(const double* roots, int n, int s, double* ws2, double* rout,
                              int ldrout, double* mout, const DevStatus* status,
                              cudaStream_t st, int* launches) {
  tsqr_cross_kernel<<<1, 512, 0, st>>>(roots, n, s, ws2, rout, ldrout, mout, status);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
