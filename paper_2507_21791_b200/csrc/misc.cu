// misc.cu — input generation and verification kernels.
//
//  gen_gaussian : seeded i.i.d. N(0,1) test matrices on the device (counter-based
//                 Philox4x32-10 keyed by (seed, global row, column) + Box-Muller), the
//                 device-side stand-in for gen_matrix's Gaussian mode
//                 (matrix_gen.cpp:18-56) at sizes where the reference's sequential
//                 mt19937_64 stream is too slow; independent of the row sharding.
//  residual     : sum of squares of X - Q R and of X (metrics.cpp:16-28), double-double
//                 partials per CTA, for full-size verification on the device.
#include <mutex>
#include <unordered_map>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {

BGS_DEV void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                          uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
  c0 = n0; c1 = n1; c2 = n2; c3 = n3;
}

BGS_DEV void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c[0], c[1], c[2], c[3], k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

}  // namespace

__global__ void gen_gaussian_kernel(unsigned long long seed, long row0, long n_local, long m,
                                    double* __restrict__ x, long ldx) {
  const long total = n_local * m;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long i = idx % n_local, j = idx / n_local;
    const unsigned long long grow = (unsigned long long)(row0 + i);
    uint32_t c[4] = {(uint32_t)grow, (uint32_t)(grow >> 32), (uint32_t)j, 0x5bd1e995u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const unsigned long long a = ((unsigned long long)c[0] << 32 | c[1]) >> 11;
    const unsigned long long b = ((unsigned long long)c[2] << 32 | c[3]) >> 11;
    const double u1 = (double)a * 0x1.0p-53, u2 = (double)b * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(1.0 - u1));
    x[i + (size_t)j * ldx] = radius * cospi(2.0 * u2);
  }
}

cudaError_t gen_gaussian_launch(unsigned long long seed, long row0, long n_local, long m,
                                double* x, long ldx, cudaStream_t st) {
  if (n_local <= 0 || m <= 0) return cudaSuccess;
  long blocks = (n_local * m + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  gen_gaussian_kernel<<<(int)blocks, 256, 0, st>>>(seed, row0, n_local, m, x, ldx);
  return cudaGetLastError();
}

__global__ void copy_cols_kernel(const double* __restrict__ src, long lds, double* __restrict__ dst,
                                 long ldd, long rows, long cols) {
  const long total = rows * cols;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const long i = idx % rows, j = idx / rows;
    dst[i + (size_t)j * ldd] = src[i + (size_t)j * lds];
  }
}

cudaError_t copy_cols_launch(const double* src, long lds, double* dst, long ldd, long rows,
                             long cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  long blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  copy_cols_kernel<<<(int)blocks, 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}

// One thread per row and a 16-column tile of R held in shared memory:
// d_ij = x_ij - sum_{k <= j} q_ik r_kj.  Partial sums of d^2 and x^2 per CTA, in
// double-double, reduced by a second tiny kernel in fixed order.
// SM = false (m > 1600: the tile does not fit shared memory): R is read from global
// memory (L1 / L2 resident) instead.
constexpr int RES_TILE = 16;
template <bool SM>
__global__ void __launch_bounds__(256)
    residual_kernel(const double* __restrict__ x, long ldx, const double* __restrict__ q, long ldq,
                    const double* __restrict__ r, long ldr, long n_rows, long m,
                    double2* __restrict__ part) {
  extern __shared__ double rt_sm[];  // (m) x RES_TILE
  __shared__ double red[2][8][2];
  double sd = 0.0, ed = 0.0, sx = 0.0, ex = 0.0;
  for (long j0 = 0; j0 < m; j0 += RES_TILE) {
    const int nj = (int)((m - j0) < RES_TILE ? (m - j0) : RES_TILE);
    const long kmax = j0 + nj;  // R upper: rows k < j0 + nj matter
    if (SM) {
      __syncthreads();
      for (long e = threadIdx.x; e < kmax * RES_TILE; e += blockDim.x) {
        const long k = e % kmax;
        const int jj = (int)(e / kmax);
        rt_sm[e] = jj < nj ? r[k + (size_t)(j0 + jj) * ldr] : 0.0;
      }
      __syncthreads();
    }
    // tile element (k, jj): shared copy, or R itself (columns past nj read as zero)
    auto rt = [&](long k, int jj) -> double {
      if (SM) return rt_sm[k + jj * kmax];
      return jj < nj ? __ldg(&r[k + (size_t)(j0 + jj) * ldr]) : 0.0;
    };
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n_rows;
         i += (long)gridDim.x * blockDim.x) {
      double acc[RES_TILE];
#pragma unroll
      for (int jj = 0; jj < RES_TILE; ++jj) acc[jj] = 0.0;
      for (long k = 0; k < kmax; ++k) {
        const double qv = q[i + (size_t)k * ldq];
#pragma unroll
        for (int jj = 0; jj < RES_TILE; ++jj) acc[jj] = fma(qv, rt(k, jj), acc[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < RES_TILE; ++jj) {
        if (jj < nj) {
          const double xv = x[i + (size_t)(j0 + jj) * ldx];
          const double d = xv - acc[jj];
          double s2, e2;
          two_sum(sd, d * d, s2, e2);
          sd = s2; ed += e2;
          two_sum(sx, xv * xv, s2, e2);
          sx = s2; ex += e2;
        }
      }
    }
  }
  // CTA reduction (fixed order)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[4] = {sd, ed, sx, ex};
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[t] += __shfl_xor_sync(0xffffffffu, v[t], o);
  if (lane == 0) {
    red[0][warp][0] = v[0]; red[0][warp][1] = v[1];
    red[1][warp][0] = v[2]; red[1][warp][1] = v[3];
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0, e = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      double s2, e2;
      two_sum(s, red[threadIdx.x][w][0], s2, e2);
      s = s2; e += e2 + red[threadIdx.x][w][1];
    }
    part[blockIdx.x * 2 + threadIdx.x] = make_double2(s, e);
  }
}

__global__ void dd_finish_kernel(const double2* part, int G, double* out) {
  const int t = threadIdx.x;
  if (t >= 2) return;
  double s = 0.0, e = 0.0;
  for (int g = 0; g < G; ++g) {
    const double2 v = part[g * 2 + t];
    double s2, e2;
    two_sum(s, v.x, s2, e2);
    s = s2; e += e2 + v.y;
  }
  out[t] = s + e;
}

cudaError_t residual_launch(const double* x, long ldx, const double* q, long ldq,
                            const double* r, long ldr, long n_rows, long m, double, double,
                            double* ws, double* out, int num_sms, cudaStream_t st) {
  const size_t smem = (size_t)m * RES_TILE * sizeof(double);
  long grid = (n_rows + 255) / 256;
  if (grid > num_sms * 2) grid = num_sms * 2;
  if (grid < 1) grid = 1;
  if (smem <= 200 * 1024) {
    cudaError_t e = ensure_smem(residual_kernel<true>, smem);
    if (e != cudaSuccess) return e;
    residual_kernel<true><<<(int)grid, 256, smem, st>>>(x, ldx, q, ldq, r, ldr, n_rows, m,
                                                        reinterpret_cast<double2*>(ws));
  } else {
    residual_kernel<false><<<(int)grid, 256, 0, st>>>(x, ldx, q, ldq, r, ldr, n_rows, m,
                                                       reinterpret_cast<double2*>(ws));
  }
  dd_finish_kernel<<<1, 32, 0, st>>>(reinterpret_cast<const double2*>(ws), (int)grid, out);
  return cudaGetLastError();
}

// ---- two_norm on the device (metrics.cpp:8-14, dense_kernels.cpp:205-239) ----
// y = A x for a symmetric m x m A (column-major): warp w of the CTA forms row i = 8 b + w as
// the dot of column i with x (coalesced), x staged in shared memory.
__global__ void __launch_bounds__(256) sym_matvec_kernel(const double* __restrict__ A, int m,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ y) {
  extern __shared__ double xs[];
  for (int k = threadIdx.x; k < m; k += blockDim.x) xs[k] = x[k];
  __syncthreads();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= m) return;
  const double* col = A + (size_t)i * m;
  double a0 = 0.0, a1 = 0.0;
  int k = lane;
  for (; k + 32 < m; k += 64) {
    a0 = fma(col[k], xs[k], a0);
    a1 = fma(col[k + 32], xs[k + 32], a1);
  }
  if (k < m) a0 = fma(col[k], xs[k], a0);
  double acc = a0 + a1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[i] = acc;
}

// nrm = ||u||_2 (one CTA, fixed order); then v = u / nrm (a second launch reads nrm).
__global__ void __launch_bounds__(256) norm2_kernel(const double* __restrict__ u, int m,
                                                    double* __restrict__ nrm) {
  __shared__ double red[8];
  double a = 0.0;
  for (int k = threadIdx.x; k < m; k += blockDim.x) a = fma(u[k], u[k], a);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    nrm[0] = sqrt(t);
  }
}

__global__ void scale_kernel(const double* __restrict__ u, int m, const double* __restrict__ nrm,
                             double* __restrict__ v) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) v[k] = nrm[0] == 0.0 ? 0.0 : u[k] / nrm[0];
}

__global__ void sub_identity_kernel(double* A, int m) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) A[k + (size_t)k * m] -= 1.0;
}

// ||A||_2 of a symmetric device matrix by power iteration on A^T A = A A (the reference's
// iteration: w = A^T A v, lambda = ||w||, v = w / lambda, stop when lambda moves by at most
// 1e-10 relative, at most 5000 rounds): sqrt(lambda).  ws: 3 m + 8 doubles.
cudaError_t sym_two_norm(double* A, int m, bool sub_identity, double* ws, double* out,
                         cudaStream_t st) {
  cudaError_t e;
  if (sub_identity) sub_identity_kernel<<<(m + 255) / 256, 256, 0, st>>>(A, m);
  double* v = ws;
  double* w = ws + m;
  double* u = ws + 2 * m;
  double* nrm = ws + 3 * m;
  std::vector<double> v0(m);
  double nv = 0.0;
  for (int i = 0; i < m; ++i) {
    v0[i] = 1.0 + (double)(i % 13) / 16.0;
    nv += v0[i] * v0[i];
  }
  nv = std::sqrt(nv);
  for (auto& t : v0) t /= nv;
  if ((e = cudaMemcpyAsync(v, v0.data(), (size_t)m * sizeof(double), cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return e;
  const size_t smem = (size_t)m * sizeof(double);
  if ((e = ensure_smem(sym_matvec_kernel, smem)) != cudaSuccess) return e;
  double lambda = 0.0, prev = 0.0;
  for (int it = 0; it < 5000; ++it) {
    sym_matvec_kernel<<<(m + 7) / 8, 256, smem, st>>>(A, m, v, w);
    sym_matvec_kernel<<<(m + 7) / 8, 256, smem, st>>>(A, m, w, u);
    norm2_kernel<<<1, 256, 0, st>>>(u, m, nrm);
    scale_kernel<<<(m + 255) / 256, 256, 0, st>>>(u, m, nrm, v);
    if ((e = cudaMemcpyAsync(&lambda, nrm, sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if (lambda == 0.0) break;
    if (it > 0 && std::fabs(lambda - prev) <= 1e-10 * lambda) break;
    prev = lambda;
  }
  *out = std::sqrt(lambda);
  return cudaGetLastError();
}

cudaError_t ensure_smem_impl(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[kernel];
  if (bytes <= have) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

}  // namespace bgs
