// small.cu — K3: replicated small factor operations, one CTA, on the device.
//
// Replaces the per-step replicated arithmetic of bcgs.cpp that the reference runs
// redundantly on every rank between synchronizations:
//   pyth_chol / chol_factor      (intraorth.cpp:158-163, dense_kernels.cpp:54-87)
//   tri_solve_left_trans         (dense_kernels.cpp:112-133)  S12 and the delayed
//                                 reprojection S2 = Y_kk^{-T}(P - Y^T Z) (bcgs.cpp:339)
//   multiply_at_b                (dense_matrix.cpp:124-139)
//   R assembly: store_column_blocks / upper_product (bcgs.cpp:35-59, 332-333)
// Semantics kept: symmetrization before Cholesky, the !(acc > 0) pivot test with a
// 1-based pivot, NotSpd diagnostics {site, block column, assumption power}, and the
// NonFiniteError check on every reduced Gram (dense_kernels.cpp:45-47).  Results go to
// device buffers read by K2; the host never waits on them.
#include "common.cuh"
#include "kernels.h"

namespace bgs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int SMAX = 16;

struct Smem {
  double a[SMAX * SMAX];
  double b[SMAX * SMAX];
  double c[SMAX * SMAX];
  double d[SMAX * SMAX];
  double sdp[SMAX * SMAX];  // previous S_diag
  int flag;
  int pivot;
};

// out(i,j) = sum_r A(r,i) B(r,j), rows x s each; one warp per entry, fixed order.
__device__ void cta_atb(const double* A, int lda, const double* B, int ldb, int rows, int s,
                        double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < s * s; e += kWarps) {
    const int i = e % s, j = e / s;
    double acc = 0.0;
    for (int r = lane; r < rows; r += 32) acc = fma(A[r + (size_t)i * lda], B[r + (size_t)j * ldb], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[i + j * s] = acc;
  }
}

// Upper Cholesky of the symmetrized a (s x s) into g; returns the 1-based failing pivot.
// Thread-serial: s <= 16 (chol_factor, dense_kernels.cpp:54-87).
__device__ int chol_serial(const double* a, int s, double* g) {
  double sym[SMAX * SMAX];
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i) sym[i + j * s] = 0.5 * (a[i + j * s] + a[j + i * s]);
  for (int k = 0; k < s * s; ++k) g[k] = 0.0;
  for (int j = 0; j < s; ++j) {
    for (int i = 0; i <= j; ++i) {
      double acc = sym[i + j * s];
      for (int k = 0; k < i; ++k) acc -= g[k + i * s] * g[k + j * s];
      if (i == j) {
        if (!(acc > 0.0)) return j + 1;
        g[j + j * s] = sqrt(acc);
      } else {
        g[i + j * s] = acc / g[i + i * s];
      }
    }
  }
  return 0;
}

// W = G^{-T} B for upper G (s x s), B (s x s) (tri_solve_left_trans).  Returns 1-based
// index of a zero diagonal entry (SingularError), else 0.
__device__ int trsm_lt_serial(const double* g, int ldg_, const double* b, int ldb, int s,
                              double* w) {
  for (int i = 0; i < s; ++i) {
    const double gii = g[i + i * ldg_];
    if (gii == 0.0) return i + 1;
    for (int j = 0; j < s; ++j) {
      double acc = b[i + j * ldb];
      for (int k = 0; k < i; ++k) acc -= g[k + i * ldg_] * w[k + j * s];
      w[i + j * s] = acc / gii;
    }
  }
  return 0;
}

__device__ void set_status(DevStatus* st, int code, int pivot, int block, int site, int kp) {
  if (atomicCAS(&st->code, 0, code) == 0) {
    st->pivot = pivot;
    st->block = block;
    st->site = site;
    st->kappa_power = kp;
    __threadfence();
  }
}

// Non-finite scan of the reduced Gram (round_accumulators' NonFiniteError).
__device__ bool gram_finite(const SmallParams& p, Smem& sh) {
  if (threadIdx.x == 0) sh.flag = 0;
  __syncthreads();
  int bad = 0;
  for (int e = threadIdx.x; e < p.gm * p.gn; e += kThreads) {
    const int i = e % p.gm, j = e / p.gm;
    if (!isfinite(p.G[i + (size_t)j * p.ldg])) bad = 1;
  }
  if (bad) atomicOr(&sh.flag, 1);
  __syncthreads();
  return sh.flag == 0;
}

// R(0:kp, k-block) = S + Y * Sd  (store_column_blocks of scol + multiply(ycol, sdiag))
__device__ void r_column(const SmallParams& p, const double* Sc, int ldsc, const double* Y,
                         int ldy, const double* Sd, int ldsd) {
  const int s = p.s, kp = p.kp;
  for (int e = threadIdx.x; e < kp * s; e += kThreads) {
    const int i = e % kp, j = e / kp;
    double acc = 0.0;
    for (int l = 0; l < s; ++l) acc += Y[i + (size_t)l * ldy] * Sd[l + j * ldsd];
    p.R[i + (size_t)(p.kp + j) * p.ldr] = Sc[i + (size_t)j * ldsc] + acc;
  }
}

// R_kk = upper_product(a, b) (bcgs.cpp:35-49); lower triangle stays exact zero.
__device__ void r_diag(const SmallParams& p, const double* a, const double* b) {
  const int s = p.s;
  for (int e = threadIdx.x; e < s * s; e += kThreads) {
    const int i = e % s, j = e / s;
    double acc = 0.0;
    if (i <= j)
      for (int k = i; k <= j; ++k) acc += a[i + k * s] * b[k + j * s];
    p.R[(p.kp + i) + (size_t)(p.kp + j) * p.ldr] = i <= j ? acc : 0.0;
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) small_kernel(const SmallParams p) {
  if (status_bad(p.status)) return;
  __shared__ Smem sh;
  const int s = p.s, kp = p.kp;
  const int tid = threadIdx.x;

  if (p.gm > 0 && !gram_finite(p, sh)) {
    if (tid == 0) set_status(p.status, ST_NON_FINITE, 0, p.k + 1, SITE_NONE, 0);
    return;
  }

  switch (p.mode) {
    case SM_COPY_RBLOCK: {
      for (int e = tid; e < s * s; e += kThreads) {
        const int i = e % s, j = e / s;
        p.R[(kp + i) + (size_t)(kp + j) * p.ldr] = i <= j ? p.rtop[i + j * p.ldrtop] : 0.0;
      }
      return;
    }
    case SM_ONESYNC_PROLOGUE: {
      // R(0,0) = R00; scol = R00^{-T} (X1^T X2)  (bcgs.cpp:264-276)
      for (int e = tid; e < s * s; e += kThreads) {
        const int i = e % s, j = e / s;
        p.R[i + (size_t)j * p.ldr] = i <= j ? p.rtop[i + j * p.ldrtop] : 0.0;
      }
      if (tid == 0) {
        sh.pivot = trsm_lt_serial(p.rtop, p.ldrtop, p.G, p.ldg, s, sh.a);
        if (sh.pivot) set_status(p.status, ST_SINGULAR, sh.pivot, 1, SITE_NONE, 0);
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads)
        p.scol_next[(e % s) + (size_t)(e / s) * p.ld_scol_next] = sh.a[e];
      if (p.os_mode == OS_PYTH) {
        // S_diag = chol(T2 - scol^T scol)  (bcgs.cpp:280-287)
        cta_atb(sh.a, s, sh.a, s, s, s, sh.b);
        __syncthreads();
        if (tid == 0) {
          for (int e = 0; e < s * s; ++e)
            sh.c[e] = p.G[(s + e % s) + (size_t)(e / s) * p.ldg] - sh.b[e];
          const int piv = chol_serial(sh.c, s, sh.d);
          if (piv) set_status(p.status, ST_NOT_SPD, piv, 2, SITE_PROLOGUE_PYTH, p.kappa_power);
          for (int e = 0; e < s * s; ++e) p.sdiag[e] = sh.d[e];
        }
      } else if (p.os_mode == OS_SKIP) {
        for (int e = tid; e < s * s; e += kThreads) p.sdiag[e] = (e % s == e / s) ? 1.0 : 0.0;
      }
      return;
    }
    case SM_ONESYNC_STEP: {
      const double* Y = p.G;             // G[0:kp, 0:s]
      const double* Om = p.G + kp;       // G[kp:kp+s, 0:s]
      for (int e = tid; e < s * s; e += kThreads) sh.sdp[e] = p.sdiag[e];
      // Y^T Y, then Y_diag = chol(Omega - Y^T Y)  (bcgs.cpp:321-327)
      cta_atb(Y, p.ldg, Y, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.c[e] = Om[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        sh.pivot = chol_serial(sh.c, s, sh.d);
        if (sh.pivot)
          set_status(p.status, ST_NOT_SPD, sh.pivot, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
        for (int e = 0; e < s * s; ++e) p.ydiag[e] = sh.d[e];
      }
      __syncthreads();
      if (sh.pivot) return;
      // R column = scol + Y S_diag; R_kk = Y_diag S_diag  (bcgs.cpp:332-333)
      r_column(p, p.scol_prev, p.ld_scol_prev, Y, p.ldg, sh.sdp, s);
      r_diag(p, sh.d, sh.sdp);
      if (!p.has_next) return;
      // S2 = Y_diag^{-T} (P - Y^T Z); scol = [Z; S2]  (bcgs.cpp:336-344)
      const double* Z = p.G + (size_t)s * p.ldg;
      const double* P = p.G + kp + (size_t)s * p.ldg;
      cta_atb(Y, p.ldg, Z, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.b[e] = P[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        sh.pivot = trsm_lt_serial(sh.d, s, sh.b, s, s, sh.c);
        if (sh.pivot) set_status(p.status, ST_SINGULAR, sh.pivot, p.k + 1, SITE_NONE, 0);
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < (kp + s) * s; e += kThreads) {
        const int i = e % (kp + s), j = e / (kp + s);
        p.scol_next[i + (size_t)j * p.ld_scol_next] =
            i < kp ? Z[i + (size_t)j * p.ldg] : sh.c[(i - kp) + j * s];
      }
      if (p.os_mode == OS_PYTH) {
        __syncthreads();
        // S_diag = chol(T - scol^T scol)  (bcgs.cpp:352-359)
        cta_atb(p.scol_next, p.ld_scol_next, p.scol_next, p.ld_scol_next, kp + s, s, sh.a);
        __syncthreads();
        if (tid == 0) {
          const double* T = p.G + kp + s + (size_t)s * p.ldg;
          for (int e = 0; e < s * s; ++e) sh.b[e] = T[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
          const int piv = chol_serial(sh.b, s, sh.d);
          if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 2, SITE_FIRST_PASS, p.kappa_power);
          for (int e = 0; e < s * s; ++e) p.sdiag[e] = sh.d[e];
        }
      } else if (p.os_mode == OS_SKIP) {
        for (int e = tid; e < s * s; e += kThreads) p.sdiag[e] = (e % s == e / s) ? 1.0 : 0.0;
      }
      return;
    }
    case SM_PIPI_PROJ: {
      // [S; T] = [Q X_k]^T X_k -> S_diag = chol(T - S^T S)  (bcgs.cpp:185-195)
      for (int e = tid; e < kp * s; e += kThreads)
        p.save[(e % kp) + (size_t)(e / kp) * p.ldsave] = p.G[(e % kp) + (size_t)(e / kp) * p.ldg];
      cta_atb(p.G, p.ldg, p.G, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.b[e] = p.G[(kp + e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        const int piv = chol_serial(sh.b, s, sh.d);
        if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_FIRST_PASS, p.kappa_power);
        for (int e = 0; e < s * s; ++e) p.sdiag[e] = sh.d[e];
      }
      return;
    }
    case SM_PIPI_REPROJ: {
      // [Y; Omega] = [Q U]^T U -> Y_diag = chol(Omega - Y^T Y); R column  (bcgs.cpp:199-216)
      for (int e = tid; e < s * s; e += kThreads) sh.sdp[e] = p.sdiag[e];
      cta_atb(p.G, p.ldg, p.G, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.b[e] = p.G[(kp + e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        sh.pivot = chol_serial(sh.b, s, sh.d);
        if (sh.pivot)
          set_status(p.status, ST_NOT_SPD, sh.pivot, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
        for (int e = 0; e < s * s; ++e) p.ydiag[e] = sh.d[e];
      }
      __syncthreads();
      if (sh.pivot) return;
      r_column(p, p.aux1, p.ldaux1, p.G, p.ldg, sh.sdp, s);
      r_diag(p, sh.d, sh.sdp);
      return;
    }
    case SM_IRO_SAVE: {
      for (int e = tid; e < kp * s; e += kThreads)
        p.save[(e % kp) + (size_t)(e / kp) * p.ldsave] = p.G[(e % kp) + (size_t)(e / kp) * p.ldg];
      return;
    }
    case SM_IRO_FINISH: {
      // R column = S1 + S2 R1; R_kk = R2 R1  (bcgs.cpp:162-164)
      for (int e = tid; e < s * s; e += kThreads) {
        sh.a[e] = p.aux2[(e % s) + (size_t)(e / s) * p.ldaux2];  // R1
        sh.b[e] = p.rtop[(e % s) + (size_t)(e / s) * p.ldrtop];  // R2
      }
      __syncthreads();
      r_column(p, p.aux1, p.ldaux1, p.G, p.ldg, sh.a, s);
      r_diag(p, sh.b, sh.a);
      return;
    }
    default:
      return;
  }
}

cudaError_t small_launch(const SmallParams& p, cudaStream_t st, int* launches) {
  if (p.s < 1 || p.s > SMAX) return cudaErrorInvalidValue;
  small_kernel<<<1, kThreads, 0, st>>>(p);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
