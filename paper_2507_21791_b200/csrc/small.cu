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
#include "reduce.cuh"

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
__device__ __noinline__ void cta_atb(const double* A, int lda, const double* B, int ldb, int rows, int s,
                        double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < s * s; e += kWarps) {
    const int i = e % s, j = e / s;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const double* Ai = A + (size_t)i * lda;
    const double* Bj = B + (size_t)j * ldb;
    int r = lane;
    for (; r + 96 < rows; r += 128) {
      a0 = fma(Ai[r], Bj[r], a0);
      a1 = fma(Ai[r + 32], Bj[r + 32], a1);
      a2 = fma(Ai[r + 64], Bj[r + 64], a2);
      a3 = fma(Ai[r + 96], Bj[r + 96], a3);
    }
    for (; r < rows; r += 32) a0 = fma(Ai[r], Bj[r], a0);
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[i + j * s] = acc;
  }
}

// Upper Cholesky of the symmetrized a (s x s) into g; returns the 1-based failing pivot.
// Thread-serial: s <= 16 (chol_factor, dense_kernels.cpp:54-87).
__device__ __noinline__ int chol_serial(const double* a, int s, double* g) {
  for (int k = 0; k < s * s; ++k) g[k] = 0.0;
  for (int j = 0; j < s; ++j) {
    for (int i = 0; i <= j; ++i) {
      double acc = 0.5 * (a[i + j * s] + a[j + i * s]);
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
__device__ __noinline__ int trsm_lt_serial(const double* g, int ldg_, const double* b, int ldb, int s,
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

// R(0:kp, k-block) = S + Y * Sd  (store_column_blocks of scol + multiply(ycol, sdiag))
__device__ __noinline__ void r_column(const SmallParams& p, const double* Sc, int ldsc, const double* Y,
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
__device__ __noinline__ void r_diag(const SmallParams& p, const double* a, const double* b) {
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

// Copies an r x c column-major global block into shared memory (ld = r) with one
// coalesced pass: all loads of a thread are independent, so the L2 latency is paid once.
__device__ __noinline__ void stage(const double* src, int ld, int r, int c, double* dst) {
  for (int e = threadIdx.x; e < r * c; e += kThreads) dst[e] = src[(e % r) + (size_t)(e / r) * ld];
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) small_kernel(SmallParams p) {
  if (status_bad(p.status)) return;
  __shared__ Smem sh;
  extern __shared__ double dyn[];
  const int s = p.s, kp = p.kp;
  const int tid = threadIdx.x;
  // dynamic shared memory: [G gm x gn][scol_prev kp x s][scol_next (kp+s) x s]
  double* gs = dyn;
  double* sprev = gs + (size_t)p.gm * p.gn;
  double* snext = sprev + (size_t)kp * s;

  // ---- stage every input with one parallel pass ----
  if (tid == 0) sh.flag = 0;
  __syncthreads();
  if (p.gm > 0) {
    int bad = 0;
    for (int e = tid; e < p.gm * p.gn; e += kThreads) {
      const double v = p.G[(e % p.gm) + (size_t)(e / p.gm) * p.ldg];
      gs[e] = v;
      bad |= !isfinite(v);
    }
    if (bad) atomicOr(&sh.flag, 1);
    p.G = gs;  // every mode below reads the Gram from shared memory
    p.ldg = p.gm;
  }
  if (MODE == SM_ONESYNC_STEP) stage(p.scol_prev, p.ld_scol_prev, kp, s, sprev);
  if (MODE == SM_PIPI_REPROJ || MODE == SM_IRO_FINISH) stage(p.aux1, p.ldaux1, kp, s, sprev);
  for (int e = tid; e < s * s; e += kThreads) {
    if (p.sdiag) sh.sdp[e] = p.sdiag[e];
    if (MODE == SM_IRO_FINISH) {
      sh.a[e] = p.aux2[(e % s) + (size_t)(e / s) * p.ldaux2];  // R1
      sh.b[e] = p.rtop[(e % s) + (size_t)(e / s) * p.ldrtop];  // R2
    }
    if (MODE == SM_ONESYNC_PROLOGUE || MODE == SM_COPY_RBLOCK)
      sh.b[e] = p.rtop[(e % s) + (size_t)(e / s) * p.ldrtop];  // root R
  }
  __syncthreads();
  if (sh.flag) {
    if (tid == 0) set_status(p.status, ST_NON_FINITE, 0, p.k + 1, SITE_NONE, 0);
    return;
  }

  switch (MODE) {
    case SM_COPY_RBLOCK: {
      for (int e = tid; e < s * s; e += kThreads) {
        const int i = e % s, j = e / s;
        p.R[(kp + i) + (size_t)(kp + j) * p.ldr] = i <= j ? sh.b[e] : 0.0;
      }
      return;
    }
    case SM_ONESYNC_PROLOGUE: {
      // R(0,0) = R00; scol = R00^{-T} (X1^T X2)  (bcgs.cpp:264-276)
      for (int e = tid; e < s * s; e += kThreads) {
        const int i = e % s, j = e / s;
        p.R[i + (size_t)j * p.ldr] = i <= j ? sh.b[e] : 0.0;
      }
      if (tid == 0) {
        sh.pivot = trsm_lt_serial(sh.b, s, p.G, p.ldg, s, sh.a);
        if (sh.pivot) set_status(p.status, ST_SINGULAR, sh.pivot, 1, SITE_NONE, 0);
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads)
        p.scol_next[(e % s) + (size_t)(e / s) * p.ld_scol_next] = sh.a[e];
      if (p.os_mode == OS_PYTH) {
        // S_diag = chol(T2 - scol^T scol)  (bcgs.cpp:280-287)
        cta_atb(sh.a, s, sh.a, s, s, s, sh.c);
        __syncthreads();
        if (tid == 0) {
          for (int e = 0; e < s * s; ++e)
            sh.c[e] = p.G[(s + e % s) + (size_t)(e / s) * p.ldg] - sh.c[e];
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
      // Y^T Y, then Y_diag = chol(Omega - Y^T Y)  (bcgs.cpp:321-327)
      cta_atb(Y, p.ldg, Y, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.c[e] = Om[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        sh.pivot = chol_serial(sh.c, s, sh.d);
        if (sh.pivot)
          set_status(p.status, ST_NOT_SPD, sh.pivot, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads) p.ydiag[e] = sh.d[e];
      // R column = scol + Y S_diag; R_kk = Y_diag S_diag  (bcgs.cpp:332-333)
      r_column(p, sprev, kp, Y, p.ldg, sh.sdp, s);
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
      const int kn = kp + s;
      for (int e = tid; e < kn * s; e += kThreads) {
        const int i = e % kn, j = e / kn;
        const double v = i < kp ? Z[i + (size_t)j * p.ldg] : sh.c[(i - kp) + j * s];
        snext[e] = v;
        p.scol_next[i + (size_t)j * p.ld_scol_next] = v;
      }
      if (p.os_mode == OS_PYTH) {
        __syncthreads();
        // S_diag = chol(T - scol^T scol)  (bcgs.cpp:352-359)
        cta_atb(snext, kn, snext, kn, kn, s, sh.a);
        __syncthreads();
        if (tid == 0) {
          const double* T = p.G + kp + s + (size_t)s * p.ldg;
          for (int e = 0; e < s * s; ++e) sh.b[e] = T[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
          const int piv = chol_serial(sh.b, s, sh.c);
          if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 2, SITE_FIRST_PASS, p.kappa_power);
          for (int e = 0; e < s * s; ++e) p.sdiag[e] = sh.c[e];
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
      cta_atb(p.G, p.ldg, p.G, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid == 0) {
        for (int e = 0; e < s * s; ++e) sh.b[e] = p.G[(kp + e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        sh.pivot = chol_serial(sh.b, s, sh.d);
        if (sh.pivot)
          set_status(p.status, ST_NOT_SPD, sh.pivot, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads) p.ydiag[e] = sh.d[e];
      r_column(p, sprev, kp, p.G, p.ldg, sh.sdp, s);
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
      r_column(p, sprev, kp, p.G, p.ldg, sh.a, s);
      r_diag(p, sh.b, sh.a);
      return;
    }
    default:
      return;
  }
}

// ---------------------------------------------------------------------------------
// SM_ONESYNC_STEP for s <= 4 (bcgs.cpp:294-367), the per-step op of the one-sync sweep:
// one pass over the kp rows of [Y | Z] = G[0:kp, 0:2s] computes Y^T Y, Y^T Z, Z^T Z (36
// dot products per thread, then a fixed-order block reduction), the R column
// S_prev + Y S_diag and the copy of Z into scol_next; thread 0 then runs the s x s
// Cholesky / triangular solves in registers.  Same operation order as chol_serial /
// trsm_lt_serial / r_diag; only the kp-long sums are grouped differently (the reference
// forms them sequentially, this path by rows-per-thread then a tree).
// ---------------------------------------------------------------------------------
namespace {
constexpr int kStepThreads = 256;

// upper Cholesky of the symmetrized 4x4 (s x s used) a into g; 1-based failing pivot
BGS_DEV int chol4(const double (&a)[16], int s, double (&g)[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) g[k] = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int i = 0; i <= j; ++i) {
      if (j < s) {
        double acc = 0.5 * (a[i + 4 * j] + a[j + 4 * i]);
#pragma unroll
        for (int k = 0; k < i; ++k) acc -= g[k + 4 * i] * g[k + 4 * j];
        if (i == j) {
          if (!(acc > 0.0)) return j + 1;
          g[j + 4 * j] = sqrt(acc);
        } else {
          g[i + 4 * j] = acc / g[i + 4 * i];
        }
      }
    }
  }
  return 0;
}

// w = g^{-T} b (g upper); 1-based index of a zero diagonal entry, else 0
BGS_DEV int trsm4(const double (&g)[16], const double (&b)[16], int s, double (&w)[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) w[k] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < s) {
      const double gii = g[i + 4 * i];
      if (gii == 0.0) return i + 1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < s) {
          double acc = b[i + 4 * j];
#pragma unroll
          for (int k = 0; k < i; ++k) acc -= g[k + 4 * i] * w[k + 4 * j];
          w[i + 4 * j] = acc / gii;
        }
      }
    }
  }
  return 0;
}
}  // namespace

__device__ __noinline__ void onesync_step4_body(const SmallParams& p) {
  const int s = p.s, kp = p.kp, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nz = p.has_next ? s : 0;  // Z columns present
  __shared__ double red[kStepThreads / 32][36];
  __shared__ double prod[36];
  __shared__ double blk[3][16];  // Omega = G[kp:, 0:s], P = G[kp:, s:2s], T = G[kp+s:, s:2s]
  __shared__ int bad_flag;
  if (tid == 0) bad_flag = 0;
  // previous S_diag (broadcast loads) and the status word, issued together
  double sdp[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) sdp[e] = ((e & 3) < s && (e >> 2) < s) ? p.sdiag[(e & 3) + s * (e >> 2)] : 0.0;
  const bool dead = status_bad(p.status);
  if (tid < 48) {  // the s x s blocks thread 0 needs later, loaded now in parallel
    const int b = tid >> 4, e = tid & 15, i = e & 3, j = e >> 2;
    double v = 0.0;
    if (i < s && j < s && (b == 0 || p.has_next)) {
      const size_t ld = p.ldg;
      v = b == 0 ? p.G[(kp + i) + j * ld]
                 : b == 1 ? p.G[(kp + i) + (s + j) * ld] : p.G[(kp + s + i) + (s + j) * ld];
    }
    blk[b][e] = v;
  }
  // ---- one pass over rows: products, R column, scol_next copy, non-finite check ----
  double acc[36];
#pragma unroll
  for (int e = 0; e < 36; ++e) acc[e] = 0.0;
  int bad = 0;
  double rcol[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = tid + h * kStepThreads;
    double y[4] = {0.0, 0.0, 0.0, 0.0}, z[4] = {0.0, 0.0, 0.0, 0.0};
    if (r < kp) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if (l < s) y[l] = p.G[r + (size_t)l * p.ldg];
        if (l < nz) z[l] = p.G[r + (size_t)(s + l) * p.ldg];
      }
#pragma unroll
      for (int l = 0; l < 4; ++l) bad |= !isfinite(y[l]) | !isfinite(z[l]);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        // R(r, kp + l) = S_prev(r, l) + sum_m Y(r, m) S_diag(m, l)
        double a = 0.0;
#pragma unroll
        for (int m2 = 0; m2 < 4; ++m2) a += y[m2] * sdp[m2 + 4 * l];
        rcol[h][l] = l < s ? p.scol_prev[r + (size_t)l * p.ld_scol_prev] + a : 0.0;
        if (l < nz) p.scol_next[r + (size_t)l * p.ld_scol_next] = z[l];
      }
    }
    // packed upper YtY (10), full YtZ (16), upper ZtZ (10)
    int e = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i <= j; ++i, ++e) acc[e] = fma(y[i], y[j], acc[e]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i, ++e) acc[e] = fma(y[i], z[j], acc[e]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i <= j; ++i, ++e) acc[e] = fma(z[i], z[j], acc[e]);
  }
  // the rest of the reduced Gram, for the non-finite check (rows kp..gm)
  for (int e = tid; e < (p.gm - kp) * p.gn; e += kStepThreads) {
    const int r = kp + e % (p.gm - kp), c = e / (p.gm - kp);
    bad |= !isfinite(p.G[r + (size_t)c * p.ldg]);
  }
  if (bad) atomicOr(&bad_flag, 1);
#pragma unroll
  for (int e = 0; e < 36; ++e) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  }
  if (lane == 0)
#pragma unroll
    for (int e = 0; e < 36; ++e) red[warp][e] = acc[e];
  __syncthreads();
  if (dead) return;
  if (tid < 36) {
    double t = 0.0;
    for (int w = 0; w < kStepThreads / 32; ++w) t += red[w][tid];
    prod[tid] = t;
  }
  if (bad_flag) {
    if (tid == 0) set_status(p.status, ST_NON_FINITE, 0, p.k + 1, SITE_NONE, 0);
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = tid + h * kStepThreads;
    if (r < kp)
#pragma unroll
      for (int l = 0; l < 4; ++l)
        if (l < s) p.R[r + (size_t)(kp + l) * p.ldr] = rcol[h][l];
  }
  __syncthreads();
  if (tid != 0) return;
  // ---- thread 0: s x s factors in registers (the s x s Gram blocks come from blk) ----
  double ytz[16], c[16], yd[16], sd[16];
  {
    int e = 0;
    double yty[16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i <= j; ++i) {
        yty[i + 4 * j] = yty[j + 4 * i] = prod[e];
        ++e;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) ytz[i + 4 * j] = prod[e++];
    // Y_diag = chol(Omega - Y^T Y)  (bcgs.cpp:321-327)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        c[i + 4 * j] = (i < s && j < s) ? blk[0][i + 4 * j] - yty[i + 4 * j] : 0.0;
  }
  int piv = chol4(c, s, yd);
  if (piv) {
    set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
    return;
  }
#pragma unroll
  for (int e = 0; e < 16; ++e)
    if ((e & 3) < s && (e >> 2) < s) p.ydiag[(e & 3) + s * (e >> 2)] = yd[e];
  // R_kk = upper_product(Y_diag, S_diag)  (bcgs.cpp:35-49, 333)
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < s && j < s) {
        double a = 0.0;
        if (i <= j)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k >= i && k <= j) a += yd[i + 4 * k] * sdp[k + 4 * j];
        p.R[(kp + i) + (size_t)(kp + j) * p.ldr] = i <= j ? a : 0.0;
      }
    }
  if (!p.has_next) return;
  // S2 = Y_diag^{-T} (P - Y^T Z); scol_next = [Z; S2]  (bcgs.cpp:336-344)
  double bm[16], s2[16];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      bm[i + 4 * j] = (i < s && j < s) ? blk[1][i + 4 * j] - ytz[i + 4 * j] : 0.0;
  piv = trsm4(yd, bm, s, s2);
  if (piv) {
    set_status(p.status, ST_SINGULAR, piv, p.k + 1, SITE_NONE, 0);
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < s && j < s) p.scol_next[(kp + i) + (size_t)j * p.ld_scol_next] = s2[i + 4 * j];
  if (p.os_mode == OS_PYTH) {
    // S_diag = chol(T - scol^T scol), scol^T scol = Z^T Z + S2^T S2  (bcgs.cpp:352-359)
    double t[16];
    int e = 26;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i <= j; ++i) {
        double a = prod[e++];
#pragma unroll
        for (int k = 0; k < 4; ++k) a += s2[k + 4 * i] * s2[k + 4 * j];
        const double v = (i < s && j < s) ? blk[2][i + 4 * j] : 0.0;
        const double vt = (i < s && j < s) ? blk[2][j + 4 * i] : 0.0;
        t[i + 4 * j] = v - a;
        t[j + 4 * i] = vt - a;
      }
    piv = chol4(t, s, sd);
    if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 2, SITE_FIRST_PASS, p.kappa_power);
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if ((k & 3) < s && (k >> 2) < s) p.sdiag[(k & 3) + s * (k >> 2)] = sd[k];
  } else if (p.os_mode == OS_SKIP) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if ((k & 3) < s && (k >> 2) < s) p.sdiag[(k & 3) + s * (k >> 2)] = (k & 3) == (k >> 2) ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(kStepThreads, 1) onesync_step4_kernel(SmallParams p) {
  onesync_step4_body(p);
}

// gram_reduce + the one-sync step in one launch: every CTA reduces its slice of the Gram,
// publishes it (fence + ticket), and the last CTA to finish runs the step on the complete
// Gram (the threadfence-reduction pattern); it also re-arms the ticket for the next launch.
static_assert(RED_THREADS == kStepThreads, "one block shape for both halves");
__global__ void __launch_bounds__(kStepThreads, 1)
    reduce_step4_kernel(const ReduceArgs r, SmallParams p, unsigned* ticket) {
  __shared__ int last;
  gram_reduce_body(r);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;
  onesync_step4_body(p);
}

bool small_mergeable(const SmallParams& p) {
  return p.mode == SM_ONESYNC_STEP && p.s <= 4 && p.kp <= 2 * kStepThreads && !p.sdiag_prev_copy;
}

cudaError_t reduce_small_launch(const ReduceArgs& r, int entries, const SmallParams& p,
                                unsigned* ticket, cudaStream_t st, int* launches) {
  if (!small_mergeable(p)) return cudaErrorInvalidValue;
  reduce_step4_kernel<<<(entries + RED_ENTRIES - 1) / RED_ENTRIES, kStepThreads, 0, st>>>(r, p,
                                                                                        ticket);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t small_launch(const SmallParams& p, cudaStream_t st, int* launches) {
  if (p.s < 1 || p.s > SMAX) return cudaErrorInvalidValue;
  if (small_mergeable(p)) {
    onesync_step4_kernel<<<1, kStepThreads, 0, st>>>(p);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const size_t smem =
      ((size_t)(p.gm > 0 ? p.gm * p.gn : 0) + (size_t)p.kp * p.s + (size_t)(p.kp + p.s) * p.s) *
      sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
#define BGS_SMALL_CASE(M)                      \
  case M:                                      \
    e = ensure_smem(small_kernel<M>, smem);    \
    if (e != cudaSuccess) return e;            \
    small_kernel<M><<<1, kThreads, smem, st>>>(p); \
    break;
  switch (p.mode) {
    BGS_SMALL_CASE(SM_ONESYNC_PROLOGUE)
    BGS_SMALL_CASE(SM_ONESYNC_STEP)
    BGS_SMALL_CASE(SM_PIPI_PROJ)
    BGS_SMALL_CASE(SM_PIPI_REPROJ)
    BGS_SMALL_CASE(SM_IRO_SAVE)
    BGS_SMALL_CASE(SM_IRO_FINISH)
    BGS_SMALL_CASE(SM_COPY_RBLOCK)
    default: return cudaErrorInvalidValue;
  }
#undef BGS_SMALL_CASE
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
