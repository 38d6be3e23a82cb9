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
#include <algorithm>

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

// Upper Cholesky of the symmetrized a (s x s) into g (shared); returns the 1-based failing
// pivot on every lane (chol_factor, dense_kernels.cpp:54-87).  One warp, lane j owning
// column j (s <= 16): rows are finished in order -- the diagonal on lane i, then row i's
// divisions in parallel.  Entry (i, j) = (0.5 (a_ij + a_ji) - sum_{k<i} g_ki g_kj) / g_ii
// with the same k order as the serial loop, so the result is the same bit for bit and the
// first failing pivot is the same; the chain is s square roots + s divisions instead of
// s (s + 1) / 2 dependent fp64 divisions / roots on one thread.
__device__ __noinline__ int chol_warp(const double* a, int s, double* g) {
  const int lane = threadIdx.x & 31;
  for (int k = lane; k < s * s; k += 32) g[k] = 0.0;
  __syncwarp();
  for (int i = 0; i < s; ++i) {
    double d = 0.0;
    if (lane == i) {
      double acc = 0.5 * (a[i + i * s] + a[i + i * s]);
      for (int k = 0; k < i; ++k) acc -= g[k + i * s] * g[k + i * s];
      d = acc;
    }
    d = __shfl_sync(0xffffffffu, d, i);
    if (!(d > 0.0)) return i + 1;
    const double gii = sqrt(d);
    if (lane > i && lane < s) {
      const int j = lane;
      double acc = 0.5 * (a[i + j * s] + a[j + i * s]);
      for (int k = 0; k < i; ++k) acc -= g[k + i * s] * g[k + j * s];
      g[i + j * s] = acc / gii;
    }
    if (lane == i) g[i + i * s] = gii;
    __syncwarp();
  }
  return 0;
}

// W = G^{-T} B for upper G (s x s), B (s x s) (tri_solve_left_trans), one warp: lane j
// solves column j (same expressions and order as the row-serial loop).  Returns the
// 1-based index of the first zero diagonal entry (SingularError) on every lane, else 0.
__device__ __noinline__ int trsm_lt_warp(const double* g, int ldg_, const double* b, int ldb, int s,
                                         double* w) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < s; ++i)
    if (g[i + i * ldg_] == 0.0) return i + 1;
  if (lane < s) {
    const int j = lane;
    for (int i = 0; i < s; ++i) {
      double acc = b[i + j * ldb];
      for (int k = 0; k < i; ++k) acc -= g[k + i * ldg_] * w[k + j * s];
      w[i + j * s] = acc / g[i + i * ldg_];
    }
  }
  __syncwarp();
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
  // batches of 8 independent loads per thread before their stores (L2 latency once per
  // batch, not per element)
  const int tot = r * c;
  for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * kThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kThreads;
      v[u] = e < tot ? src[(e % r) + (size_t)(e / r) * ld] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * kThreads;
      if (e < tot) dst[e] = v[u];
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) small_kernel(SmallParams p) {
  if (status_bad(p.status)) return;
  __shared__ Smem sh;
  extern __shared__ double dyn[];
  const int s = p.s, kp = p.kp;
  const int tid = threadIdx.x;
  // dynamic shared memory: [G gm x gn][scol_prev kp x s][scol_next (kp+s) x s], unless
  // that exceeds the budget (p.unstaged: large m x s, e.g. s = 16 at m > 400): then every
  // operand is read where it lies (global, L2-resident) with its own leading dimension
  const bool stg = !p.unstaged;
  double* gs = dyn;
  double* sprev = stg ? gs + (size_t)p.gm * p.gn : nullptr;
  double* snext = stg ? sprev + (size_t)kp * s : p.scol_next;
  int ld_prev = kp;
  const int ld_next = stg ? kp + s : p.ld_scol_next;

  // ---- stage every input with one parallel pass ----
  if (tid == 0) sh.flag = 0;
  __syncthreads();
  if (p.gm > 0) {
    int bad = 0;
    const int tot = p.gm * p.gn;
    for (int e0 = tid; e0 < tot; e0 += 8 * kThreads) {  // 8 loads in flight per thread
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kThreads;
        v[u] = e < tot ? p.G[(e % p.gm) + (size_t)(e / p.gm) * p.ldg] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kThreads;
        if (e < tot) {
          if (stg) gs[e] = v[u];
          bad |= !isfinite(v[u]);
        }
      }
    }
    if (bad) atomicOr(&sh.flag, 1);
    if (stg) {
      p.G = gs;  // every mode below reads the Gram from shared memory
      p.ldg = p.gm;
    }
  }
  if (stg) {
    if (MODE == SM_ONESYNC_STEP) stage(p.scol_prev, p.ld_scol_prev, kp, s, sprev);
      if (MODE == SM_PIPI_REPROJ || MODE == SM_IRO_FINISH || MODE == SM_CLASSIC_FINISH)
      stage(p.aux1, p.ldaux1, kp, s, sprev);
  } else if (MODE == SM_ONESYNC_STEP) {
    sprev = const_cast<double*>(p.scol_prev);
    ld_prev = p.ld_scol_prev;
  } else if (MODE == SM_PIPI_REPROJ || MODE == SM_IRO_FINISH || MODE == SM_CLASSIC_FINISH) {
    sprev = const_cast<double*>(p.aux1);
    ld_prev = p.ldaux1;
  }
  for (int e = tid; e < s * s; e += kThreads) {
    if (p.sdiag) sh.sdp[e] = p.sdiag[e];
    if (MODE == SM_IRO_FINISH) {
      sh.a[e] = p.aux2[(e % s) + (size_t)(e / s) * p.ldaux2];  // R1
      sh.b[e] = p.rtop[(e % s) + (size_t)(e / s) * p.ldrtop];  // R2
    }
    if (MODE == SM_ONESYNC_PROLOGUE || MODE == SM_COPY_RBLOCK || MODE == SM_CLASSIC_FINISH)
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
      if (tid < 32) {
        const int piv = trsm_lt_warp(sh.b, s, p.G, p.ldg, s, sh.a);
        if (tid == 0) {
          sh.pivot = piv;
          if (piv) set_status(p.status, ST_SINGULAR, piv, 1, SITE_NONE, 0);
        }
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads)
        p.scol_next[(e % s) + (size_t)(e / s) * p.ld_scol_next] = sh.a[e];
      if (p.os_mode == OS_PYTH) {
        // S_diag = chol(T2 - scol^T scol)  (bcgs.cpp:280-287)
        cta_atb(sh.a, s, sh.a, s, s, s, sh.c);
        __syncthreads();
        if (tid < 32) {
          for (int e = tid; e < s * s; e += 32)
            sh.c[e] = p.G[(s + e % s) + (size_t)(e / s) * p.ldg] - sh.c[e];
          __syncwarp();
          const int piv = chol_warp(sh.c, s, sh.d);
          if (piv && tid == 0) set_status(p.status, ST_NOT_SPD, piv, 2, SITE_PROLOGUE_PYTH, p.kappa_power);
          __syncwarp();
          for (int e = tid; e < s * s; e += 32) p.sdiag[e] = sh.d[e];
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
      if (tid < 32) {
        for (int e = tid; e < s * s; e += 32) sh.c[e] = Om[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        __syncwarp();
        const int piv = chol_warp(sh.c, s, sh.d);
        if (tid == 0) {
          sh.pivot = piv;
          if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
        }
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads) p.ydiag[e] = sh.d[e];
      // R column = scol + Y S_diag; R_kk = Y_diag S_diag  (bcgs.cpp:332-333)
      r_column(p, sprev, ld_prev, Y, p.ldg, sh.sdp, s);
      r_diag(p, sh.d, sh.sdp);
      if (!p.has_next) return;
      // S2 = Y_diag^{-T} (P - Y^T Z); scol = [Z; S2]  (bcgs.cpp:336-344)
      const double* Z = p.G + (size_t)s * p.ldg;
      const double* P = p.G + kp + (size_t)s * p.ldg;
      cta_atb(Y, p.ldg, Z, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid < 32) {
        for (int e = tid; e < s * s; e += 32) sh.b[e] = P[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        __syncwarp();
        const int piv = trsm_lt_warp(sh.d, s, sh.b, s, s, sh.c);
        if (tid == 0) {
          sh.pivot = piv;
          if (piv) set_status(p.status, ST_SINGULAR, piv, p.k + 1, SITE_NONE, 0);
        }
      }
      __syncthreads();
      if (sh.pivot) return;
      const int kn = kp + s;
      for (int e = tid; e < kn * s; e += kThreads) {
        const int i = e % kn, j = e / kn;
        const double v = i < kp ? Z[i + (size_t)j * p.ldg] : sh.c[(i - kp) + j * s];
        if (stg) snext[e] = v;
        p.scol_next[i + (size_t)j * p.ld_scol_next] = v;
      }
      if (p.os_mode == OS_PYTH) {
        __syncthreads();  // (orders the global scol_next writes too: same block)
        // S_diag = chol(T - scol^T scol)  (bcgs.cpp:352-359)
        cta_atb(snext, ld_next, snext, ld_next, kn, s, sh.a);
        __syncthreads();
        if (tid < 32) {
          const double* T = p.G + kp + s + (size_t)s * p.ldg;
          for (int e = tid; e < s * s; e += 32) sh.b[e] = T[(e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
          __syncwarp();
          const int piv = chol_warp(sh.b, s, sh.c);
          if (piv && tid == 0) set_status(p.status, ST_NOT_SPD, piv, p.k + 2, SITE_FIRST_PASS, p.kappa_power);
          __syncwarp();
          for (int e = tid; e < s * s; e += 32) p.sdiag[e] = sh.c[e];
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
      if (tid < 32) {
        for (int e = tid; e < s * s; e += 32) sh.b[e] = p.G[(kp + e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        __syncwarp();
        const int piv = chol_warp(sh.b, s, sh.d);
        if (piv && tid == 0) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_FIRST_PASS, p.kappa_power);
        __syncwarp();
        for (int e = tid; e < s * s; e += 32) p.sdiag[e] = sh.d[e];
      }
      return;
    }
    case SM_PIPI_REPROJ: {
      // [Y; Omega] = [Q U]^T U -> Y_diag = chol(Omega - Y^T Y); R column  (bcgs.cpp:199-216)
      cta_atb(p.G, p.ldg, p.G, p.ldg, kp, s, sh.a);
      __syncthreads();
      if (tid < 32) {
        for (int e = tid; e < s * s; e += 32) sh.b[e] = p.G[(kp + e % s) + (size_t)(e / s) * p.ldg] - sh.a[e];
        __syncwarp();
        const int piv = chol_warp(sh.b, s, sh.d);
        if (tid == 0) {
          sh.pivot = piv;
          if (piv) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
        }
      }
      __syncthreads();
      if (sh.pivot) return;
      for (int e = tid; e < s * s; e += kThreads) p.ydiag[e] = sh.d[e];
      r_column(p, sprev, ld_prev, p.G, p.ldg, sh.sdp, s);
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
      r_column(p, sprev, ld_prev, p.G, p.ldg, sh.a, s);
      r_diag(p, sh.b, sh.a);
      return;
    }
    case SM_CLASSIC_FINISH: {
      // store_column_blocks(R, k, S); R.set_block(k, k, R_intra)  (bcgs.cpp:126-128)
      for (int e = tid; e < kp * s; e += kThreads) {
        const int i = e % kp, j = e / kp;
        p.R[i + (size_t)(kp + j) * p.ldr] = sprev[i + (size_t)j * ld_prev];
      }
      for (int e = tid; e < s * s; e += kThreads) {
        const int i = e % s, j = e / s;
        p.R[(kp + i) + (size_t)(kp + j) * p.ldr] = i <= j ? sh.b[e] : 0.0;
      }
      return;
    }
    case SM_CHOLQR: {
      // R = chol_factor(U^T U) (intraorth.cpp:146-149); NotSpd -> "intra-block Cholesky QR"
      if (tid < 32) {
        for (int e = tid; e < s * s; e += 32) sh.c[e] = p.G[(e % s) + (size_t)(e / s) * p.ldg];
        __syncwarp();
        const int piv = chol_warp(sh.c, s, sh.d);
        if (piv && tid == 0) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_INTRA_CHOLQR, 2);
        __syncwarp();
        for (int e = tid; e < s * s; e += 32) p.sdiag[e] = sh.d[e];
      }
      return;
    }
    default:
      return;
  }
}

// ---------------------------------------------------------------------------------
// SM_ONESYNC_STEP for s <= 4 (bcgs.cpp:294-367), the per-step op of the one-sync sweep.
// It sits on the critical path between two fused kernels, so it is built for latency:
//  1. one coalesced pass over the kp rows of [Y | Z] = G[0:kp, 0:2s]: the R column
//     S_prev + Y S_diag, the copy of Z into scol_next, the non-finite check, and the rows
//     staged in shared memory;
//  2. Y^T Y, Y^T Z, Z^T Z as 36 products x 7 row chunks on 252 threads (two interleaved
//     accumulators per thread), then a fixed-order sum of the chunks;
//  3. the s x s factors on lanes 0..3 of warp 0, lane j owning column j: Cholesky row by
//     row (the diagonal on lane i, then the divisions of row i in parallel), triangular
//     solves column-parallel.
// Every entry is formed by the same expression as chol_warp / trsm_lt_warp / r_diag
// (symmetrization, the k-ordered updates, the !(acc > 0) pivot test, division by the
// diagonal); only the kp-long sums are grouped differently (the reference forms them
// sequentially, this path by row chunks).
// ---------------------------------------------------------------------------------
namespace {
constexpr int kStepThreads = 256;
constexpr int kStepRowsMax = 2 * kStepThreads;  // small_mergeable: kp <= 512
constexpr int kStepChunks = 7;                  // 36 x 7 = 252 product threads
constexpr int kYZLd = kStepRowsMax + 1;         // odd column stride: columns in distinct banks

// (left, right) staged columns of product e: packed upper Y^T Y (10), full Y^T Z (16),
// packed upper Z^T Z (10); columns 0..3 are Y, 4..7 are Z
BGS_DEV void product_cols(int e, int& cu, int& cv) {
  const bool zz = e >= 26;
  if (e >= 10 && e < 26) {
    cu = (e - 10) & 3;
    cv = 4 + ((e - 10) >> 2);
    return;
  }
  const int f = zz ? e - 26 : e;  // f = j (j + 1) / 2 + i, i <= j
  const int j = f >= 6 ? 3 : f >= 3 ? 2 : f >= 1 ? 1 : 0;
  const int i = f - j * (j + 1) / 2;
  cu = i + (zz ? 4 : 0);
  cv = j + (zz ? 4 : 0);
}

// Upper Cholesky of the symmetrized s x s block a (column-major 4 x 4, shared) on lanes
// 0..3 of one warp, lane j owning column j, the factor in registers and the cross-lane
// operands moved by shuffles (no shared-memory round trip on the chain: 1.7 -> 1.1 us per
// factorization, %globaltimer stamps).  Entry (i, j) = (0.5 (a_ij + a_ji) -
// sum_{k<i} g_ki g_kj) / g_ii, diagonal by sqrt -- chol_warp's expression and k order --,
// rows finished in order, so the first failing pivot (1-based, returned on every lane) is
// the column-ordered loop's.  The factor also goes to g in shared memory (4 x 4).
BGS_DEV int chol4_reg(const double* a, int s, double* g, int lane) {
  const int j = lane & 3;
  double c[4], gc[4];  // symmetrized column j (entries i <= j), factor column j
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    c[i] = 0.5 * (a[i + 4 * j] + a[j + 4 * i]);
    gc[i] = 0.0;
  }
  int piv = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= s) break;
    // column i of the factor so far (final since row i - 1), from lane i
    double gi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) gi[k] = __shfl_sync(0xffffffffu, gc[k], i);
    double d = c[i];  // (lane i: the diagonal, c[i] = 0.5 (a_ii + a_ii))
#pragma unroll
    for (int k = 0; k < i; ++k) d -= gi[k] * gi[k];
    d = __shfl_sync(0xffffffffu, d, i);
    if (!(d > 0.0)) {
      piv = i + 1;
      break;
    }
    const double gii = sqrt(d);
    double acc = c[i];
#pragma unroll
    for (int k = 0; k < i; ++k) acc -= gi[k] * gc[k];
    if (j > i) gc[i] = acc / gii;
    if (j == i) gc[i] = gii;
  }
  if (lane < 4)
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i + 4 * j] = (i <= j && i < s && j < s && !piv) ? gc[i] : 0.0;
  __syncwarp();
  return piv;
}

// w = g^{-T} b (tri_solve_left_trans), g upper and b in shared memory (4 x 4); lane j < s
// solves column j with g read once (broadcast) and w in registers; same expressions and
// order as trsm_lt_warp.  Returns the 1-based index of a zero diagonal (SingularError).
BGS_DEV int trsm4_reg(const double* g, const double* b, int s, double* w, int lane) {
  for (int i = 0; i < s; ++i)
    if (g[i + 4 * i] == 0.0) return i + 1;
  const int j = lane & 3;
  double gm[16], wc[4];
#pragma unroll
  for (int e = 0; e < 16; ++e) gm[e] = g[e];
#pragma unroll
  for (int i = 0; i < 4; ++i) wc[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= s) break;
    double acc = b[i + 4 * j];
#pragma unroll
    for (int k = 0; k < i; ++k) acc -= gm[k + 4 * i] * wc[k];
    wc[i] = acc / gm[i + 4 * i];
  }
  if (lane < 4)
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i + 4 * j] = (i < s && j < s) ? wc[i] : 0.0;
  __syncwarp();
  return 0;
}

}  // namespace

#ifdef BGS_STEP_STAMPS
__device__ unsigned long long g_st_min = ~0ull, g_st_red = 0ull, g_st[8], g_st_log[512 * 8];
extern "C" int bgs_dbg_step_stamps(unsigned long long* out) {  // 512 x 8, host memory
  return (int)cudaMemcpyFromSymbol(out, g_st_log, sizeof g_st_log);
}
BGS_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STAMP(i) \
  if (threadIdx.x == 0) g_st[i] = gtime();
#else
#define STAMP(i)
#endif

__device__ __forceinline__ void onesync_step4_body(const SmallParams& p) {
  const int s = p.s, kp = p.kp, tid = threadIdx.x, lane = tid & 31;
  const int nz = p.has_next ? s : 0;  // Z columns present
  __shared__ double yz[8 * kYZLd];    // [Y | Z] rows 0..kp, column stride kYZLd
  __shared__ double part[36][kStepChunks];
  __shared__ double prod[36];
  __shared__ double blk[3][16];  // Omega = G[kp:, 0:s], P = G[kp:, s:2s], T = G[kp+s:, s:2s]
  __shared__ double f_in[16], f_yd[16], f_s2[16], f_sd[16], f_sdp[16];  // s x s blocks (4 x 4)
  __shared__ int bad_flag;
  if (tid == 0) bad_flag = 0;
  if (tid < 16) {
    const int i = tid & 3, j = tid >> 2;
    f_sdp[tid] = (i < s && j < s) ? p.sdiag[i + s * j] : 0.0;
  }
  // previous S_diag (broadcast loads) and the status word, issued together
  double sdp[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) sdp[e] = ((e & 3) < s && (e >> 2) < s) ? p.sdiag[(e & 3) + s * (e >> 2)] : 0.0;
  const bool dead = status_bad(p.status);
  if (tid < 48) {  // the s x s blocks warp 0 needs later, loaded now in parallel
    const int b = tid >> 4, e = tid & 15, i = e & 3, j = e >> 2;
    double v = 0.0;
    if (i < s && j < s && (b == 0 || p.has_next)) {
      const size_t ld = p.ldg;
      v = b == 0 ? p.G[(kp + i) + j * ld]
                 : b == 1 ? p.G[(kp + i) + (s + j) * ld] : p.G[(kp + s + i) + (s + j) * ld];
    }
    blk[b][e] = v;
  }
  // ---- 1. one pass over rows: stage [Y | Z], R column, scol_next copy, non-finite check ----
  // Every load of the pass is issued before the first store (one L2 round trip: the
  // stores to scol_next could alias G as far as the compiler knows).
  double y[2][4], z[2][4], sp[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = tid + h * kStepThreads;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      y[h][l] = (r < kp && l < s) ? p.G[r + (size_t)l * p.ldg] : 0.0;
      z[h][l] = (r < kp && l < nz) ? p.G[r + (size_t)(s + l) * p.ldg] : 0.0;
      sp[h][l] = (r < kp && l < s) ? p.scol_prev[r + (size_t)l * p.ld_scol_prev] : 0.0;
    }
  }
  // the rest of the reduced Gram, for the non-finite check (rows kp..gm)
  const int tail = (p.gm - kp) * p.gn;
  const double tv = tid < tail ? p.G[kp + tid % (p.gm - kp) + (size_t)(tid / (p.gm - kp)) * p.ldg] : 0.0;
  int bad = !isfinite(tv);
  for (int e = tid + kStepThreads; e < tail; e += kStepThreads) {
    const int r = kp + e % (p.gm - kp), c = e / (p.gm - kp);
    bad |= !isfinite(p.G[r + (size_t)c * p.ldg]);
  }
  double rcol[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = tid + h * kStepThreads;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      bad |= !isfinite(y[h][l]) | !isfinite(z[h][l]);
      // R(r, kp + l) = S_prev(r, l) + sum_m Y(r, m) S_diag(m, l)
      double a = 0.0;
#pragma unroll
      for (int m2 = 0; m2 < 4; ++m2) a += y[h][m2] * sdp[m2 + 4 * l];
      rcol[h][l] = l < s ? sp[h][l] + a : 0.0;
    }
    if (r < kp) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        yz[l * kYZLd + r] = y[h][l];
        yz[(4 + l) * kYZLd + r] = z[h][l];
        if (l < nz) p.scol_next[r + (size_t)l * p.ld_scol_next] = z[h][l];
      }
    }
  }
  if (bad) atomicOr(&bad_flag, 1);
  __syncthreads();
  STAMP(2)
  if (dead) return;
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
  // ---- 2. the 36 products: row pairs (2b, 2b + 1) summed in kStepChunks contiguous
  // chunks of pairs, even / odd pairs interleaved (the merged path's order) ----
  if (tid < 36 * kStepChunks) {
    const int e = tid % 36, c = tid / 36;
    int cu, cv;
    product_cols(e, cu, cv);
    const int np = (kp + 1) / 2;
    const int len = (np + kStepChunks - 1) / kStepChunks;
    const int b0 = c * len, b1 = min(np, b0 + len);
    const double* u = yz + cu * kYZLd;
    const double* v = yz + cv * kYZLd;
    auto pair = [&](int b) {  // rows past kp are zero in yz (staged as 0 when r >= kp)
      const double p0 = __dmul_rn(u[2 * b], v[2 * b]);
      const double p1 = 2 * b + 1 < kp ? __dmul_rn(u[2 * b + 1], v[2 * b + 1]) : 0.0;
      return __dadd_rn(p0, p1);
    };
    double a0 = 0.0, a1 = 0.0;
    int b = b0;
    for (; b + 1 < b1; b += 2) {
      a0 = __dadd_rn(a0, pair(b));
      a1 = __dadd_rn(a1, pair(b + 1));
    }
    if (b < b1) a0 = __dadd_rn(a0, pair(b));
    part[e][c] = a0 + a1;
  }
  __syncthreads();
  STAMP(3)
  if (tid >= 32) return;
  for (int e = lane; e < 36; e += 32) {  // lanes 0..3 also take products 32..35
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < kStepChunks; ++c) t += part[e][c];
    prod[e] = t;
  }
  __syncwarp();
  // ---- 3. warp 0: s x s factors, lane j owning column j ----
  // Y_diag = chol(Omega - Y^T Y)  (bcgs.cpp:321-327)
  if (lane < 16) {
    const int i = lane & 3, j = lane >> 2;
    const int lo = min(i, j), hi = max(i, j);
    const double yty = prod[hi * (hi + 1) / 2 + lo];
    f_in[lane] = (i < s && j < s) ? blk[0][lane] - yty : 0.0;
  }
  __syncwarp();
  int piv = chol4_reg(f_in, s, f_yd, lane);
  STAMP(4)
  if (piv) {
    if (lane == 0) set_status(p.status, ST_NOT_SPD, piv, p.k + 1, SITE_SECOND_PASS, p.kappa_power);
    return;
  }
  if (lane < 16) {
    const int i = lane & 3, j = lane >> 2;
    if (i < s && j < s) {
      p.ydiag[i + s * j] = f_yd[lane];
      // R_kk = upper_product(Y_diag, S_diag)  (bcgs.cpp:35-49, 333)
      double a = 0.0;
      if (i <= j)
        for (int k = i; k <= j; ++k) a += f_yd[i + 4 * k] * f_sdp[k + 4 * j];
      p.R[(kp + i) + (size_t)(kp + j) * p.ldr] = i <= j ? a : 0.0;
    }
  }
  if (!p.has_next) return;
  // S2 = Y_diag^{-T} (P - Y^T Z); scol_next = [Z; S2]  (bcgs.cpp:336-344)
  if (lane < 16) {
    const int i = lane & 3, j = lane >> 2;
    f_in[lane] = (i < s && j < s) ? blk[1][lane] - prod[10 + lane] : 0.0;
  }
  __syncwarp();
  piv = trsm4_reg(f_yd, f_in, s, f_s2, lane);
  STAMP(5)
  if (piv) {
    if (lane == 0) set_status(p.status, ST_SINGULAR, piv, p.k + 1, SITE_NONE, 0);
    return;
  }
  if (lane < 16) {
    const int i = lane & 3, j = lane >> 2;
    if (i < s && j < s) p.scol_next[(kp + i) + (size_t)j * p.ld_scol_next] = f_s2[lane];
  }
  if (p.os_mode == OS_PYTH) {
    // S_diag = chol(T - scol^T scol), scol^T scol = Z^T Z + S2^T S2  (bcgs.cpp:352-359)
    __syncwarp();
    if (lane < 16) {
      const int i = lane & 3, j = lane >> 2;
      const int lo = min(i, j), hi = max(i, j);
      double a = prod[26 + hi * (hi + 1) / 2 + lo];
#pragma unroll
      for (int k = 0; k < 4; ++k) a += f_s2[k + 4 * lo] * f_s2[k + 4 * hi];
      f_in[lane] = ((i < s && j < s) ? blk[2][lane] : 0.0) - a;
    }
    __syncwarp();
    piv = chol4_reg(f_in, s, f_sd, lane);
    if (piv && lane == 0) set_status(p.status, ST_NOT_SPD, piv, p.k + 2, SITE_FIRST_PASS, p.kappa_power);
    __syncwarp();
    if (lane < 16) {
      const int i = lane & 3, j = lane >> 2;
      if (i < s && j < s) p.sdiag[i + s * j] = f_sd[lane];
    }
#ifdef BGS_STEP_STAMPS
    STAMP(6)
    if (tid == 0 && p.k < 512) {  // [k][start, reduce done, detect, pass, products, chol, trsm, end]
      unsigned long long* o = g_st_log + (size_t)p.k * 8;
      o[0] = g_st_min; o[1] = g_st_red;
      for (int i = 1; i <= 6; ++i) o[i + 1] = g_st[i];
    }
    if (tid == 0) {
      g_st_min = ~0ull;
      g_st_red = 0ull;
    }
#endif
  } else if (p.os_mode == OS_SKIP) {
    if (lane < 16) {
      const int i = lane & 3, j = lane >> 2;
      if (i < s && j < s) p.sdiag[i + s * j] = i == j ? 1.0 : 0.0;
    }
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
    reduce_step4_kernel(const ReduceArgs r, int nblk, SmallParams p, unsigned* ticket) {
  __shared__ int last;
  // The next fused kernel may launch now (programmatic dependent): its CTAs take the SMs
  // this grid frees and prefetch their first stages; they wait for this grid to complete
  // before reading anything it writes.
  griddep_launch_dependents();
#ifdef BGS_STEP_STAMPS
  const unsigned long long t_in = gtime();
#endif
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) gram_reduce_body(r, b);
#ifdef BGS_STEP_STAMPS
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(&g_st_min, t_in);
    atomicMax(&g_st_red, gtime());
  }
#endif
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;
  STAMP(1)
  onesync_step4_body(p);
}

// ---------------------------------------------------------------------------------------
// The one-sync step across ranks over peer-mapped windows (peer.cu), fused with its
// neighbours: SURVEY.md 8(f) row 4, replacing exact_allreduce (communicator.cpp:226-250)
// between fused_gram and the step's small operations.
//   A  reduce_push_kernel: every CTA reduces its slice of the local Gram partials and
//      stores the entries straight into slot (epoch & 1, rank) of EVERY rank's window
//      (NVLink / NVSwitch peer stores); the last CTA publishes flag[rank] = epoch
//      everywhere (release, system scope).
//   B  sum_step4_kernel: [acquire-spin on the P local flags: distinct GPUs only; ranks that
//      share a GPU wait with stream memory operations before the launch] every CTA adds
//      its slice of the P partials in rank order into G (same order on every rank ->
//      bitwise replicated); the last CTA runs the step.  Triggers the programmatic launch
//      of the next fused kernel at entry, like the single-GPU merged kernel.
//   AB reduce_xchg_step4_kernel: A and B in ONE launch (in-kernel spin; distinct GPUs).
// A block step is then fused kernel -> A -> B (or AB) -> fused kernel instead of fused ->
// gram_reduce -> push -> sum -> step -> fused.
BGS_DEV void peer_sum_body(const PeerView& v, unsigned epoch, int spin, unsigned long words,
                           double* __restrict__ G, DevStatus* status) {
  unsigned char* win = v.win[v.rank];
  if (spin) {
    if ((int)threadIdx.x < v.P) {
      const unsigned* f = reinterpret_cast<const unsigned*>(win) + threadIdx.x;
      if (!spin_flag_geq(f, epoch) && status)  // (pivot: the rank that never arrived, 1-based)
        set_status(status, ST_COLLECTIVE, (int)threadIdx.x + 1, 0, SITE_NONE, 0);
    }
    __syncthreads();
  }
  const double* base = reinterpret_cast<const double*>(win + kPeerFlagBytes +
                                                       (size_t)(epoch & 1u) * v.P * v.slot_bytes);
  const unsigned long sd = v.slot_bytes / sizeof(double);
  const unsigned long stride = (unsigned long)gridDim.x * blockDim.x;
  for (unsigned long i = (unsigned long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) {
    double acc = __ldcv(base + i);
    for (int r = 1; r < v.P; ++r) acc += __ldcv(base + (size_t)r * sd + i);  // rank order
    G[i] = acc;
  }
}

// true in exactly one CTA: the last one to get here (re-arms the ticket)
BGS_DEV bool last_cta(unsigned* ticket, bool system_scope) {
  __shared__ int last;
  if (system_scope) __threadfence_system(); else __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return false;
  if (system_scope) __threadfence_system(); else __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

BGS_DEV void publish_flags(const PeerView& v, unsigned epoch) {
  if ((int)threadIdx.x < v.P)
    st_release_sys(reinterpret_cast<unsigned*>(v.win[threadIdx.x]) + v.rank, epoch);
}

__global__ void __launch_bounds__(kStepThreads, 1)
    reduce_push_kernel(const ReduceArgs r, int nblk, const ReducePush push, const PeerView v,
                       unsigned epoch, unsigned* ticket) {
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) gram_reduce_body<true>(r, b, &push);
  if (!last_cta(ticket, true)) return;
  publish_flags(v, epoch);
}

__global__ void __launch_bounds__(kStepThreads, 1)
    sum_step4_kernel(const PeerView v, unsigned epoch, int spin, unsigned long words, double* G,
                     SmallParams p, unsigned* ticket) {
  griddep_launch_dependents();
  peer_sum_body(v, epoch, spin, words, G, const_cast<DevStatus*>(p.status));
  if (!last_cta(ticket, false)) return;
  onesync_step4_body(p);
}

__global__ void __launch_bounds__(kStepThreads, 1)
    reduce_xchg_step4_kernel(const ReduceArgs r, int nblk, const ReducePush push, const PeerView v,
                             unsigned epoch, unsigned long words, double* G, SmallParams p,
                             unsigned* ticket) {
  griddep_launch_dependents();
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) gram_reduce_body<true>(r, b, &push);
  if (last_cta(ticket, true)) publish_flags(v, epoch);
  // (every CTA of this grid is resident -- one wave -- so the spin cannot starve the CTA
  // that publishes this rank's flag; the peers' flags arrive over NVLink)
  __syncthreads();
  peer_sum_body(v, epoch, 1, words, G, const_cast<DevStatus*>(p.status));
  if (!last_cta(ticket + 1, false)) return;
  onesync_step4_body(p);
}

bool small_mergeable(const SmallParams& p) {
  return p.mode == SM_ONESYNC_STEP && p.s <= 4 && p.kp <= 2 * kStepThreads && !p.sdiag_prev_copy;
}

cudaError_t reduce_small_launch(const ReduceArgs& r, int entries, const SmallParams& p,
                                unsigned* ticket, int sms, cudaStream_t st, int* launches) {
  if (!small_mergeable(p)) return cudaErrorInvalidValue;
  // one wave: the step body needs ~140 registers, so one CTA per SM; extra entry blocks
  // are looped over inside the CTA instead of running as a second wave
  const int nblk = (entries + RED_ENTRIES - 1) / RED_ENTRIES;
  reduce_step4_kernel<<<std::min(nblk, sms), kStepThreads, 0, st>>>(r, nblk, p, ticket);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t reduce_push_launch(const ReduceArgs& r, int entries, const ReducePush& push,
                               const PeerView& v, unsigned epoch, unsigned* ticket, int sms,
                               cudaStream_t st, int* launches) {
  const int nblk = (entries + RED_ENTRIES - 1) / RED_ENTRIES;
  reduce_push_kernel<<<std::min(nblk, sms), kStepThreads, 0, st>>>(r, nblk, push, v, epoch, ticket);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t sum_small_launch(const PeerView& v, unsigned epoch, bool spin, unsigned long words,
                             double* G, const SmallParams& p, unsigned* ticket, int sms,
                             cudaStream_t st, int* launches) {
  if (!small_mergeable(p)) return cudaErrorInvalidValue;
  const int grid = (int)std::max<unsigned long>(1, std::min<unsigned long>(sms, (words + kStepThreads - 1) / kStepThreads));
  sum_step4_kernel<<<grid, kStepThreads, 0, st>>>(v, epoch, spin ? 1 : 0, words, G, p, ticket);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t reduce_xchg_small_launch(const ReduceArgs& r, int entries, const ReducePush& push,
                                     const PeerView& v, unsigned epoch, unsigned long words,
                                     double* G, const SmallParams& p, unsigned* ticket, int sms,
                                     cudaStream_t st, int* launches) {
  if (!small_mergeable(p)) return cudaErrorInvalidValue;
  const int nblk = (entries + RED_ENTRIES - 1) / RED_ENTRIES;
  // one wave (<= one CTA per SM: the step body's registers allow no more), see the kernel
  reduce_xchg_step4_kernel<<<std::min(nblk, sms), kStepThreads, 0, st>>>(r, nblk, push, v, epoch,
                                                                       words, G, p, ticket);
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
  size_t smem =
      ((size_t)(p.gm > 0 ? p.gm * p.gn : 0) + (size_t)p.kp * p.s + (size_t)(p.kp + p.s) * p.s) *
      sizeof(double);
  SmallParams q = p;
  q.unstaged = smem > 200 * 1024 ? 1 : 0;  // read the operands from global memory instead
  if (q.unstaged) smem = 0;
  cudaError_t e = cudaSuccess;
#define BGS_SMALL_CASE(M)                      \
  case M:                                      \
    e = ensure_smem(small_kernel<M>, smem);    \
    if (e != cudaSuccess) return e;            \
    small_kernel<M><<<1, kThreads, smem, st>>>(q); \
    break;
  switch (p.mode) {
    BGS_SMALL_CASE(SM_ONESYNC_PROLOGUE)
    BGS_SMALL_CASE(SM_ONESYNC_STEP)
    BGS_SMALL_CASE(SM_PIPI_PROJ)
    BGS_SMALL_CASE(SM_PIPI_REPROJ)
    BGS_SMALL_CASE(SM_IRO_SAVE)
    BGS_SMALL_CASE(SM_IRO_FINISH)
    BGS_SMALL_CASE(SM_COPY_RBLOCK)
    BGS_SMALL_CASE(SM_CLASSIC_FINISH)
    BGS_SMALL_CASE(SM_CHOLQR)
    default: return cudaErrorInvalidValue;
  }
#undef BGS_SMALL_CASE
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace bgs
