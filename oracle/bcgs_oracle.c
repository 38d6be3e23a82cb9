/* TEST INFRASTRUCTURE — NOT THE PRODUCT.  See bcgs_oracle.h for the contract.
 *
 * A from-scratch C restatement of the reference's CPU algorithms for the BCGS QR hot
 * path.  Every function names the reference file:line whose behaviour it restates
 * (paths relative to /root/reference/proj).  Floating-point operation order follows
 * the reference so that, compiled with -ffp-contract=off, results are BITWISE equal to
 * the reference's (checked by tests/test_oracle_pin.py against oracle/_ref).
 *
 * Differences in structure (not in results):
 *  - one address space: the P "ranks" of the reference's run_spmd are not threads here.
 *    Everything the reference computes per rank is row-local except the exact Gram
 *    (order-free, so P-independent) and the TSQR leaf plan (restated with P);
 *  - the exact accumulator is a carry-save 68 x 32-bit-digit fixed-point number
 *    (LSB weight 2^-1074) instead of the reference's 34 x 64-bit two's-complement limbs;
 *    both round the exact sum once, to nearest even, so they agree bitwise;
 *  - Gram operands are lists of column pointers (no local_concat copies).
 */
#include "bcgs_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * Error context + allocation arena
 * ---------------------------------------------------------------------------------- */
enum { E_OK = 0, E_DIM = 1, E_NOTSPD = 2, E_SINGULAR = 3, E_RANKDEF = 4, E_NONFINITE = 5,
       E_COLLECTIVE = 6, E_CONFIG = 7, E_OTHER = 8 };

typedef struct {
  jmp_buf jb;
  int code;
  int pivot;
  char msg[1024];
  void** ptrs;
  long nptr, cap;
  or_stats* st;
  int procs;
} ctx_t;

static void fail(ctx_t* c, int code, int pivot, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->msg, sizeof c->msg, fmt, ap);
  va_end(ap);
  c->code = code;
  c->pivot = pivot;
  longjmp(c->jb, 1);
}

static void* amalloc(ctx_t* c, size_t bytes) {
  void* p = calloc(1, bytes ? bytes : 1);
  if (!p) fail(c, E_OTHER, 0, "oracle: out of memory");
  if (c->nptr == c->cap) {
    c->cap = c->cap ? 2 * c->cap : 256;
    c->ptrs = (void**)realloc(c->ptrs, sizeof(void*) * (size_t)c->cap);
  }
  c->ptrs[c->nptr++] = p;
  return p;
}

static void afree(ctx_t* c, void* p) {
  if (!p) return;
  for (long i = c->nptr - 1; i >= 0; --i) {
    if (c->ptrs[i] == p) {
      c->ptrs[i] = c->ptrs[--c->nptr];
      free(p);
      return;
    }
  }
}

static void arena_release(ctx_t* c) {
  for (long i = 0; i < c->nptr; ++i) free(c->ptrs[i]);
  free(c->ptrs);
  c->ptrs = NULL;
  c->nptr = c->cap = 0;
}

/* ------------------------------------------------------------------------------------
 * Column-major matrices (dense_matrix.hpp:10-40)
 * ---------------------------------------------------------------------------------- */
typedef struct {
  long r, c;
  double* d;
} mat;
#define AT(M, i, j) ((M).d[(size_t)(j) * (size_t)(M).r + (size_t)(i)])

static mat mnew(ctx_t* c, long r, long cols) {
  mat m = {r, cols, NULL};
  m.d = (double*)amalloc(c, sizeof(double) * (size_t)(r * cols));
  return m;
}
static void mdel(ctx_t* c, mat* m) { afree(c, m->d); m->d = NULL; }
static mat meye(ctx_t* c, long n) {
  mat m = mnew(c, n, n);
  for (long i = 0; i < n; ++i) AT(m, i, i) = 1.0;
  return m;
}
/* DenseMatrix::sub (dense_matrix.cpp:23-35) */
static mat msub(ctx_t* c, mat a, long r0, long r1, long c0, long c1) {
  mat o = mnew(c, r1 - r0, c1 - c0);
  for (long j = c0; j < c1; ++j)
    for (long i = r0; i < r1; ++i) AT(o, i - r0, j - c0) = AT(a, i, j);
  return o;
}
static void mset_sub(mat dst, long r0, long c0, mat b) {
  for (long j = 0; j < b.c; ++j)
    for (long i = 0; i < b.r; ++i) AT(dst, r0 + i, c0 + j) = AT(b, i, j);
}
/* operator+ / operator- (dense_matrix.cpp:94-106) */
static mat madd(ctx_t* c, mat a, mat b, double sgn) {
  mat o = mnew(c, a.r, a.c);
  for (long k = 0; k < a.r * a.c; ++k) o.d[k] = sgn > 0 ? a.d[k] + b.d[k] : a.d[k] - b.d[k];
  return o;
}
/* multiply: fixed ijk order (dense_matrix.cpp:107-122) */
static mat mmul(ctx_t* c, mat a, mat b) {
  mat o = mnew(c, a.r, b.c);
  for (long j = 0; j < b.c; ++j)
    for (long i = 0; i < a.r; ++i) {
      double acc = 0.0;
      for (long k = 0; k < a.c; ++k) acc += AT(a, i, k) * AT(b, k, j);
      AT(o, i, j) = acc;
    }
  return o;
}
/* multiply_at_b (dense_matrix.cpp:124-139) */
static mat mmul_atb(ctx_t* c, mat a, mat b) {
  mat o = mnew(c, a.c, b.c);
  for (long j = 0; j < b.c; ++j)
    for (long i = 0; i < a.c; ++i) {
      double acc = 0.0;
      for (long k = 0; k < a.r; ++k) acc += AT(a, k, i) * AT(b, k, j);
      AT(o, i, j) = acc;
    }
  return o;
}
/* vstack (dense_matrix.cpp:141-149) */
static mat mvstack(ctx_t* c, mat a, mat b) {
  mat o = mnew(c, a.r + b.r, a.c);
  mset_sub(o, 0, 0, a);
  mset_sub(o, a.r, 0, b);
  return o;
}
/* frobenius_norm: scaled two-pass (dense_matrix.cpp:58-69) */
static double mfrob(mat a) {
  double mx = 0.0;
  for (long k = 0; k < a.r * a.c; ++k) {
    double v = fabs(a.d[k]);
    if (v > mx) mx = v;
  }
  if (mx == 0.0) return 0.0;
  double acc = 0.0;
  for (long k = 0; k < a.r * a.c; ++k) {
    double t = a.d[k] / mx;
    acc += t * t;
  }
  return mx * sqrt(acc);
}

/* ------------------------------------------------------------------------------------
 * Exact fixed-point accumulator (restates exact_sum.hpp:8-54 / exact_sum.cpp:16-157:
 * value = sum of doubles held exactly with LSB weight 2^-1074, rounded once to
 * nearest-even).  Representation: 68 signed 64-bit "digits" of base 2^32, carry-save.
 * ---------------------------------------------------------------------------------- */
#define XL 68
typedef struct {
  int64_t l[XL];
  long cnt;
  int poison;
} xacc;

static void xacc_norm(xacc* a) {
  for (int i = 0; i < XL - 1; ++i) {
    int64_t carry = a->l[i] >> 32; /* arithmetic shift: floor division */
    a->l[i] -= (int64_t)((uint64_t)carry << 32);
    a->l[i + 1] += carry;
  }
  a->cnt = 0;
}

static inline void xacc_add(xacc* a, double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff);
  uint64_t f = b & ((UINT64_C(1) << 52) - 1);
  if (e == 0x7ff) { a->poison = 1; return; }
  uint64_t mant;
  int pos;
  if (e == 0) {
    if (!f) return;
    mant = f;
    pos = 0;
  } else {
    mant = f | (UINT64_C(1) << 52);
    pos = e - 1;
  }
  int li = pos >> 5, sh = pos & 31;
  unsigned __int128 v = (unsigned __int128)mant << sh;
  int64_t d0 = (int64_t)(uint32_t)v, d1 = (int64_t)(uint32_t)(v >> 32),
          d2 = (int64_t)(uint32_t)(v >> 64);
  if (b >> 63) {
    a->l[li] -= d0; a->l[li + 1] -= d1; a->l[li + 2] -= d2;
  } else {
    a->l[li] += d0; a->l[li + 1] += d1; a->l[li + 2] += d2;
  }
  if (++a->cnt >= (1L << 29)) xacc_norm(a);
}

/* add_product: FMA two-product hi + lo (exact_sum.cpp:36-47) */
static inline void xacc_add_product(xacc* a, double x, double y) {
  double hi = x * y;
  if (!isfinite(hi)) { a->poison = 1; return; }
  double lo = fma(x, y, -hi);
  xacc_add(a, hi);
  xacc_add(a, lo);
}

static int xbit(const int64_t* mag, int pos) { return (int)((mag[pos >> 5] >> (pos & 31)) & 1); }
static int xany_below(const int64_t* mag, int pos) {
  int li = pos >> 5, sh = pos & 31;
  for (int i = 0; i < li; ++i)
    if (mag[i]) return 1;
  if (!sh) return 0;
  return (mag[li] & ((INT64_C(1) << sh) - 1)) != 0;
}

/* round_to_double: nearest, ties to even (exact_sum.cpp:122-157) */
static double xacc_round(const xacc* a0) {
  if (a0->poison) return NAN;
  xacc a = *a0;
  xacc_norm(&a);
  int neg = a.l[XL - 1] < 0;
  if (neg) {
    for (int i = 0; i < XL; ++i) a.l[i] = -a.l[i];
    xacc_norm(&a);
  }
  int top = XL - 1;
  while (top >= 0 && a.l[top] == 0) --top;
  if (top < 0) return 0.0;
  int msb = top * 32 + (31 - __builtin_clz((unsigned)a.l[top]));
  int rp = msb - 52 > 0 ? msb - 52 : 0;
  uint64_t mant = 0;
  for (int p = msb; p >= rp; --p) mant = (mant << 1) | (uint64_t)xbit(a.l, p);
  if (rp > 0) {
    int guard = xbit(a.l, rp - 1);
    int sticky = xany_below(a.l, rp - 1);
    if (guard && (sticky || (mant & 1))) ++mant;
  }
  double v = ldexp((double)mant, rp - 1074);
  return neg ? -v : v;
}

/* gram over column-pointer lists: out(i,j) = sum_k a_i[k] b_j[k], exact, rounded once
 * (gram_accumulate + round_accumulators, dense_kernels.cpp:10-52).  Returns nonzero if
 * any accumulator was poisoned (NonFiniteError in the reference). */
static int gram_cols(const double* const* acol, long ma, const double* const* bcol, long mb,
                     long n, double* out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (long t = 0; t < ma * mb; ++t) {
    long i = t % ma, j = t / ma;
    xacc acc;
    memset(&acc, 0, sizeof acc);
    const double* a = acol[i];
    const double* b = bcol[j];
    for (long k = 0; k < n; ++k) xacc_add_product(&acc, a[k], b[k]);
    if (acc.poison) bad = 1;
    out[i + j * ma] = xacc_round(&acc);
  }
  return bad;
}

static mat gram_m(ctx_t* c, mat a, mat b) {
  const double** ac = (const double**)amalloc(c, sizeof(double*) * (size_t)(a.c ? a.c : 1));
  const double** bc = (const double**)amalloc(c, sizeof(double*) * (size_t)(b.c ? b.c : 1));
  for (long j = 0; j < a.c; ++j) ac[j] = a.d + (size_t)j * a.r;
  for (long j = 0; j < b.c; ++j) bc[j] = b.d + (size_t)j * b.r;
  mat g = mnew(c, a.c, b.c);
  int bad = gram_cols(ac, a.c, bc, b.c, a.r, g.d);
  afree(c, ac);
  afree(c, bc);
  if (bad) fail(c, E_NONFINITE, 0, "reduction saw a NaN or infinity");
  return g;
}

/* ------------------------------------------------------------------------------------
 * Small dense kernels (dense_kernels.cpp:54-203)
 * ---------------------------------------------------------------------------------- */
/* chol_factor: symmetrize, upper factor, NotSpd on !(acc > 0) with 1-based pivot
 * (dense_kernels.cpp:54-87) */
static int chol_raw(mat a, mat g) {
  long n = a.r;
  double* s = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < n; ++i) s[i + j * n] = 0.5 * (AT(a, i, j) + AT(a, j, i));
  for (long k = 0; k < n * n; ++k) g.d[k] = 0.0;
  for (long j = 0; j < n; ++j) {
    for (long i = 0; i <= j; ++i) {
      double acc = s[i + j * n];
      for (long k = 0; k < i; ++k) acc -= AT(g, k, i) * AT(g, k, j);
      if (i == j) {
        if (!(acc > 0.0)) { free(s); return (int)(j + 1); }
        AT(g, j, j) = sqrt(acc);
      } else {
        AT(g, i, j) = acc / AT(g, i, i);
      }
    }
  }
  free(s);
  return 0;
}

static mat chol_factor(ctx_t* c, mat a) {
  mat g = mnew(c, a.r, a.r);
  int p = chol_raw(a, g);
  if (p) fail(c, E_NOTSPD, p, "cholesky pivot %d is not strictly positive", p);
  return g;
}

/* tri_solve_right: W G = B (dense_kernels.cpp:89-110) */
static mat tri_solve_right(ctx_t* c, mat b, mat g) {
  long n = g.r;
  mat w = mnew(c, b.r, n);
  for (long j = 0; j < n; ++j) {
    if (AT(g, j, j) == 0.0)
      fail(c, E_SINGULAR, (int)(j + 1), "triangular factor has a zero at diagonal entry %ld",
           j + 1);
    for (long i = 0; i < b.r; ++i) {
      double acc = AT(b, i, j);
      for (long k = 0; k < j; ++k) acc -= AT(w, i, k) * AT(g, k, j);
      AT(w, i, j) = acc / AT(g, j, j);
    }
  }
  return w;
}

/* tri_solve_left_trans: G^T W = B (dense_kernels.cpp:112-133) */
static mat tri_solve_left_trans(ctx_t* c, mat g, mat b) {
  long n = g.r;
  mat w = mnew(c, n, b.c);
  for (long i = 0; i < n; ++i) {
    if (AT(g, i, i) == 0.0)
      fail(c, E_SINGULAR, (int)(i + 1), "triangular factor has a zero at diagonal entry %ld",
           i + 1);
    for (long j = 0; j < b.c; ++j) {
      double acc = AT(b, i, j);
      for (long k = 0; k < i; ++k) acc -= AT(g, k, i) * AT(w, k, j);
      AT(w, i, j) = acc / AT(g, i, i);
    }
  }
  return w;
}

/* householder_qr: economic, nonnegative diag(R) (dense_kernels.cpp:135-203) */
static void householder(ctx_t* c, mat x, mat* qo, mat* ro) {
  long m = x.r, n = x.c, p = m < n ? m : n;
  mat a = mnew(c, m, n);
  memcpy(a.d, x.d, sizeof(double) * (size_t)(m * n));
  double* taus = (double*)amalloc(c, sizeof(double) * (size_t)(p + 1));
  double** vs = (double**)amalloc(c, sizeof(double*) * (size_t)(p + 1));
  for (long k = 0; k < p; ++k) {
    double mx = 0.0;
    for (long i = k; i < m; ++i) {
      double t = fabs(AT(a, i, k));
      mx = mx < t ? t : mx; /* std::max(mx, t) */
    }
    if (mx == 0.0) continue;
    double ssq = 0.0;
    for (long i = k; i < m; ++i) {
      double t = AT(a, i, k) / mx;
      ssq += t * t;
    }
    double sigma = mx * sqrt(ssq);
    double alpha = AT(a, k, k) >= 0.0 ? -sigma : sigma;
    double* v = (double*)amalloc(c, sizeof(double) * (size_t)(m - k));
    v[0] = AT(a, k, k) - alpha;
    for (long i = k + 1; i < m; ++i) v[i - k] = AT(a, i, k);
    double vtv = 0.0;
    for (long i = 0; i < m - k; ++i) vtv += v[i] * v[i];
    double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    AT(a, k, k) = alpha;
    for (long i = k + 1; i < m; ++i) AT(a, i, k) = 0.0;
    for (long j = k + 1; j < n; ++j) {
      double w = 0.0;
      for (long i = k; i < m; ++i) w += v[i - k] * AT(a, i, j);
      w *= tau;
      for (long i = k; i < m; ++i) AT(a, i, j) -= w * v[i - k];
    }
    taus[k] = tau;
    vs[k] = v;
  }
  mat r = mnew(c, p, n);
  for (long j = 0; j < n; ++j)
    for (long i = 0; i <= (j < p - 1 ? j : p - 1); ++i) AT(r, i, j) = AT(a, i, j);
  mat q = mnew(c, m, p);
  for (long i = 0; i < p; ++i) AT(q, i, i) = 1.0;
  for (long k = p - 1; k >= 0; --k) {
    double* v = vs[k];
    double tau = taus[k];
    if (tau == 0.0) continue;
    for (long j = 0; j < p; ++j) {
      double w = 0.0;
      for (long i = k; i < m; ++i) w += v[i - k] * AT(q, i, j);
      w *= tau;
      for (long i = k; i < m; ++i) AT(q, i, j) -= w * v[i - k];
    }
  }
  for (long k = 0; k < p; ++k) {
    if (AT(r, k, k) < 0.0) {
      for (long j = k; j < n; ++j) AT(r, k, j) = -AT(r, k, j);
      for (long i = 0; i < m; ++i) AT(q, i, k) = -AT(q, i, k);
    }
  }
  for (long k = 0; k < p; ++k) afree(c, vs[k]);
  afree(c, vs);
  afree(c, taus);
  mdel(c, &a);
  *qo = q;
  *ro = r;
}

/* upper_product (bcgs.cpp:35-49) */
static mat upper_product(ctx_t* c, mat a, mat b) {
  long n = a.r;
  mat o = mnew(c, n, n);
  for (long j = 0; j < n; ++j)
    for (long i = 0; i <= j; ++i) {
      double acc = 0.0;
      for (long k = i; k <= j; ++k) acc += AT(a, i, k) * AT(b, k, j);
      AT(o, i, j) = acc;
    }
  return o;
}

/* ------------------------------------------------------------------------------------
 * Sync accounting (sync_stats.hpp:13-27)
 * ---------------------------------------------------------------------------------- */
static void record(ctx_t* c, const char* label, long words) {
  or_stats* st = c->st;
  if (!st) return;
  st->sync_count += 1;
  st->words_reduced += words;
  size_t len = strlen(st->labels);
  if (len + strlen(label) + 2 < sizeof st->labels) {
    if (st->n_events) strcat(st->labels, "\n");
    strcat(st->labels, label);
  }
  st->n_events += 1;
}

/* ------------------------------------------------------------------------------------
 * Distributed-matrix helpers on the global matrix (dist_block.cpp).  Column block
 * pointers into a global column-major n x m matrix stand in for BlockSpan.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  const double* p; /* first column */
  long ncols;
} span_t;

/* fused_gram (dist_block.cpp:79-88): (concat left)^T (concat right), one sync */
static mat fused_gram(ctx_t* c, long n, const span_t* left, int nl, const span_t* right, int nr,
                      const char* label) {
  long ma = 0, mb = 0;
  for (int i = 0; i < nl; ++i) ma += left[i].ncols;
  for (int i = 0; i < nr; ++i) mb += right[i].ncols;
  const double** ac = (const double**)amalloc(c, sizeof(double*) * (size_t)(ma + 1));
  const double** bc = (const double**)amalloc(c, sizeof(double*) * (size_t)(mb + 1));
  long t = 0;
  for (int i = 0; i < nl; ++i)
    for (long j = 0; j < left[i].ncols; ++j) ac[t++] = left[i].p + (size_t)j * n;
  t = 0;
  for (int i = 0; i < nr; ++i)
    for (long j = 0; j < right[i].ncols; ++j) bc[t++] = right[i].p + (size_t)j * n;
  mat g = mnew(c, ma, mb);
  int bad = gram_cols(ac, ma, bc, mb, n, g.d);
  afree(c, ac);
  afree(c, bc);
  if (bad) fail(c, E_NONFINITE, 0, "reduction saw a NaN or infinity");
  record(c, label, ma * mb);
  return g;
}

/* local_axpy_block (dist_block.cpp:90-108): Y -= Q S, Y/Q given as column pointers */
static void axpy_block(long n, double* y, const double* q, mat s) {
  for (long j = 0; j < s.c; ++j) {
    double* yj = y + (size_t)j * n;
    for (long i = 0; i < n; ++i) {
      double acc = 0.0;
      for (long k = 0; k < s.r; ++k) acc += q[(size_t)k * n + i] * AT(s, k, j);
      yj[i] -= acc;
    }
  }
}

/* scale_right_block (dist_block.cpp:110-117) -> tri_solve_right, in place on n x s */
static void scale_right(ctx_t* c, long n, double* u, mat g) {
  mat b = {n, g.r, u};
  mat w = tri_solve_right(c, b, g);
  memcpy(u, w.d, sizeof(double) * (size_t)(n * g.r));
  mdel(c, &w);
}

/* ------------------------------------------------------------------------------------
 * TSQR over the fixed 24-slot leaf grid (intraorth.cpp:19-111, tsqr_tree.cpp,
 * communicator.cpp:252-317)
 * ---------------------------------------------------------------------------------- */
typedef struct {
  long h1, h2;
  mat q;
} tnode;

/* build_subtree (tsqr_tree.cpp:14-29) */
static mat build_subtree(ctx_t* c, mat* leaf_rs, long lo, long hi, tnode* nodes, long* nn) {
  if (lo == hi) {
    mat r = mnew(c, leaf_rs[lo].r, leaf_rs[lo].c);
    memcpy(r.d, leaf_rs[lo].d, sizeof(double) * (size_t)(r.r * r.c));
    return r;
  }
  long mid = lo + (hi - lo + 1) / 2;
  mat a = build_subtree(c, leaf_rs, lo, mid - 1, nodes, nn);
  mat b = build_subtree(c, leaf_rs, mid, hi, nodes, nn);
  mat st = mvstack(c, a, b);
  mat q, r;
  householder(c, st, &q, &r);
  nodes[*nn].h1 = a.r;
  nodes[*nn].h2 = b.r;
  nodes[*nn].q = q;
  (*nn)++;
  mdel(c, &st);
  mdel(c, &a);
  mdel(c, &b);
  return r;
}

/* propagate_subtree (tsqr_tree.cpp:31-49) */
static void propagate_subtree(ctx_t* c, tnode* nodes, long lo, long hi, long node_at, mat m,
                              mat* out) {
  if (lo == hi) {
    out[lo] = m;
    return;
  }
  tnode* nd = &nodes[node_at];
  long mid = lo + (hi - lo + 1) / 2;
  long right_internal = (hi - mid + 1) - 1;
  mat top = msub(c, nd->q, 0, nd->h1, 0, nd->q.c);
  mat bot = msub(c, nd->q, nd->h1, nd->h1 + nd->h2, 0, nd->q.c);
  mat ml = mmul(c, top, m);
  mat mr = mmul(c, bot, m);
  mdel(c, &top);
  mdel(c, &bot);
  propagate_subtree(c, nodes, lo, mid - 1, node_at - right_internal - 1, ml, out);
  propagate_subtree(c, nodes, mid, hi, node_at - 1, mr, out);
}

/* run_tsqr (intraorth.cpp:81-111) on the global n x s block xb (column pointer);
 * writes Q into qout (n x s), returns R.  `fused` (optional) rides in the same sync. */
static mat run_tsqr(ctx_t* c, long n, long s, const double* xb, double* qout, const mat* fused,
                    const char* label) {
  if (n < s)
    fail(c, E_RANKDEF, 0, "tsqr: block has %ld columns but only %ld global rows", s, n);
  const long slots = 24;
  int procs = c->procs;
  /* plan_leaves (intraorth.cpp:27-43) */
  long lw = (n + slots - 1) / slots;
  long per = (n + procs - 1) / procs;
  int aligned = 1;
  for (int r = 1; r < procs; ++r) {
    long b = (long)r * per < n ? (long)r * per : n;
    if (b < n && b % lw != 0) { aligned = 0; break; }
  }
  long total = aligned ? (n + lw - 1) / lw : procs;
  /* factor_local_leaves (intraorth.cpp:52-79), all ranks */
  mat* lq = (mat*)amalloc(c, sizeof(mat) * (size_t)total);
  mat* lr = (mat*)amalloc(c, sizeof(mat) * (size_t)total);
  long* lrow0 = (long*)amalloc(c, sizeof(long) * (size_t)total);
  for (long L = 0; L < total; ++L) {
    long g0, g1;
    if (aligned) {
      g0 = L * lw;
      g1 = g0 + lw < n ? g0 + lw : n;
    } else {
      g0 = L * per < n ? L * per : n;
      g1 = g0 + per < n ? g0 + per : n;
    }
    mat blk = mnew(c, g1 - g0, s);
    for (long j = 0; j < s; ++j)
      memcpy(blk.d + (size_t)j * blk.r, xb + (size_t)j * n + g0, sizeof(double) * (size_t)blk.r);
    householder(c, blk, &lq[L], &lr[L]);
    mdel(c, &blk);
    lrow0[L] = g0;
  }
  /* tsqr_leaf_reduce: combine_leaf_factors + fused grid (communicator.cpp:252-317) */
  tnode* nodes = (tnode*)amalloc(c, sizeof(tnode) * (size_t)(total + 1));
  long nn = 0;
  mat root = build_subtree(c, lr, 0, total - 1, nodes, &nn);
  long words = root.r * root.c + (fused ? fused->r * fused->c : 0);
  record(c, label, words);
  /* propagate_tree (tsqr_tree.cpp:62-78) */
  mat* ms = (mat*)amalloc(c, sizeof(mat) * (size_t)total);
  propagate_subtree(c, nodes, 0, total - 1, nn - 1, meye(c, root.r), ms);
  for (long L = 0; L < total; ++L) {
    if (ms[L].r != lr[L].r) fail(c, E_DIM, 0, "propagate_tree: leaf heights disagree with tree");
    mat ql = mmul(c, lq[L], ms[L]);
    for (long j = 0; j < s; ++j)
      memcpy(qout + (size_t)j * n + lrow0[L], ql.d + (size_t)j * ql.r,
             sizeof(double) * (size_t)ql.r);
    mdel(c, &ql);
    mdel(c, &ms[L]);
    mdel(c, &lq[L]);
    mdel(c, &lr[L]);
  }
  for (long k = 0; k < nn; ++k) mdel(c, &nodes[k].q);
  afree(c, nodes);
  afree(c, ms);
  afree(c, lq);
  afree(c, lr);
  afree(c, lrow0);
  return root;
}

/* ------------------------------------------------------------------------------------
 * R container (UpperTriangular, dense_matrix.cpp:170-220) + helpers (bcgs.cpp:52-80)
 * ---------------------------------------------------------------------------------- */
static void r_set_block(mat R, long s, long bi, long bj, mat b) { mset_sub(R, bi * s, bj * s, b); }
/* store_column_blocks (bcgs.cpp:52-59) */
static void store_column_blocks(mat R, long s, long col_block, mat scol) {
  mset_sub(R, 0, col_block * s, scol);
}

/* pyth_chol = chol(T - S^T S) (intraorth.cpp:158-163) with the semantic NotSpd rewrite
 * of rethrow_not_spd (bcgs.cpp:61-80) */
static mat pyth_chol_site(ctx_t* c, mat t, mat s, const char* variant, const char* site,
                          long block_1based, int kappa_power) {
  mat sts = mmul_atb(c, s, s);
  mat d = madd(c, t, sts, -1.0);
  mat g = mnew(c, d.r, d.r);
  int p = chol_raw(d, g);
  if (p) {
    char hyp[64] = "";
    if (kappa_power == 1) snprintf(hyp, sizeof hyp, "O(u) * kappa(X) <= 1");
    else if (kappa_power > 1) snprintf(hyp, sizeof hyp, "O(u) * kappa(X)^%d <= 1", kappa_power);
    fail(c, E_NOTSPD, p,
         "%s: %s for block column %ld hit a Gram matrix that is not numerically positive "
         "definite (cholesky pivot %d is not strictly positive)%s%s",
         variant, site, block_1based, p, hyp[0] ? "; likely violated working assumption: " : "",
         hyp);
  }
  mdel(c, &sts);
  mdel(c, &d);
  return g;
}

/* ------------------------------------------------------------------------------------
 * The five in-scope variants (bcgs.cpp:83-369).  x: n x m global; q: n x m output;
 * R: m x m output (zero-initialised).
 * ---------------------------------------------------------------------------------- */
#define COL(A, j) ((A) + (size_t)(j) * (size_t)n)

/* single_block (bcgs.cpp:83-90) */
static void single_block(ctx_t* c, long n, long s, const double* x, double* q, mat R) {
  mat r = run_tsqr(c, n, s, x, q, NULL, "reduce_factor_tree:tsqr");
  r_set_block(R, s, 0, 0, r);
}

/* iro_impl (bcgs.cpp:135-167): BCGSI+ */
static void iro_impl(ctx_t* c, long n, long m, long s, const double* x, double* q, mat R) {
  long qb = m / s;
  if (qb == 1) { single_block(c, n, s, x, q, R); return; }
  {
    mat r11 = run_tsqr(c, n, s, x, q, NULL, "reduce_factor_tree:tsqr");
    r_set_block(R, s, 0, 0, r11);
    mdel(c, &r11);
  }
  double* u = (double*)amalloc(c, sizeof(double) * (size_t)(n * s));
  for (long k = 1; k < qb; ++k) {
    long c0 = k * s;
    span_t L1[1] = {{q, c0}}, R1[1] = {{COL(x, c0), s}};
    mat s1 = fused_gram(c, n, L1, 1, R1, 1, "fused_gram:proj1");
    memcpy(u, COL(x, c0), sizeof(double) * (size_t)(n * s));
    axpy_block(n, u, q, s1);
    mat r1 = run_tsqr(c, n, s, u, u, NULL, "reduce_factor_tree:tsqr");
    span_t R2[1] = {{u, s}};
    mat s2 = fused_gram(c, n, L1, 1, R2, 1, "fused_gram:proj2");
    axpy_block(n, u, q, s2);
    mat r2 = run_tsqr(c, n, s, u, COL(q, c0), NULL, "reduce_factor_tree:tsqr");
    mat t = mmul(c, s2, r1);
    mat col = madd(c, s1, t, 1.0);
    store_column_blocks(R, s, k, col);
    mat rkk = upper_product(c, r2, r1);
    r_set_block(R, s, k, k, rkk);
    mdel(c, &s1); mdel(c, &r1); mdel(c, &s2); mdel(c, &r2); mdel(c, &t); mdel(c, &col);
    mdel(c, &rkk);
  }
  afree(c, u);
}

/* pipi_impl (bcgs.cpp:169-219): BCGSPIPI+ */
static void pipi_impl(ctx_t* c, long n, long m, long s, const double* x, double* q, mat R) {
  long qb = m / s;
  if (qb == 1) { single_block(c, n, s, x, q, R); return; }
  {
    mat r11 = run_tsqr(c, n, s, x, q, NULL, "reduce_factor_tree:tsqr");
    r_set_block(R, s, 0, 0, r11);
    mdel(c, &r11);
  }
  double* u = (double*)amalloc(c, sizeof(double) * (size_t)(n * s));
  for (long k = 1; k < qb; ++k) {
    long c0 = k * s;
    span_t L1[2] = {{q, c0}, {COL(x, c0), s}}, R1[1] = {{COL(x, c0), s}};
    mat m1 = fused_gram(c, n, L1, 2, R1, 1, "fused_gram:proj");
    mat scol = msub(c, m1, 0, c0, 0, s);
    mat t = msub(c, m1, c0, c0 + s, 0, s);
    mat sdiag = pyth_chol_site(c, t, scol, "BCGSPIPI+", "first-pass Pythagorean normalization",
                               k + 1, 2);
    memcpy(u, COL(x, c0), sizeof(double) * (size_t)(n * s));
    axpy_block(n, u, q, scol);
    scale_right(c, n, u, sdiag);
    span_t L2[2] = {{q, c0}, {u, s}}, R2[1] = {{u, s}};
    mat m2 = fused_gram(c, n, L2, 2, R2, 1, "fused_gram:reproj");
    mat ycol = msub(c, m2, 0, c0, 0, s);
    mat omega = msub(c, m2, c0, c0 + s, 0, s);
    mat ydiag = pyth_chol_site(c, omega, ycol, "BCGSPIPI+",
                               "second-pass Pythagorean normalization", k + 1, 2);
    axpy_block(n, u, q, ycol);
    scale_right(c, n, u, ydiag);
    memcpy(COL(q, c0), u, sizeof(double) * (size_t)(n * s));
    mat ys = mmul(c, ycol, sdiag);
    mat col = madd(c, scol, ys, 1.0);
    store_column_blocks(R, s, k, col);
    mat rkk = upper_product(c, ydiag, sdiag);
    r_set_block(R, s, k, k, rkk);
    mdel(c, &m1); mdel(c, &scol); mdel(c, &t); mdel(c, &sdiag); mdel(c, &m2); mdel(c, &ycol);
    mdel(c, &omega); mdel(c, &ydiag); mdel(c, &ys); mdel(c, &col); mdel(c, &rkk);
  }
  afree(c, u);
}

enum { MODE_PYTH = 0, MODE_SKIP = 1, MODE_TSQR = 2 };

/* onesync_impl (bcgs.cpp:233-369): BCGSI+P-1S (PythChol), BCGSI+1S (SkipNorm),
 * BCGSI+P-2S (TsqrPath) */
static void onesync_impl(ctx_t* c, long n, long m, long s, const double* x, double* q, mat R,
                         int mode, const char* name, int kappa_power) {
  long qb = m / s;
  if (qb == 1) { single_block(c, n, s, x, q, R); return; }
  double* u = (double*)amalloc(c, sizeof(double) * (size_t)(n * s));
  double* un = (double*)amalloc(c, sizeof(double) * (size_t)(n * s));
  mat scol, sdiag;
  /* prologue (bcgs.cpp:250-292) */
  if (mode == MODE_TSQR) {
    span_t L[1] = {{x, s}}, Rr[1] = {{COL(x, s), s}};
    /* tsqr_fused_gram: the Gram is computed without its own sync (intraorth.cpp:122-135) */
    const double* ac[64];
    const double* bc[64];
    mat fused = mnew(c, s, s);
    for (long j = 0; j < s; ++j) { ac[j] = COL(x, j); bc[j] = COL(x, s + j); }
    (void)L; (void)Rr;
    if (gram_cols(ac, s, bc, s, n, fused.d)) fail(c, E_NONFINITE, 0, "reduction saw a NaN or infinity");
    mat r00 = run_tsqr(c, n, s, x, q, &fused, "reduce_factor_tree:prologue");
    r_set_block(R, s, 0, 0, r00);
    scol = tri_solve_left_trans(c, r00, fused);
    memcpy(u, COL(x, s), sizeof(double) * (size_t)(n * s));
    axpy_block(n, u, q, scol);
    sdiag = run_tsqr(c, n, s, u, u, NULL, "reduce_factor_tree:tsqr");
    mdel(c, &fused);
    mdel(c, &r00);
  } else {
    int pyth = mode == MODE_PYTH;
    long lc = pyth ? 2 * s : s;
    const double* ac[128];
    const double* bc[64];
    mat fused = mnew(c, lc, s);
    for (long j = 0; j < lc; ++j) ac[j] = COL(x, j);
    for (long j = 0; j < s; ++j) bc[j] = COL(x, s + j);
    if (gram_cols(ac, lc, bc, s, n, fused.d)) fail(c, E_NONFINITE, 0, "reduction saw a NaN or infinity");
    mat r00 = run_tsqr(c, n, s, x, q, &fused, "reduce_factor_tree:prologue");
    r_set_block(R, s, 0, 0, r00);
    mat x1tx2 = msub(c, fused, 0, s, 0, s);
    scol = tri_solve_left_trans(c, r00, x1tx2);
    memcpy(u, COL(x, s), sizeof(double) * (size_t)(n * s));
    axpy_block(n, u, q, scol);
    if (pyth) {
      mat t2 = msub(c, fused, s, 2 * s, 0, s);
      sdiag = pyth_chol_site(c, t2, scol, name, "prologue Pythagorean normalization", 2,
                             kappa_power);
      scale_right(c, n, u, sdiag);
      mdel(c, &t2);
    } else {
      sdiag = meye(c, s);
    }
    mdel(c, &fused);
    mdel(c, &r00);
    mdel(c, &x1tx2);
  }
  /* main loop (bcgs.cpp:294-367) */
  for (long k = 1; k < qb; ++k) {
    long c0 = k * s;
    int has_next = k + 1 < qb;
    mat ycol, omega, z = {0, 0, NULL}, p = {0, 0, NULL}, t_next = {0, 0, NULL};
    if (has_next) {
      span_t L[3] = {{q, c0}, {u, s}, {COL(x, c0 + s), s}};
      span_t Rr[2] = {{u, s}, {COL(x, c0 + s), s}};
      mat g = fused_gram(c, n, L, mode == MODE_PYTH ? 3 : 2, Rr, 2, "fused_gram:wide");
      ycol = msub(c, g, 0, c0, 0, s);
      omega = msub(c, g, c0, c0 + s, 0, s);
      z = msub(c, g, 0, c0, s, 2 * s);
      p = msub(c, g, c0, c0 + s, s, 2 * s);
      if (mode == MODE_PYTH) t_next = msub(c, g, c0 + s, c0 + 2 * s, s, 2 * s);
      mdel(c, &g);
    } else {
      span_t L[2] = {{q, c0}, {u, s}}, Rr[1] = {{u, s}};
      mat g = fused_gram(c, n, L, 2, Rr, 1, "fused_gram:final");
      ycol = msub(c, g, 0, c0, 0, s);
      omega = msub(c, g, c0, c0 + s, 0, s);
      mdel(c, &g);
    }
    mat ydiag = pyth_chol_site(c, omega, ycol, name, "second-pass Pythagorean normalization",
                               k + 1, kappa_power);
    axpy_block(n, u, q, ycol);
    scale_right(c, n, u, ydiag);
    memcpy(COL(q, c0), u, sizeof(double) * (size_t)(n * s));
    mat ys = mmul(c, ycol, sdiag);
    mat col = madd(c, scol, ys, 1.0);
    store_column_blocks(R, s, k, col);
    mat rkk = upper_product(c, ydiag, sdiag);
    r_set_block(R, s, k, k, rkk);
    mdel(c, &ys); mdel(c, &col); mdel(c, &rkk); mdel(c, &omega);
    if (!has_next) {
      mdel(c, &ycol); mdel(c, &ydiag);
      break;
    }
    /* delayed reprojection S2 = Y_diag^{-T} (P - Y^T Z) (bcgs.cpp:336-344) */
    mat ytz = mmul_atb(c, ycol, z);
    mat pm = madd(c, p, ytz, -1.0);
    mat s2 = tri_solve_left_trans(c, ydiag, pm);
    mdel(c, &scol);
    scol = mvstack(c, z, s2);
    memcpy(un, COL(x, c0 + s), sizeof(double) * (size_t)(n * s));
    axpy_block(n, un, q, scol);
    mdel(c, &sdiag);
    if (mode == MODE_TSQR) {
      sdiag = run_tsqr(c, n, s, un, un, NULL, "reduce_factor_tree:tsqr");
    } else if (mode == MODE_PYTH) {
      sdiag = pyth_chol_site(c, t_next, scol, name, "first-pass Pythagorean normalization",
                             k + 2, kappa_power);
      scale_right(c, n, un, sdiag);
    } else {
      sdiag = meye(c, s);
    }
    double* tmp = u; u = un; un = tmp;
    mdel(c, &ycol); mdel(c, &ydiag); mdel(c, &z); mdel(c, &p); mdel(c, &ytz); mdel(c, &pm);
    mdel(c, &s2);
    if (t_next.d) mdel(c, &t_next);
  }
  afree(c, u);
  afree(c, un);
}

/* ------------------------------------------------------------------------------------
 * Public entry points
 * ---------------------------------------------------------------------------------- */
/* check_shape (bcgs.cpp:14-26) + distribute's own check (dist_block.cpp:33-36) */
int or_factor(int variant, const double* x, long n, long m, long s, int procs, double* q,
              double* r, or_stats* st) {
  ctx_t* c = (ctx_t*)calloc(1, sizeof(ctx_t));
  c->st = st;
  c->procs = procs;
  if (st) memset(st, 0, sizeof *st);
  int code = 0;
  if (setjmp(c->jb) == 0) {
    if (procs < 1) fail(c, E_DIM, 0, "run_spmd: procs must be >= 1");
    if (s <= 0 || m % s != 0) fail(c, E_DIM, 0, "distribute: block width must divide the columns");
    if (m == 0) fail(c, E_DIM, 0, "bcgs: column count must be a positive multiple of the block width");
    if (n < m) fail(c, E_DIM, 0, "bcgs: economic factorization needs at least as many rows as columns");
    if (variant < 1 || variant > 5) fail(c, E_CONFIG, 0, "oracle: variant %d out of scope", variant);
    mat R = {m, m, r};
    memset(r, 0, sizeof(double) * (size_t)(m * m));
    memset(q, 0, sizeof(double) * (size_t)(n * m));
    switch (variant) {
      case 1: iro_impl(c, n, m, s, x, q, R); break;
      case 2: pipi_impl(c, n, m, s, x, q, R); break;
      case 3: onesync_impl(c, n, m, s, x, q, R, MODE_PYTH, "BCGSI+P-1S", 2); break;
      case 4: onesync_impl(c, n, m, s, x, q, R, MODE_TSQR, "BCGSI+P-2S", 1); break;
      case 5: onesync_impl(c, n, m, s, x, q, R, MODE_SKIP, "BCGSI+1S", 3); break;
    }
  } else {
    code = c->code;
    if (st) {
      st->pivot = c->pivot;
      snprintf(st->msg, sizeof st->msg, "%s", c->msg);
    }
  }
  arena_release(c);
  free(c);
  return code;
}

void or_gram(const double* a, long n, long ma, const double* b, long mb, double* out) {
  const double** ac = (const double**)malloc(sizeof(double*) * (size_t)(ma + 1));
  const double** bc = (const double**)malloc(sizeof(double*) * (size_t)(mb + 1));
  for (long j = 0; j < ma; ++j) ac[j] = a + (size_t)j * n;
  for (long j = 0; j < mb; ++j) bc[j] = b + (size_t)j * n;
  gram_cols(ac, ma, bc, mb, n, out);
  free(ac);
  free(bc);
}

int or_householder(const double* x, long rows, long cols, double* q, double* r) {
  ctx_t* c = (ctx_t*)calloc(1, sizeof(ctx_t));
  int code = 0;
  if (setjmp(c->jb) == 0) {
    mat X = {rows, cols, (double*)x}, Q, Rm;
    householder(c, X, &Q, &Rm);
    memcpy(q, Q.d, sizeof(double) * (size_t)(Q.r * Q.c));
    memcpy(r, Rm.d, sizeof(double) * (size_t)(Rm.r * Rm.c));
  } else {
    code = c->code;
  }
  arena_release(c);
  free(c);
  return code;
}

int or_chol(const double* a, long n, double* g, int* pivot) {
  mat A = {n, n, (double*)a}, G = {n, n, g};
  int p = chol_raw(A, G);
  if (pivot) *pivot = p;
  return p ? E_NOTSPD : 0;
}

/* two_norm: power iteration on the exact Gram (dense_kernels.cpp:205-239) */
static double two_norm(ctx_t* c, mat a) {
  if (a.r * a.c == 0) return 0.0;
  mat g = gram_m(c, a, a);
  long m = g.r;
  double* v = (double*)amalloc(c, sizeof(double) * (size_t)m);
  double* w = (double*)amalloc(c, sizeof(double) * (size_t)m);
  for (long i = 0; i < m; ++i) v[i] = 1.0 + (double)(i % 13) / 16.0;
  double nv = 0.0;
  for (long i = 0; i < m; ++i) nv += v[i] * v[i];
  nv = sqrt(nv);
  for (long i = 0; i < m; ++i) v[i] /= nv;
  double lambda_prev = 0.0, lambda = 0.0;
  for (int it = 0; it < 5000; ++it) {
    for (long i = 0; i < m; ++i) {
      double acc = 0.0;
      for (long k = 0; k < m; ++k) acc += AT(g, i, k) * v[k];
      w[i] = acc;
    }
    double nw = 0.0;
    for (long i = 0; i < m; ++i) nw += w[i] * w[i];
    nw = sqrt(nw);
    if (nw == 0.0) return 0.0;
    lambda = nw;
    for (long i = 0; i < m; ++i) v[i] = w[i] / nw;
    if (fabs(lambda - lambda_prev) <= 1e-10 * lambda) break;
    lambda_prev = lambda;
  }
  return sqrt(lambda);
}

/* loss_of_orthogonality (metrics.cpp:8-14) */
double or_loo(const double* q, long n, long m) {
  ctx_t* c = (ctx_t*)calloc(1, sizeof(ctx_t));
  double out = NAN;
  if (setjmp(c->jb) == 0) {
    mat Q = {n, m, (double*)q};
    mat g = gram_m(c, Q, Q);
    for (long i = 0; i < m; ++i) AT(g, i, i) -= 1.0;
    out = two_norm(c, g);
  }
  arena_release(c);
  free(c);
  return out;
}

/* residual ||X - QR||_F / ||X||_F (metrics.cpp:16-28), multiply in ijk order */
double or_residual(const double* x, const double* q, const double* r, long n, long m) {
  double* diff = (double*)malloc(sizeof(double) * (size_t)(n * m));
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    for (long j = 0; j < m; ++j) {
      double acc = 0.0;
      for (long k = 0; k < m; ++k) acc += q[(size_t)k * n + i] * r[(size_t)j * m + k];
      diff[(size_t)j * n + i] = x[(size_t)j * n + i] - acc;
    }
  }
  mat D = {n, m, diff}, X = {n, m, (double*)x};
  double num = mfrob(D), den = mfrob(X);
  free(diff);
  return den == 0.0 ? num : num / den;
}

/* ------------------------------------------------------------------------------------
 * gen_matrix (matrix_gen.cpp:18-97): mt19937_64 + Box-Muller, column-major fill
 * ---------------------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} gstream;

static void mt_seed(gstream* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = UINT64_C(6364136223846793005) * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
  g->have_spare = 0;
}

static uint64_t mt_next(gstream* g) {
  const uint64_t UM = UINT64_C(0xFFFFFFFF80000000), LM = UINT64_C(0x7FFFFFFF);
  const uint64_t MA = UINT64_C(0xB5026F5AA96619E9);
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? MA : 0);
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & UINT64_C(0x5555555555555555);
  y ^= (y << 17) & UINT64_C(0x71D67FFFEDA60000);
  y ^= (y << 37) & UINT64_C(0xFFF7EEE000000000);
  y ^= y >> 43;
  return y;
}

static double g_unit(gstream* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

static double g_next(gstream* g) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare;
  }
  double u1 = g_unit(g), u2 = g_unit(g);
  double radius = sqrt(-2.0 * log(1.0 - u1));
  double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
  g->spare = radius * sin(angle);
  g->have_spare = 1;
  return radius * cos(angle);
}

int or_gen_matrix(long n, long m, long s, double kappa, unsigned long long seed, int dist,
                  double* x) {
  if (m < 1 || n < m || s < 1 || m % s != 0) return E_DIM;
  if (!(kappa >= 1.0)) return E_CONFIG;
  gstream* g = (gstream*)malloc(sizeof(gstream));
  mt_seed(g, seed);
  if (dist == 1) {
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < n; ++i) x[(size_t)j * n + i] = g_next(g);
    free(g);
    return 0;
  }
  ctx_t* c = (ctx_t*)calloc(1, sizeof(ctx_t));
  int code = 0;
  if (setjmp(c->jb) == 0) {
    mat gu = mnew(c, n, m), gv = mnew(c, m, m);
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < n; ++i) AT(gu, i, j) = g_next(g);
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < m; ++i) AT(gv, i, j) = g_next(g);
    mat u, ru, v, rv;
    householder(c, gu, &u, &ru);
    mdel(c, &gu);
    householder(c, gv, &v, &rv);
    for (long j = 0; j < m; ++j) {
      double sg = m == 1 ? 1.0 : pow(kappa, -(double)j / (double)(m - 1));
      for (long i = 0; i < n; ++i) AT(u, i, j) *= sg;
    }
    /* multiply(u, v.transposed()) in ijk order */
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < n; ++i) {
        double acc = 0.0;
        for (long k = 0; k < m; ++k) acc += AT(u, i, k) * AT(v, j, k);
        x[(size_t)j * n + i] = acc;
      }
  } else {
    code = c->code;
  }
  arena_release(c);
  free(c);
  free(g);
  return code;
}

/* ------------------------------------------------------------------------------------
 * variant_flops (cost_model.cpp:29-119) and expected_syncs (variant.cpp:53-71)
 * ---------------------------------------------------------------------------------- */
double or_variant_flops(int v, long n, long m, long s) {
  if (s < 1 || m < 1 || m % s != 0 || n < m) return -1.0;
  long q = m / s;
  double dn = (double)n, ds = (double)s;
  double block_qr = 4.0 * dn * ds * ds, block_scale = dn * ds * ds;
#define GU(a, b) (2.0 * dn * (a) * (b))
  if (q == 1) return block_qr;
  double f = 0.0;
  switch (v) {
    case 0:
      f = block_qr;
      for (long k = 1; k < q; ++k) f += GU(k * ds, ds) + GU(k * ds, ds) + block_qr;
      return f;
    case 1:
      f = block_qr;
      for (long k = 1; k < q; ++k) f += 2.0 * (GU(k * ds, ds) + GU(k * ds, ds) + block_qr);
      return f;
    case 2:
      f = block_qr;
      for (long k = 1; k < q; ++k)
        f += 2.0 * GU((k + 1) * ds, ds) + 2.0 * GU(k * ds, ds) + 2.0 * block_scale;
      return f;
    case 3:
      f = block_qr + GU(2.0 * ds, ds) + GU(ds, ds) + block_scale;
      for (long k = 1; k < q; ++k) {
        int hn = k + 1 < q;
        f += hn ? GU(k * ds + 2.0 * ds, 2.0 * ds) : GU(k * ds + ds, ds);
        f += GU(k * ds, ds) + block_scale;
        if (hn) f += GU((k + 1) * ds, ds) + block_scale;
      }
      return f;
    case 5:
      f = block_qr + GU(ds, ds) + GU(ds, ds);
      for (long k = 1; k < q; ++k) {
        int hn = k + 1 < q;
        f += hn ? GU(k * ds + ds, 2.0 * ds) : GU(k * ds + ds, ds);
        f += GU(k * ds, ds) + block_scale;
        if (hn) f += GU((k + 1) * ds, ds);
      }
      return f;
    case 4:
      f = block_qr + GU(ds, ds) + GU(ds, ds) + block_qr;
      for (long k = 1; k < q; ++k) {
        int hn = k + 1 < q;
        f += hn ? GU(k * ds + ds, 2.0 * ds) : GU(k * ds + ds, ds);
        f += GU(k * ds, ds) + block_scale;
        if (hn) f += GU((k + 1) * ds, ds) + block_qr;
      }
      return f;
  }
#undef GU
  return -1.0;
}

long or_expected_syncs(int v, long q) {
  if (q < 1) return -1;
  if (q == 1) return 1;
  switch (v) {
    case 0: return 2 * q - 1;
    case 1: return 4 * q - 3;
    case 2: return 2 * q - 1;
    case 3: return q;
    case 4: return 2 * q - 1;
    case 5: return q;
  }
  return -1;
}
