// kernels.h — parameter blocks and host launchers of the sm_100a kernels (K1..K4).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace bgs {

struct DevStatus;

// ---------------- K1: Gram (gram.cu) ----------------
constexpr int GRAM_FLUSH = 4;               // stages (x16 rows) between double-double folds
constexpr int GRAM_SMEM_BUDGET = 210 * 1024;  // bytes of stage ring per CTA

struct alignas(64) GramParams {
  CUtensorMap map[2];  // span 0 / span 1 sources (column-major, box 16 rows x 8 cols)
  int col0[2];         // first source column of each span
  int ncols[2];        // loaded columns of each span
  int lcols[2];        // columns of each span that are rows of the output (left operand)
  int nbox[2];         // 8-column boxes of each span
  int nboxes;          // nbox[0] + nbox[1]
  int mt_out;          // boxes used as the left operand: nbox[0] or nboxes
  int nt;              // n-tiles (set by the launcher)
  int N;               // right-operand columns (<= 32)
  int rcol[32];        // tile column of each right-operand column (-1: pad)
  long n_rows;         // rows of this shard
  long total_stages;   // set by the launcher
  int stages;          // pipeline depth (set by the launcher)
  double* partial;     // per-CTA (hi, lo) partials
  const DevStatus* status;
};

// Per-CTA partials of one shard (p.partial already offset to this shard's first CTA).
cudaError_t gram_partials_launch(GramParams& p, int grid, cudaStream_t st, int* launches);
// Deterministic double-double sum over `ctas` partial slots -> compact M x N Gram
// (M = lcols[0] + lcols[1]).
cudaError_t gram_reduce_launch(const GramParams& p, int ctas, double* out, cudaStream_t st,
                               int* launches);
int gram_n_tiles(int N);
size_t gram_partial_doubles_per_cta(int mt_out, int N);

// ---------------- K2: block update (update.cu) ----------------
struct UpdateParams {
  long n_rows;
  const double* qp;  // prefix Q[:, 0:kp]
  long ldq;
  int kp;
  int s;
  int has_a, has_b, cb_has_a;
  const double* srcA; long ld_srcA; double* dstA; long ld_dstA;
  const double* CA; long ldca; const double* TA; long ldta;
  const double* srcB; long ld_srcB; double* dstB; long ld_dstB;
  const double* CB; long ldcb; const double* TB; long ldtb;
  const DevStatus* status;
};
cudaError_t update_launch(const UpdateParams& p, int num_sms, cudaStream_t st, int* launches);

// ---------------- K3: replicated small factor ops (small.cu) ----------------
enum SmallMode : int {
  SM_ONESYNC_PROLOGUE = 1,  // scol = R00^{-T} G0[0:s]; Sd = pyth ? chol(T - scol^T scol) : I
  SM_ONESYNC_STEP = 2,      // Yd, R column, S2, next scol / Sd (bcgs.cpp:294-367)
  SM_PIPI_PROJ = 3,         // Sd = chol(T - S^T S), keep S (bcgs.cpp:185-197)
  SM_PIPI_REPROJ = 4,       // Yd = chol(Omega - Y^T Y), R column (bcgs.cpp:199-216)
  SM_IRO_SAVE = 5,          // keep S1 = Q^T X_k (bcgs.cpp:151-153)
  SM_IRO_FINISH = 6,        // R column = S1 + S2 R1, R_kk = R2 R1 (bcgs.cpp:162-164)
  SM_COPY_RBLOCK = 7,       // R(0,0) = TSQR root (bcgs.cpp:83-90, 142-146)
};
// onesync sub-modes (SDiagMode, bcgs.cpp:223-231)
enum OnesyncMode : int { OS_PYTH = 0, OS_SKIP = 1, OS_TSQR = 2 };

struct SmallParams {
  int mode;
  int os_mode;     // OnesyncMode
  int s;
  int k;           // 0-based block index of the current step
  int kp;          // k * s (prefix width)
  int has_next;
  int kappa_power;
  const double* G; int ldg;       // reduced Gram of this step
  int gm, gn;                     // its shape (checked for non-finite entries)
  double* R; int ldr;             // device R (m x m)
  const double* scol_prev; int ld_scol_prev;  // S_{1:k, k+1} from the previous step
  double* scol_next; int ld_scol_next;        // next scol ((kp+s) x s)
  double* sdiag;                  // S_{k+1,k+1}: read as previous, written as next (s x s)
  double* sdiag_prev_copy;        // scratch copy of the previous sdiag (s x s)
  double* ydiag;                  // Y_kk (s x s)
  const double* rtop; int ldrtop; // TSQR root R for prologue / copy modes
  const double* aux1; int ldaux1; // IRO: S1 / R1 ; PIPI: saved scol
  const double* aux2; int ldaux2; // IRO: R2
  double* save; int ldsave;       // where SM_IRO_SAVE / SM_PIPI_PROJ keep S
  DevStatus* status;
};
cudaError_t small_launch(const SmallParams& p, cudaStream_t st, int* launches);

// ---------------- K4: TSQR (tsqr.cu) ----------------
// Workspace for a TSQR over L leaves of width s: regions [R | Rtmp | M | Mtmp] of
// L*s*s doubles each, then node Q factors (L * 2s*s).
size_t tsqr_ws_bytes(int leaves, int s);
inline double* tsqr_ws_R(double* ws) { return ws; }
inline double* tsqr_ws_M(double* ws, int L, int s) { return ws + (size_t)2 * L * s * s; }
// Leaf QR of the rows [bounds[l], bounds[l+1]) (l < L) of a tall block: explicit Q_leaf in
// place into dst, R_leaf (s x s, nonnegative diagonal) into rleaf + l*s*s.
cudaError_t tsqr_leaf_launch(const double* src, long lds, double* dst, long ldd,
                             const long* d_bounds, int L, long hmax, int s, double* rleaf,
                             const DevStatus* status, cudaStream_t st, int* launches);
// Bottom-up combine of every tree t (leaves [tree_off[t], tree_off[t+1])) -> roots + t*s*s.
cudaError_t tsqr_up_launch(int n_trees, const int* d_tree_off, double* ws, int L, int s,
                           double* roots, const DevStatus* status, cudaStream_t st,
                           int* launches);
// Top-down: per-leaf M (region M) from each tree's root matrix mtop + t*s*s.
cudaError_t tsqr_down_launch(int n_trees, const int* d_tree_off, double* ws, int L, int s,
                             const double* mtop, const DevStatus* status, cudaStream_t st,
                             int* launches);
// Q rows of leaf l <- Q rows * M_l (in place).
cudaError_t tsqr_apply_launch(double* dst, long ldd, const long* d_bounds, int L, int s,
                              const double* M, const DevStatus* status, cudaStream_t st,
                              int* launches);
// The cross-shard tree over `n` root factors (one per rank): root R -> rout (ld ldrout),
// M_r for each rank -> mout + r*s*s.  Deterministic; identical on every rank.
cudaError_t tsqr_cross_launch(const double* roots, int n, int s, double* ws2, double* rout,
                              int ldrout, double* mout, const DevStatus* status,
                              cudaStream_t st, int* launches);

// ---------------- misc (misc.cu) ----------------
cudaError_t gen_gaussian_launch(unsigned long long seed, long row0, long n_local, long m,
                                double* x, long ldx, cudaStream_t st);
cudaError_t copy_cols_launch(const double* src, long lds, double* dst, long ldd, long rows,
                             long cols, cudaStream_t st);
// Sum of squares of (X - Q R) and of X, scaled by the host-supplied maxima, per-CTA
// partials -> out[0..1] (double-double reduced).
cudaError_t residual_launch(const double* x, long ldx, const double* q, long ldq,
                            const double* r, long ldr, long n_rows, long m, double inv_scale_d,
                            double inv_scale_x, double* ws, double* out, int num_sms,
                            cudaStream_t st);
cudaError_t maxabs_launch(const double* x, long ldx, long n_rows, long m, double* ws,
                          double* out, int num_sms, cudaStream_t st);
cudaError_t sum_into_launch(double* dst, const double* src, long count, cudaStream_t st);

}  // namespace bgs
