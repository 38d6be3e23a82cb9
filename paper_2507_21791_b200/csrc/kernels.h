// kernels.h — parameter blocks and host launchers of the sm_100a kernels (K1..K4).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace bgs {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size class (it
// is a host-synchronous driver call; doing it per launch starves the GPU).
cudaError_t ensure_smem_impl(const void* kernel, size_t bytes);
template <typename K>
inline cudaError_t ensure_smem(K kernel, size_t bytes) {
  return ensure_smem_impl(reinterpret_cast<const void*>(kernel), bytes);
}

struct DevStatus;

// ---------------- K1 / K12: the tile engine (gram.cu) ----------------
constexpr int GRAM_FLUSH = 2;                  // stages between double-double folds
// Dynamic shared memory budget per CTA: 227 KB minus the kernel's static shared memory
// and the per-block reservation (kept with margin).
constexpr int TILE_SMEM_MAX = 232448 - 2048;

struct alignas(64) TileParams {
  CUtensorMap map0[5];  // span-0 source, 3-D boxes {16, H, w}, w = 128/64/32/16/8 columns
  CUtensorMap map1[2];  // span-1 source, w = 16/8 columns
  int col0[2];          // first source column of each span
  int units_span[2];    // 8-column units loaded per span
  int lcols[2];         // columns of each span that are output rows (left operand)
  int units;            // units_span[0] + units_span[1]
  int mt_out;           // 8-column m-tiles used as the left operand (a prefix of the tile)
  int nt;               // n-tiles (set by the launcher)
  int N;                // right-operand columns (<= 32)
  int rcol[32];         // tile column of each right-operand column (-1: pad)
  long n_rows;          // rows of this shard
  long total_stages;    // set by the launcher
  int stages;           // pipeline depth
  int H;                // 16-row blocks per stage (stage rows RS = 16 H)
  double* partial;      // per-CTA (hi, lo) partials
  const DevStatus* status;
  // K12: fused block update in front of the Gram (ignored by K1)
  int upd_a, upd_b, kp, s, colA, colB;
  const double* CA; int ldca; const double* TA;
  const double* CB; int ldcb; const double* TB;
  double* dstA; long lddA;
  double* dstB; long lddB;
  unsigned long long* phase;  // BGS_TILE_PROF: per-CTA cycle counters [grid][8] (or null)
  int dbg;  // experiment mask (BGS_TILE_DBG): 1 no proxy fence, 2 no global stores,
            // 4 no update MMAs, 8 no Gram MMAs, 16 no epilogue
  int comp_t0;  // first compensated output tile (>= mt_out: none; every 4-row k-step of
                // tiles >= comp_t0 is folded into their double-double at once)
};

cudaError_t tile_launch(TileParams& p, bool upd, int grid, cudaStream_t st, int* launches);
bool tile_fused_supported(int s, int kp, int mt_out);
size_t tile_smem_bytes(int H, int stages, int units, bool upd);
// Deterministic double-double sum over `ctas` partial slots -> compact M x N Gram
// (M = lcols[0] + lcols[1]).
// ld_out > 0: write into a larger Gram (column stride ld_out; chunked left operands)
cudaError_t gram_reduce_launch(const TileParams& p, int ctas, double* out, cudaStream_t st,
                               int* launches, int ld_out = 0);
int gram_n_tiles(int N);
size_t gram_partial_doubles_per_cta(int mt_out, int N);

// ---------------- K12c: cluster-split fused update + Gram (k12.cu) ----------------
// Stages of 32 R rows on ping-pong consumer warpgroups; with cluster = 2 a CTA pair shares
// each stage: rank r loads its own span-0 units plus the extra (A-block) units it needs and
// all of span 1, and the partial block update is exchanged through distributed shared
// memory.  s <= 4, N <= 8.  One (hi, lo) partial slot per cluster.
struct alignas(64) SplitParams {
  CUtensorMap map0[5];  // span 0, boxes {16, 2, w}, w = 128/64/32/16/8
  CUtensorMap map1[2];  // span 1, w = 16/8
  int col0[2];          // first source column of each span
  int U0, U1;           // 8-column units of span 0 / span 1
  int ncols0;           // columns of span 0 (all are output rows)
  int lcols1;           // output-row columns of span 1 (rank 0 emits them)
  int s1_left;          // ceil(lcols1 / 8)
  int own_u0[4], own_n[4];  // per cluster rank: owned span-0 units
  int ext_u0[4], ext_n[4];  // per cluster rank: extra span-0 units (the A block)
  int slot_units;       // max local units over the two ranks
  int mt_out;           // global 8-column output tiles (U0 + s1_left)
  int N;                // right-operand columns (<= 8), all in span 1
  int rcol1[8];         // span-1 column of each right-operand column (-1: pad)
  long n_rows;
  long total_stages;    // 32-row stages of the shard
  int stages;           // ring depth
  int cluster;          // CTAs per cluster: 1 (whole tile per CTA), 2 or 4 (split prefix)
  int R;                // 32-row chunks per stage (1, 2, 4)
  int kw, mtw;          // k-steps / output tiles per warp (planned; selects the instance)
  int upd_a, upd_b, kp, s;
  const double* CA; int ldca; const double* TA;
  const double* CB; int ldcb; const double* TB;
  double* dstA; long lddA;
  double* dstB; long lddB;
  double* partial;      // (hi, lo) partials, one slot per (cluster, consumer group)
  const DevStatus* status;
  unsigned long long* phase;
  int dbg;
  int pdl;              // launched as a programmatic dependent of the merged reduce + step
  int comp_t0;          // first compensated output tile (>= mt_out: none; k12_ct.cu)
};
// Plans the rank split for a fused Gram of the given shape; false when K12c does not
// apply (then the caller uses tile_launch).  Fills own/ext ranges, slot_units, stages.
bool k12_plan(SplitParams& p);
size_t k12_smem_bytes(int stages, int slot_units, int R, int C);
cudaError_t k12_launch(const SplitParams& p, int grid, cudaStream_t st, int* launches);
// CTAs a launch of cluster width C may use: C x the clusters that can be co-resident
// (clusters of 4 do not tile all 148 SMs), at most `sms`
int k12_grid_cap(int C, int sms);

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
int update_max_kp(int s);

// ---------------- K2m: the s = 8 / 16 update fed by TMA (update_tma.cu) ----------------
struct alignas(64) UpdTmaParams {
  CUtensorMap map[5];  // the Q buffer, 3-D boxes {16, 2, w}, w = 128/64/32/16/8
  int col0;            // first prefix column in the map
  long n_rows;
  long total_blocks;   // 32-row blocks (set by the launcher)
  int kp, s;           // kp: multiple of 8
  int stages;          // ring depth (set by the launcher)
  int has_a, has_b, cb_has_a;
  const double* srcA; long ld_srcA; double* dstA; long ld_dstA;
  const double* CA; long ldca; const double* TA;
  const double* srcB; long ld_srcB; double* dstB; long ld_dstB;
  const double* CB; long ldcb; const double* TB;
  const DevStatus* status;
  double* coef_ws;     // >= update_tma_coef_doubles(s, kp): the packed coefficient fragments
};
cudaError_t update_tma_launch(UpdTmaParams& p, int num_sms, cudaStream_t st, int* launches);
size_t update_tma_coef_doubles(int s, int kp);
int update_tma_max_kp(int s);
size_t update_tma_smem_bytes(int s, int kp, int stages);

// ---------------- K3: replicated small factor ops (small.cu) ----------------
enum SmallMode : int {
  SM_ONESYNC_PROLOGUE = 1,  // scol = R00^{-T} G0[0:s]; Sd = pyth ? chol(T - scol^T scol) : I
  SM_ONESYNC_STEP = 2,      // Yd, R column, S2, next scol / Sd (bcgs.cpp:294-367)
  SM_PIPI_PROJ = 3,         // Sd = chol(T - S^T S), keep S (bcgs.cpp:185-197)
  SM_PIPI_REPROJ = 4,       // Yd = chol(Omega - Y^T Y), R column (bcgs.cpp:199-216)
  SM_IRO_SAVE = 5,          // keep S1 = Q^T X_k (bcgs.cpp:151-153)
  SM_IRO_FINISH = 6,        // R column = S1 + S2 R1, R_kk = R2 R1 (bcgs.cpp:162-164)
  SM_COPY_RBLOCK = 7,       // R(0,0) = TSQR root (bcgs.cpp:83-90, 142-146)
  SM_CLASSIC_FINISH = 8,    // R column = S (saved), R_kk = intra-block R (bcgs.cpp:126-128)
  SM_CHOLQR = 9,            // R_kk = chol(U^T U) -> sdiag (cholqr, intraorth.cpp:136-151)
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
  int unstaged;                   // set by small_launch: operands too large for shared memory
};
cudaError_t small_launch(const SmallParams& p, cudaStream_t st, int* launches);
// gram_reduce followed by the s <= 4 one-sync step in one launch (single-GPU contexts: the
// step needs the fully reduced Gram, so no allreduce may sit in between).
struct ReduceArgs;
ReduceArgs reduce_args(const TileParams& p, int ctas, double* out, int ld_out);
bool small_mergeable(const SmallParams& p);

cudaError_t gram_reduce_launch_args(const ReduceArgs& a, int entries, cudaStream_t st,
                                    int* launches);
cudaError_t reduce_small_launch(const ReduceArgs& r, int entries, const SmallParams& p,
                                unsigned* ticket, int sms, cudaStream_t st, int* launches);

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
// Grouped tree of one shard's leaves [leaf_base, leaf_base + Lt): up -> root_out; down from
// mtop (identity if null) -> the leaf M's (tsqr.cu).
cudaError_t tsqr_tree_up_shard(double* ws, int L, int leaf_base, int Lt, int s, double* root_out,
                               const DevStatus* status, cudaStream_t st, int* launches);
cudaError_t tsqr_tree_down_shard(double* ws, int L, int leaf_base, int Lt, int s,
                                 const double* mtop, const DevStatus* status, cudaStream_t st,
                                 int* launches);
// Apply M_leaf to one shard's Q rows, M_leaf walked down the tree from mtop in the kernel
// (replaces tsqr_tree_down_shard + tsqr_apply_launch for s in {1, 2, 4, 8, 16}).
cudaError_t tsqr_apply_path_shard(double* dst, long ldd, const long* d_bounds, double* ws, int L,
                                  int leaf_base, int Lt, int s, const double* mtop,
                                  const DevStatus* status, cudaStream_t st, int* launches);
// Q rows of leaf l <- Q rows * M_l (in place; M_l precomputed by tsqr_tree_down_shard).
cudaError_t tsqr_apply_launch(double* dst, long ldd, const long* d_bounds, int L, int s,
                              const double* M, const DevStatus* status, cudaStream_t st,
                              int* launches);
// The cross-shard tree over `n` root factors (one per rank): root R -> rout (ld ldrout),
// M_r for each rank -> mout + r*s*s.  Deterministic; identical on every rank.
cudaError_t tsqr_cross_launch(const double* roots, int n, int s, double* ws2, double* rout,
                              int ldrout, double* mout, const DevStatus* status,
                              cudaStream_t st, int* launches);

// ---------------- peer.cu: one-shot exchange over peer-mapped windows ----------------
// Window of a rank: [flags: P x u32 in kPeerFlagBytes][parity 0: P slots][parity 1: P slots]
constexpr int kPeerMaxRanks = 8;
constexpr size_t kPeerFlagBytes = 256;
struct PeerView {
  unsigned char* win[kPeerMaxRanks];  // every rank's window as mapped here (win[rank]: local)
  int P, rank;
  unsigned long slot_bytes;  // bytes per (parity, source rank) slot
};
inline size_t peer_window_bytes(int P, size_t slot_bytes) { return kPeerFlagBytes + 2 * (size_t)P * slot_bytes; }
// Store [a (na doubles) | b (nb doubles)] into slot (epoch & 1, rank) of every window, then
// flag[rank] = epoch there (release, system scope).  cnt: P zeroed u32 tickets (local).
cudaError_t peer_push_launch(const PeerView& v, const double* a, unsigned long na, const double* b,
                             unsigned long nb, unsigned epoch, unsigned* cnt, cudaStream_t st,
                             int* launches);
// recv[r * ng + i] = rank r's gather part; sum[i] = the ns partials added in rank order.
// spin: wait in the kernel for the P flags (distinct GPUs only).
// status (optional): the in-kernel wait gives up after ~8 s and records ST_COLLECTIVE there.
struct DevStatus;
cudaError_t peer_sum_launch(const PeerView& v, unsigned long ng, double* recv, unsigned long ns,
                            double* sum, unsigned epoch, bool spin, cudaStream_t st, int* launches,
                            DevStatus* status = nullptr);

// The one-sync step fused with the exchange (small.cu): A = reduce + push + flags, B =
// [spin] + rank-ordered sum + step, AB = both in one launch (in-kernel spin).
struct ReduceArgs;
struct ReducePush;
struct SmallParams;
cudaError_t reduce_push_launch(const ReduceArgs& r, int entries, const ReducePush& push,
                               const PeerView& v, unsigned epoch, unsigned* ticket, int sms,
                               cudaStream_t st, int* launches);
cudaError_t sum_small_launch(const PeerView& v, unsigned epoch, bool spin, unsigned long words,
                             double* G, const SmallParams& p, unsigned* ticket, int sms,
                             cudaStream_t st, int* launches);
cudaError_t reduce_xchg_small_launch(const ReduceArgs& r, int entries, const ReducePush& push,
                                     const PeerView& v, unsigned epoch, unsigned long words,
                                     double* G, const SmallParams& p, unsigned* ticket, int sms,
                                     cudaStream_t st, int* launches);

// ---------------- misc (misc.cu) ----------------
cudaError_t gen_gaussian_launch(unsigned long long seed, long row0, long n_local, long m,
                                double* x, long ldx, cudaStream_t st);
cudaError_t copy_cols_launch(const double* src, long lds, double* dst, long ldd, long rows,
                             long cols, cudaStream_t st);
// Sum of squares of (X - Q R) and of X, scaled by the host-supplied maxima, per-CTA
// partials -> out[0..1] (double-double reduced).
// ||A||_2 of a symmetric m x m device matrix (optionally A - I first, in place) by the
// reference's power iteration on A^T A; ws >= 3 m + 8 doubles.  Synchronizes `st`.
cudaError_t sym_two_norm(double* A, int m, bool sub_identity, double* ws, double* out,
                         cudaStream_t st);
cudaError_t residual_launch(const double* x, long ldx, const double* q, long ldq,
                            const double* r, long ldr, long n_rows, long m, double inv_scale_d,
                            double inv_scale_x, double* ws, double* out, int num_sms,
                            cudaStream_t st);

}  // namespace bgs
