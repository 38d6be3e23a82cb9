/* bgs_gpu.h — C ABI of the B200-native low-synchronization BCGS QR (paper 2507.21791).
 *
 * This is the drop-in boundary for the reference's CPU QR path.  The reference has no
 * FFI layer; its boundary is the C++ API in the headers under
 * /root/reference/proj/include/blockgs.  Each entry point below names the reference interface it replaces.
 * Plain pointers and sizes only: no torch, no C++ types.  All matrices are column-major
 * fp64 with an explicit leading dimension (dense_matrix.hpp:21-22 layout contract).
 *
 * Compute runs on hand-written sm_100a kernels (TMA + DMMA Gram, fused block update,
 * on-device small factor ops, on-device TSQR); the single synchronization of each block
 * step is one NCCL allreduce when the context spans several GPUs (or one exchange through
 * a caller-supplied host communicator, bgs_ctx_create_host_comm).  There is no CPU
 * fallback: on a host without a usable B200 every compute entry point returns
 * BGS_E_CUDA.
 */
#ifndef BGS_GPU_H
#define BGS_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 1:1 with the exception taxonomy of errors.hpp:9-51
 * (DimensionError, NotSpdError, SingularError, RankDeficientError, NonFiniteError,
 * CollectiveError, ConfigError) plus CUDA/driver failures. */
enum {
  BGS_OK = 0,
  BGS_E_DIMENSION = 1,
  BGS_E_NOT_SPD = 2,
  BGS_E_SINGULAR = 3,
  BGS_E_RANK_DEFICIENT = 4,
  BGS_E_NON_FINITE = 5,
  BGS_E_COLLECTIVE = 6, /* NCCL failure or rank mismatch */
  BGS_E_CONFIG = 7,
  BGS_E_INTERNAL = 8,
  BGS_E_CUDA = 9 /* no device / CUDA error / kernel image missing */
};

/* Variant ids: same order and meaning as blockgs::VariantId (variant.hpp:8-15). */
enum {
  BGS_BCGS = 0, /* classic BCGS: out of scope (returns BGS_E_CONFIG) */
  BGS_BCGSI_PLUS = 1,
  BGS_BCGSPIPI_PLUS = 2,
  BGS_BCGSI_PLUS_P_1S = 3,
  BGS_BCGSI_PLUS_P_2S = 4,
  BGS_BCGSI_PLUS_1S = 5
};

#define BGS_LABELS_CAP 65536

/* SyncStats (sync_stats.hpp:13-27): one event per collective rendezvous, labels in
 * issue order, '\n'-joined, using the reference's label strings. */
typedef struct {
  long sync_count;
  long words_reduced;
  int n_events;
  char labels[BGS_LABELS_CAP];
} bgs_stats;

/* Error detail.  For BGS_E_NOT_SPD, `pivot` is the 1-based Cholesky pivot
 * (NotSpdError::pivot, errors.hpp:40-44) and `msg` carries the reference's semantic
 * diagnostic (bcgs.cpp:69-80): "<variant>: <site> for block column <k> hit a Gram matrix
 * that is not numerically positive definite (...); likely violated working assumption:
 * O(u) * kappa(X)^p <= 1". */
typedef struct {
  int code;
  int pivot;
  long block; /* 1-based block column of a NotSpd abort, else 0 */
  char site[96];
  char msg[1024];
} bgs_error;

/* Per-call device timing (CUDA events on the factorization stream). */
typedef struct {
  double factor_ms; /* X resident on the device -> Q, R resident; excludes H2D/D2H */
  double total_ms;  /* whole call as seen by the host */
  long kernel_launches; /* our kernels launched by the factorization */
} bgs_timing;

typedef struct bgs_ctx bgs_ctx;

/* ---- algorithm-selection API (variant.hpp:17-39, cost_model.hpp:37) --------------- */
const char* bgs_variant_name(int variant);                 /* variant.cpp:18-34 */
int bgs_parse_variant(const char* name, int* variant, bgs_error* err); /* variant.cpp:43-51 */
long bgs_expected_syncs(int variant, long q);              /* variant.cpp:53-71 */
double bgs_variant_flops(int variant, long n, long m, long s); /* cost_model.cpp:29-119 */
int bgs_shard_rows(long n, int procs, int rank, long* row0, long* rows); /* dist_block.cpp:33-44 */

/* ---- context: device, stream, NCCL communicator, workspaces -----------------------
 * Replaces Communicator + run_spmd's per-rank setup (communicator.hpp:50-152).
 * nranks == 1: single GPU, no NCCL unless nccl_unique_id is non-null (then a one-rank
 * communicator carries the same collectives as the multi-GPU path).  nranks > 1: one
 * process (or thread) per GPU; nccl_unique_id points to the 128-byte ncclUniqueId shared
 * by all ranks. */
int bgs_ctx_create(int device, int rank, int nranks, const void* nccl_unique_id,
                   bgs_ctx** out, bgs_error* err);
/* A context whose collectives go through a caller-supplied host communicator instead of
 * NCCL -- the reference's Communicator (communicator.hpp:98-152) as a callback.  `fn` is
 * a blocking allgather: every rank passes `bytes` bytes in `send` and receives all ranks'
 * buffers in rank order in `recv` (nranks * bytes); it returns 0 on success.  Each sync
 * of the algorithm (a Gram allreduce, a TSQR root exchange with its fused Gram) is ONE
 * call: the partials are gathered and summed in rank order on the host, so R is bitwise
 * replicated (exact_allreduce, communicator.cpp:226-250).  Uses: ranks that share a GPU
 * (tests: several processes on one device, where NCCL refuses), or a transport NCCL does
 * not cover.  No kernel ever waits on another rank: the exchange is between launches. */
typedef int (*bgs_allgather_fn)(void* user, const void* send, void* recv, unsigned long bytes);
int bgs_ctx_create_host_comm(int device, int rank, int nranks, bgs_allgather_fn fn, void* user,
                             bgs_ctx** out, bgs_error* err);
/* A context whose collectives are ONE-SHOT exchanges over peer-mapped device memory
 * (SURVEY.md 8(f) row 4): exact_allreduce (communicator.cpp:226-250) and the TSQR root
 * exchange fused with its Gram allreduce (communicator.cpp:252-317) re-designed for GPUs
 * that address each other's memory -- NVLink / NVSwitch P2P between the GPUs of a node, or
 * CUDA IPC between processes.  Each rank owns a window [flags | 2 parities x nranks
 * slots]; a sync is: every rank stores its partial into its slot of EVERY window and
 * then publishes a flag there (release, system scope); every rank waits for the nranks
 * flags of its own window and adds the partials in rank order (bitwise replicated R).
 * One network traversal, no host round trip, no second phase.
 *   bgs_ctx_create_peer   allocates the window (slot_bytes 0: sized for the largest
 *                         exchange the library admits, 1 MiB per slot);
 *   bgs_ctx_peer_handle   exports it (BGS_PEER_HANDLE_BYTES; ranks allgather these);
 *   bgs_ctx_peer_attach   maps all nranks windows (handles in rank order).
 * wait_mode 0 picks how a rank waits: 2 = an acquire spin at the head of the sum kernel
 * when every rank has its own GPU; 1 = stream memory operations (cuStreamWaitValue32)
 * when ranks share a GPU, where no kernel may wait on another rank's kernel.  */
#define BGS_PEER_HANDLE_BYTES 128
int bgs_ctx_create_peer(int device, int rank, int nranks, unsigned long slot_bytes, bgs_ctx** out,
                        bgs_error* err);
int bgs_ctx_peer_handle(bgs_ctx* ctx, void* handle, bgs_error* err);
int bgs_ctx_peer_attach(bgs_ctx* ctx, const void* handles, int wait_mode, bgs_error* err);
/* Protocol self-test on one GPU: nranks emulated ranks in this process, `epochs` exchanges
 * of ng gathered + ns summed doubles; pushes, a device synchronize, then the spin flavour
 * of the sum kernel (nothing ever waits); results checked bitwise. */
int bgs_peer_selftest(int device, int nranks, long ng, long ns, int epochs, bgs_error* err);
void bgs_ctx_destroy(bgs_ctx* ctx);
int bgs_nccl_unique_id(void* out128, bgs_error* err); /* ncclGetUniqueId via the ctx's NCCL */
/* The *_device entry points below run on the context's own stream and first wait (an
 * event, no host sync) for all work queued so far on the caller's stream, so buffers the
 * caller filled asynchronously are safe to pass.  Default: the legacy default stream
 * (torch's default).  `stream` is a cudaStream_t.  Results are complete on return. */
int bgs_ctx_set_stream(bgs_ctx* ctx, void* stream);
int bgs_device_info(int device, int* sm_count, long* hbm_bytes, char* name, long name_cap);

/* ---- BcgsOptions (bcgs.hpp:19-30) ---------------------------------------------------
 * `probe` is RecurrenceProbe::on_eval: the one-sync variants (BCGSI+P-1S, BCGSI+P-2S,
 * BCGSI+1S) call it once per delayed reprojection (bcgs.cpp:339-343) with the 1-based
 * block index k of Q_k, the s x s recurrence S2 (column-major, host), and this shard's
 * rows of Q_k and X_{k+1} (host copies, n_local x s, ld n_local), so a test can form the
 * never-communicated product Q_k^T X_{k+1} directly.  `shard` is the rank (the emulated
 * shard under bgs_factor with procs > 1).  Firing it synchronizes the stream once per
 * step (a debugging hook, like the reference's).  classic_intra is accepted for API
 * parity; classic BCGS is out of scope, so it has no effect. */
typedef void (*bgs_probe_fn)(void* user, long k, const double* s2, long s, const double* q_local,
                             const double* x_local, long n_local, int shard);
typedef struct {
  int classic_intra; /* IntraorthKind: 0 Tsqr (default), 1 CholQr -- unused on this path */
  bgs_probe_fn probe;
  void* probe_user;
} bgs_options;

/* ---- drop-in for run_factor (runner.hpp:28-29, runner.cpp:39-67) ------------------
 * Host X (n x m, ldx) in; Q (n x m, ldq, gathered in rank order like gather_rows) and
 * R (m x m upper, ldr; strict lower triangle exact zeros) out.  `procs` is the
 * reference's process count: on a single-GPU context procs > 1 runs the row-sharded
 * algorithm with `procs` shards emulated on the one device (rank-ordered reductions,
 * one sync per collective), mirroring the reference's simulated backend.
 * NotSpd returns BGS_E_NOT_SPD with the diagnostic in err (FactorOutcome.ok = false). */
int bgs_factor(bgs_ctx* ctx, int variant, long n, long m, long s, int procs,
               const double* x, long ldx, double* q, long ldq, double* r, long ldr,
               bgs_stats* stats, bgs_timing* timing, bgs_error* err);
/* run_factor(v, x, s, procs, opts): the same with BcgsOptions (opts may be NULL). */
int bgs_factor_opts(bgs_ctx* ctx, int variant, long n, long m, long s, int procs,
                    const double* x, long ldx, double* q, long ldq, double* r, long ldr,
                    const bgs_options* opts, bgs_stats* stats, bgs_timing* timing,
                    bgs_error* err);

/* ---- device-resident per-rank entry (run_variant on a DistBlockMatrix,
 * bcgs.hpp:49-50).  This rank owns rows [row0, row0 + n_local) of the global n x m
 * matrix (the ceil split of dist_block.cpp:37-43).  d_x / d_q are device pointers
 * (n_local x m, leading dimensions ldx / ldq >= n_local rounded up to 16, 16-byte aligned
 * columns: the TMA tile engine reads whole 16-row blocks; rows past n_local are ignored).  R is replicated: written to
 * host memory h_r (m x m, ldr) identically on every rank.  Collectives use the ctx's
 * NCCL communicator (nranks > 1). */
int bgs_factor_device(bgs_ctx* ctx, int variant, long n, long m, long s, long row0,
                      long n_local, const double* d_x, long ldx, double* d_q, long ldq,
                      double* h_r, long ldr, bgs_stats* stats, bgs_timing* timing,
                      bgs_error* err);
/* run_variant(v, x, comm, opts) (bcgs.hpp:49-50): the same with BcgsOptions. */
int bgs_factor_device_opts(bgs_ctx* ctx, int variant, long n, long m, long s, long row0,
                           long n_local, const double* d_x, long ldx, double* d_q, long ldq,
                           double* h_r, long ldr, const bgs_options* opts, bgs_stats* stats,
                           bgs_timing* timing, bgs_error* err);

/* ---- inputs and verification on the device (matrix_gen.hpp:27, metrics.hpp:10-20) -- */
/* Seeded i.i.d. N(0,1) entries X(i,j) for global rows [row0, row0+n_local): a
 * counter-based Philox stream keyed by (seed, global row, column), so the global matrix
 * is independent of how it is sharded.  Not the reference's mt19937_64 sequence. */
int bgs_gen_gaussian_device(bgs_ctx* ctx, unsigned long long seed, long row0, long n_local,
                            long m, double* d_x, long ldx, bgs_error* err);
/* Host-side bitwise port of the reference generator's Gaussian mode
 * (matrix_gen.cpp:18-56: mt19937_64 + Box-Muller, column-major fill). */
int bgs_gen_gaussian_host(unsigned long long seed, long n, long m, double* x, long ldx);
/* Host-side bitwise port of gen_matrix (matrix_gen.cpp:18-97), both modes: gaussian != 0
 * gives the raw N(0,1) draws, gaussian == 0 the geometric family X = U diag(sigma) V^T
 * (Householder Q factors of seeded Gaussians, sigma_i = kappa^(-i/(m-1))).  Same checks
 * and error wording as the reference (DimensionError / ConfigError).  O(n m^2) on one
 * core: for driver-sized inputs (the bench configs), not for BASELINE config 5. */
int bgs_gen_matrix_host(long n, long m, long s, double kappa, unsigned long long seed,
                        int gaussian, double* x, long ldx, bgs_error* err);
/* loss_of_orthogonality = ||Q^T Q - I||_2 and residual ||X - QR||_F / ||X||_F
 * computed on the GPU for a (sharded) device-resident factorization; the Gram and the
 * residual sum are reduced over ranks with NCCL. */
/* Same metrics for host-resident X, Q, R (uploads them; single-GPU context). */
int bgs_metrics(bgs_ctx* ctx, long n, long m, const double* x, long ldx, const double* q,
                long ldq, const double* r, long ldr, double* loo, double* resid, bgs_error* err);
int bgs_metrics_device(bgs_ctx* ctx, long n, long m, long n_local, const double* d_x,
                       long ldx, const double* d_q, long ldq, const double* h_r, long ldr,
                       double* loo, double* resid, bgs_error* err);

/* ---- live per-kernel profile (CUDA events on the factorization stream) -------------
 * When enabled, every kernel class launched by the factorization is bracketed by CUDA
 * events; bgs_profile_read returns, per class, launches, summed device time and the
 * ALGORITHMIC bytes / flops those launches had to move / do.
 * Reading resets the accumulators. */
typedef struct {
  char name[32];
  long launches;
  double ms;
  double alg_bytes;
  double alg_flops;
} bgs_kernel_stat;
int bgs_profile_enable(bgs_ctx* ctx, int on);
int bgs_profile_read(bgs_ctx* ctx, bgs_kernel_stat* out, int cap, int* count);

/* ---- building blocks exposed for parity tests ------------------------------------ */
/* Tall-skinny Gram A^T B (dense_kernels.hpp:15-24) through the K1 TMA/DMMA kernel:
 * host in/out, out is ma x mb (ld = ma). */
int bgs_gram(bgs_ctx* ctx, const double* a, long n, long ma, const double* b, long mb,
             double* out, bgs_error* err);
/* TSQR of a tall block (intraorth.hpp:22-27) through the K4 kernels: host in/out. */
int bgs_tsqr(bgs_ctx* ctx, const double* x, long n, long s, double* q, double* r,
             bgs_error* err);

#ifdef __cplusplus
}
#endif
#endif /* BGS_GPU_H */
