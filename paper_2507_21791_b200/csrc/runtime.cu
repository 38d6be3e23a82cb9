// runtime.cu — host runtime and C ABI (include/bgs_gpu.h).
//
// Per-variant drivers restate the control flow of the reference's bcgs.cpp
// (onesync_impl :233-369, pipi_impl :169-219, iro_impl :135-167, single_block :83-90)
// on top of the device kernels:
//   K1 gram_*   (gram.cu)   — the tall products of fused_gram / tsqr_fused_gram
//   K2 update_* (update.cu) — local_axpy_block + scale_right_block + copies
//   K3 small_*  (small.cu)  — pyth_chol, delayed reprojection, R assembly, NotSpd
//   K4 tsqr_*   (tsqr.cu)   — run_tsqr / householder_qr / tsqr tree
// Every block step is enqueued on one CUDA stream; the host never waits inside the
// factorization.  Collectives (one per sync event, recorded with the reference's labels
// and word counts, sync_stats.hpp:13-27) are NCCL calls on a multi-GPU context; on a
// single-GPU context with procs > 1 the ranks' shards live on the one device and the
// cross-rank combine is done by the same deterministic kernels (the reference's
// "simulated" backend, communicator.hpp:98-152).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <unistd.h>

#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "../../include/bgs_gpu.h"
#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"

using namespace bgs;

namespace {

// ------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------
struct Fail {
  int code;
  std::string msg;
  int pivot = 0;
  long block = 0;
  std::string site;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

#define CUDA_OK(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) fail(BGS_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

void put_err(bgs_error* err, const Fail& f) {
  if (!err) return;
  err->code = f.code;
  err->pivot = f.pivot;
  err->block = f.block;
  snprintf(err->site, sizeof err->site, "%s", f.site.c_str());
  snprintf(err->msg, sizeof err->msg, "%s", f.msg.c_str());
}
void clear_err(bgs_error* err) {
  if (err) memset(err, 0, sizeof *err);
}

// ------------------------------------------------------------------------------------
// NCCL, loaded on demand (only multi-GPU contexts need it)
// ------------------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define LOADSYM(name)                                                      \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name)); \
  if (!api.name) return api;
  LOADSYM(GetUniqueId)
  LOADSYM(CommInitRank)
  LOADSYM(CommDestroy)
  LOADSYM(AllReduce)
  LOADSYM(AllGather)
  LOADSYM(GroupStart)
  LOADSYM(GroupEnd)
  LOADSYM(GetErrorString)
#undef LOADSYM
  api.ok = true;
  return api;
}

#define NCCL_OK(expr)                                                                    \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != ncclSuccess) fail(BGS_E_COLLECTIVE, "%s failed: %s", #expr, nccl().GetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda at link time)
// ------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

PFN_encodeTiled encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (fn) return fn;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    fail(BGS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  fn = reinterpret_cast<PFN_encodeTiled>(p);
  return fn;
}

// cuStreamWaitValue32 (GEQ, cyclic): the stream stalls until *addr reaches `value`; no
// kernel occupies an SM while it waits (the peer transport's wait between launches).
void stream_wait_geq(cudaStream_t st, unsigned* addr, unsigned value) {
  using PFN_wait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static PFN_wait fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      fail(BGS_E_CUDA, "cuStreamWaitValue32 unavailable");
    fn = reinterpret_cast<PFN_wait>(p);
  }
  const CUresult r = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) fail(BGS_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}

// The {16 rows, row block, column} 3-D view of a column-major rows x cols fp64 matrix
// used by the tile engine (gram.cu): box {16, H, w}, 128-byte swizzle.  Reads whole
// 16-row blocks, so the storage must hold ceil(rows/16)*16 rows per column (ld >= that).
CUtensorMap make_map3(const double* base, long rows, long cols, long ld, int H, int w) {
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  if (rows <= 0 || cols <= 0) return m;
  const long rb = (rows + 15) / 16;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || ld < rb * 16)
    fail(BGS_E_DIMENSION,
         "device matrices need 16-byte aligned columns and a leading dimension >= rows "
         "rounded up to 16 (got rows %ld, ld %ld)", rows, ld);
  cuuint64_t dims[3] = {16, (cuuint64_t)rb, (cuuint64_t)cols};
  cuuint64_t strides[2] = {128, (cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[3] = {16, (cuuint32_t)H, (cuuint32_t)w};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(BGS_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return m;
}

// ------------------------------------------------------------------------------------
// grow-only device buffers
// ------------------------------------------------------------------------------------
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DBuf& operator=(DBuf&&) = delete;
  ~DBuf() { release(); }  // temporaries are freed on every exit path (Fail included)
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    CUDA_OK(cudaMalloc(&p, b));
    bytes = b;
    static const bool poison = getenv("BGS_POISON") != nullptr;  // tests: NaN-fill new buffers
    if (poison) {  // (completed before any stream of the context can touch the buffer)
      CUDA_OK(cudaMemset(p, 0xFF, b));
      CUDA_OK(cudaDeviceSynchronize());
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  double* d() const { return static_cast<double*>(p); }
};

// Page-locked host buffer (grow-only): the mirrors that let bgs_factor stream pageable
// caller buffers through the copy engines.
struct HBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    CUDA_OK(cudaHostAlloc(&p, b, cudaHostAllocDefault));
    bytes = b;
  }
  ~HBuf() {
    if (p) cudaFreeHost(p);
  }
  double* d() const { return static_cast<double*>(p); }
};

// dst[:, j] = src[:, j] for j < cols (rows doubles each), columns split over host threads
void host_copy_cols(double* dst, long ldd, const double* src, long lds, long rows, long cols) {
  const int nt = (int)std::max<long>(1, std::min<long>(cols, std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
  auto work = [&](int t) {
    for (long j = t; j < cols; j += nt)
      memcpy(dst + (size_t)j * ldd, src + (size_t)j * lds, (size_t)rows * sizeof(double));
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

const char* kVariantNames[6] = {"BCGS", "BCGSI+", "BCGSPIPI+", "BCGSI+P-1S", "BCGSI+P-2S",
                                "BCGSI+1S"};

}  // namespace

// ------------------------------------------------------------------------------------
// context
// ------------------------------------------------------------------------------------
struct bgs_ctx {
  int device = 0, rank = 0, nranks = 1, sms = 148;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  // caller-supplied host communicator (bgs_ctx_create_host_comm): one allgather per sync
  bgs_allgather_fn hc_fn = nullptr;
  void* hc_user = nullptr;
  HBuf hc_send, hc_recv, hc_out;
  // peer-memory transport (bgs_ctx_create_peer, peer.cu): one-shot exchange over windows
  // every rank maps (NVLink P2P between GPUs, CUDA IPC between processes)
  struct PeerComm {
    bool on = false, attached = false;
    int wait_mode = 0;  // 1: stream memory operations, 2: acquire spin in the sum kernel
    void* window = nullptr;  // cudaMalloc'ed (IPC-exportable), local
    void* cnt = nullptr;
    void* mapped[kPeerMaxRanks] = {};  // cudaIpcOpenMemHandle results (to close)
    PeerView view{};
    unsigned epoch = 0;
  } peer;
  bool collective() const { return comm != nullptr || hc_fn != nullptr || peer.on; }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // The device-pointer entry points run on `stream` (non-blocking) but first wait for the
  // caller's work issued so far on `caller` (legacy default stream unless set with
  // bgs_ctx_set_stream): a buffer the caller filled or cleared asynchronously is ready.
  cudaStream_t caller = nullptr;
  cudaEvent_t entry = nullptr;
  // copy engines of the host drop-in (bgs_factor): X chunks in, final Q columns out
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> xfer_events;  // reusable, timing disabled
  HBuf hx, hq;                           // pinned mirrors for pageable caller buffers
  DBuf partial, G, scolA, scolB, sdiag, ydiag, save, r1, r2, rtop, R, status;
  DBuf tsqr_ws, tsqr_bounds, roots, roots_all, cross_ws, cross_m, metrics;
  DBuf coefws;  // K2m: the update coefficients packed in DMMA-fragment order
  std::vector<DBuf> sx, sq;  // per-shard device buffers of the host-API path
  std::vector<DBuf> rscr;    // per-shard right-operand scratch of chunked Grams
  DBuf ticket;               // last-CTA ticket of the merged reduce + step kernel
  // CUDA graphs of whole factorizations (bgs_factor_device): one per call signature,
  // captured on the second call with that signature (the first sizes every workspace),
  // replayed after; dropped when a workspace was reallocated since the capture.
  struct GraphEntry {
    std::string key;
    std::vector<void*> bufs;  // workspace pointers the graph was captured with
    cudaGraphExec_t exec = nullptr;
    std::unique_ptr<bgs_stats> stats;
    long launches = 0;
    std::unique_ptr<HBuf> bounds;
    int uses = 0;
  };
  std::vector<GraphEntry> graphs;
  std::vector<std::string> seen;  // signatures run once (the next call captures)
  std::vector<void*> buf_signature() const {
    return {partial.p, G.p, scolA.p, scolB.p, sdiag.p, ydiag.p, save.p, r1.p, r2.p, rtop.p, R.p,
            status.p, tsqr_ws.p, tsqr_bounds.p, roots.p, roots_all.p, cross_ws.p, cross_m.p,
            ticket.p, metrics.p, coefws.p};
  }
  int launches = 0;
  // live profiler: event pairs per launch, resolved after the stream syncs
  struct ProfClass {
    std::string name;
    long launches = 0;
    double ms = 0, bytes = 0, flops = 0;
  };
  struct ProfRec {
    int cls;
    cudaEvent_t a, b;
  };
  bool prof_on = false;
  std::vector<ProfClass> prof;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CUDA_OK(cudaEventCreate(&e));
    return e;
  }
  int prof_class(const char* name) {
    for (size_t i = 0; i < prof.size(); ++i)
      if (prof[i].name == name) return (int)i;
    prof.push_back(ProfClass{name});
    return (int)prof.size() - 1;
  }
  // Resolve recorded pairs (the stream must have completed them).
  void prof_resolve() {
    for (auto& p : pending) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) prof[p.cls].ms += ms;
      event_pool.push_back(p.a);
      event_pool.push_back(p.b);
    }
    pending.clear();
  }
  ~bgs_ctx() {
    for (DBuf* b : {&partial, &G, &scolA, &scolB, &sdiag, &ydiag, &save, &r1, &r2, &rtop, &R,
                    &status, &tsqr_ws, &tsqr_bounds, &roots, &roots_all, &cross_ws,
                    &cross_m, &metrics})
      b->release();
    for (auto& b : sx) b.release();
    for (auto& b : rscr) b.release();
    ticket.release();
    coefws.release();
    for (auto& b : sq) b.release();
    for (auto& p : pending) {
      event_pool.push_back(p.a);
      event_pool.push_back(p.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    for (void* mp : peer.mapped)
      if (mp) cudaIpcCloseMemHandle(mp);
    if (peer.window) cudaFree(peer.window);
    if (peer.cnt) cudaFree(peer.cnt);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (entry) cudaEventDestroy(entry);
    for (auto e : xfer_events) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

static long even_ld(long rows) { return std::max<long>(32, (rows + 31) & ~31L); }

// Order the context stream after everything the caller has queued on its stream.
static void order_after_caller(bgs_ctx* c) {
  CUDA_OK(cudaEventRecord(c->entry, c->caller));
  CUDA_OK(cudaStreamWaitEvent(c->stream, c->entry, 0));
}

// One row shard resident on this device: rows [row0, row0 + rows) of the global matrix.
struct Shard {
  long row0 = 0, rows = 0;
  const double* X = nullptr;
  long ldx = 0;
  double* Q = nullptr;
  long ldq = 0;
  // tile-engine views: [H index: 0 -> H=2, 1 -> H=4][box width 128/64/32/16/8]
  CUtensorMap mapX[2][5], mapQ[2][5];
  // chunked Grams: the right operand copied to a contiguous scratch (SR spans)
  double* Rs = nullptr;
  long ldr = 0;
  CUtensorMap mapR[2][5];
  void make_maps(long m) {
    for (int hi = 0; hi < 2; ++hi)
      for (int wi = 0; wi < 5; ++wi) {
        mapX[hi][wi] = make_map3(X, rows, m, ldx, 2 << hi, 128 >> wi);
        mapQ[hi][wi] = make_map3(Q, rows, m, ldq, 2 << hi, 128 >> wi);
      }
  }
  // TSQR leaf plan
  int leaf_base = 0, n_leaves = 0, bound_base = 0;
  long hmax = 0;
};

enum Src { SX = 0, SQ = 1, SR = 2 };  // X, Q, right-operand scratch (chunked Grams)

struct GSpan {
  int src = SQ;
  int col0 = 0;
  int ncols = 0;  // loaded columns
  int lcols = 0;  // left-operand (output row) columns
};

struct GramSpec {
  int nspans = 1;
  GSpan sp[2];
  int N = 0;
  int rspan[32];
  int rcol[32];
  // Gram rows >= comp_row (compact row index) are accumulated with every 4-row k-step
  // folded into a double-double (gram_ct.cu / k12_ct.cu): BCGSI+1S's U rows
  int comp_row = 1 << 30;
};
// first compensated output tile of a Gram whose span 0 has lc0 output-row columns in
// units0 8-column units (span-1 output rows follow at tile units0); mt_out: none
static int comp_tile(const GramSpec& g, int lc0, int units0, int mt_out) {
  const int r = g.comp_row;
  if (r < 0 || r >= (1 << 30)) return mt_out;
  const int t = r < lc0 ? r / 8 : units0 + (r - lc0) / 8;
  return t < mt_out ? t : mt_out;
}

class Runner {
 public:
  bgs_ctx* c;
  int variant;
  long n, m, s, q;
  int P;        // ranks of the factorization
  bool use_coll;  // a multi-rank (or one-rank NCCL) context: collectives between launches
  std::vector<Shard> sh;
  bgs_stats* stats;
  const bgs_options* opt;  // BcgsOptions (probe)
  HBuf* bounds_sink = nullptr;  // graph capture: pinned home of the TSQR leaf bounds
  long words = 0;
  DevStatus* status;
  int tsqr_L = 0;  // total leaves across local shards

  bool no_fuse = false;
  bool no_k12c = false;
  bool prof_step = false;  // BGS_PROF_STEP: one profiler class per fused block step
  int gram_max_units = 0;  // BGS_GRAM_MAXUNITS (tests): chunk unfused Grams above this
  bool no_merge_small = false;  // BGS_NO_MERGE_SMALL: separate reduce and small launches
  bool no_pdl = false;          // BGS_NO_PDL: no programmatic dependent launch of K12c
  int comp_mode = 1;            // BGS_COMP_TAIL: 0 off, 1 BCGSI+1S (default), 2 all modes
  bool no_k2m = false;          // BGS_K2M=0: the s = 8 / 16 update on K2t instead of K2m
  // Programmatic dependent launch of a fused kernel is allowed only right behind the
  // merged reduce + step kernel (nothing queued in between): that kernel writes only the
  // Gram, the small factors and the status word, which the fused kernel reads after its
  // griddepcontrol.wait; X / Q come from kernels that completed before it started.
  int merged_mark = -1, waits = 0, merged_waits = -1;
  bool pdl_next() const {
    return !no_pdl && merged_mark == c->launches && merged_waits == waits;
  }
  int tile_dbg = 0;
  bool tile_prof = false;

  Runner(bgs_ctx* ctx, int v, long n_, long m_, long s_, int P_, bool nccl_, bgs_stats* st, const bgs_options* opt_ = nullptr)
      : c(ctx), variant(v), n(n_), m(m_), s(s_), q(m_ / s_), P(P_), use_coll(nccl_), stats(st), opt(opt_) {
    const char* e = getenv("BGS_NO_FUSE");
    no_fuse = e && *e && *e != '0';
    // K12c (k12.cu) is the fused path; BGS_K12C=0 falls back to the single-CTA K12
    const char* e2 = getenv("BGS_K12C");
    no_k12c = e2 && *e2 == '0';
    const char* e3 = getenv("BGS_PROF_STEP");
    prof_step = e3 && *e3 && *e3 != '0';
    const char* e4 = getenv("BGS_GRAM_MAXUNITS");
    gram_max_units = e4 ? atoi(e4) : 0;
    const char* e5 = getenv("BGS_NO_MERGE_SMALL");
    no_merge_small = e5 && *e5 && *e5 != '0';
    const char* ek2m = getenv("BGS_K2M");
    no_k2m = ek2m && *ek2m == '0';
    const char* ect = getenv("BGS_COMP_TAIL");
    comp_mode = !ect ? 1 : (*ect == '0' ? 0 : (strcmp(ect, "all") == 0 ? 2 : 1));
    const char* e7 = getenv("BGS_NO_PEER_FUSE");
    no_peer_fuse = e7 && *e7 && *e7 != '0';
    const char* e8 = getenv("BGS_PEER_ONE");
    peer_one = e8 ? atoi(e8) : 1;
    const char* e6 = getenv("BGS_NO_PDL");
    no_pdl = e6 && *e6 && *e6 != '0';
    const char* d = getenv("BGS_TILE_DBG");
    tile_dbg = d ? atoi(d) : 0;
    const char* tp = getenv("BGS_TILE_PROF");
    tile_prof = tp && *tp && *tp != '0';
  }

  // Streaming hooks of the host drop-in (bgs_factor): X arrives in column chunks on a copy
  // stream (the compute stream waits on a chunk's event before the first kernel that reads
  // it) and Q columns leave on another copy stream as soon as they are final.
  struct XFeed {
    long chunk_cols = 0;
    std::vector<cudaEvent_t> ready;  // per chunk, recorded on the H2D stream
    int waited = 0;                  // chunks the compute stream already waits on
    // pageable caller buffers: a feeder thread records ready[i] after staging chunk i;
    // the enqueueing thread blocks until then (cudaStreamWaitEvent on a never-recorded
    // event would not wait)
    bool async_feed = false;
    std::mutex mu;
    std::condition_variable cv;
    int recorded = 0;
    bool failed = false;
  };
  XFeed* feed = nullptr;
  std::function<void(long)> on_q_final;  // Q columns [0, c) are final
  void need_x(long col_end) {
    if (!feed || col_end <= 0) return;
    const int upto = (int)std::min<long>((long)feed->ready.size(),
                                         (col_end + feed->chunk_cols - 1) / feed->chunk_cols);
    for (; feed->waited < upto; ++feed->waited, ++waits) {
      if (feed->async_feed) {
        std::unique_lock<std::mutex> lk(feed->mu);
        feed->cv.wait(lk, [&] { return feed->recorded > feed->waited || feed->failed; });
        if (feed->failed) fail(BGS_E_CUDA, "staging the pageable input failed");
      }
      CUDA_OK(cudaStreamWaitEvent(c->stream, feed->ready[feed->waited], 0));
    }
  }
  void q_final(long col_end) {
    if (on_q_final) on_q_final(col_end);
  }

  // RAII bracket of one launch (or launch group) of a kernel class for the profiler.
  struct Prof {
    bgs_ctx* c;
    int cls = -1;
    cudaEvent_t a = nullptr;
    Prof(bgs_ctx* ctx, const char* name, double bytes, double flops) : c(ctx) {
      if (!c->prof_on) return;
      cls = c->prof_class(name);
      c->prof[cls].launches += 1;
      c->prof[cls].bytes += bytes;
      c->prof[cls].flops += flops;
      a = c->get_event();
      CUDA_OK(cudaEventRecord(a, c->stream));
    }
    ~Prof() {
      if (cls < 0) return;
      cudaEvent_t b = c->get_event();
      cudaEventRecord(b, c->stream);
      c->pending.push_back({cls, a, b});
    }
  };

  void record(const char* label, long w) {
    if (!stats) return;
    stats->sync_count += 1;
    stats->words_reduced += w;
    size_t len = strlen(stats->labels);
    if (len + strlen(label) + 2 < sizeof stats->labels) {
      if (stats->n_events) strcat(stats->labels, "\n");
      strcat(stats->labels, label);
    }
    stats->n_events += 1;
  }

  const double* colp(const Shard& x, int src, long col) const {
    return src == SX ? x.X + (size_t)col * x.ldx : x.Q + (size_t)col * x.ldq;
  }
  double* qcol(const Shard& x, long col) const { return x.Q + (size_t)col * x.ldq; }

  // ---------------- setup ----------------
  void setup() {
    const size_t ss = (size_t)s * s;
    c->status.ensure(sizeof(DevStatus));
    status = reinterpret_cast<DevStatus*>(c->status.p);
    CUDA_OK(cudaMemsetAsync(status, 0, sizeof(DevStatus), c->stream));
    c->ticket.ensure(64);
    CUDA_OK(cudaMemsetAsync(c->ticket.p, 0, 64, c->stream));
    c->R.ensure((size_t)m * m * sizeof(double));
    CUDA_OK(cudaMemsetAsync(c->R.p, 0, (size_t)m * m * sizeof(double), c->stream));
    const long Mmax = m + 2 * s + 16;
    c->G.ensure((size_t)Mmax * 32 * sizeof(double) + 4096);
    c->scolA.ensure((size_t)(m + s) * s * sizeof(double));
    c->scolB.ensure((size_t)(m + s) * s * sizeof(double));
    c->save.ensure((size_t)(m + s) * s * sizeof(double));
    for (DBuf* b : {&c->sdiag, &c->ydiag, &c->r1, &c->r2, &c->rtop}) b->ensure(ss * sizeof(double) + 64);
    for (auto& x : sh) x.make_maps(m);
    // Gram partial slots: every shard's CTAs
    const int boxes_max = (int)((m + 2 * s + 7) / 8) + 2;
    const size_t per_cta = gram_partial_doubles_per_cta(boxes_max, std::min<long>(2 * s, 32));
    c->partial.ensure(per_cta * sizeof(double) * (size_t)grid_total() + 64);
    // TSQR leaf plan
    const long lw = s <= 4 ? 1024 : (s <= 8 ? 512 : 256);
    std::vector<long> bounds;
    int leaf = 0;
    for (auto& x : sh) {
      long L = x.rows <= 0 ? 1 : (x.rows + lw - 1) / lw;
      if (x.rows > 0) L = std::max<long>(1, std::min<long>(L, x.rows / s));
      x.leaf_base = leaf;
      x.n_leaves = (int)L;
      x.bound_base = (int)bounds.size();
      x.hmax = 0;
      for (long l = 0; l <= L; ++l) {
        const long b = x.rows * l / L;
        bounds.push_back(b);
        if (l > 0) x.hmax = std::max(x.hmax, b - bounds[bounds.size() - 2]);
      }
      leaf += (int)L;
    }
    tsqr_L = leaf;
    c->tsqr_ws.ensure(tsqr_ws_bytes(tsqr_L, (int)s) + 64);
    c->tsqr_bounds.ensure(bounds.size() * sizeof(long));
    const void* bsrc = bounds.data();
    if (bounds_sink) {  // graph capture: the copy node must read memory that outlives the call
      bounds_sink->ensure(bounds.size() * sizeof(long) + 64);
      memcpy(bounds_sink->p, bounds.data(), bounds.size() * sizeof(long));
      bsrc = bounds_sink->p;
    }
    CUDA_OK(cudaMemcpyAsync(c->tsqr_bounds.p, bsrc, bounds.size() * sizeof(long),
                            cudaMemcpyHostToDevice, c->stream));
    c->roots.ensure((size_t)sh.size() * ss * sizeof(double) + 64);
    c->roots_all.ensure((size_t)P * ss * sizeof(double) + 64);
    c->cross_ws.ensure(tsqr_ws_bytes(P, (int)s) + 64);
    c->cross_m.ensure((size_t)P * ss * sizeof(double) + 64);
    // BGS_POISON=2 (tests): NaN-fill every workspace at the start of EVERY factorization, not
    // only when it is allocated: whatever an earlier call left behind (finite, so invisible to
    // BGS_POISON=1) must not be read before this call writes it.
    static const int poison_level = [] {
      const char* e = getenv("BGS_POISON");
      return e ? atoi(e) : 0;
    }();
    if (poison_level >= 2)
      for (DBuf* b : {&c->G, &c->scolA, &c->scolB, &c->save, &c->sdiag, &c->ydiag, &c->r1, &c->r2,
                      &c->rtop, &c->partial, &c->tsqr_ws, &c->roots, &c->roots_all, &c->cross_ws,
                      &c->cross_m, &c->coefws})
        if (b->p && b->bytes) CUDA_OK(cudaMemsetAsync(b->p, 0xFF, b->bytes, c->stream));
  }

  int grid_for(const Shard& x) const {
    const int per = std::max(1, c->sms / (int)sh.size());
    const long stages = (x.rows + 63) / 64;
    return (int)std::max<long>(1, std::min<long>(per, stages));
  }
  int grid_total() const {
    int g = 0;
    for (auto& x : sh) g += grid_for(x);
    return g;
  }

  // ---------------- collectives (between launches; no kernel waits on a rank) ----------
  // Sum of every rank's n doubles at d (in place), identical bits on every rank.
  void allreduce(double* d, size_t n) {
    if (c->comm) {
      Prof pr(c, "nccl_allreduce", (double)n * 8.0, 0.0);
      NCCL_OK(nccl().AllReduce(d, d, n, ncclDouble, ncclSum, c->comm, c->stream));
      return;
    }
    exchange(nullptr, 0, nullptr, d, n);
  }
  // One sync: allgather of ng doubles (send -> recv, rank-major) and allreduce of ns
  // doubles at sum (in place).  NCCL: one group.  Host communicator: one allgather of the
  // packed [gather | partial] buffer, the partials summed in rank order on the host.
  void exchange(const double* send, size_t ng, double* recv, double* sum, size_t ns) {
    if (c->comm) {
      NCCL_OK(nccl().GroupStart());
      if (ng) NCCL_OK(nccl().AllGather(send, recv, ng, ncclDouble, c->comm, c->stream));
      if (ns) NCCL_OK(nccl().AllReduce(sum, sum, ns, ncclDouble, ncclSum, c->comm, c->stream));
      NCCL_OK(nccl().GroupEnd());
      return;
    }
    if (c->peer.on) {
      peer_exchange(send, ng, recv, sum, ns);
      return;
    }
    if (!c->hc_fn) fail(BGS_E_INTERNAL, "collective on a context without a communicator");
    flush_reduce();
    Prof pr(c, "host_exchange", (double)(ng + ns) * 8.0 * P, 0.0);
    const size_t w = ng + ns;
    c->hc_send.ensure(w * sizeof(double) + 64);
    c->hc_recv.ensure((size_t)P * w * sizeof(double) + 64);
    c->hc_out.ensure(((size_t)P * ng + ns) * sizeof(double) + 64);
    double* hs = c->hc_send.d();
    if (ng) CUDA_OK(cudaMemcpyAsync(hs, send, ng * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (ns) CUDA_OK(cudaMemcpyAsync(hs + ng, sum, ns * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));  // (also retires the previous exchange's H2D)
    double* hr = c->hc_recv.d();
    if (c->hc_fn(c->hc_user, hs, hr, (unsigned long)(w * sizeof(double))) != 0)
      fail(BGS_E_COLLECTIVE, "host communicator allgather failed (rank %d of %d)", c->rank, P);
    double* ho = c->hc_out.d();
    for (int r = 0; r < P; ++r) memcpy(ho + (size_t)r * ng, hr + (size_t)r * w, ng * sizeof(double));
    for (size_t i = 0; i < ns; ++i) {
      double acc = hr[ng + i];
      for (int r = 1; r < P; ++r) acc += hr[(size_t)r * w + ng + i];  // rank order
      ho[(size_t)P * ng + i] = acc;
    }
    if (ng) CUDA_OK(cudaMemcpyAsync(recv, ho, (size_t)P * ng * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (ns) CUDA_OK(cudaMemcpyAsync(sum, ho + (size_t)P * ng, ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }

  // The sync over peer-mapped windows (peer.cu): push to every rank, wait for the P flags
  // (stream memory operations, or a spin in the sum kernel on distinct GPUs), sum in rank
  // order out of the local window.  No host round trip.
  void peer_exchange(const double* send, size_t ng, double* recv, double* sum, size_t ns) {
    bgs_ctx::PeerComm& pc = c->peer;
    if (!pc.attached) fail(BGS_E_COLLECTIVE, "peer context: bgs_ctx_peer_attach was not called");
    if ((ng + ns) * sizeof(double) > pc.view.slot_bytes)
      fail(BGS_E_CONFIG, "peer window slot (%lu bytes) is smaller than the exchange payload (%zu bytes)",
           pc.view.slot_bytes, (ng + ns) * sizeof(double));
    flush_reduce();
    Prof pr(c, "peer_exchange", (double)(ng + ns) * 8.0 * P, 0.0);
    const unsigned ep = ++pc.epoch;
    CUDA_OK(peer_push_launch(pc.view, send, ng, sum, ns, ep, static_cast<unsigned*>(pc.cnt), c->stream,
                             &c->launches));
    if (pc.wait_mode == 1) {
      for (int r = 0; r < pc.view.P; ++r) {
        if (r == pc.view.rank) continue;  // (stream order covers the local push)
        stream_wait_geq(c->stream, reinterpret_cast<unsigned*>(pc.window) + r, ep);
      }
      ++waits;
    }
    CUDA_OK(peer_sum_launch(pc.view, ng, recv, ns, sum, ep, pc.wait_mode == 2, c->stream, &c->launches,
                            status));
  }

  // RecurrenceProbe::on_eval (bcgs.cpp:339-343): S2 of step k and this rank's rows of Q_k
  // (block k, final once the update of step k has run) and X_{k+1}, as host copies.
  void fire_probe(long k, const double* s2_dev, int ld_s2) {
    if (!opt || !opt->probe) return;
    flush_reduce();
    CUDA_OK(cudaStreamSynchronize(c->stream));
    std::vector<double> s2((size_t)s * s);
    CUDA_OK(cudaMemcpy2D(s2.data(), s * sizeof(double), s2_dev, (size_t)ld_s2 * sizeof(double),
                         s * sizeof(double), s, cudaMemcpyDeviceToHost));
    for (size_t t = 0; t < sh.size(); ++t) {
      const Shard& x = sh[t];
      const long nl = std::max<long>(x.rows, 0);
      std::vector<double> ql((size_t)nl * s + 1), xl((size_t)nl * s + 1);
      if (nl) {
        CUDA_OK(cudaMemcpy2D(ql.data(), nl * sizeof(double), x.Q + (size_t)(k * s) * x.ldq,
                             x.ldq * sizeof(double), nl * sizeof(double), s, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy2D(xl.data(), nl * sizeof(double), x.X + (size_t)((k + 1) * s) * x.ldx,
                             x.ldx * sizeof(double), nl * sizeof(double), s, cudaMemcpyDeviceToHost));
      }
      opt->probe(opt->probe_user, k + 1, s2.data(), s, ql.data(), xl.data(), nl,
                 use_coll ? c->rank : (int)t);
    }
  }

  // ---------------- K1 / K12 + reduction + (NCCL) allreduce ----------------
  // Fused block update carried in front of the Gram (K12); dst columns are Q columns.
  struct Fuse {
    bool a = false, b = false;
    int kp = 0;
    const double* CA = nullptr; int ldca = 0; const double* TA = nullptr; long dstA = 0;
    const double* CB = nullptr; int ldcb = 0; const double* TB = nullptr; long dstB = 0;
  };

  // K12c (k12.cu): the fused update + Gram split over CTA pairs.  Returns -1 when the
  // shape is not covered (the caller then uses the single-CTA tile engine).
  // Structural K12c parameters of a fused Gram spec + the plan; false if K12c cannot run it.
  bool split_params(const GramSpec& sp, bool a, bool b, int kp, SplitParams& p) const {
    memset(&p, 0, sizeof p);
    if (no_k12c || sp.nspans != 2 || sp.N > 8 || sp.sp[0].lcols != sp.sp[0].ncols) return false;
    for (int j = 0; j < sp.N; ++j) {
      if (sp.rspan[j] != 1) return false;
      p.rcol1[j] = sp.rcol[j];
    }
    for (int j = sp.N; j < 8; ++j) p.rcol1[j] = -1;
    p.N = sp.N;
    p.U0 = (sp.sp[0].ncols + 7) / 8;
    p.U1 = (sp.sp[1].ncols + 7) / 8;
    p.ncols0 = sp.sp[0].ncols;
    p.lcols1 = sp.sp[1].lcols;
    p.col0[0] = sp.sp[0].col0;
    p.col0[1] = sp.sp[1].col0;
    p.upd_a = a;
    p.upd_b = b;
    p.kp = kp;
    p.s = (int)s;
    if (!k12_plan(p)) return false;
    p.comp_t0 = comp_tile(sp, sp.sp[0].ncols, p.U0, p.mt_out);
    // K12c compensates exactly the span-1 left unit (U_{k+1}, X_{k+2} as output rows)
    if (p.comp_t0 < p.mt_out && !(p.comp_t0 == p.U0 && p.s1_left == 1)) return false;
    for (auto& x : sh)
      if (x.rows > 0 && grid_for(x) < p.cluster) return false;
    return true;
  }

  int gram_split(const GramSpec& sp, const char* label, bool count_sync, bool do_allreduce,
                 const Fuse& fz, const int units[2], const int lc[2]) {
    SplitParams p;
    if (!split_params(sp, fz.a, fz.b, fz.kp, p)) return -1;
    p.CA = fz.CA; p.ldca = fz.ldca; p.TA = fz.TA;
    p.CB = fz.CB; p.ldcb = fz.ldcb; p.TB = fz.TB;
    p.status = status;
    p.dbg = tile_dbg;
    (void)units;
    static const int prof_minkp = [] {
      const char* e = getenv("BGS_PROF_MINKP");
      return e ? atoi(e) : 0;
    }();
    static const int prof_maxkp = [] {
      const char* e = getenv("BGS_PROF_MAXKP");
      return e ? atoi(e) : 1 << 30;
    }();
    if (tile_prof && fz.kp >= prof_minkp && fz.kp <= prof_maxkp) {
      c->metrics.ensure((size_t)512 * 16 * sizeof(unsigned long long) + 64);
      p.phase = reinterpret_cast<unsigned long long*>(c->metrics.p) + 256 * 16;
    }
    const int M = lc[0] + lc[1];
    const size_t per_slot = gram_partial_doubles_per_cta(p.mt_out, p.N);
    int slot_base = 0;
    for (auto& x : sh) {
      const int grid = p.cluster >= 2 ? std::min(grid_for(x) / p.cluster * p.cluster, k12_grid_cap(p.cluster, c->sms)) : grid_for(x);
      if (x.rows > 0) {
        for (int wi = 0; wi < 5; ++wi)
          p.map0[wi] = sp.sp[0].src == SX ? x.mapX[0][wi] : x.mapQ[0][wi];
        for (int wi = 0; wi < 2; ++wi)
          p.map1[wi] = sp.sp[1].src == SX ? x.mapX[0][3 + wi] : x.mapQ[0][3 + wi];
        p.n_rows = x.rows;
        p.total_stages = (x.rows + 32 * p.R - 1) / (32 * p.R);
        p.partial = c->partial.d() + per_slot * slot_base;
        p.dstA = x.Q + (size_t)fz.dstA * x.ldq;
        p.lddA = x.ldq;
        p.dstB = x.Q + (size_t)fz.dstB * x.ldq;
        p.lddB = x.ldq;
        const int nout = (fz.a ? 1 : 0) + (fz.b ? 1 : 0);
        const double bytes = 8.0 * x.rows * (sp.sp[0].ncols + sp.sp[1].ncols) + 8.0 * x.rows * s * nout;
        const double flops = 2.0 * x.rows * (double)M * sp.N + 2.0 * x.rows * (double)fz.kp * s * nout;
        char cls[64] = "fused_update_gram";
        if (prof_step) snprintf(cls, sizeof cls, "fused_update_gram@kp%04d", fz.kp);
        Prof pr(c, cls, bytes, flops);
        p.pdl = pdl_next() && !pr.a ? 1 : 0;  // (profiling events in between: plain launch)
        CUDA_OK(k12_launch(p, grid, c->stream, &c->launches));
        slot_base += grid / p.cluster;
      } else {
        CUDA_OK(cudaMemsetAsync(c->partial.d() + per_slot * slot_base, 0,
                                per_slot * sizeof(double), c->stream));
        slot_base += 1;
      }
    }
    TileParams rp;
    memset(&rp, 0, sizeof rp);
    rp.partial = c->partial.d();
    rp.mt_out = p.mt_out;
    rp.N = p.N;
    rp.units_span[0] = p.U0;
    rp.lcols[0] = lc[0];
    rp.lcols[1] = lc[1];
    rp.status = status;
    reduce(rp, slot_base, c->G.d(), 0, (double)slot_base * per_slot * 8.0);
    if (use_coll && do_allreduce) allreduce_after_reduce(c->G.d(), (size_t)M * p.N);
    if (count_sync) record(label, (long)M * p.N);
    return M;
  }

  // A Gram reduction held back so the one-sync step's small op can run in the same launch
  // (reduce_step4_kernel).  Only inside onesync(), only on single-GPU contexts (no
  // allreduce may sit between the two); every other launch flushes it first.
  // On a peer-memory context (peer.cu) the cross-rank exchange of that Gram is held back
  // with it (xchg): reduce -> push -> flags and [wait] -> rank-ordered sum -> step then run
  // as two launches, or one (small.cu: reduce_push / sum_step4 / reduce_xchg_step4).
  struct PendingReduce {
    bool on = false;
    ReduceArgs a;
    int entries = 0;
    double bytes = 0.0;
    bool xchg = false;   // an allreduce of `words` doubles at a.out follows the reduction
    size_t words = 0;
  };
  PendingReduce pend;
  bool defer_reduce = false;
  bool no_peer_fuse = false;  // BGS_NO_PEER_FUSE: separate reduce / push / sum / step launches
  int peer_one = 1;           // BGS_PEER_ONE=0: never the single-launch form (A then B)
  bool peer_fusable() const {
    return c->peer.on && c->peer.attached && !no_peer_fuse && !c->comm && !c->hc_fn;
  }
  void flush_reduce() {
    if (!pend.on) return;
    pend.on = false;
    {
      Prof pr(c, "gram_reduce", pend.bytes, 0.0);
      CUDA_OK(gram_reduce_launch_args(pend.a, pend.entries, c->stream, &c->launches));
    }
    if (pend.xchg) {
      pend.xchg = false;
      allreduce(pend.a.out, pend.words);
    }
  }
  // the allreduce that follows a reduction into d: rides with a held-back reduction
  void allreduce_after_reduce(double* d, size_t n) {
    if (pend.on && pend.a.out == d) {
      pend.xchg = true;
      pend.words = n;
      return;
    }
    allreduce(d, n);
  }
  // launch (or hold back) the reduction of `slots` partial slots described by rp
  void reduce(const TileParams& rp, int slots, double* out, int ld_out, double bytes) {
    if (defer_reduce && (!use_coll || peer_fusable()) && !gout) {
      pend.on = true;
      pend.a = reduce_args(rp, slots, out, ld_out);
      pend.entries = rp.mt_out * 8 * 8 * gram_n_tiles(rp.N);
      pend.bytes = bytes;
      return;
    }
    Prof pr(c, "gram_reduce", bytes, 0.0);
    CUDA_OK(gram_reduce_launch(rp, slots, out, c->stream, &c->launches, ld_out));
  }

  static const CUtensorMap& map_of(const Shard& x, int src, int hi, int wi) {
    return src == SX ? x.mapX[hi][wi] : src == SQ ? x.mapQ[hi][wi] : x.mapR[hi][wi];
  }
  double* gout = nullptr;  // chunked Grams: where this chunk's rows go (ld gout_ld)
  int gout_ld = 0;

  // A left operand wider than one CTA's shared memory holds (H = 2, 2 stages; e.g. m = 800):
  // copy the right operand (<= 32 columns) into a contiguous scratch, run the tile engine
  // over column chunks of the left operand, each chunk writing its rows of the Gram; then
  // one allreduce / sync record for the whole Gram, as before.
  int gram_chunked(const GramSpec& sp, const char* label, bool count_sync, bool do_allreduce) {
    const int N = sp.N;
    struct Run {
      int src, col0, n;
    };
    std::vector<Run> left;
    int M = 0;
    for (int i = 0; i < sp.nspans; ++i)
      if (sp.sp[i].lcols > 0) {
        left.push_back({sp.sp[i].src, sp.sp[i].col0, sp.sp[i].lcols});
        M += sp.sp[i].lcols;
      }
    for (int j = 0; j < N; ++j)
      if (sp.sp[sp.rspan[j]].src == SX) need_x(sp.sp[sp.rspan[j]].col0 + sp.rcol[j] + 1);
    if (c->rscr.size() < sh.size()) c->rscr.resize(sh.size());
    for (size_t i = 0; i < sh.size(); ++i) {
      Shard& x = sh[i];
      if (x.rows <= 0) continue;
      x.ldr = even_ld(x.rows);
      c->rscr[i].ensure((size_t)x.ldr * 32 * sizeof(double) + 256);
      x.Rs = c->rscr[i].d();
      for (int j = 0; j < N; ++j) {
        const GSpan& g = sp.sp[sp.rspan[j]];
        CUDA_OK(copy_cols_launch(colp(x, g.src, g.col0 + sp.rcol[j]), g.src == SX ? x.ldx : x.ldq,
                                 x.Rs + (size_t)j * x.ldr, x.ldr, x.rows, 1, c->stream));
      }
      for (int hi = 0; hi < 2; ++hi)
        for (int wi = 0; wi < 5; ++wi) x.mapR[hi][wi] = make_map3(x.Rs, x.rows, N, x.ldr, 2 << hi, 128 >> wi);
    }
    const int runits = (N + 7) / 8;
    int cu = 1;
    while (tile_smem_bytes(2, 2, cu + 1 + runits, false) <= (size_t)TILE_SMEM_MAX) ++cu;
    if (gram_max_units > runits) cu = std::min(cu, gram_max_units - runits);
    const int cw = 8 * cu;
    int row_off = 0;
    for (const Run& r : left)
      for (int c0 = 0; c0 < r.n; c0 += cw) {
        const int len = std::min(cw, r.n - c0);
        GramSpec g = spec2(r.src, r.col0 + c0, len, len, SR, 0, N, 0);
        add_right(g, 1, 0, N);
        if (sp.comp_row < row_off + len) g.comp_row = std::max(0, sp.comp_row - row_off);
        gout = c->G.d() + row_off;
        gout_ld = M;
        gram(g, "", false, false);
        gout = nullptr;
        gout_ld = 0;
        row_off += len;
      }
    if (use_coll && do_allreduce) allreduce(c->G.d(), (size_t)M * N);
    if (count_sync) record(label, (long)M * N);
    return M;
  }

  // Returns M (rows of the compact Gram written to c->G, ld = M).
  int gram(const GramSpec& sp, const char* label, bool count_sync = true,
           bool do_allreduce = true, const Fuse* fz = nullptr) {
    flush_reduce();
    for (int i = 0; i < sp.nspans; ++i)
      if (sp.sp[i].src == SX) need_x(sp.sp[i].col0 + sp.sp[i].ncols);
    TileParams p;
    memset(&p, 0, sizeof p);
    int units[2] = {0, 0}, lc[2] = {0, 0};
    for (int i = 0; i < sp.nspans; ++i) {
      units[i] = (sp.sp[i].ncols + 7) / 8;
      lc[i] = sp.sp[i].lcols;
    }
    const bool span1_left = sp.nspans == 2 && lc[1] > 0;
    if (span1_left && lc[0] != sp.sp[0].ncols) fail(BGS_E_INTERNAL, "gram: bad left layout");
    p.units_span[0] = units[0];
    p.units_span[1] = units[1];
    p.units = units[0] + units[1];
    p.mt_out = span1_left ? units[0] + (lc[1] + 7) / 8 : (lc[0] + 7) / 8;
    p.N = sp.N;
    for (int i = 0; i < 2; ++i) {
      p.col0[i] = sp.sp[i].col0;
      p.lcols[i] = lc[i];
    }
    p.comp_t0 = comp_tile(sp, lc[0], units[0], p.mt_out);
    for (int j = 0; j < 32; ++j)
      p.rcol[j] = j < sp.N ? (sp.rspan[j] == 0 ? sp.rcol[j] : 8 * units[0] + sp.rcol[j]) : -1;
    p.status = status;
    p.dbg = tile_dbg;
    if (tile_prof) {
      c->metrics.ensure((size_t)512 * 16 * sizeof(unsigned long long) + 64);
      p.phase = reinterpret_cast<unsigned long long*>(c->metrics.p);
    }
    const bool upd = fz != nullptr;
    if (!upd && !gout && (tile_smem_bytes(2, 2, p.units, false) > (size_t)TILE_SMEM_MAX ||
                          (gram_max_units > 0 && p.units > gram_max_units)))
      return gram_chunked(sp, label, count_sync, do_allreduce);
    if (upd) {
      const int M = gram_split(sp, label, count_sync, do_allreduce, *fz, units, lc);
      if (M >= 0) return M;
    }
    if (upd) {
      if (!tile_fused_supported((int)s, fz->kp, p.mt_out) || sp.N > 8)
        fail(BGS_E_INTERNAL, "gram: fused update not supported for this shape");
      p.upd_a = fz->a;
      p.upd_b = fz->b;
      p.kp = fz->kp;
      p.s = (int)s;
      p.colA = fz->kp;
      p.colB = 8 * units[0];
      p.CA = fz->CA; p.ldca = fz->ldca; p.TA = fz->TA;
      p.CB = fz->CB; p.ldcb = fz->ldcb; p.TB = fz->TB;
    }
    // Tallest stage (longest contiguous run per column) that keeps >= 3 (H=4) or >= 2
    // (H=2) stages in flight within the CTA's shared memory.
    int H = 0, S = 0;
    for (int h : {4, 2}) {
      const size_t one = tile_smem_bytes(h, 1, p.units, upd) - tile_smem_bytes(h, 0, p.units, upd);
      const size_t fixed = tile_smem_bytes(h, 0, p.units, upd);
      const int smax = (int)((TILE_SMEM_MAX - fixed) / one);
      if (smax >= (h == 4 ? 3 : 2)) {
        H = h;
        S = std::min(smax, 8);
        break;
      }
    }
    if (!H) fail(BGS_E_CONFIG, "gram: a %d-column tile does not fit in shared memory", 8 * p.units);
    p.H = H;
    p.stages = S;
    const int hi = H == 4 ? 1 : 0;
    const int M = lc[0] + (span1_left ? lc[1] : 0);
    const size_t per_cta = gram_partial_doubles_per_cta(p.mt_out, p.N);
    int cta_base = 0;
    double flops_upd = 0.0, bytes_upd = 0.0;
    for (auto& x : sh) {
      const int grid = grid_for(x);
      if (x.rows > 0) {
        for (int wi = 0; wi < 5; ++wi) p.map0[wi] = map_of(x, sp.sp[0].src, hi, wi);
        if (sp.nspans == 2)
          for (int wi = 0; wi < 2; ++wi) p.map1[wi] = map_of(x, sp.sp[1].src, hi, 3 + wi);
        p.n_rows = x.rows;
        p.partial = c->partial.d() + per_cta * cta_base;
        if (upd) {
          p.dstA = x.Q + (size_t)fz->dstA * x.ldq;
          p.lddA = x.ldq;
          p.dstB = x.Q + (size_t)fz->dstB * x.ldq;
          p.lddB = x.ldq;
          const int nout = (fz->a ? 1 : 0) + (fz->b ? 1 : 0);
          bytes_upd = 8.0 * x.rows * s * nout;  // the written blocks
          flops_upd = 2.0 * x.rows * (double)fz->kp * s * nout;
        }
        const double bytes = 8.0 * x.rows * (sp.sp[0].ncols + (sp.nspans == 2 ? sp.sp[1].ncols : 0));
        char cls[64];
        snprintf(cls, sizeof cls, "%s", upd ? "fused_update_gram" : "gram");
        if (upd && prof_step) snprintf(cls, sizeof cls, "fused_update_gram@kp%04d", fz->kp);
        Prof pr(c, cls, bytes + bytes_upd, 2.0 * x.rows * (double)M * sp.N + flops_upd);
        CUDA_OK(tile_launch(p, upd, grid, c->stream, &c->launches));
      } else {
        CUDA_OK(cudaMemsetAsync(c->partial.d() + per_cta * cta_base, 0,
                                per_cta * grid * sizeof(double), c->stream));
      }
      cta_base += grid;
    }
    p.partial = c->partial.d();
    reduce(p, cta_base, gout ? gout : c->G.d(), gout ? gout_ld : 0, (double)cta_base * per_cta * 8.0);
    if (use_coll && do_allreduce) allreduce_after_reduce(c->G.d(), (size_t)M * p.N);
    if (count_sync) record(label, (long)M * p.N);
    return M;
  }

  // ---------------- K2 ----------------
  struct Upd {
    int kp = 0;
    bool has_a = false, has_b = false, cb_has_a = false;
    int srcA = SQ; long colA = 0; long dstA = 0;  // dst always in Q
    const double* CA = nullptr; long ldca = 0; const double* TA = nullptr;
    int srcB = SX; long colB = 0; long dstB = 0;
    const double* CB = nullptr; long ldcb = 0; const double* TB = nullptr;
  };
  void update(const Upd& u) {
    flush_reduce();
    if (u.has_a && u.srcA == SX) need_x(u.colA + s);
    if (u.has_b && u.srcB == SX) need_x(u.colB + s);
    for (auto& x : sh) {
      if (x.rows <= 0) continue;
      UpdateParams p;
      memset(&p, 0, sizeof p);
      p.n_rows = x.rows;
      p.qp = x.Q;
      p.ldq = x.ldq;
      p.kp = u.kp;
      p.s = (int)s;
      p.has_a = u.has_a;
      p.has_b = u.has_b;
      p.cb_has_a = u.cb_has_a;
      if (u.has_a) {
        p.srcA = colp(x, u.srcA, u.colA);
        p.ld_srcA = u.srcA == SX ? x.ldx : x.ldq;
        p.dstA = qcol(x, u.dstA);
        p.ld_dstA = x.ldq;
        p.CA = u.CA; p.ldca = u.ldca; p.TA = u.TA; p.ldta = s;
      }
      if (u.has_b) {
        p.srcB = colp(x, u.srcB, u.colB);
        p.ld_srcB = u.srcB == SX ? x.ldx : x.ldq;
        p.dstB = qcol(x, u.dstB);
        p.ld_dstB = x.ldq;
        p.CB = u.CB; p.ldcb = u.ldcb; p.TB = u.TB; p.ldtb = s;
      }
      p.status = status;
      const int nout = (u.has_a ? 1 : 0) + (u.has_b ? 1 : 0);
      Prof pr(c, "update", 8.0 * x.rows * ((double)u.kp + 2.0 * s * nout),
              2.0 * x.rows * (double)u.kp * s * nout + (double)x.rows * s * s * nout);
      // A prefix longer than one launch's coefficient panel (s = 16 past m ~ 880): chained
      // launches over column chunks, in place; the triangular factors and B's coupling to A
      // act in the last one.
      static const int kmax_env = [] {
        const char* e = getenv("BGS_UPDATE_MAXKP");  // tests: force the chained path
        return e ? atoi(e) : 0;
      }();
      // s = 5..16 with kp a multiple of 8: K2m (update_tma.cu), TMA-fed; BGS_K2M=0: K2t
      if (!no_k2m && s >= 5 && s <= 16 && u.kp >= 8 && u.kp % 8 == 0) {
        int km = update_tma_max_kp((int)s) & ~7;
        if (kmax_env > 0) km = std::min(km, std::max(8, kmax_env & ~7));
        for (int c0 = 0; c0 < u.kp; c0 += km) {
          const int c1 = std::min(u.kp, c0 + km);
          const bool last = c1 == u.kp;
          UpdTmaParams q;
          memset(&q, 0, sizeof q);
          for (int wi = 0; wi < 5; ++wi) q.map[wi] = x.mapQ[0][wi];  // boxes {16, 2, w}
          q.col0 = c0;
          q.n_rows = x.rows;
          q.kp = c1 - c0;
          q.s = (int)s;
          q.has_a = u.has_a;
          q.has_b = u.has_b;
          q.cb_has_a = last ? u.cb_has_a : 0;
          q.status = status;
          c->coefws.ensure(update_tma_coef_doubles((int)s, q.kp) * sizeof(double) + 64);
          q.coef_ws = c->coefws.d();
          if (u.has_a) {
            q.srcA = c0 > 0 ? p.dstA : p.srcA; q.ld_srcA = c0 > 0 ? p.ld_dstA : p.ld_srcA;
            q.dstA = p.dstA; q.ld_dstA = p.ld_dstA;
            q.CA = u.CA + c0; q.ldca = u.ldca; q.TA = last ? u.TA : nullptr;
          }
          if (u.has_b) {
            q.srcB = c0 > 0 ? p.dstB : p.srcB; q.ld_srcB = c0 > 0 ? p.ld_dstB : p.ld_srcB;
            q.dstB = p.dstB; q.ld_dstB = p.ld_dstB;
            q.CB = u.CB + c0; q.ldcb = u.ldcb; q.TB = last ? u.TB : nullptr;
          }
          CUDA_OK(update_tma_launch(q, c->sms, c->stream, &c->launches));
        }
        continue;
      }
      int kmax = update_max_kp((int)s);
      if (kmax_env > 0) kmax = std::min(kmax, std::max(4, kmax_env & ~3));
      if (u.kp <= kmax) {
        CUDA_OK(update_launch(p, c->sms, c->stream, &c->launches));
        continue;
      }
      for (int c0 = 0; c0 < u.kp; c0 += kmax) {
        const int c1 = std::min(u.kp, c0 + kmax);
        const bool last = c1 == u.kp;
        UpdateParams pc = p;
        pc.kp = c1 - c0;
        pc.qp = x.Q + (size_t)c0 * x.ldq;
        if (u.has_a) {
          pc.CA = u.CA + c0;
          pc.TA = last ? u.TA : nullptr;
          if (c0 > 0) { pc.srcA = pc.dstA; pc.ld_srcA = pc.ld_dstA; }
        }
        if (u.has_b) {
          pc.CB = u.CB + c0;
          pc.TB = last ? u.TB : nullptr;
          pc.cb_has_a = last ? u.cb_has_a : 0;
          if (c0 > 0) { pc.srcB = pc.dstB; pc.ld_srcB = pc.ld_dstB; }
        }
        CUDA_OK(update_launch(pc, c->sms, c->stream, &c->launches));
      }
    }
  }

  // ---------------- K3 ----------------
  void small(SmallParams p) {
    p.s = (int)s;
    p.R = c->R.d();
    p.ldr = (int)m;
    p.status = status;
    if (pend.on && pend.xchg && small_mergeable(p)) {
      // the step across ranks: reduce + push + flags, [wait], rank-ordered sum + step
      bgs_ctx::PeerComm& pc = c->peer;
      if (pend.words * sizeof(double) > pc.view.slot_bytes)
        fail(BGS_E_CONFIG, "peer window slot (%lu bytes) is smaller than the exchange payload (%zu bytes)",
             pc.view.slot_bytes, pend.words * sizeof(double));
      pend.on = false;
      pend.xchg = false;
      const unsigned ep = ++pc.epoch;
      ReducePush push;
      memset(&push, 0, sizeof push);
      push.n = pc.view.P;
      for (int r = 0; r < pc.view.P; ++r)
        push.dst[r] = reinterpret_cast<double*>(
            pc.view.win[r] + kPeerFlagBytes +
            ((size_t)(ep & 1u) * pc.view.P + pc.view.rank) * pc.view.slot_bytes);
      unsigned* tk = static_cast<unsigned*>(c->ticket.p);
      if (pc.wait_mode == 2 && peer_one) {
        Prof pr(c, "reduce_xchg_small", pend.bytes, 0.0);
        CUDA_OK(reduce_xchg_small_launch(pend.a, pend.entries, push, pc.view, ep, pend.words,
                                         pend.a.out, p, tk, c->sms, c->stream, &c->launches));
      } else {
        {
          Prof pr(c, "reduce_push", pend.bytes, 0.0);
          CUDA_OK(reduce_push_launch(pend.a, pend.entries, push, pc.view, ep, tk, c->sms, c->stream,
                                     &c->launches));
        }
        if (pc.wait_mode == 1) {
          for (int r = 0; r < pc.view.P; ++r) {
            if (r == pc.view.rank) continue;  // (stream order covers the local push)
            stream_wait_geq(c->stream, reinterpret_cast<unsigned*>(pc.window) + r, ep);
          }
          ++waits;
        }
        Prof pr(c, "sum_small", (double)pend.words * 8.0 * pc.view.P, 0.0);
        CUDA_OK(sum_small_launch(pc.view, ep, pc.wait_mode == 2, pend.words, pend.a.out, p, tk,
                                 c->sms, c->stream, &c->launches));
      }
      merged_mark = c->launches;
      merged_waits = waits;
      return;
    }
    if (pend.on && !pend.xchg && small_mergeable(p)) {
      pend.on = false;
      Prof pr(c, "reduce_small", pend.bytes, 0.0);
      CUDA_OK(reduce_small_launch(pend.a, pend.entries, p, static_cast<unsigned*>(c->ticket.p),
                                  c->sms, c->stream, &c->launches));
      merged_mark = c->launches;
      merged_waits = waits;
      return;
    }
    flush_reduce();
    Prof pr(c, "small", 0.0, 0.0);
    CUDA_OK(small_launch(p, c->stream, &c->launches));
  }

  // ---------------- K4: TSQR of an n x s block -> Q block, root R -> rout ----------------
  // fusedG/fusedCount: a Gram computed before this call that rides in the same
  // rendezvous (tsqr_fused_gram, intraorth.cpp:122-135).
  void tsqr(int src, long scol_, long dcol, double* rout, int ldrout, const char* label,
            long fused_words = 0, double* fusedG = nullptr) {
    flush_reduce();
    if (src == SX) need_x(scol_ + s);
    const size_t ss = (size_t)s * s;
    double* ws = c->tsqr_ws.d();
    const long* bounds = static_cast<const long*>(c->tsqr_bounds.p);
    for (auto& x : sh) {
      Prof pr(c, "tsqr_leaf", 16.0 * x.rows * s, 8.0 * x.rows * s * s);
      CUDA_OK(tsqr_leaf_launch(colp(x, src, scol_), src == SX ? x.ldx : x.ldq, qcol(x, dcol),
                               x.ldq, bounds + x.bound_base, x.n_leaves, x.hmax, (int)s,
                               tsqr_ws_R(ws) + (size_t)x.leaf_base * ss, status, c->stream,
                               &c->launches));
    }
    {
      Prof pr(c, "tsqr_tree", 0.0, 0.0);
      for (size_t t = 0; t < sh.size(); ++t)
        CUDA_OK(tsqr_tree_up_shard(ws, tsqr_L, sh[t].leaf_base, sh[t].n_leaves, (int)s,
                                   c->roots.d() + t * ss, status, c->stream, &c->launches));
    }
    const double* all_roots = c->roots.d();
    if (use_coll) {
      // one rendezvous: allgather of the per-rank roots + the fused Gram's allreduce
      exchange(c->roots.d(), ss, c->roots_all.d(), fusedG, fusedG ? (size_t)fused_words : 0);
      all_roots = c->roots_all.d();
    }
    const double* mtop = nullptr;  // identity: a single shard's root is the global root
    if (P == 1 && sh.size() == 1) {
      CUDA_OK(cudaMemcpy2DAsync(rout, (size_t)ldrout * sizeof(double), all_roots, s * sizeof(double),
                                s * sizeof(double), s, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      Prof pr(c, "tsqr_tree", 0.0, 0.0);
      CUDA_OK(tsqr_cross_launch(all_roots, P, (int)s, c->cross_ws.d(), rout, ldrout,
                                c->cross_m.d(), status, c->stream, &c->launches));
      mtop = c->cross_m.d() + (use_coll ? (size_t)c->rank * ss : 0);
    }
    for (size_t t = 0; t < sh.size(); ++t) {
      const Shard& x = sh[t];
      Prof pr(c, "tsqr_apply", 16.0 * x.rows * s, 2.0 * x.rows * s * s);
      CUDA_OK(tsqr_apply_path_shard(qcol(x, dcol), x.ldq, bounds + x.bound_base, ws, tsqr_L,
                                    x.leaf_base, x.n_leaves, (int)s, mtop ? mtop + t * ss : nullptr,
                                    status, c->stream, &c->launches));
    }
    record(label, (long)ss + fused_words);
  }

  // ---------------- variant drivers ----------------
  static GramSpec spec1(int src, int col0, int ncols, int lcols) {
    GramSpec g;
    g.nspans = 1;
    g.sp[0] = {src, col0, ncols, lcols};
    return g;
  }
  static GramSpec spec2(int src0, int col0, int n0, int l0, int src1, int col1, int n1, int l1) {
    GramSpec g;
    g.nspans = 2;
    g.sp[0] = {src0, col0, n0, l0};
    g.sp[1] = {src1, col1, n1, l1};
    return g;
  }
  static void add_right(GramSpec& g, int span, int col, int cnt) {
    for (int j = 0; j < cnt; ++j) {
      g.rspan[g.N + j] = span;
      g.rcol[g.N + j] = col + j;
    }
    g.N += cnt;
  }

  double* Rd() { return c->R.d(); }

  // q = 1 (bcgs.cpp:83-90)
  void single_block() { tsqr(SX, 0, 0, Rd(), (int)m, "reduce_factor_tree:tsqr"); }

  // Can the block update producing the left operand of `g` be fused in front of it?
  bool fuse_ok(const GramSpec& g, int kp) const {
    if (no_fuse || s > 4 || g.N > 8) return false;
    int units = 0;
    for (int i = 0; i < g.nspans; ++i) units += (g.sp[i].ncols + 7) / 8;
    const bool span1_left = g.nspans == 2 && g.sp[1].lcols > 0;
    const int mt_out = span1_left ? (g.sp[0].ncols + 7) / 8 + (g.sp[1].lcols + 7) / 8
                                  : (g.sp[0].lcols + 7) / 8;
    if (tile_fused_supported((int)s, kp, mt_out) &&
        tile_smem_bytes(2, 2, units, true) <= (size_t)TILE_SMEM_MAX)
      return true;
    SplitParams p;  // K12c can take shapes the single-CTA K12 cannot (CTA pairs)
    return split_params(g, true, true, kp, p);
  }

  // Gram of one-sync step j over [Q_{1:j} U_j (X_{j+1})] when U_j already sits in Q
  // block j (unfused layout; fused_gram:wide / :final, bcgs.cpp:303-319).
  GramSpec onesync_spec_unfused(int mode, long j) const {
    const int si = (int)s, kp = (int)(j * s);
    GramSpec g;
    if (j + 1 < q) {
      g = spec2(SQ, 0, kp + si, kp + si, SX, kp + si, si, mode == OS_PYTH ? si : 0);
      add_right(g, 0, kp, si);
      add_right(g, 1, 0, si);
    } else {
      g = spec1(SQ, 0, kp + si, kp + si);
      add_right(g, 0, kp, si);
    }
    if (comp_tail(mode)) g.comp_row = kp;  // U_j in Q block j
    return g;
  }
  // BCGSI+1S carries U unnormalized: its Gram rows U^T [U X] feed Y_diag = chol(Omega -
  // Y^T Y) and S2 directly, so they get the compensated accumulation (DESIGN.md
  // "Numerics").  BGS_COMP_TAIL=0: off; =all: every one-sync mode (experiments).
  bool comp_tail(int mode) const {
    return comp_mode == 2 || (comp_mode == 1 && mode == OS_SKIP);
  }
  // The same Gram on the tile of a fused update: Q_{1:j} in span 0, [X_j -> U_j, X_{j+1}]
  // in span 1 (U_j produced in place by the update).
  GramSpec onesync_spec_fused(int mode, long j) const {
    const int si = (int)s, kp = (int)(j * s);
    const bool wide = j + 1 < q;
    GramSpec g = spec2(SQ, 0, kp, kp, SX, kp, wide ? 2 * si : si,
                       (wide && mode == OS_PYTH) ? 2 * si : si);
    add_right(g, 1, 0, si);
    if (wide) add_right(g, 1, si, si);
    if (comp_tail(mode)) g.comp_row = kp;  // U_j: the first span-1 output row
    return g;
  }

  // onesync_impl (bcgs.cpp:233-369); modes PythChol (P-1S), SkipNorm (I+1S), TsqrPath (P-2S)
  void onesync(int mode, int kappa_power) {
    if (q == 1) return single_block();
    defer_reduce = !no_merge_small;
    struct Undefer {
      Runner* r;
      ~Undefer() { r->defer_reduce = false; }
    } undefer{this};
    const int si = (int)s;
    double* scol_cur = c->scolA.d();
    double* scol_nxt = c->scolB.d();
    double* sdiag = c->sdiag.d();
    double* ydiag = c->ydiag.d();
    const bool fusable = mode != OS_TSQR;
    int M;
    // ---- prologue: TSQR(X_1) with the first Gram in the same rendezvous ----
    {
      const int lc = mode == OS_PYTH ? 2 * si : si;
      GramSpec g = spec1(SX, 0, 2 * si, lc);
      add_right(g, 0, si, si);
      const int M0 = gram(g, "", /*count_sync=*/false, /*do_allreduce=*/false);
      tsqr(SX, 0, 0, c->rtop.d(), si, "reduce_factor_tree:prologue", (long)M0 * si, c->G.d());
      SmallParams sp;
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_ONESYNC_PROLOGUE;
      sp.os_mode = mode;
      sp.kappa_power = kappa_power;
      sp.G = c->G.d(); sp.ldg = M0; sp.gm = M0; sp.gn = si;
      sp.rtop = c->rtop.d(); sp.ldrtop = si;
      sp.scol_next = scol_cur; sp.ld_scol_next = si;
      sp.sdiag = sdiag;
      small(sp);
      // U_2 = (X_2 - Q_1 S_12) S_22^{-1}, then the Gram of step 1 (fused when possible)
      const char* lab = q > 2 ? "fused_gram:wide" : "fused_gram:final";
      GramSpec gf = onesync_spec_fused(mode, 1);
      if (fusable && fuse_ok(gf, si)) {
        Fuse fz;
        fz.b = true;
        fz.kp = si;
        fz.CB = scol_cur; fz.ldcb = si;
        fz.TB = mode == OS_PYTH ? sdiag : nullptr;
        fz.dstB = si;
        M = gram(gf, lab, true, true, &fz);
      } else {
        Upd u;
        u.kp = si;
        u.has_b = true;
        u.srcB = SX; u.colB = si; u.dstB = si;
        u.CB = scol_cur; u.ldcb = si;
        u.TB = mode == OS_PYTH ? sdiag : nullptr;
        update(u);
        if (mode == OS_TSQR) tsqr(SQ, si, si, sdiag, si, "reduce_factor_tree:tsqr");
        M = gram(onesync_spec_unfused(mode, 1), lab);
      }
    }
    // ---- block steps ----
    for (long k = 1; k < q; ++k) {
      const int kp = (int)(k * s);
      const bool has_next = k + 1 < q;
      SmallParams sp;
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_ONESYNC_STEP;
      sp.os_mode = mode;
      sp.k = (int)k;
      sp.kp = kp;
      sp.has_next = has_next;
      sp.kappa_power = kappa_power;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = has_next ? 2 * si : si;
      sp.scol_prev = scol_cur; sp.ld_scol_prev = kp;
      sp.scol_next = scol_nxt; sp.ld_scol_next = kp + si;
      sp.sdiag = sdiag;
      sp.ydiag = ydiag;
      small(sp);
      if (!has_next) {
        // Q_q = (U_q - Q_{1:q-1} Y) Y_qq^{-1}  (bcgs.cpp:329-331)
        Upd u;
        u.kp = kp;
        u.has_a = true;
        u.srcA = SQ; u.colA = kp; u.dstA = kp;
        u.CA = c->G.d(); u.ldca = M; u.TA = ydiag;
        update(u);
        q_final(m);
        break;
      }
      // Q_k = (U_k - Q_{1:k} Y) Y_kk^{-1}; U_{k+1} = (X_{k+1} - Q_{1:k+1} [Z; S2]) S^{-1};
      // then the Gram of step k+1 — one pass over Q_{1:k} when fused.
      const char* lab = k + 2 < q ? "fused_gram:wide" : "fused_gram:final";
      GramSpec gf = onesync_spec_fused(mode, k + 1);
      gf.sp[0].ncols = gf.sp[0].lcols = kp + si;  // span 0 = [Q_{1:k} | U_k -> Q_k]
      if (comp_tail(mode)) gf.comp_row = kp + si;  // U_{k+1}: span 1
      // (span 1 still starts at X block k+1)
      if (fusable && fuse_ok(gf, kp)) {
        Fuse fz;
        fz.a = fz.b = true;
        fz.kp = kp;
        fz.CA = c->G.d(); fz.ldca = M; fz.TA = ydiag; fz.dstA = kp;
        fz.CB = scol_nxt; fz.ldcb = kp + si; fz.TB = mode == OS_PYTH ? sdiag : nullptr;
        fz.dstB = kp + si;
        M = gram(gf, lab, true, true, &fz);
      } else {
        Upd u;
        u.kp = kp;
        u.has_a = true;
        u.srcA = SQ; u.colA = kp; u.dstA = kp;
        u.CA = c->G.d(); u.ldca = M; u.TA = ydiag;
        u.has_b = true;
        u.cb_has_a = true;
        u.srcB = SX; u.colB = kp + si; u.dstB = kp + si;
        u.CB = scol_nxt; u.ldcb = kp + si;
        u.TB = mode == OS_PYTH ? sdiag : nullptr;
        update(u);
        if (mode == OS_TSQR) tsqr(SQ, kp + si, kp + si, sdiag, si, "reduce_factor_tree:tsqr");
        M = gram(onesync_spec_unfused(mode, k + 1), lab);
      }
      fire_probe(k, scol_nxt + kp, kp + si);  // S2 = rows kp.. of the next scol
      q_final(kp + si);  // later steps only write columns >= kp + s
      std::swap(scol_cur, scol_nxt);
    }
  }

  // classic_impl (bcgs.cpp:92-133): one projection, then the intra-block QR (TSQR, or
  // Cholesky QR when BcgsOptions::classic_intra says so) of X_k - Q_{1:k} S.
  void intra_qr(int src, long col, long k) {
    const int si = (int)s;
    const bool chol = opt && opt->classic_intra == 1;
    if (!chol) {
      tsqr(src, col, col, c->r1.d(), si, "reduce_factor_tree:tsqr");
      return;
    }
    // cholqr (intraorth.cpp:136-151): G = U^T U (one sync), R = chol(G), Q = U R^{-1}
    GramSpec g = spec1(src, (int)col, si, si);
    add_right(g, 0, 0, si);
    const int M = gram(g, "fused_gram:cholqr");
    SmallParams sp;
    memset(&sp, 0, sizeof sp);
    sp.mode = SM_CHOLQR;
    sp.k = (int)k;
    sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
    sp.sdiag = c->r1.d();
    small(sp);
    Upd u;
    u.kp = 0;
    u.has_a = true;
    u.srcA = src; u.colA = col; u.dstA = col;
    u.TA = c->r1.d();
    update(u);
  }
  void classic() {
    if (q == 1) return single_block();
    const int si = (int)s;
    SmallParams sp;
    memset(&sp, 0, sizeof sp);
    intra_qr(SX, 0, 0);
    sp.mode = SM_CLASSIC_FINISH;  // R(0,0)
    sp.rtop = c->r1.d(); sp.ldrtop = si;
    small(sp);
    for (long k = 1; k < q; ++k) {
      const int kp = (int)(k * s);
      GramSpec g = spec2(SQ, 0, kp, kp, SX, kp, si, 0);
      add_right(g, 1, 0, si);
      const int M = gram(g, "fused_gram:proj");
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_IRO_SAVE;
      sp.k = (int)k; sp.kp = kp;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
      sp.save = c->save.d(); sp.ldsave = kp;
      small(sp);
      Upd u;
      u.kp = kp;
      u.has_a = true;
      u.srcA = SX; u.colA = kp; u.dstA = kp;
      u.CA = c->save.d(); u.ldca = kp; u.TA = nullptr;
      update(u);
      intra_qr(SQ, kp, k);
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_CLASSIC_FINISH;
      sp.k = (int)k; sp.kp = kp;
      sp.aux1 = c->save.d(); sp.ldaux1 = kp;
      sp.rtop = c->r1.d(); sp.ldrtop = si;
      small(sp);
    }
  }

  // pipi_impl (bcgs.cpp:169-219)
  void pipi() {
    if (q == 1) return single_block();
    const int si = (int)s;
    tsqr(SX, 0, 0, Rd(), (int)m, "reduce_factor_tree:tsqr");
    // [S; T] = [Q_1 X_2]^T X_2
    GramSpec g0 = spec2(SQ, 0, si, si, SX, si, si, si);
    add_right(g0, 1, 0, si);
    int M = gram(g0, "fused_gram:proj");
    for (long k = 1; k < q; ++k) {
      const int kp = (int)(k * s);
      SmallParams sp;
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_PIPI_PROJ;
      sp.k = (int)k; sp.kp = kp; sp.kappa_power = 2;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
      sp.save = c->save.d(); sp.ldsave = kp;
      sp.sdiag = c->sdiag.d();
      small(sp);
      // U = (X_k - Q S) S_kk^{-1}, then [Y; Omega] = [Q U]^T U  (bcgs.cpp:196-204)
      GramSpec gr = spec2(SQ, 0, kp, kp, SX, kp, si, si);
      add_right(gr, 1, 0, si);
      if (fuse_ok(gr, kp)) {
        Fuse fz;
        fz.b = true;
        fz.kp = kp;
        fz.CB = c->save.d(); fz.ldcb = kp; fz.TB = c->sdiag.d(); fz.dstB = kp;
        M = gram(gr, "fused_gram:reproj", true, true, &fz);
      } else {
        Upd u;
        u.kp = kp;
        u.has_a = true;
        u.srcA = SX; u.colA = kp; u.dstA = kp;
        u.CA = c->save.d(); u.ldca = kp; u.TA = c->sdiag.d();
        update(u);
        GramSpec g2 = spec1(SQ, 0, kp + si, kp + si);
        add_right(g2, 0, kp, si);
        M = gram(g2, "fused_gram:reproj");
      }
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_PIPI_REPROJ;
      sp.k = (int)k; sp.kp = kp; sp.kappa_power = 2;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
      sp.aux1 = c->save.d(); sp.ldaux1 = kp;
      sp.sdiag = c->sdiag.d();
      sp.ydiag = c->ydiag.d();
      small(sp);
      // Q_k = (U - Q Y) Y_kk^{-1}, then the next step's [Q X_{k+1}]^T X_{k+1}
      if (k + 1 < q) {
        GramSpec gp = spec2(SQ, 0, kp + si, kp + si, SX, kp + si, si, si);
        add_right(gp, 1, 0, si);
        if (fuse_ok(gp, kp)) {
          Fuse fz;
          fz.a = true;
          fz.kp = kp;
          fz.CA = c->G.d(); fz.ldca = M; fz.TA = c->ydiag.d(); fz.dstA = kp;
          M = gram(gp, "fused_gram:proj", true, true, &fz);
          continue;
        }
      }
      Upd u2;
      u2.kp = kp;
      u2.has_a = true;
      u2.srcA = SQ; u2.colA = kp; u2.dstA = kp;
      u2.CA = c->G.d(); u2.ldca = M; u2.TA = c->ydiag.d();
      update(u2);
      if (k + 1 < q) {
        GramSpec gp = spec2(SQ, 0, kp + si, kp + si, SX, kp + si, si, si);
        add_right(gp, 1, 0, si);
        M = gram(gp, "fused_gram:proj");
      }
    }
  }

  // iro_impl (bcgs.cpp:135-167)
  void iro() {
    if (q == 1) return single_block();
    const int si = (int)s;
    tsqr(SX, 0, 0, Rd(), (int)m, "reduce_factor_tree:tsqr");
    for (long k = 1; k < q; ++k) {
      const int kp = (int)(k * s);
      GramSpec g = spec2(SQ, 0, kp, kp, SX, kp, si, 0);
      add_right(g, 1, 0, si);
      int M = gram(g, "fused_gram:proj1");
      SmallParams sp;
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_IRO_SAVE;
      sp.k = (int)k; sp.kp = kp;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
      sp.save = c->save.d(); sp.ldsave = kp;
      small(sp);
      Upd u;
      u.kp = kp;
      u.has_a = true;
      u.srcA = SX; u.colA = kp; u.dstA = kp;
      u.CA = c->save.d(); u.ldca = kp; u.TA = nullptr;
      update(u);
      tsqr(SQ, kp, kp, c->r1.d(), si, "reduce_factor_tree:tsqr");
      GramSpec g2 = spec1(SQ, 0, kp + si, kp);
      add_right(g2, 0, kp, si);
      M = gram(g2, "fused_gram:proj2");
      Upd u2;
      u2.kp = kp;
      u2.has_a = true;
      u2.srcA = SQ; u2.colA = kp; u2.dstA = kp;
      u2.CA = c->G.d(); u2.ldca = M; u2.TA = nullptr;
      update(u2);
      tsqr(SQ, kp, kp, c->r2.d(), si, "reduce_factor_tree:tsqr");
      memset(&sp, 0, sizeof sp);
      sp.mode = SM_IRO_FINISH;
      sp.k = (int)k; sp.kp = kp;
      sp.G = c->G.d(); sp.ldg = M; sp.gm = M; sp.gn = si;
      sp.aux1 = c->save.d(); sp.ldaux1 = kp;
      sp.aux2 = c->r1.d(); sp.ldaux2 = si;
      sp.rtop = c->r2.d(); sp.ldrtop = si;
      small(sp);
    }
  }

  void dump_phase_profile() {
    if (!tile_prof) return;
    std::vector<unsigned long long> h(512 * 16);
    cudaMemcpy(h.data(), c->metrics.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double tot[16] = {0};
    for (int b = 0; b < 256; ++b)
      for (int i = 0; i < 16; ++i) tot[i] += (double)h[b * 16 + i];
    const double st = tot[9] > 0 ? tot[9] : 1;
    fprintf(stderr,
            "[tile phases] stages %.0f | cycles per stage (thread 0): wait %.0f update %.0f "
            "reduce %.0f epilogue %.0f gram %.0f fence+arrive %.0f refill %.0f (empty-wait %.0f) "
            "flush %.0f | total %.0f\n",
            tot[9], tot[0] / st, tot[1] / st, tot[2] / st, tot[3] / st, tot[4] / st, tot[6] / st,
            tot[7] / st, tot[10] / st, tot[8] / st, tot[5] / st);
    // K12c: [cta][group][full-wait, update, exchange, epilogue, gram, total, stages]
    double kt[8] = {0};
    for (int b = 0; b < 160; ++b)  // (cells from 2560 on hold CTA 0's timeline)
      for (int g = 0; g < 2; ++g)
        for (int i = 0; i < 7; ++i) kt[i] += (double)h[256 * 16 + b * 16 + 8 * g + i];
    if (kt[6] > 0)
      fprintf(stderr,
              "[k12c phases] group-stages %.0f | cycles per group-stage: full-wait %.0f update %.0f "
              "exchange %.0f epilogue %.0f gram %.0f | total %.0f\n",
              kt[6], kt[0] / kt[6], kt[1] / kt[6], kt[2] / kt[6], kt[3] / kt[6], kt[4] / kt[6],
              kt[5] / kt[6]);
    // K12c timeline of CTA 0 in the last profiled launch: [group][stage][6 stamps]
    constexpr int kTl0 = 4096 + 2560;
    if (getenv("BGS_TIMELINE") && h[kTl0] != 0) {
      const unsigned long long base = std::min(h[kTl0], h[kTl0 + 48 * 6]);
      for (int g = 0; g < 2; ++g)
        for (int j = 0; j < 48; ++j) {
          const unsigned long long* t = &h[kTl0 + (g * 48 + j) * 6];
          if (!t[0]) continue;
          fprintf(stderr, "[k12c timeline] g %d j %2d:", g, j);
          for (int i = 0; i < 6; ++i) fprintf(stderr, " %llu", t[i] - base);
          fprintf(stderr, "\n");
        }
    }
  }

  void run() {
    if (tile_prof) {
      c->metrics.ensure((size_t)512 * 16 * sizeof(unsigned long long) + 64);
      CUDA_OK(cudaMemsetAsync(c->metrics.p, 0, 512 * 16 * sizeof(unsigned long long), c->stream));
    }
    setup();
    switch (variant) {
      case BGS_BCGS: classic(); break;
      case BGS_BCGSI_PLUS: iro(); break;
      case BGS_BCGSPIPI_PLUS: pipi(); break;
      case BGS_BCGSI_PLUS_P_1S: onesync(OS_PYTH, 2); break;
      case BGS_BCGSI_PLUS_P_2S: onesync(OS_TSQR, 1); break;
      case BGS_BCGSI_PLUS_1S: onesync(OS_SKIP, 3); break;
      default: fail(BGS_E_CONFIG, "variant %d is out of scope", variant);
    }
    flush_reduce();
    q_final(m);
  }

  // Converts the device status word into the reference's exception semantics.
  void check_status() {
    DevStatus h;
    CUDA_OK(cudaMemcpy(&h, status, sizeof h, cudaMemcpyDeviceToHost));
    if (h.code == 0) return;
    Fail f;
    f.code = h.code;
    f.pivot = h.pivot;
    f.block = h.block;
    if (h.code == ST_NOT_SPD) {
      const char* site = h.site == SITE_PROLOGUE_PYTH ? "prologue Pythagorean normalization"
                         : h.site == SITE_FIRST_PASS  ? "first-pass Pythagorean normalization"
                         : h.site == SITE_INTRA_CHOLQR ? "intra-block Cholesky QR"
                                                      : "second-pass Pythagorean normalization";
      f.site = site;
      std::string hyp;
      if (h.kappa_power == 1) hyp = "O(u) * kappa(X) <= 1";
      else if (h.kappa_power > 1) hyp = "O(u) * kappa(X)^" + std::to_string(h.kappa_power) + " <= 1";
      char buf[1024];
      snprintf(buf, sizeof buf,
               "%s: %s for block column %d hit a Gram matrix that is not numerically positive "
               "definite (cholesky pivot %d is not strictly positive)%s%s",
               kVariantNames[variant], site, h.block, h.pivot,
               hyp.empty() ? "" : "; likely violated working assumption: ", hyp.c_str());
      f.msg = buf;
    } else if (h.code == ST_NON_FINITE) {
      f.msg = "reduction saw a NaN or infinity";
      if (getenv("BGS_DEBUG_STATUS")) f.msg += " (block column " + std::to_string(h.block) + ")";
    } else if (h.code == ST_SINGULAR) {
      f.msg = "triangular factor has a zero at diagonal entry " + std::to_string(h.pivot);
    } else if (h.code == ST_COLLECTIVE) {
      f.msg = "peer exchange: rank " + std::to_string(h.pivot - 1) +
              " never published its flag (gave up after ~8 s; rank " + std::to_string(c->rank) + " of " +
              std::to_string(c->nranks) + ")";
    } else {
      f.msg = "device status " + std::to_string(h.code);
    }
    throw f;
  }
};

void validate(int variant, long n, long m, long s, int procs) {
  if (procs < 1) fail(BGS_E_DIMENSION, "run_spmd: procs must be >= 1");
  if (s <= 0 || m % s != 0) fail(BGS_E_DIMENSION, "distribute: block width must divide the columns");
  if (m == 0)
    fail(BGS_E_DIMENSION, "bcgs: column count must be a positive multiple of the block width");
  if (n < m)
    fail(BGS_E_DIMENSION, "bcgs: economic factorization needs at least as many rows as columns");
  if (variant < 0 || variant > 5) fail(BGS_E_CONFIG, "unknown variant id %d", variant);
  if (s > 16) fail(BGS_E_CONFIG, "block width s = %ld exceeds the supported maximum 16", s);
  if (m > 4096) fail(BGS_E_CONFIG, "m = %ld exceeds the supported maximum 4096", m);
}

void select_device(bgs_ctx* c) {
  if (!c) fail(BGS_E_CUDA, "null context");
  CUDA_OK(cudaSetDevice(c->device));
}

}  // namespace

// Leading dimension of library-owned device buffers: rows rounded up to 32 (the tile
// engine's TMA view reads whole 16-row blocks; 32 keeps 256-byte column alignment).

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

const char* bgs_variant_name(int v) { return (v >= 0 && v < 6) ? kVariantNames[v] : nullptr; }

int bgs_parse_variant(const char* name, int* variant, bgs_error* err) {
  clear_err(err);
  std::string key(name ? name : "");
  for (auto& ch : key) ch = (char)std::toupper((unsigned char)ch);
  for (int v = 0; v < 6; ++v) {
    if (key == kVariantNames[v]) {
      if (variant) *variant = v;
      return BGS_OK;
    }
  }
  if (err) {
    err->code = BGS_E_CONFIG;
    snprintf(err->msg, sizeof err->msg,
             "unknown variant '%s' (expected one of BCGS, BCGSI+, BCGSPIPI+, BCGSI+P-1S, "
             "BCGSI+P-2S, BCGSI+1S)",
             name ? name : "");
  }
  return BGS_E_CONFIG;
}

long bgs_expected_syncs(int v, long q) {
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

double bgs_variant_flops(int v, long n, long m, long s) {
  if (s < 1 || m < 1 || m % s != 0 || n < m) return -1.0;
  const long q = m / s;
  const double dn = (double)n, ds = (double)s;
  const double block_qr = 4.0 * dn * ds * ds, block_scale = dn * ds * ds;
  auto gu = [dn](double a, double b) { return 2.0 * dn * a * b; };
  if (q == 1) return block_qr;
  double f = 0.0;
  switch (v) {
    case 0:
      f = block_qr;
      for (long k = 1; k < q; ++k) f += gu(k * ds, ds) * 2 + block_qr;
      return f;
    case 1:
      f = block_qr;
      for (long k = 1; k < q; ++k) f += 2.0 * (gu(k * ds, ds) + gu(k * ds, ds) + block_qr);
      return f;
    case 2:
      f = block_qr;
      for (long k = 1; k < q; ++k)
        f += 2.0 * gu((k + 1) * ds, ds) + 2.0 * gu(k * ds, ds) + 2.0 * block_scale;
      return f;
    case 3:
      f = block_qr + gu(2.0 * ds, ds) + gu(ds, ds) + block_scale;
      for (long k = 1; k < q; ++k) {
        const bool hn = k + 1 < q;
        f += hn ? gu(k * ds + 2.0 * ds, 2.0 * ds) : gu(k * ds + ds, ds);
        f += gu(k * ds, ds) + block_scale;
        if (hn) f += gu((k + 1) * ds, ds) + block_scale;
      }
      return f;
    case 5:
      f = block_qr + gu(ds, ds) + gu(ds, ds);
      for (long k = 1; k < q; ++k) {
        const bool hn = k + 1 < q;
        f += hn ? gu(k * ds + ds, 2.0 * ds) : gu(k * ds + ds, ds);
        f += gu(k * ds, ds) + block_scale;
        if (hn) f += gu((k + 1) * ds, ds);
      }
      return f;
    case 4:
      f = block_qr + gu(ds, ds) + gu(ds, ds) + block_qr;
      for (long k = 1; k < q; ++k) {
        const bool hn = k + 1 < q;
        f += hn ? gu(k * ds + ds, 2.0 * ds) : gu(k * ds + ds, ds);
        f += gu(k * ds, ds) + block_scale;
        if (hn) f += gu((k + 1) * ds, ds) + block_qr;
      }
      return f;
  }
  return -1.0;
}

int bgs_shard_rows(long n, int procs, int rank, long* row0, long* rows) {
  if (procs < 1 || rank < 0 || rank >= procs || n < 0) return BGS_E_DIMENSION;
  const long per = (n + procs - 1) / procs;
  const long r0 = std::min((long)rank * per, n);
  const long r1 = std::min(r0 + per, n);
  if (row0) *row0 = r0;
  if (rows) *rows = r1 - r0;
  return BGS_OK;
}

int bgs_device_info(int device, int* sm_count, long* hbm_bytes, char* name, long name_cap) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return BGS_E_CUDA;
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (hbm_bytes) *hbm_bytes = (long)prop.totalGlobalMem;
  if (name && name_cap > 0) snprintf(name, (size_t)name_cap, "%s", prop.name);
  return BGS_OK;
}

int bgs_nccl_unique_id(void* out128, bgs_error* err) {
  clear_err(err);
  try {
    if (!nccl().ok) fail(BGS_E_COLLECTIVE, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    NCCL_OK(nccl().GetUniqueId(&id));
    memcpy(out128, &id, sizeof id);
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

int bgs_ctx_create(int device, int rank, int nranks, const void* uid, bgs_ctx** out,
                   bgs_error* err) {
  clear_err(err);
  *out = nullptr;
  bgs_ctx* c = new bgs_ctx();
  try {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
      fail(BGS_E_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    if (device < 0 || device >= ndev) fail(BGS_E_CUDA, "device %d out of range", device);
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    CUDA_OK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(BGS_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200)", device,
           prop.major, prop.minor);
    c->sms = prop.multiProcessorCount;
    CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreate(&c->e0));
    CUDA_OK(cudaEventCreate(&c->e1));
    CUDA_OK(cudaEventCreateWithFlags(&c->entry, cudaEventDisableTiming));
    // an NCCL communicator for every multi-rank context, and for a one-rank context
    // whose caller passes an id (the collective path on one GPU: tests, bring-up)
    if (nranks > 1 || uid) {
      if (!uid) fail(BGS_E_COLLECTIVE, "nranks > 1 needs an ncclUniqueId");
      if (!nccl().ok) fail(BGS_E_COLLECTIVE, "libnccl.so.2 could not be loaded");
      ncclUniqueId id;
      memcpy(&id, uid, sizeof id);
      NCCL_OK(nccl().CommInitRank(&c->comm, nranks, id, rank));
    }
    *out = c;
    return BGS_OK;
  } catch (const Fail& f) {
    delete c;
    put_err(err, f);
    return f.code;
  }
}

int bgs_ctx_create_host_comm(int device, int rank, int nranks, bgs_allgather_fn fn, void* user,
                             bgs_ctx** out, bgs_error* err) {
  clear_err(err);
  *out = nullptr;
  if (!fn || nranks < 1 || rank < 0 || rank >= nranks) {
    if (err) {
      err->code = BGS_E_COLLECTIVE;
      snprintf(err->msg, sizeof err->msg, "host communicator: need fn and 0 <= rank < nranks");
    }
    return BGS_E_COLLECTIVE;
  }
  bgs_ctx* c = nullptr;
  // a plain single-GPU context, then the communicator
  const int rc = bgs_ctx_create(device, 0, 1, nullptr, &c, err);
  if (rc != BGS_OK) return rc;
  c->rank = rank;
  c->nranks = nranks;
  c->hc_fn = fn;
  c->hc_user = user;
  *out = c;
  return BGS_OK;
}

// ---- peer-memory transport (peer.cu) ----
namespace {
// The 128-byte blob ranks exchange: the IPC handle of the window plus what attach checks.
struct PeerBlob {
  cudaIpcMemHandle_t ipc;  // 64 bytes
  unsigned char uuid[16];  // the GPU (ranks on one GPU must not spin on each other)
  int rank, nranks;
  unsigned long slot_bytes;
  long pid;
  unsigned long window;  // the window's address in the exporting process (same-process attach)
  char pad[16];
};
static_assert(sizeof(PeerBlob) == BGS_PEER_HANDLE_BYTES, "peer blob layout");
}  // namespace

int bgs_ctx_create_peer(int device, int rank, int nranks, unsigned long slot_bytes, bgs_ctx** out,
                        bgs_error* err) {
  clear_err(err);
  *out = nullptr;
  if (nranks < 1 || nranks > kPeerMaxRanks || rank < 0 || rank >= nranks) {
    if (err) {
      err->code = BGS_E_COLLECTIVE;
      snprintf(err->msg, sizeof err->msg, "peer context: need 0 <= rank < nranks <= %d", kPeerMaxRanks);
    }
    return BGS_E_COLLECTIVE;
  }
  bgs_ctx* c = nullptr;
  const int rc = bgs_ctx_create(device, 0, 1, nullptr, &c, err);
  if (rc != BGS_OK) return rc;
  try {
    c->rank = rank;
    c->nranks = nranks;
    // default slot: the largest exchange validate() admits, (m + 2s) x 2s Gram + an s x s root
    if (!slot_bytes) slot_bytes = ((4096ul + 32) * 32 + 256 + 64) * sizeof(double);
    slot_bytes = (slot_bytes + 255) / 256 * 256;
    const size_t wb = peer_window_bytes(nranks, slot_bytes);
    CUDA_OK(cudaMalloc(&c->peer.window, wb));  // plain cudaMalloc: IPC-exportable
    CUDA_OK(cudaMemset(c->peer.window, 0, wb));
    CUDA_OK(cudaMalloc(&c->peer.cnt, 64));
    CUDA_OK(cudaMemset(c->peer.cnt, 0, 64));
    CUDA_OK(cudaDeviceSynchronize());
    c->peer.on = true;
    c->peer.view.P = nranks;
    c->peer.view.rank = rank;
    c->peer.view.slot_bytes = slot_bytes;
    c->peer.view.win[rank] = static_cast<unsigned char*>(c->peer.window);
    *out = c;
    return BGS_OK;
  } catch (const Fail& f) {
    delete c;
    put_err(err, f);
    return f.code;
  }
}

int bgs_ctx_peer_handle(bgs_ctx* c, void* handle, bgs_error* err) {
  clear_err(err);
  try {
    if (!c || !c->peer.on) fail(BGS_E_COLLECTIVE, "not a peer context");
    CUDA_OK(cudaSetDevice(c->device));
    PeerBlob b;
    memset(&b, 0, sizeof b);
    CUDA_OK(cudaIpcGetMemHandle(&b.ipc, c->peer.window));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, c->device));
    memcpy(b.uuid, &prop.uuid, 16);
    b.rank = c->rank;
    b.nranks = c->nranks;
    b.slot_bytes = c->peer.view.slot_bytes;
    b.pid = (long)getpid();
    b.window = reinterpret_cast<unsigned long>(c->peer.window);
    memcpy(handle, &b, sizeof b);
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

int bgs_ctx_peer_attach(bgs_ctx* c, const void* handles, int wait_mode, bgs_error* err) {
  clear_err(err);
  try {
    if (!c || !c->peer.on) fail(BGS_E_COLLECTIVE, "not a peer context");
    if (c->peer.attached) fail(BGS_E_COLLECTIVE, "peer context already attached");
    if (wait_mode < 0 || wait_mode > 2) fail(BGS_E_CONFIG, "peer wait mode must be 0 (auto), 1 (stream) or 2 (spin)");
    CUDA_OK(cudaSetDevice(c->device));
    const int P = c->nranks;
    const PeerBlob* hb = static_cast<const PeerBlob*>(handles);
    bool shared_gpu = false;
    for (int r = 0; r < P; ++r) {
      PeerBlob b;
      memcpy(&b, hb + r, sizeof b);
      if (b.rank != r || b.nranks != P || b.slot_bytes != c->peer.view.slot_bytes)
        fail(BGS_E_COLLECTIVE, "peer handle %d does not match (rank %d of %d, slot %lu bytes)", r,
             b.rank, b.nranks, b.slot_bytes);
      for (int t = 0; t < r; ++t)
        if (memcmp(hb[t].uuid, b.uuid, 16) == 0) shared_gpu = true;
      if (r == c->rank) continue;
      if (b.pid == (long)getpid()) {
        // a rank of this process (one process driving several contexts): its window is a
        // plain device pointer here; on another GPU it needs peer access
        cudaPointerAttributes at;
        CUDA_OK(cudaPointerGetAttributes(&at, reinterpret_cast<void*>(b.window)));
        if (at.device != c->device) {
          cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); e = cudaSuccess; }
          CUDA_OK(e);
        }
        c->peer.view.win[r] = reinterpret_cast<unsigned char*>(b.window);
      } else {
        void* mp = nullptr;
        CUDA_OK(cudaIpcOpenMemHandle(&mp, b.ipc, cudaIpcMemLazyEnablePeerAccess));
        c->peer.mapped[r] = mp;
        c->peer.view.win[r] = static_cast<unsigned char*>(mp);
      }
    }
    // Ranks that share a GPU must never wait inside a kernel (nothing guarantees their
    // kernels run at the same time): the wait is then a stream memory operation.
    if (wait_mode == 2 && shared_gpu && P > 1)
      fail(BGS_E_CONFIG, "peer wait mode 2 (spin) needs every rank on its own GPU");
    c->peer.wait_mode = wait_mode ? wait_mode : (shared_gpu ? 1 : 2);
    c->peer.attached = true;
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

// Protocol self-test on ONE GPU without any cross-launch waiting (B200_PROFILING.md): P
// emulated ranks in this process; every epoch all ranks push (no waits), the device is
// synchronized, then every rank runs the SPIN flavour of the sum kernel -- its flags are
// already there -- and the sums must equal the rank-ordered host sum bitwise on all ranks.
int bgs_peer_selftest(int device, int nranks, long ng, long ns, int epochs, bgs_error* err) {
  clear_err(err);
  std::vector<bgs_ctx*> cs((size_t)std::max(nranks, 0), nullptr);
  int rc = BGS_OK;
  try {
    if (nranks < 1 || nranks > kPeerMaxRanks || ng < 0 || ns < 1 || epochs < 1)
      fail(BGS_E_CONFIG, "peer selftest: bad arguments");
    const size_t w = (size_t)(ng + ns);
    std::vector<PeerBlob> blobs((size_t)nranks);
    for (int r = 0; r < nranks; ++r) {
      bgs_error e2;
      if (bgs_ctx_create_peer(device, r, nranks, w * sizeof(double), &cs[r], &e2) != BGS_OK)
        fail(e2.code, "%s", e2.msg);
      if (bgs_ctx_peer_handle(cs[r], &blobs[r], &e2) != BGS_OK) fail(e2.code, "%s", e2.msg);
    }
    for (int r = 0; r < nranks; ++r) {
      bgs_error e2;
      // mode 1 passes the shared-GPU check; the sum kernels below still spin (on flags
      // that are already set)
      if (bgs_ctx_peer_attach(cs[r], blobs.data(), 1, &e2) != BGS_OK) fail(e2.code, "%s", e2.msg);
    }
    std::vector<DBuf> gin((size_t)nranks), sin((size_t)nranks), gout((size_t)nranks);
    std::vector<std::vector<double>> hg((size_t)nranks), hs((size_t)nranks);
    std::mt19937_64 gen(777);
    for (int ep = 1; ep <= epochs; ++ep) {
      for (int r = 0; r < nranks; ++r) {
        hg[r].resize((size_t)ng + 1);
        hs[r].resize((size_t)ns);
        for (auto& v : hg[r]) v = (double)(long)(gen() >> 11) * 0x1p-53 - 0.5;
        for (auto& v : hs[r]) v = ((double)(long)(gen() >> 11) * 0x1p-53 - 0.5) * (double)(1 << (gen() % 40));
        gin[r].ensure(((size_t)ng + 1) * 8);
        sin[r].ensure((size_t)ns * 8);
        gout[r].ensure(((size_t)ng * nranks + 1) * 8);
        CUDA_OK(cudaMemcpy(gin[r].p, hg[r].data(), (size_t)ng * 8, cudaMemcpyHostToDevice));
        CUDA_OK(cudaMemcpy(sin[r].p, hs[r].data(), (size_t)ns * 8, cudaMemcpyHostToDevice));
      }
      for (int r = 0; r < nranks; ++r) {
        bgs_ctx* c = cs[r];
        c->peer.epoch = (unsigned)ep;
        CUDA_OK(peer_push_launch(c->peer.view, gin[r].d(), (unsigned long)ng, sin[r].d(),
                                 (unsigned long)ns, (unsigned)ep, static_cast<unsigned*>(c->peer.cnt),
                                 c->stream, nullptr));
      }
      CUDA_OK(cudaDeviceSynchronize());  // every flag of this epoch is set: nothing below waits
      for (int r = 0; r < nranks; ++r)
        CUDA_OK(peer_sum_launch(cs[r]->peer.view, (unsigned long)ng, gout[r].d(), (unsigned long)ns,
                                sin[r].d(), (unsigned)ep, true, cs[r]->stream, nullptr));
      CUDA_OK(cudaDeviceSynchronize());
      std::vector<double> want((size_t)ns), got((size_t)ns), gg((size_t)ng * nranks + 1);
      for (long i = 0; i < ns; ++i) {
        double acc = hs[0][(size_t)i];
        for (int r = 1; r < nranks; ++r) acc += hs[r][(size_t)i];
        want[(size_t)i] = acc;
      }
      for (int r = 0; r < nranks; ++r) {
        CUDA_OK(cudaMemcpy(got.data(), sin[r].p, (size_t)ns * 8, cudaMemcpyDeviceToHost));
        if (memcmp(got.data(), want.data(), (size_t)ns * 8) != 0)
          fail(BGS_E_INTERNAL, "peer selftest: rank %d epoch %d: sum differs from the rank-ordered sum", r, ep);
        if (ng) {
          CUDA_OK(cudaMemcpy(gg.data(), gout[r].p, (size_t)ng * nranks * 8, cudaMemcpyDeviceToHost));
          for (int t = 0; t < nranks; ++t)
            if (memcmp(gg.data() + (size_t)t * ng, hg[t].data(), (size_t)ng * 8) != 0)
              fail(BGS_E_INTERNAL, "peer selftest: rank %d epoch %d: gathered part of rank %d differs", r, ep, t);
        }
      }
    }
  } catch (const Fail& f) {
    put_err(err, f);
    rc = f.code;
  }
  for (bgs_ctx* c : cs) bgs_ctx_destroy(c);
  return rc;
}

int bgs_ctx_set_stream(bgs_ctx* c, void* stream) {
  if (!c) return BGS_E_CUDA;
  c->caller = static_cast<cudaStream_t>(stream);
  return BGS_OK;
}

void bgs_ctx_destroy(bgs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  delete c;
}


int bgs_factor(bgs_ctx* c, int variant, long n, long m, long s, int procs, const double* x,
               long ldx, double* q, long ldq, double* r, long ldr, bgs_stats* stats,
               bgs_timing* timing, bgs_error* err) {
  return bgs_factor_opts(c, variant, n, m, s, procs, x, ldx, q, ldq, r, ldr, nullptr, stats,
                         timing, err);
}

int bgs_factor_opts(bgs_ctx* c, int variant, long n, long m, long s, int procs, const double* x,
                    long ldx, double* q, long ldq, double* r, long ldr, const bgs_options* opts,
                    bgs_stats* stats, bgs_timing* timing, bgs_error* err) {
  clear_err(err);
  if (stats) memset(stats, 0, sizeof *stats);
  if (timing) memset(timing, 0, sizeof *timing);
  const auto t0 = std::chrono::steady_clock::now();
  try {
    if (!c) fail(BGS_E_CUDA, "null context");
    validate(variant, n, m, s, procs);
    if (ldx < n || ldq < n || ldr < m) fail(BGS_E_DIMENSION, "leading dimension too small");
    if (c->nranks > 1) fail(BGS_E_CONFIG, "bgs_factor runs on a single-GPU context; use bgs_factor_device per rank");
    select_device(c);
    Runner run(c, variant, n, m, s, procs, false, stats, opts);
    // Stream X in and Q out on copy engines, overlapped with the factorization, when both
    // host buffers are pinned (pageable copies would block the enqueueing thread).
    auto pinned = [](const void* p) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return a.type == cudaMemoryTypeHost;
    };
    const char* nsio = getenv("BGS_NO_STREAM_IO");
    const bool stream_io = !(nsio && *nsio && *nsio != '0');
    // pageable caller buffers go through rings of pinned slots: a feeder thread copies X
    // chunks into them (host threads) ahead of the H2D copies, a drainer thread copies
    // finished Q chunks out of them (the driver's own staging of pageable memory runs at
    // a fraction of the copy engines' rate: 0.5-0.7 s vs 0.08 s at config 2)
    const bool mirror_x = stream_io && !pinned(x), mirror_q = stream_io && !pinned(q);
    c->sx.resize(std::max<size_t>(c->sx.size(), (size_t)procs));
    c->sq.resize(std::max<size_t>(c->sq.size(), (size_t)procs));
    for (int rk = 0; rk < procs; ++rk) {
      long r0, rows;
      bgs_shard_rows(n, procs, rk, &r0, &rows);
      Shard sh;
      sh.row0 = r0;
      sh.rows = rows;
      sh.ldx = sh.ldq = even_ld(rows);
      c->sx[rk].ensure((size_t)sh.ldx * m * sizeof(double) + 256);
      c->sq[rk].ensure((size_t)sh.ldq * m * sizeof(double) + 256);
      sh.X = c->sx[rk].d();
      sh.Q = c->sq[rk].d();
      if (rows > 0 && !stream_io)
        CUDA_OK(cudaMemcpy2DAsync(c->sx[rk].p, sh.ldx * sizeof(double), x + r0, ldx * sizeof(double),
                                  rows * sizeof(double), m, cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemsetAsync(c->sq[rk].p, 0, (size_t)sh.ldq * m * sizeof(double), c->stream));
      run.sh.push_back(sh);
    }
    Runner::XFeed feed;
    long q_done = 0;
    constexpr int kRing = 3;  // pinned slots per direction
    std::thread feeder, drainer;
    struct DrainItem {
      long c0, c1;
      int slot;
    };
    std::deque<DrainItem> dq;
    std::mutex dmu;
    std::condition_variable dcv;
    long q_pushed = 0, q_drained = 0;
    bool q_closed = false, drain_failed = false;
    cudaEvent_t qev[kRing] = {nullptr, nullptr, nullptr};
    size_t slot_doubles = 0, need = 0;
    int nch = 0;
    std::function<void(int, const double*, long)> enqueue_x;  // (outlives the setup block)
    // joins the helper threads on every exit path (errors included)
    struct Joiner {
      std::thread* t[2];
      std::mutex* mu;
      std::condition_variable* cv;
      bool* closed;
      ~Joiner() {
        {
          std::lock_guard<std::mutex> lk(*mu);
          *closed = true;
        }
        cv->notify_all();
        for (auto* x : t)
          if (x->joinable()) x->join();
      }
    } joiner{{&feeder, &drainer}, &dmu, &dcv, &q_closed};
    if (stream_io) {
      if (!c->h2d) CUDA_OK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
      if (!c->d2h) CUDA_OK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
      // chunks of whole blocks, ~16 columns (128 MB at n = 1e6)
      feed.chunk_cols = s * std::max<long>(1, 16 / s);
      nch = (int)((m + feed.chunk_cols - 1) / feed.chunk_cols);
      need = (size_t)nch + (size_t)(m / feed.chunk_cols) + 4;
      while (c->xfer_events.size() < need + kRing) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->xfer_events.push_back(e);
      }
      for (int k = 0; k < kRing; ++k) qev[k] = c->xfer_events[need + k];
      slot_doubles = (size_t)n * feed.chunk_cols;
      if (mirror_x) c->hx.ensure((size_t)kRing * slot_doubles * sizeof(double));
      if (mirror_q) c->hq.ensure((size_t)kRing * slot_doubles * sizeof(double));
      for (int ch = 0; ch < nch; ++ch) feed.ready.push_back(c->xfer_events[ch]);
      // H2D of chunk ch from host memory src (leading dimension lds, row 0 = global row 0)
      enqueue_x = [&](int ch, const double* src, long lds) {
        const long c0 = ch * feed.chunk_cols, nc = std::min(feed.chunk_cols, m - c0);
        for (const Shard& sh : run.sh)
          if (sh.rows > 0)
            CUDA_OK(cudaMemcpy2DAsync(const_cast<double*>(sh.X) + (size_t)c0 * sh.ldx,
                                      sh.ldx * sizeof(double), src + sh.row0, lds * sizeof(double),
                                      sh.rows * sizeof(double), nc, cudaMemcpyHostToDevice, c->h2d));
        CUDA_OK(cudaEventRecord(feed.ready[ch], c->h2d));
      };
      if (!mirror_x) {
        for (int ch = 0; ch < nch; ++ch) enqueue_x(ch, x + (size_t)ch * feed.chunk_cols * ldx, ldx);
      } else {
        feed.async_feed = true;
        feeder = std::thread([&] {
          try {
            cudaSetDevice(c->device);
            for (int ch = 0; ch < nch; ++ch) {
              const int k = ch % kRing;
              if (ch >= kRing) CUDA_OK(cudaEventSynchronize(feed.ready[ch - kRing]));  // slot free
              const long c0 = ch * feed.chunk_cols, nc = std::min(feed.chunk_cols, m - c0);
              double* slot = c->hx.d() + (size_t)k * slot_doubles;
              host_copy_cols(slot, n, x + (size_t)c0 * ldx, ldx, n, nc);
              enqueue_x(ch, slot, n);
              {
                std::lock_guard<std::mutex> lk(feed.mu);
                feed.recorded = ch + 1;
              }
              feed.cv.notify_all();
            }
          } catch (...) {
            std::lock_guard<std::mutex> lk(feed.mu);
            feed.failed = true;
            feed.cv.notify_all();
          }
        });
      }
      run.feed = &feed;
      if (mirror_q) {
        drainer = std::thread([&] {
          cudaSetDevice(c->device);
          for (;;) {
            DrainItem it;
            {
              std::unique_lock<std::mutex> lk(dmu);
              dcv.wait(lk, [&] { return !dq.empty() || q_closed; });
              if (dq.empty()) return;
              it = dq.front();
            }
            if (cudaEventSynchronize(qev[it.slot]) != cudaSuccess) {
              std::lock_guard<std::mutex> lk(dmu);
              drain_failed = true;
              dq.clear();
              dcv.notify_all();
              return;
            }
            host_copy_cols(q + (size_t)it.c0 * ldq, ldq, c->hq.d() + (size_t)it.slot * slot_doubles, n, n,
                           it.c1 - it.c0);
            {
              std::lock_guard<std::mutex> lk(dmu);
              dq.pop_front();
              ++q_drained;
            }
            dcv.notify_all();
          }
        });
      }
      size_t next_ev = (size_t)nch;
      run.on_q_final = [&, next_ev](long cend) mutable {
        if (cend <= q_done || (cend < m && cend - q_done < feed.chunk_cols)) return;
        cudaEvent_t e = c->xfer_events[next_ev];
        next_ev = next_ev + 1 < need ? next_ev + 1 : (size_t)nch;
        CUDA_OK(cudaEventRecord(e, c->stream));
        CUDA_OK(cudaStreamWaitEvent(c->d2h, e, 0));
        if (!mirror_q) {
          for (const Shard& sh : run.sh)
            if (sh.rows > 0)
              CUDA_OK(cudaMemcpy2DAsync(q + sh.row0 + (size_t)q_done * ldq, ldq * sizeof(double),
                                        sh.Q + (size_t)q_done * sh.ldq, sh.ldq * sizeof(double),
                                        sh.rows * sizeof(double), cend - q_done,
                                        cudaMemcpyDeviceToHost, c->d2h));
          q_done = cend;
          return;
        }
        // pieces of <= chunk_cols columns, one ring slot each
        while (q_done < cend) {
          const long c1 = std::min(cend, q_done + feed.chunk_cols);
          const int k = (int)(q_pushed % kRing);
          {
            std::unique_lock<std::mutex> lk(dmu);  // the slot's previous piece is drained
            dcv.wait(lk, [&] { return q_drained + kRing > q_pushed || drain_failed; });
            if (drain_failed) fail(BGS_E_CUDA, "draining Q to the pageable output failed");
          }
          double* slot = c->hq.d() + (size_t)k * slot_doubles;
          for (const Shard& sh : run.sh)
            if (sh.rows > 0)
              CUDA_OK(cudaMemcpy2DAsync(slot + sh.row0, n * sizeof(double),
                                        sh.Q + (size_t)q_done * sh.ldq, sh.ldq * sizeof(double),
                                        sh.rows * sizeof(double), c1 - q_done,
                                        cudaMemcpyDeviceToHost, c->d2h));
          CUDA_OK(cudaEventRecord(qev[k], c->d2h));
          {
            std::lock_guard<std::mutex> lk(dmu);
            dq.push_back({q_done, c1, k});
            ++q_pushed;
          }
          dcv.notify_all();
          q_done = c1;
        }
      };
    }
    c->launches = 0;
    CUDA_OK(cudaEventRecord(c->e0, c->stream));
    run.run();
    CUDA_OK(cudaEventRecord(c->e1, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    CUDA_OK(cudaGetLastError());
    c->prof_resolve();
    if (stream_io) CUDA_OK(cudaStreamSynchronize(c->d2h));
    if (feeder.joinable()) feeder.join();
    if (mirror_q) {
      std::unique_lock<std::mutex> lk(dmu);  // every piece copied out to the caller
      dcv.wait(lk, [&] { return q_drained == q_pushed || drain_failed; });
      if (drain_failed) fail(BGS_E_CUDA, "draining Q to the pageable output failed");
    }
    run.check_status();
    for (int rk = 0; rk < procs && !stream_io; ++rk) {
      const Shard& sh = run.sh[rk];
      if (sh.rows > 0)
        CUDA_OK(cudaMemcpy2DAsync(q + sh.row0, ldq * sizeof(double), sh.Q, sh.ldq * sizeof(double),
                                  sh.rows * sizeof(double), m, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_OK(cudaMemcpy2DAsync(r, ldr * sizeof(double), c->R.p, m * sizeof(double),
                              m * sizeof(double), m, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    if (timing) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->e0, c->e1);
      timing->factor_ms = ms;
      timing->kernel_launches = c->launches;
      timing->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return BGS_OK;
  } catch (const Fail& f) {
    if (c && c->h2d) cudaStreamSynchronize(c->h2d);
    if (c && c->d2h) cudaStreamSynchronize(c->d2h);
    if (c && c->stream) cudaStreamSynchronize(c->stream);
    put_err(err, f);
    return f.code;
  }
}

int bgs_factor_device(bgs_ctx* c, int variant, long n, long m, long s, long row0, long n_local,
                      const double* d_x, long ldx, double* d_q, long ldq, double* h_r, long ldr,
                      bgs_stats* stats, bgs_timing* timing, bgs_error* err) {
  return bgs_factor_device_opts(c, variant, n, m, s, row0, n_local, d_x, ldx, d_q, ldq, h_r, ldr,
                                nullptr, stats, timing, err);
}

int bgs_factor_device_opts(bgs_ctx* c, int variant, long n, long m, long s, long row0,
                           long n_local, const double* d_x, long ldx, double* d_q, long ldq,
                           double* h_r, long ldr, const bgs_options* opts, bgs_stats* stats,
                           bgs_timing* timing, bgs_error* err) {
  clear_err(err);
  if (stats) memset(stats, 0, sizeof *stats);
  if (timing) memset(timing, 0, sizeof *timing);
  const auto t0 = std::chrono::steady_clock::now();
  try {
    if (!c) fail(BGS_E_CUDA, "null context");
    validate(variant, n, m, s, c->nranks);
    long e0r, erows;
    bgs_shard_rows(n, c->nranks, c->rank, &e0r, &erows);
    if (row0 != e0r || n_local != erows)
      fail(BGS_E_DIMENSION, "rank %d must own rows [%ld, %ld) of the ceil split", c->rank, e0r,
           e0r + erows);
    if (ldx < n_local || ldq < n_local || ldr < m) fail(BGS_E_DIMENSION, "leading dimension too small");
    select_device(c);
    order_after_caller(c);
    Runner run(c, variant, n, m, s, c->nranks, c->collective(), stats, opts);
    Shard sh;
    sh.row0 = row0;
    sh.rows = n_local;
    sh.X = d_x;
    sh.ldx = ldx;
    sh.Q = d_q;
    sh.ldq = ldq;
    run.sh.push_back(sh);
    c->launches = 0;
    // The whole factorization is one CUDA graph on repeated calls (BGS_GRAPH=0: plain
    // launches).  Not with a host communicator (its exchanges synchronize), a probe, or
    // the profilers.
    const char* eg = getenv("BGS_GRAPH");
    const bool graphable = !(eg && *eg == '0') && !c->hc_fn && !c->peer.on && !(opts && opts->probe) &&
                           !c->prof_on && !run.tile_prof && !run.prof_step;
    std::string key;
    if (graphable) {
      char kb[512];
      snprintf(kb, sizeof kb, "%d %ld %ld %ld %ld %ld %p %ld %p %ld %d | %d %d %d %d %d %d %d %d",
               variant, n, m, s, row0, n_local, (const void*)d_x, ldx, (void*)d_q, ldq,
               opts ? opts->classic_intra : 0, run.no_fuse, run.no_k12c, run.gram_max_units,
               run.no_merge_small, run.no_pdl, run.comp_mode, run.no_k2m, run.tile_dbg);
      key = kb;
      for (const char* ev : {"BGS_K12C_PLAN", "BGS_K12C_MAXS", "BGS_K12C_MINS", "BGS_K12C_KWMAX", "BGS_UPDATE_MAXKP",
                             "BGS_TSQR_GENERIC", "BGS_K2_SCALAR"}) {
        const char* v = getenv(ev);
        key += std::string(" ") + (v ? v : "-");
      }
    }
    auto body = [&]() {
      // For s not a multiple of 4 the fused kernel's last k-step reads a few Q columns that
      // are not computed yet (zero coefficients): they must hold finite values.
      if (s % 4 && n_local > 0)
        CUDA_OK(cudaMemset2DAsync(d_q, ldq * sizeof(double), 0, n_local * sizeof(double), m,
                                  c->stream));
      run.run();
    };
    bgs_ctx::GraphEntry* ge = nullptr;
    if (graphable) {
      for (auto& g : c->graphs)
        if (g.key == key) ge = &g;
      if (ge && ge->bufs != c->buf_signature()) {  // a workspace moved: capture again
        cudaGraphExecDestroy(ge->exec);
        c->graphs.erase(c->graphs.begin() + (ge - c->graphs.data()));
        ge = nullptr;
      }
      if (!ge && std::find(c->seen.begin(), c->seen.end(), key) != c->seen.end()) {
        // second call with this signature: capture (every workspace is sized already)
        if (c->graphs.size() >= 8) {
          cudaGraphExecDestroy(c->graphs.front().exec);
          c->graphs.erase(c->graphs.begin());
        }
        c->graphs.emplace_back();
        bgs_ctx::GraphEntry& g = c->graphs.back();
        g.key = key;
        g.stats.reset(new bgs_stats());
        g.bounds.reset(new HBuf());
        // (pinned memory cannot be allocated while capturing: size it for the leaf plan
        // of setup(), at most ceil(rows / 256) leaves + 1 bounds)
        g.bounds->ensure(((size_t)(n_local + 255) / 256 + 4) * sizeof(long) + 64);
        run.stats = g.stats.get();
        run.bounds_sink = g.bounds.get();
        cudaGraph_t graph = nullptr;
        CUDA_OK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
          body();
        } catch (...) {
          cudaStreamEndCapture(c->stream, &graph);
          if (graph) cudaGraphDestroy(graph);
          c->graphs.pop_back();
          throw;
        }
        CUDA_OK(cudaStreamEndCapture(c->stream, &graph));
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) {
          c->graphs.pop_back();
          fail(BGS_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
        }
        g.launches = c->launches;
        g.bufs = c->buf_signature();
        ge = &g;
        run.stats = stats;
      }
    }
    CUDA_OK(cudaEventRecord(c->e0, c->stream));
    if (ge) {
      run.status = reinterpret_cast<DevStatus*>(c->status.p);  // (set by setup() otherwise)
      CUDA_OK(cudaGraphLaunch(ge->exec, c->stream));
      ge->uses += 1;
      if (stats) memcpy(stats, ge->stats.get(), sizeof *stats);
      c->launches = (int)ge->launches;
    } else {
      body();
      if (graphable && std::find(c->seen.begin(), c->seen.end(), key) == c->seen.end()) {
        if (c->seen.size() >= 64) c->seen.erase(c->seen.begin());
        c->seen.push_back(key);
      }
    }
    CUDA_OK(cudaEventRecord(c->e1, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    CUDA_OK(cudaGetLastError());
    c->prof_resolve();
    run.dump_phase_profile();
    run.check_status();
    if (h_r)
      CUDA_OK(cudaMemcpy2D(h_r, ldr * sizeof(double), c->R.p, m * sizeof(double), m * sizeof(double),
                           m, cudaMemcpyDeviceToHost));
    if (timing) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->e0, c->e1);
      timing->factor_ms = ms;
      timing->kernel_launches = c->launches;
      timing->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return BGS_OK;
  } catch (const Fail& f) {
    if (c && c->stream) cudaStreamSynchronize(c->stream);
    put_err(err, f);
    return f.code;
  }
}

int bgs_gen_gaussian_device(bgs_ctx* c, unsigned long long seed, long row0, long n_local, long m,
                            double* d_x, long ldx, bgs_error* err) {
  clear_err(err);
  try {
    select_device(c);
    order_after_caller(c);
    CUDA_OK(gen_gaussian_launch(seed, row0, n_local, m, d_x, ldx, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

// matrix_gen.cpp:18-56 (GaussianStream + gaussian_matrix): std::mt19937_64 is fully
// specified by the C++ standard, so the draw sequence matches the reference's bitwise
// on the same libm.
int bgs_gen_gaussian_host(unsigned long long seed, long n, long m, double* x, long ldx) {
  if (n < 0 || m < 0 || ldx < n) return BGS_E_DIMENSION;
  std::mt19937_64 g(seed);
  bool have = false;
  double spare = 0.0;
  auto unit = [&g]() { return static_cast<double>(g() >> 11) * 0x1.0p-53; };
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < n; ++i) {
      double v;
      if (have) {
        have = false;
        v = spare;
      } else {
        const double u1 = unit(), u2 = unit();
        const double radius = std::sqrt(-2.0 * std::log(1.0 - u1));
        const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = radius * std::sin(angle);
        have = true;
        v = radius * std::cos(angle);
      }
      x[i + (size_t)j * ldx] = v;
    }
  return BGS_OK;
}

int bgs_metrics_device(bgs_ctx* c, long n, long m, long n_local, const double* d_x, long ldx,
                       const double* d_q, long ldq, const double* h_r, long ldr, double* loo,
                       double* resid, bgs_error* err) {
  clear_err(err);
  try {
    select_device(c);
    order_after_caller(c);
    (void)n;
    const int si = 32;
    // Q^T Q in panels of 32 right columns through K1 (+ allreduce), assembled on the device
    Runner run(c, BGS_BCGSI_PLUS_P_1S, std::max(n, m), m, 1, c->nranks, c->collective(), nullptr);
    Shard sh;
    sh.rows = n_local;
    sh.X = d_x; sh.ldx = ldx;
    sh.Q = const_cast<double*>(d_q); sh.ldq = ldq;
    run.sh.push_back(sh);
    c->status.ensure(sizeof(DevStatus));
    run.status = reinterpret_cast<DevStatus*>(c->status.p);
    CUDA_OK(cudaMemsetAsync(run.status, 0, sizeof(DevStatus), c->stream));
    run.sh[0].make_maps(m);
    const size_t per_cta = gram_partial_doubles_per_cta((int)((m + 7) / 8) + 1, si);
    c->partial.ensure(per_cta * sizeof(double) * (size_t)run.grid_total() + 64);
    c->G.ensure((size_t)(m + 16) * 32 * sizeof(double) + 4096);
    DBuf dgram, dws;
    dgram.ensure((size_t)m * m * sizeof(double));
    dws.ensure((size_t)(3 * m + 8) * sizeof(double));
    for (long j0 = 0; j0 < m; j0 += si) {
      const int nb = (int)std::min<long>(si, m - j0);
      GramSpec g = Runner::spec1(SQ, 0, (int)m, (int)m);
      run.add_right(g, 0, (int)j0, nb);
      run.gram(g, "", false, true);
      CUDA_OK(cudaMemcpyAsync(dgram.d() + (size_t)j0 * m, c->G.p, (size_t)m * nb * sizeof(double),
                              cudaMemcpyDeviceToDevice, c->stream));
    }
    // two_norm(Q^T Q - I) (dense_kernels.cpp:205-239) by power iteration on the device:
    // O(m^2) per round instead of the O(m^3) host product it replaces (m = 4096 took minutes)
    double lnorm = 0.0;
    CUDA_OK(sym_two_norm(dgram.d(), (int)m, true, dws.d(), &lnorm, c->stream));
    if (loo) *loo = lnorm;

    // residual
    // per-CTA (d^2, x^2) double-double partials: <= 2*sms CTAs x 2 double2, then 2 results
    const size_t part_doubles = (size_t)2 * c->sms * 4;
    c->metrics.ensure((part_doubles + 8) * sizeof(double));
    double* out2 = c->metrics.d() + part_doubles;
    DBuf dr;
    dr.ensure((size_t)m * m * sizeof(double));
    CUDA_OK(cudaMemcpy2DAsync(dr.p, m * sizeof(double), h_r, ldr * sizeof(double), m * sizeof(double),
                              m, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(residual_launch(d_x, ldx, d_q, ldq, dr.d(), m, n_local, m, 1.0, 1.0, c->metrics.d(),
                            out2, c->sms, c->stream));
    if (c->collective()) run.allreduce(out2, 2);
    double h[2];
    CUDA_OK(cudaMemcpyAsync(h, out2, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    dr.release();
    if (resid) *resid = h[1] == 0.0 ? std::sqrt(h[0]) : std::sqrt(h[0]) / std::sqrt(h[1]);
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

int bgs_metrics(bgs_ctx* c, long n, long m, const double* x, long ldx, const double* q, long ldq,
                const double* r, long ldr, double* loo, double* resid, bgs_error* err) {
  clear_err(err);
  try {
    select_device(c);
    if (n < 1 || m < 1 || ldx < n || ldq < n || ldr < m) fail(BGS_E_DIMENSION, "bgs_metrics: shape");
    const long ld = even_ld(n);
    DBuf dx, dq;
    dx.ensure((size_t)ld * m * sizeof(double));
    dq.ensure((size_t)ld * m * sizeof(double));
    CUDA_OK(cudaMemcpy2DAsync(dx.p, ld * sizeof(double), x, ldx * sizeof(double), n * sizeof(double),
                              m, cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpy2DAsync(dq.p, ld * sizeof(double), q, ldq * sizeof(double), n * sizeof(double),
                              m, cudaMemcpyHostToDevice, c->stream));
    const int rc = bgs_metrics_device(c, n, m, n, dx.d(), ld, dq.d(), ld, r, ldr, loo, resid, err);
    dx.release();
    dq.release();
    return rc;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

int bgs_profile_enable(bgs_ctx* c, int on) {
  if (!c) return BGS_E_CUDA;
  c->prof_on = on != 0;
  return BGS_OK;
}

int bgs_profile_read(bgs_ctx* c, bgs_kernel_stat* out, int cap, int* count) {
  if (!c) return BGS_E_CUDA;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->prof_resolve();
  int n = 0;
  for (auto& p : c->prof) {
    if (n < cap && out) {
      memset(&out[n], 0, sizeof out[n]);
      snprintf(out[n].name, sizeof out[n].name, "%s", p.name.c_str());
      out[n].launches = p.launches;
      out[n].ms = p.ms;
      out[n].alg_bytes = p.bytes;
      out[n].alg_flops = p.flops;
    }
    ++n;
  }
  if (count) *count = n;
  c->prof.clear();
  return BGS_OK;
}

int bgs_gram(bgs_ctx* c, const double* a, long n, long ma, const double* b, long mb, double* out,
             bgs_error* err) {
  clear_err(err);
  try {
    select_device(c);
    if (n < 1 || ma < 1 || mb < 1 || mb > 32 || ma > 4096) fail(BGS_E_DIMENSION, "bgs_gram: shape");
    const long ld = even_ld(n);
    DBuf da, db;
    da.ensure((size_t)ld * ma * sizeof(double));
    db.ensure((size_t)ld * mb * sizeof(double));
    CUDA_OK(cudaMemcpy2DAsync(da.p, ld * sizeof(double), a, n * sizeof(double), n * sizeof(double), ma,
                              cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaMemcpy2DAsync(db.p, ld * sizeof(double), b, n * sizeof(double), n * sizeof(double), mb,
                              cudaMemcpyHostToDevice, c->stream));
    Runner run(c, BGS_BCGSI_PLUS_P_1S, n, std::max(ma, mb), 1, 1, false, nullptr);
    Shard sh;
    sh.rows = n;
    sh.Q = da.d(); sh.ldq = ld;
    sh.X = db.d(); sh.ldx = ld;
    run.sh.push_back(sh);
    for (int hi = 0; hi < 2; ++hi)
      for (int wi = 0; wi < 5; ++wi) {
        run.sh[0].mapQ[hi][wi] = make_map3(da.d(), n, ma, ld, 2 << hi, 128 >> wi);
        run.sh[0].mapX[hi][wi] = make_map3(db.d(), n, mb, ld, 2 << hi, 128 >> wi);
      }
    c->status.ensure(sizeof(DevStatus));
    run.status = reinterpret_cast<DevStatus*>(c->status.p);
    CUDA_OK(cudaMemsetAsync(run.status, 0, sizeof(DevStatus), c->stream));
    const size_t per_cta = gram_partial_doubles_per_cta((int)((ma + 7) / 8), (int)mb);
    c->partial.ensure(per_cta * sizeof(double) * (size_t)run.grid_total() + 64);
    c->G.ensure((size_t)ma * mb * sizeof(double) + 64);
    GramSpec g = Runner::spec2(SQ, 0, (int)ma, (int)ma, SX, 0, (int)mb, 0);
    run.add_right(g, 1, 0, (int)mb);
    run.gram(g, "", false, false);
    CUDA_OK(cudaMemcpyAsync(out, c->G.p, (size_t)ma * mb * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    run.check_status();
    da.release();
    db.release();
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

int bgs_tsqr(bgs_ctx* c, const double* x, long n, long s, double* q, double* r, bgs_error* err) {
  clear_err(err);
  try {
    select_device(c);
    if (s < 1 || s > 16) fail(BGS_E_CONFIG, "bgs_tsqr: 1 <= s <= 16");
    if (n < s) fail(BGS_E_RANK_DEFICIENT, "tsqr: block has %ld columns but only %ld global rows", s, n);
    const long ld = even_ld(n);
    DBuf dx, dq;
    dx.ensure((size_t)ld * s * sizeof(double));
    dq.ensure((size_t)ld * s * sizeof(double));
    CUDA_OK(cudaMemcpy2DAsync(dx.p, ld * sizeof(double), x, n * sizeof(double), n * sizeof(double), s,
                              cudaMemcpyHostToDevice, c->stream));
    Runner run(c, BGS_BCGSI_PLUS, n, s, s, 1, false, nullptr);
    Shard sh;
    sh.rows = n;
    sh.X = dx.d(); sh.ldx = ld;
    sh.Q = dq.d(); sh.ldq = ld;
    run.sh.push_back(sh);
    run.setup();
    run.tsqr(SX, 0, 0, c->rtop.d(), (int)s, "reduce_factor_tree:tsqr");
    CUDA_OK(cudaStreamSynchronize(c->stream));
    CUDA_OK(cudaGetLastError());
    run.check_status();  // rank-deficient leaves / non-finite input
    CUDA_OK(cudaMemcpy2D(q, n * sizeof(double), dq.p, ld * sizeof(double), n * sizeof(double), s,
                         cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(r, c->rtop.p, (size_t)s * s * sizeof(double), cudaMemcpyDeviceToHost));
    dx.release();
    dq.release();
    return BGS_OK;
  } catch (const Fail& f) {
    put_err(err, f);
    return f.code;
  }
}

}  // extern "C"
