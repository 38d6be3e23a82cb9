// runner_gpu.cpp — blockgs::gpu::run_factor over the C ABI (see runner_gpu.hpp).
#include "runner_gpu.hpp"

#include <memory>
#include <mutex>
#include <sstream>
#include <string>

#include "bgs_gpu.h"
#include "blockgs/errors.hpp"
#include "blockgs/metrics.hpp"

namespace blockgs::gpu {

namespace {

// One context per process (device 0), created on first use: the C ABI call is blocking
// and not concurrent on one context (bgs_gpu.h), so calls are serialized here.
struct Ctx {
  bgs_ctx* c = nullptr;
  std::mutex mu;
  Ctx() {
    bgs_error e{};
    if (bgs_ctx_create(0, 0, 1, nullptr, &c, &e) != BGS_OK) {
      c = nullptr;
      err = e.msg;
    }
  }
  ~Ctx() { bgs_ctx_destroy(c); }
  std::string err;
};

Ctx& ctx() {
  static Ctx g;
  return g;
}

[[noreturn]] void rethrow(int rc, const bgs_error& e) {
  const std::string msg = e.msg;
  switch (rc) {
    case BGS_E_DIMENSION: throw DimensionError(msg);
    case BGS_E_SINGULAR: throw SingularError(msg, e.pivot);
    case BGS_E_RANK_DEFICIENT: throw RankDeficientError(msg);
    case BGS_E_NON_FINITE: throw NonFiniteError(msg);
    case BGS_E_COLLECTIVE: throw CollectiveError(msg);
    case BGS_E_CONFIG: throw ConfigError(msg);
    default: throw Error("bgs_factor: " + msg);
  }
}

// RecurrenceProbe::on_eval trampoline: host copies -> DenseMatrix views
struct ProbeCtx {
  const RecurrenceProbe* probe;
};

void probe_tramp(void* user, long k, const double* s2, long s, const double* q_local,
                 const double* x_local, long n_local, int /*shard*/) {
  const auto* p = static_cast<const ProbeCtx*>(user);
  DenseMatrix S2(s, s), Ql(n_local, s), Xl(n_local, s);
  for (long j = 0; j < s; ++j) {
    for (long i = 0; i < s; ++i) S2(i, j) = s2[i + j * s];
    for (long i = 0; i < n_local; ++i) {
      Ql(i, j) = q_local[i + j * n_local];
      Xl(i, j) = x_local[i + j * n_local];
    }
  }
  p->probe->on_eval(k, S2, Ql, Xl);
}

}  // namespace

FactorOutcome run_factor(VariantId v, const DenseMatrix& x, long s, int procs,
                         const BcgsOptions& opts) {
  Ctx& g = ctx();
  if (!g.c) throw Error("no usable B200 (the GPU path has no CPU fallback): " + g.err);
  std::lock_guard<std::mutex> lock(g.mu);
  const long n = x.rows(), m = x.cols();
  FactorOutcome out;
  DenseMatrix q(n, m), r(m, m);
  auto st = std::make_unique<bgs_stats>();
  bgs_timing tm{};
  bgs_error err{};
  ProbeCtx pc{opts.probe};
  bgs_options o{};
  o.classic_intra = static_cast<int>(opts.classic_intra);
  if (opts.probe && opts.probe->on_eval) {
    o.probe = probe_tramp;
    o.probe_user = &pc;
  }
  const int rc = bgs_factor_opts(g.c, static_cast<int>(v), n, m, s, procs, x.data().data(),
                                 n > 0 ? n : 1, q.data().data(), n > 0 ? n : 1,
                                 r.data().data(), m > 0 ? m : 1, &o, st.get(), &tm, &err);
  if (rc == BGS_E_NOT_SPD) {  // runner.cpp:56-61
    out.ok = false;
    out.error = err.msg;
    out.not_spd_pivot = err.pivot;
    return out;
  }
  if (rc != BGS_OK) rethrow(rc, err);
  out.ok = true;
  out.q = std::move(q);
  out.r = UpperTriangular::from_dense(r, s);  // strict lower triangle is exact zero
  // SyncStats: counts and words from the GPU run, labels one per event in issue order
  out.stats.sync_count = st->sync_count;
  out.stats.words_reduced = st->words_reduced;
  std::istringstream labels(st->labels);
  for (std::string l; std::getline(labels, l);)
    if (!l.empty()) {
      out.stats.event_labels.push_back(l);
      ++out.stats.label_counts[l];
    }
  out.loo = loss_of_orthogonality(out.q);  // metrics.cpp:8-14
  ResidualResult res = residual(x, out.q, out.r.to_dense());
  out.resid = res.value;
  out.x_was_zero = res.x_was_zero;
  return out;
}

}  // namespace blockgs::gpu
