// Test infrastructure only (oracle/_ref): a thin extern "C" shim over the UNMODIFIED
// reference library compiled from /root/reference/proj/src by oracle/Makefile.
// It lets pytest (ctypes) and bench.py's reference arm call the reference's own
// gen_matrix (proj/src/matrix_gen.cpp:60-97), run_variant under run_spmd
// (proj/include/blockgs/communicator.hpp:281-330, proj/src/bcgs.cpp:414-431) and the
// exact metrics (proj/src/metrics.cpp:8-28).  Nothing here is shipped or measured as
// the product.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "blockgs/bcgs.hpp"
#include "blockgs/communicator.hpp"
#include "blockgs/cost_model.hpp"
#include "blockgs/dense_kernels.hpp"
#include "blockgs/dist_block.hpp"
#include "blockgs/errors.hpp"
#include "blockgs/matrix_gen.hpp"
#include "blockgs/metrics.hpp"
#include "blockgs/runner.hpp"
#include "blockgs/variant.hpp"

using namespace blockgs;

namespace {
void set_msg(char* buf, long cap, const std::string& s) {
  if (!buf || cap <= 0) return;
  std::strncpy(buf, s.c_str(), static_cast<size_t>(cap - 1));
  buf[cap - 1] = 0;
}
// Error codes shared with include/bgs_gpu.h (BGS_E_*).
int code_of(const std::exception& e) {
  if (dynamic_cast<const NotSpdError*>(&e)) return 2;
  if (dynamic_cast<const DimensionError*>(&e)) return 1;
  if (dynamic_cast<const SingularError*>(&e)) return 3;
  if (dynamic_cast<const RankDeficientError*>(&e)) return 4;
  if (dynamic_cast<const NonFiniteError*>(&e)) return 5;
  if (dynamic_cast<const CollectiveError*>(&e)) return 6;
  if (dynamic_cast<const ConfigError*>(&e)) return 7;
  return 8;
}
}  // namespace

extern "C" {

// X (n x m, col-major, ld = n) = gen_matrix({n, m, s, kappa, seed, dist}); dist 0 = geometric, 1 = gaussian.
int ref_gen_matrix(long n, long m, long s, double kappa, unsigned long long seed, int dist,
                   double* x, char* msg, long msgcap) {
  try {
    MatrixSpec spec;
    spec.n = n; spec.m = m; spec.s = s; spec.kappa = kappa; spec.seed = seed;
    spec.distribution = dist == 1 ? MatrixDistribution::RandomGaussian
                                  : MatrixDistribution::GeometricSingularValues;
    DenseMatrix g = gen_matrix(spec);
    std::memcpy(x, g.data().data(), sizeof(double) * static_cast<size_t>(n * m));
    return 0;
  } catch (const std::exception& e) {
    set_msg(msg, msgcap, e.what());
    return code_of(e);
  }
}

// Runs run_variant on `procs` simulated ranks (threads) and gathers Q.  Returns 0 on
// success, an error code otherwise (NotSpd: 2, pivot in *pivot).  Timing covers
// distribute + run_variant only (stats and gather excluded), as SURVEY.md §8(d).
// labels: '\n'-joined event labels (factorization phase).  Metrics optional.
// BcgsOptions::classic_intra for the following ref_factor calls (0 Tsqr, 1 CholQr).
static int g_classic_intra = 0;
void ref_set_classic_intra(int kind) { g_classic_intra = kind; }

int ref_factor(int variant, const double* xin, long n, long m, long s, int procs,
               int want_metrics, double* q, double* r, long* sync_count, long* words,
               char* labels, long labcap, double* loo, double* resid, double* seconds,
               int* pivot, char* msg, long msgcap) {
  try {
    DenseMatrix x(n, m);
    std::memcpy(x.data().data(), xin, sizeof(double) * static_cast<size_t>(n * m));
    VariantId v = all_variants().at(static_cast<size_t>(variant));
    struct View { DenseMatrix q; UpperTriangular r; SyncStats st; double secs; };
    auto [views, st] = run_spmd(procs, [&](Communicator& comm) {
      auto t0 = std::chrono::steady_clock::now();
      DistBlockMatrix xd = distribute(x, s, comm);
      BcgsOptions opts;
      opts.classic_intra = g_classic_intra ? IntraorthKind::CholQr : IntraorthKind::Tsqr;
      BcgsResult res = run_variant(v, xd, comm, opts);
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      DenseMatrix qf = gather(res.q);
      return View{std::move(qf), std::move(res.r), std::move(res.stats), secs};
    });
    (void)st;
    double worst = 0;
    for (auto& vw : views) worst = std::max(worst, vw.secs);
    if (seconds) *seconds = worst;
    const View& v0 = views[0];
    if (q) std::memcpy(q, v0.q.data().data(), sizeof(double) * static_cast<size_t>(n * m));
    if (r) std::memcpy(r, v0.r.to_dense().data().data(), sizeof(double) * static_cast<size_t>(m * m));
    if (sync_count) *sync_count = v0.st.sync_count;
    if (words) *words = v0.st.words_reduced;
    std::string lab;
    for (size_t i = 0; i < v0.st.event_labels.size(); ++i) {
      if (i) lab += "\n";
      lab += v0.st.event_labels[i];
    }
    set_msg(labels, labcap, lab);
    if (want_metrics) {
      if (loo) *loo = loss_of_orthogonality(v0.q);
      if (resid) *resid = residual(x, v0.q, v0.r.to_dense()).value;
    }
    return 0;
  } catch (const NotSpdError& e) {
    if (pivot) *pivot = e.pivot;
    set_msg(msg, msgcap, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_msg(msg, msgcap, e.what());
    return code_of(e);
  }
}

double ref_loo(const double* qin, long n, long m) {
  DenseMatrix q(n, m);
  std::memcpy(q.data().data(), qin, sizeof(double) * static_cast<size_t>(n * m));
  return loss_of_orthogonality(q);
}

double ref_residual(const double* xin, const double* qin, const double* rin, long n, long m) {
  DenseMatrix x(n, m), q(n, m), r(m, m);
  std::memcpy(x.data().data(), xin, sizeof(double) * static_cast<size_t>(n * m));
  std::memcpy(q.data().data(), qin, sizeof(double) * static_cast<size_t>(n * m));
  std::memcpy(r.data().data(), rin, sizeof(double) * static_cast<size_t>(m * m));
  return residual(x, q, r).value;
}

// a^T b with exact accumulation, rounded once (dense_kernels.cpp:29-34).
void ref_gram(const double* a, long n, long ma, const double* b, long mb, double* out) {
  DenseMatrix A(n, ma), B(n, mb);
  std::memcpy(A.data().data(), a, sizeof(double) * static_cast<size_t>(n * ma));
  std::memcpy(B.data().data(), b, sizeof(double) * static_cast<size_t>(n * mb));
  DenseMatrix g = gram(A, B);
  std::memcpy(out, g.data().data(), sizeof(double) * static_cast<size_t>(ma * mb));
}

// householder_qr (dense_kernels.cpp:135-203): q (rows x p), r (p x cols), p = min(rows, cols).
void ref_householder(const double* xin, long rows, long cols, double* q, double* r) {
  DenseMatrix x(rows, cols);
  std::memcpy(x.data().data(), xin, sizeof(double) * static_cast<size_t>(rows * cols));
  QrResult qr = householder_qr(x);
  std::memcpy(q, qr.q.data().data(), sizeof(double) * static_cast<size_t>(qr.q.size()));
  std::memcpy(r, qr.r.data().data(), sizeof(double) * static_cast<size_t>(qr.r.size()));
}

double ref_variant_flops(int variant, long n, long m, long s) {
  return variant_flops(all_variants().at(static_cast<size_t>(variant)), n, m, s);
}

long ref_expected_syncs(int variant, long q) {
  return expected_syncs(all_variants().at(static_cast<size_t>(variant)), q);
}

}  // extern "C"
