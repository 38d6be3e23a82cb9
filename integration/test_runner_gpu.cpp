// test_runner_gpu.cpp — the reference's callers' view of the drop-in: the same inputs
// through the reference's run_factor (CPU, the unmodified library in oracle/_ref) and
// through blockgs::gpu::run_factor (runner_gpu.cpp -> libbgs_gpu.so), compared with the
// north_star tolerances: R to 1e-10 (normwise, and entrywise on |R_ij| >= 1e-3 max|R|),
// LOO / residual within 10x, SyncStats identical.  Also acceptance C8
// (acceptance.cpp:477-511) through the shim's BcgsOptions::probe, and the error contract.
// One JSON line per check; exit status 0 iff all pass.  Test infrastructure (tests/).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "blockgs/dense_kernels.hpp"
#include "blockgs/errors.hpp"
#include "blockgs/matrix_gen.hpp"
#include "blockgs/runner.hpp"
#include "blockgs/variant.hpp"
#include "runner_gpu.hpp"

using namespace blockgs;

namespace {

constexpr double kU = 1.1102230246251565e-16;
int g_fail = 0;

struct Case {
  VariantId v;
  long n, m, s;
  int procs;
  double kappa;
  bool gaussian;
};

DenseMatrix make(const Case& c, std::uint64_t seed) {
  MatrixSpec sp;
  sp.n = c.n;
  sp.m = c.m;
  sp.s = c.s;
  sp.kappa = c.kappa;
  sp.seed = seed;
  sp.distribution = c.gaussian ? MatrixDistribution::RandomGaussian
                               : MatrixDistribution::GeometricSingularValues;
  return gen_matrix(sp);
}

void compare(const Case& c, std::uint64_t seed) {
  const DenseMatrix x = make(c, seed);
  const FactorOutcome ref = run_factor(c.v, x, c.s, c.procs);
  const FactorOutcome gpu = gpu::run_factor(c.v, x, c.s, c.procs);
  bool pass = ref.ok && gpu.ok;
  double rn = NAN, re = NAN;
  if (pass) {
    const DenseMatrix& a = gpu.r.to_dense();
    const DenseMatrix& b = ref.r.to_dense();
    double mx = 0.0, dmax = 0.0;
    for (long j = 0; j < c.m; ++j)
      for (long i = 0; i < c.m; ++i) mx = std::fmax(mx, std::fabs(b(i, j)));
    re = 0.0;
    for (long j = 0; j < c.m; ++j)
      for (long i = 0; i < c.m; ++i) {
        const double d = std::fabs(a(i, j) - b(i, j));
        dmax = std::fmax(dmax, d);
        if (std::fabs(b(i, j)) >= 1e-3 * mx) re = std::fmax(re, d / std::fabs(b(i, j)));
        if (i > j && a(i, j) != 0.0) pass = false;  // exact-zero lower triangle
      }
    rn = dmax / mx;
    pass = pass && rn <= 1e-10 && re <= 1e-10;
    pass = pass && gpu.loo <= 10 * std::fmax(ref.loo, kU) && gpu.resid <= 10 * std::fmax(ref.resid, kU);
    pass = pass && gpu.stats.sync_count == ref.stats.sync_count &&
           gpu.stats.words_reduced == ref.stats.words_reduced &&
           gpu.stats.event_labels == ref.stats.event_labels &&
           gpu.stats.label_counts == ref.stats.label_counts;
  }
  if (!pass) ++g_fail;
  std::printf("{\"check\": \"factor\", \"variant\": \"%s\", \"n\": %ld, \"m\": %ld, \"s\": %ld, "
              "\"procs\": %d, \"kappa\": %g, \"gaussian\": %d, \"ref_ok\": %d, \"gpu_ok\": %d, "
              "\"r_norm\": %.3e, \"r_entry\": %.3e, \"loo\": %.3e, \"loo_ref\": %.3e, "
              "\"resid\": %.3e, \"resid_ref\": %.3e, \"syncs\": %ld, \"syncs_ref\": %ld, "
              "\"pass\": %s}\n",
              variant_name(c.v).c_str(), c.n, c.m, c.s, c.procs, c.kappa, c.gaussian ? 1 : 0,
              ref.ok ? 1 : 0, gpu.ok ? 1 : 0, rn, re, gpu.loo, ref.loo, gpu.resid, ref.resid,
              gpu.stats.sync_count, ref.stats.sync_count, pass ? "true" : "false");
}

// acceptance.cpp:477-511 through the GPU shim
void c8() {
  for (double kappa : {1e1, 1e3}) {
    Case c{VariantId::BcgsIp1s, 100, 16, 4, 1, kappa, false};
    const DenseMatrix x = make(c, 12345);
    double worst = 0.0;
    long fires = 0;
    RecurrenceProbe probe;
    probe.on_eval = [&](long, const DenseMatrix& s2, const DenseMatrix& q_blk,
                        const DenseMatrix& x_blk) {
      const DenseMatrix direct = gram(q_blk, x_blk);
      for (long j = 0; j < s2.cols(); ++j)
        for (long i = 0; i < s2.rows(); ++i)
          worst = std::fmax(worst, std::fabs(s2(i, j) - direct(i, j)));
      ++fires;
    };
    BcgsOptions opts;
    opts.probe = &probe;
    const FactorOutcome out = gpu::run_factor(VariantId::BcgsIp1s, x, 4, 1, opts);
    const bool pass = out.ok && fires == 2 && worst <= 1e-10;
    if (!pass) ++g_fail;
    std::printf("{\"check\": \"C8\", \"kappa\": %g, \"fires\": %ld, \"worst\": %.3e, \"pass\": %s}\n",
                kappa, fires, worst, pass ? "true" : "false");
  }
}

void errors() {
  // NotSpd far outside the working assumption: ok = false on both sides, same variant /
  // wording of the diagnostic (bcgs.cpp:69-80)
  {
    Case c{VariantId::BcgsIp1s, 400, 32, 4, 1, 1e15, false};
    const DenseMatrix x = make(c, 7);
    const FactorOutcome ref = run_factor(c.v, x, c.s, 1);
    const FactorOutcome gpu = gpu::run_factor(c.v, x, c.s, 1);
    const std::string head = "BCGSI+P-1S: ";
    const bool pass = !ref.ok && !gpu.ok && gpu.error.rfind(head, 0) == 0 &&
                      gpu.error.find("likely violated working assumption") != std::string::npos &&
                      gpu.not_spd_pivot >= 1;
    if (!pass) ++g_fail;
    std::printf("{\"check\": \"not_spd\", \"ref_ok\": %d, \"gpu_ok\": %d, \"pivot\": %d, "
                "\"pass\": %s}\n", ref.ok ? 1 : 0, gpu.ok ? 1 : 0, gpu.not_spd_pivot,
                pass ? "true" : "false");
  }
  // DimensionError: s does not divide m (bcgs.cpp:14-26 / distribute)
  {
    DenseMatrix x(50, 10);
    int got_ref = 0, got_gpu = 0;
    try {
      (void)run_factor(VariantId::BcgsIp1s, x, 4, 1);
    } catch (const DimensionError&) {
      got_ref = 1;
    }
    try {
      (void)gpu::run_factor(VariantId::BcgsIp1s, x, 4, 1);
    } catch (const DimensionError&) {
      got_gpu = 1;
    }
    const bool pass = got_ref && got_gpu;
    if (!pass) ++g_fail;
    std::printf("{\"check\": \"dimension_error\", \"ref\": %d, \"gpu\": %d, \"pass\": %s}\n",
                got_ref, got_gpu, pass ? "true" : "false");
  }
  // NonFiniteError on a NaN input
  {
    Case c{VariantId::BcgsIp1s, 200, 16, 4, 1, 1.0, true};
    DenseMatrix x = make(c, 3);
    x(5, 7) = NAN;
    int got_gpu = 0;
    try {
      (void)gpu::run_factor(VariantId::BcgsIp1s, x, 4, 1);
    } catch (const NonFiniteError&) {
      got_gpu = 1;
    }
    if (!got_gpu) ++g_fail;
    std::printf("{\"check\": \"non_finite\", \"gpu\": %d, \"pass\": %s}\n", got_gpu,
                got_gpu ? "true" : "false");
  }
}

}  // namespace

int main() {
  const std::vector<Case> cases = {
      {VariantId::BcgsIp1s, 100000, 64, 4, 1, 1.0, true},  // BASELINE config 1
      {VariantId::BcgsIp1s, 2000, 64, 4, 4, 1e4, false},
      {VariantId::BcgsIp2s, 2000, 64, 4, 3, 1e6, false},
      {VariantId::BcgsI1s, 2000, 48, 4, 1, 1e3, false},
      {VariantId::BcgsPipiPlus, 2000, 64, 8, 2, 1e4, false},
      {VariantId::BcgsIro, 2000, 64, 16, 1, 1e8, false},
      {VariantId::BcgsIp1s, 777, 36, 3, 5, 1e2, true},
  };
  std::uint64_t seed = 12345;
  for (const Case& c : cases) compare(c, seed++);
  c8();
  errors();
  std::printf("{\"summary\": true, \"failures\": %d}\n", g_fail);
  return g_fail ? 1 : 0;
}
