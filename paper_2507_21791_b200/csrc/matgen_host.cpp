// matgen_host.cpp — host-side port of the reference's test-matrix generator
// (gen_matrix, proj/src/matrix_gen.cpp:18-97), bit for bit: the mt19937_64 + Box-Muller
// Gaussian stream (:18-56), and the geometric family X = (U diag(sigma)) V^T with U, V the
// sign-fixed Householder Q factors (householder_qr, dense_kernels.cpp:135-203) of seeded
// Gaussian matrices and sigma_i = kappa^(-i/(m-1)) (:81-96).  Input generation for the
// driver (paper_2507_21791_b200/cli.py: `bench --config`, `factor`, `verify`) so a
// reference config produces the reference's exact X; not on the factorization path.
// Compiled by g++ without FMA contraction (x86-64 baseline, -ffp-contract=off): every
// operation rounds like the reference's -O3 build.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "bgs_gpu.h"

namespace {

struct Gauss {
  std::mt19937_64 g;
  bool have = false;
  double spare = 0.0;
  explicit Gauss(unsigned long long seed) : g(seed) {}
  double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double next() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = unit(), u2 = unit();
    const double radius = std::sqrt(-2.0 * std::log(1.0 - u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare = radius * std::sin(angle);
    have = true;
    return radius * std::cos(angle);
  }
};

// Column-major rows x cols.
struct Mat {
  long r = 0, c = 0;
  std::vector<double> a;
  Mat(long rr, long cc) : r(rr), c(cc), a((size_t)rr * cc, 0.0) {}
  double& operator()(long i, long j) { return a[(size_t)j * r + i]; }
};

// Explicit Q (rows x p) of the Householder QR with the reference's canonical sign
// (nonnegative R diagonal); same loops, same operation order.
Mat householder_q(Mat a) {
  const long m = a.r, n = a.c, p = std::min(m, n);
  std::vector<double> taus((size_t)p, 0.0);
  std::vector<std::vector<double>> vs((size_t)p);
  std::vector<double> rdiag((size_t)p, 0.0);
  for (long k = 0; k < p; ++k) {
    double mx = 0.0;
    for (long i = k; i < m; ++i) mx = std::max(mx, std::fabs(a(i, k)));
    if (mx == 0.0) continue;
    double ssq = 0.0;
    for (long i = k; i < m; ++i) {
      const double t = a(i, k) / mx;
      ssq += t * t;
    }
    const double sigma = mx * std::sqrt(ssq);
    const double alpha = a(k, k) >= 0.0 ? -sigma : sigma;
    std::vector<double> v((size_t)(m - k));
    v[0] = a(k, k) - alpha;
    for (long i = k + 1; i < m; ++i) v[(size_t)(i - k)] = a(i, k);
    double vtv = 0.0;
    for (double t : v) vtv += t * t;
    const double tau = vtv == 0.0 ? 0.0 : 2.0 / vtv;
    a(k, k) = alpha;
    for (long i = k + 1; i < m; ++i) a(i, k) = 0.0;
    for (long j = k + 1; j < n; ++j) {
      double w = 0.0;
      for (long i = k; i < m; ++i) w += v[(size_t)(i - k)] * a(i, j);
      w *= tau;
      for (long i = k; i < m; ++i) a(i, j) -= w * v[(size_t)(i - k)];
    }
    taus[(size_t)k] = tau;
    vs[(size_t)k] = std::move(v);
  }
  for (long k = 0; k < p; ++k) rdiag[(size_t)k] = a(k, k);
  Mat q(m, p);
  for (long i = 0; i < p; ++i) q(i, i) = 1.0;
  for (long k = p - 1; k >= 0; --k) {
    const std::vector<double>& v = vs[(size_t)k];
    const double tau = taus[(size_t)k];
    if (tau == 0.0) continue;
    for (long j = 0; j < p; ++j) {
      double w = 0.0;
      for (long i = k; i < m; ++i) w += v[(size_t)(i - k)] * q(i, j);
      w *= tau;
      for (long i = k; i < m; ++i) q(i, j) -= w * v[(size_t)(i - k)];
    }
  }
  for (long k = 0; k < p; ++k)
    if (rdiag[(size_t)k] < 0.0)
      for (long i = 0; i < m; ++i) q(i, k) = -q(i, k);
  return q;
}

Mat gaussian_matrix(long rows, long cols, Gauss& g) {
  Mat m(rows, cols);
  for (long j = 0; j < cols; ++j)
    for (long i = 0; i < rows; ++i) m(i, j) = g.next();
  return m;
}

void put(bgs_error* err, int code, const char* msg) {
  if (!err) return;
  std::memset(err, 0, sizeof *err);
  err->code = code;
  std::strncpy(err->msg, msg, sizeof err->msg - 1);
}

}  // namespace

extern "C" int bgs_gen_matrix_host(long n, long m, long s, double kappa, unsigned long long seed,
                                   int gaussian, double* x, long ldx, bgs_error* err) {
  // matrix_gen.cpp:60-79: the reference's argument checks and wording
  if (m < 1) return put(err, BGS_E_DIMENSION, "gen_matrix: column count must be at least 1"), BGS_E_DIMENSION;
  if (n < m)
    return put(err, BGS_E_DIMENSION, "gen_matrix: need n >= m for an economic test matrix"), BGS_E_DIMENSION;
  if (s < 1 || m % s != 0)
    return put(err, BGS_E_DIMENSION,
               "gen_matrix: column count must be a positive multiple of the block width"),
           BGS_E_DIMENSION;
  if (!(kappa >= 1.0)) return put(err, BGS_E_CONFIG, "gen_matrix: kappa must be at least 1"), BGS_E_CONFIG;
  if (ldx < n) return put(err, BGS_E_DIMENSION, "gen_matrix: ldx < n"), BGS_E_DIMENSION;
  Gauss g(seed);
  if (gaussian) {
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < n; ++i) x[(size_t)j * ldx + i] = g.next();
    return BGS_OK;
  }
  Mat u = householder_q(gaussian_matrix(n, m, g));
  Mat v = householder_q(gaussian_matrix(m, m, g));
  std::vector<double> sigma((size_t)m);
  for (long i = 0; i < m; ++i)
    sigma[(size_t)i] = m == 1 ? 1.0 : std::pow(kappa, -static_cast<double>(i) / static_cast<double>(m - 1));
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < n; ++i) u(i, j) *= sigma[(size_t)j];
  // multiply(u, v^T) (dense_matrix.cpp:107-122): out(i, j) = sum_k u(i, k) v(j, k)
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < n; ++i) {
      double acc = 0.0;
      for (long k = 0; k < m; ++k) acc += u(i, k) * v(j, k);
      x[(size_t)j * ldx + i] = acc;
    }
  return BGS_OK;
}
