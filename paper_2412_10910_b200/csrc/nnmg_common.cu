// Error state, launch counter and the host-side 1D tables.
#include "nnmg_common.cuh"

#include <atomic>
#include <algorithm>
#include <cmath>

namespace nnmg {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }
void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }
uint64_t launch_count() { return g_launches.load(); }

namespace {

// Legendre P_n and P_n' at x (long double recurrence)
void legendre(int n, long double x, long double& p, long double& dp) {
  long double p0 = 1.0L, p1 = x;
  if (n == 0) {
    p = 1.0L;
    dp = 0.0L;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    long double pk = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = pk;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0L);
}

// Gauss-Legendre nodes/weights on [-1,1], ascending (numpy leggauss order)
void gauss_legendre(int n, std::vector<long double>& x, std::vector<long double>& w) {
  x.resize(n);
  w.resize(n);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < n; ++i) {
    long double z = std::cos(pi * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 100; ++it) {
      long double p, dp;
      legendre(n, z, p, dp);
      long double dz = p / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-30L) break;
    }
    long double p, dp;
    legendre(n, z, p, dp);
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
}

// Gauss-Lobatto nodes on [-1,1]: endpoints and roots of P'_{n-1}
std::vector<long double> gauss_lobatto(int n) {
  std::vector<long double> x(n);
  x[0] = -1.0L;
  x[n - 1] = 1.0L;
  const int N = n - 1;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 1; i < N; ++i) {
    long double z = -std::cos(pi * i / N);
    for (int it = 0; it < 100; ++it) {
      long double p, dp;
      legendre(N, z, p, dp);
      // (1-z^2) P'' = 2 z P' - N(N+1) P
      long double d2p = (2.0L * z * dp - N * (N + 1) * p) / (1.0L - z * z);
      long double dz = dp / d2p;
      z -= dz;
      if (std::fabs(dz) < 1e-30L) break;
    }
    x[i] = z;
  }
  return x;
}

}  // namespace

Tables make_tables(int degree) {
  NNMG_REQUIRE(degree >= 1 && degree <= kMaxDegree, kUnsupported,
               "polynomial degree must be in [1, " + std::to_string(kMaxDegree) + "]");
  Tables t{};
  const int n1 = degree + 1;
  t.n1 = n1;
  std::vector<long double> gx, gw;
  gauss_legendre(n1, gx, gw);
  std::vector<long double> lob = gauss_lobatto(n1);
  std::vector<long double> q(n1), nd(n1), den(n1);
  for (int i = 0; i < n1; ++i) {
    q[i] = 0.5L * (gx[i] + 1.0L);
    nd[i] = 0.5L * (lob[i] + 1.0L);
    t.xq[i] = static_cast<double>(q[i]);
    t.w[i] = static_cast<double>(0.5L * gw[i]);
  }
  nd[0] = 0.0L;
  nd[n1 - 1] = 1.0L;
  for (int i = 0; i < n1; ++i) {
    t.nodes[i] = static_cast<double>(nd[i]);
    long double d = 1.0L;
    for (int j = 0; j < n1; ++j)
      if (j != i) d *= (nd[i] - nd[j]);
    den[i] = d;
    t.denom[i] = static_cast<double>(d);
    t.rdenom[i] = static_cast<double>(1.0L / d);
  }
  for (int a = 0; a < n1; ++a) {
    for (int i = 0; i < n1; ++i) {
      long double v = 1.0L;
      for (int j = 0; j < n1; ++j)
        if (j != i) v *= (q[a] - nd[j]);
      t.S[a][i] = static_cast<double>(v / den[i]);
      long double dv = 0.0L;
      for (int k = 0; k < n1; ++k) {
        if (k == i) continue;
        long double term = 1.0L;
        for (int j = 0; j < n1; ++j)
          if (j != i && j != k) term *= (q[a] - nd[j]);
        dv += term;
      }
      t.D[a][i] = static_cast<double>(dv / den[i]);
      // Lagrange polynomials through the Gauss points, derivative at x_a
      long double gden = 1.0L;
      for (int j = 0; j < n1; ++j)
        if (j != i) gden *= (q[i] - q[j]);
      long double gd = 0.0L;
      for (int k = 0; k < n1; ++k) {
        if (k == i) continue;
        long double term = 1.0L;
        for (int j = 0; j < n1; ++j)
          if (j != i && j != k) term *= (q[a] - q[j]);
        gd += term;
      }
      t.Dc[a][i] = static_cast<double>(gd / gden);
    }
  }
  for (int a = 0; a < kMaxN1; ++a)
    for (int i = 0; i < kMaxN1; ++i) {
      t.S32[a][i] = static_cast<float>(t.S[a][i]);
      t.Dc32[a][i] = static_cast<float>(t.Dc[a][i]);
    }
  for (int i = 0; i < kMaxN1; ++i) {
    t.nodes32[i] = static_cast<float>(t.nodes[i]);
    t.rdenom32[i] = static_cast<float>(t.rdenom[i]);
  }
  return t;
}

}  // namespace nnmg
