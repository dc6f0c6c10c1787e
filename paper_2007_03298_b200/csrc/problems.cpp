// Host-side problem setup (see problems.hpp for the reference lines).
#include "problems.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>

namespace dssb {

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;  // the value of std::numbers::pi

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace

HostRng HostRng::for_stream(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t iteration) {
  uint64_t s = mix64(seed + 0x9e3779b97f4a7c15ULL);
  s = mix64(s ^ purpose);
  s = mix64(s ^ rank);
  s = mix64(s ^ iteration);
  return HostRng(s);
}

uint64_t HostRng::next_u64() {
  state_ += 0x9e3779b97f4a7c15ULL;
  return mix64(state_);
}

double HostRng::uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

uint64_t HostRng::uniform_below(uint64_t n) {
  if (n == 0) throw std::invalid_argument("uniform_below: n must be positive");
  const uint64_t limit = std::numeric_limits<uint64_t>::max() - std::numeric_limits<uint64_t>::max() % n;
  uint64_t v = next_u64();
  while (v >= limit) v = next_u64();
  return v % n;
}

double HostRng::gaussian() {
  const double u1 = 1.0 - uniform01();
  const double u2 = uniform01();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

namespace {

// seeded_unit_vector (problems.cpp:106-113)
std::vector<double> seeded_unit_vector(size_t d, HostRng& rng) {
  std::vector<double> u(d);
  for (double& v : u) v = rng.gaussian();
  double acc = 0.0;
  for (double v : u) acc += v * v;
  const double n = std::sqrt(acc);
  if (n < 1e-12) throw std::runtime_error("seeded_unit_vector: degenerate draw");
  for (double& v : u) v /= n;
  return u;
}

}  // namespace

void quadratic_problem(uint64_t seed, int d, double delta0, std::vector<double>& wstar, std::vector<double>& w0) {
  if (d < 1) throw std::invalid_argument("problem.d must be >= 1 (got " + std::to_string(d) + ")");
  if (delta0 <= 0.0) throw std::invalid_argument("problem.delta0 must be > 0");
  const size_t n = static_cast<size_t>(d);
  HostRng center = HostRng::for_stream(seed, kStreamDataGen, 1, 0);
  wstar.resize(n);
  for (double& v : wstar) v = center.gaussian();
  HostRng init = HostRng::for_stream(seed, kStreamInitParams, 0, 0);
  const std::vector<double> u = seeded_unit_vector(n, init);
  w0 = wstar;
  const double r = std::sqrt(delta0);
  for (size_t i = 0; i < n; ++i) w0[i] += r * u[i];
}

void logistic_dataset(uint64_t seed, int d, int M, std::vector<double>& x, std::vector<double>& y) {
  if (d < 1) throw std::invalid_argument("problem.d must be >= 1 (got " + std::to_string(d) + ")");
  if (M < 1) throw std::invalid_argument("logistic requires problem.M >= 1");
  const size_t n = static_cast<size_t>(d);
  HostRng rng = HostRng::for_stream(seed, kStreamDataGen, 0, 0);
  std::vector<double> w = seeded_unit_vector(n, rng);
  for (double& v : w) v *= 3.0;
  x.assign(static_cast<size_t>(M) * n, 0.0);
  y.assign(static_cast<size_t>(M), 1.0);
  for (int i = 0; i < M; ++i) {
    double margin = 0.0;
    for (size_t j = 0; j < n; ++j) {
      const double v = rng.gaussian();
      x[static_cast<size_t>(i) * n + j] = v;
      margin += v * w[j];
    }
    const double p = 1.0 / (1.0 + std::exp(-margin));
    y[static_cast<size_t>(i)] = rng.uniform01() < p ? 1.0 : -1.0;
  }
}

namespace {

// dense helpers (problems.cpp:18-65): sequential sums from 0.0
double dot_seq(const std::vector<double>& a, const std::vector<double>& b) {
  double acc = 0.0;
  for (size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
  return acc;
}

double norm_seq(const std::vector<double>& v) {
  double acc = 0.0;
  for (double x : v) acc += x * x;
  return std::sqrt(acc);
}

std::vector<double> matvec_seq(const std::vector<double>& a, const std::vector<double>& x) {
  const size_t d = x.size();
  std::vector<double> out(d, 0.0);
  for (size_t i = 0; i < d; ++i) {
    double acc = 0.0;
    for (size_t j = 0; j < d; ++j) acc += a[i * d + j] * x[j];
    out[i] = acc;
  }
  return out;
}

// Cholesky solve of an SPD system (problems.cpp:36-63)
std::vector<double> spd_solve(std::vector<double> a, std::vector<double> b) {
  const size_t d = b.size();
  for (size_t j = 0; j < d; ++j) {
    double diag = a[j * d + j];
    for (size_t k = 0; k < j; ++k) diag -= a[j * d + k] * a[j * d + k];
    if (diag <= 0.0) throw std::runtime_error("spd_solve: matrix not positive definite");
    const double root = std::sqrt(diag);
    a[j * d + j] = root;
    for (size_t i = j + 1; i < d; ++i) {
      double v = a[i * d + j];
      for (size_t k = 0; k < j; ++k) v -= a[i * d + k] * a[j * d + k];
      a[i * d + j] = v / root;
    }
  }
  for (size_t i = 0; i < d; ++i) {
    double v = b[i];
    for (size_t k = 0; k < i; ++k) v -= a[i * d + k] * b[k];
    b[i] = v / a[i * d + i];
  }
  for (size_t ii = d; ii > 0; --ii) {
    const size_t i = ii - 1;
    double v = b[i];
    for (size_t k = i + 1; k < d; ++k) v -= a[k * d + i] * b[k];
    b[i] = v / a[i * d + i];
  }
  return b;
}

// power iteration from the uniform start (problems.cpp:67-82)
double max_eigenvalue(const std::vector<double>& a, size_t d) {
  std::vector<double> v(d, 1.0 / std::sqrt(static_cast<double>(d)));
  double lambda = 0.0;
  for (int it = 0; it < 1000; ++it) {
    std::vector<double> av = matvec_seq(a, v);
    const double n = norm_seq(av);
    if (n == 0.0) return 0.0;
    for (size_t i = 0; i < d; ++i) av[i] /= n;
    const double next = dot_seq(av, matvec_seq(a, av));
    const bool converged = std::abs(next - lambda) <= 1e-13 * std::max(1.0, std::abs(next));
    lambda = next;
    v = std::move(av);
    if (converged && it > 2) break;
  }
  return lambda;
}

double sigmoid(double z) { return 1.0 / (1.0 + std::exp(-z)); }
double softplus(double z) { return z > 0.0 ? z + std::log1p(std::exp(-z)) : std::log1p(std::exp(z)); }

double logistic_full_loss(const double* x, const double* y, int M, size_t d, double l2, const std::vector<double>& w) {
  double acc = 0.0;
  for (int i = 0; i < M; ++i) {
    const double* xi = x + static_cast<size_t>(i) * d;
    double z = 0.0;
    for (size_t j = 0; j < d; ++j) z += xi[j] * w[j];
    acc += softplus(-y[i] * z);
  }
  acc /= static_cast<double>(M);
  if (l2 > 0.0) acc += 0.5 * l2 * dot_seq(w, w);
  return acc;
}

}  // namespace

LogisticConstants logistic_constants(const double* x, const double* y, int M, int d_in, double l2) {
  if (d_in < 1 || M < 1) throw std::invalid_argument("logistic: empty dataset");
  const size_t d = static_cast<size_t>(d_in);
  LogisticConstants out;
  std::vector<double> gram(d * d, 0.0);
  for (int i = 0; i < M; ++i) {
    const double* xi = x + static_cast<size_t>(i) * d;
    for (size_t a = 0; a < d; ++a) {
      for (size_t b = a; b < d; ++b) gram[a * d + b] += xi[a] * xi[b];
    }
  }
  for (size_t a = 0; a < d; ++a) {
    for (size_t b = 0; b < a; ++b) gram[a * d + b] = gram[b * d + a];
  }
  out.smoothness = max_eigenvalue(gram, d) / (4.0 * static_cast<double>(M)) + l2;
  if (!(l2 > 0.0)) return out;
  // damped Newton to |grad| <= 1e-12 (problems.cpp:372-413)
  std::vector<double> w(d, 0.0);
  for (int it = 0; it < 200; ++it) {
    std::vector<double> g(d, 0.0);
    std::vector<double> h(d * d, 0.0);
    for (int i = 0; i < M; ++i) {
      const double* xi = x + static_cast<size_t>(i) * d;
      const double yi = y[i];
      double z = 0.0;
      for (size_t j = 0; j < d; ++j) z += xi[j] * w[j];
      const double s = sigmoid(-yi * z);
      const double curv = s * (1.0 - s);
      for (size_t j = 0; j < d; ++j) {
        g[j] += -yi * s * xi[j];
        for (size_t k = j; k < d; ++k) h[j * d + k] += curv * xi[j] * xi[k];
      }
    }
    const double inv_m = 1.0 / static_cast<double>(M);
    for (size_t j = 0; j < d; ++j) {
      g[j] = g[j] * inv_m + l2 * w[j];
      for (size_t k = 0; k < j; ++k) h[j * d + k] = h[k * d + j];
      for (size_t k = j; k < d; ++k) h[j * d + k] *= inv_m;
      h[j * d + j] += l2;
    }
    if (norm_seq(g) <= 1e-12) {
      out.w_opt = w;
      out.f_star = logistic_full_loss(x, y, M, d, l2, w);
      return out;
    }
    const std::vector<double> dir = spd_solve(h, g);
    const double f0 = logistic_full_loss(x, y, M, d, l2, w);
    const double allowance = 64.0 * std::numeric_limits<double>::epsilon() * (1.0 + std::abs(f0));
    double step = 1.0;
    for (int half = 0; half < 60; ++half) {
      std::vector<double> trial = w;
      for (size_t j = 0; j < d; ++j) trial[j] -= step * dir[j];
      if (logistic_full_loss(x, y, M, d, l2, trial) <= f0 + allowance) {
        w = std::move(trial);
        break;
      }
      step *= 0.5;
    }
  }
  throw std::runtime_error("logistic optimum solve did not reach tolerance 1e-12");
}

void mlp_dataset(uint64_t seed, int d, int M, std::vector<double>& x, std::vector<double>& y) {
  if (d < 1) throw std::invalid_argument("problem.d must be >= 1 (got " + std::to_string(d) + ")");
  if (M < 1) throw std::invalid_argument("tiny-mlp requires problem.M >= 1");
  const size_t n = static_cast<size_t>(d);
  HostRng rng = HostRng::for_stream(seed, kStreamDataGen, 0, 0);
  std::vector<double> teacher = seeded_unit_vector(n, rng);
  for (double& v : teacher) v *= 2.0;
  x.assign(static_cast<size_t>(M) * n, 0.0);
  y.assign(static_cast<size_t>(M), 0.0);
  for (int i = 0; i < M; ++i) {
    double z = 0.0;
    for (size_t j = 0; j < n; ++j) {
      const double v = rng.gaussian();
      x[static_cast<size_t>(i) * n + j] = v;
      z += v * teacher[j];
    }
    y[static_cast<size_t>(i)] = std::sin(z);
  }
}

void mlp_initial_params(uint64_t seed, int d_in, int hidden, std::vector<double>& w) {
  if (hidden < 1 || hidden > 32) {
    throw std::invalid_argument("problem.hidden must be in [1, 32] (got " + std::to_string(hidden) + ")");
  }
  const size_t d = static_cast<size_t>(d_in);
  const size_t h = static_cast<size_t>(hidden);
  HostRng rng = HostRng::for_stream(seed, kStreamInitParams, 0, 0);
  w.assign(h * d + 2 * h + 1, 0.0);
  const double s1 = 1.0 / std::sqrt(static_cast<double>(d));
  for (size_t i = 0; i < h * d; ++i) w[i] = s1 * rng.gaussian();
  const double s2 = 1.0 / std::sqrt(static_cast<double>(h));
  for (size_t i = 0; i < h; ++i) w[h * d + h + i] = s2 * rng.gaussian();
}

void make_shards(int dataset_size, int workers, uint64_t seed, std::vector<int>& indices,
                 std::vector<int>& offsets) {
  if (workers < 1) throw std::invalid_argument("make_shards: workers must be >= 1");
  if (dataset_size < workers) {
    throw std::invalid_argument("make_shards: dataset smaller than worker count (" +
                                std::to_string(dataset_size) + " < " + std::to_string(workers) + ")");
  }
  std::vector<int> perm(static_cast<size_t>(dataset_size));
  for (int i = 0; i < dataset_size; ++i) perm[static_cast<size_t>(i)] = i;
  HostRng rng = HostRng::for_stream(seed, kStreamShard, 0, 0);
  for (size_t i = perm.size() - 1; i > 0; --i) {
    const size_t j = static_cast<size_t>(rng.uniform_below(i + 1));
    std::swap(perm[i], perm[j]);
  }
  // round-robin deal: worker w gets perm[w], perm[w + W], ... in that order
  offsets.assign(static_cast<size_t>(workers) + 1, 0);
  indices.resize(perm.size());
  for (int w = 0; w < workers; ++w) {
    const int cnt = dataset_size / workers + (w < dataset_size % workers ? 1 : 0);
    offsets[static_cast<size_t>(w) + 1] = offsets[static_cast<size_t>(w)] + cnt;
  }
  for (size_t i = 0; i < perm.size(); ++i) {
    const size_t w = i % static_cast<size_t>(workers);
    indices[static_cast<size_t>(offsets[w]) + i / static_cast<size_t>(workers)] = perm[i];
  }
}

void epoch_order(const int* shard, int size, uint64_t seed, int rank, long epoch, int* out) {
  for (int i = 0; i < size; ++i) out[i] = shard[i];
  if (size == 0) return;
  HostRng rng = HostRng::for_stream(seed, kStreamEpochOrder, static_cast<uint64_t>(rank),
                                    static_cast<uint64_t>(epoch));
  for (size_t i = static_cast<size_t>(size) - 1; i > 0; --i) {
    const size_t j = static_cast<size_t>(rng.uniform_below(i + 1));
    std::swap(out[i], out[j]);
  }
}

}  // namespace dssb
