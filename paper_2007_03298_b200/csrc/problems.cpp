// Host-side problem setup (see problems.hpp for the reference lines).
#include "problems.hpp"

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

void logistic_dataset(uint64_t seed, int d, int M, std::vector<double>& x, std::vector<double>& y) {
  if (d < 1) throw std::invalid_argument("problem.d must be >= 1 (got " + std::to_string(d) + ")");
  if (M < 1) throw std::invalid_argument("logistic requires problem.M >= 1");
  const size_t n = static_cast<size_t>(d);
  HostRng rng = HostRng::for_stream(seed, kStreamDataGen, 0, 0);
  // seeded_unit_vector (problems.cpp:106-113), scaled by 3
  std::vector<double> w(n);
  for (double& v : w) v = rng.gaussian();
  double acc = 0.0;
  for (double v : w) acc += v * v;
  const double nrm = std::sqrt(acc);
  if (nrm < 1e-12) throw std::runtime_error("seeded_unit_vector: degenerate draw");
  for (double& v : w) v /= nrm;
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
