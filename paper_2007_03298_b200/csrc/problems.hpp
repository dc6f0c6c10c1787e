// Host-side problem setup for the device gradient producers: the
// reference's SplitMix64 streams, the synthetic logistic dataset, the data
// shards and the per-epoch shard orders.
//
// These run once per run (setup), not per iteration, and are bit-exact
// restatements of the reference's host code.  They are compiled with the
// host compiler and the same libm as the reference, and FMA contraction is
// off:
//   Rng                /root/reference/proj/src/rng.cpp:9-51
//   quadratic w*, w0   /root/reference/proj/src/problems.cpp:157-165
//   logistic dataset   /root/reference/proj/src/problems.cpp:230-250
//   logistic L, f*     /root/reference/proj/src/problems.cpp:18-82,292-416
//   tiny-MLP data, w0  /root/reference/proj/src/problems.cpp:436-476
//   make_shards        /root/reference/proj/src/problems.cpp:642-662
//   epoch_order        /root/reference/proj/src/problems.cpp:664-674
#pragma once

#include <cstdint>
#include <vector>

namespace dssb {

// rng.hpp:42-47 stream purposes
constexpr uint64_t kStreamDataGen = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kStreamInitParams = 0xbf58476d1ce4e5b9ULL;
constexpr uint64_t kStreamShard = 0x94d049bb133111ebULL;
constexpr uint64_t kStreamBatch = 0xd6e8feb86659fd93ULL;
constexpr uint64_t kStreamGradientNoise = 0xa0761d6478bd642fULL;
constexpr uint64_t kStreamEpochOrder = 0xe7037ed1a0b428dbULL;

class HostRng {
 public:
  explicit HostRng(uint64_t state) : state_(state) {}
  static HostRng for_stream(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t iteration);
  uint64_t next_u64();
  double uniform01();
  uint64_t uniform_below(uint64_t n);
  double gaussian();

 private:
  uint64_t state_;
};

// Synthetic logistic data (problems.cpp:230-250): x is M x d row-major,
// y in {-1, +1}.
void logistic_dataset(uint64_t seed, int d, int M, std::vector<double>& x, std::vector<double>& y);

// TinyMlpProblem's data and start (problems.cpp:436-476): x is M x d
// gaussians, y = sin(x . teacher) with teacher = 2 * a seeded unit vector;
// params [W1 (hidden x d) | b1 | w2 | b2] with W1, w2 seeded gaussians
// scaled by 1/sqrt(d), 1/sqrt(hidden) and zero biases.
void mlp_dataset(uint64_t seed, int d, int M, std::vector<double>& x, std::vector<double>& y);
void mlp_initial_params(uint64_t seed, int d, int hidden, std::vector<double>& w);

// LogisticProblem::finish_setup (problems.cpp:346-416): the smoothness
// bound (power iteration on X^T X / 4M, + l2) and, for l2 > 0, the optimum
// by damped Newton (w_opt, f* = full_loss(w_opt)).  Setup-time host code.
struct LogisticConstants {
  double smoothness = 0.0;
  double f_star = 0.0;
  std::vector<double> w_opt;
};
LogisticConstants logistic_constants(const double* x, const double* y, int M, int d, double l2);

// Isotropic quadratic (A = mu*I) optimum and start (problems.cpp:157-165):
// w* = gaussians of (seed, kDataGen, 1, 0); w0 = w* + sqrt(delta0) * u, u the
// normalised gaussians of (seed, kInitParams, 0, 0).
void quadratic_problem(uint64_t seed, int d, double delta0, std::vector<double>& wstar, std::vector<double>& w0);

// CSR shards: worker w owns indices[offsets[w] .. offsets[w+1]).
void make_shards(int dataset_size, int workers, uint64_t seed, std::vector<int>& indices,
                 std::vector<int>& offsets);

void epoch_order(const int* shard, int size, uint64_t seed, int rank, long epoch, int* out);

}  // namespace dssb
