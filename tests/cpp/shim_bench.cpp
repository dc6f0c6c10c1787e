// Timing of the drop-in path: the reference's own run_training
// (sync.cpp:284-463, DS-Sync branch :347-374) on an isotropic quadratic,
// linked two ways by oracle/Makefile:
//
//   _ref/shim_bench        the unmodified reference objects
//   _ref/shim_bench_b200   the same objects with apply_step / sync_round /
//                          make_partition / ring,tree,ps_allreduce_avg served
//                          by the B200 library (tests/cpp/b200_shim.cpp)
//
// Both binaries run the same Problem, options and seeds, so their final
// params must be bit-identical; the wall times are the drop-in's own cost
// (host<->device copies on every call) against the reference's CPU path.
//
// The reference's QuadraticProblem stores a dense d x d matrix (F10 in
// infeasible at d = 1M); this Problem is the same objective with
// A = mu * I written elementwise -- w*, w0 and the gradient noise drawn from
// the reference's Rng streams exactly as problems.cpp:157-193 draws them.
//
//   shim_bench <d> <iterations> <W> <N> <lockstep|parallel> <params_out.bin>
// prints one JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dssync/optim.hpp"
#include "dssync/problems.hpp"
#include "dssync/rng.hpp"
#include "dssync/sync.hpp"

using namespace dssync;

namespace {

class IsoQuadratic final : public Problem {
 public:
  IsoQuadratic(int d, double mu, double sigma, double delta0, uint64_t seed) {
    spec_.kind = "quadratic";
    spec_.d = d;
    spec_.mu = spec_.L = mu;
    spec_.sigma = sigma;
    spec_.delta0 = delta0;
    spec_.seed = seed;
    Rng center = Rng::for_stream(seed, streams::kDataGen, 1, 0);
    w_star_.resize(static_cast<size_t>(d));
    for (double& x : w_star_) x = center.gaussian();
    Rng init = Rng::for_stream(seed, streams::kInitParams, 0, 0);
    ParamVector u(static_cast<size_t>(d));
    for (double& x : u) x = init.gaussian();
    const double n = norm(u);
    w0_ = w_star_;
    const double r = std::sqrt(delta0);
    for (size_t i = 0; i < u.size(); ++i) w0_[i] += r * (u[i] / n);
  }
  const DatasetSpec& spec() const override { return spec_; }
  int dim() const override { return spec_.d; }
  int dataset_size() const override { return 0; }
  ParamVector initial_params() const override { return w0_; }
  GradSample stochastic_gradient(const ParamVector& w, std::span<const int>, Rng& rng) const override {
    GradSample out;
    out.grad.resize(w.size());
    const double scale = spec_.sigma / std::sqrt(static_cast<double>(w.size()));
    double loss = 0.0;
    for (size_t i = 0; i < w.size(); ++i) {
      const double diff = w[i] - w_star_[i];
      double g = spec_.mu * diff;
      loss += diff * g;
      if (spec_.sigma > 0.0) g += scale * rng.gaussian();
      out.grad[i] = g;
    }
    out.loss = 0.5 * loss;
    return out;
  }
  double full_loss(const ParamVector& w) const override {
    double acc = 0.0;
    for (size_t i = 0; i < w.size(); ++i) {
      const double diff = w[i] - w_star_[i];
      acc += diff * (spec_.mu * diff);
    }
    return 0.5 * acc;
  }
  ParamVector full_gradient(const ParamVector& w) const override {
    ParamVector g(w.size());
    for (size_t i = 0; i < w.size(); ++i) g[i] = spec_.mu * (w[i] - w_star_[i]);
    return g;
  }
  bool has_optimum() const override { return true; }
  const ParamVector& optimum() const override { return w_star_; }
  double true_suboptimality(const ParamVector& w) const override { return full_loss(w); }
  double smoothness() const override { return spec_.L; }
  double strong_convexity() const override { return spec_.mu; }

 private:
  DatasetSpec spec_;
  ParamVector w_star_, w0_;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: shim_bench d iterations W N lockstep|parallel params_out.bin\n");
    return 2;
  }
  const int d = std::atoi(argv[1]);
  const long T = std::atol(argv[2]);
  const int W = std::atoi(argv[3]);
  const int N = std::atoi(argv[4]);
  const bool parallel = std::strcmp(argv[5], "parallel") == 0;
  IsoQuadratic problem(d, 1.0, 0.5, 4.0, 7);
  SyncStrategy s;
  s.kind = StrategyKind::DsSync;
  s.topology = Topology::Ring;
  s.world = {W, N};
  RunOptions o;
  o.iterations = T;
  o.seed = 1;
  o.optimizer.kind = OptimizerKind::SgdMomentum;
  o.optimizer.hp.weight_decay = 1e-4;
  o.lr = constant_lr(0.05);
  o.mode = parallel ? ExecutionMode::Parallel : ExecutionMode::Lockstep;
  const auto t0 = std::chrono::steady_clock::now();
  const RunResult r = run_training(problem, s, o);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (FILE* f = std::fopen(argv[6], "wb")) {
    for (const WorkerState& ws : r.final_workers) std::fwrite(ws.params.data(), sizeof(double), ws.params.size(), f);
    std::fclose(f);
  }
  std::printf("{\"d\": %d, \"iterations\": %ld, \"W\": %d, \"N\": %d, \"mode\": \"%s\", \"seconds\": %.4f, "
              "\"ms_per_iteration\": %.3f, \"final_suboptimality\": %.17g}\n",
              d, T, W, N, parallel ? "parallel" : "lockstep", sec, 1e3 * sec / static_cast<double>(T),
              r.traces.back().suboptimality);
  return 0;
}
