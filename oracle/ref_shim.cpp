// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdssync_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (to pin the oracle and generate
// golden fixtures) and by bench.py's reference arm / cpu_baseline leg.  It
// contains no reference code, only calls into the reference's public API
// (namespace dssync): make_partition, group_of, check_mixing, validate,
// apply_step, sync_round, run_training, ring/tree/ps_allreduce_avg,
// make_problem, make_shards, Rng.
#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dssync/comm.hpp"
#include "dssync/config.hpp"
#include "dssync/errors.hpp"
#include "dssync/metrics.hpp"
#include "dssync/optim.hpp"
#include "dssync/param.hpp"
#include "dssync/problems.hpp"
#include "dssync/rng.hpp"
#include "dssync/schedule.hpp"
#include "dssync/sync.hpp"

using namespace dssync;

namespace {

void put(char* buf, int len, const std::string& s) {
  if (buf && len > 0) {
    std::strncpy(buf, s.c_str(), static_cast<size_t>(len) - 1);
    buf[len - 1] = 0;
  }
}

// 0 ok, 1 invalid_argument, 2 DivergenceError, 3 runtime_error, 4 ConfigError
template <typename F>
int guarded(char* err, int errlen, int* rank, long* it, F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    put(err, errlen, e.what());
    return 4;
  } catch (const DivergenceError& e) {
    if (rank) *rank = e.rank;
    if (it) *it = e.iteration;
    put(err, errlen, e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    put(err, errlen, e.what());
    return 1;
  } catch (const std::exception& e) {
    put(err, errlen, e.what());
    return 3;
  }
}

OptimizerState make_opt(int kind, const double* hp, double alpha) {
  OptimizerState s;
  s.kind = static_cast<OptimizerKind>(kind);
  s.hp.alpha = alpha;
  s.hp.momentum = hp[0];
  s.hp.beta1 = hp[1];
  s.hp.beta2 = hp[2];
  s.hp.epsilon = hp[3];
  s.hp.weight_decay = hp[4];
  return s;
}

SyncStrategy make_strategy(int kind, int topo, int W, int N, int servers) {
  SyncStrategy s;
  s.kind = static_cast<StrategyKind>(kind);
  s.topology = static_cast<Topology>(topo);
  s.world = {W, N};
  s.num_servers = servers;
  return s;
}

// WorkerState rows <-> flat [W][d] arrays.  Moments are materialised (the
// reference allocates zeros lazily on the first step, optim.cpp:63,73-74,
// which is numerically identical to starting from explicit zeros).
std::vector<WorkerState> load_workers(int W, long d, int opt, const double* hp, const long* steps,
                                      const double* w, const double* m1, const double* m2) {
  std::vector<WorkerState> ws(static_cast<size_t>(W));
  for (int k = 0; k < W; ++k) {
    WorkerState& x = ws[static_cast<size_t>(k)];
    x.rank = k;
    x.params.assign(w + static_cast<long>(k) * d, w + static_cast<long>(k + 1) * d);
    x.opt = make_opt(opt, hp, 0.0);
    if (steps) x.opt.step_count = steps[k];
    if (m1 && opt != 0) x.opt.first_moment.assign(m1 + static_cast<long>(k) * d, m1 + static_cast<long>(k + 1) * d);
    if (m2 && opt >= 2) x.opt.second_moment.assign(m2 + static_cast<long>(k) * d, m2 + static_cast<long>(k + 1) * d);
  }
  return ws;
}

void store_workers(const std::vector<WorkerState>& ws, long d, long* steps, double* w, double* m1, double* m2) {
  for (size_t k = 0; k < ws.size(); ++k) {
    std::memcpy(w + static_cast<long>(k) * d, ws[k].params.data(), sizeof(double) * static_cast<size_t>(d));
    if (steps) steps[k] = ws[k].opt.step_count;
    if (m1 && !ws[k].opt.first_moment.empty()) {
      std::memcpy(m1 + static_cast<long>(k) * d, ws[k].opt.first_moment.data(), sizeof(double) * static_cast<size_t>(d));
    }
    if (m2 && !ws[k].opt.second_moment.empty()) {
      std::memcpy(m2 + static_cast<long>(k) * d, ws[k].opt.second_moment.data(), sizeof(double) * static_cast<size_t>(d));
    }
  }
}

AllReduceResult collective(int topo, int servers, const std::vector<int>& members,
                           const std::vector<ParamVector>& inputs) {
  switch (topo) {
    case 1: return tree_allreduce_avg(members, inputs);
    case 2: return ps_allreduce_avg(members, inputs, servers);
    default: return ring_allreduce_avg(members, inputs);
  }
}

// local_iteration's optimizer part (sync.cpp:244-266): alpha into the
// state, apply_step, wrap runtime failures as DivergenceError(rank, t).
void local_step(WorkerState& ws, const ParamVector& grad, double alpha, long t) {
  ws.opt.hp.alpha = alpha;
  try {
    StepResult r = apply_step(ws.opt, ws.params, grad);
    ws.params = std::move(r.params);
    ws.opt = std::move(r.state);
  } catch (const DivergenceError&) {
    throw;
  } catch (const std::runtime_error& e) {
    throw DivergenceError(ws.rank, t, e.what());
  }
}

template <typename F>
void parallel_for(size_t n, int threads, F&& fn) {
  // run_training's Parallel mode fan-out (sync.cpp:103-129): lowest index wins.
  if (threads <= 1 || n <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  const size_t th = std::min<size_t>(static_cast<size_t>(threads), n);
  std::vector<std::exception_ptr> errs(n);
  std::vector<std::thread> pool;
  for (size_t j = 0; j < th; ++j) {
    pool.emplace_back([&, j] {
      for (size_t i = j; i < n; i += th) {
        try {
          fn(i);
        } catch (...) {
          errs[i] = std::current_exception();
        }
      }
    });
  }
  for (auto& t : pool) t.join();
  for (auto& e : errs) {
    if (e) std::rethrow_exception(e);
  }
}

}  // namespace

extern "C" {

int ref_validate_world(int W, int N, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] { validate(WorldConfig{W, N}); });
}

int ref_validate_strategy(int kind, int topo, int W, int N, int servers, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] { validate(make_strategy(kind, topo, W, N, servers)); });
}

int ref_is_square_mode(int W, int N) { return is_square_mode(WorldConfig{W, N}) ? 1 : 0; }

int ref_make_partition(int W, int N, long t, int* members, int* offsets, int* n_groups, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    const GroupPartition p = make_partition(WorldConfig{W, N}, t);
    int pos = 0;
    offsets[0] = 0;
    for (size_t g = 0; g < p.groups.size(); ++g) {
      for (int x : p.groups[g]) members[pos++] = x;
      offsets[g + 1] = pos;
    }
    *n_groups = static_cast<int>(p.groups.size());
  });
}

int ref_group_of(int W, int N, long t, int rank, int* members, int* count, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    const std::vector<int> g = group_of(WorldConfig{W, N}, t, rank);
    for (size_t i = 0; i < g.size(); ++i) members[i] = g[i];
    *count = static_cast<int>(g.size());
  });
}

int ref_check_mixing(int W, int N, long t) {
  try {
    return check_mixing(WorldConfig{W, N}, t) ? 1 : 0;
  } catch (...) {
    return -1;
  }
}

// Collective over explicit inputs; values[0] written to out, counts returned.
int ref_allreduce(int topo, int servers, int m, long d, const double* inputs, double* out, long* steps,
                  long* msgs, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    std::vector<int> members(static_cast<size_t>(m));
    std::vector<ParamVector> in(static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) {
      members[static_cast<size_t>(k)] = k;
      in[static_cast<size_t>(k)].assign(inputs + static_cast<long>(k) * d, inputs + static_cast<long>(k + 1) * d);
    }
    const AllReduceResult r = collective(topo, servers, members, in);
    for (int k = 0; k < m; ++k) {
      if (r.values[static_cast<size_t>(k)] != r.values[0]) throw std::runtime_error("members disagree");
    }
    std::memcpy(out, r.values[0].data(), sizeof(double) * static_cast<size_t>(d));
    *steps = r.steps.serial_steps;
    *msgs = r.steps.total_messages;
  });
}

int ref_mean_of(int m, long d, const double* inputs, double* out, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    std::vector<ParamVector> in(static_cast<size_t>(m));
    for (int k = 0; k < m; ++k) in[static_cast<size_t>(k)].assign(inputs + static_cast<long>(k) * d, inputs + static_cast<long>(k + 1) * d);
    const ParamVector r = mean_of(in);
    std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(d));
  });
}

// apply_step (optim.cpp:46-98) on one row; moments in/out (zeros = fresh).
int ref_apply_step(int opt, const double* hp, double alpha, long* step_count, long d, double* w,
                   const double* g, double* m1, double* m2, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    OptimizerState s = make_opt(opt, hp, alpha);
    s.step_count = *step_count;
    if (opt != 0 && m1) s.first_moment.assign(m1, m1 + d);
    if (opt >= 2 && m2) s.second_moment.assign(m2, m2 + d);
    const StepResult r = apply_step(s, ParamVector(w, w + d), ParamVector(g, g + d));
    std::memcpy(w, r.params.data(), sizeof(double) * static_cast<size_t>(d));
    if (m1 && !r.state.first_moment.empty()) std::memcpy(m1, r.state.first_moment.data(), sizeof(double) * static_cast<size_t>(d));
    if (m2 && !r.state.second_moment.empty()) std::memcpy(m2, r.state.second_moment.data(), sizeof(double) * static_cast<size_t>(d));
    *step_count = r.state.step_count;
  });
}

// sync_round (sync.cpp:268-282) on [W][d] params.
int ref_sync_round(int kind, int topo, int W, int N, int servers, long t, long d, double* w, long* steps,
                   long* msgs, int* err_rank, long* err_it, char* err, int errlen) {
  return guarded(err, errlen, err_rank, err_it, [&] {
    std::vector<WorkerState> ws = load_workers(W, d, 0, std::vector<double>(5, 0.0).data(), nullptr, w, nullptr, nullptr);
    const SyncRoundOutcome o = sync_round(ws, make_strategy(kind, topo, W, N, servers), t);
    store_workers(ws, d, nullptr, w, nullptr, nullptr);
    *steps = o.critical_path_steps;
    *msgs = o.total_messages;
  });
}

// One DS-Sync iteration with explicit gradients: every worker's local step
// (sync.cpp:348-362) then sync_round (sync.cpp:364-373).
int ref_ds_iteration(int topo, int W, int N, long d, long t, int opt, const double* hp, double alpha,
                     long* steps, double* w, const double* g, double* m1, double* m2, int* err_rank,
                     long* err_it, char* err, int errlen) {
  return guarded(err, errlen, err_rank, err_it, [&] {
    std::vector<WorkerState> ws = load_workers(W, d, opt, hp, steps, w, m1, m2);
    for (int k = 0; k < W; ++k) {
      local_step(ws[static_cast<size_t>(k)], ParamVector(g + static_cast<long>(k) * d, g + static_cast<long>(k + 1) * d), alpha, t);
    }
    sync_round(ws, make_strategy(1, topo, W, N, 1), t);
    store_workers(ws, d, steps, w, m1, m2);
  });
}

// One BSP iteration with explicit gradients (sync.cpp:375-428): collective
// over all gradients, then every worker steps with the mean.
int ref_bsp_iteration(int topo, int servers, int W, long d, long t, int opt, const double* hp, double alpha,
                      long* steps, double* w, const double* g, double* m1, double* m2, int* err_rank,
                      long* err_it, char* err, int errlen) {
  return guarded(err, errlen, err_rank, err_it, [&] {
    std::vector<WorkerState> ws = load_workers(W, d, opt, hp, steps, w, m1, m2);
    std::vector<int> members(static_cast<size_t>(W));
    std::vector<ParamVector> in(static_cast<size_t>(W));
    for (int k = 0; k < W; ++k) {
      members[static_cast<size_t>(k)] = k;
      in[static_cast<size_t>(k)].assign(g + static_cast<long>(k) * d, g + static_cast<long>(k + 1) * d);
    }
    AllReduceResult r;
    try {
      r = collective(topo, servers, members, in);
    } catch (const std::runtime_error& e) {
      throw DivergenceError(0, t, e.what());
    }
    for (int k = 0; k < W; ++k) local_step(ws[static_cast<size_t>(k)], r.values[static_cast<size_t>(k)], alpha, t);
    store_workers(ws, d, steps, w, m1, m2);
  });
}

// format_double (metrics.cpp:13-17) of n values, '\n'-joined into buf.
int ref_format_doubles(const double* v, long n, char* buf, long len) {
  std::string out;
  for (long i = 0; i < n; ++i) {
    out += format_double(v[i]);
    out += '\n';
  }
  if (static_cast<long>(out.size()) + 1 > len) return 1;
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return 0;
}

// Gaussians of stream (seed, purpose, rank, it) (rng.cpp:20-51).
void ref_gaussians(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t it, long n, double* out) {
  Rng r = Rng::for_stream(seed, purpose, rank, it);
  for (long i = 0; i < n; ++i) out[i] = r.gaussian();
}

uint64_t ref_next_u64(uint64_t* state) {
  Rng r(*state);
  const uint64_t v = r.next_u64();
  *state += 0x9e3779b97f4a7c15ULL;
  return v;
}

// Quadratic problem (L == mu: A = mu*I) optimum and start point.
int ref_quadratic_init(uint64_t seed, int d, double mu, double delta0, double* wstar, double* w0, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "quadratic";
    s.d = d;
    s.mu = mu;
    s.L = mu;
    s.sigma = 0.0;
    s.delta0 = delta0;
    s.seed = seed;
    auto p = make_problem(s);
    std::memcpy(wstar, p->optimum().data(), sizeof(double) * static_cast<size_t>(d));
    const ParamVector x = p->initial_params();
    std::memcpy(w0, x.data(), sizeof(double) * static_cast<size_t>(d));
  });
}

// Full trajectory of run_training on the isotropic quadratic, replayed
// through the public API so every per-iteration gradient is recorded:
//   grads_out  [T][W][d]  the stochastic gradient each worker used at t
//   params_out [T][W][d]  every worker's params after iteration t
// The replay is then checked against run_training itself (same options):
// *matches = 1 iff final params agree bit for bit.  When trace_* are given,
// run_training's IterationTrace (sync.hpp:63-74) is recorded per t:
//   trace_gmean [T][d], trace_loss [T][W], trace_scalars [T][5] =
//   {mean_post_sync_loss, suboptimality, critical_path_steps,
//    total_messages, simulated_comm_time}.
int ref_quadratic_run(int kind, int topo, int W, int N, int d, double mu, double sigma, double delta0,
                      uint64_t problem_seed, uint64_t run_seed, int T, int opt, const double* hp,
                      double alpha, double* grads_out, double* params_out, int* matches, char* err,
                      int errlen, double* trace_gmean, double* trace_loss, double* trace_scalars,
                      char* csv_out, long csv_len) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "quadratic";
    s.d = d;
    s.mu = mu;
    s.L = mu;
    s.sigma = sigma;
    s.delta0 = delta0;
    s.seed = problem_seed;
    auto problem = make_problem(s);
    const SyncStrategy strat = make_strategy(kind, topo, W, N, 1);
    RunOptions o;
    o.iterations = T;
    o.seed = run_seed;
    o.optimizer = make_opt(opt, hp, alpha);
    o.lr = constant_lr(alpha);

    std::vector<WorkerState> ws(static_cast<size_t>(W));
    for (int k = 0; k < W; ++k) {
      ws[static_cast<size_t>(k)].rank = k;
      ws[static_cast<size_t>(k)].params = problem->initial_params();
      ws[static_cast<size_t>(k)].opt = o.optimizer;
    }
    for (int t = 0; t < T; ++t) {
      std::vector<ParamVector> grads(static_cast<size_t>(W));
      for (int k = 0; k < W; ++k) {
        Rng noise = Rng::for_stream(run_seed, streams::kGradientNoise, static_cast<uint64_t>(k), static_cast<uint64_t>(t));
        grads[static_cast<size_t>(k)] = problem->stochastic_gradient(ws[static_cast<size_t>(k)].params, {}, noise).grad;
        std::memcpy(grads_out + (static_cast<long>(t) * W + k) * d, grads[static_cast<size_t>(k)].data(), sizeof(double) * static_cast<size_t>(d));
      }
      if (kind == 1) {
        for (int k = 0; k < W; ++k) local_step(ws[static_cast<size_t>(k)], grads[static_cast<size_t>(k)], alpha, t);
        sync_round(ws, strat, t);
      } else {
        std::vector<int> members(static_cast<size_t>(W));
        for (int k = 0; k < W; ++k) members[static_cast<size_t>(k)] = k;
        const AllReduceResult r = collective(topo, 1, members, grads);
        for (int k = 0; k < W; ++k) local_step(ws[static_cast<size_t>(k)], r.values[static_cast<size_t>(k)], alpha, t);
      }
      for (int k = 0; k < W; ++k) {
        std::memcpy(params_out + (static_cast<long>(t) * W + k) * d, ws[static_cast<size_t>(k)].params.data(), sizeof(double) * static_cast<size_t>(d));
      }
    }
    const RunResult rr = run_training(*problem, strat, o);
    *matches = 1;
    for (int k = 0; k < W; ++k) {
      if (rr.final_workers[static_cast<size_t>(k)].params != ws[static_cast<size_t>(k)].params) *matches = 0;
    }
    if (trace_gmean) {
      for (int t = 0; t < T; ++t) {
        const IterationTrace& tr = rr.traces[static_cast<size_t>(t)];
        std::memcpy(trace_gmean + static_cast<long>(t) * d, tr.global_mean_params.data(), sizeof(double) * static_cast<size_t>(d));
        for (int k = 0; k < W; ++k) trace_loss[static_cast<long>(t) * W + k] = tr.post_sync_loss[static_cast<size_t>(k)];
        double* sc = trace_scalars + static_cast<long>(t) * 5;
        sc[0] = tr.mean_post_sync_loss;
        sc[1] = tr.suboptimality;
        sc[2] = static_cast<double>(tr.critical_path_steps);
        sc[3] = static_cast<double>(tr.total_messages);
        sc[4] = tr.simulated_comm_time;
      }
    }
    if (csv_out) {  // the reference's own metrics file for this run (metrics.cpp:37-56)
      const std::string csv = metrics_csv(rr.traces);
      if (static_cast<long>(csv.size()) + 1 > csv_len) throw std::runtime_error("csv buffer too small");
      std::memcpy(csv_out, csv.c_str(), csv.size() + 1);
    }
  });
}

// C1 (acceptance.cpp:239-258): logistic d=20 M=2000 seed 11, batch 8,
// replacement sampling, DS W=4 N=2 (or BSP), step_decay_lr(1.0, 0.5, 75).
// Replays run_training's batches (sample_batch, sync.cpp:153-166) and
// gradients through the public API, recording them, and checks the replay
// against run_training.
int ref_logistic_run(int kind, int W, int N, int d, int M, double l2, uint64_t problem_seed,
                     uint64_t run_seed, int batch, int T, int opt, const double* hp, double alpha0,
                     double factor, long every, int sampling, double* grads_out, double* params_out,
                     double* alphas_out, int* batches_out, int* matches, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "logistic";
    s.d = d;
    s.M = M;
    s.mu = l2;
    s.seed = problem_seed;
    auto problem = make_problem(s);
    const SyncStrategy strat = make_strategy(kind, 0, W, N, 1);
    RunOptions o;
    o.iterations = T;
    o.seed = run_seed;
    o.batch_size = batch;
    o.optimizer = make_opt(opt, hp, alpha0);
    o.lr = step_decay_lr(alpha0, factor, every);
    o.sampling = sampling ? SamplingMode::Epoch : SamplingMode::Replacement;
    const std::vector<Shard> shards = make_shards(problem->dataset_size(), W, run_seed);
    std::vector<WorkerState> ws(static_cast<size_t>(W));
    for (int k = 0; k < W; ++k) {
      ws[static_cast<size_t>(k)].rank = k;
      ws[static_cast<size_t>(k)].params = problem->initial_params();
      ws[static_cast<size_t>(k)].opt = o.optimizer;
      ws[static_cast<size_t>(k)].shard = shards[static_cast<size_t>(k)];
    }
    for (int t = 0; t < T; ++t) {
      const double alpha = o.lr.alpha(t);
      alphas_out[t] = alpha;
      std::vector<ParamVector> grads(static_cast<size_t>(W));
      for (int k = 0; k < W; ++k) {
        const WorkerState& x = ws[static_cast<size_t>(k)];
        // sample_batch (sync.cpp:153-179), restated: it is not in a public header
        std::vector<int> b(static_cast<size_t>(batch));
        if (!sampling) {
          Rng br = Rng::for_stream(run_seed, streams::kBatch, static_cast<uint64_t>(k), static_cast<uint64_t>(t));
          for (auto& idx : b) idx = x.shard.indices[br.uniform_below(x.shard.indices.size())];
        } else {
          const long size = static_cast<long>(x.shard.indices.size());
          long pos = static_cast<long>(t) * batch;
          for (auto& idx : b) {
            idx = epoch_order(x.shard, run_seed, k, pos / size)[static_cast<size_t>(pos % size)];
            ++pos;
          }
        }
        std::memcpy(batches_out + (static_cast<long>(t) * W + k) * batch, b.data(), sizeof(int) * static_cast<size_t>(batch));
        Rng noise = Rng::for_stream(run_seed, streams::kGradientNoise, static_cast<uint64_t>(k), static_cast<uint64_t>(t));
        grads[static_cast<size_t>(k)] = problem->stochastic_gradient(x.params, b, noise).grad;
        std::memcpy(grads_out + (static_cast<long>(t) * W + k) * d, grads[static_cast<size_t>(k)].data(), sizeof(double) * static_cast<size_t>(d));
      }
      if (kind == 1) {
        for (int k = 0; k < W; ++k) local_step(ws[static_cast<size_t>(k)], grads[static_cast<size_t>(k)], alpha, t);
        sync_round(ws, strat, t);
      } else {
        std::vector<int> members(static_cast<size_t>(W));
        for (int k = 0; k < W; ++k) members[static_cast<size_t>(k)] = k;
        const AllReduceResult r = ring_allreduce_avg(members, grads);
        for (int k = 0; k < W; ++k) local_step(ws[static_cast<size_t>(k)], r.values[static_cast<size_t>(k)], alpha, t);
      }
      for (int k = 0; k < W; ++k) {
        std::memcpy(params_out + (static_cast<long>(t) * W + k) * d, ws[static_cast<size_t>(k)].params.data(), sizeof(double) * static_cast<size_t>(d));
      }
    }
    const RunResult rr = run_training(*problem, strat, o);
    *matches = 1;
    for (int k = 0; k < W; ++k) {
      if (rr.final_workers[static_cast<size_t>(k)].params != ws[static_cast<size_t>(k)].params) *matches = 0;
    }
  });
}

// y_i * x_i of the logistic dataset through the public Problem API: with
// l2 = 0, w = 0 and the one-example batch {i}, stochastic_gradient is
// (-y_i * 0.5) * x_i exactly (problems.cpp:265-290), so -2 * grad = y_i * x_i.
// The model depends on the data only through these products.
int ref_logistic_yx(uint64_t seed, int d, int M, double* out, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "logistic";
    s.d = d;
    s.M = M;
    s.mu = 0.0;
    s.seed = seed;
    auto problem = make_problem(s);
    const ParamVector w(static_cast<size_t>(d), 0.0);
    Rng noise(0);
    for (int i = 0; i < M; ++i) {
      const int b[1] = {i};
      const GradSample g = problem->stochastic_gradient(w, std::span<const int>(b, 1), noise);
      for (int j = 0; j < d; ++j) out[static_cast<long>(i) * d + j] = -2.0 * g.grad[static_cast<size_t>(j)];
    }
  });
}

// load_logistic_csv through make_problem (problems.cpp:572-640): M, d and
// y_i * x_i (as ref_logistic_yx) when out is non-null.
int ref_load_csv(const char* path, double l2, double* out, int cap, int* M, int* d, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "logistic";
    s.csv = path;
    s.mu = l2;
    auto problem = make_problem(s);
    *M = problem->dataset_size();
    *d = problem->dim();
    if (!out || static_cast<long>(*M) * *d > cap) return;
    const ParamVector w(static_cast<size_t>(*d), 0.0);
    const std::unique_ptr<Problem> p0 = [&] {
      DatasetSpec z = s;
      z.mu = 0.0;
      return make_problem(z);
    }();
    Rng noise(0);
    for (int i = 0; i < *M; ++i) {
      const int b[1] = {i};
      const GradSample g = p0->stochastic_gradient(w, std::span<const int>(b, 1), noise);
      for (int j = 0; j < *d; ++j) out[static_cast<long>(i) * *d + j] = -2.0 * g.grad[static_cast<size_t>(j)];
    }
  });
}

int ref_make_shards(int M, int W, uint64_t seed, int* indices, int* offsets, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    const std::vector<Shard> sh = make_shards(M, W, seed);
    int n = 0;
    offsets[0] = 0;
    for (int w = 0; w < W; ++w) {
      for (int i : sh[static_cast<size_t>(w)].indices) indices[n++] = i;
      offsets[w + 1] = n;
    }
  });
}

int ref_epoch_order(const int* shard, int size, uint64_t seed, int rank, long epoch, int* out) {
  Shard s;
  s.indices.assign(shard, shard + size);
  const std::vector<int> o = epoch_order(s, seed, rank, epoch);
  for (int i = 0; i < size; ++i) out[i] = o[static_cast<size_t>(i)];
  return 0;
}

// The reference's `dssync run` (tools/main.cpp:34-55) through its public
// API: load_run_config, make_problem, build_run_options, run_training,
// metrics_csv / summary_json / atomic_write_file into out_dir.
int ref_cmd_run(const char* config_path, const char* out_dir, char* err, int errlen, int* rank, long* it) {
  return guarded(err, errlen, rank, it, [&] {
    const RunConfig cfg = load_run_config(config_path);
    std::unique_ptr<Problem> problem = make_problem(cfg.problem);
    std::vector<SeedOutcome> outcomes;
    for (uint64_t seed : cfg.seeds) {
      const RunOptions opts = build_run_options(cfg, *problem, seed);
      const RunResult result = run_training(*problem, cfg.strategy, opts);
      const IterationTrace& last = result.traces.back();
      outcomes.push_back({seed, last.mean_post_sync_loss, last.suboptimality});
      atomic_write_file(std::string(out_dir) + "/metrics_seed" + std::to_string(seed) + ".csv",
                        metrics_csv(result.traces));
    }
    atomic_write_file(std::string(out_dir) + "/summary.json", summary_json(cfg, outcomes));
  });
}

// parse_run_config only: 0 or 4 (ConfigError) with the message.
int ref_parse_config(const char* text, char* err, int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] { (void)parse_run_config(text); });
}

// Tiny-MLP run (problems.cpp:436-570: running statistics = EMA of the hidden
// pre-activations, stats_dim = hidden), DS or BSP, replayed through the
// public API with the fold_running_stats EMA restated (sync.cpp:193-201:
// rs = 0.9*rs + 0.1*obs), recording per t:
//   grads [T][W][dim], obs [T][W][h], params [T][W][dim], stats [T][W][h]
// and checked against run_training's final params and running_stats.
int ref_mlp_run(int kind, int W, int N, int d_in, int M, int hidden, uint64_t problem_seed, uint64_t run_seed,
                int batch, int T, int opt, const double* hp, double alpha, double* grads_out, double* obs_out,
                double* params_out, double* stats_out, double* w0_out, int* batches_out, int* matches, char* err,
                int errlen) {
  return guarded(err, errlen, nullptr, nullptr, [&] {
    DatasetSpec s;
    s.kind = "tiny-mlp";
    s.d = d_in;
    s.M = M;
    s.hidden = hidden;
    s.seed = problem_seed;
    auto problem = make_problem(s);
    const int dim = problem->dim();
    const int h = problem->stats_dim();
    const SyncStrategy strat = make_strategy(kind, 0, W, N, 1);
    RunOptions o;
    o.iterations = T;
    o.seed = run_seed;
    o.batch_size = batch;
    o.optimizer = make_opt(opt, hp, alpha);
    o.lr = constant_lr(alpha);
    const std::vector<Shard> shards = make_shards(problem->dataset_size(), W, run_seed);
    std::vector<WorkerState> ws(static_cast<size_t>(W));
    for (int k = 0; k < W; ++k) {
      ws[static_cast<size_t>(k)].rank = k;
      ws[static_cast<size_t>(k)].params = problem->initial_params();
      ws[static_cast<size_t>(k)].running_stats.assign(static_cast<size_t>(h), 0.0);
      ws[static_cast<size_t>(k)].opt = o.optimizer;
      ws[static_cast<size_t>(k)].shard = shards[static_cast<size_t>(k)];
    }
    std::memcpy(w0_out, ws[0].params.data(), sizeof(double) * static_cast<size_t>(dim));
    auto ema = [](WorkerState& x, const ParamVector& obs) {
      for (size_t i = 0; i < x.running_stats.size(); ++i) x.running_stats[i] = 0.9 * x.running_stats[i] + 0.1 * obs[i];
    };
    for (int t = 0; t < T; ++t) {
      std::vector<GradSample> smp(static_cast<size_t>(W));
      for (int k = 0; k < W; ++k) {
        const WorkerState& x = ws[static_cast<size_t>(k)];
        Rng br = Rng::for_stream(run_seed, streams::kBatch, static_cast<uint64_t>(k), static_cast<uint64_t>(t));
        std::vector<int> b(static_cast<size_t>(batch));
        for (auto& idx : b) idx = x.shard.indices[br.uniform_below(x.shard.indices.size())];
        std::memcpy(batches_out + (static_cast<long>(t) * W + k) * batch, b.data(), sizeof(int) * static_cast<size_t>(batch));
        Rng noise = Rng::for_stream(run_seed, streams::kGradientNoise, static_cast<uint64_t>(k), static_cast<uint64_t>(t));
        smp[static_cast<size_t>(k)] = problem->stochastic_gradient(x.params, b, noise);
        std::memcpy(grads_out + (static_cast<long>(t) * W + k) * dim, smp[static_cast<size_t>(k)].grad.data(), sizeof(double) * static_cast<size_t>(dim));
        std::memcpy(obs_out + (static_cast<long>(t) * W + k) * h, smp[static_cast<size_t>(k)].stats_observation.data(), sizeof(double) * static_cast<size_t>(h));
      }
      if (kind == 1) {  // DS: local step, EMA, then params ++ stats averaged in groups
        for (int k = 0; k < W; ++k) {
          local_step(ws[static_cast<size_t>(k)], smp[static_cast<size_t>(k)].grad, alpha, t);
          ema(ws[static_cast<size_t>(k)], smp[static_cast<size_t>(k)].stats_observation);
        }
        sync_round(ws, strat, t);
      } else {  // BSP: EMA, one collective on grad ++ stats, then the step with the mean grad
        std::vector<int> members(static_cast<size_t>(W));
        std::vector<ParamVector> in(static_cast<size_t>(W));
        for (int k = 0; k < W; ++k) {
          ema(ws[static_cast<size_t>(k)], smp[static_cast<size_t>(k)].stats_observation);
          members[static_cast<size_t>(k)] = k;
          in[static_cast<size_t>(k)] = smp[static_cast<size_t>(k)].grad;
          in[static_cast<size_t>(k)].insert(in[static_cast<size_t>(k)].end(), ws[static_cast<size_t>(k)].running_stats.begin(),
                                            ws[static_cast<size_t>(k)].running_stats.end());
        }
        const AllReduceResult r = ring_allreduce_avg(members, in);
        for (int k = 0; k < W; ++k) {
          const ParamVector& pl = r.values[static_cast<size_t>(k)];
          ws[static_cast<size_t>(k)].running_stats.assign(pl.begin() + dim, pl.end());
          local_step(ws[static_cast<size_t>(k)], ParamVector(pl.begin(), pl.begin() + dim), alpha, t);
        }
      }
      for (int k = 0; k < W; ++k) {
        std::memcpy(params_out + (static_cast<long>(t) * W + k) * dim, ws[static_cast<size_t>(k)].params.data(), sizeof(double) * static_cast<size_t>(dim));
        std::memcpy(stats_out + (static_cast<long>(t) * W + k) * h, ws[static_cast<size_t>(k)].running_stats.data(), sizeof(double) * static_cast<size_t>(h));
      }
    }
    const RunResult rr = run_training(*problem, strat, o);
    *matches = 1;
    for (int k = 0; k < W; ++k) {
      if (rr.final_workers[static_cast<size_t>(k)].params != ws[static_cast<size_t>(k)].params) *matches = 0;
      if (rr.final_workers[static_cast<size_t>(k)].running_stats != ws[static_cast<size_t>(k)].running_stats) *matches = 0;
    }
  });
}

// ---------------------------------------------------------------------------
// CPU baseline: the reference's own per-iteration DS / BSP work on
// resident WorkerStates — apply_step for every worker (sync.cpp:348-362,
// threaded like run_training's Parallel mode) and each group's
// ring_allreduce_avg over concat'ed payloads, written back
// (sync.cpp:203-240,364-370).  The group table is passed in because the
// reference's make_partition rejects the rectangular C2/C3 shapes; every
// arithmetic op is the reference's.
struct RefBench {
  std::vector<WorkerState> ws;
  std::vector<ParamVector> grads;
  long d = 0;
};

void* ref_bench_create(int W, long d, int opt, const double* hp, uint64_t seed, int threads) {
  // Synthetic O(1) inputs from counter-addressed reference Rng streams, so
  // they can be generated on every host thread: the common start w0 in
  // 1M-element chunks, each worker's gradient from its own stream.
  auto* b = new RefBench;
  b->d = d;
  b->ws.resize(static_cast<size_t>(W));
  b->grads.resize(static_cast<size_t>(W));
  const long chunk = 1L << 20;
  ParamVector w0(static_cast<size_t>(d));
  parallel_for(static_cast<size_t>((d + chunk - 1) / chunk), threads, [&](size_t c) {
    Rng r = Rng::for_stream(seed, streams::kInitParams, c, 0);
    const long hi = std::min(d, static_cast<long>(c + 1) * chunk);
    for (long i = static_cast<long>(c) * chunk; i < hi; ++i) w0[static_cast<size_t>(i)] = r.gaussian();
  });
  parallel_for(static_cast<size_t>(W), threads, [&](size_t k) {
    WorkerState& x = b->ws[k];
    x.rank = static_cast<int>(k);
    x.params = w0;
    x.opt = make_opt(opt, hp, 0.0);
    Rng r = Rng::for_stream(seed, streams::kGradientNoise, k, 0);
    ParamVector g(static_cast<size_t>(d));
    for (auto& v : g) v = 0.01 * r.gaussian();
    b->grads[k] = std::move(g);
  });
  return b;
}

void ref_bench_destroy(void* h) { delete static_cast<RefBench*>(h); }

int ref_bench_ds_step(void* h, long t, double alpha, const int* members, const int* offsets, int n_groups,
                      int threads, char* err, int errlen) {
  auto* b = static_cast<RefBench*>(h);
  return guarded(err, errlen, nullptr, nullptr, [&] {
    parallel_for(b->ws.size(), threads, [&](size_t k) { local_step(b->ws[k], b->grads[k], alpha, t); });
    parallel_for(static_cast<size_t>(n_groups), threads, [&](size_t g) {
      std::vector<int> mem(members + offsets[g], members + offsets[g + 1]);
      std::vector<ParamVector> in;
      in.reserve(mem.size());
      for (int r : mem) in.push_back(b->ws[static_cast<size_t>(r)].params);  // concat_payload
      AllReduceResult red;
      try {
        red = ring_allreduce_avg(mem, in);
      } catch (const std::runtime_error& e) {
        throw DivergenceError(mem[0], t, e.what());
      }
      for (size_t i = 0; i < mem.size(); ++i) b->ws[static_cast<size_t>(mem[i])].params = std::move(red.values[i]);
    });
  });
}

int ref_bench_bsp_step(void* h, long t, double alpha, int threads, char* err, int errlen) {
  auto* b = static_cast<RefBench*>(h);
  return guarded(err, errlen, nullptr, nullptr, [&] {
    const int W = static_cast<int>(b->ws.size());
    std::vector<int> members(static_cast<size_t>(W));
    for (int k = 0; k < W; ++k) members[static_cast<size_t>(k)] = k;
    AllReduceResult red = ring_allreduce_avg(members, b->grads);
    parallel_for(b->ws.size(), threads, [&](size_t k) { local_step(b->ws[k], red.values[k], alpha, t); });
  });
}

// The group table the reference bench arm uses, built without the product
// library.  Legal shapes (W = N*N or N = W) come from the reference's own
// make_partition (schedule.cpp:31-54).  The rectangular C2/C3 shapes
// (W = N*K) are rejected by the reference's validate (schedule.cpp:8-24);
// for them this applies the builder's documented extension of
// schedule.cpp:49, g(x) = t even ? x / N : x % N, which reduces to the
// reference's rule when K = N.  Returns 1 for shapes neither rule covers.
int ref_bench_partition(int W, int N, int rect, long t, int* members, int* offsets, int* n_groups, char* err,
                        int errlen) {
  bool legal = true;
  try {
    validate(WorldConfig{W, N});
  } catch (const std::invalid_argument&) {
    legal = false;
  }
  if (legal) return ref_make_partition(W, N, t, members, offsets, n_groups, err, errlen);
  if (!rect || N <= 0 || W % N != 0 || t < 0) {
    put(err, errlen, "ref_bench_partition: shape is neither legal nor rectangular");
    return 1;
  }
  const int K = W / N;
  const int ng = (t % 2 == 0) ? K : N;
  int pos = 0;
  offsets[0] = 0;
  for (int g = 0; g < ng; ++g) {
    for (int x = 0; x < W; ++x) {
      if (((t % 2 == 0) ? x / N : x % N) == g) members[pos++] = x;
    }
    offsets[g + 1] = pos;
  }
  *n_groups = ng;
  return 0;
}

// The stock reference iteration on a legal shape: apply_step for every
// worker (threaded, like run_training's Parallel mode, sync.cpp:348-362)
// followed by the reference's own sync_round (sync.cpp:268-282), which
// syncs the groups one after another on the calling thread.
int ref_bench_stock_step(void* h, int N, long t, double alpha, int threads, char* err, int errlen) {
  auto* b = static_cast<RefBench*>(h);
  return guarded(err, errlen, nullptr, nullptr, [&] {
    parallel_for(b->ws.size(), threads, [&](size_t k) { local_step(b->ws[k], b->grads[k], alpha, t); });
    sync_round(b->ws, make_strategy(1, 0, static_cast<int>(b->ws.size()), N, 1), t);
  });
}

// Host memory the bench holds (params + grads + optimizer moments), bytes.
long ref_bench_bytes(void* h) {
  auto* b = static_cast<RefBench*>(h);
  long n = 0;
  for (size_t k = 0; k < b->ws.size(); ++k) {
    n += static_cast<long>(b->ws[k].params.size() + b->grads[k].size() + b->ws[k].opt.first_moment.size() +
                           b->ws[k].opt.second_moment.size());
  }
  return n * static_cast<long>(sizeof(double));
}

}  // extern "C"
