// C-ABI entry points of the gradient producers and their problem setup:
// the isotropic quadratic (QuadraticProblem with A = mu*I,
// problems.cpp:120-224) and logistic regression with device batch sampling
// (problems.cpp:226-430, sync.cpp:153-191).  Setup runs on the host,
// bit-exact (problems.cpp here); every iteration's work runs on the device.
#include "context.cuh"

using namespace dssb;

extern "C" int dss_quadratic_gradients(dss_ctx* c, long t, uint64_t seed, double mu, double sigma) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (!(mu > 0.0)) throw std::invalid_argument("quadratic requires problem.mu > 0");
    if (sigma < 0.0) throw std::invalid_argument("problem.sigma must be >= 0");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const double scale = sigma > 0.0 ? sigma / std::sqrt(static_cast<double>(c->d)) : 0.0;
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      GradArgs<T> a{};
      a.w = static_cast<const T*>(c->w);
      a.g = static_cast<T*>(c->g);
      a.wstar = static_cast<const T*>(c->wstar);
      a.ld = c->d_pad;
      a.d = c->d;
      a.nlocal = c->P;
      a.mu = mu;
      a.scale = scale;
      for (int k = 0; k < c->P; ++k) {
        a.s0[k] = stream_state(seed, kGradientNoise, static_cast<uint64_t>(grank(c, c->first + k)),
                               static_cast<uint64_t>(t));
      }
      dim3 grid(grid_x(c, c->d_pad, c->P), c->P);
      TimedLaunch tl(c, DSS_KIND_GRADIENT);
      quad_grad_kernel<T><<<grid, kThreads, 0, c->stream>>>(a);
      ck(cudaGetLastError(), "quad_grad_kernel launch");
    };
    if (c->cfg.dtype == DSS_F64) {
      run(static_cast<double*>(nullptr));
    } else {
      run(static_cast<float*>(nullptr));
    }
    return DSS_OK;
  });
}

extern "C" int dss_quadratic_init(dss_ctx* c, uint64_t problem_seed, double delta0) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (!(delta0 > 0.0)) throw std::invalid_argument("problem.delta0 must be > 0");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    // scratch rows, freed on every exit (after the stream is drained)
    struct Scratch {
      double *ws = nullptr, *u = nullptr, *ss = nullptr;
      cudaStream_t st;
      ~Scratch() {
        cudaStreamSynchronize(st);
        cudaFree(ws);
        cudaFree(u);
        cudaFree(ss);
      }
    } sc{nullptr, nullptr, nullptr, c->stream};
    double*& ws = sc.ws;
    double*& u = sc.u;
    double*& ss = sc.ss;
    ck(cudaMalloc(&ws, sizeof(double) * c->d), "cudaMalloc");
    ck(cudaMalloc(&u, sizeof(double) * c->d), "cudaMalloc");
    const int gx = grid_x(c, c->d, 1);
    ck(cudaMalloc(&ss, sizeof(double) * (1 + static_cast<size_t>(gx))), "cudaMalloc");
    gaussian_fill_kernel<<<gx, kThreads, 0, c->stream>>>(ws, c->d, stream_state(problem_seed, kDataGen, 1, 0));
    gaussian_fill_kernel<<<gx, kThreads, 0, c->stream>>>(u, c->d, stream_state(problem_seed, kInitParams, 0, 0));
    sumsq_kernel<<<gx, kThreads, 0, c->stream>>>(u, c->d, ss + 1);
    sumsq_finish<<<1, 1, 0, c->stream>>>(ss + 1, gx, ss);
    const double r = std::sqrt(delta0);
    const int gp = grid_x(c, c->d_pad, 1);
    if (c->cfg.dtype == DSS_F64) {
      compose_init_kernel<double><<<gp, kThreads, 0, c->stream>>>(ws, u, ss, c->d, c->d_pad, r,
                                                                 static_cast<double*>(c->wstar),
                                                                 static_cast<double*>(c->w));
      broadcast_row_kernel<double><<<grid_x(c, c->d_pad * c->P, 1), kThreads, 0, c->stream>>>(
          static_cast<double*>(c->w), c->d_pad, c->P, static_cast<double*>(c->w));
    } else {
      compose_init_kernel<float><<<gp, kThreads, 0, c->stream>>>(ws, u, ss, c->d, c->d_pad, r,
                                                                static_cast<float*>(c->wstar),
                                                                static_cast<float*>(c->w));
      broadcast_row_kernel<float><<<grid_x(c, c->d_pad * c->P, 1), kThreads, 0, c->stream>>>(
          static_cast<float*>(c->w), c->d_pad, c->P, static_cast<float*>(c->w));
    }
    ck(cudaGetLastError(), "init kernels");
    ck(cudaStreamSynchronize(c->stream), "init sync");
    return DSS_OK;
  });
}

extern "C" int dss_set_optimum(dss_ctx* c, const void* host, long n) {
  if (!c || !host) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (n < 0 || n > c->d) throw std::invalid_argument("optimum length exceeds dim");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaMemcpyAsync(c->wstar, host, static_cast<size_t>(n) * c->esz, cudaMemcpyHostToDevice, c->stream),
       "set_optimum");
    ck(cudaStreamSynchronize(c->stream), "set_optimum sync");
    return DSS_OK;
  });
}

extern "C" int dss_quadratic_losses(dss_ctx* c, double mu, int exact, double* losses, double* suboptimality) {
  if (!c || !losses) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    if (!c->d_loss) c->d_loss = static_cast<double*>(dalloc(c, sizeof(double) * (c->P + 1)));
    const int rows = c->P + (suboptimality ? 1 : 0);
    if (!c->d_loss_rows) {  // every local row, then the global-mean row (after dss_global_mean)
      std::vector<void*> ptrs;
      for (int k = 0; k < c->P; ++k) {
        ptrs.push_back(static_cast<char*>(c->w) + static_cast<size_t>(k) * c->d_pad * c->esz);
      }
      ptrs.push_back(c->mg);
      c->d_loss_rows = upload_table(c, ptrs);
    }
    void** d_ptrs = c->d_loss_rows;
    ck(cudaMemsetAsync(c->d_loss, 0, sizeof(double) * (c->P + 1), c->stream), "loss reset");
    dim3 grid(grid_x(c, c->d, rows), rows);
    if (exact) {
      if (c->cfg.dtype == DSS_F64) {
        quad_loss_exact_kernel<double><<<rows, 32, 0, c->stream>>>(reinterpret_cast<const double* const*>(d_ptrs),
                                                                  static_cast<const double*>(c->wstar), c->d, mu,
                                                                  c->d_loss);
      } else {
        quad_loss_exact_kernel<float><<<rows, 32, 0, c->stream>>>(reinterpret_cast<const float* const*>(d_ptrs),
                                                                 static_cast<const float*>(c->wstar), c->d, mu,
                                                                 c->d_loss);
      }
    } else if (c->cfg.dtype == DSS_F64) {
      quad_loss_kernel<double><<<grid, kThreads, 0, c->stream>>>(reinterpret_cast<const double* const*>(d_ptrs),
                                                                 static_cast<const double*>(c->wstar), c->d, mu, c->d_loss);
    } else {
      quad_loss_kernel<float><<<grid, kThreads, 0, c->stream>>>(reinterpret_cast<const float* const*>(d_ptrs),
                                                                static_cast<const float*>(c->wstar), c->d, mu, c->d_loss);
    }
    ck(cudaGetLastError(), "quad_loss_kernel launch");
    std::vector<double> h(static_cast<size_t>(rows));
    ck(cudaMemcpyAsync(h.data(), c->d_loss, sizeof(double) * rows, cudaMemcpyDeviceToHost, c->stream), "loss readback");
    ck(cudaStreamSynchronize(c->stream), "loss sync");
    for (int k = 0; k < c->P; ++k) losses[k] = h[static_cast<size_t>(k)];
    if (suboptimality) *suboptimality = h[static_cast<size_t>(c->P)];
    return DSS_OK;
  });
}

// ====================== logistic problem on the device ======================

extern "C" int dss_logistic_dataset(uint64_t seed, int d, int M, double* x, double* y) {
  if (!x || !y) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    std::vector<double> hx, hy;
    logistic_dataset(seed, d, M, hx, hy);
    std::memcpy(x, hx.data(), sizeof(double) * hx.size());
    std::memcpy(y, hy.data(), sizeof(double) * hy.size());
    return DSS_OK;
  });
}

extern "C" int dss_quadratic_problem(uint64_t seed, int d, double delta0, double* wstar, double* w0) {
  if (!wstar || !w0) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    std::vector<double> ws, x0;
    quadratic_problem(seed, d, delta0, ws, x0);
    std::memcpy(wstar, ws.data(), sizeof(double) * ws.size());
    std::memcpy(w0, x0.data(), sizeof(double) * x0.size());
    return DSS_OK;
  });
}

extern "C" int dss_logistic_constants(const double* x, const double* y, int M, int d, double l2,
                                      double* smoothness, double* f_star, double* w_opt) {
  if (!x || !y || !smoothness || !f_star) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    if (l2 < 0.0) throw std::invalid_argument("logistic l2 must be >= 0");
    const LogisticConstants k = logistic_constants(x, y, M, d, l2);
    *smoothness = k.smoothness;
    *f_star = l2 > 0.0 ? k.f_star : std::nan("");
    if (w_opt && l2 > 0.0) std::copy(k.w_opt.begin(), k.w_opt.end(), w_opt);
    return DSS_OK;
  });
}

extern "C" int dss_make_shards(int dataset_size, int workers, uint64_t seed, int* indices, int* offsets) {
  if (!indices || !offsets) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    std::vector<int> idx, off;
    make_shards(dataset_size, workers, seed, idx, off);
    std::copy(idx.begin(), idx.end(), indices);
    std::copy(off.begin(), off.end(), offsets);
    return DSS_OK;
  });
}

extern "C" int dss_epoch_order(const int* shard, int size, uint64_t seed, int rank, long epoch, int* out) {
  if ((!shard || !out) && size > 0) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    if (size < 0) throw std::invalid_argument("epoch_order: size must be >= 0");
    epoch_order(shard, size, seed, rank, epoch, out);
    return DSS_OK;
  });
}

namespace dssb {

void free_logistic(dss_ctx* c) {
  for (void* p : c->logi.mem) {
    char* user = static_cast<char*>(p) + c->guard;
    c->guarded.erase(std::remove_if(c->guarded.begin(), c->guarded.end(),
                                    [&](const std::pair<char*, size_t>& gb) { return gb.first == user; }),
                     c->guarded.end());
    cudaFree(p);
  }
  c->logi.mem.clear();
  c->logi.ready = false;
}

template <typename P>
P* logi_alloc(dss_ctx* c, size_t n) {
  void* p = nullptr;
  const size_t g = static_cast<size_t>(c->guard), bytes = std::max<size_t>(n, 1) * sizeof(P);
  ck(cudaMalloc(&p, bytes + 2 * g), "cudaMalloc");
  c->logi.mem.push_back(p);
  char* user = static_cast<char*>(p) + g;
  if (g) {  // guard bands, as dalloc (checked by dss_check_guards)
    ck(cudaMemset(p, kGuardByte, g), "guard");
    ck(cudaMemset(user + bytes, kGuardByte, g), "guard");
    c->guarded.push_back({user, bytes});
  }
  return reinterpret_cast<P*>(user);
}

// w as doubles [d] + the -y*s factors [batch]
size_t logistic_smem(long d, long batch) { return sizeof(double) * static_cast<size_t>(d + batch); }
constexpr long kLogisticMaxSmem = 200 * 1024;

}  // namespace dssb

namespace {

size_t mlp_smem(long dim, int batch, int hidden) {
  return sizeof(double) * static_cast<size_t>(dim + 3L * batch * hidden + batch);
}

// Upload a dataset problem (x: M x d_feat, y: M) and shard it over the world
// (make_shards(M, W, run_seed), sync.cpp:300); this GPU keeps its workers'
// shards, the epoch-order cache and the batch rows.
void dataset_setup(dss_ctx* c, const double* x, const double* y, int M, int d_feat, int hidden, double l2,
                   int batch_size, int sampling, uint64_t run_seed) {
  if (batch_size < 1) throw std::invalid_argument("batch_size must be >= 1");
  if (sampling != DSS_SAMPLING_REPLACEMENT && sampling != DSS_SAMPLING_EPOCH) {
    throw std::invalid_argument("sampling must be replacement or epoch");
  }
  ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
  ck(cudaStreamSynchronize(c->stream), "stream sync");
  free_logistic(c);
  std::vector<int> idx, off;
  make_shards(M, c->cfg.strategy.world_size, run_seed, idx, off);
  // this GPU's workers' shards in local-row order (their global ranks need not be contiguous)
  std::vector<int> local_off(static_cast<size_t>(c->P) + 1, 0), local_idx;
  long max_shard = 0;
  for (int k = 0; k < c->P; ++k) {
    const size_t r = static_cast<size_t>(grank(c, c->first + k));
    local_idx.insert(local_idx.end(), idx.begin() + off[r], idx.begin() + off[r + 1]);
    const int n = off[r + 1] - off[r];
    local_off[static_cast<size_t>(k) + 1] = local_off[static_cast<size_t>(k)] + n;
    max_shard = std::max<long>(max_shard, n);
  }
  auto& L = c->logi;
  const size_t xn = static_cast<size_t>(M) * d_feat;
  L.x = logi_alloc<double>(c, xn);
  L.y = logi_alloc<double>(c, static_cast<size_t>(M));
  L.shard = logi_alloc<int>(c, static_cast<size_t>(local_off.back()));
  L.shard_off = logi_alloc<int>(c, local_off.size());
  L.order = logi_alloc<int>(c, static_cast<size_t>(c->P) * max_shard);
  L.order_epoch = logi_alloc<long>(c, static_cast<size_t>(c->P));
  L.batch = logi_alloc<int>(c, static_cast<size_t>(c->P) * batch_size);
  ck(cudaMemcpy(L.x, x, sizeof(double) * xn, cudaMemcpyHostToDevice), "dataset x upload");
  ck(cudaMemcpy(L.y, y, sizeof(double) * M, cudaMemcpyHostToDevice), "dataset y upload");
  ck(cudaMemcpy(L.shard, local_idx.data(), sizeof(int) * local_off.back(), cudaMemcpyHostToDevice), "shard upload");
  ck(cudaMemcpy(L.shard_off, local_off.data(), sizeof(int) * local_off.size(), cudaMemcpyHostToDevice),
     "shard upload");
  ck(cudaMemset(L.order_epoch, 0xff, sizeof(long) * c->P), "epoch init");  // -1
  ck(cudaMemset(L.batch, 0, sizeof(int) * c->P * batch_size), "batch init");
  L.max_shard = max_shard;
  L.M = M;
  L.B = batch_size;
  L.sampling = sampling;
  L.d_feat = d_feat;
  L.hidden = hidden;
  L.l2 = l2;
  L.seed = run_seed;
  L.ready = true;
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) {
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
       "smem attr");
  }
}

}  // namespace

extern "C" int dss_logistic_setup(dss_ctx* c, const double* x, const double* y, int M, double l2, int batch_size,
                                  int sampling, uint64_t run_seed) {
  if (!c || !x || !y) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (M < 1) throw std::invalid_argument("logistic requires problem.M >= 1");
    if (!(l2 >= 0.0)) throw std::invalid_argument("problem.mu must be >= 0");
    if (batch_size >= 1 && static_cast<long>(logistic_smem(c->d, batch_size)) > kLogisticMaxSmem) {
      throw std::invalid_argument("logistic on the device supports (dim + batch_size) * 8 B <= 200 KiB");
    }
    dataset_setup(c, x, y, M, static_cast<int>(c->d), 0, l2, batch_size, sampling, run_seed);
    allow_smem(logistic_grad_kernel<double>, logistic_smem(c->d, batch_size));
    allow_smem(logistic_grad_kernel<float>, logistic_smem(c->d, batch_size));
    return DSS_OK;
  });
}

extern "C" int dss_mlp_setup(dss_ctx* c, const double* x, const double* y, int M, int d_in, int hidden,
                             int batch_size, int sampling, uint64_t run_seed) {
  if (!c || !x || !y) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (M < 1) throw std::invalid_argument("tiny-mlp requires problem.M >= 1");
    if (d_in < 1) throw std::invalid_argument("problem.d must be >= 1 (got " + std::to_string(d_in) + ")");
    if (hidden < 1 || hidden > 32) {
      throw std::invalid_argument("problem.hidden must be in [1, 32] (got " + std::to_string(hidden) + ")");
    }
    const long dim = static_cast<long>(hidden) * d_in + 2 * hidden + 1;
    if (c->d != dim) throw std::invalid_argument("tiny-mlp: the context dim must be hidden * d + 2 * hidden + 1");
    if (c->s != hidden) throw std::invalid_argument("tiny-mlp: the context stats_dim must equal hidden");
    if (batch_size >= 1 && static_cast<long>(mlp_smem(dim, batch_size, hidden)) > kLogisticMaxSmem) {
      throw std::invalid_argument("tiny-mlp on the device supports (dim + 3 * batch * hidden + batch) * 8 B <= 200 KiB");
    }
    dataset_setup(c, x, y, M, d_in, hidden, 0.0, batch_size, sampling, run_seed);
    allow_smem(mlp_grad_kernel<double>, mlp_smem(dim, batch_size, hidden));
    allow_smem(mlp_grad_kernel<float>, mlp_smem(dim, batch_size, hidden));
    return DSS_OK;
  });
}

namespace dssb {

LogisticArgs logistic_args(dss_ctx* c, long t) {
  const auto& L = c->logi;
  LogisticArgs a{};
  a.x = L.x;
  a.y = L.y;
  a.shard = L.shard;
  a.shard_off = L.shard_off;
  a.order = L.order;
  a.order_epoch = L.order_epoch;
  a.batch = L.batch;
  a.max_shard = L.max_shard;
  a.ld = c->d_pad;
  a.d = L.d_feat;
  a.hidden = L.hidden;
  a.obs_ld = c->s_pad;
  a.B = L.B;
  a.sampling = L.sampling;
  a.l2 = L.l2;
  a.seed = L.seed;
  a.t = t;
  a.rank_of = c->d_rank_of;
  a.gerr = c->d_gerr;
  return a;
}

void launch_logistic(dss_ctx* c, long t) {
  const LogisticArgs a = logistic_args(c, t);
  TimedLaunch tl(c, DSS_KIND_GRADIENT);
  if (c->cfg.dtype == DSS_F64) {
    logistic_grad_kernel<double><<<c->P, 128, logistic_smem(c->d, c->logi.B), c->stream>>>(
        a, static_cast<const double*>(c->w), static_cast<double*>(c->g));
  } else {
    logistic_grad_kernel<float><<<c->P, 128, logistic_smem(c->d, c->logi.B), c->stream>>>(
        a, static_cast<const float*>(c->w), static_cast<float*>(c->g));
  }
  ck(cudaGetLastError(), "logistic_grad_kernel launch");
}

}  // namespace

extern "C" int dss_logistic_gradients(dss_ctx* c, long t) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (!c->logi.ready || c->logi.hidden) throw std::invalid_argument("dss_logistic_setup has not been called");
    if (t < 0) throw std::invalid_argument("iteration must be >= 0");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    launch_logistic(c, t);
    return DSS_OK;
  });
}

extern "C" int dss_logistic_steps(dss_ctx* c, long t0, long n, const double* alphas, int check, dss_outcome* last) {
  if (!c || (!alphas && n > 0)) return fail(c, DSS_EINVAL, "null argument");
  if (small_path(c, n) && small_bytes(c) <= 32768 && c->logi.ready && !c->logi.hidden && c->d <= kSmallLogiMaxDim &&
      c->logi.B <= kSmallLogiMaxBatch) {
    // the whole run in one CTA: sampling, gradient, step and group fold
    const int st = guard(c, [&]() -> int {
      if (t0 < 0) throw std::invalid_argument("iteration must be >= 0");
      for (long i = 0; i < n; ++i) {
        if (!std::isfinite(alphas[i]) || alphas[i] < 0.0) {
          throw std::invalid_argument("learning rate at t=" + std::to_string(t0 + i) + " must be finite and >= 0");
        }
      }
      ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
      if (c->cfg.dtype == DSS_F64) {
        run_small<double>(c, t0, n, alphas, true);
      } else {
        run_small<float>(c, t0, n, alphas, true);
      }
      if (last) *last = round_outcome(c->cfg.strategy, t0 + n - 1, c->d + c->s);
      return DSS_OK;
    });
    if (st != DSS_OK) return st;
    if (check) return dss_check(c);
    return DSS_OK;
  }
  for (long i = 0; i < n; ++i) {
    int st = dss_logistic_gradients(c, t0 + i);
    if (st == DSS_OK) st = dss_step(c, t0 + i, alphas[i], 0, last);
    if (st != DSS_OK) return st;
  }
  if (check) return dss_check(c);
  return DSS_OK;
}

extern "C" int dss_mlp_gradients(dss_ctx* c, long t) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (!c->logi.ready || !c->logi.hidden) throw std::invalid_argument("dss_mlp_setup has not been called");
    if (t < 0) throw std::invalid_argument("iteration must be >= 0");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const LogisticArgs a = logistic_args(c, t);
    const size_t smem = mlp_smem(c->d, c->logi.B, c->logi.hidden);
    TimedLaunch tl(c, DSS_KIND_GRADIENT);
    if (c->cfg.dtype == DSS_F64) {
      mlp_grad_kernel<double><<<c->P, 128, smem, c->stream>>>(a, static_cast<const double*>(c->w),
                                                              static_cast<double*>(c->g),
                                                              static_cast<double*>(c->stats_obs));
    } else {
      mlp_grad_kernel<float><<<c->P, 128, smem, c->stream>>>(a, static_cast<const float*>(c->w),
                                                             static_cast<float*>(c->g),
                                                             static_cast<float*>(c->stats_obs));
    }
    ck(cudaGetLastError(), "mlp_grad_kernel launch");
    return DSS_OK;
  });
}

extern "C" int dss_mlp_losses(dss_ctx* c, int exact, double* losses) {
  if (!c || !losses) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (!c->logi.ready || !c->logi.hidden) throw std::invalid_argument("dss_mlp_setup has not been called");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    if (!c->d_loss) c->d_loss = static_cast<double*>(dalloc(c, sizeof(double) * (c->P + 1)));
    const auto& L = c->logi;
    if (c->cfg.dtype == DSS_F64) {
      mlp_loss_kernel<double><<<c->P, kThreads, 0, c->stream>>>(static_cast<const double*>(c->w), c->d_pad, L.x, L.y,
                                                               L.d_feat, L.hidden, L.M, exact, c->d_loss);
    } else {
      mlp_loss_kernel<float><<<c->P, kThreads, 0, c->stream>>>(static_cast<const float*>(c->w), c->d_pad, L.x, L.y,
                                                              L.d_feat, L.hidden, L.M, exact, c->d_loss);
    }
    ck(cudaGetLastError(), "mlp_loss_kernel launch");
    ck(cudaMemcpyAsync(losses, c->d_loss, sizeof(double) * c->P, cudaMemcpyDeviceToHost, c->stream), "loss readback");
    ck(cudaStreamSynchronize(c->stream), "loss sync");
    return DSS_OK;
  });
}

extern "C" int dss_mlp_dataset(uint64_t seed, int d, int M, double* x, double* y) {
  if (!x || !y) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    std::vector<double> hx, hy;
    mlp_dataset(seed, d, M, hx, hy);
    std::memcpy(x, hx.data(), sizeof(double) * hx.size());
    std::memcpy(y, hy.data(), sizeof(double) * hy.size());
    return DSS_OK;
  });
}

extern "C" int dss_mlp_initial_params(uint64_t seed, int d, int hidden, double* w) {
  if (!w) return fail(nullptr, DSS_EINVAL, "null argument");
  return guard(nullptr, [&]() -> int {
    std::vector<double> hw;
    mlp_initial_params(seed, d, hidden, hw);
    std::memcpy(w, hw.data(), sizeof(double) * hw.size());
    return DSS_OK;
  });
}

extern "C" int dss_logistic_batch(dss_ctx* c, int* out) {
  if (!c || !out) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (!c->logi.ready) throw std::invalid_argument("dss_logistic_setup has not been called");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaMemcpyAsync(out, c->logi.batch, sizeof(int) * c->P * c->logi.B, cudaMemcpyDeviceToHost, c->stream),
       "batch download");
    ck(cudaStreamSynchronize(c->stream), "batch sync");
    return DSS_OK;
  });
}

extern "C" int dss_logistic_losses(dss_ctx* c, int exact, double* losses) {
  if (!c || !losses) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (!c->logi.ready || c->logi.hidden) throw std::invalid_argument("dss_logistic_setup has not been called");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    if (!c->d_loss) c->d_loss = static_cast<double*>(dalloc(c, sizeof(double) * (c->P + 1)));
    const auto& L = c->logi;
    if (c->cfg.dtype == DSS_F64) {
      logistic_loss_kernel<double><<<c->P, kThreads, 0, c->stream>>>(static_cast<const double*>(c->w), c->d_pad, L.x,
                                                                     L.y, static_cast<int>(c->d), L.M, L.l2, exact,
                                                                     c->d_loss);
    } else {
      logistic_loss_kernel<float><<<c->P, kThreads, 0, c->stream>>>(static_cast<const float*>(c->w), c->d_pad, L.x,
                                                                    L.y, static_cast<int>(c->d), L.M, L.l2, exact,
                                                                    c->d_loss);
    }
    ck(cudaGetLastError(), "logistic_loss_kernel launch");
    ck(cudaMemcpyAsync(losses, c->d_loss, sizeof(double) * c->P, cudaMemcpyDeviceToHost, c->stream), "loss readback");
    ck(cudaStreamSynchronize(c->stream), "loss sync");
    return DSS_OK;
  });
}

