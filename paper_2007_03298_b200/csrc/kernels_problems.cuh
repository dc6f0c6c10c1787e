// Gradient producers on the device: the isotropic quadratic
// (problems.cpp:173-200), logistic regression with batch sampling
// (problems.cpp:265-305, sync.cpp:153-191), initial rows, losses, and the
// running-stats EMA (sync.cpp:193-201).
#pragma once

#include "kernel_common.cuh"

namespace dssb {

// ---- logistic regression with device batch sampling ------------------------
// LogisticProblem::stochastic_gradient (problems.cpp:265-290) fed by
// sample_batch (sync.cpp:153-179): one CTA per local worker.  Thread 0 draws
// the batch from the worker's shard with the reference's SplitMix64 streams
// (integer work: bit-exact indices), then the CTA walks the batch in order:
// the products x_j * w_j in parallel, their sum sequentially from 0.0 (the
// reference's dot order), and the per-feature accumulation -y*s*x_j in
// parallel (each feature's sum keeps the reference's sample order).  Every
// add/mul is an explicit _rn op; the only inexact step against the
// reference is exp() in the sigmoid (CUDA's libdevice vs glibc, <= 1 ulp).

__device__ __forceinline__ uint64_t stream_state_dev(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t it) {
  uint64_t s = mix64(seed + 0x9e3779b97f4a7c15ULL);
  s = mix64(s ^ purpose);
  s = mix64(s ^ rank);
  return mix64(s ^ it);
}

struct DevRng {  // Rng::next_u64 / uniform_below (rng.cpp:28-43)
  uint64_t s;
  __device__ __forceinline__ uint64_t next() {
    s += 0x9e3779b97f4a7c15ULL;
    return mix64(s);
  }
  __device__ __forceinline__ uint64_t below(uint64_t n) {
    const uint64_t limit = ~0ULL - ~0ULL % n;
    uint64_t v = next();
    while (v >= limit) v = next();
    return v % n;
  }
};

constexpr uint64_t kBatchStream = 0xd6e8feb86659fd93ULL;       // rng.hpp:45
constexpr uint64_t kEpochOrderStream = 0xe7037ed1a0b428dbULL;  // rng.hpp:47

// A dataset problem on the device: logistic regression (hidden = 0) or
// the tiny MLP (hidden units, running-stat observations into obs).
struct LogisticArgs {
  const double* x;        // [M][d] row-major (d = features)
  const double* y;        // [M] labels in {-1, +1} (logistic) / targets (MLP)
  const int* shard;       // local workers' shards, concatenated
  const int* shard_off;   // [P + 1]
  int* order;             // [P][max_shard] cached epoch order (epoch sampling)
  long* order_epoch;      // [P] epoch held in order (-1 = none)
  int* batch;             // [P][B] the sampled indices
  long max_shard;
  long ld;                // row stride of w / g
  int d, B, sampling;     // sampling: 0 replacement, 1 epoch
  double l2;
  uint64_t seed;
  long t;
  const int* rank_of;     // local row -> global rank (RNG streams, shards, error keys)
  unsigned long long* gerr;  // gradient failure latch: t << 32 | rank
  int hidden;             // MLP hidden units (0: logistic)
  long obs_ld;            // MLP: row stride of the running-stat observation rows
};

__device__ __forceinline__ double softplus_dev(double z) {  // problems.cpp:338-341
  return z > 0.0 ? __dadd_rn(z, log1p(exp(-z))) : log1p(exp(z));
}

// sample_batch (sync.cpp:153-179) for local worker k, into a.batch[k].
__device__ inline void sample_batch_dev(const LogisticArgs& a, int k) {
  const int rank = a.rank_of[k];
  const int* sh = a.shard + a.shard_off[k];
  const long size = a.shard_off[k + 1] - a.shard_off[k];
  int* bt = a.batch + static_cast<long>(k) * a.B;
  if (a.sampling == 0) {
    DevRng r{stream_state_dev(a.seed, kBatchStream, static_cast<uint64_t>(rank), static_cast<uint64_t>(a.t))};
    for (int b = 0; b < a.B; ++b) bt[b] = sh[r.below(static_cast<uint64_t>(size))];
    return;
  }
  int* ord = a.order + static_cast<long>(k) * a.max_shard;
  long pos = a.t * a.B;
  for (int b = 0; b < a.B; ++b, ++pos) {
    const long epoch = pos / size;
    if (a.order_epoch[k] != epoch) {  // epoch_order (problems.cpp:664-674)
      for (long i = 0; i < size; ++i) ord[i] = sh[i];
      DevRng r{stream_state_dev(a.seed, kEpochOrderStream, static_cast<uint64_t>(rank), static_cast<uint64_t>(epoch))};
      for (long i = size - 1; i > 0; --i) {
        const long j = static_cast<long>(r.below(static_cast<uint64_t>(i + 1)));
        const int tmp = ord[i];
        ord[i] = ord[j];
        ord[j] = tmp;
      }
      a.order_epoch[k] = epoch;
    }
    bt[b] = ord[pos % size];
  }
}

// Replacement sampling (sync.cpp:160-166) with the draws spread over
// threads: draw b of the stream is mix64(s0 + (b+1) * phi) unless an earlier
// draw was rejected by uniform_below (probability size / 2^64 per draw), so
// thread `lane` of `width` takes draws lane, lane + width, ...; if any draw
// is rejected, thread 0 redoes the batch sequentially.  `sync` is the
// barrier of the participating group (warp or block); bt is visible to the
// group on return.  Epoch sampling stays on thread 0 (its per-epoch order is
// one sequential shuffle, cached).
template <typename Sync, typename Any>
__device__ void sample_batch_par(const LogisticArgs& a, int k, int lane, int width, Sync sync, Any any) {
  if (a.sampling != 0) {
    if (lane == 0) sample_batch_dev(a, k);
    sync();
    return;
  }
  const int rank = a.rank_of[k];
  const int* sh = a.shard + a.shard_off[k];
  const uint64_t n = static_cast<uint64_t>(a.shard_off[k + 1] - a.shard_off[k]);
  int* bt = a.batch + static_cast<long>(k) * a.B;
  const uint64_t s0 = stream_state_dev(a.seed, kBatchStream, static_cast<uint64_t>(rank), static_cast<uint64_t>(a.t));
  const uint64_t limit = ~0ULL - ~0ULL % n;
  bool rejected = false;
  for (int b = lane; b < a.B; b += width) {
    const uint64_t v = mix64(s0 + static_cast<uint64_t>(b + 1) * 0x9e3779b97f4a7c15ULL);
    if (v >= limit) {
      rejected = true;
    } else {
      bt[b] = sh[v % n];
    }
  }
  if (any(rejected)) {
    if (lane == 0) sample_batch_dev(a, k);
  }
  sync();
}

// Is the batch loss of checked_gradient (problems.cpp:277-287, sync.cpp:186)
// finite?  Every term softplus(nz) <= max(nz, 0) + log 2, so when the
// largest nz, the batch size and the l2 term keep the sum far below the
// overflow threshold the loss is finite without evaluating log1p/exp on the
// critical path.  Otherwise (exploding params only) the exact loss is
// evaluated in the reference's order.
template <typename T>
__device__ bool logistic_loss_finite(const LogisticArgs& a, const int* bt, const T* wr, double max_nz, bool nan_nz) {
  if (nan_nz) return false;
  double dd = 0.0;
  if (a.l2 > 0.0) {
    for (int j = 0; j < a.d; ++j) dd = __dadd_rn(dd, __dmul_rn(static_cast<double>(wr[j]), static_cast<double>(wr[j])));
  }
  const double reg = __dmul_rn(__dmul_rn(0.5, a.l2), dd);
  if (max_nz < 1e300 / static_cast<double>(a.B) && reg < 1e300) return true;
  double loss = 0.0;
  for (int b = 0; b < a.B; ++b) {
    const double* x = a.x + static_cast<long>(bt[b]) * a.d;
    double z = 0.0;
    for (int j = 0; j < a.d; ++j) z = __dadd_rn(z, __dmul_rn(x[j], static_cast<double>(wr[j])));
    loss = __dadd_rn(loss, softplus_dev(__dmul_rn(-a.y[bt[b]], z)));
  }
  loss = __dmul_rn(loss, __ddiv_rn(1.0, static_cast<double>(a.B)));
  if (a.l2 > 0.0) loss = __dadd_rn(loss, reg);
  return isfinite(loss);
}


template <typename T> struct GradArgs {
  const T* w;
  T* g;
  const T* wstar;
  long ld;
  long d;      // real dimension (padding gets g = 0)
  int nlocal;
  double mu;
  double scale;  // sigma / sqrt(d); 0 disables noise
  uint64_t s0[kMaxLocal];  // for_stream(seed, kGradientNoise, rank, t) per local worker
};

// g_i = (0 + mu*(w_i - w*_i)) + scale * gaussian_i   (problems.cpp:173-193 with
// A = mu*I: the dense matvec over exact zeros reduces to +0 + mu*x_i).
template <typename T>
__global__ void __launch_bounds__(kThreads) quad_grad_kernel(const GradArgs<T> a) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  const int k = blockIdx.y;
  const T* w = a.w + static_cast<long>(k) * a.ld;
  T* g = a.g + static_cast<long>(k) * a.ld;
  const T mu = static_cast<T>(a.mu);
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.ld; i += stride) {
    if (i >= a.d) {
      g[i] = T(0);
      continue;
    }
    T grad = add_(T(0), mul_(mu, sub_(w[i], a.wstar[i])));
    if (a.scale > 0.0) {
      const double n = __dmul_rn(a.scale, gaussian_at(a.s0[k], static_cast<uint64_t>(i)));
      grad = add_(grad, static_cast<T>(n));
    }
    g[i] = grad;
  }
}

// Gaussian fill of one row (w* or the init direction u), in double.
static __global__ void gaussian_fill_kernel(double* out, long d, uint64_t s0) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d; i += stride) {
    out[i] = gaussian_at(s0, static_cast<uint64_t>(i));
  }
}

// Sum of squares in a fixed order: per thread a strided sum, a warp
// butterfly, the warps in order into partial[blockIdx.x]; sumsq_finish adds
// the block partials in block order.  The same grid always gives the same
// bits (every rank of a multi-GPU run computes the same start row).
static __global__ void sumsq_kernel(const double* x, long d, double* partial) {
  __shared__ double part[kThreads / 32];
  double acc = 0.0;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d; i += stride) {
    acc = __dadd_rn(acc, __dmul_rn(x[i], x[i]));
  }
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s = __dadd_rn(s, part[i]);
    partial[blockIdx.x] = s;
  }
}

static __global__ void sumsq_finish(const double* partial, int n, double* out) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, partial[i]);
  *out = s;
}

// w*_T = T(w*), row_T = T(w* + r * (u / |u|)) (problems.cpp:106-113,161-165)
template <typename T>
__global__ void compose_init_kernel(const double* wstar, const double* u, const double* sumsq, long d,
                                    long ld, double r, T* wstar_out, T* row_out) {
  const double n = __dsqrt_rn(*sumsq);
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < ld; i += stride) {
    if (i < d) {
      wstar_out[i] = static_cast<T>(wstar[i]);
      row_out[i] = static_cast<T>(__dadd_rn(wstar[i], __dmul_rn(r, __ddiv_rn(u[i], n))));
    } else {
      wstar_out[i] = T(0);
      row_out[i] = T(0);
    }
  }
}

// full_loss of the isotropic quadratic per row (problems.cpp:195-200 with
// A = mu*I): 0.5 * sum_i (w_i - w*_i) * (mu * (w_i - w*_i)), accumulated in
// fp64 (a parallel sum: tolerance parity, not order-exact).  blockIdx.y =
// row; out[row] += block partial.
template <typename T>
__global__ void quad_loss_kernel(const T* const* rows, const T* wstar, long d, double mu, double* out) {
  __shared__ double part[kThreads / 32];
  const T* w = rows[blockIdx.y];
  double acc = 0.0;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d; i += stride) {
    const double diff = static_cast<double>(w[i]) - static_cast<double>(wstar[i]);
    acc += diff * (mu * diff);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += part[i];
    atomicAdd(out + blockIdx.y, 0.5 * s);
  }
}

// The same loss in the reference's exact operation order (problems.cpp:
// 195-200: diff = w - w*, matvec(mu*I) = mu*diff, dot sequential from 0.0,
// times 0.5): one thread per row walks i ascending.  Bit-exact with the
// reference; meant for traces and metrics files, not for huge d.
template <typename T>
__global__ void quad_loss_exact_kernel(const T* const* rows, const T* wstar, long d, double mu, double* out) {
  if (threadIdx.x != 0) return;
  const T* w = rows[blockIdx.x];
  double acc = 0.0;
  for (long i = 0; i < d; ++i) {
    const double diff = __dsub_rn(static_cast<double>(w[i]), static_cast<double>(wstar[i]));
    acc = __dadd_rn(acc, __dmul_rn(diff, __dadd_rn(0.0, __dmul_rn(mu, diff))));
  }
  out[blockIdx.x] = __dmul_rn(0.5, acc);
}

// fold_running_stats (sync.cpp:193-201): rs = 0.9 * rs + 0.1 * obs, the
// constants rounded once to T.
template <typename T>
__global__ void stats_ema_kernel(T* rs, const T* obs, long n) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  const T a = static_cast<T>(0.9), b = static_cast<T>(0.1);
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    rs[i] = add_(mul_(a, rs[i]), mul_(b, obs[i]));
  }
}

template <typename T>
__global__ void broadcast_row_kernel(T* base, long ld, int rows, const T* src) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  const long n = ld * rows;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    base[i] = src[i % ld];
  }
}

// One CTA per local worker.  All margins first (thread b: z_b summed in the
// reference's feature order, then -y_b * sigmoid(-y_b z_b)), then every
// feature's gradient sum in example order (thread j): the reference's
// additions in the reference's order (problems.cpp:273-289), with a
// critical path of d + B steps.  Dynamic shared memory: w as doubles [d],
// the -y*s factors [B], and a reduction scratch.
template <typename T>
__global__ void __launch_bounds__(128) logistic_grad_kernel(const LogisticArgs a, const T* __restrict__ w,
                                                            T* __restrict__ g) {
  extern __shared__ double sh[];
  __shared__ double red_max[4];
  __shared__ int red_nan;
  const int k = blockIdx.x;
  const int d = a.d;
  double* wd = sh;
  double* ys = sh + d;
  const T* wr = w + static_cast<long>(k) * a.ld;
  if (threadIdx.x == 0) red_nan = 0;
  sample_batch_par(a, k, threadIdx.x, blockDim.x, [] { __syncthreads(); },
                   [](bool p) { return __syncthreads_or(p) != 0; });
  for (int j = threadIdx.x; j < d; j += blockDim.x) wd[j] = static_cast<double>(wr[j]);
  __syncthreads();
  const int* bt = a.batch + static_cast<long>(k) * a.B;
  double max_nz = 0.0;
  bool nan_nz = false;
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
    const int idx = bt[b];
    const double* x = a.x + static_cast<long>(idx) * d;
    double z = 0.0;
    for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(x[j], wd[j]));
    const double y = a.y[idx];
    const double nz = __dmul_rn(-y, z);
    ys[b] = __dmul_rn(-y, __ddiv_rn(1.0, __dadd_rn(1.0, exp(-nz))));  // sigmoid (problems.cpp:337)
    max_nz = fmax(max_nz, nz);
    nan_nz = nan_nz || isnan(nz);
  }
  for (int off = 16; off > 0; off >>= 1) max_nz = fmax(max_nz, __shfl_xor_sync(0xffffffffu, max_nz, off));
  if ((threadIdx.x & 31) == 0) red_max[threadIdx.x >> 5] = max_nz;
  if (nan_nz) red_nan = 1;
  __syncthreads();
  const double inv = __ddiv_rn(1.0, static_cast<double>(a.B));
  bool bad = false;
  T* gr = g + static_cast<long>(k) * a.ld;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < a.B; ++b) acc = __dadd_rn(acc, __dmul_rn(ys[b], a.x[static_cast<long>(bt[b]) * d + j]));
    double v = __dmul_rn(acc, inv);
    if (a.l2 > 0.0) v = __dadd_rn(v, __dmul_rn(a.l2, wd[j]));
    bad = bad || !isfinite(v);
    gr[j] = static_cast<T>(v);
  }
  for (long j = d + threadIdx.x; j < a.ld; j += blockDim.x) gr[j] = T(0);
  if (threadIdx.x == 0) {
    double m = red_max[0];
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) m = fmax(m, red_max[i]);
    bad = bad || !logistic_loss_finite(a, bt, wr, m, red_nan != 0);
  }
  // checked_gradient (sync.cpp:181-191): DivergenceError(rank, t)
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    atomicMin(a.gerr, (static_cast<unsigned long long>(a.t) << 32) | static_cast<unsigned int>(a.rank_of[k]));
  }
}

// LogisticProblem::full_loss (problems.cpp:292-305) of local row blockIdx.x:
// mean softplus(-y z) + 0.5 * l2 * |w|^2.  exact = 1: one thread in the
// reference's order (libdevice exp/log1p: tolerance, not bit-exact);
// exact = 0: a parallel fp64 reduction over the examples.
template <typename T>
__global__ void __launch_bounds__(kThreads) logistic_loss_kernel(const T* w, long ld, const double* x, const double* y,
                                                                 int d, int M, double l2, int exact, double* out) {
  __shared__ double part[kThreads / 32];
  const T* wr = w + static_cast<long>(blockIdx.x) * ld;
  double acc = 0.0;
  if (exact) {
    if (threadIdx.x != 0) return;
    for (int i = 0; i < M; ++i) {
      const double* xi = x + static_cast<long>(i) * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(xi[j], static_cast<double>(wr[j])));
      acc = __dadd_rn(acc, softplus_dev(__dmul_rn(-y[i], z)));
    }
  } else {
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      const double* xi = x + static_cast<long>(i) * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(xi[j], static_cast<double>(wr[j])));
      acc += softplus_dev(__dmul_rn(-y[i], z));
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    acc = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) acc += part[i];
  }
  acc = __ddiv_rn(acc, static_cast<double>(M));
  if (l2 > 0.0) {
    double dd = 0.0;
    for (int j = 0; j < d; ++j) dd = __dadd_rn(dd, __dmul_rn(static_cast<double>(wr[j]), static_cast<double>(wr[j])));
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(0.5, l2), dd));
  }
  out[blockIdx.x] = acc;
}

// TinyMlpProblem::stochastic_gradient (problems.cpp:478-503) of local
// worker blockIdx.x: one hidden tanh layer, scalar output, squared loss.
// Params [W1 (h x d) | b1 (h) | w2 (h) | b2]; the observation is the mean
// hidden pre-activation (the running-stats input, sync.cpp:193-201).  As
// for the logistic kernel, every example's forward pass is computed first
// (thread per (example, unit): z summed in the reference's feature order,
// then thread per example: the output summed in unit order), then every
// gradient element's sum over the examples is taken in example order --
// the reference's additions in the reference's order.  Dynamic shared
// memory: w as doubles [dim], z / tanh(z) / dz [B][h], err [B].
template <typename T>
__global__ void __launch_bounds__(128) mlp_grad_kernel(const LogisticArgs a, const T* __restrict__ w,
                                                       T* __restrict__ g, T* __restrict__ obs) {
  extern __shared__ double sh[];
  const int k = blockIdx.x;
  const int d = a.d, h = a.hidden, B = a.B;
  const long dim = static_cast<long>(h) * d + 2 * h + 1;
  double* wd = sh;
  double* zs = wd + dim;
  double* as = zs + static_cast<long>(B) * h;
  double* dz = as + static_cast<long>(B) * h;
  double* er = dz + static_cast<long>(B) * h;
  const T* wr = w + static_cast<long>(k) * a.ld;
  sample_batch_par(a, k, threadIdx.x, blockDim.x, [] { __syncthreads(); },
                   [](bool p) { return __syncthreads_or(p) != 0; });
  for (long e = threadIdx.x; e < dim; e += blockDim.x) wd[e] = static_cast<double>(wr[e]);
  __syncthreads();
  const int* bt = a.batch + static_cast<long>(k) * B;
  const long hd = static_cast<long>(h) * d;
  // forward, hidden layer: z_i = b1_i + sum_j W1_ij x_j (problems.cpp:550-556)
  for (long u = threadIdx.x; u < static_cast<long>(B) * h; u += blockDim.x) {
    const int b = static_cast<int>(u / h), i = static_cast<int>(u % h);
    const double* x = a.x + static_cast<long>(bt[b]) * d;
    double z = wd[hd + i];
    for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(wd[static_cast<long>(i) * d + j], x[j]));
    zs[u] = z;
    as[u] = tanh(z);
  }
  __syncthreads();
  // output and error: out = b2 + sum_i w2_i a_i; err = out - y
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    double out = wd[hd + 2 * h];
    for (int i = 0; i < h; ++i) out = __dadd_rn(out, __dmul_rn(wd[hd + h + i], as[static_cast<long>(b) * h + i]));
    er[b] = __dsub_rn(out, a.y[bt[b]]);
  }
  __syncthreads();
  // dz = err * w2_i * (1 - a_i^2)
  for (long u = threadIdx.x; u < static_cast<long>(B) * h; u += blockDim.x) {
    const int b = static_cast<int>(u / h), i = static_cast<int>(u % h);
    dz[u] = __dmul_rn(__dmul_rn(er[b], wd[hd + h + i]), __dsub_rn(1.0, __dmul_rn(as[u], as[u])));
  }
  __syncthreads();
  const double inv = __ddiv_rn(1.0, static_cast<double>(B));
  bool bad = false;
  T* gr = g + static_cast<long>(k) * a.ld;
  for (long e = threadIdx.x; e < dim; e += blockDim.x) {
    double acc = 0.0;
    if (e < hd) {  // W1_ij += dz_i x_j
      const int i = static_cast<int>(e / d), j = static_cast<int>(e % d);
      for (int b = 0; b < B; ++b) {
        acc = __dadd_rn(acc, __dmul_rn(dz[static_cast<long>(b) * h + i], a.x[static_cast<long>(bt[b]) * d + j]));
      }
    } else if (e < hd + h) {  // b1_i += dz_i
      const int i = static_cast<int>(e - hd);
      for (int b = 0; b < B; ++b) acc = __dadd_rn(acc, dz[static_cast<long>(b) * h + i]);
    } else if (e < hd + 2 * h) {  // w2_i += err a_i
      const int i = static_cast<int>(e - hd - h);
      for (int b = 0; b < B; ++b) acc = __dadd_rn(acc, __dmul_rn(er[b], as[static_cast<long>(b) * h + i]));
    } else {  // b2 += err
      for (int b = 0; b < B; ++b) acc = __dadd_rn(acc, er[b]);
    }
    const double v = __dmul_rn(acc, inv);
    bad = bad || !isfinite(v);
    gr[e] = static_cast<T>(v);
  }
  for (long e = dim + threadIdx.x; e < a.ld; e += blockDim.x) gr[e] = T(0);
  for (int i = threadIdx.x; i < h; i += blockDim.x) {  // observation: mean pre-activation
    double acc = 0.0;
    for (int b = 0; b < B; ++b) acc = __dadd_rn(acc, zs[static_cast<long>(b) * h + i]);
    obs[static_cast<long>(k) * a.obs_ld + i] = static_cast<T>(__dmul_rn(acc, inv));
  }
  if (threadIdx.x == 0) {  // the batch loss, for checked_gradient (sync.cpp:186)
    double loss = 0.0;
    for (int b = 0; b < B; ++b) loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(0.5, er[b]), er[b]));
    bad = bad || !isfinite(__dmul_rn(loss, inv));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    atomicMin(a.gerr, (static_cast<unsigned long long>(a.t) << 32) | static_cast<unsigned int>(a.rank_of[k]));
  }
}

// TinyMlpProblem::full_loss (problems.cpp:516-526) of local row blockIdx.x:
// mean 0.5 * err^2 over the dataset.  exact = 1: one thread in the
// reference's order; exact = 0: a parallel reduction over the examples.
template <typename T>
__global__ void __launch_bounds__(kThreads) mlp_loss_kernel(const T* w, long ld, const double* x, const double* y,
                                                            int d, int h, int M, int exact, double* out) {
  __shared__ double part[kThreads / 32];
  const T* wr = w + static_cast<long>(blockIdx.x) * ld;
  const long hd = static_cast<long>(h) * d;
  auto err_of = [&](int m) {
    const double* xi = x + static_cast<long>(m) * d;
    double o = static_cast<double>(wr[hd + 2 * h]);
    for (int i = 0; i < h; ++i) {
      double z = static_cast<double>(wr[hd + i]);
      for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(static_cast<double>(wr[static_cast<long>(i) * d + j]), xi[j]));
      o = __dadd_rn(o, __dmul_rn(static_cast<double>(wr[hd + h + i]), tanh(z)));
    }
    return __dsub_rn(o, y[m]);
  };
  double acc = 0.0;
  if (exact) {
    if (threadIdx.x != 0) return;
    for (int m = 0; m < M; ++m) {
      const double e = err_of(m);
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(0.5, e), e));
    }
  } else {
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
      const double e = err_of(m);
      acc += 0.5 * e * e;
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x != 0) return;
    acc = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) acc += part[i];
  }
  out[blockIdx.x] = __ddiv_rn(acc, static_cast<double>(M));
}

}  // namespace dssb
