/*
 * dssync_b200.h — C-ABI of the B200-native DS-Sync (divide-and-shuffle
 * synchronization, arXiv 2007.03298) step.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * exposes it as free C++ functions in namespace dssync (static lib, no FFI):
 *
 *   make_partition  /root/reference/proj/include/dssync/schedule.hpp:37  (src/schedule.cpp:31-54)
 *   group_of        /root/reference/proj/include/dssync/schedule.hpp:40  (src/schedule.cpp:56-65)
 *   check_mixing    /root/reference/proj/include/dssync/schedule.hpp:45  (src/schedule.cpp:67-90)
 *   validate(World) /root/reference/proj/include/dssync/schedule.hpp:23  (src/schedule.cpp:8-24)
 *   validate(Strat) /root/reference/proj/include/dssync/sync.hpp:43      (src/sync.cpp:47-66)
 *   apply_step      /root/reference/proj/include/dssync/optim.hpp:51-52  (src/optim.cpp:46-98)
 *   sync_round      /root/reference/proj/include/dssync/sync.hpp:128-129 (src/sync.cpp:268-282)
 *   run_training DS branch  src/sync.cpp:347-374, BSP branch src/sync.cpp:375-428
 *   mean_of / ring|tree|ps_allreduce_avg  src/param.cpp:42-53, src/comm.cpp:78-289
 *   QuadraticProblem::stochastic_gradient (A = mu*I)  src/problems.cpp:134-136,173-193
 *
 * Everything here is plain C: opaque handle, C scalars, host pointers and
 * sizes.  No torch types.  Every entry point returns a dss_status; the text
 * of the last failure (same wording as the reference's exceptions) and, for
 * divergence, the (rank, iteration) pair the reference's DivergenceError
 * carries (errors.hpp:16-25) are available through dss_last_error().
 *
 * Product path only: there is no CPU fallback.  Device entry points fail
 * with DSS_ECUDA when no B200 is present.
 */
#ifndef DSSYNC_B200_H_
#define DSSYNC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (sync.cpp/schedule.cpp exceptions -> ints) ------------ */
typedef enum {
  DSS_OK = 0,
  DSS_EINVAL = 1,     /* std::invalid_argument (schedule.cpp:8-24, sync.cpp:47-66, comm.cpp:56-72) */
  DSS_EDIVERGED = 2,  /* dssync::DivergenceError(rank, iteration) (errors.hpp:16-25) */
  DSS_ECUDA = 3,      /* CUDA runtime failure / no device */
  DSS_ENCCL = 4,      /* peer/IPC failure on the multi-GPU path */
  DSS_ERUNTIME = 5    /* std::runtime_error outside the training loop (param.cpp:28-32) */
} dss_status;

/* ---- enums mirror the reference's enum classes, same ordinal order ------ */
typedef enum { DSS_VANILLA_SGD = 0, DSS_SGD_MOMENTUM = 1, DSS_ADAM = 2, DSS_ADAMW = 3 } dss_optimizer_kind; /* optim.hpp:11 */
typedef enum { DSS_BSP = 0, DSS_DS_SYNC = 1 } dss_strategy_kind;  /* sync.hpp:14 */
typedef enum { DSS_RING = 0, DSS_TREE = 1, DSS_PS = 2 } dss_topology; /* sync.hpp:15 */
typedef enum { DSS_F32 = 0, DSS_F64 = 1 } dss_dtype;
typedef enum { DSS_SAMPLING_REPLACEMENT = 0, DSS_SAMPLING_EPOCH = 1 } dss_sampling; /* sync.hpp SamplingMode */

/* Worker-major device buffers, [local_workers][d_pad]. */
typedef enum {
  DSS_BUF_PARAMS = 0,   /* WorkerState::params            (sync.hpp:57) */
  DSS_BUF_GRADS = 1,    /* GradSample::grad                (problems.hpp:31) */
  DSS_BUF_MOMENT1 = 2,  /* OptimizerState::first_moment    (optim.hpp:31) */
  DSS_BUF_MOMENT2 = 3,  /* OptimizerState::second_moment   (optim.hpp:32) */
  DSS_BUF_STATS = 4,    /* WorkerState::running_stats      (sync.hpp:58), rows of stats_dim */
  DSS_BUF_STATS_OBS = 5 /* GradSample::stats_observation   (problems.hpp:32), rows of stats_dim */
} dss_buffer;

/* OptimizerHyperparams (optim.hpp:16-23); alpha is passed per step. */
typedef struct {
  double momentum;
  double beta1;
  double beta2;
  double epsilon;
  double weight_decay;
} dss_hparams;

/* SyncStrategy (sync.hpp:34-39) + WorldConfig (schedule.hpp:17-20). */
typedef struct {
  int kind;         /* dss_strategy_kind */
  int topology;     /* dss_topology; the arithmetic is topology-independent (comm.hpp:71-74) */
  int world_size;   /* W */
  int group_size;   /* N */
  int num_servers;  /* ps only */
  int rectangular;  /* 0 = reference rules (W == N*N or W == N).  1 = builder extension
                       W = N*K: even t -> K blocks of N, odd t -> N combs of K.
                       Not part of the reference: parity there is pinned only by the oracle. */
} dss_strategy;

/* SyncRoundOutcome (sync.hpp:119-122). */
typedef struct {
  long critical_path_steps;
  long total_messages;
} dss_outcome;

/* Context configuration.  One context per process/GPU. */
typedef struct {
  dss_strategy strategy;
  int optimizer;        /* dss_optimizer_kind */
  dss_hparams hp;
  int dtype;            /* dss_dtype */
  long dim;             /* d, parameters per worker */
  int device;           /* CUDA ordinal */
  int rank;             /* this GPU's index among n_gpus (process rank) */
  int n_gpus;           /* G; world_size must be a multiple of G.  Workers are packed
                           contiguously: gpu(k) = k / (W/G) */
  int path;             /* 0 = auto (two-shot for groups with one member per GPU, ordered
                           chain fold when some GPU holds several members).
                           1 = (one GPU) route every multi-member group through the
                           two-shot kernels with virtual owners: exercises the multi-GPU
                           fold on a single device for parity tests.
                           2 = (several GPUs) every spanning group uses the chain fold.
                           3 = (several GPUs) two-shot groups use the unfused pull fold
                           (step, barrier, fold) instead of the fused push kernel.
                           4 = (several GPUs) as 0 but never one-shot.  Path 0 folds a
                           schedule parity one-shot (every member GPU gathers every
                           member row and folds it for its own members; no peer stores
                           into params, no next-iteration barrier) when its spanning
                           groups are pairs with one member per GPU, or rows are at
                           most 512 KiB.
                           Results are bit-identical on every path. */
  long stats_dim;       /* running_stats per worker (0 = none).  They travel with the
                           params (DS, sync_round) or the gradients (BSP) through the same
                           ordered group fold, without an optimizer step
                           (sync.cpp:203-213, 386-411). */
  int placement;        /* worker placement over the GPUs (DS-Sync, n_gpus > 1):
                           0 = contiguous packing, gpu(k) = k / (W/G).
                           1 = tiled: the K x N (block x comb) grid of W = N*K workers is
                           cut into gr x gc tiles, one per GPU, so blocks span gc GPUs
                           and combs gr GPUs; (gr, gc) minimises the cross-GPU rows of
                           the busier schedule parity (dss_placement).  Groups, fold
                           order and results are unchanged; only which GPU holds which
                           worker.  Ignored (contiguous) for BSP and single-group worlds.
                           2 = auto: the tiling where contiguous packing would leave an
                           ordered chain >= 3 GPUs deep (C3 / C4 on 4 GPUs) and rows
                           are past the one-shot size (512 KiB), else contiguous. */
} dss_config;

typedef struct dss_ctx dss_ctx;

/* ======================= host-only schedule (no GPU) ===================== */

/* validate(WorldConfig) (schedule.cpp:8-24); rectangular=1 accepts W % N == 0. */
int dss_validate_world(int world_size, int group_size, int rectangular);

/* validate(SyncStrategy) (sync.cpp:47-66). */
int dss_validate_strategy(const dss_strategy* s);

/* is_square_mode (schedule.cpp:26-29). Returns 1/0, or -1 on invalid input. */
int dss_is_square_mode(int world_size, int group_size);

/* make_partition (schedule.cpp:31-54) / partition_for (sync.cpp:131-141 when
 * kind == BSP).  Writes the groups as CSR: members[0..W) grouped, ascending
 * inside each group; offsets[0..n_groups]; *n_groups.  members must hold W
 * ints and offsets W+1 ints. */
int dss_partition(const dss_strategy* s, long t, int* members, int* offsets, int* n_groups);

/* group_of (schedule.cpp:56-65): members of rank's group, *count of them. */
int dss_group_of(const dss_strategy* s, long t, int rank, int* members, int* count);

/* check_mixing (schedule.cpp:67-90): 1 true, 0 false, <0 error status negated. */
int dss_check_mixing(const dss_strategy* s, long t);

/* Closed-form SyncRoundOutcome of one round at iteration t: max over groups
 * of the collective's serial steps, sum of its messages (comm.cpp:78-289:
 * ring 2m-1 / 2m-1, tree 3log2m / m*log2m + 2(m-1), ps 2m / 2*m*min(P, dim)). */
int dss_round_outcome(const dss_strategy* s, long t, long payload_dim, dss_outcome* out);

/* Worker placement: gpu_of[k] and row_of[k] (the local row on that GPU) for
 * every global rank k of a context created with this strategy, n_gpus,
 * placement mode (dss_config.placement), dim and dtype (auto mode keeps
 * rows of the one-shot size contiguous; dim = 0 ignores the row size);
 * *gr / *gc receive the tiling (0, 0 for contiguous packing).  Host only. */
int dss_placement(const dss_strategy* s, int n_gpus, int placement, long dim, int dtype, int* gpu_of, int* row_of,
                  int* gr, int* gc);

/* Multi-GPU plan for (strategy, t, n_gpus, rank): how many groups this GPU
 * folds locally, how many span GPUs, and the [lo, hi) element slice this GPU
 * owns in each spanning group (two-shot ownership).  Host-only, for tests. */
typedef struct {
  int local_groups;      /* groups whose members all live on this GPU */
  int spanning_groups;   /* groups with members on this GPU and on others */
  int owned_slices;      /* two-shot groups in which this GPU owns a non-empty slice */
  long owned_elems;      /* sum of owned slice lengths */
  int chain_groups;      /* spanning groups folded by the ordered chain (several members on a GPU) */
} dss_plan_summary;
int dss_plan(const dss_strategy* s, long t, long dim, int n_gpus, int rank,
             dss_plan_summary* out, long* slice_lo, long* slice_hi, int* slice_group, int max_slices);

/* ============================ device context ============================= */

int dss_create(const dss_config* cfg, dss_ctx** out);
int dss_destroy(dss_ctx* ctx);

/* Run all device work on exactly this stream (e.g. the caller's current
 * stream); NULL means the CUDA legacy default stream.  Contexts start on a
 * private non-blocking stream. */
int dss_set_stream(dss_ctx* ctx, void* cuda_stream);

/* First global rank hosted here and how many (P = W / n_gpus). */
int dss_local_workers(const dss_ctx* ctx, int* first_rank, int* count);
/* Global ranks of this GPU's workers in local-row order (count entries): the
 * row order of dss_upload_all / dss_download_all.  Contiguous packing gives
 * first_rank, first_rank + 1, ...; with the tiled placement first_rank is -1
 * and the ranks come from here. */
int dss_local_ranks(const dss_ctx* ctx, int* ranks);

/* Padded row length in elements (multiple of 64) and element size in bytes. */
long dss_row_stride(const dss_ctx* ctx);
int dss_elem_size(const dss_ctx* ctx);

/* Device address of a worker row (global rank hosted here), for zero-copy
 * interop (e.g. wrapping into a framework tensor for the NCCL baseline). */
int dss_device_ptr(dss_ctx* ctx, int buffer, int rank, void** out);

/* Host <-> device copies of one worker's row: n elements of the context's
 * dtype (n <= dim).  Stream-ordered; dss_download synchronizes. */
int dss_upload(dss_ctx* ctx, int buffer, int rank, const void* host, long n);
int dss_download(dss_ctx* ctx, int buffer, int rank, void* host, long n);

/* Whole-buffer copies for every local worker: host is [P][dim] contiguous.
 * Async w.r.t. the host when the host memory is pinned. */
int dss_upload_all(dss_ctx* ctx, int buffer, const void* host);
int dss_download_all(dss_ctx* ctx, int buffer, void* host);

/* Fill a buffer of every local worker with a copy of one host row. */
int dss_broadcast_row(dss_ctx* ctx, int buffer, const void* host_row);

/* OptimizerState::step_count per worker (optim.hpp:33).  Bias corrections
 * use 1 - pow(beta, step_count + 1) in double on the host (optim.cpp:76-78). */
int dss_set_step_count(dss_ctx* ctx, int rank, long step_count);
long dss_get_step_count(const dss_ctx* ctx, int rank);

/* ---- the hot path ---- */

/* One full iteration at t with learning rate alpha:
 *   DS-Sync: every worker apply_step(own w, own g) then every group averages
 *            its stepped params in ascending-rank order (sync.cpp:347-374),
 *            fused: each element is read once and written once.
 *   BSP:     the world averages gradients in ascending-rank order, then every
 *            worker apply_step(own w, mean g) (sync.cpp:375-428).
 * Non-finite results are latched on the device; they surface as
 * DSS_EDIVERGED from dss_check() (or from this call when check != 0). */
int dss_step(dss_ctx* ctx, long t, double alpha, int check, dss_outcome* out);

/* n consecutive iterations t0 .. t0+n-1 (alphas[i] for iteration t0+i) in
 * one call: the run_training loop body (sync.cpp:323-459, sync part) without
 * a host round trip per iteration.  On one GPU, small worlds run the whole
 * batch in one launch: one CTA up to 32 KB per array, a cooperative
 * resident grid with a barrier between iterations up to 16 workers and
 * 1 MB (DS) / 4 MB (BSP) per array.  Same bits as n dss_step calls. */
int dss_steps(dss_ctx* ctx, long t0, long n, const double* alphas, int check, dss_outcome* last);

/* One iteration fed from and returned to HOST memory, pipelined across
 * calls: host_grads ([local_workers][dim], pinned) is copied in on a copy
 * stream, the iteration runs, and the resulting params are snapshotted on
 * the device and copied out to host_params ([local_workers][dim], pinned) on
 * a second copy stream -- so iteration t's copy-out overlaps iteration t+1's
 * copy-in.  host_params of iteration t is complete once the next
 * dss_step_host or dss_host_sync returns; host_grads may be reused as soon
 * as the next call returns.  Collective on several GPUs (like dss_step). */
int dss_step_host(dss_ctx* ctx, long t, double alpha, const void* host_grads, void* host_params);
/* Wait for every outstanding dss_step_host copy. */
int dss_host_sync(dss_ctx* ctx);

/* sync_round (sync.cpp:268-282): group averaging only, no optimizer step.
 * Optimizer state untouched. */
int dss_sync_round(dss_ctx* ctx, long t, int check, dss_outcome* out);

/* apply_step (optim.cpp:46-98) for every local worker with its own gradient,
 * no averaging. */
int dss_apply_step(dss_ctx* ctx, double alpha, int check);

/* fold_running_stats (sync.cpp:193-201) for every local worker:
 * running_stats = 0.9 * running_stats + 0.1 * stats_observation (the
 * DSS_BUF_STATS_OBS rows).  Call it where the reference does: after the local
 * step's gradient (DS) / before the collective (BSP), i.e. before dss_step. */
int dss_running_stats_update(dss_ctx* ctx);

/* Synthetic gradients of the isotropic quadratic (problems.cpp:134-136,173-193):
 *   g_k = mu * (w_k - w*) + (sigma / sqrt(d)) * gaussian_i(seed, kGradientNoise, k, t)
 * with the reference's SplitMix64 stream (rng.cpp:20-51), counter-addressed. */
int dss_quadratic_gradients(dss_ctx* ctx, long t, uint64_t seed, double mu, double sigma);

/* w* = gaussians of stream (problem_seed, kDataGen, 1, 0) (problems.cpp:157-159)
 * and every worker's params = w* + sqrt(delta0) * u, u the normalised
 * gaussian vector of stream (problem_seed, kInitParams, 0, 0) (problems.cpp:161-165).
 * Device-generated at full size: tolerance-level parity with the reference
 * (the Box-Muller log/cos are libdevice's, and |u|^2 is a fixed-order tree
 * sum rather than the reference's sequential loop), but deterministic: the
 * same call gives the same bits on every run and every rank.  The bit-exact
 * host generator is dss_quadratic_problem. */
int dss_quadratic_init(dss_ctx* ctx, uint64_t problem_seed, double delta0);
/* Upload an explicit optimum w* (dim elements of the context dtype). */
int dss_set_optimum(dss_ctx* ctx, const void* host, long n);

/* ---- per-iteration trace (run_training post-round, sync.cpp:430-458) ---- */
/* global_mean_params = mean_of_ptrs over all W workers' params
 * (param.cpp:59-70): ascending fold x 1/W, bit-exact; dim elements of the
 * context dtype written to host_mean on every rank (collective on multi-GPU). */
int dss_global_mean(dss_ctx* ctx, void* host_mean);
/* post_sync_loss of every local worker, full_loss of the isotropic quadratic
 * 0.5 * sum_i (w_i - w*_i) * (mu * (w_i - w*_i)) (problems.cpp:195-200).
 * exact = 0: parallel fp64 device reduction (tolerance parity);
 * exact = 1: the reference's sequential operation order, bit-exact (one
 * thread per row: for traces / metrics files, not for huge d).
 * losses: local_workers doubles.  suboptimality (optional) = full_loss of the
 * row written by the last dss_global_mean (true_suboptimality, sync.cpp:585). */
int dss_quadratic_losses(dss_ctx* ctx, double mu, int exact, double* losses, double* suboptimality);

/* ---- logistic regression on the device (config C1 end to end) ----------- */
/* LogisticProblem's synthetic dataset (problems.cpp:230-250), host, bit-exact:
 * x: M*d doubles (row-major), y: M labels in {-1, +1}. */
int dss_logistic_dataset(uint64_t seed, int d, int M, double* x, double* y);
/* QuadraticProblem's optimum and start for A = mu*I (problems.cpp:157-165),
 * host, bit-exact: wstar, w0 = d doubles each (cf. dss_quadratic_init, the
 * device-side generator of these rows for huge d, equal within tolerance). */
int dss_quadratic_problem(uint64_t seed, int d, double delta0, double* wstar, double* w0);
/* LogisticProblem::finish_setup (problems.cpp:346-416), host, bit-exact:
 * the smoothness bound (power iteration on X^T X / 4M, + l2) and, when
 * l2 > 0, the damped-Newton optimum w_opt (d doubles, optional) and
 * f* = full_loss(w_opt) (NaN when l2 == 0: no optimum). */
int dss_logistic_constants(const double* x, const double* y, int M, int d, double l2, double* smoothness,
                           double* f_star, double* w_opt);
/* make_shards (problems.cpp:642-662), host, bit-exact: worker w owns
 * indices[offsets[w] .. offsets[w+1]) (indices: M ints, offsets: workers+1). */
int dss_make_shards(int dataset_size, int workers, uint64_t seed, int* indices, int* offsets);
/* epoch_order (problems.cpp:664-674), host, bit-exact: out = size ints. */
int dss_epoch_order(const int* shard, int size, uint64_t seed, int rank, long epoch, int* out);
/* Upload the dataset (x: M*dim doubles, y: M) and shard it over the world
 * with make_shards(M, world_size, run_seed) (sync.cpp:300); each iteration
 * then samples batch_size examples per worker on the device (sample_batch,
 * sync.cpp:153-179, DSS_SAMPLING_*) with the run seed's streams. */
int dss_logistic_setup(dss_ctx* ctx, const double* x, const double* y, int M, double l2, int batch_size,
                       int sampling, uint64_t run_seed);
/* Gradient rows of every local worker at iteration t: checked_gradient +
 * LogisticProblem::stochastic_gradient (sync.cpp:181-191, problems.cpp:265-290),
 * computed in fp64 from the worker's params and stored in the context dtype.
 * Batch indices are bit-exact; the gradient is within libdevice-vs-glibc exp
 * rounding of the reference.  A non-finite gradient or batch loss latches
 * DivergenceError(rank, t, "non-finite stochastic gradient") (see dss_check). */
int dss_logistic_gradients(dss_ctx* ctx, long t);
/* n iterations of (dss_logistic_gradients(t), dss_step(t, alphas[i])). */
int dss_logistic_steps(dss_ctx* ctx, long t0, long n, const double* alphas, int check, dss_outcome* last);
/* ---- tiny MLP on the device (running statistics, acceptance.cpp:328-402) -- */
/* TinyMlpProblem's data (problems.cpp:436-460) and initial_params
 * (:466-476), host, bit-exact: x = M*d doubles, y = M targets; w = hidden*d
 * + 2*hidden + 1 doubles ([W1 | b1 | w2 | b2]). */
int dss_mlp_dataset(uint64_t seed, int d, int M, double* x, double* y);
int dss_mlp_initial_params(uint64_t seed, int d, int hidden, double* w);
/* Upload the MLP data and shard it as dss_logistic_setup does.  The context
 * needs dim = hidden*d + 2*hidden + 1 and stats_dim = hidden. */
int dss_mlp_setup(dss_ctx* ctx, const double* x, const double* y, int M, int d, int hidden, int batch_size,
                  int sampling, uint64_t run_seed);
/* Gradient rows (DSS_BUF_GRADS) and running-stat observations
 * (DSS_BUF_STATS_OBS: the mean hidden pre-activations) of every local
 * worker at iteration t (TinyMlpProblem::stochastic_gradient,
 * problems.cpp:478-503, via checked_gradient).  Follow with
 * dss_running_stats_update and dss_step, as run_training does. */
int dss_mlp_gradients(dss_ctx* ctx, long t);
/* TinyMlpProblem::full_loss (problems.cpp:516-526) of every local worker. */
int dss_mlp_losses(dss_ctx* ctx, int exact, double* losses);
/* Indices sampled by the last dss_logistic_gradients: [local_workers][batch]. */
int dss_logistic_batch(dss_ctx* ctx, int* out);
/* LogisticProblem::full_loss (problems.cpp:292-305) of every local worker:
 * exact = 1 in the reference's order (one thread per row), 0 parallel. */
int dss_logistic_losses(dss_ctx* ctx, int exact, double* losses);

/* Latched divergence check (synchronizes).  DSS_OK or DSS_EDIVERGED. */
int dss_check(dss_ctx* ctx);
/* Clear latched divergence flags. */
int dss_clear_error(dss_ctx* ctx);

/* Text of the last failure; *rank / *iteration are set for DSS_EDIVERGED
 * (else -1).  Returns the status of the last failure. */
int dss_last_error(const dss_ctx* ctx, char* buf, size_t len, int* rank, long* iteration);
/* Text of the last failure of a context-free call (schedule functions). */
int dss_last_global_error(char* buf, size_t len);

/* ---- per-kernel timing (CUDA events on the launching stream) ---- */
/* When enabled, every hot-path kernel launch is bracketed by events; the
 * totals over the launches since the last reset are returned. */
int dss_enable_timing(dss_ctx* ctx, int on);
int dss_kernel_times(dss_ctx* ctx, double* total_ms, long* launches, double* max_launch_ms);
/* Same events split by kernel kind: arrays of DSS_KIND_COUNT entries
 * (total ms, launches) since the last call to either timing query. */
enum {
  DSS_KIND_GROUP = 0,    /* ds_group_kernel: fused step + ordered fold (or in-place step) */
  DSS_KIND_FOLD = 1,     /* fold_kernel: two-shot ordered fold over NVLink peers */
  DSS_KIND_BSP = 2,      /* bsp_kernel: fused gradient fold + step */
  DSS_KIND_BARRIER = 3,  /* barrier_kernel: cross-GPU flag barrier */
  DSS_KIND_GRADIENT = 4, /* quad_grad_kernel: synthetic gradients */
  DSS_KIND_CHAIN = 5,    /* chain_partial_kernel: ordered chain fold, partial pass over NVLink */
  DSS_KIND_CHAIN_MEAN = 6, /* chain_mean_kernel: the chain's mean pass */
  DSS_KIND_COUNT = 7
};
int dss_kernel_times_by_kind(dss_ctx* ctx, double* total_ms, long* launches);
/* gpu_launches: hot-path kernels launched since creation (all kinds). */
long dss_launch_count(const dss_ctx* ctx);

/* ---- diagnostics ---- */
/* With DSS_GUARD_BYTES=n in the environment at dss_create, every device
 * allocation of the context carries n bytes (rounded up to 256) of 0xA5 on
 * both sides.  dss_check_guards synchronizes the context's stream and
 * counts overwritten guard bytes (*corrupted; DSS_ERUNTIME when nonzero):
 * an out-of-bounds-write check that needs no compute-sanitizer.  Without
 * the variable it checks nothing and returns DSS_OK. */
int dss_check_guards(dss_ctx* ctx, long* corrupted);

/* Single-device emulation of a G-GPU world (tests): n contexts created on
 * ONE device as ranks 0..n-1 of an n-GPU world (identical configuration)
 * are wired to each other's buffers directly and share one stream.
 * dss_emulate_step then runs one DS-Sync iteration of every rank in two
 * passes in rank order -- local steps, push phase 1 and the chain's partial
 * pass, then push phase 2, the pull folds and the chain's mean pass -- so
 * every cross-rank flag a kernel waits on was released by an earlier launch
 * on the stream (no concurrently spinning launches).  The kernels, tables
 * and flag protocol are the multi-GPU ones; results equal a real G-GPU run
 * bit for bit.  DS-Sync only. */
int dss_emulate_attach(dss_ctx** ctxs, int n);
int dss_emulate_step(dss_ctx** ctxs, int n, long t, double alpha, int check);

/* ---- multi-GPU (one process per GPU over NVLink/NVSwitch) ---- */
/* CUDA IPC handles of this GPU's params, grads, mean-gradient, barrier-flag,
 * chain-row, chain-flag, running-stats, push-staging and push-flag buffers
 * (9 x 64 B), then a 160-B layout fingerprint (dtype, dims, world,
 * optimizer, path, chain and one-shot geometry): DSS_IPC_BYTES bytes
 * written to out.  dss_ipc_attach fails with DSS_EINVAL when any rank's
 * fingerprint differs from this context's. */
#define DSS_IPC_BYTES 736
int dss_ipc_export(dss_ctx* ctx, void* out);
/* Map every GPU's exported handles (n_gpus * DSS_IPC_BYTES bytes, rank
 * order, own entry ignored).  Must be called on every rank before the first
 * multi-GPU dss_step.  Requires peer access between all GPUs. */
int dss_ipc_attach(dss_ctx* ctx, const void* all_handles);
/* Cross-GPU barrier over the flag buffers (also used by tests). */
int dss_barrier(dss_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* DSSYNC_B200_H_ */
