// Host-side context of the C ABI (include/dssync_b200.h): the per-GPU
// device state (struct dss_ctx), the launch tables built from the schedule,
// and the helpers shared by the engine (engine.cu: plans, launches, the
// iteration flow) and the entry points (dssync_b200.cu, problems_abi.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

#include <nvtx3/nvToolsExt.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "dssync_b200.h"
#include "kernels.cuh"
#include "problems.hpp"
#include "schedule.hpp"

#ifndef DSS_CHAIN_LAZY_MEAN
#define DSS_CHAIN_LAZY_MEAN 1
#endif

namespace dssb {


extern thread_local std::string g_last_global_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PeerError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

inline uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Rng::for_stream (rng.cpp:20-26): the state the stream starts from.
inline uint64_t stream_state(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t iteration) {
  uint64_t s = mix64_host(seed + 0x9e3779b97f4a7c15ULL);
  s = mix64_host(s ^ purpose);
  s = mix64_host(s ^ rank);
  s = mix64_host(s ^ iteration);
  return s;
}

constexpr uint64_t kDataGen = 0x9e3779b97f4a7c15ULL;        // rng.hpp:40
constexpr uint64_t kInitParams = 0xbf58476d1ce4e5b9ULL;     // rng.hpp:41
constexpr uint64_t kGradientNoise = 0xa0761d6478bd642fULL;  // rng.hpp:44

inline const char* collective_name(int topology) {
  switch (topology) {
    case DSS_TREE: return "tree_allreduce_avg";
    case DSS_PS: return "ps_allreduce_avg";
    default: return "ring_allreduce_avg";
  }
}

// Device CSR table of groups for one launch of ds_group_kernel.
struct GroupLaunch {
  int size = 0;     // uniform group size of this launch (0 = mixed)
  int groups = 0;
  int* d_members = nullptr;
  int* d_offsets = nullptr;
  std::vector<int> members;  // host copy (slots, group after group)
};

struct FoldLaunch {
  int entries = 0;
  int uniform_m = 0;  // src count if uniform, else 0
  long max_len = 0;   // longest slice (elements)
  FoldEntry* d_entries = nullptr;
  void** d_src = nullptr;
  void** d_dst = nullptr;
};

struct ChainLaunch {
  int na = 0, nb = 0;              // kernel A / kernel B entries on this GPU
  ChainEntry* d_a = nullptr;
  ChainEntry* d_b = nullptr;
  void** d_src = nullptr;          // member rows
  void** d_dst = nullptr;          // mean destinations
  int* d_src_lr = nullptr;         // local row index of each member
  int* d_dst_lr = nullptr;         // local row index of each destination
  int opt_mem = -1;                // fused step on the members (DS), kOptNone = fold only
  int opt_dst = -1;                // fused step of the destinations with the mean (BSP)
  std::vector<ChainEntry> hb;      // host copies of the kernel B entries and destinations
  std::vector<void*> hdst;
};

// Deferred chain mean pass (DSS_CHAIN_LAZY_MEAN): a stage-0 GPU of two-GPU
// chains skips kernel B (copying the mean that arrived in place into its
// other members' rows) when the next parity's groups are all local; that
// step's fused kernel waits for the mean chunks and reads every aliased
// member's params from the row the mean arrived in.
struct LazyPlan {
  bool ok = false;
  int nf = 0;
  const unsigned long long* flags[4] = {};  // kernel B entries' receive flags (chunk-indexed)
  int alias[8] = {};                         // local row -> row holding its params
  int rows[8] = {};                          // next parity's group members (local rows), group after group
  int nr = 0, m = 0;
};

struct PushLaunch {
  bool oneshot = false;
  bool bsp = false;                // one-shot BSP: push gradients, fold, step the replicas
  int* d_dst_lr = nullptr;         // BSP: local row of each dst
  int items = 0, folds = 0;
  void** d_item_dst = nullptr;
  unsigned long long** d_item_flag = nullptr;
  int* d_item_gpu = nullptr;       // one-shot: destination GPU of each item_dst entry
  PushItem* d_items = nullptr;
  PushFold* d_folds = nullptr;
  void** d_dst = nullptr;
};

struct ParityPlan {
  PushLaunch push;                     // fused two-shot (DS step, one member per GPU)
  bool any_push = false;               // identical on every GPU
  bool built = false;
  bool any_spanning = false;  // identical on every GPU
  bool any_twoshot = false;   // identical on every GPU
  bool any_chain = false;     // identical on every GPU
  std::vector<GroupLaunch> local;      // fused step+fold launches
  GroupLaunch spanning_step;           // singleton in-place steps of spanning members
  FoldLaunch fold;                     // owned two-shot slices
  ChainLaunch chain;                   // ordered chain-fold groups
};

}  // namespace dssb

struct dss_ctx {
  dss_config cfg{};
  int P = 0;            // local workers
  int first = 0;        // first SLOT here (slot = gpu * P + local row)
  // worker placement: slot of every global rank and its inverse (identity for
  // contiguous packing); every plan and kernel table works in slots, error
  // keys carry global ranks (rank_of: local row -> global rank on the device)
  std::vector<int> slot_of, rank_of_slot;
  bool placed = false;
  int tile_gr = 0, tile_gc = 0;
  int* d_rank_of = nullptr;
  long d = 0, d_pad = 0;
  int esz = 4;
  int sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;

  void* w = nullptr;
  void* g = nullptr;
  void* m1 = nullptr;
  void* m2 = nullptr;
  void* mg = nullptr;     // mean gradient row (BSP over several GPUs)
  void* stats = nullptr;      // [P][s_pad] running statistics
  void* stats_obs = nullptr;  // [P][s_pad] batch observations
  long s = 0, s_pad = 0;
  std::vector<void*> peer_stats;
  void* wstar = nullptr;  // quadratic optimum row
  unsigned long long* d_err = nullptr;
  unsigned long long* d_gerr = nullptr;  // gradient-producer failures: t << 32 | rank
  unsigned long long* d_timeout = nullptr;
  unsigned long long* flags = nullptr;  // [G] barrier words, written by peers
  unsigned long long** d_peer_flags = nullptr;
  unsigned long long* h_err = nullptr;  // pinned readback

  // chain fold: receive rows [2 (partial, mean)][slots][d_pad] and their
  // per-chunk epoch flags [2][slots][n_chunks], both peer-mapped
  void* chain_buf = nullptr;
  unsigned long long* chain_flags = nullptr;
  int chain_slots = 0;
  long chain_chunk = 0, chain_nchunks = 0;
  unsigned long long chain_epoch = 0;
  std::vector<void*> peer_chain_buf;
  std::vector<unsigned long long*> peer_chain_flags;
  // fused two-shot staging: each GPU's owned slices, S rows each, + flags
  void* push_buf = nullptr;
  unsigned long long* push_flags = nullptr;
  std::vector<void*> peer_push_buf;
  std::vector<unsigned long long*> peer_push_flags;
  int push_occupancy = 0;
  // one-shot area after the two-shot staging: [B][P][R][d_pad] rows +
  // [B][P][R][n_chunks] flags (R = oneshot_rows, B = DSS_ONESHOT_BUFFERS),
  // rotated by the one-shot launch count
  bool oneshot[2] = {false, false};  // per schedule parity (same on every GPU)
  long oneshot_base_elems = 0, oneshot_base_flags = 0;
  long oneshot_half_elems = 0, oneshot_half_flags = 0;
  long oneshot_rows = 0;  // staging rows per group slot: the largest group size
  long oneshot_ack_off = 0;  // push_flags offset of the [G] acks (same on every GPU)
  unsigned long long** d_oneshot_ack_peer = nullptr;  // [G] peers' ack arrays
  unsigned long long oneshot_seq = 0;
  // dss_step_host pipeline
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_in = nullptr, ev_free = nullptr, ev_snap = nullptr, ev_out = nullptr;
  void* snapshot = nullptr;
  bool host_pipe = false;

  std::vector<long> step_count;
  std::vector<void*> peer_w, peer_g, peer_mg;
  std::vector<unsigned long long*> peer_flag;
  std::vector<void*> opened;  // IPC mappings to close
  bool attached = false;
  unsigned long long epoch = 0;
  bool pending_remote = false;
  bool chain_split = false;         // DS chains: per-parity partial rows and flags (see dss_step)
  bool pending_chain_only = false;  // the pending remote work is DS step chains only
  unsigned long long xgpu_ops = 0;           // cross-GPU launches so far (barrier, fold, push, chain)
  unsigned long long bsp_chain_mark = ~0ull; // xgpu_ops right after the last chain-only BSP step
  // split barrier after DS two-shot push steps (DSS_PUSH_SPLIT_BARRIER):
  // the push kernel arrives (barrier words <- epoch) and the next DS step's
  // first kernel waits, in place of a barrier launch between the steps
  unsigned long long split_mark = ~0ull;  // xgpu_ops right after an arriving push
  unsigned long long wait_epoch = 0;      // pending wait for the next launch (0: none)
  unsigned* d_arrive_count = nullptr;     // the push kernel's CTA counter
  dssb::LazyPlan lazy_plan[2];            // [chain parity]: its deferred mean pass, consumed at the other parity
  std::function<void()> lazy_b;           // the deferred kernel B launch (empty: none pending)
  unsigned long long lazy_epoch = 0;
  int lazy_parity = -1;                   // parity whose step consumes it
  bool lazy_consume = false;              // set by dss_step around guard(): do not flush on entry
  bool defer_b = false;                   // the next chain launch defers its kernel B
  bool allow_defer = false;               // dss_steps: another step of the same call follows
  bool arrive_next_push = false;          // the next push launch arrives

  dssb::ParityPlan step_plan[2];   // DS (or BSP at [0])
  dssb::ParityPlan sync_plan[2];   // sync_round (no step)
  dssb::ParityPlan mean_plan;      // ordered fold of every worker's params into mg (trace)
  dssb::ParityPlan stats_plan[2];  // running-stats fold per parity (DS) / world group at [0] (BSP)
  double* d_loss = nullptr;  // [P + 1] loss accumulators (trace)
  void** d_loss_rows = nullptr;  // [P + 1] rows the trace losses read: local params, then mg

  // logistic problem on the device (dss_logistic_setup)
  struct {
    bool ready = false;
    double* x = nullptr;       // [M][d]
    double* y = nullptr;       // [M]
    int* shard = nullptr;      // local shards, concatenated
    int* shard_off = nullptr;  // [P + 1]
    int* order = nullptr;      // [P][max_shard]
    long* order_epoch = nullptr;
    int* batch = nullptr;      // [P][B]
    long max_shard = 0;
    int M = 0, B = 0, sampling = 0;
    int d_feat = 0;            // features per example (logistic: dim)
    int hidden = 0;            // tiny MLP hidden units (0: logistic)
    double l2 = 0.0;
    uint64_t seed = 0;
    std::vector<void*> mem;
  } logi;                      // the dataset problem (logistic or tiny MLP)
  dssb::GroupLaunch apply_launch;  // singleton groups of every local worker

  // tiny-problem multi-iteration path (dss_steps)
  int* d_small_members[2] = {nullptr, nullptr};
  int* d_small_offsets[2] = {nullptr, nullptr};
  int small_ngroups[2] = {0, 0};
  double* d_small_buf = nullptr;  // [n] alphas, [n][P] bc1, [n][P] bc2
  unsigned* d_small_bar = nullptr;  // grid barrier of the persistent multi-CTA variant
  long small_cap = 0;
  std::vector<double> h_small;

  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending;
  std::vector<int> ev_kind;
  double kind_ms[DSS_KIND_COUNT] = {};
  long kind_n[DSS_KIND_COUNT] = {};
  std::vector<cudaEvent_t> ev_pool;
  long launches = 0;

  int last_status = DSS_OK;
  std::string last_error;
  int last_rank = -1;
  long last_iteration = -1;

  std::vector<void*> allocations;
  // guard bands (DSS_GUARD_BYTES, debug): every device allocation gets
  // `guard` bytes of 0xA5 on both sides, checked by dss_check_guards --
  // an out-of-bounds-write detector where compute-sanitizer is unavailable
  long guard = 0;
  std::vector<std::pair<char*, size_t>> guarded;  // (user pointer, user bytes)
  // single-device emulation of a G-GPU world (dss_emulate_*): every virtual
  // rank's context lives on one device and shares one stream; a step runs in
  // two passes over the ranks in order (pass 1: local steps, push phase 1,
  // chain partial pass; pass 2: push phase 2, pull folds, chain mean pass),
  // so every flag a kernel waits on was released by an earlier launch
  bool emulated = false;
  int emu_pass = 0;  // 0: normal (not emulating); 1 / 2: the pass being issued
};

namespace dssb {

inline int fail(dss_ctx* c, int status, const std::string& msg, int rank = -1, long it = -1) {
  if (c) {
    c->last_status = status;
    c->last_error = msg;
    c->last_rank = rank;
    c->last_iteration = it;
  }
  g_last_global_error = msg;
  return status;
}

void flush_lazy(dss_ctx* c);

// Every C-ABI entry point runs through guard: a deferred chain mean pass is
// launched first unless the call is the DS step that consumes it.
template <typename F>
int guard(dss_ctx* c, F&& f) {
  try {
    if (c) {
      if (c->lazy_b && !c->lazy_consume) flush_lazy(c);
      c->lazy_consume = false;
    }
    return f();
  } catch (const std::invalid_argument& e) {
    return fail(c, DSS_EINVAL, e.what());
  } catch (const CudaError& e) {
    return fail(c, DSS_ECUDA, e.what());
  } catch (const PeerError& e) {
    return fail(c, DSS_ENCCL, e.what());
  } catch (const std::exception& e) {
    return fail(c, DSS_ERUNTIME, e.what());
  }
}

constexpr unsigned char kGuardByte = 0xA5;

inline void* dalloc(dss_ctx* c, size_t bytes) {
  void* p = nullptr;
  const size_t g = static_cast<size_t>(c->guard);
  ck(cudaMalloc(&p, bytes + 2 * g), "cudaMalloc");
  c->allocations.push_back(p);
  char* user = static_cast<char*>(p) + g;
  if (g) {
    ck(cudaMemsetAsync(p, kGuardByte, g, c->stream), "guard");
    ck(cudaMemsetAsync(user + bytes, kGuardByte, g, c->stream), "guard");
    c->guarded.push_back({user, bytes});
  }
  ck(cudaMemsetAsync(user, 0, bytes, c->stream), "cudaMemset");
  return user;
}

template <typename T>
T* upload_table(dss_ctx* c, const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* p = static_cast<T*>(dalloc(c, v.size() * sizeof(T)));
  ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream),
     "table upload");
  ck(cudaStreamSynchronize(c->stream), "table upload sync");
  return p;
}

inline bool multi(const dss_ctx* c) { return c->cfg.n_gpus > 1; }

// The schedule of iteration t in slot space (see dss_ctx::slot_of).
inline Partition part_at(const dss_ctx* c, long t) {
  Partition p = make_partition(c->cfg.strategy, t);
  return c->placed ? to_slots(p, c->slot_of) : p;
}
// Global rank of a slot (error keys and DivergenceError carry global ranks).
inline int grank(const dss_ctx* c, int slot) { return c->rank_of_slot[static_cast<size_t>(slot)]; }
inline bool force_fold(const dss_ctx* c) { return c->cfg.path == 1 && !multi(c); }
inline bool force_chain(const dss_ctx* c) { return c->cfg.path == 2 && multi(c); }
inline bool use_push(const dss_ctx* c) { return multi(c) && c->cfg.path != 3; }  // path 3: unfused pull two-shot (A/B)

struct OwnedSlot {
  int group;
  int S;
  long lo, hi;
  long stage_off;
  long flag_off;
  long nch;
};

struct RowGeom {
  void* base;
  long len;  // logical row length (dim or stats_dim)
  long ld;   // padded row stride
};

// ---- launch helpers ---------------------------------------------------------

// NVTX ranges (header-only NVTX3: a no-op unless a tool is attached) around
// every hot launch, named by kernel kind, and around each API iteration, so
// an nsys / ncu timeline shows the DS-Sync phases.  DSS_NVTX=0 removes them.
#ifndef DSS_NVTX
#define DSS_NVTX 1
#endif
inline const char* kind_name(int k) {
  static const char* names[DSS_KIND_COUNT] = {"dss:group", "dss:fold", "dss:bsp", "dss:barrier",
                                              "dss:gradient", "dss:chain", "dss:chain_mean"};
  return k >= 0 && k < DSS_KIND_COUNT ? names[k] : "dss:?";
}
struct NvtxRange {
  explicit NvtxRange(const char* name) {
    if (DSS_NVTX) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (DSS_NVTX) nvtxRangePop();
  }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct TimedLaunch {
  dss_ctx* c;
  int kind;
  cudaEvent_t b = nullptr, e = nullptr;
  NvtxRange range;
  TimedLaunch(dss_ctx* cc, int k) : c(cc), kind(k), range(kind_name(k)) {
    ++c->launches;
    if (!c->timing) return;
    for (cudaEvent_t* ev : {&b, &e}) {
      if (!c->ev_pool.empty()) {
        *ev = c->ev_pool.back();
        c->ev_pool.pop_back();
      } else {
        ck(cudaEventCreate(ev), "cudaEventCreate");
      }
    }
    ck(cudaEventRecord(b, c->stream), "cudaEventRecord");
  }
  ~TimedLaunch() {
    if (!c->timing) return;
    cudaEventRecord(e, c->stream);
    c->ev_pending.emplace_back(b, e);
    c->ev_kind.push_back(kind);
  }
};

inline int grid_x(const dss_ctx* c, long nvec, int ys) {
  const long want = static_cast<long>(c->sms) * (2048 / kThreads);
  long gx = (want + ys - 1) / ys;
  const long need = (nvec + kThreads - 1) / kThreads;
  gx = std::min(gx, need);
  return static_cast<int>(std::max(1L, std::min(gx, 65535L)));
}

template <typename T>
StepConsts<T> consts(const dss_ctx* c, double alpha) {
  const dss_hparams& h = c->cfg.hp;
  StepConsts<T> k;
  k.alpha = static_cast<T>(alpha);
  k.wd = static_cast<T>(h.weight_decay);
  k.mom = static_cast<T>(h.momentum);
  k.b1 = static_cast<T>(h.beta1);
  k.omb1 = static_cast<T>(1.0 - h.beta1);
  k.b2 = static_cast<T>(h.beta2);
  k.omb2 = static_cast<T>(1.0 - h.beta2);
  k.eps = static_cast<T>(h.epsilon);
  k.awd = static_cast<T>(alpha * h.weight_decay);
  return k;
}

template <typename Args>
void fill_bias(const dss_ctx* c, Args& a) {
  // only Adam / AdamW read the bias corrections; workers usually share one
  // step count, so pow() runs once per distinct count (host launch cost)
  if (c->cfg.optimizer != DSS_ADAM && c->cfg.optimizer != DSS_ADAMW) return;
  const dss_hparams& h = c->cfg.hp;
  long last = -1;
  double b1 = 0.0, b2 = 0.0;
  for (int k = 0; k < c->P; ++k) {
    const long sc = c->step_count[static_cast<size_t>(k)];
    if (sc != last) {
      const double t = static_cast<double>(sc + 1);
      b1 = 1.0 - std::pow(h.beta1, t);  // optim.cpp:76-77
      b2 = 1.0 - std::pow(h.beta2, t);  // optim.cpp:78
      last = sc;
    }
    a.bc1[k] = b1;
    a.bc2[k] = b2;
  }
}

// ---- engine (engine.cu) -----------------------------------------------------

GroupLaunch make_group_launch(dss_ctx* c, const std::vector<std::vector<int>>& groups);
std::vector<OwnedSlot> owned_layout(const dss_ctx* c, const Partition& part, int q, long chunk, long* stage_total,
                                    long* flag_total);
// All launch tables of the context (both schedule parities, sync rounds,
// the trace mean, running stats); after dss_ipc_attach on several GPUs.
void build_plans(dss_ctx* c);

void launch_groups_any(dss_ctx* c, const GroupLaunch& gl, int opt, long t, double alpha, const void* g, long g_ld,
                       int step_phase, int sync_phase = 1, void* rows = nullptr, long rows_ld = 0);
void launch_fold_any(dss_ctx* c, const FoldLaunch& fl, long t);
void launch_chain_any(dss_ctx* c, const ChainLaunch& cl, long t, double alpha = 0.0);
void launch_push_any(dss_ctx* c, const PushLaunch& pl, long t, double alpha);
template <typename T>
void launch_bsp(dss_ctx* c, long t, double alpha);

// Cross-GPU flag barrier (no-op on one GPU).
void barrier(dss_ctx* c);
// Barrier if peers may still be writing into our rows.
void quiesce(dss_ctx* c, bool allow_chain_skip = false);
void flush_wait(dss_ctx* c, unsigned long long epoch = 0);
dssb::LazyPlan build_lazy(dss_ctx* c, int p);
void launch_lazy_any(dss_ctx* c, const dssb::LazyPlan& lp, long t, double alpha);
void fold_stats(dss_ctx* c, long t, bool barrier_done);
void bump_steps(dss_ctx* c);
int check_impl(dss_ctx* c);
int check_rank(dss_ctx* c, int rank, int* lr);
RowGeom geom(dss_ctx* c, int buffer);

// Small worlds (engine.cu): whole iterations in one launch when every
// worker is on this GPU and all rows fit DSS_PERSIST_MAX_BYTES -- one CTA up
// to 32 KB, else a resident grid with a barrier between iterations;
// logistic = 1 (one CTA only) adds the device gradient phase
// (problems_abi.cu).
bool small_path(const dss_ctx* c, long n);
long small_bytes(const dss_ctx* c);
template <typename T>
void run_small(dss_ctx* c, long t0, long n, const double* alphas, bool logistic = false);

// Logistic problem state on the device (problems_abi.cu).
LogisticArgs logistic_args(dss_ctx* c, long t);
void free_logistic(dss_ctx* c);

}  // namespace dssb
