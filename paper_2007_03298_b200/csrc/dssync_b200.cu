// C-ABI implementation: device-resident worker state, the host driver of
// the DS-Sync / BSP iteration, and kernel dispatch.
//
// Host driver restates run_training's DS branch (sync.cpp:347-374), BSP
// branch (sync.cpp:375-428) and sync_round (sync.cpp:268-282) over
// device-resident worker-major buffers.  One context per GPU (process).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "dssync_b200.h"
#include "kernels.cuh"
#include "problems.hpp"
#include "schedule.hpp"

using namespace dssb;

namespace {

thread_local std::string g_last_global_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PeerError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Rng::for_stream (rng.cpp:20-26): the state the stream starts from.
uint64_t stream_state(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t iteration) {
  uint64_t s = mix64_host(seed + 0x9e3779b97f4a7c15ULL);
  s = mix64_host(s ^ purpose);
  s = mix64_host(s ^ rank);
  s = mix64_host(s ^ iteration);
  return s;
}

constexpr uint64_t kDataGen = 0x9e3779b97f4a7c15ULL;        // rng.hpp:40
constexpr uint64_t kInitParams = 0xbf58476d1ce4e5b9ULL;     // rng.hpp:41
constexpr uint64_t kGradientNoise = 0xa0761d6478bd642fULL;  // rng.hpp:44

const char* collective_name(int topology) {
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
};

struct PushLaunch {
  bool oneshot = false;
  int items = 0, folds = 0;
  void** d_item_dst = nullptr;
  unsigned long long** d_item_flag = nullptr;
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

}  // namespace

struct dss_ctx {
  dss_config cfg{};
  int P = 0;            // local workers
  int first = 0;        // first global rank here
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
  // one-shot (small rows): double-buffered staging [2][P][G][d_pad] + flags [2][P][G][n_chunks]
  // one-shot area after the two-shot staging: [2][P][G][d_pad] rows +
  // [2][P][G][n_chunks] flags, double-buffered by one-shot launch count
  bool oneshot[2] = {false, false};  // per schedule parity (same on every GPU)
  long oneshot_base_elems = 0, oneshot_base_flags = 0;
  long oneshot_half_elems = 0, oneshot_half_flags = 0;
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

  ParityPlan step_plan[2];   // DS (or BSP at [0])
  ParityPlan sync_plan[2];   // sync_round (no step)
  ParityPlan mean_plan;      // ordered fold of every worker's params into mg (trace)
  ParityPlan stats_plan[2];  // running-stats fold per parity (DS) / world group at [0] (BSP)
  double* d_loss = nullptr;  // [P + 1] loss accumulators (trace)

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
    double l2 = 0.0;
    uint64_t seed = 0;
    std::vector<void*> mem;
  } logi;
  GroupLaunch apply_launch;  // singleton groups of every local worker

  // tiny-problem multi-iteration path (dss_steps)
  int* d_small_members[2] = {nullptr, nullptr};
  int* d_small_offsets[2] = {nullptr, nullptr};
  int small_ngroups[2] = {0, 0};
  double* d_small_buf = nullptr;  // [n] alphas, [n][P] bc1, [n][P] bc2
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
};

namespace {

int fail(dss_ctx* c, int status, const std::string& msg, int rank = -1, long it = -1) {
  if (c) {
    c->last_status = status;
    c->last_error = msg;
    c->last_rank = rank;
    c->last_iteration = it;
  }
  g_last_global_error = msg;
  return status;
}

template <typename F>
int guard(dss_ctx* c, F&& f) {
  try {
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

void* dalloc(dss_ctx* c, size_t bytes) {
  void* p = nullptr;
  ck(cudaMalloc(&p, bytes), "cudaMalloc");
  ck(cudaMemsetAsync(p, 0, bytes, c->stream), "cudaMemset");
  c->allocations.push_back(p);
  return p;
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

GroupLaunch make_group_launch(dss_ctx* c, const std::vector<std::vector<int>>& groups) {
  GroupLaunch gl;
  if (groups.empty()) return gl;
  std::vector<int> members, offsets{0};
  gl.size = static_cast<int>(groups[0].size());
  for (const auto& g : groups) {
    if (static_cast<int>(g.size()) != gl.size) gl.size = 0;
    members.insert(members.end(), g.begin(), g.end());
    offsets.push_back(static_cast<int>(members.size()));
  }
  gl.groups = static_cast<int>(groups.size());
  gl.d_members = upload_table(c, members);
  gl.d_offsets = upload_table(c, offsets);
  return gl;
}

// Local-group launches bucketed by group size so each uses a templated,
// fully unrolled member loop.
std::vector<GroupLaunch> make_bucketed(dss_ctx* c, const std::vector<std::vector<int>>& groups) {
  std::vector<GroupLaunch> out;
  std::vector<int> sizes;
  for (const auto& g : groups) {
    if (std::find(sizes.begin(), sizes.end(), static_cast<int>(g.size())) == sizes.end()) {
      sizes.push_back(static_cast<int>(g.size()));
    }
  }
  for (int s : sizes) {
    std::vector<std::vector<int>> b;
    for (const auto& g : groups) {
      if (static_cast<int>(g.size()) == s) b.push_back(g);
    }
    out.push_back(make_group_launch(c, b));
  }
  return out;
}

bool multi(const dss_ctx* c) { return c->cfg.n_gpus > 1; }
bool force_fold(const dss_ctx* c) { return c->cfg.path == 1 && !multi(c); }

void* row_ptr(dss_ctx* c, const std::vector<void*>& bases, int rank) {
  const int gpu = rank / c->P;
  const int lr = rank - gpu * c->P;
  return static_cast<char*>(bases[static_cast<size_t>(gpu)]) +
         static_cast<size_t>(lr) * c->d_pad * c->esz;
}

// Row of a rank hosted on THIS GPU inside a local buffer.
void* row_ptr(dss_ctx* c, const std::vector<void*>&, int rank, void* local_base) {
  return static_cast<char*>(local_base) + static_cast<size_t>(rank - c->first) * c->d_pad * c->esz;
}

bool force_chain(const dss_ctx* c) { return c->cfg.path == 2 && multi(c); }
bool use_push(const dss_ctx* c) { return multi(c) && c->cfg.path != 3; }  // path 3: unfused pull two-shot (A/B)

// Staging layout of GPU q's owned two-shot slices at parity t: for each
// owned slice (plan order) its group, S, [lo, hi), element offset in q's
// staging buffer (S rows of hi-lo) and flag offset (S rows of n_chunks).
struct OwnedSlot {
  int group;
  int S;
  long lo, hi;
  long stage_off;
  long flag_off;
  long nch;
};
std::vector<OwnedSlot> owned_layout(const dss_ctx* c, const Partition& part, int q, long chunk,
                                    long* stage_total, long* flag_total) {
  const GpuPlan gp = make_plan(part, c->cfg.strategy.world_size, c->cfg.n_gpus, q, c->d_pad, force_chain(c));
  std::vector<OwnedSlot> out;
  long so = 0, fo = 0;
  for (const Slice& sl : gp.owned) {
    OwnedSlot o{};
    o.group = sl.group;
    std::vector<int> gpus;
    for (int j = 0; j < part.size(sl.group); ++j) {
      const int gpu = part.group(sl.group)[j] / c->P;
      if (gpus.empty() || gpus.back() != gpu) gpus.push_back(gpu);
    }
    o.S = static_cast<int>(gpus.size());
    o.lo = sl.lo;
    o.hi = sl.hi;
    o.nch = (sl.hi - sl.lo + chunk - 1) / chunk;
    o.stage_off = so;
    o.flag_off = fo;
    so += static_cast<long>(o.S) * (sl.hi - sl.lo);
    fo += static_cast<long>(o.S) * o.nch;
    out.push_back(o);
  }
  if (stage_total) *stage_total = so;
  if (flag_total) *flag_total = fo;
  return out;
}

void* chain_row(dss_ctx* c, void* base, int region, int slot) {
  return static_cast<char*>(base) +
         (static_cast<size_t>(region) * c->chain_slots + slot) * c->d_pad * c->esz;
}
unsigned long long* chain_flag(dss_ctx* c, unsigned long long* base, int region, int slot) {
  return base + (static_cast<size_t>(region) * c->chain_slots + slot) * c->chain_nchunks;
}

// Chain-fold launch tables for this GPU's roles.  members of role i are
// rows of `member_base` (local); its mean lands in dsts[i] (local rows).
ChainLaunch build_chain(dss_ctx* c, const std::vector<ChainRole>& roles, void* member_base,
                        const std::vector<std::vector<void*>>& dsts, int err_phase, int opt_mem = kOptNone,
                        int opt_dst = kOptNone, const std::vector<std::vector<int>>& dst_lrs = {}) {
  ChainLaunch cl;
  cl.opt_mem = opt_mem;
  cl.opt_dst = opt_dst;
  std::vector<ChainEntry> ea, eb;
  std::vector<void*> src, dst;
  std::vector<int> src_lr, dst_lr;
  for (size_t i = 0; i < roles.size(); ++i) {
    const ChainRole& r = roles[i];
    if (r.slot >= c->chain_slots || r.next_slot >= c->chain_slots || r.mean_next_slot >= c->chain_slots) {
      throw std::logic_error("chain slot out of range");
    }
    ChainEntry a{};
    a.stage = r.stage;
    a.last = r.stage == r.S - 1;
    a.run_beg = static_cast<int>(src.size());
    a.run_cnt = static_cast<int>(r.run.size());
    for (int k : r.run) {
      src.push_back(static_cast<char*>(member_base) + static_cast<size_t>(k - c->first) * c->d_pad * c->esz);
      src_lr.push_back(k - c->first);
    }
    a.dst_beg = static_cast<int>(dst.size());
    a.dst_cnt = static_cast<int>(dsts[i].size());
    dst.insert(dst.end(), dsts[i].begin(), dsts[i].end());
    for (size_t q = 0; q < dsts[i].size(); ++q) {
      dst_lr.push_back(i < dst_lrs.size() && q < dst_lrs[i].size() ? dst_lrs[i][q] : 0);
    }
    a.recv = chain_row(c, c->chain_buf, 0, r.slot);
    a.recv_flags = chain_flag(c, c->chain_flags, 0, r.slot);
    if (!a.last) {
      a.send = chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.next_gpu)], 0, r.next_slot);
      a.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.next_gpu)], 0, r.next_slot);
    } else {
      a.send = chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
      a.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
    }
    a.err_rank = r.first_member;
    a.err_phase = err_phase;
    a.m = r.m;
    ea.push_back(a);
    if (r.stage <= r.S - 2) {
      ChainEntry b = a;
      b.last = 0;
      b.recv = chain_row(c, c->chain_buf, 1, r.slot);
      b.recv_flags = chain_flag(c, c->chain_flags, 1, r.slot);
      if (r.stage < r.S - 2) {
        b.send = chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
        b.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
      } else {
        b.send = nullptr;
        b.send_flags = nullptr;
      }
      eb.push_back(b);
    }
  }
  cl.na = static_cast<int>(ea.size());
  cl.nb = static_cast<int>(eb.size());
  cl.d_a = upload_table(c, ea);
  cl.d_b = upload_table(c, eb);
  cl.d_src = upload_table(c, src);
  cl.d_dst = upload_table(c, dst);
  cl.d_src_lr = upload_table(c, src_lr);
  cl.d_dst_lr = upload_table(c, dst_lr);
  return cl;
}

// Fused two-shot tables of parity t for this GPU (one member per GPU in
// every two-shot group).
PushLaunch build_oneshot(dss_ctx* c, const Partition& part);

PushLaunch build_push(dss_ctx* c, const Partition& part, long t) {
  (void)t;
  if (c->oneshot[t & 1]) return build_oneshot(c, part);
  PushLaunch pl;
  const int G = c->cfg.n_gpus;
  const int me = c->cfg.rank;
  const long CH = c->chain_chunk;
  std::vector<std::vector<OwnedSlot>> lay(static_cast<size_t>(G));
  for (int q = 0; q < G; ++q) lay[static_cast<size_t>(q)] = owned_layout(c, part, q, CH, nullptr, nullptr);
  auto find_slot = [&](int q, int group) -> const OwnedSlot& {
    for (const OwnedSlot& o : lay[static_cast<size_t>(q)]) {
      if (o.group == group) return o;
    }
    throw std::logic_error("push: owner slot not found");
  };
  std::vector<PushItem> items;
  std::vector<void*> item_dst;
  std::vector<unsigned long long*> item_flag;
  std::vector<std::pair<long, long>> item_keys;  // (chunk-major, owner) order key, index
  std::vector<PushFold> folds;
  std::vector<void*> dst;
  const GpuPlan gp = make_plan(part, c->cfg.strategy.world_size, G, me, c->d_pad, force_chain(c));
  for (int gi : gp.spanning_groups) {
    bool chain = false;
    for (const ChainRole& r : gp.chain) chain = chain || r.group == gi;
    if (chain) continue;
    const int* mem = part.group(gi);
    const int m = part.size(gi);
    std::vector<int> gpus;
    int my_member = -1, j = -1;
    for (int q = 0; q < m; ++q) {
      const int gpu = mem[q] / c->P;
      if (gpus.empty() || gpus.back() != gpu) gpus.push_back(gpu);
      if (gpu == me) {
        my_member = mem[q];
        j = static_cast<int>(gpus.size()) - 1;
      }
    }
    const int S = static_cast<int>(gpus.size());
    if (S != m) throw std::logic_error("push two-shot needs one member per GPU");
    for (int oo = 0; oo < S; ++oo) {  // my member's chunks of every owner's slice
      const int o = (oo + j) % S;       // start at a different owner on every GPU
      const OwnedSlot& sl = find_slot(gpus[static_cast<size_t>(o)], gi);
      const long L = sl.hi - sl.lo;
      char* stage = static_cast<char*>(c->peer_push_buf[static_cast<size_t>(gpus[static_cast<size_t>(o)])]) +
                    static_cast<size_t>(sl.stage_off + static_cast<long>(j) * L) * c->esz;
      unsigned long long* flags = c->peer_push_flags[static_cast<size_t>(gpus[static_cast<size_t>(o)])] +
                                  sl.flag_off + static_cast<long>(j) * sl.nch;
      for (long ch = 0; ch < sl.nch; ++ch) {
        PushItem it{};
        it.lr = my_member - c->first;
        it.lo = sl.lo + ch * CH;
        it.hi = std::min(sl.hi, it.lo + CH);
        it.dst_beg = static_cast<int>(item_dst.size());
        it.ndst = 1;
        item_dst.push_back(stage + static_cast<size_t>(it.lo - sl.lo) * c->esz);
        item_flag.push_back(flags + ch);
        it.rank = my_member;
        item_keys.push_back({ch * 64 + oo, static_cast<long>(items.size())});
        items.push_back(it);
      }
    }
    const OwnedSlot& mine = find_slot(me, gi);  // the chunks I fold
    const long L = mine.hi - mine.lo;
    const int dst_beg = static_cast<int>(dst.size());
    for (int q = 0; q < m; ++q) dst.push_back(row_ptr(c, c->peer_w, mem[q]));
    for (long ch = 0; ch < mine.nch; ++ch) {
      PushFold f{};
      f.lo = mine.lo + ch * CH;
      f.hi = std::min(mine.hi, f.lo + CH);
      f.stage = static_cast<char*>(c->push_buf) + static_cast<size_t>(mine.stage_off + (f.lo - mine.lo)) * c->esz;
      f.stage_ld = L;
      f.flags = c->push_flags + mine.flag_off + ch;
      f.flag_ld = mine.nch;
      f.S = S;
      f.dst_beg = dst_beg;
      f.n_dst = m;
      f.err_rank = mem[0];
      folds.push_back(f);
    }
  }
  // interleave phase-1 items chunk-major across owners (each GPU starting at
  // a different owner) so every owner's inbound link is busy from the start
  std::stable_sort(item_keys.begin(), item_keys.end(),
                   [](const std::pair<long, long>& x, const std::pair<long, long>& y) { return x.first < y.first; });
  std::vector<PushItem> ordered;
  ordered.reserve(items.size());
  for (const auto& k : item_keys) ordered.push_back(items[static_cast<size_t>(k.second)]);
  items.swap(ordered);
  pl.items = static_cast<int>(items.size());
  pl.folds = static_cast<int>(folds.size());
  pl.d_item_dst = upload_table(c, item_dst);
  pl.d_item_flag = upload_table(c, item_flag);
  pl.d_items = upload_table(c, items);
  pl.d_folds = upload_table(c, folds);
  pl.d_dst = upload_table(c, dst);
  return pl;
}

// One-shot tables of parity t for this GPU: my member's stepped row goes to
// every member GPU's staging (row lr_o * G + j on GPU o, lr_o the member's
// local row there, j my position in the group); every GPU folds all S rows
// of its own member in ascending order and keeps the mean locally.
PushLaunch build_oneshot(dss_ctx* c, const Partition& part) {
  PushLaunch pl;
  pl.oneshot = true;
  const int G = c->cfg.n_gpus;
  const int me = c->cfg.rank;
  const long CH = c->chain_chunk;
  const long nch = c->chain_nchunks;
  const GpuPlan gp = make_plan(part, c->cfg.strategy.world_size, G, me, c->d_pad, force_chain(c));
  std::vector<PushItem> items;
  std::vector<void*> item_dst;
  std::vector<unsigned long long*> item_flag;
  std::vector<PushFold> folds;
  std::vector<void*> dst;
  for (int gi : gp.spanning_groups) {
    bool chain = false;
    for (const ChainRole& r : gp.chain) chain = chain || r.group == gi;
    if (chain) continue;
    const int* mem = part.group(gi);
    const int m = part.size(gi);
    int j = -1, my_member = -1;
    for (int q = 0; q < m; ++q) {
      if (mem[q] / c->P == me) {
        j = q;
        my_member = mem[q];
      }
    }
    if (j < 0) continue;
    // one item per chunk of my member: stepped once, stored to all m
    // stagings (every GPU starting at a different destination)
    for (long ch = 0; ch < nch; ++ch) {
      PushItem it{};
      it.lr = my_member - c->first;
      it.lo = ch * CH;
      it.hi = std::min(c->d_pad, it.lo + CH);
      it.dst_beg = static_cast<int>(item_dst.size());
      it.ndst = m;
      it.rank = my_member;
      for (int oo = 0; oo < m; ++oo) {
        const int o = (oo + j) % m;
        const int gpu = mem[o] / c->P;
        const long row = static_cast<long>(mem[o] - gpu * c->P) * G + j;
        item_dst.push_back(static_cast<char*>(c->peer_push_buf[static_cast<size_t>(gpu)]) +
                           static_cast<size_t>(row * c->d_pad + it.lo) * c->esz);
        item_flag.push_back(c->peer_push_flags[static_cast<size_t>(gpu)] + row * nch + ch);
      }
      items.push_back(it);
    }
    const long row0 = static_cast<long>(my_member - c->first) * G;
    const int dst_beg = static_cast<int>(dst.size());
    dst.push_back(static_cast<char*>(c->w) + static_cast<size_t>(my_member - c->first) * c->d_pad * c->esz);
    for (long ch = 0; ch < nch; ++ch) {
      PushFold f{};
      f.lo = ch * CH;
      f.hi = std::min(c->d_pad, f.lo + CH);
      f.stage = static_cast<char*>(c->push_buf) + static_cast<size_t>(row0 * c->d_pad + f.lo) * c->esz;
      f.stage_ld = c->d_pad;
      f.flags = c->push_flags + row0 * nch + ch;
      f.flag_ld = nch;
      f.S = m;
      f.dst_beg = dst_beg;
      f.n_dst = 1;
      f.err_rank = mem[0];
      folds.push_back(f);
    }
  }
  // chunk-major across this GPU's groups
  std::vector<PushItem> ordered;
  ordered.reserve(items.size());
  const size_t ng = nch ? items.size() / static_cast<size_t>(nch) : 0;
  for (long ch = 0; ch < nch; ++ch) {
    for (size_t g = 0; g < ng; ++g) ordered.push_back(items[g * static_cast<size_t>(nch) + static_cast<size_t>(ch)]);
  }
  pl.items = static_cast<int>(ordered.size());
  pl.folds = static_cast<int>(folds.size());
  pl.d_item_dst = upload_table(c, item_dst);
  pl.d_item_flag = upload_table(c, item_flag);
  pl.d_items = upload_table(c, ordered);
  pl.d_folds = upload_table(c, folds);
  pl.d_dst = upload_table(c, dst);
  return pl;
}

// Build the launch tables of one parity.  with_step: DS iteration (local
// steps fused); otherwise sync_round (fold only).
ParityPlan build_plan(dss_ctx* c, long t, bool with_step) {
  ParityPlan pp;
  const dss_strategy& s = c->cfg.strategy;
  const Partition part = make_partition(s, t);
  const int G = multi(c) ? c->cfg.n_gpus : 1;
  std::vector<std::vector<int>> local, span_members;
  std::vector<Slice> owned;

  if (force_fold(c)) {
    // Every multi-member group takes the two-shot path with one virtual
    // owner per member (slices split m ways), all on this device.
    for (int gi = 0; gi < part.n_groups(); ++gi) {
      const int* mem = part.group(gi);
      const int m = part.size(gi);
      if (m == 1) {
        local.push_back({mem[0]});
        continue;
      }
      pp.any_spanning = true;
      for (int j = 0; j < m; ++j) span_members.push_back({mem[j]});
      for (int j = 0; j < m; ++j) {
        Slice sl;
        sl.group = gi;
        slice_range(c->d_pad, m, j, &sl.lo, &sl.hi);
        if (sl.hi > sl.lo) owned.push_back(sl);
      }
    }
  } else {
    const GpuPlan gp = make_plan(part, s.world_size, G, multi(c) ? c->cfg.rank : 0, c->d_pad, force_chain(c));
    pp.any_spanning = gp.any_spanning_globally;
    pp.any_twoshot = gp.any_twoshot_globally;
    pp.any_chain = gp.any_chain_globally;
    for (int gi : gp.local_groups) {
      local.emplace_back(part.group(gi), part.group(gi) + part.size(gi));
    }
    // Members of chain groups are stepped inside the chain's partial pass
    // (fused step + ordered fold); only two-shot members step separately.
    std::vector<int> chain_members;
    for (const ChainRole& r : gp.chain) chain_members.insert(chain_members.end(), r.run.begin(), r.run.end());
    for (int r : gp.spanning_local_members) {
      const bool in_chain = std::find(chain_members.begin(), chain_members.end(), r) != chain_members.end();
      if (!(with_step && in_chain)) span_members.push_back({r});
    }
    owned = gp.owned;
    if (!gp.chain.empty()) {
      std::vector<std::vector<void*>> dsts;
      std::vector<std::vector<int>> lrs;
      for (const ChainRole& r : gp.chain) {
        std::vector<void*> d;
        std::vector<int> l;
        for (int k : r.run) {
          d.push_back(row_ptr(c, std::vector<void*>(static_cast<size_t>(G), nullptr), k, c->w));
          l.push_back(k - c->first);
        }
        dsts.push_back(d);
        lrs.push_back(l);
      }
      pp.chain = build_chain(c, gp.chain, c->w, dsts, s.kind == DSS_BSP ? 0 : 1,
                             with_step ? c->cfg.optimizer : kOptNone, kOptNone, lrs);
    }
  }
  if (force_fold(c)) pp.any_twoshot = pp.any_spanning;

  pp.local = make_bucketed(c, local);
  if (with_step && use_push(c) && pp.any_twoshot) {
    // Fused two-shot: this GPU's two-shot members are stepped inside the
    // push kernel; owned slices are folded there too.
    pp.any_push = true;
    pp.push = build_push(c, part, t);
    std::vector<std::vector<int>> rest;  // chain members are stepped in the chain
    (void)rest;
    span_members.clear();
    owned.clear();
  }
  if (with_step) pp.spanning_step = make_group_launch(c, span_members);

  if (!owned.empty()) {
    std::vector<FoldEntry> entries;
    std::vector<void*> src, dst;
    std::vector<void*> wb = multi(c) ? c->peer_w : std::vector<void*>{c->w};
    FoldLaunch& fl = pp.fold;
    fl.uniform_m = part.size(owned[0].group);
    for (const Slice& sl : owned) {
      const int* mem = part.group(sl.group);
      const int m = part.size(sl.group);
      if (m != fl.uniform_m) fl.uniform_m = 0;
      FoldEntry e{};
      e.src_beg = static_cast<int>(src.size());
      e.src_cnt = m;
      e.dst_beg = static_cast<int>(dst.size());
      e.dst_cnt = m;
      e.lo = sl.lo;
      e.hi = sl.hi;
      e.err_rank = mem[0];
      e.err_phase = s.kind == DSS_BSP ? 0 : 1;
      if (m > kMaxFold) throw std::invalid_argument("group spans more members than the fold kernel holds (64)");
      for (int j = 0; j < m; ++j) {
        void* p = row_ptr(c, wb, mem[j]);
        src.push_back(p);
        dst.push_back(p);
      }
      fl.max_len = std::max(fl.max_len, sl.hi - sl.lo);
      entries.push_back(e);
    }
    fl.entries = static_cast<int>(entries.size());
    fl.d_entries = upload_table(c, entries);
    fl.d_src = upload_table(c, src);
    fl.d_dst = upload_table(c, dst);
  }
  pp.built = true;
  return pp;
}

// BSP across GPUs: this GPU's owned slice of the world group folds all W
// gradients (peer rows) and writes the mean gradient slice into every GPU's
// mean-gradient row.
ParityPlan build_bsp_multi_plan(dss_ctx* c) {
  ParityPlan pp;
  const int G = c->cfg.n_gpus;
  const int W = c->cfg.strategy.world_size;
  const Partition part = make_partition(c->cfg.strategy, 0);  // one all-world group
  const GpuPlan gp = make_plan(part, W, G, c->cfg.rank, c->d_pad, force_chain(c));
  pp.any_spanning = true;
  pp.any_twoshot = gp.any_twoshot_globally;
  pp.any_chain = gp.any_chain_globally;
  std::vector<std::vector<int>> singles;
  for (int k = 0; k < c->P; ++k) singles.push_back({c->first + k});
  pp.spanning_step = make_group_launch(c, singles);
  if (!gp.chain.empty()) {
    // packed BSP: ordered chain over the gradient rows; as each chunk of the
    // mean gradient arrives, every local replica steps with it in place
    // (fused fold -> step, no mean-gradient row round trip)
    std::vector<void*> reps;
    std::vector<int> lrs;
    for (int k = 0; k < c->P; ++k) {
      reps.push_back(static_cast<char*>(c->w) + static_cast<size_t>(k) * c->d_pad * c->esz);
      lrs.push_back(k);
    }
    pp.chain = build_chain(c, gp.chain, c->g, {reps}, 0, kOptNone, c->cfg.optimizer, {lrs});
  }
  if (!gp.owned.empty()) {
    const Slice sl = gp.owned[0];
    FoldEntry e{};
    std::vector<void*> src, dst;
    e.src_beg = 0;
    e.src_cnt = W;
    e.dst_beg = 0;
    e.dst_cnt = G;
    e.lo = sl.lo;
    e.hi = sl.hi;
    e.err_rank = 0;
    e.err_phase = 0;
    if (W > kMaxFold) throw std::invalid_argument("multi-GPU BSP supports at most 64 workers");
    for (int k = 0; k < W; ++k) src.push_back(row_ptr(c, c->peer_g, k));
    for (int q = 0; q < G; ++q) dst.push_back(c->peer_mg[static_cast<size_t>(q)]);
    pp.fold.entries = 1;
    pp.fold.uniform_m = W;
    pp.fold.max_len = sl.hi - sl.lo;
    pp.fold.d_entries = upload_table(c, std::vector<FoldEntry>{e});
    pp.fold.d_src = upload_table(c, src);
    pp.fold.d_dst = upload_table(c, dst);
  }
  pp.built = true;
  return pp;
}

// global_mean_params = mean_of_ptrs over all W workers (param.cpp:59-70):
// one all-world group over the params rows, mean into mg (every GPU).
ParityPlan build_mean_plan(dss_ctx* c) {
  ParityPlan pp;
  const int W = c->cfg.strategy.world_size;
  dss_strategy world = c->cfg.strategy;
  world.kind = DSS_BSP;
  world.group_size = W;
  world.rectangular = 0;
  const Partition part = make_partition(world, 0);
  if (!multi(c)) {
    if (W > kMaxFold) throw std::invalid_argument("global mean supports at most 64 workers per GPU");
    FoldEntry e{};
    std::vector<void*> src, dst{c->mg};
    e.src_beg = 0;
    e.src_cnt = W;
    e.dst_beg = 0;
    e.dst_cnt = 1;
    e.lo = 0;
    e.hi = c->d_pad;
    e.err_rank = 0;
    e.err_phase = 1;
    for (int k = 0; k < W; ++k) src.push_back(static_cast<char*>(c->w) + static_cast<size_t>(k) * c->d_pad * c->esz);
    pp.any_spanning = true;
    pp.any_twoshot = true;
    pp.fold.entries = 1;
    pp.fold.uniform_m = W;
    pp.fold.max_len = c->d_pad;
    pp.fold.d_entries = upload_table(c, std::vector<FoldEntry>{e});
    pp.fold.d_src = upload_table(c, src);
    pp.fold.d_dst = upload_table(c, dst);
    pp.built = true;
    return pp;
  }
  const int G = c->cfg.n_gpus;
  const GpuPlan gp = make_plan(part, W, G, c->cfg.rank, c->d_pad, force_chain(c));
  pp.any_spanning = true;
  pp.any_twoshot = gp.any_twoshot_globally;
  pp.any_chain = gp.any_chain_globally;
  if (!gp.chain.empty()) pp.chain = build_chain(c, gp.chain, c->w, {std::vector<void*>{c->mg}}, 1);
  if (!gp.owned.empty()) {
    if (W > kMaxFold) throw std::invalid_argument("global mean supports at most 64 workers");
    const Slice sl = gp.owned[0];
    FoldEntry e{};
    std::vector<void*> src, dst;
    e.src_beg = 0;
    e.src_cnt = W;
    e.dst_beg = 0;
    e.dst_cnt = G;
    e.lo = sl.lo;
    e.hi = sl.hi;
    e.err_rank = 0;
    e.err_phase = 1;
    for (int k = 0; k < W; ++k) src.push_back(row_ptr(c, c->peer_w, k));
    for (int q = 0; q < G; ++q) dst.push_back(c->peer_mg[static_cast<size_t>(q)]);
    pp.fold.entries = 1;
    pp.fold.uniform_m = W;
    pp.fold.max_len = sl.hi - sl.lo;
    pp.fold.d_entries = upload_table(c, std::vector<FoldEntry>{e});
    pp.fold.d_src = upload_table(c, src);
    pp.fold.d_dst = upload_table(c, dst);
  }
  pp.built = true;
  return pp;
}

// Running statistics ride the same schedule as their payload (params for DS
// and sync_round, the world group for BSP): local groups fold in the group
// kernel (no step); groups spanning GPUs are tiny rows, always two-shot
// slices over the peers' stats rows.
ParityPlan build_stats_plan(dss_ctx* c, const Partition& part) {
  ParityPlan pp;
  const int G = multi(c) ? c->cfg.n_gpus : 1;
  const int W = c->cfg.strategy.world_size;
  std::vector<std::vector<int>> local;
  std::vector<FoldEntry> entries;
  std::vector<void*> src, dst;
  long max_len = 0;
  int uniform_m = -1;
  for (int gi = 0; gi < part.n_groups(); ++gi) {
    const int* mem = part.group(gi);
    const int m = part.size(gi);
    std::vector<int> gpus;
    for (int j = 0; j < m; ++j) {
      const int gpu = mem[j] / c->P;
      if (gpus.empty() || gpus.back() != gpu) gpus.push_back(gpu);
    }
    if (gpus.size() > 1) pp.any_spanning = pp.any_twoshot = true;
    const int me = multi(c) ? c->cfg.rank : 0;
    const auto it = std::find(gpus.begin(), gpus.end(), me);
    if (it == gpus.end()) continue;
    if (gpus.size() == 1) {
      local.emplace_back(mem, mem + m);
      continue;
    }
    if (m > kMaxFold) throw std::invalid_argument("group spans more members than the fold kernel holds (64)");
    long lo = 0, hi = 0;
    slice_range(c->s_pad, static_cast<int>(gpus.size()), static_cast<int>(it - gpus.begin()), &lo, &hi);
    if (hi <= lo) continue;
    FoldEntry e{};
    e.src_beg = static_cast<int>(src.size());
    e.src_cnt = m;
    e.dst_beg = static_cast<int>(dst.size());
    e.dst_cnt = m;
    e.lo = lo;
    e.hi = hi;
    e.err_rank = c->cfg.strategy.kind == DSS_BSP ? 0 : mem[0];
    e.err_phase = c->cfg.strategy.kind == DSS_BSP ? 0 : 1;
    for (int j = 0; j < m; ++j) {
      const int gpu = mem[j] / c->P;
      void* p = static_cast<char*>(c->peer_stats[static_cast<size_t>(gpu)]) +
                static_cast<size_t>(mem[j] - gpu * c->P) * c->s_pad * c->esz;
      src.push_back(p);
      dst.push_back(p);
    }
    uniform_m = uniform_m < 0 ? m : (uniform_m == m ? m : 0);
    max_len = std::max(max_len, hi - lo);
    entries.push_back(e);
  }
  (void)G;
  (void)W;
  pp.local = make_bucketed(c, local);
  if (!entries.empty()) {
    pp.fold.entries = static_cast<int>(entries.size());
    pp.fold.uniform_m = uniform_m < 0 ? 0 : uniform_m;
    pp.fold.max_len = max_len;
    pp.fold.d_entries = upload_table(c, entries);
    pp.fold.d_src = upload_table(c, src);
    pp.fold.d_dst = upload_table(c, dst);
  }
  pp.built = true;
  return pp;
}

void build_stats_plans(dss_ctx* c) {
  if (c->s == 0) return;
  const dss_strategy& s = c->cfg.strategy;
  for (int p = 0; p < (s.kind == DSS_DS_SYNC ? 2 : 1); ++p) c->stats_plan[p] = build_stats_plan(c, make_partition(s, p));
}

void build_plans(dss_ctx* c) {
  const dss_strategy& s = c->cfg.strategy;
  if (s.kind == DSS_DS_SYNC) {
    for (int p = 0; p < 2; ++p) c->step_plan[p] = build_plan(c, p, true);
  } else if (multi(c)) {
    c->step_plan[0] = build_bsp_multi_plan(c);
  }
  for (int p = 0; p < 2; ++p) c->sync_plan[p] = build_plan(c, p, false);
  if (c->cfg.strategy.world_size <= kMaxFold || multi(c)) c->mean_plan = build_mean_plan(c);
  build_stats_plans(c);
}

// ---- launch helpers ---------------------------------------------------------

struct TimedLaunch {
  dss_ctx* c;
  int kind;
  cudaEvent_t b = nullptr, e = nullptr;
  TimedLaunch(dss_ctx* cc, int k) : c(cc), kind(k) {
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

int grid_x(const dss_ctx* c, long nvec, int ys) {
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
  const dss_hparams& h = c->cfg.hp;
  for (int k = 0; k < c->P; ++k) {
    const double t = static_cast<double>(c->step_count[static_cast<size_t>(k)] + 1);
    a.bc1[k] = 1.0 - std::pow(h.beta1, t);  // optim.cpp:76-77
    a.bc2[k] = 1.0 - std::pow(h.beta2, t);  // optim.cpp:78
  }
}

template <typename T, int OPT, int M>
void launch_group_t(dss_ctx* c, const GroupArgs<T>& a, int groups) {
  dim3 grid(grid_x(c, a.nvec, groups), groups);
  TimedLaunch tl(c, DSS_KIND_GROUP);
  ds_group_kernel<T, OPT, M><<<grid, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "ds_group_kernel launch");
}

// Shared-memory-staged variant for groups of 8 with stateful optimizers
// (DSS_GROUP_BULK=1; default off until measured better).
#ifndef DSS_GROUP_BULK
#define DSS_GROUP_BULK 0
#endif

template <typename T, int OPT>
void launch_group_bulk(dss_ctx* c, const GroupArgs<T>& a, const GroupLaunch& gl) {
  constexpr int A = (OPT == kAdam || OPT == kAdamW) ? 4 : (OPT == kMomentum ? 3 : 2);
  const size_t smem = static_cast<size_t>(kBulkStages) * 8 * A * kBulkTE * sizeof(T);
  static bool attr_set = false;
  if (!attr_set) {
    ck(cudaFuncSetAttribute(ds_group_bulk_kernel<T, OPT, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)),
       "bulk smem attribute");
    attr_set = true;
  }
  const int tiles = static_cast<int>((a.ld + kBulkTE - 1) / kBulkTE);
  dim3 grid(std::max(1, std::min(tiles, (c->sms + gl.groups - 1) / gl.groups)), gl.groups);
  TimedLaunch tl(c, DSS_KIND_GROUP);
  ds_group_bulk_kernel<T, OPT, 8><<<grid, kThreads + 32, smem, c->stream>>>(a, c->d_timeout);
  ck(cudaGetLastError(), "ds_group_bulk_kernel launch");
}

template <typename T, int OPT>
void launch_group_m(dss_ctx* c, const GroupArgs<T>& a, const GroupLaunch& gl) {
  if constexpr (OPT == kMomentum || OPT == kAdam || OPT == kAdamW) {
    if (DSS_GROUP_BULK && std::is_same_v<T, float> && gl.size == 8 && a.g_ld == a.ld &&
        a.w == static_cast<T*>(c->w)) {
      launch_group_bulk<T, OPT>(c, a, gl);
      return;
    }
  }
  switch (gl.size) {
    case 1: launch_group_t<T, OPT, 1>(c, a, gl.groups); break;
    case 2: launch_group_t<T, OPT, 2>(c, a, gl.groups); break;
    case 3: launch_group_t<T, OPT, 3>(c, a, gl.groups); break;
    case 4: launch_group_t<T, OPT, 4>(c, a, gl.groups); break;
    case 8: launch_group_t<T, OPT, 8>(c, a, gl.groups); break;
    default: launch_group_t<T, OPT, 0>(c, a, gl.groups); break;
  }
}

// opt < 0: fold only (sync_round); otherwise the optimizer kind.
template <typename T>
void launch_groups(dss_ctx* c, const GroupLaunch& gl, int opt, long t, double alpha,
                   const void* g, long g_ld, int step_phase, int sync_phase, void* rows = nullptr, long rows_ld = 0) {
  if (gl.groups == 0) return;
  GroupArgs<T> a{};
  a.w = static_cast<T*>(rows ? rows : c->w);  // rows: fold-only over another row set (running stats)
  a.g = static_cast<const T*>(g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = rows ? rows_ld : c->d_pad;
  a.g_ld = g_ld;
  a.nvec = a.ld / Vec<T>::n;
  a.first_rank = c->first;
  a.members = gl.d_members;
  a.offsets = gl.d_offsets;
  a.step_phase = step_phase;
  a.sync_phase = sync_phase;
  a.t = t;
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  a.err = c->d_err;
  switch (opt) {
    case kOptNone: launch_group_m<T, kOptNone>(c, a, gl); break;
    case kSgd: launch_group_m<T, kSgd>(c, a, gl); break;
    case kMomentum: launch_group_m<T, kMomentum>(c, a, gl); break;
    case kAdam: launch_group_m<T, kAdam>(c, a, gl); break;
    case kAdamW: launch_group_m<T, kAdamW>(c, a, gl); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

void launch_groups_any(dss_ctx* c, const GroupLaunch& gl, int opt, long t, double alpha,
                       const void* g, long g_ld, int step_phase, int sync_phase = 1, void* rows = nullptr,
                       long rows_ld = 0) {
  if (c->cfg.dtype == DSS_F64) {
    launch_groups<double>(c, gl, opt, t, alpha, g, g_ld, step_phase, sync_phase, rows, rows_ld);
  } else {
    launch_groups<float>(c, gl, opt, t, alpha, g, g_ld, step_phase, sync_phase, rows, rows_ld);
  }
}

template <typename T, int M>
void launch_fold_t(dss_ctx* c, const FoldLaunch& fl, long t) {
  FoldArgs<T> a{};
  a.src = reinterpret_cast<T* const*>(fl.d_src);
  a.dst = reinterpret_cast<T* const*>(fl.d_dst);
  a.entries = fl.d_entries;
  a.t = t;
  a.err = c->d_err;
  dim3 grid(grid_x(c, fl.max_len / Vec<T>::n, fl.entries), fl.entries);
  TimedLaunch tl(c, DSS_KIND_FOLD);
  fold_kernel<T, M><<<grid, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "fold_kernel launch");
}

template <typename T>
void launch_fold(dss_ctx* c, const FoldLaunch& fl, long t) {
  if (fl.entries == 0) return;
  switch (fl.uniform_m) {
    case 2: launch_fold_t<T, 2>(c, fl, t); break;
    case 4: launch_fold_t<T, 4>(c, fl, t); break;
    case 8: launch_fold_t<T, 8>(c, fl, t); break;
    default: launch_fold_t<T, 0>(c, fl, t); break;
  }
}

void launch_fold_any(dss_ctx* c, const FoldLaunch& fl, long t) {
  if (c->cfg.dtype == DSS_F64) {
    launch_fold<double>(c, fl, t);
  } else {
    launch_fold<float>(c, fl, t);
  }
}

template <typename T, int OPTM, int OPTD>
void launch_chain_t(dss_ctx* c, const ChainLaunch& cl, ChainArgs<T>& a) {
  // Kernel B follows kernel A on the stream.  Measured alternatives that
  // lost at 2 GPUs (C2 / C3 iters/s against 3108 / 480 for this schedule):
  // B concurrently on a side stream with A giving up CTA slots (2534 / 369),
  // and both passes in one persistent kernel with lagged mean-pass units
  // (2300 / stalled).
  if (cl.na > 0) {
    a.entries = cl.d_a;
    a.n_entries = cl.na;
    const long units = c->chain_nchunks * cl.na;
    TimedLaunch tl(c, DSS_KIND_CHAIN);
    chain_partial_kernel<T, OPTM, OPTD><<<static_cast<int>(std::min<long>(units, c->sms * long{DSS_CHAIN_CTAS_PER_SM})),
                                          kThreads, 0, c->stream>>>(a);
    ck(cudaGetLastError(), "chain_partial_kernel launch");
  }
  if (cl.nb > 0) {
    a.entries = cl.d_b;
    a.n_entries = cl.nb;
    const long units = c->chain_nchunks * cl.nb;
    TimedLaunch tl(c, DSS_KIND_CHAIN_MEAN);
    chain_mean_kernel<T, OPTD><<<static_cast<int>(std::min<long>(units, c->sms * long{DSS_CHAIN_CTAS_PER_SM})),
                                 kThreads, 0, c->stream>>>(a);
    ck(cudaGetLastError(), "chain_mean_kernel launch");
  }
}

template <typename T, int OPTM>
void launch_chain_d(dss_ctx* c, const ChainLaunch& cl, ChainArgs<T>& a) {
  switch (cl.opt_dst) {
    case kOptNone: launch_chain_t<T, OPTM, kOptNone>(c, cl, a); break;
    case kSgd: launch_chain_t<T, kOptNone, kSgd>(c, cl, a); break;
    case kMomentum: launch_chain_t<T, kOptNone, kMomentum>(c, cl, a); break;
    case kAdam: launch_chain_t<T, kOptNone, kAdam>(c, cl, a); break;
    case kAdamW: launch_chain_t<T, kOptNone, kAdamW>(c, cl, a); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

template <typename T>
void launch_chain(dss_ctx* c, const ChainLaunch& cl, long t, double alpha) {
  ++c->chain_epoch;  // same sequence on every GPU: flags compare against it
  if (cl.opt_mem != kOptNone && cl.opt_dst != kOptNone) throw std::logic_error("chain: one fused step only");
  ChainArgs<T> a{};
  a.src = reinterpret_cast<T* const*>(cl.d_src);
  a.dst = reinterpret_cast<T* const*>(cl.d_dst);
  a.src_lr = cl.d_src_lr;
  a.dst_lr = cl.d_dst_lr;
  a.chunk = c->chain_chunk;
  a.len = c->d_pad;
  a.n_chunks = c->chain_nchunks;
  a.epoch = c->chain_epoch;
  a.t = t;
  a.err = c->d_err;
  a.timeout = c->d_timeout;
  a.stage = static_cast<T*>(c->mg);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.first_rank = c->first;
  a.step_phase = c->cfg.strategy.kind == DSS_BSP ? 1 : 0;
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  switch (cl.opt_mem) {
    case kOptNone: launch_chain_d<T, kOptNone>(c, cl, a); break;
    case kSgd: launch_chain_t<T, kSgd, kOptNone>(c, cl, a); break;
    case kMomentum: launch_chain_t<T, kMomentum, kOptNone>(c, cl, a); break;
    case kAdam: launch_chain_t<T, kAdam, kOptNone>(c, cl, a); break;
    case kAdamW: launch_chain_t<T, kAdamW, kOptNone>(c, cl, a); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

void launch_chain_any(dss_ctx* c, const ChainLaunch& cl, long t, double alpha = 0.0) {
  if (c->cfg.dtype == DSS_F64) {
    launch_chain<double>(c, cl, t, alpha);
  } else {
    launch_chain<float>(c, cl, t, alpha);
  }
}

template <typename T, int OPT>
void launch_push_t(dss_ctx* c, const PushLaunch& pl, long t, double alpha) {
  ++c->chain_epoch;  // flags compare against the shared epoch sequence
  PushArgs<T> a{};
  a.items = pl.d_items;
  a.n_items = pl.items;
  a.item_dst = pl.d_item_dst;
  a.item_flag = pl.d_item_flag;
  a.folds = pl.d_folds;
  a.n_folds = pl.folds;
  a.dst = reinterpret_cast<T* const*>(pl.d_dst);
  a.w = static_cast<T*>(c->w);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.first_rank = c->first;
  a.t = t;
  a.epoch = c->chain_epoch;
  a.err = c->d_err;
  a.timeout = c->d_timeout;
  if (pl.oneshot) {
    // alternate staging buffers: a GPU can only push launch n+2 after every
    // peer pushed launch n+1, i.e. after every peer finished folding launch n
    const long par = static_cast<long>(c->oneshot_seq++ & 1);
    a.stage_shift = (c->oneshot_base_elems + par * c->oneshot_half_elems) * c->esz;
    a.flag_shift = c->oneshot_base_flags + par * c->oneshot_half_flags;
  }
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  int occ = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, push_twoshot_kernel<T, OPT>, kThreads, 0), "occupancy");
  // fully resident grid: phase-1 work can never wait behind spinning CTAs
  const long grid = std::max(1L, std::min<long>(static_cast<long>(std::max(occ, 1)) * c->sms,
                                                std::max(pl.items, pl.folds)));
  TimedLaunch tl(c, DSS_KIND_FOLD);
  push_twoshot_kernel<T, OPT><<<static_cast<int>(grid), kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "push_twoshot_kernel launch");
}

template <typename T>
void launch_push(dss_ctx* c, const PushLaunch& pl, long t, double alpha) {
  switch (c->cfg.optimizer) {
    case kSgd: launch_push_t<T, kSgd>(c, pl, t, alpha); break;
    case kMomentum: launch_push_t<T, kMomentum>(c, pl, t, alpha); break;
    case kAdam: launch_push_t<T, kAdam>(c, pl, t, alpha); break;
    case kAdamW: launch_push_t<T, kAdamW>(c, pl, t, alpha); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

void launch_push_any(dss_ctx* c, const PushLaunch& pl, long t, double alpha) {
  if (c->cfg.dtype == DSS_F64) {
    launch_push<double>(c, pl, t, alpha);
  } else {
    launch_push<float>(c, pl, t, alpha);
  }
}

template <typename T, int OPT, int WT>
void launch_bsp_t(dss_ctx* c, const BspArgs<T>& a) {
  dim3 grid(grid_x(c, a.nvec, 1), 1);
  TimedLaunch tl(c, DSS_KIND_BSP);
  bsp_kernel<T, OPT, WT><<<grid, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "bsp_kernel launch");
}

template <typename T, int OPT>
void launch_bsp_w(dss_ctx* c, const BspArgs<T>& a) {
  switch (a.nw) {
    case 2: launch_bsp_t<T, OPT, 2>(c, a); break;
    case 4: launch_bsp_t<T, OPT, 4>(c, a); break;
    case 8: launch_bsp_t<T, OPT, 8>(c, a); break;
    default: launch_bsp_t<T, OPT, 0>(c, a); break;
  }
}

template <typename T>
void launch_bsp(dss_ctx* c, long t, double alpha) {
  BspArgs<T> a{};
  a.w = static_cast<T*>(c->w);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.nvec = c->d_pad / Vec<T>::n;
  a.nw = c->P;
  a.t = t;
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  a.err = c->d_err;
  switch (c->cfg.optimizer) {
    case kSgd: launch_bsp_w<T, kSgd>(c, a); break;
    case kMomentum: launch_bsp_w<T, kMomentum>(c, a); break;
    case kAdam: launch_bsp_w<T, kAdam>(c, a); break;
    case kAdamW: launch_bsp_w<T, kAdamW>(c, a); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

void barrier(dss_ctx* c) {
  if (!multi(c)) return;
  if (!c->attached) throw PeerError("multi-GPU context used before dss_ipc_attach");
  ++c->epoch;
  TimedLaunch tl(c, DSS_KIND_BARRIER);
  barrier_kernel<<<1, 32 * ((c->cfg.n_gpus + 31) / 32), 0, c->stream>>>(
      c->d_peer_flags, c->flags, c->cfg.rank, c->cfg.n_gpus, c->epoch, c->d_timeout);
  ck(cudaGetLastError(), "barrier_kernel launch");
}

// Peers may still be writing group means into our rows (two-shot phase 2 of
// the previous round): wait for them before touching the rows again.
void quiesce(dss_ctx* c) {
  if (c->pending_remote && multi(c)) barrier(c);
  c->pending_remote = false;
}

// Fold the running statistics of iteration t (DS: the parity's groups; BSP:
// the world).  barrier_done: a cross-GPU barrier already ordered every GPU's
// stats update before this point in the current iteration.
void fold_stats(dss_ctx* c, long t, bool barrier_done) {
  if (c->s == 0) return;
  const ParityPlan& sp = c->stats_plan[c->cfg.strategy.kind == DSS_DS_SYNC ? (t & 1) : 0];
  const int phase = c->cfg.strategy.kind == DSS_BSP ? 0 : 1;
  for (const GroupLaunch& gl : sp.local) {
    launch_groups_any(c, gl, kOptNone, t, 0.0, nullptr, 0, 0, phase, c->stats, c->s_pad);
  }
  if (sp.any_twoshot) {
    if (multi(c) && !barrier_done) barrier(c);
    launch_fold_any(c, sp.fold, t);
    c->pending_remote = multi(c);
  }
}

void bump_steps(dss_ctx* c) {
  for (auto& s : c->step_count) ++s;
}

int check_impl(dss_ctx* c) {
  ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  ck(cudaMemcpy(c->h_err, c->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost), "err readback");
  unsigned long long timeout = 0;
  if (c->d_timeout) {
    ck(cudaMemcpy(&timeout, c->d_timeout, sizeof(timeout), cudaMemcpyDeviceToHost), "timeout readback");
  }
  if (timeout) return fail(c, DSS_ENCCL, "cross-GPU barrier timed out (peer did not arrive)");
  unsigned long long gkey = ~0ull;
  ck(cudaMemcpy(&gkey, c->d_gerr, sizeof(gkey), cudaMemcpyDeviceToHost), "err readback");
  const unsigned long long key = *c->h_err;
  if (key == ~0ull && gkey == ~0ull) return DSS_OK;
  long t = static_cast<long>(key >> 34);
  const int phase = static_cast<int>((key >> 32) & 3);
  int rank = static_cast<int>(key & 0xffffffffu);
  std::string what;
  const bool bsp = c->cfg.strategy.kind == DSS_BSP;
  const bool local_step = bsp ? phase == 1 : phase == 0;
  // A gradient failure (checked_gradient, sync.cpp:181-191) wins over an
  // iteration-t step/collective failure unless it comes later in the
  // reference's order: DS runs gradient + step per worker in rank order
  // (sync.cpp:348-361), BSP computes every gradient before the collective.
  bool grad = false;
  if (gkey != ~0ull) {
    const long gt = static_cast<long>(gkey >> 32);
    const int gr = static_cast<int>(gkey & 0xffffffffu);
    grad = key == ~0ull || gt < t || (gt == t && (bsp || !local_step || gr <= rank));
    if (grad) {
      t = gt;
      rank = gr;
    }
  }
  if (grad) {
    what = "non-finite stochastic gradient";
  } else if (local_step) {
    what = "apply_step: non-finite value in result";  // optim.cpp:96 via sync.cpp:257-261
  } else {
    what = std::string(collective_name(c->cfg.strategy.topology)) + ": non-finite value in result";
  }
  // DivergenceError text (errors.hpp:17-19)
  const std::string msg = "worker " + std::to_string(rank) + " diverged at iteration " +
                          std::to_string(t) + ": " + what;
  return fail(c, DSS_EDIVERGED, msg, rank, t);
}

int check_rank(dss_ctx* c, int rank, int* lr) {
  if (rank < c->first || rank >= c->first + c->P) {
    throw std::invalid_argument("rank " + std::to_string(rank) + " is not hosted on this GPU");
  }
  *lr = rank - c->first;
  return DSS_OK;
}

struct RowGeom {
  void* base;
  long len;  // logical row length (dim or stats_dim)
  long ld;   // padded row stride
};

RowGeom geom(dss_ctx* c, int buffer) {
  switch (buffer) {
    case DSS_BUF_PARAMS: return {c->w, c->d, c->d_pad};
    case DSS_BUF_GRADS: return {c->g, c->d, c->d_pad};
    case DSS_BUF_MOMENT1:
      if (!c->m1) throw std::invalid_argument("optimizer has no first moment buffer");
      return {c->m1, c->d, c->d_pad};
    case DSS_BUF_MOMENT2:
      if (!c->m2) throw std::invalid_argument("optimizer has no second moment buffer");
      return {c->m2, c->d, c->d_pad};
    case DSS_BUF_STATS:
    case DSS_BUF_STATS_OBS:
      if (c->s == 0) throw std::invalid_argument("context has no running statistics (stats_dim = 0)");
      return {buffer == DSS_BUF_STATS ? c->stats : c->stats_obs, c->s, c->s_pad};
    default: throw std::invalid_argument("unknown buffer id");
  }
}

}  // namespace

// ============================ schedule (host) ===============================

extern "C" int dss_validate_world(int world_size, int group_size, int rectangular) {
  return guard(nullptr, [&]() -> int {
    validate_world(world_size, group_size, rectangular != 0);
    return DSS_OK;
  });
}

extern "C" int dss_validate_strategy(const dss_strategy* s) {
  return guard(nullptr, [&]() -> int {
    if (!s) throw std::invalid_argument("null strategy");
    validate_strategy(*s);
    return DSS_OK;
  });
}

extern "C" int dss_is_square_mode(int world_size, int group_size) {
  return is_square_mode(world_size, group_size) ? 1 : 0;
}

extern "C" int dss_partition(const dss_strategy* s, long t, int* members, int* offsets, int* n_groups) {
  return guard(nullptr, [&]() -> int {
    if (!s || !members || !offsets || !n_groups) throw std::invalid_argument("null argument");
    if (s->kind == DSS_BSP) validate_strategy(*s);
    const Partition p = make_partition(*s, t);
    std::copy(p.members.begin(), p.members.end(), members);
    std::copy(p.offsets.begin(), p.offsets.end(), offsets);
    *n_groups = p.n_groups();
    return DSS_OK;
  });
}

extern "C" int dss_group_of(const dss_strategy* s, long t, int rank, int* members, int* count) {
  return guard(nullptr, [&]() -> int {
    if (!s || !members || !count) throw std::invalid_argument("null argument");
    const std::vector<int> g = group_of(*s, t, rank);
    std::copy(g.begin(), g.end(), members);
    *count = static_cast<int>(g.size());
    return DSS_OK;
  });
}

extern "C" int dss_check_mixing(const dss_strategy* s, long t) {
  int result = 0;
  const int st = guard(nullptr, [&]() -> int {
    if (!s) throw std::invalid_argument("null strategy");
    result = check_mixing(*s, t) ? 1 : 0;
    return DSS_OK;
  });
  return st == DSS_OK ? result : -st;
}

extern "C" int dss_round_outcome(const dss_strategy* s, long t, long payload_dim, dss_outcome* out) {
  return guard(nullptr, [&]() -> int {
    if (!s || !out) throw std::invalid_argument("null argument");
    validate_strategy(*s);
    *out = round_outcome(*s, t, payload_dim);
    return DSS_OK;
  });
}

extern "C" int dss_plan(const dss_strategy* s, long t, long dim, int n_gpus, int rank,
                        dss_plan_summary* out, long* slice_lo, long* slice_hi, int* slice_group,
                        int max_slices) {
  return guard(nullptr, [&]() -> int {
    if (!s || !out) throw std::invalid_argument("null argument");
    validate_strategy(*s);
    if (n_gpus < 1 || s->world_size % n_gpus != 0) {
      throw std::invalid_argument("world_size must be a multiple of n_gpus");
    }
    if (rank < 0 || rank >= n_gpus) throw std::invalid_argument("gpu rank out of range");
    const Partition p = make_partition(*s, t);
    const GpuPlan gp = make_plan(p, s->world_size, n_gpus, rank, pad_dim(dim));
    out->local_groups = static_cast<int>(gp.local_groups.size());
    out->spanning_groups = static_cast<int>(gp.spanning_groups.size());
    out->owned_slices = static_cast<int>(gp.owned.size());
    out->chain_groups = static_cast<int>(gp.chain.size());
    out->owned_elems = 0;
    for (size_t i = 0; i < gp.owned.size(); ++i) {
      out->owned_elems += gp.owned[i].hi - gp.owned[i].lo;
      if (static_cast<int>(i) < max_slices) {
        if (slice_lo) slice_lo[i] = gp.owned[i].lo;
        if (slice_hi) slice_hi[i] = gp.owned[i].hi;
        if (slice_group) slice_group[i] = gp.owned[i].group;
      }
    }
    return DSS_OK;
  });
}

extern "C" int dss_last_global_error(char* buf, size_t len) {
  if (buf && len) {
    std::snprintf(buf, len, "%s", g_last_global_error.c_str());
  }
  return DSS_OK;
}

// ============================== context =====================================

extern "C" int dss_create(const dss_config* cfg, dss_ctx** out) {
  if (!cfg || !out) return fail(nullptr, DSS_EINVAL, "null argument");
  *out = nullptr;
  auto c = std::make_unique<dss_ctx>();
  int st = guard(c.get(), [&]() -> int {
    c->cfg = *cfg;
    const dss_strategy& s = cfg->strategy;
    validate_strategy(s);
    if (cfg->dim < 1) throw std::invalid_argument("dim must be >= 1");
    if (cfg->dtype != DSS_F32 && cfg->dtype != DSS_F64) throw std::invalid_argument("unknown dtype");
    if (cfg->optimizer < DSS_VANILLA_SGD || cfg->optimizer > DSS_ADAMW) {
      throw std::invalid_argument("unknown optimizer kind");
    }
    if (cfg->n_gpus < 1 || s.world_size % cfg->n_gpus != 0) {
      throw std::invalid_argument("world_size must be a multiple of n_gpus");
    }
    if (cfg->rank < 0 || cfg->rank >= cfg->n_gpus) throw std::invalid_argument("rank out of range");
    c->P = s.world_size / cfg->n_gpus;
    if (c->P > kMaxLocal) {
      throw std::invalid_argument("at most " + std::to_string(kMaxLocal) + " workers per GPU");
    }
    c->first = cfg->rank * c->P;
    c->d = cfg->dim;
    c->d_pad = pad_dim(cfg->dim);
    c->esz = cfg->dtype == DSS_F64 ? 8 : 4;
    c->step_count.assign(static_cast<size_t>(c->P), 0);

    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (cfg->device < 0 || cfg->device >= ndev) throw CudaError("no CUDA device " + std::to_string(cfg->device));
    ck(cudaSetDevice(cfg->device), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cfg->device), "sm count");
    ck(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own_stream;

    const size_t rows = static_cast<size_t>(c->P) * c->d_pad * c->esz;
    c->w = dalloc(c.get(), rows);
    c->g = dalloc(c.get(), rows);
    if (cfg->optimizer != DSS_VANILLA_SGD) c->m1 = dalloc(c.get(), rows);
    if (cfg->optimizer == DSS_ADAM || cfg->optimizer == DSS_ADAMW) c->m2 = dalloc(c.get(), rows);
    c->mg = dalloc(c.get(), static_cast<size_t>(c->d_pad) * c->esz);
    if (cfg->stats_dim < 0) throw std::invalid_argument("stats_dim must be >= 0");
    if (cfg->path < 0 || cfg->path > 4) throw std::invalid_argument("path must be 0..4");
    c->s = cfg->stats_dim;
    c->s_pad = c->s > 0 ? pad_dim(c->s) : 0;
    // running statistics rows (always allocated: an IPC handle needs a buffer)
    c->stats = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(c->P) * c->s_pad * c->esz));
    c->stats_obs = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(c->P) * c->s_pad * c->esz));
    c->wstar = dalloc(c.get(), static_cast<size_t>(c->d_pad) * c->esz);
    c->d_err = static_cast<unsigned long long*>(dalloc(c.get(), sizeof(unsigned long long)));
    ck(cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream), "err init");
    c->d_gerr = static_cast<unsigned long long*>(dalloc(c.get(), sizeof(unsigned long long)));
    ck(cudaMemsetAsync(c->d_gerr, 0xff, sizeof(unsigned long long), c->stream), "err init");
    c->d_timeout = static_cast<unsigned long long*>(dalloc(c.get(), sizeof(unsigned long long)));
    c->flags = static_cast<unsigned long long*>(
        dalloc(c.get(), sizeof(unsigned long long) * static_cast<size_t>(std::max(cfg->n_gpus, 32))));
    ck(cudaMallocHost(&c->h_err, sizeof(unsigned long long)), "cudaMallocHost");

    std::vector<std::vector<int>> singles;
    for (int k = 0; k < c->P; ++k) singles.push_back({c->first + k});
    c->apply_launch = make_group_launch(c.get(), singles);
    if (multi(c.get())) {
      // chain-fold receive rows and flags, sized for the worst parity (the
      // plan is global, so every GPU computes the same slot count)
      int slots = 0;
      for (long t = 0; t < (s.kind == DSS_DS_SYNC ? 2 : 1); ++t) {
        const GpuPlan gp = make_plan(make_partition(s, t), s.world_size, cfg->n_gpus, cfg->rank, c->d_pad,
                                     force_chain(c.get()));
        slots = std::max(slots, gp.max_chain_slots);
      }
      dss_strategy world = s;  // the all-world group of the global-mean trace
      world.kind = DSS_BSP;
      world.group_size = s.world_size;
      world.rectangular = 0;
      slots = std::max(slots, make_plan(make_partition(world, 0), s.world_size, cfg->n_gpus, cfg->rank, c->d_pad,
                                        force_chain(c.get())).max_chain_slots);
      c->chain_slots = slots;
      c->chain_chunk = std::min<long>(c->d_pad, DSS_CHAIN_CHUNK);
      c->chain_nchunks = (c->d_pad + c->chain_chunk - 1) / c->chain_chunk;
      c->chain_buf = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(2) * slots * c->d_pad * c->esz));
      // Fused two-shot staging of the owned slices, worst parity and worst
      // GPU: the one-shot area starts after it at the same offset on every
      // GPU, because a pusher applies its own offset to the peer's buffer.
      long ps = 0, pf = 0;
      for (long t = 0; t < (s.kind == DSS_DS_SYNC ? 2 : 1); ++t) {
        const Partition part = make_partition(s, t);
        for (int q = 0; q < cfg->n_gpus; ++q) {
          long st = 0, fl = 0;
          owned_layout(c.get(), part, q, c->chain_chunk, &st, &fl);
          ps = std::max(ps, st);
          pf = std::max(pf, fl);
        }
      }
      // One-shot per schedule parity: every member GPU gathers every
      // member's row.  Same NVLink bytes as two-shot for pairs (S = 2) and
      // no barrier before the next iteration; for S > 2 only small rows.
      for (long t = 0; t < 2; ++t) {
        if (s.kind != DSS_DS_SYNC || !use_push(c.get()) || force_chain(c.get()) || cfg->path == 4) break;
        const Partition part = make_partition(s, t);
        bool ok = true;
        for (int gi = 0; gi < part.n_groups(); ++gi) {
          std::vector<int> gpus;
          for (int q = 0; q < part.size(gi); ++q) gpus.push_back(part.group(gi)[q] / c->P);
          const bool spans = gpus.front() != gpus.back();
          const bool one_each = std::adjacent_find(gpus.begin(), gpus.end()) == gpus.end();
          if (spans && one_each && part.size(gi) > 2 && c->d_pad * c->esz > DSS_ONESHOT_MAX_BYTES) ok = false;
        }
        c->oneshot[t] = ok;
      }
      if (c->oneshot[0] || c->oneshot[1]) {
        c->oneshot_base_elems = ps;
        c->oneshot_base_flags = pf;
        c->oneshot_half_elems = static_cast<long>(c->P) * cfg->n_gpus * c->d_pad;
        c->oneshot_half_flags = static_cast<long>(c->P) * cfg->n_gpus * c->chain_nchunks;
        ps += 2 * c->oneshot_half_elems;
        pf += 2 * c->oneshot_half_flags;
      }
      c->push_buf = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(ps) * c->esz));
      c->push_flags = static_cast<unsigned long long*>(
          dalloc(c.get(), std::max<size_t>(64, sizeof(unsigned long long) * static_cast<size_t>(pf))));
      c->chain_flags = static_cast<unsigned long long*>(dalloc(
          c.get(), std::max<size_t>(64, sizeof(unsigned long long) * 2 * slots * c->chain_nchunks)));
    } else {
      c->peer_stats = {c->stats};
      build_plans(c.get());
    }
    ck(cudaStreamSynchronize(c->stream), "create sync");
    return DSS_OK;
  });
  if (st != DSS_OK) {
    g_last_global_error = c->last_error;
    dss_destroy(c.release());
    return st;
  }
  *out = c.release();
  return DSS_OK;
}

namespace {
void free_logistic(dss_ctx* c);
}  // namespace

extern "C" int dss_destroy(dss_ctx* c) {
  if (!c) return DSS_OK;
  if (c->cfg.device >= 0) cudaSetDevice(c->cfg.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocations) cudaFree(p);
  for (auto& pr : c->ev_pending) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->h_err) cudaFreeHost(c->h_err);
  free_logistic(c);
  if (c->copy_in) cudaStreamSynchronize(c->copy_in), cudaStreamDestroy(c->copy_in);
  if (c->copy_out) cudaStreamSynchronize(c->copy_out), cudaStreamDestroy(c->copy_out);
  for (cudaEvent_t e : {c->ev_in, c->ev_free, c->ev_snap, c->ev_out}) {
    if (e) cudaEventDestroy(e);
  }
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return DSS_OK;
}

extern "C" int dss_set_stream(dss_ctx* c, void* s) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(c->stream), "stream switch sync");
    c->stream = static_cast<cudaStream_t>(s);  // exactly this stream; NULL = legacy default stream
    return DSS_OK;
  });
}

extern "C" int dss_local_workers(const dss_ctx* c, int* first_rank, int* count) {
  if (!c || !first_rank || !count) return DSS_EINVAL;
  *first_rank = c->first;
  *count = c->P;
  return DSS_OK;
}

extern "C" long dss_row_stride(const dss_ctx* c) { return c ? c->d_pad : -1; }
extern "C" int dss_elem_size(const dss_ctx* c) { return c ? c->esz : -1; }

extern "C" int dss_device_ptr(dss_ctx* c, int buffer, int rank, void** out) {
  if (!c || !out) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    int lr = 0;
    check_rank(c, rank, &lr);
    const RowGeom gm = geom(c, buffer);
    *out = static_cast<char*>(gm.base) + static_cast<size_t>(lr) * gm.ld * c->esz;
    return DSS_OK;
  });
}

extern "C" int dss_upload(dss_ctx* c, int buffer, int rank, const void* host, long n) {
  if (!c || !host) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    int lr = 0;
    check_rank(c, rank, &lr);
    const RowGeom gm = geom(c, buffer);
    if (n < 0 || n > gm.len) throw std::invalid_argument("upload length exceeds the row length");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    char* dst = static_cast<char*>(gm.base) + static_cast<size_t>(lr) * gm.ld * c->esz;
    ck(cudaMemcpyAsync(dst, host, static_cast<size_t>(n) * c->esz, cudaMemcpyHostToDevice, c->stream),
       "upload");
    ck(cudaStreamSynchronize(c->stream), "upload sync");
    return DSS_OK;
  });
}

extern "C" int dss_download(dss_ctx* c, int buffer, int rank, void* host, long n) {
  if (!c || !host) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    int lr = 0;
    check_rank(c, rank, &lr);
    const RowGeom gm = geom(c, buffer);
    if (n < 0 || n > gm.len) throw std::invalid_argument("download length exceeds the row length");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const char* src = static_cast<const char*>(gm.base) + static_cast<size_t>(lr) * gm.ld * c->esz;
    ck(cudaMemcpyAsync(host, src, static_cast<size_t>(n) * c->esz, cudaMemcpyDeviceToHost, c->stream),
       "download");
    ck(cudaStreamSynchronize(c->stream), "download sync");
    return DSS_OK;
  });
}

extern "C" int dss_upload_all(dss_ctx* c, int buffer, const void* host) {
  if (!c || !host) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const RowGeom gm = geom(c, buffer);
    const size_t row = static_cast<size_t>(gm.len) * c->esz;
    ck(cudaMemcpy2DAsync(gm.base, static_cast<size_t>(gm.ld) * c->esz, host, row, row,
                         static_cast<size_t>(c->P), cudaMemcpyHostToDevice, c->stream),
       "upload_all");
    return DSS_OK;
  });
}

extern "C" int dss_download_all(dss_ctx* c, int buffer, void* host) {
  if (!c || !host) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const RowGeom gm = geom(c, buffer);
    const size_t row = static_cast<size_t>(gm.len) * c->esz;
    ck(cudaMemcpy2DAsync(host, row, gm.base, static_cast<size_t>(gm.ld) * c->esz, row,
                         static_cast<size_t>(c->P), cudaMemcpyDeviceToHost, c->stream),
       "download_all");
    ck(cudaStreamSynchronize(c->stream), "download_all sync");
    return DSS_OK;
  });
}

extern "C" int dss_broadcast_row(dss_ctx* c, int buffer, const void* host_row) {
  if (!c || !host_row) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const RowGeom gm = geom(c, buffer);
    char* base = static_cast<char*>(gm.base);
    const size_t row = static_cast<size_t>(gm.len) * c->esz;
    for (int k = 0; k < c->P; ++k) {
      ck(cudaMemcpyAsync(base + static_cast<size_t>(k) * gm.ld * c->esz, host_row, row,
                         cudaMemcpyHostToDevice, c->stream),
         "broadcast_row");
    }
    ck(cudaStreamSynchronize(c->stream), "broadcast sync");
    return DSS_OK;
  });
}

extern "C" int dss_set_step_count(dss_ctx* c, int rank, long step_count) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    int lr = 0;
    check_rank(c, rank, &lr);
    if (step_count < 0) throw std::invalid_argument("step_count must be >= 0");
    c->step_count[static_cast<size_t>(lr)] = step_count;
    return DSS_OK;
  });
}

extern "C" long dss_get_step_count(const dss_ctx* c, int rank) {
  if (!c || rank < c->first || rank >= c->first + c->P) return -1;
  return c->step_count[static_cast<size_t>(rank - c->first)];
}

// ------------------------------- hot path ------------------------------------

extern "C" int dss_step(dss_ctx* c, long t, double alpha, int check, dss_outcome* out) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (t < 0) throw std::invalid_argument("iteration must be >= 0");
    // run_training (sync.cpp:324-328) / check_step_args (optim.cpp:33-35)
    if (!std::isfinite(alpha) || alpha < 0.0) {
      throw std::invalid_argument("learning rate at t=" + std::to_string(t) + " must be finite and >= 0");
    }
    if (multi(c) && !c->attached) throw PeerError("multi-GPU context used before dss_ipc_attach");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const dss_strategy& s = c->cfg.strategy;
    const int opt = c->cfg.optimizer;
    if (s.kind == DSS_DS_SYNC) {
      const ParityPlan& pp = c->step_plan[t & 1];
      quiesce(c);
      // Local groups: fused apply_step + ordered fold + broadcast.
      for (const GroupLaunch& gl : pp.local) launch_groups_any(c, gl, opt, t, alpha, c->g, c->d_pad, 0);
      if (pp.any_spanning) {
        // Members of spanning groups step in place.  Two-shot groups: after
        // every GPU has stepped, each owner folds its slice over NVLink.
        // Chain groups: the ordered partial/mean passes (flag-synchronised
        // per chunk, no barrier).
        launch_groups_any(c, pp.spanning_step, opt, t, alpha, c->g, c->d_pad, 0);
        bool barrier_done = false;
        if (pp.any_push) {
          launch_push_any(c, pp.push, t, alpha);  // fused step + push two-shot
        } else if (pp.any_twoshot) {
          if (multi(c)) barrier(c);
          barrier_done = true;
          launch_fold_any(c, pp.fold, t);
        }
        if (pp.any_chain) launch_chain_any(c, pp.chain, t, alpha);
        // one-shot writes no peer params: the next iteration needs no barrier
        c->pending_remote = multi(c) && (pp.any_chain || !(pp.any_push && pp.push.oneshot));
        fold_stats(c, t, barrier_done);
      } else {
        fold_stats(c, t, false);
      }
    } else if (!multi(c)) {
      if (c->cfg.dtype == DSS_F64) {
        launch_bsp<double>(c, t, alpha);
      } else {
        launch_bsp<float>(c, t, alpha);
      }
      fold_stats(c, t, false);
    } else {
      // BSP over GPUs: barrier (gradients final everywhere), ordered fold of
      // all W gradients into every GPU's mean-gradient row, barrier, local
      // apply_step of every replica with the shared mean gradient.
      // Packed GPUs (P >= 2) use the ordered chain over the gradient rows
      // instead: every GPU forwards one partial row, not P rows.
      const ParityPlan& pp = c->step_plan[0];
      c->pending_remote = false;
      barrier(c);
      if (pp.any_twoshot) {
        launch_fold_any(c, pp.fold, t);
        barrier(c);
      }
      if (pp.any_chain) {
        launch_chain_any(c, pp.chain, t, alpha);  // fold -> replica step, fused per chunk
        c->pending_remote = true;
      } else {
        launch_groups_any(c, pp.spanning_step, opt, t, alpha, c->mg, 0, 1);
      }
      fold_stats(c, t, true);
    }
    bump_steps(c);
    if (out) *out = round_outcome(s, t, c->d + c->s);
    if (check) return check_impl(c);
    return DSS_OK;
  });
}

extern "C" int dss_step_host(dss_ctx* c, long t, double alpha, const void* host_grads, void* host_params) {
  if (!c || !host_grads || !host_params) return fail(c, DSS_EINVAL, "null argument");
  int st = guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    if (!c->host_pipe) {
      ck(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking), "copy stream");
      ck(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking), "copy stream");
      for (cudaEvent_t* e : {&c->ev_in, &c->ev_free, &c->ev_snap, &c->ev_out}) {
        ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
      }
      c->snapshot = dalloc(c, static_cast<size_t>(c->P) * c->d_pad * c->esz);
      ck(cudaEventRecord(c->ev_free, c->stream), "event");
      ck(cudaEventRecord(c->ev_out, c->copy_out), "event");
      c->host_pipe = true;
    }
    const size_t row = static_cast<size_t>(c->d) * c->esz;
    const size_t ld = static_cast<size_t>(c->d_pad) * c->esz;
    // copy-in: once the previous iteration no longer reads the gradients
    ck(cudaStreamWaitEvent(c->copy_in, c->ev_free, 0), "wait");
    ck(cudaMemcpy2DAsync(c->g, ld, host_grads, row, row, static_cast<size_t>(c->P), cudaMemcpyHostToDevice,
                         c->copy_in),
       "grads H2D");
    ck(cudaEventRecord(c->ev_in, c->copy_in), "event");
    ck(cudaStreamWaitEvent(c->stream, c->ev_in, 0), "wait");
    // the previous call's copy-out (running concurrently with this copy-in)
    // must land before we return: that is the API's completion point
    ck(cudaEventSynchronize(c->ev_out), "previous copy-out");
    return DSS_OK;
  });
  if (st != DSS_OK) return st;
  st = dss_step(c, t, alpha, 0, nullptr);
  if (st != DSS_OK) return st;
  return guard(c, [&]() -> int {
    const size_t row = static_cast<size_t>(c->d) * c->esz;
    const size_t ld = static_cast<size_t>(c->d_pad) * c->esz;
    quiesce(c);  // peers' mean stores into our rows (and reads of our grads) are done
    ck(cudaEventRecord(c->ev_free, c->stream), "event");
    ck(cudaStreamWaitEvent(c->stream, c->ev_out, 0), "wait");  // previous copy-out done with the snapshot
    ck(cudaMemcpyAsync(c->snapshot, c->w, static_cast<size_t>(c->P) * ld, cudaMemcpyDeviceToDevice, c->stream),
       "params snapshot");
    ck(cudaEventRecord(c->ev_snap, c->stream), "event");
    ck(cudaStreamWaitEvent(c->copy_out, c->ev_snap, 0), "wait");
    ck(cudaMemcpy2DAsync(host_params, row, c->snapshot, ld, row, static_cast<size_t>(c->P), cudaMemcpyDeviceToHost,
                         c->copy_out),
       "params D2H");
    ck(cudaEventRecord(c->ev_out, c->copy_out), "event");
    return DSS_OK;
  });
}

extern "C" int dss_host_sync(dss_ctx* c) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    if (c->host_pipe) {
      ck(cudaStreamSynchronize(c->copy_in), "copy-in sync");
      ck(cudaStreamSynchronize(c->copy_out), "copy-out sync");
    }
    ck(cudaStreamSynchronize(c->stream), "stream sync");
    return DSS_OK;
  });
}

namespace {

// Worlds small enough that one CTA beats one launch per iteration.
bool small_path(const dss_ctx* c, long n) {
  const long bytes = static_cast<long>(c->P) * c->d_pad * c->esz;
  return !multi(c) && c->cfg.path == 0 && c->s == 0 && n >= 2 && bytes <= 32768 && c->P <= kMaxLocal;
}

template <typename T, int OPT>
void launch_small_t(dss_ctx* c, const SmallArgs<T>& a) {
  TimedLaunch tl(c, c->cfg.strategy.kind == DSS_BSP ? DSS_KIND_BSP : DSS_KIND_GROUP);
  small_steps_kernel<T, OPT><<<1, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "small_steps_kernel launch");
}

LogisticArgs logistic_args(dss_ctx* c, long t);

template <typename T>
void run_small(dss_ctx* c, long t0, long n, const double* alphas, bool logistic = false) {
  const int P = c->P;
  const dss_strategy& s = c->cfg.strategy;
  if (!c->d_small_members[0]) {  // schedule tables of both parities, once
    for (int p = 0; p < 2; ++p) {
      const Partition part = make_partition(s, p);
      c->d_small_members[p] = upload_table(c, part.members);
      c->d_small_offsets[p] = upload_table(c, part.offsets);
      c->small_ngroups[p] = part.n_groups();
    }
  }
  const long need = n * (1 + 2L * P);
  if (need > c->small_cap) {
    c->d_small_buf = static_cast<double*>(dalloc(c, sizeof(double) * need));
    c->small_cap = need;
  }
  c->h_small.resize(static_cast<size_t>(need));
  double* ha = c->h_small.data();
  double* h1 = ha + n;
  double* h2 = h1 + n * P;
  const dss_hparams& h = c->cfg.hp;
  for (long i = 0; i < n; ++i) {
    ha[i] = alphas[i];
    for (int k = 0; k < P; ++k) {  // optim.cpp:76-78 per worker and iteration
      const double tt = static_cast<double>(c->step_count[static_cast<size_t>(k)] + i + 1);
      h1[i * P + k] = 1.0 - std::pow(h.beta1, tt);
      h2[i * P + k] = 1.0 - std::pow(h.beta2, tt);
    }
  }
  ck(cudaMemcpyAsync(c->d_small_buf, ha, sizeof(double) * need, cudaMemcpyHostToDevice, c->stream),
     "small-path tables");
  SmallArgs<T> a{};
  a.w = static_cast<T*>(c->w);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.nvec = c->d_pad / Vec<T>::n;
  a.nw = P;
  for (int p = 0; p < 2; ++p) {
    a.members[p] = c->d_small_members[p];
    a.offsets[p] = c->d_small_offsets[p];
    a.ngroups[p] = c->small_ngroups[p];
  }
  a.bsp = s.kind == DSS_BSP ? 1 : 0;
  a.t0 = t0;
  a.n = static_cast<int>(n);
  a.alpha = c->d_small_buf;
  a.bc1 = c->d_small_buf + n;
  a.bc2 = c->d_small_buf + n + n * P;
  a.wd = h.weight_decay;
  a.c = consts<T>(c, 0.0);
  a.err = c->d_err;
  if (logistic) {
    a.logistic = 1;
    a.lg = logistic_args(c, t0);
  }
  switch (c->cfg.optimizer) {
    case kSgd: launch_small_t<T, kSgd>(c, a); break;
    case kMomentum: launch_small_t<T, kMomentum>(c, a); break;
    case kAdam: launch_small_t<T, kAdam>(c, a); break;
    case kAdamW: launch_small_t<T, kAdamW>(c, a); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
  // the host table buffer is reused by the next call: wait for the copy
  ck(cudaStreamSynchronize(c->stream), "small-path sync");
  for (auto& sc : c->step_count) sc += n;
}

}  // namespace

extern "C" int dss_steps(dss_ctx* c, long t0, long n, const double* alphas, int check, dss_outcome* last) {
  if (!c || (!alphas && n > 0)) return fail(c, DSS_EINVAL, "null argument");
  if (small_path(c, n)) {
    const int st = guard(c, [&]() -> int {
      if (t0 < 0) throw std::invalid_argument("iteration must be >= 0");
      for (long i = 0; i < n; ++i) {
        if (!std::isfinite(alphas[i]) || alphas[i] < 0.0) {
          throw std::invalid_argument("learning rate at t=" + std::to_string(t0 + i) + " must be finite and >= 0");
        }
      }
      ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
      if (c->cfg.dtype == DSS_F64) {
        run_small<double>(c, t0, n, alphas);
      } else {
        run_small<float>(c, t0, n, alphas);
      }
      if (last) *last = round_outcome(c->cfg.strategy, t0 + n - 1, c->d + c->s);
      return DSS_OK;
    });
    if (st != DSS_OK) return st;
    if (check) return dss_check(c);
    return DSS_OK;
  }
  for (long i = 0; i < n; ++i) {
    const int st = dss_step(c, t0 + i, alphas[i], 0, last);
    if (st != DSS_OK) return st;
  }
  if (check) return dss_check(c);
  return DSS_OK;
}

extern "C" int dss_sync_round(dss_ctx* c, long t, int check, dss_outcome* out) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    const dss_strategy& s = c->cfg.strategy;
    validate_strategy(s);  // sync.cpp:270
    if (t < 0 && s.kind == DSS_DS_SYNC) throw std::invalid_argument("iteration must be >= 0");
    if (multi(c) && !c->attached) throw PeerError("multi-GPU context used before dss_ipc_attach");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const ParityPlan& pp = c->sync_plan[s.kind == DSS_DS_SYNC ? (t & 1) : 0];
    quiesce(c);
    const int phase = s.kind == DSS_BSP ? 0 : 1;  // collective failure: members[0] (sync.cpp:233-235)
    for (const GroupLaunch& gl : pp.local) launch_groups_any(c, gl, kOptNone, t, 0.0, nullptr, 0, 0, phase);
    if (pp.any_spanning) {
      if (pp.any_twoshot) {
        if (multi(c)) barrier(c);
        launch_fold_any(c, pp.fold, t);
      }
      if (pp.any_chain) launch_chain_any(c, pp.chain, t);
      c->pending_remote = multi(c);
    }
    fold_stats(c, t, pp.any_twoshot);
    if (out) *out = round_outcome(s, t, c->d + c->s);
    if (check) return check_impl(c);
    return DSS_OK;
  });
}

extern "C" int dss_running_stats_update(dss_ctx* c) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (c->s == 0) return DSS_OK;  // the problem has no running statistics (sync.cpp:194)
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    const long n = static_cast<long>(c->P) * c->s_pad;
    if (c->cfg.dtype == DSS_F64) {
      stats_ema_kernel<double><<<grid_x(c, n, 1), kThreads, 0, c->stream>>>(static_cast<double*>(c->stats),
                                                                          static_cast<const double*>(c->stats_obs), n);
    } else {
      stats_ema_kernel<float><<<grid_x(c, n, 1), kThreads, 0, c->stream>>>(static_cast<float*>(c->stats),
                                                                         static_cast<const float*>(c->stats_obs), n);
    }
    ck(cudaGetLastError(), "stats_ema_kernel launch");
    return DSS_OK;
  });
}

extern "C" int dss_apply_step(dss_ctx* c, double alpha, int check) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    if (!std::isfinite(alpha) || alpha < 0.0) {
      throw std::invalid_argument("apply_step: alpha must be finite and >= 0");  // optim.cpp:33-35
    }
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    launch_groups_any(c, c->apply_launch, c->cfg.optimizer, 0, alpha, c->g, c->d_pad, 0);
    bump_steps(c);
    if (check) return check_impl(c);
    return DSS_OK;
  });
}

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
        a.s0[k] = stream_state(seed, kGradientNoise, static_cast<uint64_t>(c->first + k), static_cast<uint64_t>(t));
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
    double *ws = nullptr, *u = nullptr, *ss = nullptr;
    ck(cudaMalloc(&ws, sizeof(double) * c->d), "cudaMalloc");
    ck(cudaMalloc(&u, sizeof(double) * c->d), "cudaMalloc");
    ck(cudaMalloc(&ss, sizeof(double)), "cudaMalloc");
    ck(cudaMemsetAsync(ss, 0, sizeof(double), c->stream), "memset");
    const int gx = grid_x(c, c->d, 1);
    gaussian_fill_kernel<<<gx, kThreads, 0, c->stream>>>(ws, c->d, stream_state(problem_seed, kDataGen, 1, 0));
    gaussian_fill_kernel<<<gx, kThreads, 0, c->stream>>>(u, c->d, stream_state(problem_seed, kInitParams, 0, 0));
    sumsq_kernel<<<gx, kThreads, 0, c->stream>>>(u, c->d, ss);
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
    cudaFree(ws);
    cudaFree(u);
    cudaFree(ss);
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

extern "C" int dss_global_mean(dss_ctx* c, void* host_mean) {
  if (!c || !host_mean) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (!c->mean_plan.built) throw std::invalid_argument("global mean supports at most 64 workers per GPU");
    if (multi(c) && !c->attached) throw PeerError("multi-GPU context used before dss_ipc_attach");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const ParityPlan& pp = c->mean_plan;
    quiesce(c);
    if (pp.any_twoshot) {
      if (multi(c)) barrier(c);
      launch_fold_any(c, pp.fold, 0);
      if (multi(c)) barrier(c);
    }
    if (pp.any_chain) {
      if (multi(c)) barrier(c);
      launch_chain_any(c, pp.chain, 0);
      if (multi(c)) c->pending_remote = true;
    }
    ck(cudaMemcpyAsync(host_mean, c->mg, static_cast<size_t>(c->d) * c->esz, cudaMemcpyDeviceToHost, c->stream),
       "global mean download");
    ck(cudaStreamSynchronize(c->stream), "global mean sync");
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
    std::vector<void*> ptrs;
    for (int k = 0; k < c->P; ++k) ptrs.push_back(static_cast<char*>(c->w) + static_cast<size_t>(k) * c->d_pad * c->esz);
    if (suboptimality) ptrs.push_back(c->mg);  // after dss_global_mean
    void** d_ptrs = upload_table(c, ptrs);
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
    cudaFree(d_ptrs);
    c->allocations.erase(std::find(c->allocations.begin(), c->allocations.end(), static_cast<void*>(d_ptrs)));
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

namespace {

void free_logistic(dss_ctx* c) {
  for (void* p : c->logi.mem) cudaFree(p);
  c->logi.mem.clear();
  c->logi.ready = false;
}

template <typename P>
P* logi_alloc(dss_ctx* c, size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(P)), "cudaMalloc");
  c->logi.mem.push_back(p);
  return static_cast<P*>(p);
}

// w as doubles [d] + the -y*s factors [batch]
size_t logistic_smem(long d, long batch) { return sizeof(double) * static_cast<size_t>(d + batch); }
constexpr long kLogisticMaxSmem = 200 * 1024;

}  // namespace

extern "C" int dss_logistic_setup(dss_ctx* c, const double* x, const double* y, int M, double l2, int batch_size,
                                  int sampling, uint64_t run_seed) {
  if (!c || !x || !y) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (M < 1) throw std::invalid_argument("logistic requires problem.M >= 1");
    if (!(l2 >= 0.0)) throw std::invalid_argument("problem.mu must be >= 0");
    if (batch_size < 1) throw std::invalid_argument("batch_size must be >= 1");
    if (sampling != DSS_SAMPLING_REPLACEMENT && sampling != DSS_SAMPLING_EPOCH) {
      throw std::invalid_argument("sampling must be replacement or epoch");
    }
    if (static_cast<long>(logistic_smem(c->d, batch_size)) > kLogisticMaxSmem) {
      throw std::invalid_argument("logistic on the device supports (dim + batch_size) * 8 B <= 200 KiB");
    }
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(c->stream), "stream sync");
    free_logistic(c);
    // make_shards over the whole world (sync.cpp:300); keep this GPU's rows
    std::vector<int> idx, off;
    make_shards(M, c->cfg.strategy.world_size, run_seed, idx, off);
    std::vector<int> local_off(static_cast<size_t>(c->P) + 1, 0);
    long max_shard = 0;
    for (int k = 0; k < c->P; ++k) {
      const int n = off[static_cast<size_t>(c->first + k) + 1] - off[static_cast<size_t>(c->first + k)];
      local_off[static_cast<size_t>(k) + 1] = local_off[static_cast<size_t>(k)] + n;
      max_shard = std::max<long>(max_shard, n);
    }
    auto& L = c->logi;
    const size_t xn = static_cast<size_t>(M) * c->d;
    L.x = logi_alloc<double>(c, xn);
    L.y = logi_alloc<double>(c, static_cast<size_t>(M));
    L.shard = logi_alloc<int>(c, static_cast<size_t>(local_off.back()));
    L.shard_off = logi_alloc<int>(c, local_off.size());
    L.order = logi_alloc<int>(c, static_cast<size_t>(c->P) * max_shard);
    L.order_epoch = logi_alloc<long>(c, static_cast<size_t>(c->P));
    L.batch = logi_alloc<int>(c, static_cast<size_t>(c->P) * batch_size);
    ck(cudaMemcpy(L.x, x, sizeof(double) * xn, cudaMemcpyHostToDevice), "logistic x upload");
    ck(cudaMemcpy(L.y, y, sizeof(double) * M, cudaMemcpyHostToDevice), "logistic y upload");
    ck(cudaMemcpy(L.shard, idx.data() + off[static_cast<size_t>(c->first)], sizeof(int) * local_off.back(),
                  cudaMemcpyHostToDevice), "shard upload");
    ck(cudaMemcpy(L.shard_off, local_off.data(), sizeof(int) * local_off.size(), cudaMemcpyHostToDevice),
       "shard upload");
    ck(cudaMemset(L.order_epoch, 0xff, sizeof(long) * c->P), "epoch init");  // -1
    ck(cudaMemset(L.batch, 0, sizeof(int) * c->P * batch_size), "batch init");
    if (logistic_smem(c->d, batch_size) > 48 * 1024) {
      ck(cudaFuncSetAttribute(logistic_grad_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(logistic_smem(c->d, batch_size))), "smem attr");
      ck(cudaFuncSetAttribute(logistic_grad_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(logistic_smem(c->d, batch_size))), "smem attr");
    }
    L.max_shard = max_shard;
    L.M = M;
    L.B = batch_size;
    L.sampling = sampling;
    L.l2 = l2;
    L.seed = run_seed;
    L.ready = true;
    return DSS_OK;
  });
}

namespace {

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
  a.d = static_cast<int>(c->d);
  a.B = L.B;
  a.sampling = L.sampling;
  a.l2 = L.l2;
  a.seed = L.seed;
  a.t = t;
  a.first_rank = c->first;
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
    if (!c->logi.ready) throw std::invalid_argument("dss_logistic_setup has not been called");
    if (t < 0) throw std::invalid_argument("iteration must be >= 0");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    quiesce(c);
    launch_logistic(c, t);
    return DSS_OK;
  });
}

extern "C" int dss_logistic_steps(dss_ctx* c, long t0, long n, const double* alphas, int check, dss_outcome* last) {
  if (!c || (!alphas && n > 0)) return fail(c, DSS_EINVAL, "null argument");
  if (small_path(c, n) && c->logi.ready && c->d <= kSmallLogiMaxDim && c->logi.B <= kSmallLogiMaxBatch) {
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
    if (!c->logi.ready) throw std::invalid_argument("dss_logistic_setup has not been called");
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

extern "C" int dss_check(dss_ctx* c) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    return check_impl(c);
  });
}

extern "C" int dss_clear_error(dss_ctx* c) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream), "err reset");
    ck(cudaMemsetAsync(c->d_gerr, 0xff, sizeof(unsigned long long), c->stream), "err reset");
    ck(cudaMemsetAsync(c->d_timeout, 0, sizeof(unsigned long long), c->stream), "timeout reset");
    ck(cudaStreamSynchronize(c->stream), "err reset sync");
    c->last_status = DSS_OK;
    c->last_error.clear();
    c->last_rank = -1;
    c->last_iteration = -1;
    return DSS_OK;
  });
}

extern "C" int dss_last_error(const dss_ctx* c, char* buf, size_t len, int* rank, long* iteration) {
  if (!c) {
    if (buf && len) std::snprintf(buf, len, "%s", g_last_global_error.c_str());
    return DSS_EINVAL;
  }
  if (buf && len) std::snprintf(buf, len, "%s", c->last_error.c_str());
  if (rank) *rank = c->last_rank;
  if (iteration) *iteration = c->last_iteration;
  return c->last_status;
}

extern "C" int dss_enable_timing(dss_ctx* c, int on) {
  if (!c) return DSS_EINVAL;
  c->timing = on != 0;
  return DSS_OK;
}

namespace {
void drain_events(dss_ctx* c) {
  ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
  ck(cudaStreamSynchronize(c->stream), "timing sync");
  for (size_t i = 0; i < c->ev_pending.size(); ++i) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->ev_pending[i].first, c->ev_pending[i].second), "cudaEventElapsedTime");
    c->kind_ms[c->ev_kind[i]] += ms;
    c->kind_n[c->ev_kind[i]] += 1;
    c->ev_pool.push_back(c->ev_pending[i].first);
    c->ev_pool.push_back(c->ev_pending[i].second);
  }
  c->ev_pending.clear();
  c->ev_kind.clear();
}
}  // namespace

extern "C" int dss_kernel_times(dss_ctx* c, double* total_ms, long* launches, double* max_launch_ms) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(c->stream), "timing sync");
    double tot = 0.0, mx = 0.0;
    for (size_t i = 0; i < c->ev_pending.size(); ++i) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, c->ev_pending[i].first, c->ev_pending[i].second), "cudaEventElapsedTime");
      tot += ms;
      mx = std::max(mx, static_cast<double>(ms));
    }
    const long n = static_cast<long>(c->ev_pending.size());
    drain_events(c);
    for (int k = 0; k < DSS_KIND_COUNT; ++k) {
      c->kind_ms[k] = 0.0;
      c->kind_n[k] = 0;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = n;
    if (max_launch_ms) *max_launch_ms = mx;
    return DSS_OK;
  });
}

extern "C" int dss_kernel_times_by_kind(dss_ctx* c, double* total_ms, long* launches) {
  if (!c || !total_ms || !launches) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    drain_events(c);
    for (int k = 0; k < DSS_KIND_COUNT; ++k) {
      total_ms[k] = c->kind_ms[k];
      launches[k] = c->kind_n[k];
      c->kind_ms[k] = 0.0;
      c->kind_n[k] = 0;
    }
    return DSS_OK;
  });
}

extern "C" long dss_launch_count(const dss_ctx* c) { return c ? c->launches : -1; }

// ------------------------------- multi-GPU -----------------------------------

extern "C" int dss_ipc_export(dss_ctx* c, void* out) {
  if (!c || !out) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    if (!multi(c)) throw std::invalid_argument("dss_ipc_export needs n_gpus > 1");
    cudaIpcMemHandle_t h[9];
    ck(cudaIpcGetMemHandle(&h[0], c->w), "cudaIpcGetMemHandle(params)");
    ck(cudaIpcGetMemHandle(&h[1], c->g), "cudaIpcGetMemHandle(grads)");
    ck(cudaIpcGetMemHandle(&h[2], c->mg), "cudaIpcGetMemHandle(mean grad)");
    ck(cudaIpcGetMemHandle(&h[3], c->flags), "cudaIpcGetMemHandle(flags)");
    ck(cudaIpcGetMemHandle(&h[4], c->chain_buf), "cudaIpcGetMemHandle(chain rows)");
    ck(cudaIpcGetMemHandle(&h[5], c->chain_flags), "cudaIpcGetMemHandle(chain flags)");
    ck(cudaIpcGetMemHandle(&h[6], c->stats), "cudaIpcGetMemHandle(running stats)");
    ck(cudaIpcGetMemHandle(&h[7], c->push_buf), "cudaIpcGetMemHandle(push staging)");
    ck(cudaIpcGetMemHandle(&h[8], c->push_flags), "cudaIpcGetMemHandle(push flags)");
    std::memcpy(out, h, sizeof(h));
    return DSS_OK;
  });
}

extern "C" int dss_ipc_attach(dss_ctx* c, const void* all) {
  if (!c || !all) return fail(c, DSS_EINVAL, "null argument");
  return guard(c, [&]() -> int {
    if (!multi(c)) throw std::invalid_argument("dss_ipc_attach needs n_gpus > 1");
    if (c->attached) throw std::invalid_argument("already attached");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const int G = c->cfg.n_gpus;
    c->peer_w.assign(static_cast<size_t>(G), nullptr);
    c->peer_g.assign(static_cast<size_t>(G), nullptr);
    c->peer_mg.assign(static_cast<size_t>(G), nullptr);
    c->peer_flag.assign(static_cast<size_t>(G), nullptr);
    c->peer_chain_buf.assign(static_cast<size_t>(G), nullptr);
    c->peer_chain_flags.assign(static_cast<size_t>(G), nullptr);
    c->peer_stats.assign(static_cast<size_t>(G), nullptr);
    c->peer_push_buf.assign(static_cast<size_t>(G), nullptr);
    c->peer_push_flags.assign(static_cast<size_t>(G), nullptr);
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(all);
    for (int r = 0; r < G; ++r) {
      if (r == c->cfg.rank) {
        c->peer_w[static_cast<size_t>(r)] = c->w;
        c->peer_g[static_cast<size_t>(r)] = c->g;
        c->peer_mg[static_cast<size_t>(r)] = c->mg;
        c->peer_flag[static_cast<size_t>(r)] = c->flags;
        c->peer_chain_buf[static_cast<size_t>(r)] = c->chain_buf;
        c->peer_chain_flags[static_cast<size_t>(r)] = c->chain_flags;
        c->peer_stats[static_cast<size_t>(r)] = c->stats;
        c->peer_push_buf[static_cast<size_t>(r)] = c->push_buf;
        c->peer_push_flags[static_cast<size_t>(r)] = c->push_flags;
        continue;
      }
      void* p[9];
      for (int b = 0; b < 9; ++b) {
        cudaError_t e = cudaIpcOpenMemHandle(&p[b], h[r * 9 + b], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          throw PeerError("cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + cudaGetErrorString(e));
        }
        c->opened.push_back(p[b]);
      }
      c->peer_w[static_cast<size_t>(r)] = p[0];
      c->peer_g[static_cast<size_t>(r)] = p[1];
      c->peer_mg[static_cast<size_t>(r)] = p[2];
      c->peer_flag[static_cast<size_t>(r)] = static_cast<unsigned long long*>(p[3]);
      c->peer_chain_buf[static_cast<size_t>(r)] = p[4];
      c->peer_chain_flags[static_cast<size_t>(r)] = static_cast<unsigned long long*>(p[5]);
      c->peer_stats[static_cast<size_t>(r)] = p[6];
      c->peer_push_buf[static_cast<size_t>(r)] = p[7];
      c->peer_push_flags[static_cast<size_t>(r)] = static_cast<unsigned long long*>(p[8]);
    }
    c->d_peer_flags = upload_table(c, c->peer_flag);
    build_plans(c);
    c->attached = true;
    barrier(c);
    ck(cudaStreamSynchronize(c->stream), "attach sync");
    return check_impl(c) == DSS_OK ? DSS_OK : c->last_status;
  });
}

extern "C" int dss_barrier(dss_ctx* c) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    barrier(c);
    return DSS_OK;
  });
}
