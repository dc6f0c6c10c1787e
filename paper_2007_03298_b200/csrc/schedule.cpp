// Host schedule: restates /root/reference/proj/src/schedule.cpp:8-90 and
// sync.cpp:47-66,131-141 (same rules, same error wording), plus the
// rectangular W = N*K extension and the multi-GPU two-shot plan.
#include "schedule.hpp"

#include <algorithm>
#include <cstdio>

namespace dssb {

namespace {

bool is_power_of_two(long n) { return n > 0 && (n & (n - 1)) == 0; }

}  // namespace

void validate_world(int world_size, int group_size, bool rectangular) {
  // schedule.cpp:9-16
  if (world_size < 1) {
    throw std::invalid_argument("world_size must be >= 1 (got " + std::to_string(world_size) + ")");
  }
  if (group_size < 1) {
    throw std::invalid_argument("group_size must be >= 1 (got " + std::to_string(group_size) + ")");
  }
  const long n = group_size;
  if (rectangular) {
    if (world_size % group_size != 0) {
      throw std::invalid_argument(
          "rectangular schedule needs world_size to be a multiple of group_size (got world_size=" +
          std::to_string(world_size) + ", group_size=" + std::to_string(group_size) + ")");
    }
    return;
  }
  // schedule.cpp:17-23
  if (world_size != n * n && world_size != group_size) {
    throw std::invalid_argument(
        "world_size must equal group_size^2, or group_size for a single full group (got "
        "world_size=" +
        std::to_string(world_size) + ", group_size=" + std::to_string(group_size) + ")");
  }
}

bool is_square_mode(int world_size, int group_size) {
  // schedule.cpp:26-29
  const long n = group_size;
  return world_size == n * n && world_size != group_size;
}

void validate_strategy(const dss_strategy& s) {
  // sync.cpp:47-66
  validate_world(s.world_size, s.group_size, s.rectangular != 0);
  if (s.kind == DSS_BSP && s.group_size != s.world_size) {
    throw std::invalid_argument(
        "bsp runs one group spanning the world; set group_size equal to world_size");
  }
  if (s.kind == DSS_DS_SYNC && s.topology == DSS_PS) {
    throw std::invalid_argument("ds-sync has no parameter-server variant; use topology ring or tree");
  }
  if (s.topology == DSS_TREE && !is_power_of_two(s.group_size)) {
    throw std::invalid_argument("tree topology requires power-of-two groups (group_size=" +
                                std::to_string(s.group_size) + ")");
  }
  if (s.topology == DSS_TREE && s.rectangular && s.world_size != s.group_size &&
      !is_power_of_two(s.world_size / s.group_size)) {
    throw std::invalid_argument("tree topology requires power-of-two groups (comb size=" +
                                std::to_string(s.world_size / s.group_size) + ")");
  }
  if (s.topology == DSS_PS && s.num_servers < 1) {
    throw std::invalid_argument("ps topology needs num_servers >= 1 (got " +
                                std::to_string(s.num_servers) + ")");
  }
  if (s.kind != DSS_BSP && s.kind != DSS_DS_SYNC) throw std::invalid_argument("unknown strategy");
  if (s.topology < DSS_RING || s.topology > DSS_PS) throw std::invalid_argument("unknown topology");
}

Partition make_partition(const dss_strategy& s, long t) {
  const int W = s.world_size;
  Partition part;
  part.iteration = t;
  if (s.kind == DSS_BSP) {
    // partition_for (sync.cpp:131-139): one all-world group, no validation
    // beyond the caller's validate(strategy).
    part.members.resize(static_cast<size_t>(W));
    for (int x = 0; x < W; ++x) part.members[static_cast<size_t>(x)] = x;
    part.offsets = {0, W};
    return part;
  }
  validate_world(W, s.group_size, s.rectangular != 0);  // schedule.cpp:32
  if (t < 0) throw std::invalid_argument("iteration must be >= 0");  // schedule.cpp:33

  const int n = s.group_size;
  const bool single = (W == n);  // single-group layout (schedule.cpp:38-43)
  if (single || W == 1) {
    part.members.resize(static_cast<size_t>(W));
    for (int x = 0; x < W; ++x) part.members[static_cast<size_t>(x)] = x;
    part.offsets = {0, W};
    return part;
  }
  // Square mode: g(x) = t even ? x / n : x % n (schedule.cpp:45-50).  The
  // rectangular extension uses the same rule with W = n * k: k blocks of n
  // on even t, n combs of k on odd t.  Visiting x ascending and bucketing
  // keeps every group ascending by construction (schedule.cpp:52).
  const int k = W / n;
  const bool even = (t % 2 == 0);
  const int groups = even ? k : n;
  const int size = even ? n : k;
  part.members.resize(static_cast<size_t>(W));
  part.offsets.resize(static_cast<size_t>(groups) + 1);
  for (int g = 0; g <= groups; ++g) part.offsets[static_cast<size_t>(g)] = g * size;
  std::vector<int> fill(static_cast<size_t>(groups), 0);
  for (int x = 0; x < W; ++x) {
    const int g = even ? x / n : x % n;
    part.members[static_cast<size_t>(g * size + fill[static_cast<size_t>(g)]++)] = x;
  }
  return part;
}

std::vector<int> group_of(const dss_strategy& s, long t, int rank) {
  // schedule.cpp:56-65
  if (rank < 0 || rank >= s.world_size) {
    throw std::invalid_argument("rank out of range: " + std::to_string(rank));
  }
  const Partition p = make_partition(s, t);
  for (int g = 0; g < p.n_groups(); ++g) {
    const int* b = p.group(g);
    if (std::find(b, b + p.size(g), rank) != b + p.size(g)) return std::vector<int>(b, b + p.size(g));
  }
  throw std::logic_error("partition does not cover rank");
}

bool check_mixing(const dss_strategy& s, long t) {
  // schedule.cpp:67-90: every group at t meets every group at t+1 in exactly
  // one worker (linear merge of two sorted lists).
  const Partition now = make_partition(s, t);
  const Partition next = make_partition(s, t + 1);
  for (int a = 0; a < now.n_groups(); ++a) {
    for (int b = 0; b < next.n_groups(); ++b) {
      const int* x = now.group(a);
      const int* y = next.group(b);
      int i = 0, j = 0, common = 0;
      while (i < now.size(a) && j < next.size(b)) {
        if (x[i] == y[j]) {
          ++common;
          ++i;
          ++j;
        } else if (x[i] < y[j]) {
          ++i;
        } else {
          ++j;
        }
      }
      if (common != 1) return false;
    }
  }
  return true;
}

namespace {

// Serial steps and messages of one collective over m members (comm.cpp).
void collective_counts(int topology, long m, int servers, long dim, long* steps, long* msgs) {
  if (topology == DSS_RING) {  // comm.cpp:78-123: 2m-1 hops, lone member none
    *steps = m == 1 ? 0 : 2 * m - 1;
    *msgs = *steps;
  } else if (topology == DSS_TREE) {  // comm.cpp:125-214
    if (m == 1) {
      *steps = 0;
      *msgs = 0;
      return;
    }
    long depth = 0;
    while ((1L << depth) < m) ++depth;
    *steps = 3 * depth;
    *msgs = m * depth + 2 * (m - 1);
  } else {  // ps, comm.cpp:216-289: 2m serial steps, every non-empty slice pushed and pulled
    const long nonempty = std::min<long>(servers, dim);
    *steps = 2 * m;
    *msgs = 2 * m * nonempty;
  }
}

}  // namespace

dss_outcome round_outcome(const dss_strategy& s, long t, long payload_dim) {
  // sync_round (sync.cpp:276-281): max serial steps over groups, sum of messages.
  const Partition p = make_partition(s, t);
  dss_outcome out{0, 0};
  for (int g = 0; g < p.n_groups(); ++g) {
    long steps = 0, msgs = 0;
    collective_counts(s.topology, p.size(g), s.num_servers, payload_dim, &steps, &msgs);
    out.critical_path_steps = std::max(out.critical_path_steps, steps);
    out.total_messages += msgs;
  }
  return out;
}

void slice_range(long d_pad, int s, int j, long* lo, long* hi) {
  // Near-equal contiguous slices (sizes differ by at most one chunk), the
  // same split rule the reference's parameter servers use (comm.cpp:229-236).
  const long chunks = d_pad / kRowAlign;
  const long base = chunks / s;
  const long rem = chunks % s;
  const long c0 = j * base + std::min<long>(j, rem);
  const long c1 = c0 + base + (j < rem ? 1 : 0);
  *lo = c0 * kRowAlign;
  *hi = c1 * kRowAlign;
}

Tiling choose_tiling(const dss_strategy& s, int G) {
  Tiling best;
  const int W = s.world_size, N = s.group_size;
  if (s.kind != DSS_DS_SYNC || G <= 1 || N <= 0 || W == N || W % N != 0) return best;
  const int K = W / N;
  long best_busy = -1, best_total = -1;
  for (int gr = G; gr >= 1; --gr) {  // larger gr first: ties keep whole blocks on a GPU
    if (G % gr) continue;
    const int gc = G / gr;
    if (K % gr || N % gc) continue;
    const long even = static_cast<long>(K) * (gc - 1);  // K blocks, each over gc GPUs
    const long odd = static_cast<long>(N) * (gr - 1);   // N combs, each over gr GPUs
    const long busy = std::max(even, odd), total = even + odd;
    if (best_busy < 0 || busy < best_busy || (busy == best_busy && total < best_total)) {
      best = {gr, gc};
      best_busy = busy;
      best_total = total;
    }
  }
  return best;
}

Tiling choose_placement(const dss_strategy& s, int G, int mode, long row_bytes, long oneshot_bytes) {
  if (mode == 0 || G <= 1) return Tiling{};
  if (mode == 1) return choose_tiling(s, G);
  if (oneshot_bytes > 0 && row_bytes > 0 && row_bytes <= oneshot_bytes) return Tiling{};
  // auto: is there a deep chain under contiguous packing?
  const int W = s.world_size, P = W / G;
  bool deep_chain = false;
  for (long t = 0; t < 2 && !deep_chain && s.kind == DSS_DS_SYNC; ++t) {
    const Partition part = make_partition(s, t);
    for (int g = 0; g < part.n_groups() && !deep_chain; ++g) {
      std::vector<int> per(static_cast<size_t>(G), 0);
      for (int j = 0; j < part.size(g); ++j) ++per[static_cast<size_t>(part.group(g)[j] / P)];
      int span = 0, most = 0;
      for (int x : per) {
        span += x > 0;
        most = std::max(most, x);
      }
      deep_chain = span >= 3 && most >= 2;
    }
  }
  return deep_chain ? choose_tiling(s, G) : Tiling{};
}

std::vector<int> placement_slots(const dss_strategy& s, int G, const Tiling& t) {
  const int W = s.world_size;
  std::vector<int> slot(static_cast<size_t>(W));
  if (t.gr == 0) {
    for (int k = 0; k < W; ++k) slot[static_cast<size_t>(k)] = k;
    return slot;
  }
  const int N = s.group_size, K = W / N, P = W / G;
  const int Kt = K / t.gr, Nt = N / t.gc;
  for (int k = 0; k < W; ++k) {
    const int b = k / N, c = k % N;
    const int gpu = (b / Kt) * t.gc + c / Nt;
    slot[static_cast<size_t>(k)] = gpu * P + (b % Kt) * Nt + c % Nt;
  }
  return slot;
}

Partition to_slots(const Partition& part, const std::vector<int>& slot_of) {
  Partition out = part;
  for (int& m : out.members) m = slot_of[static_cast<size_t>(m)];
  return out;
}

GpuPlan make_plan(const Partition& part, int world_size, int n_gpus, int rank, long d_pad, bool force_chain,
                  bool no_chain) {
  GpuPlan plan;
  const int per = world_size / n_gpus;
  std::vector<int> slots_used(static_cast<size_t>(n_gpus), 0);
  // chain slot of (gpu, group): index of the group among the chain groups
  // that include that GPU, in ascending group order -- every rank computes
  // the same table, so senders know their receivers' slots.
  std::vector<std::vector<int>> slot_of(static_cast<size_t>(part.n_groups()));
  for (int g = 0; g < part.n_groups(); ++g) {
    const int* mem = part.group(g);
    const int m = part.size(g);
    std::vector<int> gpus;   // ascending, distinct (members are ascending)
    std::vector<int> count;  // members per GPU
    for (int j = 0; j < m; ++j) {
      const int gpu = mem[j] / per;
      if (gpus.empty() || gpus.back() != gpu) {
        gpus.push_back(gpu);
        count.push_back(0);
      }
      ++count.back();
    }
    const bool spanning = gpus.size() > 1;
    if (spanning) plan.any_spanning_globally = true;
    const bool chain =
        spanning && !no_chain && (force_chain || *std::max_element(count.begin(), count.end()) >= 2);
    slot_of[static_cast<size_t>(g)].assign(static_cast<size_t>(n_gpus), -1);
    if (chain) {
      plan.any_chain_globally = true;
      for (int gpu : gpus) slot_of[static_cast<size_t>(g)][static_cast<size_t>(gpu)] = slots_used[static_cast<size_t>(gpu)]++;
    } else if (spanning) {
      plan.any_twoshot_globally = true;
    }
    const auto it = std::find(gpus.begin(), gpus.end(), rank);
    if (it == gpus.end()) continue;
    if (!spanning) {
      plan.local_groups.push_back(g);
      continue;
    }
    plan.spanning_groups.push_back(g);
    for (int j = 0; j < m; ++j) {
      if (mem[j] / per == rank) plan.spanning_local_members.push_back(mem[j]);
    }
    const int S = static_cast<int>(gpus.size());
    const int pos = static_cast<int>(it - gpus.begin());
    if (chain) {
      ChainRole r;
      r.group = g;
      r.stage = pos;
      r.S = S;
      r.m = m;
      r.first_member = mem[0];
      for (int j = 0; j < m; ++j) {
        if (mem[j] / per == rank) r.run.push_back(mem[j]);
      }
      if (pos + 1 < S) r.next_gpu = gpus[static_cast<size_t>(pos + 1)];
      if (pos == S - 1) {
        r.mean_next_gpu = gpus[0];
      } else if (pos + 1 <= S - 2) {
        r.mean_next_gpu = gpus[static_cast<size_t>(pos + 1)];
      }
      plan.chain.push_back(r);
      continue;
    }
    Slice sl;
    sl.group = g;
    slice_range(d_pad, S, pos, &sl.lo, &sl.hi);
    if (sl.hi > sl.lo) plan.owned.push_back(sl);
  }
  for (ChainRole& r : plan.chain) {
    const auto& so = slot_of[static_cast<size_t>(r.group)];
    r.slot = so[static_cast<size_t>(rank)];
    if (r.next_gpu >= 0) r.next_slot = so[static_cast<size_t>(r.next_gpu)];
    if (r.mean_next_gpu >= 0) r.mean_next_slot = so[static_cast<size_t>(r.mean_next_gpu)];
  }
  plan.max_chain_slots = *std::max_element(slots_used.begin(), slots_used.end());
  std::sort(plan.spanning_local_members.begin(), plan.spanning_local_members.end());
  return plan;
}

}  // namespace dssb
