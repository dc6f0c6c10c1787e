// Host-side divide-and-shuffle schedule and the multi-GPU launch plan.
//
// The schedule is computed on the host exactly as the reference computes it
// (/root/reference/proj/src/schedule.cpp:8-90, sync.cpp:47-66,131-141) so
// group membership is bit-exact every iteration; the device only ever sees
// the resulting CSR tables.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "dssync_b200.h"

namespace dssb {

// Row padding in elements: 64 elements = 256 B (f32) / 512 B (f64), so every
// worker row starts on a 256-B boundary and holds whole 16/32-B vectors.
constexpr long kRowAlign = 64;

inline long pad_dim(long d) { return (d + kRowAlign - 1) / kRowAlign * kRowAlign; }

// CSR partition: groups[g] = members[offsets[g] .. offsets[g+1]), ascending.
struct Partition {
  long iteration = 0;
  std::vector<int> members;
  std::vector<int> offsets;
  int n_groups() const { return static_cast<int>(offsets.size()) - 1; }
  int size(int g) const { return offsets[g + 1] - offsets[g]; }
  const int* group(int g) const { return members.data() + offsets[g]; }
};

// validate(WorldConfig) (schedule.cpp:8-24).  rectangular relaxes the
// shape rule to W % N == 0 (builder extension).
void validate_world(int world_size, int group_size, bool rectangular);
bool is_square_mode(int world_size, int group_size);
// validate(SyncStrategy) (sync.cpp:47-66).
void validate_strategy(const dss_strategy& s);

// make_partition (schedule.cpp:31-54) for DS-Sync; partition_for
// (sync.cpp:131-141) returns the single all-world group under BSP.
Partition make_partition(const dss_strategy& s, long t);
std::vector<int> group_of(const dss_strategy& s, long t, int rank);
bool check_mixing(const dss_strategy& s, long t);

// Closed-form SyncRoundOutcome (comm.cpp:78-289 step/message counts).
dss_outcome round_outcome(const dss_strategy& s, long t, long payload_dim);

// ---------------------------------------------------------------------------
// Multi-GPU plan.  W workers packed contiguously over G GPUs, P = W / G per
// GPU, gpu(k) = k / P.  A group whose members all sit on one
// GPU is folded there by the fused step kernel.  A group spanning S GPUs is
// two-shot: every member GPU steps its own members in place, then the GPU at
// position j of the group's (ascending) GPU list owns the j-th of S
// near-equal slices of the padded row (in kRowAlign chunks) and folds that
// slice over all members in ascending rank order, writing the mean to every
// member.  One owner per element keeps the reference's fold order exactly.
struct Slice {
  int group = 0;  // index in the Partition
  long lo = 0;    // element range [lo, hi) of the padded row
  long hi = 0;
};

// A spanning group with several members on some GPU is folded by the
// ordered chain instead (kernels.cuh chain_*): this GPU's role in it.
struct ChainRole {
  int group = 0;        // index in the Partition
  int slot = 0;         // this GPU's receive-buffer slot for the group
  int stage = 0;        // position j in the group's ascending GPU list
  int S = 0;            // GPUs spanned
  int m = 0;            // members
  int first_member = 0;
  std::vector<int> run; // this GPU's members, ascending (contiguous in the fold order)
  int next_gpu = -1;    // partial pass successor (stage j+1), -1 at the last stage
  int next_slot = -1;
  int mean_next_gpu = -1;  // mean pass successor: last -> g_0 -> g_1 -> ... -> g_{S-2}
  int mean_next_slot = -1;
};

struct GpuPlan {
  std::vector<int> local_groups;     // groups entirely on this GPU
  std::vector<int> spanning_groups;  // groups with members here and elsewhere
  std::vector<int> spanning_local_members;  // this GPU's members of spanning groups (ascending)
  std::vector<Slice> owned;          // two-shot slices this GPU folds
  std::vector<ChainRole> chain;      // chain-fold groups this GPU takes part in
  bool any_spanning_globally = false;  // some group spans GPUs
  bool any_twoshot_globally = false;   // some spanning group is two-shot (barrier before the fold)
  bool any_chain_globally = false;
  int max_chain_slots = 0;           // over all GPUs: receive slots needed
};

// ---------------------------------------------------------------------------
// Worker placement over G GPUs.  Slot v = gpu * P + local row.  Contiguous
// packing is slot(k) = k.  The tiled placement (DS-Sync only, W = N * K:
// block b = k / N, comb c = k % N, a K x N grid) cuts the grid into
// gr x gc tiles of (K/gr) x (N/gc) workers, one tile per GPU, local rows in
// ascending rank order.  Every block then spans gc GPUs and every comb gr
// GPUs, each GPU's members of a group forming one contiguous run of the
// ascending fold order (what the chain fold needs).  choose_tiling picks the
// (gr, gc) with the fewest cross-GPU row transfers in the busier parity
// (sum over groups of 2 (S - 1) rows), then the fewest overall.
struct Tiling {
  int gr = 0, gc = 0;  // 0: contiguous packing
};
Tiling choose_tiling(const dss_strategy& s, int n_gpus);
// placement mode 2 (auto): the tiling only where contiguous packing leaves an
// ordered chain three or more GPUs deep (a group with several members on a
// GPU that spans >= 3 GPUs: C3 / C4 on 4 GPUs); contiguous packing otherwise
// (its one-member-per-GPU groups take the push two-shot, which measured
// faster than the chains a tiling would create: C2 on 4 GPUs 3501 vs 3103
// iters/s, profiles/r02/placement_ab_g4.jsonl).
// Rows of at most `oneshot_bytes` (the one-shot regime, 0 = no limit) stay
// contiguous in auto mode too: there contiguous packing keeps one parity
// GPU-local while a tiling makes both parities exchange (W=64 on 4 GPUs at
// 1 KB-256 KB: 0.53-0.73x, profiles/r02/sweeps/).
Tiling choose_placement(const dss_strategy& s, int n_gpus, int mode, long row_bytes = 0, long oneshot_bytes = 0);
// slot_of[k] for every global rank k (identity for contiguous packing).
std::vector<int> placement_slots(const dss_strategy& s, int n_gpus, const Tiling& t);
// The partition with every member replaced by its slot (member order, i.e.
// the ascending-rank fold order, kept).
Partition to_slots(const Partition& part, const std::vector<int>& slot_of);

// force_chain: every spanning group takes the chain path (tests); otherwise
// only groups with >= 2 members on some GPU (where the chain moves fewer
// NVLink bytes than the two-shot).  no_chain: no group takes the chain (a
// one-shot parity: every spanning group is gathered whole by every member
// GPU).
GpuPlan make_plan(const Partition& part, int world_size, int n_gpus, int rank, long d_pad,
                  bool force_chain = false, bool no_chain = false);

// [lo, hi) of the j-th of s near-equal chunk-aligned slices of [0, d_pad).
void slice_range(long d_pad, int s, int j, long* lo, long* hi);

}  // namespace dssb
