// The engine behind the C ABI: launch tables built from the host schedule
// (per parity: fused local groups, two-shot / one-shot push, ordered chain),
// kernel dispatch, and the cross-GPU flow pieces (barrier, quiesce, the
// running-stats fold, the divergence check).
#include "context.cuh"

namespace dssb {

thread_local std::string g_last_global_error;

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
  gl.members = members;
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


// Staging layout of GPU q's owned two-shot slices at parity t: for each
// owned slice (plan order) its group, S, [lo, hi), element offset in q's
// staging buffer (S rows of hi-lo) and flag offset (S rows of n_chunks).
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
// Flags: [parity][region][slot][chunk] (one parity unless chain_split).
unsigned long long* chain_flag(dss_ctx* c, unsigned long long* base, int region, int slot, int parity = 0) {
  return base + (static_cast<size_t>(parity * 2 + region) * c->chain_slots + slot) * c->chain_nchunks;
}

// Chain-fold launch tables for this GPU's roles.  members of role i are
// rows of `member_base` (local); its mean lands in dsts[i] (local rows).
// inplace (a Partition, params rows): the mean travels straight into the
// receiving GPU's first member row of the group instead of a receive row,
// and the mean pass there copies it to the other members (one row write
// less per group and GPU).
ChainLaunch build_chain(dss_ctx* c, const std::vector<ChainRole>& roles, void* member_base,
                        const std::vector<std::vector<void*>>& dsts, int err_phase, int opt_mem = kOptNone,
                        int opt_dst = kOptNone, const std::vector<std::vector<int>>& dst_lrs = {},
                        const Partition* inplace = nullptr, int parity = 0) {
  // chain_split (DS, in-place means): parity 1's partials use the region-1
  // rows (free: the means land in the members' rows) and its own flags
  const int pf = c->chain_split ? parity : 0;
  const int prow = pf ? 1 : 0;
  if (pf && !inplace) throw std::logic_error("chain: parity-split rows need in-place means");
  auto first_member_row = [&](int group, int gpu) -> void* {
    const int* mem = inplace->group(group);
    for (int q = 0; q < inplace->size(group); ++q) {
      if (mem[q] / c->P == gpu) return row_ptr(c, c->peer_w, mem[q]);
    }
    throw std::logic_error("chain: receiver holds no member of the group");
  };
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
    a.recv = chain_row(c, c->chain_buf, prow, r.slot);
    a.recv_flags = chain_flag(c, c->chain_flags, 0, r.slot, pf);
    if (!a.last) {
      a.send = chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.next_gpu)], prow, r.next_slot);
      a.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.next_gpu)], 0, r.next_slot, pf);
    } else {
      a.send = inplace ? first_member_row(r.group, r.mean_next_gpu)
                       : chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
      a.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot, pf);
    }
    a.err_rank = grank(c, r.first_member);
    a.err_phase = err_phase;
    a.m = r.m;
    ea.push_back(a);
    if (r.stage <= r.S - 2) {
      ChainEntry b = a;
      b.last = 0;
      b.recv = inplace ? dsts[i][0] : chain_row(c, c->chain_buf, 1, r.slot);
      b.dst_skip = inplace ? 1 : 0;
      b.recv_flags = chain_flag(c, c->chain_flags, 1, r.slot, pf);
      if (r.stage < r.S - 2) {
        b.send = inplace ? first_member_row(r.group, r.mean_next_gpu)
                         : chain_row(c, c->peer_chain_buf[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot);
        b.send_flags = chain_flag(c, c->peer_chain_flags[static_cast<size_t>(r.mean_next_gpu)], 1, r.mean_next_slot, pf);
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
  cl.hb = eb;
  cl.hdst = dst;
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
        it.rank = grank(c, my_member);
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
      f.err_rank = grank(c, mem[0]);
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

// One-shot tables of parity t for this GPU.  Every member's stepped row
// goes to every GPU of its group: row slot * R + q of GPU o's staging, with
// slot = the local row there of the group's first member on o, q the
// member's position in the group and R the largest group size.  Every GPU
// then folds all m rows of each of its groups in member order and stores
// the mean into its own members only.
PushLaunch build_oneshot(dss_ctx* c, const Partition& part) {
  PushLaunch pl;
  pl.oneshot = true;
  const int G = c->cfg.n_gpus;
  const int me = c->cfg.rank;
  const long CH = c->chain_chunk;
  const long nch = c->chain_nchunks;
  const long R = c->oneshot_rows;
  const GpuPlan gp = make_plan(part, c->cfg.strategy.world_size, G, me, c->d_pad, force_chain(c), true);
  std::vector<PushItem> items;
  std::vector<void*> item_dst;
  std::vector<unsigned long long*> item_flag;
  std::vector<int> item_gpu;
  std::vector<PushFold> folds;
  std::vector<void*> dst;
  std::vector<int> dst_lr;
  for (int gi : gp.spanning_groups) {
    const int* mem = part.group(gi);
    const int m = part.size(gi);
    if (m > R) throw std::logic_error("one-shot: group larger than the staging rows");
    std::vector<int> gpus, slot;  // distinct GPUs of the group and the group's slot on each
    for (int q = 0; q < m; ++q) {
      const int gpu = mem[q] / c->P;
      if (gpus.empty() || gpus.back() != gpu) {
        gpus.push_back(gpu);
        slot.push_back(mem[q] - gpu * c->P);
      }
    }
    const int S = static_cast<int>(gpus.size());
    int j = -1;  // my position among the group's GPUs
    for (int o = 0; o < S; ++o) j = gpus[static_cast<size_t>(o)] == me ? o : j;
    if (j < 0) continue;
    std::vector<int> mine;
    for (int q = 0; q < m; ++q) {
      if (mem[q] / c->P == me) mine.push_back(q);
    }
    // one item per (local member, chunk): stepped once, stored to all S
    // GPUs, every GPU starting at a different destination
    for (int q : mine) {
      for (long ch = 0; ch < nch; ++ch) {
        PushItem it{};
        it.lr = mem[q] - c->first;
        it.lo = ch * CH;
        it.hi = std::min(c->d_pad, it.lo + CH);
        it.dst_beg = static_cast<int>(item_dst.size());
        it.ndst = S;
        it.rank = grank(c, mem[q]);
        for (int oo = 0; oo < S; ++oo) {
          const int o = (oo + j) % S;
          const int gpu = gpus[static_cast<size_t>(o)];
          const long row = static_cast<long>(slot[static_cast<size_t>(o)]) * R + q;
          item_dst.push_back(static_cast<char*>(c->peer_push_buf[static_cast<size_t>(gpu)]) +
                             static_cast<size_t>(row * c->d_pad + it.lo) * c->esz);
          item_flag.push_back(c->peer_push_flags[static_cast<size_t>(gpu)] + row * nch + ch);
          item_gpu.push_back(gpu);
        }
        items.push_back(it);
      }
    }
    const long row0 = static_cast<long>(slot[static_cast<size_t>(j)]) * R;
    const int dst_beg = static_cast<int>(dst.size());
    for (int q : mine) {
      dst.push_back(static_cast<char*>(c->w) + static_cast<size_t>(mem[q] - c->first) * c->d_pad * c->esz);
      dst_lr.push_back(mem[q] - c->first);
    }
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
      f.n_dst = static_cast<int>(mine.size());
      f.err_rank = grank(c, mem[0]);
      folds.push_back(f);
    }
  }
  // chunk-major across this GPU's members
  std::vector<PushItem> ordered;
  ordered.reserve(items.size());
  const size_t nm = nch ? items.size() / static_cast<size_t>(nch) : 0;
  for (long ch = 0; ch < nch; ++ch) {
    for (size_t g = 0; g < nm; ++g) ordered.push_back(items[g * static_cast<size_t>(nch) + static_cast<size_t>(ch)]);
  }
  pl.items = static_cast<int>(ordered.size());
  pl.folds = static_cast<int>(folds.size());
  pl.d_item_dst = upload_table(c, item_dst);
  pl.d_item_flag = upload_table(c, item_flag);
  pl.d_items = upload_table(c, ordered);
  pl.d_folds = upload_table(c, folds);
  pl.d_dst = upload_table(c, dst);
  pl.d_dst_lr = upload_table(c, dst_lr);
  pl.d_item_gpu = upload_table(c, item_gpu);
  if (!c->d_oneshot_ack_peer) {
    std::vector<unsigned long long*> acks;
    for (int q = 0; q < G; ++q) acks.push_back(c->peer_push_flags[static_cast<size_t>(q)] + c->oneshot_ack_off);
    c->d_oneshot_ack_peer = upload_table(c, acks);
  }
  return pl;
}

// Build the launch tables of one parity.  with_step: DS iteration (local
// steps fused); otherwise sync_round (fold only).
ParityPlan build_plan(dss_ctx* c, long t, bool with_step) {
  ParityPlan pp;
  const dss_strategy& s = c->cfg.strategy;
  const Partition part = part_at(c, t);
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
    const GpuPlan gp = make_plan(part, s.world_size, G, multi(c) ? c->cfg.rank : 0, c->d_pad, force_chain(c),
                                 with_step && c->oneshot[t & 1]);
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
                             with_step ? c->cfg.optimizer : kOptNone, kOptNone, lrs,
                             DSS_CHAIN_INPLACE && multi(c) ? &part : nullptr, static_cast<int>(t & 1));
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
      e.err_rank = grank(c, mem[0]);
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
  if (c->oneshot[0]) {
    // small rows: every GPU gathers all W gradient rows, folds them in rank
    // order and steps its replicas (one kernel, no barrier)
    pp.any_spanning = true;
    pp.any_push = true;
    pp.push = build_oneshot(c, part);
    pp.push.bsp = true;
    return pp;
  }
  // Rows up to 4 MiB with at most 4 replicas per GPU: the pull two-shot (one
  // hop) beats the ordered chain (G stages): W=16 on 4 GPUs +32% at 1 MB,
  // +23% at 4 MB; the chain wins with more replicas per GPU or longer rows
  // (profiles/r02/sweeps/bsp_chain_ab_g4.md)
  const bool pull = DSS_BSP_PULL ||
                    (c->P <= DSS_BSP_PULL_MAX_P && c->d_pad * c->esz <= DSS_BSP_PULL_MAX_BYTES);
  const GpuPlan gp = make_plan(part, W, G, c->cfg.rank, c->d_pad, force_chain(c), pull && !force_chain(c));
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
  if (c->placed) {
    // tiled placement: rank order visits the GPUs several times, so the
    // ordered chain does not apply; GPU j folds slice j of all W rows (peer
    // loads in rank order) into every GPU's mean row
    pp.any_spanning = pp.any_twoshot = true;
    long lo = 0, hi = 0;
    slice_range(c->d_pad, G, c->cfg.rank, &lo, &hi);
    if (hi > lo) {
      if (W > kMaxFold) throw std::invalid_argument("global mean supports at most 64 workers");
      FoldEntry e{};
      std::vector<void*> src, dst;
      e.src_cnt = W;
      e.dst_cnt = G;
      e.lo = lo;
      e.hi = hi;
      e.err_rank = 0;
      e.err_phase = 1;
      for (int k = 0; k < W; ++k) src.push_back(row_ptr(c, c->peer_w, c->slot_of[static_cast<size_t>(k)]));
      for (int q = 0; q < G; ++q) dst.push_back(c->peer_mg[static_cast<size_t>(q)]);
      pp.fold.entries = 1;
      pp.fold.uniform_m = W;
      pp.fold.max_len = hi - lo;
      pp.fold.d_entries = upload_table(c, std::vector<FoldEntry>{e});
      pp.fold.d_src = upload_table(c, src);
      pp.fold.d_dst = upload_table(c, dst);
    }
    pp.built = true;
    return pp;
  }
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
    e.err_rank = c->cfg.strategy.kind == DSS_BSP ? 0 : grank(c, mem[0]);
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

// Deferred mean pass of parity p's chains on this GPU (LazyPlan): only when
// every chain entry here with a mean pass is a stage 0 of a two-GPU chain
// (the mean arrives in place, nothing to forward) and the other parity's
// groups are all local, one launch of 2 or 4 rows per group over all P <= 4
// rows.
LazyPlan build_lazy(dss_ctx* c, int p) {
  LazyPlan lp;
  if (!DSS_CHAIN_LAZY_MEAN || !multi(c) || c->s != 0 || !c->chain_split) return lp;
  const ParityPlan& pp = c->step_plan[p];
  const ParityPlan& pq = c->step_plan[1 - p];
  if (!pp.any_chain || pp.any_push || pp.any_twoshot || !pp.local.empty()) return lp;
  const ChainLaunch& cl = pp.chain;
  if (cl.nb == 0 || cl.nb > 4 || cl.opt_dst != kOptNone) return lp;
  if (pq.any_spanning || pq.local.size() != 1) return lp;
  const GroupLaunch& gl = pq.local[0];
  if ((gl.size != 2 && gl.size != 4) || (c->P != 2 && c->P != 4) || gl.groups * gl.size != c->P) return lp;
  const size_t row_bytes = static_cast<size_t>(c->d_pad) * c->esz;
  auto row_of = [&](const void* ptr) {
    return static_cast<int>((static_cast<const char*>(ptr) - static_cast<const char*>(c->w)) / row_bytes);
  };
  for (int r = 0; r < c->P; ++r) lp.alias[r] = r;
  for (const ChainEntry& b : cl.hb) {
    if (!b.dst_skip || b.send || b.dst_cnt < 1 || b.recv != cl.hdst[static_cast<size_t>(b.dst_beg)]) return lp;
    const int src = row_of(b.recv);
    for (int q = 1; q < b.dst_cnt; ++q) lp.alias[row_of(cl.hdst[static_cast<size_t>(b.dst_beg + q)])] = src;
    lp.flags[lp.nf++] = b.recv_flags;
  }
  for (int i = 0; i < c->P; ++i) lp.rows[i] = gl.members[static_cast<size_t>(i)] - c->first;
  lp.nr = c->P;
  lp.m = gl.size;
  lp.ok = true;
  return lp;
}

void build_stats_plans(dss_ctx* c) {
  if (c->s == 0) return;
  const dss_strategy& s = c->cfg.strategy;
  for (int p = 0; p < (s.kind == DSS_DS_SYNC ? 2 : 1); ++p) c->stats_plan[p] = build_stats_plan(c, part_at(c, p));
}

void build_plans(dss_ctx* c) {
  const dss_strategy& s = c->cfg.strategy;
  if (s.kind == DSS_DS_SYNC) {
    for (int p = 0; p < 2; ++p) c->step_plan[p] = build_plan(c, p, true);
    for (int p = 0; p < 2; ++p) c->lazy_plan[p] = build_lazy(c, p);
  } else if (multi(c)) {
    c->step_plan[0] = build_bsp_multi_plan(c);
  }
  for (int p = 0; p < 2; ++p) c->sync_plan[p] = build_plan(c, p, false);
  if (c->cfg.strategy.world_size <= kMaxFold || multi(c)) c->mean_plan = build_mean_plan(c);
  build_stats_plans(c);
}

// ---- launch helpers ---------------------------------------------------------

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
  if (a.wait_flags) flush_wait(c, a.wait_epoch);
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

// fp32 groups of 8 with these optimizers (bit OPT: momentum, Adam, AdamW)
// take the narrow-vector kernel.  Momentum only: on an unthrottled box the
// narrow kernel was +0.6-0.7% at both C3 and the C4 slice
// (profiles/r02/narrow_group_kernel_ab.jsonl), but the C4 slice's AdamW
// step runs power-capped (sw_power_cap, SM clocks 1650-1780 MHz), and there
// its extra load instructions cost 1.9% (5908 vs 6018 GB/s for the 16-B
// kernel; C3 stays +0.4% narrow: profiles/r02/power_ab_{c3,c4slice}.jsonl)
#ifndef DSS_GROUP_NARROW
#define DSS_GROUP_NARROW 2
#endif

template <int OPT>
void launch_group_narrow(dss_ctx* c, const GroupArgs<float>& a, int groups) {
  if (a.wait_flags) flush_wait(c, a.wait_epoch);
  dim3 grid(grid_x(c, a.nvec * 2, groups), groups);
  TimedLaunch tl(c, DSS_KIND_GROUP);
  ds_group_narrow_kernel<OPT, 8><<<grid, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "ds_group_narrow_kernel launch");
}

template <typename T, int OPT>
void launch_group_m(dss_ctx* c, const GroupArgs<T>& a, const GroupLaunch& gl) {
  if constexpr (std::is_same_v<T, float> && OPT != kOptNone) {
    if (((DSS_GROUP_NARROW >> OPT) & 1) && gl.size == 8 && a.g_ld == a.ld) {
      launch_group_narrow<OPT>(c, a, gl.groups);
      return;
    }
  }
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
  if (c->wait_epoch) {  // first launch of a step after an arriving push: wait in every CTA
    a.wait_flags = c->flags;
    a.wait_n = c->cfg.n_gpus;
    a.wait_epoch = c->wait_epoch;
    a.timeout = c->d_timeout;
    c->wait_epoch = 0;
  }
  a.w = static_cast<T*>(rows ? rows : c->w);  // rows: fold-only over another row set (running stats)
  a.g = static_cast<const T*>(g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = rows ? rows_ld : c->d_pad;
  a.g_ld = g_ld;
  a.nvec = a.ld / Vec<T>::n;
  a.first_rank = c->first;
  a.rank_of = c->d_rank_of;
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
                       const void* g, long g_ld, int step_phase, int sync_phase, void* rows,
                       long rows_ld) {
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
  flush_wait(c);
  ++c->xgpu_ops;
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
  // (2300 / stalled).  Round 2: both passes in one cooperative kernel, every
  // CTA taking its partial-pass units then its mean-pass units (no lag):
  // bit-exact but slower everywhere -- C2 @2 GPUs 3200 -> 2790, C3 @4 (tiled)
  // 744 -> 572, C4 @4 32.1 -> 21.3 (profiles/r02/chain_fused_ab_g*.jsonl).
  if (cl.na > 0 && c->emu_pass != 2) {
    a.entries = cl.d_a;
    a.n_entries = cl.na;
    const long units = c->chain_nchunks * cl.na;
    TimedLaunch tl(c, DSS_KIND_CHAIN);
    chain_partial_kernel<T, OPTM, OPTD><<<static_cast<int>(std::min<long>(units, c->sms * long{DSS_CHAIN_CTAS_PER_SM})),
                                          kThreads, 0, c->stream>>>(a);
    ck(cudaGetLastError(), "chain_partial_kernel launch");
  }
  if (cl.nb > 0 && c->emu_pass != 1 && c->defer_b) {
    // deferred: the next step's fused kernel (or flush_lazy) takes it
    ChainArgs<T> b = a;
    b.entries = cl.d_b;
    b.n_entries = cl.nb;
    const int grid = static_cast<int>(std::min<long>(c->chain_nchunks * cl.nb, c->sms * long{DSS_CHAIN_CTAS_PER_SM}));
    c->lazy_epoch = a.epoch;
    c->lazy_b = [c, b, grid]() {
      TimedLaunch tl(c, DSS_KIND_CHAIN_MEAN);
      chain_mean_kernel<T, OPTD><<<grid, kThreads, 0, c->stream>>>(b);
      ck(cudaGetLastError(), "chain_mean_kernel launch (deferred)");
    };
  } else if (cl.nb > 0 && c->emu_pass != 1) {
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
  if (c->emu_pass != 2) ++c->chain_epoch;  // same sequence on every GPU: flags compare against it
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
  a.rank_of = c->d_rank_of;
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

void launch_chain_any(dss_ctx* c, const ChainLaunch& cl, long t, double alpha) {
  struct ResetDefer {  // defer_b covers this one launch, even if it throws
    dss_ctx* c;
    ~ResetDefer() { c->defer_b = false; }
  } reset{c};
  flush_wait(c);
  ++c->xgpu_ops;
  if (c->cfg.dtype == DSS_F64) {
    launch_chain<double>(c, cl, t, alpha);
  } else {
    launch_chain<float>(c, cl, t, alpha);
  }
}

#ifndef DSS_PUSH_COOP
#define DSS_PUSH_COOP 1
#endif

template <typename T, int OPT>
void launch_push_t(dss_ctx* c, const PushLaunch& pl, long t, double alpha) {
  // emulation pass 2 repeats pass 1's launch numbers (epoch, one-shot seq)
  if (c->emu_pass != 2) ++c->chain_epoch;  // flags compare against the shared epoch sequence
  PushArgs<T> a{};
  a.items = pl.d_items;
  a.n_items = c->emu_pass == 2 ? 0 : pl.items;  // emulation: phase 1 and phase 2 as two launches
  a.item_dst = pl.d_item_dst;
  a.item_flag = pl.d_item_flag;
  a.folds = pl.d_folds;
  a.n_folds = c->emu_pass == 1 ? 0 : pl.folds;
  a.dst = reinterpret_cast<T* const*>(pl.d_dst);
  a.dst_lr = pl.d_dst_lr;
  a.w = static_cast<T*>(c->w);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.first_rank = c->first;
  a.rank_of = c->d_rank_of;
  a.t = t;
  a.epoch = c->chain_epoch;
  a.err = c->d_err;
  a.timeout = c->d_timeout;
  a.me = c->cfg.rank;
  a.n_gpus = c->cfg.n_gpus;
  if (c->wait_epoch) {
    a.wait_flags = c->flags;
    a.wait_epoch = c->wait_epoch;
    c->wait_epoch = 0;
  }
  if (c->arrive_next_push) {
    c->arrive_next_push = false;
    ++c->epoch;
    a.arrive_flags = c->d_peer_flags;
    a.arrive_epoch = c->epoch;
    a.arrive_count = c->d_arrive_count;
  }
  if (pl.oneshot) {
    // rotate the staging buffers; the kernel's acks keep a push from
    // overwriting a buffer its destination still reads (see PushArgs::seq)
    if (c->emu_pass != 2) ++c->oneshot_seq;
    const long par = static_cast<long>((c->oneshot_seq - 1) % DSS_ONESHOT_BUFFERS);
    a.stage_shift = (c->oneshot_base_elems + par * c->oneshot_half_elems) * c->esz;
    a.flag_shift = c->oneshot_base_flags + par * c->oneshot_half_flags;
    a.seq = c->oneshot_seq;  // 1, 2, ...: this launch's number
    a.ack_peer = c->d_oneshot_ack_peer;
    a.ack_mine = c->push_flags + c->oneshot_ack_off;
    a.item_gpu = pl.d_item_gpu;
    a.me = c->cfg.rank;
    a.n_gpus = c->cfg.n_gpus;
  }
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  auto kern = pl.bsp ? push_twoshot_kernel<T, OPT, true> : push_twoshot_kernel<T, OPT, false>;
  // Phase-2 CTAs spin on flags that phase-1 CTAs of this and other GPUs
  // release, so every CTA must be resident at once: a cooperative launch
  // guarantees it (or fails the launch) whatever else shares the GPU.  The
  // occupancy query runs once per instantiation.
  static int occ[2] = {-1, -1};
  int& o = occ[pl.bsp ? 1 : 0];
  if (o < 0) {
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, 0), "occupancy");
    o = std::max(o, 1);
  }
  const long grid = std::max(1L, std::min<long>(static_cast<long>(o) * c->sms, std::max(a.n_items, a.n_folds)));
  TimedLaunch tl(c, DSS_KIND_FOLD);
  if (DSS_PUSH_COOP) {
    void* args[] = {&a};
    ck(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(static_cast<unsigned>(grid)),
                                   dim3(kThreads), args, 0, c->stream),
       "push_twoshot_kernel cooperative launch");
  } else {
    kern<<<static_cast<int>(grid), kThreads, 0, c->stream>>>(a);
    ck(cudaGetLastError(), "push_twoshot_kernel launch");
  }
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
  ++c->xgpu_ops;
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
  if (!multi(c) || c->emulated) return;  // emulation: the launch order already serialises the ranks
  if (!c->attached) throw PeerError("multi-GPU context used before dss_ipc_attach");
  flush_lazy(c);
  c->wait_epoch = 0;  // a full barrier subsumes a pending split wait (flags only grow)
  ++c->epoch;
  ++c->xgpu_ops;
  TimedLaunch tl(c, DSS_KIND_BARRIER);
  barrier_kernel<<<1, 32 * ((c->cfg.n_gpus + 31) / 32), 0, c->stream>>>(
      c->d_peer_flags, c->flags, c->cfg.rank, c->cfg.n_gpus, c->epoch, c->d_timeout);
  ck(cudaGetLastError(), "barrier_kernel launch");
}

// Peers may still be writing group means into our rows (two-shot phase 2 of
// the previous round): wait for them before touching the rows again.
// allow_chain_skip (DS steps only): remote work that is DS step chains only
// needs no barrier before the next DS step -- see dss_step.
// allow_chain_skip also lets a DS step that follows an arriving two-shot push
// step (and nothing cross-GPU after it) wait in its first kernel instead.
void quiesce(dss_ctx* c, bool allow_chain_skip) {
  if (c->pending_remote && multi(c) && !(allow_chain_skip && c->pending_chain_only)) {
    if (allow_chain_skip && c->split_mark == c->xgpu_ops) {
      c->wait_epoch = c->epoch;
    } else {
      barrier(c);
    }
  }
  if (!allow_chain_skip) flush_wait(c);
  c->pending_remote = false;
  c->pending_chain_only = false;
}

// 2 CTAs per SM: C2 on 2 GPUs 3468-3480 iters/s against 3419-3435 at 4 and
// 8 (profiles/r02/sweeps/lazy_mean_ctas_ab_g2.jsonl), 3450-3460 against
// 3419-3431 at 3 and 3267-3272 at 1 (lazy_mean_ctas_ab2_g2.jsonl)
#ifndef DSS_LAZY_CTAS_PER_SM
#define DSS_LAZY_CTAS_PER_SM 2
#endif

void flush_lazy(dss_ctx* c) {
  if (!c->lazy_b) return;
  std::function<void()> f = std::move(c->lazy_b);
  c->lazy_b = nullptr;
  c->lazy_parity = -1;
  f();
}

template <typename T, int OPT, int NR, int M>
void launch_lazy_t(dss_ctx* c, const LazyArgs<T>& a) {
  const int grid = static_cast<int>(std::min<long>(a.n_chunks, c->sms * long{DSS_LAZY_CTAS_PER_SM}));
  TimedLaunch tl(c, DSS_KIND_GROUP);
  lazy_groups_kernel<T, OPT, NR, M><<<grid, kThreads, 0, c->stream>>>(a);
  ck(cudaGetLastError(), "lazy_groups_kernel launch");
}

template <typename T, int OPT>
void launch_lazy_o(dss_ctx* c, const LazyPlan& lp, const LazyArgs<T>& a) {
  if (lp.nr == 2) {
    launch_lazy_t<T, OPT, 2, 2>(c, a);
  } else if (lp.m == 2) {
    launch_lazy_t<T, OPT, 4, 2>(c, a);
  } else {
    launch_lazy_t<T, OPT, 4, 4>(c, a);
  }
}

template <typename T>
void launch_lazy(dss_ctx* c, const LazyPlan& lp, long t, double alpha) {
  LazyArgs<T> a{};
  a.w = static_cast<T*>(c->w);
  a.g = static_cast<const T*>(c->g);
  a.m1 = static_cast<T*>(c->m1);
  a.m2 = static_cast<T*>(c->m2);
  a.ld = c->d_pad;
  a.chunk = c->chain_chunk;
  a.len = c->d_pad;
  a.n_chunks = c->chain_nchunks;
  for (int i = 0; i < lp.nf; ++i) a.flags[i] = lp.flags[i];
  a.nf = lp.nf;
  a.epoch = c->lazy_epoch;
  a.timeout = c->d_timeout;
  for (int r = 0; r < lp.nr; ++r) {
    a.alias[r] = lp.alias[r];
    a.rows[r] = lp.rows[r];
    a.rank[r] = c->rank_of_slot[static_cast<size_t>(c->first + r)];
  }
  a.t = t;
  a.step_phase = 0;
  a.sync_phase = 1;
  a.err = c->d_err;
  a.c = consts<T>(c, alpha);
  fill_bias(c, a);
  switch (c->cfg.optimizer) {
    case kSgd: launch_lazy_o<T, kSgd>(c, lp, a); break;
    case kMomentum: launch_lazy_o<T, kMomentum>(c, lp, a); break;
    case kAdam: launch_lazy_o<T, kAdam>(c, lp, a); break;
    case kAdamW: launch_lazy_o<T, kAdamW>(c, lp, a); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
}

// The DS step of the consuming parity: the deferred mean pass and the local
// groups' step in one launch (LazyPlan).
void launch_lazy_any(dss_ctx* c, const LazyPlan& lp, long t, double alpha) {
  flush_wait(c);
  c->lazy_b = nullptr;
  c->lazy_parity = -1;
  if (c->cfg.dtype == DSS_F64) {
    launch_lazy<double>(c, lp, t, alpha);
  } else {
    launch_lazy<float>(c, lp, t, alpha);
  }
}

// Launch the waiting half of the split barrier on its own if still pending
// (epoch: a wait taken from a launch that cannot wait itself).
void flush_wait(dss_ctx* c, unsigned long long epoch) {
  if (!epoch) {
    epoch = c->wait_epoch;
    c->wait_epoch = 0;
  }
  if (!epoch) return;
  TimedLaunch tl(c, DSS_KIND_BARRIER);
  split_wait_kernel<<<1, 32 * ((c->cfg.n_gpus + 31) / 32), 0, c->stream>>>(c->flags, c->cfg.n_gpus, epoch,
                                                                           c->d_timeout);
  ck(cudaGetLastError(), "split_wait_kernel launch");
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
    c->pending_chain_only = false;
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
  const int slot = rank >= 0 && rank < static_cast<int>(c->slot_of.size()) ? c->slot_of[static_cast<size_t>(rank)] : -1;
  if (slot < c->first || slot >= c->first + c->P) {
    throw std::invalid_argument("rank " + std::to_string(rank) + " is not hosted on this GPU");
  }
  *lr = slot - c->first;
  return DSS_OK;
}


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

// ---- tiny worlds: whole iterations in one CTA (dss_steps, dss_logistic_steps)

// Worlds small enough that one CTA beats one launch per iteration.
long small_bytes(const dss_ctx* c) { return static_cast<long>(c->P) * c->d_pad * c->esz; }

// One launch for the whole batch: always up to 32 KB per array (one CTA);
// the resident grid where it beats one launch per iteration of the
// templated kernels (measured sweep: up to 16 workers; DS up to 1 MB per
// array, BSP up to 4 MB).
bool small_path(const dss_ctx* c, long n) {
  if (multi(c) || c->cfg.path != 0 || c->s != 0 || n < 2 || c->P > kMaxLocal) return false;
  const long bytes = small_bytes(c);
  if (bytes <= 32768) return true;
  const bool bsp = c->cfg.strategy.kind == DSS_BSP;
  const int max_workers = bsp ? DSS_PERSIST_MAX_WORKERS_BSP : DSS_PERSIST_MAX_WORKERS_DS;
  return bytes <= (bsp ? DSS_PERSIST_MAX_BYTES_BSP : DSS_PERSIST_MAX_BYTES) && c->P <= max_workers;
}

template <typename T, int OPT>
void launch_small_t(dss_ctx* c, SmallArgs<T>& a, int grid) {
  TimedLaunch tl(c, c->cfg.strategy.kind == DSS_BSP ? DSS_KIND_BSP : DSS_KIND_GROUP);
  if (grid == 1) {
    const long units = a.bsp ? a.nvec : std::max(a.ngroups[0], a.ngroups[1]) * a.nvec;
    if (DSS_SMALL_WIDE && !a.logistic && units > kThreads) {
      small_steps_kernel<T, OPT, kSmallWide><<<1, kSmallWide, 0, c->stream>>>(a);
    } else {
      small_steps_kernel<T, OPT><<<1, kThreads, 0, c->stream>>>(a);
    }
    ck(cudaGetLastError(), "small_steps_kernel launch");
    return;
  }
  // persistent grid with a barrier between iterations: cooperative launch
  // guarantees every CTA is resident (at most what fits the SMs)
  static int occ = -1;
  if (occ < 0) {
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, small_steps_kernel<T, OPT>, kThreads, 0), "occupancy");
    occ = std::max(occ, 1);
  }
  grid = std::min(grid, occ * c->sms);
  void* args[] = {&a};
  ck(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(small_steps_kernel<T, OPT>), dim3(grid),
                                 dim3(kThreads), args, 0, c->stream),
     "small_steps_kernel cooperative launch");
}

template <typename T>
void run_small(dss_ctx* c, long t0, long n, const double* alphas, bool logistic) {
  const int P = c->P;
  const dss_strategy& s = c->cfg.strategy;
  if (!c->d_small_members[0]) {  // schedule tables of both parities, once
    for (int p = 0; p < 2; ++p) {
      const Partition part = part_at(c, p);
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
  // one CTA for tiny worlds (and the logistic phase, one warp per worker);
  // above 32 KB a resident grid (up to two CTAs per SM), barrier between iterations
  int grid = 1;
  if (!logistic && small_bytes(c) > 32768) {
    const long units = a.bsp ? a.nvec : std::max(a.ngroups[0], a.ngroups[1]) * a.nvec;
    grid = static_cast<int>(std::min<long>(2L * c->sms, (units + kThreads - 1) / kThreads));
    grid = std::max(grid, 1);
  }
  if (grid > 1) {
    if (!c->d_small_bar) c->d_small_bar = static_cast<unsigned*>(dalloc(c, sizeof(unsigned)));
    ck(cudaMemsetAsync(c->d_small_bar, 0, sizeof(unsigned), c->stream), "barrier reset");
    a.bar = c->d_small_bar;
  }
  switch (c->cfg.optimizer) {
    case kSgd: launch_small_t<T, kSgd>(c, a, grid); break;
    case kMomentum: launch_small_t<T, kMomentum>(c, a, grid); break;
    case kAdam: launch_small_t<T, kAdam>(c, a, grid); break;
    case kAdamW: launch_small_t<T, kAdamW>(c, a, grid); break;
    default: throw std::invalid_argument("unknown optimizer kind");
  }
  // the host table buffer is reused by the next call: wait for the copy
  ck(cudaStreamSynchronize(c->stream), "small-path sync");
  for (auto& sc : c->step_count) sc += n;
}

template void launch_bsp<float>(dss_ctx* c, long t, double alpha);
template void launch_bsp<double>(dss_ctx* c, long t, double alpha);
template void run_small<float>(dss_ctx* c, long t0, long n, const double* alphas, bool logistic);
template void run_small<double>(dss_ctx* c, long t0, long n, const double* alphas, bool logistic);

}  // namespace dssb
