// C-ABI entry points (include/dssync_b200.h): context lifetime, data
// movement, the DS-Sync / BSP iteration, sync_round, apply_step, timing and
// the multi-GPU handshake.
//
// The iteration restates run_training's DS branch (sync.cpp:347-374), BSP
// branch (sync.cpp:375-428) and sync_round (sync.cpp:268-282) over
// device-resident worker-major buffers.  One context per GPU (process).
#include "context.cuh"

using namespace dssb;

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
    {
      const Tiling tl = choose_placement(s, cfg->n_gpus, cfg->placement,
                                         pad_dim(cfg->dim) * (cfg->dtype == DSS_F64 ? 8 : 4), DSS_ONESHOT_MAX_BYTES);
      c->slot_of = placement_slots(s, cfg->n_gpus, tl);
      c->rank_of_slot.assign(c->slot_of.size(), 0);
      for (size_t k = 0; k < c->slot_of.size(); ++k) {
        c->rank_of_slot[static_cast<size_t>(c->slot_of[k])] = static_cast<int>(k);
        c->placed = c->placed || c->slot_of[k] != static_cast<int>(k);
      }
      c->tile_gr = c->placed ? tl.gr : 0;
      c->tile_gc = c->placed ? tl.gc : 0;
    }
    if (cfg->placement < 0 || cfg->placement > 2) throw std::invalid_argument("placement must be 0, 1 or 2");
    c->d = cfg->dim;
    c->d_pad = pad_dim(cfg->dim);
    c->esz = cfg->dtype == DSS_F64 ? 8 : 4;
    c->step_count.assign(static_cast<size_t>(c->P), 0);

    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (cfg->device < 0 || cfg->device >= ndev) throw CudaError("no CUDA device " + std::to_string(cfg->device));
    ck(cudaSetDevice(cfg->device), "cudaSetDevice");
    ck(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cfg->device), "sm count");
    if (const char* gb = std::getenv("DSS_GUARD_BYTES")) {  // debug: guard bands around every allocation
      const long v = std::atol(gb);
      c->guard = v > 0 ? (v + 255) / 256 * 256 : 0;
    }
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
    c->d_arrive_count = static_cast<unsigned*>(dalloc(c.get(), sizeof(unsigned)));
    ck(cudaMallocHost(&c->h_err, sizeof(unsigned long long)), "cudaMallocHost");

    {
      std::vector<int> rk(static_cast<size_t>(c->P));
      for (int l = 0; l < c->P; ++l) rk[static_cast<size_t>(l)] = c->rank_of_slot[static_cast<size_t>(c->first + l)];
      c->d_rank_of = upload_table(c.get(), rk);
    }
    std::vector<std::vector<int>> singles;
    for (int k = 0; k < c->P; ++k) singles.push_back({c->first + k});
    c->apply_launch = make_group_launch(c.get(), singles);
    if (multi(c.get())) {
      // chain-fold receive rows and flags, sized for the worst parity (the
      // plan is global, so every GPU computes the same slot count)
      int slots = 0;
      for (long t = 0; t < (s.kind == DSS_DS_SYNC ? 2 : 1); ++t) {
        const GpuPlan gp = make_plan(part_at(c.get(), t), s.world_size, cfg->n_gpus, cfg->rank, c->d_pad,
                                     force_chain(c.get()));
        slots = std::max(slots, gp.max_chain_slots);
      }
      dss_strategy world = s;  // the all-world group of the global-mean trace
      world.kind = DSS_BSP;
      world.group_size = s.world_size;
      world.rectangular = 0;
      if (!c->placed) {  // placed worlds fold the global mean two-shot (build_mean_plan)
        slots = std::max(slots, make_plan(make_partition(world, 0), s.world_size, cfg->n_gpus, cfg->rank, c->d_pad,
                                          force_chain(c.get())).max_chain_slots);
      }
      c->chain_slots = slots;
      // DS-Sync with rows of 80 MiB or more prefers longer chunks than the packed BSP
      // chain and than small rows (profiles/r02/chain_chunk_ab_g{2,4}.jsonl,
      // 16384 vs 8192: DS C2 @2 3204 -> 3250, C2 @4 3480 -> 3560, C3 @4
      // 744 -> 753, C4 @4 32.0 -> 33.1 iters/s; but BSP C3 @4 768 -> 690,
      // and the sweep's 64 KB - 64 MB rows lose up to 40%,
      // profiles/r02/chain_chunk_sweep_ab_g4.jsonl)
      const bool long_chunks = s.kind == DSS_DS_SYNC && c->d_pad * c->esz >= DSS_CHAIN_CHUNK_DS_MIN_BYTES;
      long chunk = long_chunks ? DSS_CHAIN_CHUNK_DS : DSS_CHAIN_CHUNK;
      // small rows: shorter chunks, so the chain and one-shot work units
      // (chunk x group) spread over the SMs instead of serialising a whole
      // row's member loads on a few CTAs
      const bool bsp = s.kind == DSS_BSP;
      const long min_chunk = bsp ? DSS_BSP_CHAIN_CHUNK_MIN : DSS_CHAIN_CHUNK_MIN;
      const long min_chunks = bsp ? DSS_BSP_CHAIN_MIN_CHUNKS : DSS_CHAIN_MIN_CHUNKS;
      while (chunk > min_chunk && c->d_pad < chunk * min_chunks) chunk /= 2;
      c->chain_chunk = std::min<long>(c->d_pad, chunk);
      c->chain_nchunks = (c->d_pad + c->chain_chunk - 1) / c->chain_chunk;
      c->chain_buf = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(2) * slots * c->d_pad * c->esz));
      // Fused two-shot staging of the owned slices, worst parity and worst
      // GPU: the one-shot area starts after it at the same offset on every
      // GPU, because a pusher applies its own offset to the peer's buffer.
      long ps = 0, pf = 0;
      for (long t = 0; t < (s.kind == DSS_DS_SYNC ? 2 : 1); ++t) {
        const Partition part = part_at(c.get(), t);
        for (int q = 0; q < cfg->n_gpus; ++q) {
          long st = 0, fl = 0;
          owned_layout(c.get(), part, q, c->chain_chunk, &st, &fl);
          ps = std::max(ps, st);
          pf = std::max(pf, fl);
        }
      }
      // One-shot per schedule parity: every member GPU gathers every
      // member's row and folds it for its own members.  Pairs with one
      // member per GPU move the same NVLink bytes as two-shot and skip the
      // next iteration's barrier, so they go one-shot at any size; any
      // other spanning group (larger, or several members per GPU: the
      // chain) only for rows of at most DSS_ONESHOT_MAX_BYTES.
      long rows = 0;
      const bool small_rows = c->d_pad * c->esz <= DSS_ONESHOT_MAX_BYTES;
      // BSP: gather all W gradient rows (build_bsp_multi_plan).  Each fold
      // unit reads all W rows of a chunk, so only for small worlds or small
      // totals: at 4 GPUs W=4 / 16 gain 2.4x / 1.9x at 1 KB rows; at 2 GPUs
      // W=64 gains 15-26% up to 16 KB rows and loses 40% at 256 KB
      // (profiles/r02/small_rows_ab_g2.jsonl).
      // Worlds of up to 4 take it up to 4 MiB in total (W=4 at 1 MB rows:
      // +34% on 2 and 4 GPUs; profiles/r02/sweeps/oneshot_max_ab_g*.jsonl).
      const long bsp_total = static_cast<long>(s.world_size) * c->d_pad * c->esz;
      if (s.kind == DSS_BSP && use_push(c.get()) && !force_chain(c.get()) && cfg->path != 4 &&
          ((small_rows && s.world_size <= DSS_BSP_ONESHOT_MAX_W) || bsp_total <= DSS_BSP_ONESHOT_MAX_TOTAL ||
           (s.world_size <= 4 && bsp_total <= DSS_BSP_ONESHOT_SMALL_W_TOTAL))) {
        c->oneshot[0] = true;
        rows = s.world_size;
      }
      for (long t = 0; t < 2; ++t) {
        if (s.kind != DSS_DS_SYNC || !use_push(c.get()) || force_chain(c.get()) || cfg->path == 4) break;
        const Partition part = part_at(c.get(), t);
        const bool small = c->d_pad * c->esz <= DSS_ONESHOT_MAX_BYTES;
        bool ok = true;
        long rmax = 0;
        for (int gi = 0; gi < part.n_groups(); ++gi) {
          std::vector<int> gpus;
          for (int q = 0; q < part.size(gi); ++q) gpus.push_back(part.group(gi)[q] / c->P);
          if (gpus.front() == gpus.back()) continue;  // local group
          const bool one_each = std::adjacent_find(gpus.begin(), gpus.end()) == gpus.end();
          if (!(one_each && part.size(gi) == 2) && !small) ok = false;
          rmax = std::max<long>(rmax, part.size(gi));
        }
        c->oneshot[t] = ok && rmax > 0;
        if (c->oneshot[t]) rows = std::max(rows, rmax);
      }
      if (c->oneshot[0] || c->oneshot[1]) {
        c->oneshot_rows = rows;
        c->oneshot_base_elems = ps;
        c->oneshot_base_flags = pf;
        c->oneshot_half_elems = static_cast<long>(c->P) * rows * c->d_pad;
        c->oneshot_half_flags = static_cast<long>(c->P) * rows * c->chain_nchunks;
        ps += DSS_ONESHOT_BUFFERS * c->oneshot_half_elems;
        pf += DSS_ONESHOT_BUFFERS * c->oneshot_half_flags;
        c->oneshot_ack_off = pf;  // [G] one-shot launches each peer has started
        pf += cfg->n_gpus;
      }
      c->push_buf = dalloc(c.get(), std::max<size_t>(256, static_cast<size_t>(ps) * c->esz));
      c->chain_split = s.kind == DSS_DS_SYNC && DSS_CHAIN_INPLACE && DSS_DS_CHAIN_NO_BARRIER;
      c->push_flags = static_cast<unsigned long long*>(
          dalloc(c.get(), std::max<size_t>(64, sizeof(unsigned long long) * static_cast<size_t>(pf))));
      c->chain_flags = static_cast<unsigned long long*>(dalloc(
          c.get(), std::max<size_t>(64, sizeof(unsigned long long) * (c->chain_split ? 4 : 2) * slots *
                                            c->chain_nchunks)));
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

extern "C" int dss_destroy(dss_ctx* c) {
  if (!c) return DSS_OK;
  if (c->cfg.device >= 0) cudaSetDevice(c->cfg.device);
  if (c->emulated) {
    cudaDeviceSynchronize();  // the shared stream may belong to another (already destroyed) context
  } else if (c->stream) {
    cudaStreamSynchronize(c->stream);
  }
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
  *first_rank = c->placed ? -1 : c->first;
  *count = c->P;
  return DSS_OK;
}

extern "C" int dss_local_ranks(const dss_ctx* c, int* ranks) {
  if (!c || !ranks) return DSS_EINVAL;
  for (int l = 0; l < c->P; ++l) ranks[l] = c->rank_of_slot[static_cast<size_t>(c->first + l)];
  return DSS_OK;
}

extern "C" int dss_placement(const dss_strategy* s, int n_gpus, int placement, long dim, int dtype, int* gpu_of,
                             int* row_of, int* gr, int* gc) {
  if (!s || n_gpus < 1 || s->world_size < 1 || s->world_size % n_gpus) {
    return fail(nullptr, DSS_EINVAL, "dss_placement: world_size must be a multiple of n_gpus");
  }
  return guard(nullptr, [&]() -> int {
    if (placement < 0 || placement > 2) throw std::invalid_argument("placement must be 0, 1 or 2");
    const long row_bytes = dim > 0 ? pad_dim(dim) * (dtype == DSS_F64 ? 8 : 4) : 0;
    const Tiling tl = choose_placement(*s, n_gpus, placement, row_bytes, DSS_ONESHOT_MAX_BYTES);
    const std::vector<int> slot = placement_slots(*s, n_gpus, tl);
    const int P = s->world_size / n_gpus;
    for (size_t k = 0; k < slot.size(); ++k) {
      if (gpu_of) gpu_of[k] = slot[k] / P;
      if (row_of) row_of[k] = slot[k] % P;
    }
    if (gr) *gr = tl.gr;
    if (gc) *gc = tl.gc;
    return DSS_OK;
  });
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
  if (!c || rank < 0 || rank >= static_cast<int>(c->slot_of.size())) return -1;
  const int slot = c->slot_of[static_cast<size_t>(rank)];
  if (slot < c->first || slot >= c->first + c->P) return -1;
  return c->step_count[static_cast<size_t>(slot - c->first)];
}

// ------------------------------- hot path ------------------------------------

#ifndef DSS_PUSH_SPLIT_BARRIER
#define DSS_PUSH_SPLIT_BARRIER 1
#endif

extern "C" int dss_step(dss_ctx* c, long t, double alpha, int check, dss_outcome* out) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  c->lazy_consume = true;  // guard() leaves a deferred mean pass to the step below
  NvtxRange range(c->cfg.strategy.kind == DSS_DS_SYNC ? "dss_step ds-sync" : "dss_step bsp");
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
      const bool first = c->emu_pass != 2, second = c->emu_pass != 1;  // emulation passes (both when not emulating)
      if (first) {
        // Back-to-back DS steps whose cross-GPU work is chains only skip the
        // opening barrier.  Groups depend only on the parity and each parity
        // has its own partial rows and flags (chain_split), so a row or flag
        // refilled at t+1 was last used at t-1 by the same group; its sender
        // has finished t-1 (a non-last stage waits in kernel B for every
        // chunk's mean, which exists only after every stage folded that
        // chunk), so the receiver consumed it.  A member row written in place
        // at t+1 is written only after its GPU's own t+1 partial, i.e. after
        // that GPU finished t; and every GPU's kernel B waited for all of its
        // in-place means of t before its t+1 launches.  Anything else in
        // between (two-shot, push, sync_round, global mean) keeps the barrier.
        // A chain step of the other parity may have left its mean pass to
        // this step (LazyPlan): this step's local groups then run fused with
        // it; any other order launches the deferred pass first.
        const bool lazy = c->lazy_b && c->lazy_parity == static_cast<int>(t & 1) && second &&
                          c->lazy_plan[(t + 1) & 1].ok;
        if (c->lazy_b && !lazy) flush_lazy(c);
        quiesce(c, true);
        if (lazy) {
          launch_lazy_any(c, c->lazy_plan[(t + 1) & 1], t, alpha);
        } else {
          // Local groups: fused apply_step + ordered fold + broadcast.
          for (const GroupLaunch& gl : pp.local) launch_groups_any(c, gl, opt, t, alpha, c->g, c->d_pad, 0);
        }
      }
      if (pp.any_spanning) {
        // Members of spanning groups step in place.  Two-shot groups: after
        // every GPU has stepped, each owner folds its slice over NVLink.
        // Chain groups: the ordered partial/mean passes (flag-synchronised
        // per chunk, no barrier).
        if (first) launch_groups_any(c, pp.spanning_step, opt, t, alpha, c->g, c->d_pad, 0);
        bool barrier_done = false;
        // A two-shot push with nothing cross-GPU after it arrives at the split
        // barrier itself: the next DS step waits in its first kernel instead
        // of opening with a barrier launch (quiesce).  The plan flags are the
        // same on every GPU, so every GPU arrives and waits at the same epochs.
        const bool split = DSS_PUSH_SPLIT_BARRIER && multi(c) && !c->emulated && pp.any_push &&
                           !pp.push.oneshot && !pp.any_chain && c->s == 0;  // (any_push: no pull fold)
        if (pp.any_push) {
          c->arrive_next_push = split;
          launch_push_any(c, pp.push, t, alpha);  // fused step + push two-shot
          if (split) c->split_mark = c->xgpu_ops;
        } else if (pp.any_twoshot && second) {
          if (multi(c)) barrier(c);
          barrier_done = true;
          launch_fold_any(c, pp.fold, t);
        }
        if (pp.any_chain) {
          c->defer_b = c->allow_defer && c->lazy_plan[t & 1].ok && !c->emulated && c->emu_pass == 0;
          launch_chain_any(c, pp.chain, t, alpha);
          c->defer_b = false;
          if (c->lazy_b) c->lazy_parity = static_cast<int>((t + 1) & 1);
        }
        if (!second) return DSS_OK;  // emulation pass 1 ends here
        // one-shot writes no peer params: the next iteration needs no barrier
        c->pending_remote = multi(c) && (pp.any_chain || !(pp.any_push && pp.push.oneshot));
        c->pending_chain_only = c->chain_split && pp.any_chain && !pp.any_push && !pp.any_twoshot;
        fold_stats(c, t, barrier_done);
      } else {
        if (!second) return DSS_OK;
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
      if (pp.any_push) {
        // one-shot: push the gradients, fold all W, step the replicas
        quiesce(c);
        launch_push_any(c, pp.push, t, alpha);
        c->pending_remote = false;
        fold_stats(c, t, false);
        bump_steps(c);
        if (out) *out = round_outcome(s, t, c->d + c->s);
        if (check) return check_impl(c);
        return DSS_OK;
      }
      c->pending_remote = false;
      // Back-to-back chain-only BSP steps skip the opening barrier: the chain
      // reads only this GPU's gradients, writes peers' staging rows only, and
      // has the same partners every iteration, so a GPU that starts step t+1
      // has received step t's mean for every chunk -- every GPU has already
      // consumed every staging row of step t that t+1 overwrites (the mean
      // of a chunk exists only after all its partials were folded, and a
      // mean row is refilled only after its reader has started t+1, i.e.
      // finished t).  Any other cross-GPU launch in between restores it.
      const bool chain_only = pp.any_chain && !pp.any_twoshot;
      if (!(chain_only && DSS_BSP_CHAIN_NO_BARRIER && c->xgpu_ops == c->bsp_chain_mark)) barrier(c);
      if (pp.any_twoshot) {
        launch_fold_any(c, pp.fold, t);
        barrier(c);
      }
      if (pp.any_chain) {
        launch_chain_any(c, pp.chain, t, alpha);  // fold -> replica step, fused per chunk
        c->pending_remote = true;
        if (chain_only) c->bsp_chain_mark = c->xgpu_ops;
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
  // An element-chunked variant (each chunk's copy-in, step and copy-out
  // overlapping the neighbours', no snapshot) was built, checked bit-exact
  // and measured slower: C2 56.1 (this path) vs 42.3 / 49.6 / 54.6 iters/s
  // with 2 / 4 / 8 chunks (profiles/r02/e2e_chunked_ab.jsonl).
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
    // the closed-form round outcome (a host partition) only for the last iteration
    // a mean pass may be deferred only to the next step of this same call:
    // no caller code can read the rows in between, and none stays pending
    c->allow_defer = i + 1 < n;
    const int st = dss_step(c, t0 + i, alphas[i], 0, i + 1 == n ? last : nullptr);
    c->allow_defer = false;
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

// Layout fingerprint exported beside the IPC handles: peers index each
// other's buffers with their own geometry (row stride, chain slots, one-shot
// offsets, ...), so every rank must have been created with the same
// configuration.  Attach rejects a peer whose fingerprint differs.
namespace {
constexpr int kFingerprintWords = 20;
void fingerprint(const dss_ctx* c, long long* f) {
  const long long v[kFingerprintWords] = {
      0x4453535942323030LL,  // "DSSYB200"
      c->cfg.dtype, c->cfg.optimizer, c->cfg.strategy.kind, c->cfg.strategy.topology,
      c->cfg.strategy.world_size, c->cfg.strategy.group_size, c->cfg.strategy.rectangular,
      c->cfg.n_gpus, c->P, c->d, c->d_pad, c->s, c->chain_slots, c->chain_chunk,
      c->oneshot_base_elems, c->oneshot_half_elems, c->oneshot_rows, c->oneshot_ack_off,
      c->cfg.path * 1000003LL + c->guard + (static_cast<long long>(c->tile_gr * 64 + c->tile_gc) << 40) +
          (static_cast<long long>(c->chain_split) << 60)};
  std::memcpy(f, v, sizeof(v));
}
}  // namespace

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
    static_assert(sizeof(h) + kFingerprintWords * sizeof(long long) == DSS_IPC_BYTES, "DSS_IPC_BYTES");
    fingerprint(c, reinterpret_cast<long long*>(static_cast<char*>(out) + sizeof(h)));
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
    long long mine[kFingerprintWords];
    fingerprint(c, mine);
    for (int r = 0; r < G; ++r) {
      const char* blob = static_cast<const char*>(all) + static_cast<size_t>(r) * DSS_IPC_BYTES;
      if (std::memcmp(blob + 9 * sizeof(cudaIpcMemHandle_t), mine, sizeof(mine)) != 0) {
        throw std::invalid_argument("dss_ipc_attach: rank " + std::to_string(r) +
                                    " was created with a different configuration (dtype, dims, world, "
                                    "optimizer or path) than rank " + std::to_string(c->cfg.rank));
      }
    }
    for (int r = 0; r < G; ++r) {
      const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(static_cast<const char*>(all) +
                                                                  static_cast<size_t>(r) * DSS_IPC_BYTES);
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
        cudaError_t e = cudaIpcOpenMemHandle(&p[b], h[b], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          throw PeerError("cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + cudaGetErrorString(e));
        }
        c->opened.push_back(p[b]);
      }
      for (int b = 0; b < 9; ++b) p[b] = static_cast<char*>(p[b]) + c->guard;  // guard bands: user region
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

// ---- single-device emulation of a G-GPU world (tests) ------------------------

extern "C" int dss_emulate_attach(dss_ctx** ctxs, int n) {
  if (!ctxs || n < 2) return fail(nullptr, DSS_EINVAL, "dss_emulate_attach: need >= 2 contexts");
  return guard(nullptr, [&]() -> int {
    for (int r = 0; r < n; ++r) {
      dss_ctx* c = ctxs[r];
      if (!c || c->cfg.n_gpus != n || c->cfg.rank != r || c->cfg.device != ctxs[0]->cfg.device || c->attached) {
        throw std::invalid_argument("dss_emulate_attach: context r must be rank r of an n-GPU world, all on one "
                                    "device, not yet attached");
      }
      long long a[kFingerprintWords], b[kFingerprintWords];
      fingerprint(c, a);
      fingerprint(ctxs[0], b);
      if (std::memcmp(a, b, sizeof(a)) != 0) {
        throw std::invalid_argument("dss_emulate_attach: rank " + std::to_string(r) +
                                    " was created with a different configuration");
      }
    }
    ck(cudaSetDevice(ctxs[0]->cfg.device), "cudaSetDevice");
    for (int r = 0; r < n; ++r) ck(cudaStreamSynchronize(ctxs[r]->stream), "emulate attach sync");
    for (int r = 0; r < n; ++r) {
      dss_ctx* c = ctxs[r];
      c->peer_w.assign(static_cast<size_t>(n), nullptr);
      c->peer_g = c->peer_mg = c->peer_chain_buf = c->peer_stats = c->peer_push_buf = c->peer_w;
      c->peer_flag.assign(static_cast<size_t>(n), nullptr);
      c->peer_chain_flags = c->peer_push_flags = c->peer_flag;
      for (int q = 0; q < n; ++q) {  // same device, same process: the peers' buffers directly
        const dss_ctx* p = ctxs[q];
        c->peer_w[static_cast<size_t>(q)] = p->w;
        c->peer_g[static_cast<size_t>(q)] = p->g;
        c->peer_mg[static_cast<size_t>(q)] = p->mg;
        c->peer_flag[static_cast<size_t>(q)] = p->flags;
        c->peer_chain_buf[static_cast<size_t>(q)] = p->chain_buf;
        c->peer_chain_flags[static_cast<size_t>(q)] = p->chain_flags;
        c->peer_stats[static_cast<size_t>(q)] = p->stats;
        c->peer_push_buf[static_cast<size_t>(q)] = p->push_buf;
        c->peer_push_flags[static_cast<size_t>(q)] = p->push_flags;
      }
      c->stream = ctxs[0]->stream;  // one stream: launches run in issue order
      c->emulated = true;
      c->d_peer_flags = upload_table(c, c->peer_flag);
      build_plans(c);
      c->attached = true;
    }
    ck(cudaStreamSynchronize(ctxs[0]->stream), "emulate attach sync");
    return DSS_OK;
  });
}

extern "C" int dss_emulate_step(dss_ctx** ctxs, int n, long t, double alpha, int check) {
  if (!ctxs || n < 2) return fail(nullptr, DSS_EINVAL, "dss_emulate_step: need >= 2 contexts");
  for (int r = 0; r < n; ++r) {
    if (!ctxs[r] || !ctxs[r]->emulated) return fail(ctxs[r], DSS_EINVAL, "dss_emulate_step: not emulate-attached");
    if (ctxs[r]->cfg.strategy.kind != DSS_DS_SYNC) return fail(ctxs[r], DSS_EINVAL, "dss_emulate_step: DS-Sync only");
  }
  // pass 1 in rank order (chain stages only wait on lower GPU indices), then
  // pass 2 in rank order (push folds, pull folds, the mean pass g0 -> g1 -> ...)
  for (int pass = 1; pass <= 2; ++pass) {
    for (int r = 0; r < n; ++r) {
      ctxs[r]->emu_pass = pass;
      const int st = dss_step(ctxs[r], t, alpha, 0, nullptr);
      ctxs[r]->emu_pass = 0;
      if (st != DSS_OK) return st;
    }
  }
  if (check) {
    for (int r = 0; r < n; ++r) {
      if (const int st = dss_check(ctxs[r])) return st;
    }
  }
  return DSS_OK;
}

extern "C" int dss_check_guards(dss_ctx* c, long* corrupted) {
  if (!c) return fail(nullptr, DSS_EINVAL, "null context");
  return guard(c, [&]() -> int {
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(c->stream), "guard sync");
    long bad = 0, first = -1;
    std::vector<unsigned char> h(static_cast<size_t>(c->guard));
    for (size_t i = 0; i < c->guarded.size(); ++i) {
      const auto& gb = c->guarded[i];
      for (const char* band : {gb.first - c->guard, gb.first + gb.second}) {
        ck(cudaMemcpy(h.data(), band, h.size(), cudaMemcpyDeviceToHost), "guard readback");
        for (unsigned char v : h) {
          if (v != kGuardByte) {
            ++bad;
            if (first < 0) first = static_cast<long>(i);
          }
        }
      }
    }
    if (corrupted) *corrupted = bad;
    if (bad) {
      return fail(c, DSS_ERUNTIME, "guard bands overwritten: " + std::to_string(bad) + " bytes (first in allocation " +
                                       std::to_string(first) + " of " + std::to_string(c->guarded.size()) + ")");
    }
    return DSS_OK;
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
