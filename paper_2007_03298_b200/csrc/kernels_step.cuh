// One GPU: the fused DS-Sync group step (apply_step of every member, ordered
// fold, x 1/m, broadcast), the fused BSP step, and whole iterations of tiny
// worlds in one CTA.
#pragma once

#include "kernel_common.cuh"
#include "kernels_problems.cuh"

namespace dssb {

// ---- fused DS-Sync group step ---------------------------------------------
template <typename T> struct GroupArgs {
  T* w;           // [P][ld] local params (row = global rank - first_rank)
  const T* g;     // [P][ld] gradients; g_ld == 0 -> one shared row (BSP multi-GPU)
  T* m1;
  T* m2;
  long ld;
  long g_ld;
  long nvec;      // vectors per row to process
  int first_rank;       // first slot on this GPU: local row = member slot - first_rank
  const int* rank_of;   // local row -> global rank (error keys)
  const int* members;  // CSR over the groups of this launch (slots; = global ranks for contiguous packing)
  const int* offsets;
  int step_phase;      // error phase for a failed local step
  int sync_phase;      // error phase for a failed group mean
  long t;
  StepConsts<T> c;
  double bc1[kMaxLocal];  // per local worker bias corrections (optim.cpp:76-78)
  double bc2[kMaxLocal];
  unsigned long long* err;
  // split barrier (first kernel after a two-shot push step): wait for every
  // GPU's barrier word to reach wait_epoch before touching rows; null: none
  const unsigned long long* wait_flags;
  int wait_n;
  unsigned long long wait_epoch;
  unsigned long long* timeout;
};

// blockIdx.y = group of this launch; threads stride over the row's vectors.
// Per element vector: for each member in ascending order load w, g, state;
// step; store state; fold.  Then scale once and store the mean to every
// member: each element of every array is read once and written once.
template <int OPT, int M>
constexpr int group_min_blocks() {
  return (OPT == kMomentum && M == 8)                    ? DSS_MIN_BLOCKS_M8_MOMENTUM
         : ((OPT == kAdam || OPT == kAdamW) && M == 8) ? DSS_MIN_BLOCKS_M8_ADAM
                                                        : DSS_MIN_BLOCKS;
}

template <typename T, int OPT, int M>
__global__ void __launch_bounds__(kThreads, group_min_blocks<OPT, M>()) ds_group_kernel(const GroupArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  split_wait(a.wait_flags, a.wait_n, a.wait_epoch, a.timeout);
  const int beg = a.offsets[blockIdx.y];
  const int m = M > 0 ? M : a.offsets[blockIdx.y + 1] - beg;
  const int lead = a.rank_of[a.members[beg] - a.first_rank];  // members[0]: a failed group mean's rank
  // 1.0 / m in double, rounded once to T (param.cpp:49 / comm.cpp:107)
  const T inv = static_cast<T>(1.0 / static_cast<double>(m));
  unsigned long long bad = ~0ull;

  // Per-member local row index hoisted out of the element loop (registers
  // for the templated group sizes); 64-bit offsets and bias corrections are
  // derived per use to keep register pressure low at M = 8.
  constexpr int RM = M > 0 ? M : 1;
  int lrow[RM];
  if constexpr (M > 0) {
#pragma unroll
    for (int j = 0; j < M; ++j) lrow[j] = a.members[beg + j] - a.first_rank;
  }

  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < a.nvec; e += stride) {
    const long off = e * VN;
    Pack<T> acc;
    if constexpr (M > 0) {
      // Templated group size: issue a chunk of members' loads first (w, g
      // and optimizer state of CH members in flight at once), then step,
      // store state and fold in ascending member order.  Without this split
      // a member's state stores would pin the next member's loads behind
      // them (the compiler cannot prove the rows do not alias).  Stateful
      // optimizers carry 3-4 arrays per member, so groups of 8 work in
      // chunks of 4 members to stay within 128 registers (2 CTAs / SM).
      constexpr int CH = OPT == kMomentum ? (M > DSS_CHUNK_MOMENTUM ? DSS_CHUNK_MOMENTUM : M)
                         : (OPT == kAdam || OPT == kAdamW) ? (M > DSS_CHUNK_ADAM ? DSS_CHUNK_ADAM : M)
                                                           : M;
#pragma unroll
      for (int c0 = 0; c0 < M; c0 += CH) {
        Pack<T> xs[CH], gs[CH], s1[CH], s2[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int j = c0 + q;
          const long rj = static_cast<long>(lrow[j]) * a.ld + off;
          xs[q] = ldv(a.w + rj);
          if constexpr (OPT != kOptNone) gs[q] = ldv(a.g + static_cast<long>(lrow[j]) * a.g_ld + off);
          if constexpr (OPT != kOptNone && OPT != kSgd) s1[q] = ldv(a.m1 + rj);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2[q] = ldv(a.m2 + rj);
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int j = c0 + q;
          if constexpr (OPT != kOptNone) {
            const long rj = static_cast<long>(lrow[j]) * a.ld + off;
            T b1j = T(1), b2j = T(1);
            if constexpr (OPT == kAdam || OPT == kAdamW) {
              b1j = static_cast<T>(a.bc1[lrow[j]]);
              b2j = static_cast<T>(a.bc2[lrow[j]]);
            }
            step_pack<T, OPT>(xs[q], gs[q], s1[q], s2[q], a.c, b1j, b2j);
            bool ok = true;
#pragma unroll
            for (int l = 0; l < VN; ++l) ok = ok && finite_(xs[q].v[l]);
            if constexpr (OPT != kSgd) stv(a.m1 + rj, s1[q]);
            if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + rj, s2[q]);
            if (!ok) {
              const unsigned long long k = err_key(a.t, a.step_phase, a.rank_of[lrow[j]]);
              bad = k < bad ? k : bad;
            }
          }
          if (j == 0) {
            acc = xs[q];
          } else {
#pragma unroll
            for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], xs[q].v[l]);
          }
        }
      }
    } else {
      // Any group size: stream members one at a time (acc in registers).
#pragma unroll 4
      for (int j = 0; j < m; ++j) {
        const int rk = a.members[beg + j];
        const int lr = rk - a.first_rank;
        const long rj = static_cast<long>(lr) * a.ld;
        const long gj = static_cast<long>(lr) * a.g_ld;
        Pack<T> x = ldv(a.w + rj + off);
        if constexpr (OPT != kOptNone) {
          const T b1j = static_cast<T>(a.bc1[lr]);
          const T b2j = static_cast<T>(a.bc2[lr]);
          const Pack<T> gv = ldv(a.g + gj + off);
          Pack<T> s1, s2;
          if constexpr (OPT != kSgd) s1 = ldv(a.m1 + rj + off);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + rj + off);
          step_pack<T, OPT>(x, gv, s1, s2, a.c, b1j, b2j);
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) ok = ok && finite_(x.v[l]);
          if constexpr (OPT != kSgd) stv(a.m1 + rj + off, s1);
          if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + rj + off, s2);
          if (!ok) {
            const unsigned long long k = err_key(a.t, a.step_phase, a.rank_of[lr]);
            bad = k < bad ? k : bad;
          }
        }
        if (j == 0) {
          acc = x;
        } else {
#pragma unroll
          for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x.v[l]);
        }
      }
    }
    if (M != 1) {
      bool ok = true;
#pragma unroll
      for (int l = 0; l < VN; ++l) {
        acc.v[l] = mul_(acc.v[l], inv);
        ok = ok && finite_(acc.v[l]);
      }
      if (!ok) {
        const unsigned long long k = err_key(a.t, a.sync_phase, lead);
        bad = k < bad ? k : bad;
      }
    }
    if constexpr (M > 0) {
#pragma unroll
      for (int j = 0; j < M; ++j) stv(a.w + static_cast<long>(lrow[j]) * a.ld + off, acc);
    } else {
#pragma unroll 4
      for (int j = 0; j < m; ++j) stv(a.w + static_cast<long>(a.members[beg + j] - a.first_rank) * a.ld + off, acc);
    }
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}

// ---- narrow-vector group step (fp32, 8-B vectors, every member in flight) ---
// ds_group_kernel with float2 instead of float4 per thread: half the
// registers per member, so a stateful group of 8 issues every member's
// w, g and state loads at once (no second load phase) within the 2-CTA/SM
// register budget.  Same arithmetic, same order.
template <int OPT, int M>
__global__ void __launch_bounds__(kThreads, 2) ds_group_narrow_kernel(const GroupArgs<float> a) {
  const int beg = a.offsets[blockIdx.y];
  const int lead = a.rank_of[a.members[beg] - a.first_rank];
  const float inv = static_cast<float>(1.0 / static_cast<double>(M));
  unsigned long long bad = ~0ull;
  int lrow[M];
#pragma unroll
  for (int j = 0; j < M; ++j) lrow[j] = a.members[beg + j] - a.first_rank;
  const long nv2 = a.nvec * 2;  // float2 vectors per row
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < nv2; e += stride) {
    const long off = e * 2;
    float2 xs[M], gs[M], s1[M], s2[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const long rj = static_cast<long>(lrow[j]) * a.ld + off;
      xs[j] = __ldcs(reinterpret_cast<const float2*>(a.w + rj));
      gs[j] = __ldcs(reinterpret_cast<const float2*>(a.g + static_cast<long>(lrow[j]) * a.g_ld + off));
      if constexpr (OPT != kSgd) s1[j] = __ldcs(reinterpret_cast<const float2*>(a.m1 + rj));
      if constexpr (OPT == kAdam || OPT == kAdamW) s2[j] = __ldcs(reinterpret_cast<const float2*>(a.m2 + rj));
    }
    float2 acc;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const long rj = static_cast<long>(lrow[j]) * a.ld + off;
      float b1j = 1.f, b2j = 1.f;
      if constexpr (OPT == kAdam || OPT == kAdamW) {
        b1j = static_cast<float>(a.bc1[lrow[j]]);
        b2j = static_cast<float>(a.bc2[lrow[j]]);
      }
      float m1a = 0.f, m1b = 0.f, m2a = 0.f, m2b = 0.f;
      if constexpr (OPT != kSgd) {
        m1a = s1[j].x;
        m1b = s1[j].y;
      }
      if constexpr (OPT == kAdam || OPT == kAdamW) {
        m2a = s2[j].x;
        m2b = s2[j].y;
      }
      const float xa = step_elem<float, OPT>(xs[j].x, gs[j].x, m1a, m2a, a.c, b1j, b2j);
      const float xb = step_elem<float, OPT>(xs[j].y, gs[j].y, m1b, m2b, a.c, b1j, b2j);
      if constexpr (OPT != kSgd) __stcs(reinterpret_cast<float2*>(a.m1 + rj), make_float2(m1a, m1b));
      if constexpr (OPT == kAdam || OPT == kAdamW) __stcs(reinterpret_cast<float2*>(a.m2 + rj), make_float2(m2a, m2b));
      if (!(finite_(xa) && finite_(xb))) {
        const unsigned long long k = err_key(a.t, a.step_phase, a.rank_of[lrow[j]]);
        bad = k < bad ? k : bad;
      }
      if (j == 0) {
        acc = make_float2(xa, xb);
      } else {
        acc.x = add_(acc.x, xa);
        acc.y = add_(acc.y, xb);
      }
    }
    acc.x = mul_(acc.x, inv);
    acc.y = mul_(acc.y, inv);
    if (!(finite_(acc.x) && finite_(acc.y))) {
      const unsigned long long k = err_key(a.t, a.sync_phase, lead);
      bad = k < bad ? k : bad;
    }
#pragma unroll
    for (int j = 0; j < M; ++j) __stcs(reinterpret_cast<float2*>(a.w + static_cast<long>(lrow[j]) * a.ld + off), acc);
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}

// ---- shared-memory-staged group step (cp.async.bulk + mbarrier ring) -------
// Same arithmetic as ds_group_kernel; for groups of 8 with stateful
// optimizers, where holding every member's w/g/m/v in registers caps the
// bytes in flight.  A producer warp streams each tile's member rows into a
// ring of NS shared-memory stages with 1-D TMA bulk copies
// (cp.async.bulk.shared::cluster.global, completion on an mbarrier); 8
// consumer warps step + fold from shared memory and store the state and the
// mean straight to HBM.
#ifndef DSS_BULK_TE
#define DSS_BULK_TE 256
#endif
#ifndef DSS_BULK_STAGES
#define DSS_BULK_STAGES 4
#endif
constexpr int kBulkTE = DSS_BULK_TE;          // elements per tile row
constexpr int kBulkStages = DSS_BULK_STAGES;  // ring depth

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait (~20 s): a broken pipeline latches a timeout instead of hanging
__device__ __forceinline__ bool mbar_wait(unsigned long long* bar, unsigned parity, unsigned long long* timeout) {
  unsigned long long start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (!mbar_try_wait(bar, parity)) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > 20000000000ull) {
      atomicExch(timeout, 1ull);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <typename T, int OPT, int M>
__global__ void __launch_bounds__(kThreads + 32, 1) ds_group_bulk_kernel(const GroupArgs<T> a,
                                                                         unsigned long long* timeout) {
  constexpr int A = (OPT == kAdam || OPT == kAdamW) ? 4 : (OPT == kMomentum ? 3 : 2);  // w, g, m1, m2
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);  // [NS][M][A][TE]
  __shared__ __align__(8) unsigned long long full[kBulkStages], empty[kBulkStages];
  const int tiles_per_row = static_cast<int>((a.ld + kBulkTE - 1) / kBulkTE);
  const long n_tiles = static_cast<long>(gridDim.y) * tiles_per_row;
  const int grp = blockIdx.y;
  const int beg = a.offsets[grp];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // tiles of this group handled by this CTA: x = blockIdx.x, blockIdx.x + gridDim.x, ...
  const int n_mine = tiles_per_row > static_cast<int>(blockIdx.x)
                         ? (tiles_per_row - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                         : 0;
  (void)n_tiles;
  if (threadIdx.x >= kThreads) {
    // producer warp: one lane issues every bulk copy
    if (threadIdx.x == kThreads) {
      for (int i = 0; i < n_mine; ++i) {
        const int s = i % kBulkStages;
        const int r = i / kBulkStages;
        if (r > 0 && !mbar_wait(&empty[s], static_cast<unsigned>((r - 1) & 1), timeout)) break;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const long e0 = static_cast<long>(blockIdx.x + i * gridDim.x) * kBulkTE;
        const long len = a.ld - e0 < kBulkTE ? a.ld - e0 : kBulkTE;
        const unsigned bytes = static_cast<unsigned>(len * sizeof(T));
        mbar_expect_tx(&full[s], bytes * M * A);
        T* st = stage + static_cast<long>(s) * M * A * kBulkTE;
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const long row = static_cast<long>(a.members[beg + j] - a.first_rank) * a.ld + e0;
          bulk_g2s(st + (j * A + 0) * kBulkTE, a.w + row, bytes, &full[s]);
          bulk_g2s(st + (j * A + 1) * kBulkTE, a.g + row, bytes, &full[s]);
          if constexpr (A >= 3) bulk_g2s(st + (j * A + 2) * kBulkTE, a.m1 + row, bytes, &full[s]);
          if constexpr (A >= 4) bulk_g2s(st + (j * A + 3) * kBulkTE, a.m2 + row, bytes, &full[s]);
        }
      }
    }
    return;
  }
  // consumers: thread x owns element e0 + x of every tile
  const int lead = a.rank_of[a.members[beg] - a.first_rank];
  const T inv = static_cast<T>(1.0 / static_cast<double>(M));
  int lr[M];
  T b1[M], b2[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    lr[j] = a.members[beg + j] - a.first_rank;
    b1[j] = static_cast<T>(a.bc1[lr[j]]);
    b2[j] = static_cast<T>(a.bc2[lr[j]]);
  }
  unsigned long long bad = ~0ull;
  for (int i = 0; i < n_mine; ++i) {
    const int s = i % kBulkStages;
    if (!mbar_wait(&full[s], static_cast<unsigned>((i / kBulkStages) & 1), timeout)) break;
    const long e0 = static_cast<long>(blockIdx.x + i * gridDim.x) * kBulkTE;
    const long len = a.ld - e0 < kBulkTE ? a.ld - e0 : kBulkTE;
    const T* st = stage + static_cast<long>(s) * M * A * kBulkTE;
    for (int x = threadIdx.x; x < len; x += kThreads) {
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        T w = st[(j * A + 0) * kBulkTE + x];
        const T gj = st[(j * A + 1) * kBulkTE + x];
        T s1 = T(0), s2 = T(0);
        if constexpr (A >= 3) s1 = st[(j * A + 2) * kBulkTE + x];
        if constexpr (A >= 4) s2 = st[(j * A + 3) * kBulkTE + x];
        w = step_elem<T, OPT>(w, gj, s1, s2, a.c, b1[j], b2[j]);
        const long gi = static_cast<long>(lr[j]) * a.ld + e0 + x;
        if constexpr (A >= 3) __stcs(a.m1 + gi, s1);
        if constexpr (A >= 4) __stcs(a.m2 + gi, s2);
        if (!finite_(w)) {
          const unsigned long long k = err_key(a.t, a.step_phase, a.rank_of[lr[j]]);
          bad = k < bad ? k : bad;
        }
        acc = j == 0 ? w : add_(acc, w);
      }
      acc = mul_(acc, inv);
      if (!finite_(acc)) {
        const unsigned long long k = err_key(a.t, a.sync_phase, lead);
        bad = k < bad ? k : bad;
      }
#pragma unroll
      for (int j = 0; j < M; ++j) __stcs(a.w + static_cast<long>(lr[j]) * a.ld + e0 + x, acc);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}

// ---- fused BSP step on one GPU --------------------------------------------
// gm = (sum_k g_k ascending) * (1/W) (sync.cpp:389-402 via mean_of order),
// then every worker w_k' = apply_step(w_k, gm) (sync.cpp:406-421).
template <typename T> struct BspArgs {
  T* w;
  const T* g;
  T* m1;
  T* m2;
  long ld;
  long nvec;
  int nw;  // W (all local)
  long t;
  StepConsts<T> c;
  double bc1[kMaxLocal];
  double bc2[kMaxLocal];
  unsigned long long* err;
};

template <typename T, int OPT, int WT>
__global__ void __launch_bounds__(kThreads, DSS_MIN_BLOCKS) bsp_kernel(const BspArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  const int nw = WT > 0 ? WT : a.nw;
  const T inv = static_cast<T>(1.0 / static_cast<double>(nw));
  unsigned long long bad = ~0ull;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < a.nvec; e += stride) {
    const long off = e * VN;
    Pack<T> gm;
    // params/state of the first BCH workers are loaded with the gradients;
    // the rest stream behind (stateful optimizers at W = 8 would otherwise
    // need > 128 registers)
    constexpr int BCH = WT == 0 ? 1 : (OPT != kSgd && WT > 4 ? 4 : WT);
    Pack<T> xs[BCH], s1[BCH], s2[BCH];
    if constexpr (WT > 0) {
      // every gradient and the first chunk of params/state in flight before
      // the first store
      Pack<T> gs[WT];
#pragma unroll
      for (int k = 0; k < WT; ++k) {
        const long r = static_cast<long>(k) * a.ld + off;
        gs[k] = ldv(a.g + r);
        if (k < BCH) {
          xs[k] = ldv(a.w + r);
          if constexpr (OPT != kSgd) s1[k] = ldv(a.m1 + r);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2[k] = ldv(a.m2 + r);
        }
      }
      gm = gs[0];
#pragma unroll
      for (int k = 1; k < WT; ++k) {
#pragma unroll
        for (int l = 0; l < VN; ++l) gm.v[l] = add_(gm.v[l], gs[k].v[l]);
      }
    } else {
      // any W: gradients in batches of 8 loads in flight, folded in order
      gm = ldv(a.g + off);
      int k = 1;
      for (; k + 8 <= nw; k += 8) {
        Pack<T> gb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) gb[q] = ldv(a.g + static_cast<long>(k + q) * a.ld + off);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
          for (int l = 0; l < VN; ++l) gm.v[l] = add_(gm.v[l], gb[q].v[l]);
        }
      }
      for (; k < nw; ++k) {
        const Pack<T> x = ldv(a.g + static_cast<long>(k) * a.ld + off);
#pragma unroll
        for (int l = 0; l < VN; ++l) gm.v[l] = add_(gm.v[l], x.v[l]);
      }
    }
    bool okm = true;
#pragma unroll
    for (int l = 0; l < VN; ++l) {
      gm.v[l] = mul_(gm.v[l], inv);
      okm = okm && finite_(gm.v[l]);
    }
    if (!okm) {  // collective failure -> DivergenceError(0, t) (sync.cpp:399-401)
      const unsigned long long k = err_key(a.t, 0, 0);
      bad = k < bad ? k : bad;
    }
    auto step_store = [&](int k, Pack<T>& x, Pack<T>& m1v, Pack<T>& m2v) {
      const long r = static_cast<long>(k) * a.ld + off;
      const T b1 = static_cast<T>(a.bc1[k]);
      const T b2 = static_cast<T>(a.bc2[k]);
      step_pack<T, OPT>(x, gm, m1v, m2v, a.c, b1, b2);
      bool ok = true;
#pragma unroll
      for (int l = 0; l < VN; ++l) ok = ok && finite_(x.v[l]);
      stv(a.w + r, x);
      if constexpr (OPT != kSgd) stv(a.m1 + r, m1v);
      if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, m2v);
      if (!ok) {
        const unsigned long long kk = err_key(a.t, 1, k);
        bad = kk < bad ? kk : bad;
      }
    };
    if constexpr (WT > 0) {
#pragma unroll
      for (int k = 0; k < BCH; ++k) step_store(k, xs[k], s1[k], s2[k]);
      // the remaining workers in chunks of BCH: a chunk's params and state
      // are all in flight before its first store
#pragma unroll
      for (int k0 = BCH; k0 < WT; k0 += BCH) {
#pragma unroll
        for (int q = 0; q < BCH; ++q) {
          if (k0 + q < WT) {
            const long r = static_cast<long>(k0 + q) * a.ld + off;
            xs[q] = ldv(a.w + r);
            if constexpr (OPT != kSgd) s1[q] = ldv(a.m1 + r);
            if constexpr (OPT == kAdam || OPT == kAdamW) s2[q] = ldv(a.m2 + r);
          }
        }
#pragma unroll
        for (int q = 0; q < BCH; ++q) {
          if (k0 + q < WT) step_store(k0 + q, xs[q], s1[q], s2[q]);
        }
      }
    } else {
      // any W: workers in batches of 4 whose loads are all in flight before
      // the batch's first store
      int k = 0;
      for (; k + 4 <= nw; k += 4) {
        Pack<T> x[4], m1v[4], m2v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long r = static_cast<long>(k + q) * a.ld + off;
          x[q] = ldv(a.w + r);
          if constexpr (OPT != kSgd) m1v[q] = ldv(a.m1 + r);
          if constexpr (OPT == kAdam || OPT == kAdamW) m2v[q] = ldv(a.m2 + r);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) step_store(k + q, x[q], m1v[q], m2v[q]);
      }
      for (; k < nw; ++k) {
        const long r = static_cast<long>(k) * a.ld + off;
        Pack<T> x, m1v, m2v;
        x = ldv(a.w + r);
        if constexpr (OPT != kSgd) m1v = ldv(a.m1 + r);
        if constexpr (OPT == kAdam || OPT == kAdamW) m2v = ldv(a.m2 + r);
        step_store(k, x, m1v, m2v);
      }
    }
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}


// ---- many iterations of a tiny problem in one CTA ---------------------------
// C1-sized worlds (W * d_pad of a few thousand elements) are launch-latency
// bound: one CTA runs n consecutive DS (or BSP) iterations with a
// __syncthreads() between them instead of a kernel launch.  The schedule of
// both parities, per-iteration alpha (and alpha*wd) and per-worker bias
// corrections live in device memory.  Same arithmetic as the other kernels.
template <typename T> struct SmallArgs {
  T* w;
  const T* g;
  T* m1;
  T* m2;
  long ld;
  long nvec;
  int nw;               // W (all local)
  const int* members[2];
  const int* offsets[2];
  int ngroups[2];
  int bsp;              // 1: world fold of the gradients, then every worker steps
  long t0;
  int n;
  const double* alpha;  // [n]
  const double* bc1;    // [n][nw]
  const double* bc2;
  double wd;
  StepConsts<T> c;      // alpha / awd overwritten per iteration
  unsigned long long* err;
  int logistic;         // 1: each iteration first computes the logistic gradients (lg) into g
  LogisticArgs lg;
  unsigned* bar;        // grid barrier counter (zero at launch) when gridDim.x > 1
};

// Barrier across a fully resident grid: arrival count on a zeroed counter,
// target = (iteration + 1) * gridDim.x.  The release fence publishes this
// CTA's stores of the iteration before its arrival.
__device__ __forceinline__ void small_grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

constexpr int kSmallLogiMaxDim = 256;    // features per worker in the fused small-world logistic path
constexpr int kSmallLogiMaxBatch = 256;  // batch size there

// Logistic gradients of every worker at iteration t inside the one-CTA
// small-world kernel: one warp per worker.  The reference walks the batch
// example by example (problems.cpp:273-282), but an example's margin only
// depends on w, so all margins are computed at once (lane b: z_b summed in
// feature order) and then every feature's sum is taken in example order
// (lane j): the same additions in the same order, with the critical path
// d + B steps long instead of B * (d + sigmoid).
template <typename T>
__device__ void small_logistic_grads(const SmallArgs<T>& a, long t, T* g) {
  constexpr int Q = kSmallLogiMaxDim / 32;
  __shared__ double wsm[kThreads / 32][kSmallLogiMaxDim];
  __shared__ double ysm[kThreads / 32][kSmallLogiMaxBatch];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  LogisticArgs L = a.lg;
  L.t = t;
  const int d = L.d;
  for (int k = warp; k < a.nw; k += kThreads / 32) {
    sample_batch_par(L, k, lane, 32, [] { __syncwarp(); }, [](bool p) { return __any_sync(0xffffffffu, p); });
    const T* wr = a.w + static_cast<long>(k) * a.ld;
    for (int j = lane; j < d; j += 32) wsm[warp][j] = static_cast<double>(wr[j]);
    __syncwarp();
    const int* bt = L.batch + static_cast<long>(k) * L.B;
    // every example's margin at once (lane b): z_b in the reference's
    // feature order, then -y_b * sigmoid(-y_b z_b)
    double max_nz = 0.0;
    bool nan_nz = false;
    for (int b = lane; b < L.B; b += 32) {
      const int idx = bt[b];
      const double* x = L.x + static_cast<long>(idx) * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = __dadd_rn(z, __dmul_rn(x[j], wsm[warp][j]));
      const double y = L.y[idx];
      const double nz = __dmul_rn(-y, z);
      ysm[warp][b] = __dmul_rn(-y, __ddiv_rn(1.0, __dadd_rn(1.0, exp(-nz))));
      max_nz = fmax(max_nz, nz);
      nan_nz = nan_nz || isnan(nz);
    }
    for (int off = 16; off > 0; off >>= 1) max_nz = fmax(max_nz, __shfl_xor_sync(0xffffffffu, max_nz, off));
    nan_nz = __any_sync(0xffffffffu, nan_nz);
    __syncwarp();
    // then every feature (lane j): the gradient sum in example order
    const double inv = __ddiv_rn(1.0, static_cast<double>(L.B));
    bool bad = false;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      if (j < d) {
        double acc = 0.0;
        for (int b = 0; b < L.B; ++b) acc = __dadd_rn(acc, __dmul_rn(ysm[warp][b], L.x[static_cast<long>(bt[b]) * d + j]));
        double v = __dmul_rn(acc, inv);
        if (L.l2 > 0.0) v = __dadd_rn(v, __dmul_rn(L.l2, wsm[warp][j]));
        bad = bad || !isfinite(v);
        g[static_cast<long>(k) * a.ld + j] = static_cast<T>(v);
      }
    }
    if (lane == 0) bad = bad || !logistic_loss_finite(L, bt, wr, max_nz, nan_nz);
    if (__any_sync(0xffffffffu, bad) && lane == 0) {
      atomicMin(L.gerr, (static_cast<unsigned long long>(t) << 32) | static_cast<unsigned int>(L.rank_of[k]));
    }
    __syncwarp();
  }
}

// NT = kThreads for the logistic phase and the resident grid; a one-CTA
// batch with more element vectors than kThreads runs wide (kSmallWide
// threads) so more rows are in flight per member-ordered load round.
template <typename T, int OPT, int NT = kThreads>
__global__ void __launch_bounds__(NT) small_steps_kernel(const SmallArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  unsigned long long bad = ~0ull;
  StepConsts<T> c = a.c;
  // both parities' schedule tables in shared memory: the group -> member
  // lookups are then not global-load rounds ahead of every row load
  __shared__ int s_members[2][kMaxLocal];
  __shared__ int s_offsets[2][kMaxLocal + 1];
  __shared__ T s_inv[2][kMaxLocal];  // 1/m per group, the same value every unit computed before
  if (!a.bsp) {
    for (int p = 0; p < 2; ++p) {
      for (int k = threadIdx.x; k < a.nw; k += blockDim.x) s_members[p][k] = a.members[p][k];
      for (int k = threadIdx.x; k <= a.ngroups[p]; k += blockDim.x) s_offsets[p][k] = a.offsets[p][k];
      for (int k = threadIdx.x; k < a.ngroups[p]; k += blockDim.x) {
        s_inv[p][k] = static_cast<T>(1.0 / static_cast<double>(a.offsets[p][k + 1] - a.offsets[p][k]));
      }
    }
    __syncthreads();
  }
  // this thread's first (group, element vector) unit; later units advance by
  // nthreads with a carry instead of a 64-bit divide per unit
  const long tid0 = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int grp0 = a.bsp ? 0 : static_cast<int>(tid0 / a.nvec);
  const long vec0 = a.bsp ? 0 : tid0 - static_cast<long>(grp0) * a.nvec;
  double alpha_next = a.alpha[0];  // next iteration's step size, loaded one iteration ahead
  for (int i = 0; i < a.n; ++i) {
    const long t = a.t0 + i;
    const double alpha_i = alpha_next;
    if (i + 1 < a.n) alpha_next = a.alpha[i + 1];
    c.alpha = static_cast<T>(alpha_i);
    c.awd = static_cast<T>(alpha_i * a.wd);
    if constexpr (NT == kThreads) {
      if (a.logistic) {
        small_logistic_grads(a, t, const_cast<T*>(a.g));
        __syncthreads();
      }
    }
    const long tid = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long nthreads = static_cast<long>(gridDim.x) * blockDim.x;
    if (a.bsp) {
      const T inv = static_cast<T>(1.0 / static_cast<double>(a.nw));
      for (long e = tid; e < a.nvec; e += nthreads) {
        const long off = e * VN;
        Pack<T> gm = ldv(a.g + off);
        // rank order; loads 4 rows ahead of the dependent adds
        for (int k0 = 1; k0 < a.nw; k0 += 4) {
          Pack<T> xs[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (k0 + q < a.nw) xs[q] = ldv(a.g + static_cast<long>(k0 + q) * a.ld + off);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (k0 + q < a.nw) {
#pragma unroll
              for (int l = 0; l < VN; ++l) gm.v[l] = add_(gm.v[l], xs[q].v[l]);
            }
          }
        }
        bool okm = true;
#pragma unroll
        for (int l = 0; l < VN; ++l) {
          gm.v[l] = mul_(gm.v[l], inv);
          okm = okm && finite_(gm.v[l]);
        }
        if (!okm) {
          const unsigned long long k = err_key(t, 0, 0);
          bad = k < bad ? k : bad;
        }
        for (int k0 = 0; k0 < a.nw; k0 += 4) {  // replicas, loads of 4 in flight
          Pack<T> xs[4], s1[4], s2[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (k0 + q < a.nw) {
              const long r = static_cast<long>(k0 + q) * a.ld + off;
              xs[q] = ldv(a.w + r);
              if constexpr (OPT != kSgd) s1[q] = ldv(a.m1 + r);
              if constexpr (OPT == kAdam || OPT == kAdamW) s2[q] = ldv(a.m2 + r);
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k0 + q;
            if (k < a.nw) {
              const long r = static_cast<long>(k) * a.ld + off;
              const T b1 = static_cast<T>(a.bc1[static_cast<long>(i) * a.nw + k]);
              const T b2 = static_cast<T>(a.bc2[static_cast<long>(i) * a.nw + k]);
              step_pack<T, OPT>(xs[q], gm, s1[q], s2[q], c, b1, b2);
              bool ok = true;
#pragma unroll
              for (int l = 0; l < VN; ++l) ok = ok && finite_(xs[q].v[l]);
              stv(a.w + r, xs[q]);
              if constexpr (OPT != kSgd) stv(a.m1 + r, s1[q]);
              if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2[q]);
              if (!ok) {
                const unsigned long long kk = err_key(t, 1, k);
                bad = kk < bad ? kk : bad;
              }
            }
          }
        }
      }
    } else {
      const int p = static_cast<int>(t & 1);
      const int* members = s_members[p];
      const int* offsets = s_offsets[p];
      const int ngroups = a.ngroups[p];
      const long nvec = a.nvec;
      const long units = static_cast<long>(ngroups) * nvec;
      int grp = grp0;
      long vec = vec0;
      for (long u = tid; u < units;) {
        const long off = vec * VN;
        const int beg = offsets[grp];
        const int m = offsets[grp + 1] - beg;
        Pack<T> acc;
        for (int j = 0; j < m; ++j) {
          const int k = members[beg + j];
          const long r = static_cast<long>(k) * a.ld + off;
          Pack<T> x = ldv(a.w + r);
          const Pack<T> gv = ldv(a.g + r);
          Pack<T> s1, s2;
          if constexpr (OPT != kSgd) s1 = ldv(a.m1 + r);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + r);
          const T b1 = static_cast<T>(a.bc1[static_cast<long>(i) * a.nw + k]);
          const T b2 = static_cast<T>(a.bc2[static_cast<long>(i) * a.nw + k]);
          step_pack<T, OPT>(x, gv, s1, s2, c, b1, b2);
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) ok = ok && finite_(x.v[l]);
          if constexpr (OPT != kSgd) stv(a.m1 + r, s1);
          if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2);
          if (!ok) {
            const unsigned long long kk = err_key(t, 0, k);
            bad = kk < bad ? kk : bad;
          }
          if (j == 0) {
            acc = x;
          } else {
#pragma unroll
            for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x.v[l]);
          }
        }
        if (m > 1) {
          const T inv = s_inv[p][grp];
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) {
            acc.v[l] = mul_(acc.v[l], inv);
            ok = ok && finite_(acc.v[l]);
          }
          if (!ok) {
            const unsigned long long kk = err_key(t, 1, members[beg]);
            bad = kk < bad ? kk : bad;
          }
        }
        for (int j = 0; j < m; ++j) stv(a.w + static_cast<long>(members[beg + j]) * a.ld + off, acc);
        u += nthreads;
        if (u >= units) break;
        vec += nthreads;
        if (vec >= nvec) {
          if (vec < 2 * nvec) {
            vec -= nvec;
            ++grp;
          } else {  // rows shorter than the thread count
            const long q = vec / nvec;
            grp += static_cast<int>(q);
            vec -= q * nvec;
          }
        }
      }
    }
    // iteration t's rows are final before t+1 reads them
    if (gridDim.x == 1) {
      __syncthreads();
    } else {
      small_grid_barrier(a.bar, static_cast<unsigned>(i + 1) * gridDim.x);
    }
  }
  if (bad != ~0ull) atomicMin(a.err, bad);
}

}  // namespace dssb
