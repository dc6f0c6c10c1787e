// sm_100a kernels of the DS-Sync step.
//
// Bandwidth-bound elementwise/reduction work: no tensor cores.  Every
// kernel streams worker rows with 128-bit vector loads/stores, one thread
// per vector, grid sized in multiples of the 148 SMs.  The reduction axis is
// the *member* axis (group size <= 8 typically) and its order is pinned by
// the reference (param.hpp:21-24): acc = x_0; acc += x_k ascending;
// acc *= 1/m.  One thread owns an element vector and folds all members in
// registers in that order, so no tree/shuffle ever re-associates the sum.
//
// All arithmetic goes through explicit round-to-nearest intrinsics
// (__fadd_rn/__dmul_rn ...), which are never contracted into FMA, matching
// the reference's SSE2 build without FMA contraction.  The file
// is also compiled with -fmad=false.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dssb {

constexpr int kThreads = 256;
constexpr int kMaxLocal = 128;  // local workers per GPU carried in kernel params

// Tuning knobs (compile-time; the defaults are the measured best, see
// DESIGN.md).  Members whose loads are issued together before the first
// state store, per optimizer, and the CTAs/SM the register cap targets.
#ifndef DSS_CHUNK_MOMENTUM
#define DSS_CHUNK_MOMENTUM 8
#endif
#ifndef DSS_CHUNK_ADAM
#define DSS_CHUNK_ADAM 4
#endif
#ifndef DSS_MIN_BLOCKS
#define DSS_MIN_BLOCKS 2
#endif
#ifndef DSS_MIN_BLOCKS_M8_MOMENTUM
#define DSS_MIN_BLOCKS_M8_MOMENTUM 1
#endif
// Chain fold pipelining: elements per chunk (one flag each) and resident
// CTAs per SM.  Small chunks and ~one round of CTAs per GPU let stage j+1
// start one round after stage j instead of after the whole row.
#ifndef DSS_CHAIN_CHUNK
#define DSS_CHAIN_CHUNK 8192
#endif
#ifndef DSS_CHAIN_CTAS_PER_SM
#define DSS_CHAIN_CTAS_PER_SM 8
#endif
// Rows up to this many bytes fold one-shot over NVLink (every member GPU
// gathers every member's row) instead of two-shot.
#ifndef DSS_ONESHOT_MAX_BYTES
#define DSS_ONESHOT_MAX_BYTES (512L << 10)
#endif
// 1: full system fence before each chunk's release flag; 0: rely on the
// cumulativity of st.release.sys after the CTA barrier (lighter).
#ifndef DSS_CHAIN_FENCE
#define DSS_CHAIN_FENCE 0
#endif

enum OptKind : int { kOptNone = -1, kSgd = 0, kMomentum = 1, kAdam = 2, kAdamW = 3 };

// ---- exact scalar ops ------------------------------------------------------
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ bool finite_(float a) { return isfinite(a); }
__device__ __forceinline__ bool finite_(double a) { return isfinite(a); }

// ---- 16-byte vectors ---------------------------------------------------------
template <typename T> struct Vec;
template <> struct Vec<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <> struct Vec<double> {
  using type = double2;
  static constexpr int n = 2;
};

template <typename T> struct Pack {
  T v[Vec<T>::n];
};

// Streaming loads/stores (evict-first): every byte is touched once per
// iteration and the working set is far larger than L2.
template <typename T>
__device__ __forceinline__ Pack<T> ldv(const T* p) {
  Pack<T> r;
  typename Vec<T>::type x = __ldcs(reinterpret_cast<const typename Vec<T>::type*>(p));
  static_assert(sizeof(x) == sizeof(r), "pack");
  *reinterpret_cast<typename Vec<T>::type*>(r.v) = x;
  return r;
}
template <typename T>
__device__ __forceinline__ void stv(T* p, const Pack<T>& r) {
  __stcs(reinterpret_cast<typename Vec<T>::type*>(p),
         *reinterpret_cast<const typename Vec<T>::type*>(r.v));
}
// Peer/remote rows: cache-global accesses (no L1 allocation); peer
// addresses bypass the local L2 anyway.
template <typename T>
__device__ __forceinline__ Pack<T> ldv_cg(const T* p) {
  Pack<T> r;
  *reinterpret_cast<typename Vec<T>::type*>(r.v) =
      __ldcg(reinterpret_cast<const typename Vec<T>::type*>(p));
  return r;
}
template <typename T>
__device__ __forceinline__ void stv_cg(T* p, const Pack<T>& r) {
  __stcg(reinterpret_cast<typename Vec<T>::type*>(p),
         *reinterpret_cast<const typename Vec<T>::type*>(r.v));
}

// ---- optimizer constants for one launch (rounded once from double) ---------
template <typename T> struct StepConsts {
  T alpha;   // a
  T wd;      // weight_decay
  T mom;     // momentum
  T b1, omb1;  // beta1, 1 - beta1 (computed in double, optim.cpp:84)
  T b2, omb2;  // beta2, 1 - beta2
  T eps;
  T awd;     // a * weight_decay (optim.cpp:89, left-to-right)
};

// apply_step for one element (optim.cpp:56-91).  Operator order is the
// reference's, left to right:
//   sgd:      ge = g + wd*w;               w' = w - a*ge
//   momentum: ge = g + wd*w; b = mom*b + ge; w' = w - a*b
//   adam(w):  ge = adam ? g + wd*w : g
//             m = b1*m + (1-b1)*ge;  v = b2*v + ((1-b2)*ge)*ge
//             w' = w - (a*(m/bc1)) / (sqrt(v/bc2) + eps);  adamw: w' -= (a*wd)*w
template <typename T, int OPT>
__device__ __forceinline__ T step_elem(T w, T g, T& m1, T& m2, const StepConsts<T>& c, T bc1, T bc2) {
  if constexpr (OPT == kSgd) {
    const T ge = add_(g, mul_(c.wd, w));
    return sub_(w, mul_(c.alpha, ge));
  } else if constexpr (OPT == kMomentum) {
    const T ge = add_(g, mul_(c.wd, w));
    m1 = add_(mul_(c.mom, m1), ge);
    return sub_(w, mul_(c.alpha, m1));
  } else {
    const T ge = (OPT == kAdam) ? add_(g, mul_(c.wd, w)) : g;
    m1 = add_(mul_(c.b1, m1), mul_(c.omb1, ge));
    m2 = add_(mul_(c.b2, m2), mul_(mul_(c.omb2, ge), ge));
    const T mhat = div_(m1, bc1);
    const T vhat = div_(m2, bc2);
    T out = sub_(w, div_(mul_(c.alpha, mhat), add_(sqrt_(vhat), c.eps)));
    if constexpr (OPT == kAdamW) out = sub_(out, mul_(c.awd, w));
    return out;
  }
}

// ---- divergence latch ----------------------------------------------------
// key = t << 34 | phase << 32 | rank; atomicMin keeps the earliest iteration,
// then phase (DS: 0 local step before 1 group sync, sync.cpp:348-370; BSP:
// 0 gradient collective before 1 step, sync.cpp:389-421), then lowest rank
// (sync.cpp:126-128).
__device__ __forceinline__ unsigned long long err_key(long t, int phase, int rank) {
  return (static_cast<unsigned long long>(t) << 34) |
         (static_cast<unsigned long long>(phase) << 32) | static_cast<unsigned int>(rank);
}

__device__ __forceinline__ void latch_error(unsigned long long* err, unsigned long long key) {
  // warp-aggregate: one atomic per warp that saw a failure
  const unsigned mask = __activemask();
  unsigned long long k = key;
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(mask, k, off);
    k = o < k ? o : k;
  }
  if ((threadIdx.x & 31) == (__ffs(mask) - 1) && k != ~0ull) atomicMin(err, k);
}

// ---- fused DS-Sync group step ---------------------------------------------
template <typename T> struct GroupArgs {
  T* w;           // [P][ld] local params (row = global rank - first_rank)
  const T* g;     // [P][ld] gradients; g_ld == 0 -> one shared row (BSP multi-GPU)
  T* m1;
  T* m2;
  long ld;
  long g_ld;
  long nvec;      // vectors per row to process
  int first_rank;
  const int* members;  // CSR over the groups of this launch (global ranks)
  const int* offsets;
  int step_phase;      // error phase for a failed local step
  int sync_phase;      // error phase for a failed group mean
  long t;
  StepConsts<T> c;
  double bc1[kMaxLocal];  // per local worker bias corrections (optim.cpp:76-78)
  double bc2[kMaxLocal];
  unsigned long long* err;
};

// blockIdx.y = group of this launch; threads stride over the row's vectors.
// Per element vector: for each member in ascending order load w, g, state;
// step; store state; fold.  Then scale once and store the mean to every
// member: each element of every array is read once and written once.
template <int OPT, int M>
constexpr int group_min_blocks() {
  return (OPT == kMomentum && M == 8) ? DSS_MIN_BLOCKS_M8_MOMENTUM : DSS_MIN_BLOCKS;
}

template <typename T, int OPT, int M>
__global__ void __launch_bounds__(kThreads, group_min_blocks<OPT, M>()) ds_group_kernel(const GroupArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  const int beg = a.offsets[blockIdx.y];
  const int m = M > 0 ? M : a.offsets[blockIdx.y + 1] - beg;
  const int lead = a.members[beg];
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
            bool ok = true;
#pragma unroll
            for (int l = 0; l < VN; ++l) {
              xs[q].v[l] = step_elem<T, OPT>(xs[q].v[l], gs[q].v[l], s1[q].v[l], s2[q].v[l], a.c, b1j, b2j);
              ok = ok && finite_(xs[q].v[l]);
            }
            if constexpr (OPT != kSgd) stv(a.m1 + rj, s1[q]);
            if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + rj, s2[q]);
            if (!ok) {
              const unsigned long long k = err_key(a.t, a.step_phase, lrow[j] + a.first_rank);
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
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) {
            x.v[l] = step_elem<T, OPT>(x.v[l], gv.v[l], s1.v[l], s2.v[l], a.c, b1j, b2j);
            ok = ok && finite_(x.v[l]);
          }
          if constexpr (OPT != kSgd) stv(a.m1 + rj + off, s1);
          if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + rj + off, s2);
          if (!ok) {
            const unsigned long long k = err_key(a.t, a.step_phase, rk);
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
  const int lead = a.members[beg];
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
          const unsigned long long k = err_key(a.t, a.step_phase, a.first_rank + lr[j]);
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
      bool ok = true;
#pragma unroll
      for (int l = 0; l < VN; ++l) {
        x.v[l] = step_elem<T, OPT>(x.v[l], gm.v[l], m1v.v[l], m2v.v[l], a.c, b1, b2);
        ok = ok && finite_(x.v[l]);
      }
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
      for (int k = 0; k < WT; ++k) {
        Pack<T> x, m1v, m2v;
        if (k < BCH) {
          x = xs[k];
          m1v = s1[k];
          m2v = s2[k];
        } else {
          const long r = static_cast<long>(k) * a.ld + off;
          x = ldv(a.w + r);
          if constexpr (OPT != kSgd) m1v = ldv(a.m1 + r);
          if constexpr (OPT == kAdam || OPT == kAdamW) m2v = ldv(a.m2 + r);
        }
        step_store(k, x, m1v, m2v);
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
__device__ __forceinline__ uint64_t mix64(uint64_t z);

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

struct LogisticArgs {
  const double* x;        // [M][d] row-major
  const double* y;        // [M] labels in {-1, +1}
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
  int first_rank;
  unsigned long long* gerr;  // gradient failure latch: t << 32 | rank
};

__device__ __forceinline__ double softplus_dev(double z) {  // problems.cpp:338-341
  return z > 0.0 ? __dadd_rn(z, log1p(exp(-z))) : log1p(exp(z));
}

// sample_batch (sync.cpp:153-179) for local worker k, into a.batch[k].
__device__ void sample_batch_dev(const LogisticArgs& a, int k) {
  const int rank = a.first_rank + k;
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
  const int rank = a.first_rank + k;
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
};

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
      atomicMin(L.gerr, (static_cast<unsigned long long>(t) << 32) | static_cast<unsigned int>(L.first_rank + k));
    }
    __syncwarp();
  }
}

template <typename T, int OPT>
__global__ void __launch_bounds__(kThreads) small_steps_kernel(const SmallArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  unsigned long long bad = ~0ull;
  StepConsts<T> c = a.c;
  for (int i = 0; i < a.n; ++i) {
    const long t = a.t0 + i;
    c.alpha = static_cast<T>(a.alpha[i]);
    c.awd = static_cast<T>(a.alpha[i] * a.wd);
    if (a.logistic) {
      small_logistic_grads(a, t, const_cast<T*>(a.g));
      __syncthreads();
    }
    if (a.bsp) {
      const T inv = static_cast<T>(1.0 / static_cast<double>(a.nw));
      for (long e = threadIdx.x; e < a.nvec; e += blockDim.x) {
        const long off = e * VN;
        Pack<T> gm = ldv(a.g + off);
        for (int k = 1; k < a.nw; ++k) {
          const Pack<T> x = ldv(a.g + static_cast<long>(k) * a.ld + off);
#pragma unroll
          for (int l = 0; l < VN; ++l) gm.v[l] = add_(gm.v[l], x.v[l]);
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
        for (int k = 0; k < a.nw; ++k) {
          const long r = static_cast<long>(k) * a.ld + off;
          Pack<T> x = ldv(a.w + r);
          Pack<T> s1, s2;
          if constexpr (OPT != kSgd) s1 = ldv(a.m1 + r);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + r);
          const T b1 = static_cast<T>(a.bc1[static_cast<long>(i) * a.nw + k]);
          const T b2 = static_cast<T>(a.bc2[static_cast<long>(i) * a.nw + k]);
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) {
            x.v[l] = step_elem<T, OPT>(x.v[l], gm.v[l], s1.v[l], s2.v[l], c, b1, b2);
            ok = ok && finite_(x.v[l]);
          }
          stv(a.w + r, x);
          if constexpr (OPT != kSgd) stv(a.m1 + r, s1);
          if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2);
          if (!ok) {
            const unsigned long long kk = err_key(t, 1, k);
            bad = kk < bad ? kk : bad;
          }
        }
      }
    } else {
      const int p = static_cast<int>(t & 1);
      const int* members = a.members[p];
      const int* offsets = a.offsets[p];
      const long units = static_cast<long>(a.ngroups[p]) * a.nvec;
      for (long u = threadIdx.x; u < units; u += blockDim.x) {
        const int grp = static_cast<int>(u / a.nvec);
        const long off = (u % a.nvec) * VN;
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
          bool ok = true;
#pragma unroll
          for (int l = 0; l < VN; ++l) {
            x.v[l] = step_elem<T, OPT>(x.v[l], gv.v[l], s1.v[l], s2.v[l], c, b1, b2);
            ok = ok && finite_(x.v[l]);
          }
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
          const T inv = static_cast<T>(1.0 / static_cast<double>(m));
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
      }
    }
    __syncthreads();  // iteration t's rows are final before t+1 reads them
  }
  if (bad != ~0ull) atomicMin(a.err, bad);
}

// ---- ordered fold + broadcast over (possibly peer-mapped) rows ------------
// Two-shot slice owner: for e in [lo, hi): acc = src_0; acc += src_j
// ascending; acc *= 1/m; store to every dst.  src/dst are device pointers to
// row starts; for a group spanning GPUs they are NVLink peer mappings, so
// this kernel is the cross-GPU collective itself (P2P loads and stores over
// NVSwitch from inside the kernel, no NCCL).
struct FoldEntry {
  int src_beg, src_cnt;  // into the src pointer table
  int dst_beg, dst_cnt;  // into the dst pointer table
  long lo, hi;           // element range (multiples of the vector width)
  int err_rank;          // members[0] (sync.cpp:233-235) or 0 for BSP (sync.cpp:401)
  int err_phase;
};

template <typename T> struct FoldArgs {
  T* const* src;
  T* const* dst;
  const FoldEntry* entries;
  long t;
  unsigned long long* err;
};

constexpr int kMaxFold = 64;  // members (sources) / destinations per entry held in shared memory

template <typename T, int M>
__global__ void __launch_bounds__(kThreads) fold_kernel(const FoldArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  // Entry and its peer-pointer lists are read once into shared memory: the
  // element loop then has no dependent pointer loads in front of its NVLink
  // accesses (the stores could alias the tables, so the compiler would
  // otherwise reload them every iteration).
  __shared__ FoldEntry en;
  __shared__ T* s_src[kMaxFold];
  __shared__ T* s_dst[kMaxFold];
  if (threadIdx.x == 0) en = a.entries[blockIdx.y];
  __syncthreads();
  for (int q = threadIdx.x; q < en.src_cnt; q += blockDim.x) s_src[q] = a.src[en.src_beg + q];
  for (int q = threadIdx.x; q < en.dst_cnt; q += blockDim.x) s_dst[q] = a.dst[en.dst_beg + q];
  __syncthreads();
  const int m = M > 0 ? M : en.src_cnt;
  const int nd = en.dst_cnt;
  const T inv = static_cast<T>(1.0 / static_cast<double>(m));
  constexpr int RM = M > 0 ? M : 1;
  T* src[RM];
  if constexpr (M > 0) {
#pragma unroll
    for (int j = 0; j < M; ++j) src[j] = s_src[j];
  }
  unsigned long long bad = ~0ull;
  const long v0 = en.lo / VN, v1 = en.hi / VN;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = v0 + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < v1; e += stride) {
    const long off = e * VN;
    Pack<T> acc;
    if constexpr (M > 0) {
      // all member loads (local and NVLink peer) in flight, then the
      // ordered fold
      Pack<T> x[M];
#pragma unroll
      for (int j = 0; j < M; ++j) x[j] = ldv_cg(src[j] + off);
      acc = x[0];
#pragma unroll
      for (int j = 1; j < M; ++j) {
#pragma unroll
        for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x[j].v[l]);
      }
    } else {
      acc = ldv_cg(s_src[0] + off);
#pragma unroll 4
      for (int j = 1; j < m; ++j) {
        const Pack<T> x = ldv_cg(s_src[j] + off);
#pragma unroll
        for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x.v[l]);
      }
    }
    bool ok = true;
#pragma unroll
    for (int l = 0; l < VN; ++l) {
      acc.v[l] = mul_(acc.v[l], inv);
      ok = ok && finite_(acc.v[l]);
    }
    if (!ok) {
      const unsigned long long k = err_key(a.t, en.err_phase, en.err_rank);
      bad = k < bad ? k : bad;
    }
    for (int q = 0; q < nd; ++q) stv_cg(s_dst[q] + off, acc);
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
  // Peer stores must be performed system-wide before the next cross-GPU
  // barrier lets the owners of those rows read them.
  __threadfence_system();
}

// ---- cross-GPU barrier over NVLink-mapped flag words ------------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Thread j tells GPU j "rank reached epoch", then waits until GPU j has told
// us the same.  Bounded spin (~20 s of globaltimer) so a broken peer cannot
// wedge the GPU: on timeout the barrier latches a failure instead.
__global__ void barrier_kernel(unsigned long long* const* peer_flags, unsigned long long* my_flags,
                               int rank, int n, unsigned long long epoch, unsigned long long* timeout) {
  const int j = threadIdx.x;
  if (j >= n) return;
  __threadfence_system();
  st_release_sys(peer_flags[j] + rank, epoch);
  unsigned long long start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (ld_acquire_sys(my_flags + j) < epoch) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > 20000000000ull) {
      atomicExch(timeout, 1ull);
      break;
    }
  }
  __threadfence_system();
}

// ---- ordered chain fold across GPUs (comm.cpp:96-110) -------
// A group spanning GPUs g_0 < ... < g_{S-1}, each holding a contiguous run
// of its ascending members, is folded as the reference's ring does: the
// partial leaves g_0 after its run, every next GPU *continues* the same
// left-to-right fold with its own run (acc = (...(p + x_a) + x_{a+1}) ...),
// the last GPU scales by 1/m.  The mean then travels g_{S-1} -> g_0 -> g_1
// -> ... -> g_{S-2}.  Both passes are pipelined over chunks of the row with
// per-chunk epoch flags in the receiver's memory (st.release.sys /
// ld.acquire.sys), so each GPU moves ~2 rows over NVLink per group instead
// of one per member, and the fold order is bit-exact.
struct ChainEntry {
  int stage;          // position j of this GPU in the group's GPU list
  int last;           // j == S-1
  int run_beg, run_cnt;   // this GPU's members: rows in the src pointer table
  int dst_beg, dst_cnt;   // where the mean lands on this GPU
  void* recv;         // local partial-receive row (j > 0) / mean-receive row (kernel B)
  unsigned long long* recv_flags;  // local flags [n_chunks]
  void* send;         // next GPU's receive row (remote), or nullptr
  unsigned long long* send_flags;  // next GPU's flags (remote), or nullptr
  int err_rank;
  int err_phase;
  int m;              // group size (1/m)
};

template <typename T> struct ChainArgs {
  T* const* src;      // member rows (local)
  T* const* dst;      // mean destinations (local)
  const int* src_lr;  // local row index of each src entry (fused member step)
  const int* dst_lr;  // local row index of each dst entry (fused BSP replica step)
  const ChainEntry* entries;
  int n_entries;
  long chunk;         // elements per chunk (multiple of 64)
  long len;           // row length (d_pad)
  long n_chunks;
  unsigned long long epoch;
  long t;
  unsigned long long* err;
  unsigned long long* timeout;
  // fused optimizer step (DS: on the members before they are folded; BSP: on
  // every local replica with the mean gradient as it arrives)
  T* stage;           // local row the mean is parked in before the replica step (BSP)
  const T* g;
  T* m1;
  T* m2;
  long ld;
  int first_rank;
  int step_phase;
  StepConsts<T> c;
  double bc1[kMaxLocal];
  double bc2[kMaxLocal];
};

__device__ __forceinline__ bool chain_wait(const unsigned long long* flag, unsigned long long epoch,
                                           unsigned long long* timeout) {
  unsigned long long start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (ld_acquire_sys(flag) < epoch) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > 20000000000ull) {
      atomicExch(timeout, 1ull);
      return false;
    }
  }
  return true;
}

// apply_step of one local row's vector at `off` with gradient gv (in
// registers); state read and written in place.  Returns the stepped params.
template <typename T, int OPT>
__device__ __forceinline__ Pack<T> chain_step(const ChainArgs<T>& a, T* wrow, int lr, long off, const Pack<T>& gv,
                                              unsigned long long& bad, int phase) {
  constexpr int VN = Vec<T>::n;
  const long r = static_cast<long>(lr) * a.ld + off;
  Pack<T> x = ldv(wrow + off);
  Pack<T> s1, s2;
  if constexpr (OPT != kSgd) s1 = ldv(a.m1 + r);
  if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + r);
  const T b1 = static_cast<T>(a.bc1[lr]);
  const T b2 = static_cast<T>(a.bc2[lr]);
  bool ok = true;
#pragma unroll
  for (int l = 0; l < VN; ++l) {
    x.v[l] = step_elem<T, OPT>(x.v[l], gv.v[l], s1.v[l], s2.v[l], a.c, b1, b2);
    ok = ok && finite_(x.v[l]);
  }
  if constexpr (OPT != kSgd) stv(a.m1 + r, s1);
  if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2);
  if (!ok) {
    const unsigned long long k = err_key(a.t, phase, a.first_rank + lr);
    bad = k < bad ? k : bad;
  }
  return x;
}

// Step up to 4 local rows (lr[q], params at wrow[q]) with gradients gv[q]
// in one load phase: every row's params and state are in flight before the
// first store (the per-row path would expose one HBM latency per row).
template <typename T, int OPT, int B>
__device__ __forceinline__ void chain_step_batch(const ChainArgs<T>& a, T* const* wrow, const int* lr, long off,
                                                 const Pack<T>* gv, Pack<T>* out, unsigned long long& bad, int phase) {
  constexpr int VN = Vec<T>::n;
  Pack<T> x[B], s1[B], s2[B];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const long r = static_cast<long>(lr[q]) * a.ld + off;
    x[q] = ldv(wrow[q] + off);
    if constexpr (OPT != kSgd) s1[q] = ldv(a.m1 + r);
    if constexpr (OPT == kAdam || OPT == kAdamW) s2[q] = ldv(a.m2 + r);
  }
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const long r = static_cast<long>(lr[q]) * a.ld + off;
    const T b1 = static_cast<T>(a.bc1[lr[q]]);
    const T b2 = static_cast<T>(a.bc2[lr[q]]);
    bool ok = true;
#pragma unroll
    for (int l = 0; l < VN; ++l) {
      x[q].v[l] = step_elem<T, OPT>(x[q].v[l], gv[q].v[l], s1[q].v[l], s2[q].v[l], a.c, b1, b2);
      ok = ok && finite_(x[q].v[l]);
    }
    if constexpr (OPT != kSgd) stv(a.m1 + r, s1[q]);
    if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2[q]);
    if (!ok) {
      const unsigned long long k = err_key(a.t, phase, a.first_rank + lr[q]);
      bad = k < bad ? k : bad;
    }
    out[q] = x[q];
  }
}

// Deliver the mean vector of one element range on this GPU: store it to the
// destinations (OPTD none) or step every local replica with it (BSP, OPTD),
// replicas in batches of 4.
template <typename T, int OPTD>
__device__ __forceinline__ void chain_deliver(const ChainArgs<T>& a, const ChainEntry& en, long off,
                                              const Pack<T>& mean, unsigned long long& bad) {
  if constexpr (OPTD == kOptNone) {
    for (int q = 0; q < en.dst_cnt; ++q) stv(a.dst[en.dst_beg + q] + off, mean);
  } else {
    const Pack<T> gv[4] = {mean, mean, mean, mean};
    Pack<T> out[4];
    int q = 0;
    for (; q + 4 <= en.dst_cnt; q += 4) {
      chain_step_batch<T, OPTD, 4>(a, a.dst + en.dst_beg + q, a.dst_lr + en.dst_beg + q, off, gv, out, bad, 1);
#pragma unroll
      for (int b = 0; b < 4; ++b) stv(a.dst[en.dst_beg + q + b] + off, out[b]);
    }
    for (; q < en.dst_cnt; ++q) {
      chain_step_batch<T, OPTD, 1>(a, a.dst + en.dst_beg + q, a.dst_lr + en.dst_beg + q, off, gv, out, bad, 1);
      stv(a.dst[en.dst_beg + q] + off, out[0]);
    }
  }
}

// Kernel A: the ordered partial pass.  Work unit = (chunk, entry), visited
// chunk-major so every chain advances together.  A CTA only ever waits on a
// flag written by the previous GPU's kernel A, which itself only waits on
// GPUs before it: no cycle, no same-GPU dependency.  OPTM != none fuses the
// members' optimizer step into the pass (DS): the stepped params are folded
// straight from registers and never written back -- each member row is read
// once (w, g, state) and written once (state now, the mean later) while the
// chunk's partial goes over NVLink.
template <typename T, int OPTM, int OPTD>
__device__ __forceinline__ void chain_unit_a(const ChainArgs<T>& a, const ChainEntry* entries, int n_entries, long u,
                                             ChainEntry& en, int& ok_flag, unsigned long long& bad) {
  constexpr int VN = Vec<T>::n;
  const long c = u / n_entries;
  const int ei = static_cast<int>(u % n_entries);
  if (threadIdx.x == 0) {
    en = entries[ei];
    ok_flag = 1;
    if (en.stage > 0) ok_flag = chain_wait(en.recv_flags + c, a.epoch, a.timeout) ? 1 : 0;
  }
  __syncthreads();
  const long lo = c * a.chunk;
  const long hi = lo + a.chunk < a.len ? lo + a.chunk : a.len;
  const T inv = static_cast<T>(1.0 / static_cast<double>(en.m));
  if (ok_flag) {
    for (long e = lo / VN + threadIdx.x; e < hi / VN; e += blockDim.x) {
      const long off = e * VN;
      Pack<T> acc;
      if constexpr (OPTM != kOptNone) {
        // fused member step, members in load batches of up to 4, folded
        // in ascending order straight from registers
        int j = 0;
        bool first = en.stage == 0;
        if (!first) acc = ldv_cg(static_cast<const T*>(en.recv) + off);
        while (j < en.run_cnt) {
          const int nb = en.run_cnt - j >= 4 ? 4 : (en.run_cnt - j >= 2 ? 2 : 1);
          Pack<T> gv[4], x[4];
          const int* lrs = a.src_lr + en.run_beg + j;
          for (int q = 0; q < nb; ++q) gv[q] = ldv(a.g + static_cast<long>(lrs[q]) * a.ld + off);
          if (nb == 4) {
            chain_step_batch<T, OPTM, 4>(a, a.src + en.run_beg + j, lrs, off, gv, x, bad, a.step_phase);
          } else if (nb == 2) {
            chain_step_batch<T, OPTM, 2>(a, a.src + en.run_beg + j, lrs, off, gv, x, bad, a.step_phase);
          } else {
            chain_step_batch<T, OPTM, 1>(a, a.src + en.run_beg + j, lrs, off, gv, x, bad, a.step_phase);
          }
          for (int q = 0; q < nb; ++q) {
            if (first) {
              acc = x[q];
              first = false;
            } else {
#pragma unroll
              for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x[q].v[l]);
            }
          }
          j += nb;
        }
      } else {
        int j0 = 0;
        if (en.stage == 0) {
          acc = ldv(a.src[en.run_beg] + off);
          j0 = 1;
        } else {
          acc = ldv_cg(static_cast<const T*>(en.recv) + off);
        }
        for (int j = j0; j < en.run_cnt; ++j) {
          const Pack<T> x = ldv(a.src[en.run_beg + j] + off);
#pragma unroll
          for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x.v[l]);
        }
      }
      if (!en.last) {
        stv_cg(static_cast<T*>(en.send) + off, acc);
      } else {
        bool ok = true;
#pragma unroll
        for (int l = 0; l < VN; ++l) {
          acc.v[l] = mul_(acc.v[l], inv);
          ok = ok && finite_(acc.v[l]);
        }
        if (!ok) {
          const unsigned long long k = err_key(a.t, en.err_phase, en.err_rank);
          bad = k < bad ? k : bad;
        }
        if (en.send) stv_cg(static_cast<T*>(en.send) + off, acc);
        if constexpr (OPTD == kOptNone) {
          chain_deliver<T, OPTD>(a, en, off, acc, bad);
        } else {
          stv(a.stage + off, acc);  // replicas step after the flag is out
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && en.send) {
    if (DSS_CHAIN_FENCE) __threadfence_system();
    st_release_sys(en.send_flags + c, a.epoch);
  }
  if constexpr (OPTD != kOptNone) {
    // the next GPU already has this chunk: now step the local replicas
    // with it, off the inter-GPU critical path
    if (ok_flag && en.last) {
      for (long e = lo / VN + threadIdx.x; e < hi / VN; e += blockDim.x) {
        const long off = e * VN;
        chain_deliver<T, OPTD>(a, en, off, ldv(a.stage + off), bad);
      }
    }
  }
  __syncthreads();
}

// Kernel A: the ordered partial pass.  Work unit = (chunk, entry), visited
// chunk-major so every chain advances together.  A CTA only ever waits on a
// flag written by the previous GPU's kernel A, which itself only waits on
// GPUs before it: no cycle, no same-GPU dependency.  OPTM != none fuses the
// members' optimizer step into the pass (DS): the stepped params are folded
// straight from registers and never written back -- each member row is read
// once (w, g, state) and written once (state now, the mean later) while the
// chunk's partial goes over NVLink.
template <typename T, int OPTM, int OPTD>
__global__ void __launch_bounds__(kThreads) chain_partial_kernel(const ChainArgs<T> a) {
  __shared__ ChainEntry en;
  __shared__ int ok_flag;
  const long units = a.n_chunks * a.n_entries;
  unsigned long long bad = ~0ull;
  for (long u = blockIdx.x; u < units; u += gridDim.x) {
    chain_unit_a<T, OPTM, OPTD>(a, a.entries, a.n_entries, u, en, ok_flag, bad);
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}

// Kernel B: the mean pass g_{S-1} -> g_0 -> ... -> g_{S-2}: wait for the
// chunk, deliver it on this GPU (store, or step the replicas: BSP), forward.
template <typename T, int OPTD>
__device__ __forceinline__ void chain_unit_b(const ChainArgs<T>& a, const ChainEntry* entries, int n_entries, long u,
                                             ChainEntry& en, int& ok_flag, unsigned long long& bad) {
  constexpr int VN = Vec<T>::n;
  const long c = u / n_entries;
  const int ei = static_cast<int>(u % n_entries);
  if (threadIdx.x == 0) {
    en = entries[ei];
    ok_flag = chain_wait(en.recv_flags + c, a.epoch, a.timeout) ? 1 : 0;
  }
  __syncthreads();
  const long lo = c * a.chunk;
  const long hi = lo + a.chunk < a.len ? lo + a.chunk : a.len;
  if (ok_flag) {
    for (long e = lo / VN + threadIdx.x; e < hi / VN; e += blockDim.x) {
      const long off = e * VN;
      const Pack<T> mean = ldv_cg(static_cast<const T*>(en.recv) + off);
      if (en.send) stv_cg(static_cast<T*>(en.send) + off, mean);
      if constexpr (OPTD == kOptNone) chain_deliver<T, OPTD>(a, en, off, mean, bad);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && en.send) {
    if (DSS_CHAIN_FENCE) __threadfence_system();
    st_release_sys(en.send_flags + c, a.epoch);
  }
  if constexpr (OPTD != kOptNone) {
    // forwarded: now the (HBM-heavy) replica step, off the critical path
    if (ok_flag) {
      for (long e = lo / VN + threadIdx.x; e < hi / VN; e += blockDim.x) {
        const long off = e * VN;
        chain_deliver<T, OPTD>(a, en, off, ldv_cg(static_cast<const T*>(en.recv) + off), bad);
      }
    }
  }
  __syncthreads();
}

template <typename T, int OPTD>
__global__ void __launch_bounds__(kThreads) chain_mean_kernel(const ChainArgs<T> a) {
  __shared__ ChainEntry en;
  __shared__ int ok_flag;
  const long units = a.n_chunks * a.n_entries;
  unsigned long long bad = ~0ull;
  for (long u = blockIdx.x; u < units; u += gridDim.x) {
    chain_unit_b<T, OPTD>(a, a.entries, a.n_entries, u, en, ok_flag, bad);
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
}

// ---- fused two-shot (push) over NVLink ------------------------------------
// For groups with one member per GPU.  One persistent kernel per iteration:
//   phase 1  each GPU steps its member chunk by chunk and pushes the stepped
//            chunk straight into the slice owner's staging row (row = the
//            member's position j in the group), releasing a per-chunk flag;
//   phase 2  the owner of each slice waits for the S flags of a chunk, folds
//            rows 0..S-1 in ascending member order, scales, and stores the
//            mean into every member's params row (peer stores).
// The HBM step overlaps the NVLink push.  The grid is sized to be fully
// resident, so every CTA finishes its phase-1 items before any CTA can spin
// in phase 2 -- no CTA waits on work that cannot be scheduled.
struct PushItem {        // phase 1: one chunk of my member, stepped once, pushed to ndst stagings
  int lr;                // my member's local row
  long lo, hi;           // element range
  int dst_beg, ndst;     // destinations in the item tables: two-shot 1 (the slice owner), one-shot S
  int rank;              // member's global rank (error key)
};
struct PushFold {        // phase 2: one chunk of a slice this GPU owns
  long lo, hi;           // element range
  const void* stage;     // staging row 0 of the slice, positioned at lo
  long stage_ld;         // elements between staging rows (slice length)
  const unsigned long long* flags;  // flag of (row 0, this chunk); rows are flag_ld apart
  long flag_ld;
  int S;                 // rows (= members)
  int dst_beg;           // member param-row pointers in the dst table
  int n_dst;             // two-shot: S (every member, peer stores); one-shot: 1 (my member)
  int err_rank;          // members[0]
};

template <typename T> struct PushArgs {
  const PushItem* items;
  int n_items;
  void* const* item_dst;                     // staging row j of a destination, positioned at the item's lo
  unsigned long long* const* item_flag;      // its flag for (row j, chunk)
  const PushFold* folds;
  int n_folds;
  T* const* dst;         // member param rows (local or peer)
  T* w;
  const T* g;
  T* m1;
  T* m2;
  long ld;
  int first_rank;
  long t;
  unsigned long long epoch;
  unsigned long long* err;
  unsigned long long* timeout;
  long stage_shift;      // one-shot: bytes to this launch's staging buffer (double-buffered), else 0
  long flag_shift;       // one-shot: flags to this launch's flag set, else 0
  StepConsts<T> c;
  double bc1[kMaxLocal];
  double bc2[kMaxLocal];
};

// Two-shot (each slice owner folds and stores the mean to every member) or
// one-shot (every member GPU receives every member's stepped row and folds
// it for its own member; small rows: no remote stores into params, so the
// next iteration needs no barrier).  Same kernel, different tables.
template <typename T, int OPT>
__global__ void __launch_bounds__(kThreads) push_twoshot_kernel(const PushArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  __shared__ PushItem it;
  __shared__ PushFold fo;
  __shared__ int ok_flag;
  __shared__ T* sdst[kMaxFold];
  unsigned long long bad = ~0ull;
  // phase 1: step + push
  for (int u = blockIdx.x; u < a.n_items; u += gridDim.x) {
    if (threadIdx.x == 0) it = a.items[u];
    __syncthreads();
    if (threadIdx.x < it.ndst) {
      sdst[threadIdx.x] = reinterpret_cast<T*>(static_cast<char*>(a.item_dst[it.dst_beg + threadIdx.x]) + a.stage_shift);
    }
    __syncthreads();
    const long r = static_cast<long>(it.lr) * a.ld;
    const T b1 = static_cast<T>(a.bc1[it.lr]);
    const T b2 = static_cast<T>(a.bc2[it.lr]);
    for (long e = it.lo / VN + threadIdx.x; e < it.hi / VN; e += blockDim.x) {
      const long off = e * VN;
      Pack<T> x = ldv(a.w + r + off);
      const Pack<T> gv = ldv(a.g + r + off);
      Pack<T> s1, s2;
      if constexpr (OPT != kSgd) s1 = ldv(a.m1 + r + off);
      if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + r + off);
      bool ok = true;
#pragma unroll
      for (int l = 0; l < VN; ++l) {
        x.v[l] = step_elem<T, OPT>(x.v[l], gv.v[l], s1.v[l], s2.v[l], a.c, b1, b2);
        ok = ok && finite_(x.v[l]);
      }
      if constexpr (OPT != kSgd) stv(a.m1 + r + off, s1);
      if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r + off, s2);
      if (!ok) {
        const unsigned long long k = err_key(a.t, 0, it.rank);
        bad = k < bad ? k : bad;
      }
      for (int q = 0; q < it.ndst; ++q) stv_cg(sdst[q] + (off - it.lo), x);
    }
    __syncthreads();
    if (threadIdx.x < it.ndst) st_release_sys(a.item_flag[it.dst_beg + threadIdx.x] + a.flag_shift, a.epoch);
    __syncthreads();
  }
  // phase 2: ordered fold of owned chunks
  for (int u = blockIdx.x; u < a.n_folds; u += gridDim.x) {
    if (threadIdx.x == 0) {
      fo = a.folds[u];
      ok_flag = 1;
      for (int j = 0; j < fo.S && ok_flag; ++j) {
        ok_flag = chain_wait(fo.flags + a.flag_shift + j * fo.flag_ld, a.epoch, a.timeout);
      }
    }
    __syncthreads();
    if (ok_flag) {
      const T inv = static_cast<T>(1.0 / static_cast<double>(fo.S));
      const T* st = reinterpret_cast<const T*>(static_cast<const char*>(fo.stage) + a.stage_shift);
      for (long e = fo.lo / VN + threadIdx.x; e < fo.hi / VN; e += blockDim.x) {
        const long off = e * VN;
        const long so = off - fo.lo;
        Pack<T> acc = ldv_cg(st + so);
        for (int j = 1; j < fo.S; ++j) {
          const Pack<T> x = ldv_cg(st + j * fo.stage_ld + so);
#pragma unroll
          for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x.v[l]);
        }
        bool ok = true;
#pragma unroll
        for (int l = 0; l < VN; ++l) {
          acc.v[l] = mul_(acc.v[l], inv);
          ok = ok && finite_(acc.v[l]);
        }
        if (!ok) {
          const unsigned long long k = err_key(a.t, 1, fo.err_rank);
          bad = k < bad ? k : bad;
        }
        for (int q = 0; q < fo.n_dst; ++q) stv_cg(a.dst[fo.dst_beg + q] + off, acc);
      }
    }
    __syncthreads();
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
  __threadfence_system();
}

// ---- synthetic gradients: SplitMix64 + Box-Muller (rng.cpp:8-51) -----------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// i-th gaussian of the stream whose state after for_stream is s0: draws
// 2i and 2i+1 (0-based), draw j = mix64(s0 + (j+1) * phi) (rng.cpp:28-31).
__device__ __forceinline__ double gaussian_at(uint64_t s0, uint64_t i) {
  const uint64_t phi = 0x9e3779b97f4a7c15ULL;
  const uint64_t x = mix64(s0 + (2 * i + 1) * phi);
  const uint64_t y = mix64(s0 + (2 * i + 2) * phi);
  const double u1 = __dsub_rn(1.0, __dmul_rn(static_cast<double>(x >> 11), 0x1.0p-53));
  const double u2 = __dmul_rn(static_cast<double>(y >> 11), 0x1.0p-53);
  // sqrt(-2 log u1) * cos(2 pi u2), the argument rounded as (2.0*pi)*u2
  return __dmul_rn(__dsqrt_rn(__dmul_rn(-2.0, log(u1))),
                   cos(__dmul_rn(6.283185307179586232, u2)));
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
__global__ void gaussian_fill_kernel(double* out, long d, uint64_t s0) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d; i += stride) {
    out[i] = gaussian_at(s0, static_cast<uint64_t>(i));
  }
}

__global__ void sumsq_kernel(const double* x, long d, double* out) {
  __shared__ double part[kThreads / 32];
  double acc = 0.0;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d; i += stride) {
    acc += x[i] * x[i];
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += part[i];
    atomicAdd(out, s);
  }
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
    atomicMin(a.gerr, (static_cast<unsigned long long>(a.t) << 32) | static_cast<unsigned int>(a.first_rank + k));
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

}  // namespace dssb
