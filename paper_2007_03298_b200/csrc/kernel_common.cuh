// Shared pieces of the sm_100a kernels: tuning knobs, exact scalar ops,
// 16-byte vectors, the optimizer step of one element (optim.cpp:46-98),
// the divergence latch and the reference's SplitMix64 / Box-Muller stream.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dssb {

constexpr int kThreads = 256;
#ifndef DSS_MAX_LOCAL
#define DSS_MAX_LOCAL 128
#endif
constexpr int kMaxLocal = DSS_MAX_LOCAL;  // local workers per GPU carried in kernel params

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
#ifndef DSS_MIN_BLOCKS_M8_ADAM
#define DSS_MIN_BLOCKS_M8_ADAM DSS_MIN_BLOCKS
#endif
// Single-GPU worlds of at most this many bytes per state array run a whole
// dss_steps batch in one launch (a resident grid with a barrier between
// iterations above 32 KB) instead of one launch per iteration.  Measured
// against per-iteration launches: +40-100% for 4 workers at 16 KB-1 MB
// total, +10-20% for 16 workers, a loss at 4 MB.
// One-CTA batches (<= 32 KB per array) with more element vectors than
// kThreads run with kSmallWide threads: more member rows in flight.
#ifndef DSS_SMALL_WIDE
#define DSS_SMALL_WIDE 1
#endif
constexpr int kSmallWide = 512;

#ifndef DSS_PERSIST_MAX_BYTES
#define DSS_PERSIST_MAX_BYTES (1L << 20)
#endif
#ifndef DSS_PERSIST_MAX_BYTES_BSP
#define DSS_PERSIST_MAX_BYTES_BSP (4L << 20)
#endif
#ifndef DSS_PERSIST_MAX_WORKERS_DS
#define DSS_PERSIST_MAX_WORKERS_DS 16
#endif
#ifndef DSS_PERSIST_MAX_WORKERS_BSP
#define DSS_PERSIST_MAX_WORKERS_BSP 16
#endif
// 1: the chain's mean is sent straight into the receiving GPU's first
// member row (DS steps and sync rounds), not into a receive row.
#ifndef DSS_CHAIN_INPLACE
#define DSS_CHAIN_INPLACE 1
#endif
// One-shot staging buffers in rotation: a push into a peer waits until the
// peer has started the launch DSS_ONESHOT_BUFFERS - 1 back, i.e. finished
// the last launch that used the same buffer.
#ifndef DSS_ONESHOT_BUFFERS
#define DSS_ONESHOT_BUFFERS 3
#endif
#ifndef DSS_ONESHOT_ACK_RELAXED
#define DSS_ONESHOT_ACK_RELAXED 1
#endif
// Chain fold pipelining: elements per chunk (one flag each) and resident
// CTAs per SM.  Small chunks and ~one round of CTAs per GPU let stage j+1
// start one round after stage j instead of after the whole row.
#ifndef DSS_CHAIN_CHUNK
#define DSS_CHAIN_CHUNK 8192
#endif
#ifndef DSS_CHAIN_CHUNK_DS
#define DSS_CHAIN_CHUNK_DS 16384
#endif
#ifndef DSS_CHAIN_CHUNK_DS_MIN_BYTES
#define DSS_CHAIN_CHUNK_DS_MIN_BYTES (80L << 20)
#endif
// rows shorter than DSS_CHAIN_MIN_CHUNKS chunks use shorter chunks, down to
// DSS_CHAIN_CHUNK_MIN elements (0: off)
#ifndef DSS_CHAIN_MIN_CHUNKS
#define DSS_CHAIN_MIN_CHUNKS 64
#endif
#ifndef DSS_CHAIN_CHUNK_MIN
#define DSS_CHAIN_CHUNK_MIN 1024
#endif
// BSP folds all of a GPU's rows in every chain unit: more, shorter chunks
// Packed BSP across GPUs by the pull two-shot (every GPU folds its slice of
// all W rows, peer loads) instead of the ordered chain: always (A/B knob),
// or for rows of at most DSS_BSP_PULL_MAX_BYTES with at most
// DSS_BSP_PULL_MAX_P replicas per GPU
#ifndef DSS_BSP_PULL
#define DSS_BSP_PULL 0
#endif
#ifndef DSS_DS_CHAIN_NO_BARRIER
#define DSS_DS_CHAIN_NO_BARRIER 1
#endif
#ifndef DSS_BSP_CHAIN_NO_BARRIER
#define DSS_BSP_CHAIN_NO_BARRIER 1
#endif
#ifndef DSS_BSP_PULL_MAX_P
#define DSS_BSP_PULL_MAX_P 4
#endif
#ifndef DSS_BSP_PULL_MAX_BYTES
#define DSS_BSP_PULL_MAX_BYTES (4L << 20)
#endif
#ifndef DSS_BSP_CHAIN_MIN_CHUNKS
#define DSS_BSP_CHAIN_MIN_CHUNKS 1184  // 148 SMs x 8 resident chain CTAs
#endif
// (Also measured and dropped: stepping the replicas in kernel B, 2 / 4 / 8
// replicas per entry, instead of on the CTA that folded the chunk -- equal
// or slower at 4 GPUs, W = 16 / 64, 16 KB - 64 MB rows;
// profiles/r02/sweeps/bsp_chain_ab_g4.md.)
#ifndef DSS_BSP_CHAIN_CHUNK_MIN
#define DSS_BSP_CHAIN_CHUNK_MIN DSS_CHAIN_CHUNK_MIN
#endif
// BSP over several GPUs gathers all W gradient rows (one-shot) for small
// rows up to this world size, or while W rows total at most
// DSS_BSP_ONESHOT_MAX_TOTAL bytes
#ifndef DSS_BSP_ONESHOT_MAX_W
#define DSS_BSP_ONESHOT_MAX_W 16
#endif
#ifndef DSS_BSP_ONESHOT_MAX_TOTAL
#define DSS_BSP_ONESHOT_MAX_TOTAL (1L << 20)
#endif
#ifndef DSS_BSP_ONESHOT_SMALL_W_TOTAL
#define DSS_BSP_ONESHOT_SMALL_W_TOTAL (4L << 20)  // worlds of up to 4
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

// apply_step over one 16-B vector of one worker (optim.cpp:56-91 per
// element).  A branch-free fp32 Adam sequence (the intrinsics' fast paths
// spelled out, one range flag per vector, exact fallback) was built, proven
// bit-identical on the device and measured slower: C4-slice DS 6030 vs 6123
// GB/s, BSP 5305 vs 5617 (profiles/r02/adamw_ab.jsonl).
template <typename T, int OPT>
__device__ __forceinline__ void step_pack(Pack<T>& x, const Pack<T>& g, Pack<T>& m1, Pack<T>& m2,
                                          const StepConsts<T>& c, T bc1, T bc2) {
  constexpr int VN = Vec<T>::n;
#pragma unroll
  for (int l = 0; l < VN; ++l) x.v[l] = step_elem<T, OPT>(x.v[l], g.v[l], m1.v[l], m2.v[l], c, bc1, bc2);
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

// ---- split cross-GPU barrier: the waiting half -----------------------------
// A two-shot push kernel ends by storing its epoch into every GPU's barrier
// flag word (the arriving half, see push_twoshot_kernel); the first kernel of
// the next step waits here, every CTA before touching any row, instead of a
// separate barrier launch.  Thread j polls GPU j's word (bounded, ~20 s of
// globaltimer, then the timeout is latched as in barrier_kernel).
__device__ __forceinline__ void split_wait(const unsigned long long* flags, int n, unsigned long long epoch,
                                           unsigned long long* timeout) {
  if (!flags) return;
  if (static_cast<int>(threadIdx.x) < n) {
    unsigned long long start, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + threadIdx.x) : "memory");
      if (v >= epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - start > 20000000000ull) {
        atomicExch(timeout, 1ull);
        break;
      }
    }
  }
  __syncthreads();
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

}  // namespace dssb
