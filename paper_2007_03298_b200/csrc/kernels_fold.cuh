// Across GPUs over NVLink peer memory: the two-shot pull fold, the flag
// barrier, the ordered chain fold (partial and mean passes) and the fused
// push kernel (two-shot or one-shot).
#pragma once

#include "kernel_common.cuh"

namespace dssb {

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
static __global__ void barrier_kernel(unsigned long long* const* peer_flags, unsigned long long* my_flags,
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

// The waiting half of the split barrier on its own, for a step whose first
// launch cannot wait itself.
static __global__ void split_wait_kernel(const unsigned long long* my_flags, int n, unsigned long long epoch,
                                         unsigned long long* timeout) {
  split_wait(my_flags, n, epoch, timeout);
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
  int dst_skip;       // 1: the mean was received straight into dst[0] (in-place delivery)
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
  const int* rank_of;  // local row -> global rank (error keys)
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
  step_pack<T, OPT>(x, gv, s1, s2, a.c, b1, b2);
  bool ok = true;
#pragma unroll
  for (int l = 0; l < VN; ++l) ok = ok && finite_(x.v[l]);
  if constexpr (OPT != kSgd) stv(a.m1 + r, s1);
  if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2);
  if (!ok) {
    const unsigned long long k = err_key(a.t, phase, a.rank_of[lr]);
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
    step_pack<T, OPT>(x[q], gv[q], s1[q], s2[q], a.c, b1, b2);
    bool ok = true;
#pragma unroll
    for (int l = 0; l < VN; ++l) ok = ok && finite_(x[q].v[l]);
    if constexpr (OPT != kSgd) stv(a.m1 + r, s1[q]);
    if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2[q]);
    if (!ok) {
      const unsigned long long k = err_key(a.t, phase, a.rank_of[lr[q]]);
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
    for (int q = en.dst_skip; q < en.dst_cnt; ++q) stv(a.dst[en.dst_beg + q] + off, mean);
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

// ---- deferred chain mean pass fused into the next step's local groups -----
// After a two-GPU chain step the stage-0 GPU holds each group's mean in one
// member row (delivered in place by the last stage); instead of copying it to
// the group's other local members (kernel B), the next step -- whose groups
// are all local -- reads every member's params through alias[] from the row
// the mean landed in.  Unit = chain chunk: thread j waits for entry j's mean
// flag of the chunk, then every thread steps all NR local rows of its
// element vector (all loads before any store: aliased rows are read by
// other groups), folds each group of M in ascending order, scales by 1/M
// and stores the means.  Same arithmetic and order as ds_group_kernel.
template <typename T> struct LazyArgs {
  T* w;
  const T* g;
  T* m1;
  T* m2;
  long ld;
  long chunk, len, n_chunks;
  const unsigned long long* flags[4];
  int nf;
  unsigned long long epoch;
  unsigned long long* timeout;
  int alias[8];
  int rows[8];
  int rank[8];  // global rank of local row r
  long t;
  int step_phase, sync_phase;
  unsigned long long* err;
  StepConsts<T> c;
  double bc1[kMaxLocal];
  double bc2[kMaxLocal];
};

template <typename T, int OPT, int NR, int M>
__global__ void __launch_bounds__(kThreads) lazy_groups_kernel(const LazyArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  __shared__ int ok;
  unsigned long long bad = ~0ull;
  const T inv = static_cast<T>(1.0 / static_cast<double>(M));
  for (long ch = blockIdx.x; ch < a.n_chunks; ch += gridDim.x) {
    if (threadIdx.x == 0) ok = 1;
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < a.nf && !chain_wait(a.flags[threadIdx.x] + ch, a.epoch, a.timeout)) ok = 0;
    __syncthreads();
    const long lo = ch * a.chunk;
    const long hi = lo + a.chunk < a.len ? lo + a.chunk : a.len;
    if (ok) {
      for (long e = lo / VN + threadIdx.x; e < hi / VN; e += blockDim.x) {
        const long off = e * VN;
        Pack<T> x[NR], gv[NR], s1[NR], s2[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const long rr = static_cast<long>(a.rows[r]) * a.ld + off;
          x[r] = ldv(a.w + static_cast<long>(a.alias[a.rows[r]]) * a.ld + off);
          gv[r] = ldv(a.g + rr);
          if constexpr (OPT != kSgd) s1[r] = ldv(a.m1 + rr);
          if constexpr (OPT == kAdam || OPT == kAdamW) s2[r] = ldv(a.m2 + rr);
        }
#pragma unroll
        for (int g0 = 0; g0 < NR; g0 += M) {
          Pack<T> acc;
#pragma unroll
          for (int j = 0; j < M; ++j) {
            const int r = g0 + j;
            const int lr = a.rows[r];
            const long rr = static_cast<long>(lr) * a.ld + off;
            T b1 = T(1), b2 = T(1);
            if constexpr (OPT == kAdam || OPT == kAdamW) {
              b1 = static_cast<T>(a.bc1[lr]);
              b2 = static_cast<T>(a.bc2[lr]);
            }
            step_pack<T, OPT>(x[r], gv[r], s1[r], s2[r], a.c, b1, b2);
            bool okv = true;
#pragma unroll
            for (int l = 0; l < VN; ++l) okv = okv && finite_(x[r].v[l]);
            if constexpr (OPT != kSgd) stv(a.m1 + rr, s1[r]);
            if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + rr, s2[r]);
            if (!okv) {
              const unsigned long long k = err_key(a.t, a.step_phase, a.rank[lr]);
              bad = k < bad ? k : bad;
            }
            if (j == 0) {
              acc = x[r];
            } else {
#pragma unroll
              for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x[r].v[l]);
            }
          }
          if (M != 1) {
            bool okm = true;
#pragma unroll
            for (int l = 0; l < VN; ++l) {
              acc.v[l] = mul_(acc.v[l], inv);
              okm = okm && finite_(acc.v[l]);
            }
            if (!okm) {
              const unsigned long long k = err_key(a.t, a.sync_phase, a.rank[a.rows[g0]]);
              bad = k < bad ? k : bad;
            }
          }
#pragma unroll
          for (int j = 0; j < M; ++j) stv(a.w + static_cast<long>(a.rows[g0 + j]) * a.ld + off, acc);
        }
      }
    }
    __syncthreads();
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
  const int* dst_lr;     // BSP: local row of each dst (its optimizer state and bias corrections)
  T* w;
  const T* g;
  T* m1;
  T* m2;
  long ld;
  int first_rank;
  const int* rank_of;  // local row -> global rank (error keys)
  long t;
  unsigned long long epoch;
  unsigned long long* err;
  unsigned long long* timeout;
  long stage_shift;      // one-shot: bytes to this launch's staging buffer (rotated), else 0
  long flag_shift;       // one-shot: flags to this launch's flag set, else 0
  // one-shot flow control: this is one-shot launch `seq` (1, 2, ...) on
  // buffer (seq - 1) % B, B = DSS_ONESHOT_BUFFERS.  At the start every GPU
  // records seq in each peer's acks[me]; a push into GPU q's buffer waits
  // for acks[q] >= seq - B + 1, i.e. for q to have started launch
  // seq - B + 1 and so finished launch seq - B, the previous user of the
  // same buffer (consecutive launches may have other peers).
  unsigned long long seq; // 0: two-shot (no flow control)
  unsigned long long* const* ack_peer;  // [G] each GPU's ack array
  unsigned long long* ack_mine;         // [G] this GPU's ack array
  const int* item_gpu;                  // destination GPU of each item_dst entry
  int me, n_gpus;
  // split barrier.  wait_*: as GroupArgs (this launch is the first of its
  // step).  arrive_epoch != 0 (two-shot, no chain or fold after it): the last
  // CTA to finish stores arrive_epoch into every GPU's barrier word
  // (arrive_flags[j] + me), after every CTA's phase-2 stores; arrive_count
  // is a local CTA counter, zero between launches.
  const unsigned long long* wait_flags;
  unsigned long long wait_epoch;
  unsigned long long* const* arrive_flags;
  unsigned long long arrive_epoch;
  unsigned* arrive_count;
  StepConsts<T> c;
  double bc1[kMaxLocal];
  double bc2[kMaxLocal];
};

// Two-shot (each slice owner folds and stores the mean to every member) or
// one-shot (every member GPU receives every member's stepped row and folds
// it for its own member; small rows: no remote stores into params, so the
// next iteration needs no barrier).  Same kernel, different tables.
// BSP = true (one-shot over the world): phase 1 pushes the raw gradient
// rows, phase 2 folds all W of them in rank order and steps every local
// replica with the mean gradient (sync.cpp:389-421).
template <typename T, int OPT, bool BSP = false>
__global__ void __launch_bounds__(kThreads) push_twoshot_kernel(const PushArgs<T> a) {
  constexpr int VN = Vec<T>::n;
  __shared__ PushItem it;
  __shared__ PushFold fo;
  __shared__ T* sdst[kMaxFold];
  __shared__ unsigned long long sok;  // bit q: destination q may be written (its flow-control wait succeeded)
  unsigned long long bad = ~0ull;
  split_wait(a.wait_flags, a.n_gpus, a.wait_epoch, a.timeout);
  if (a.seq && blockIdx.x == 0 && threadIdx.x < a.n_gpus) {
    // "I have started launch seq".  The reads this releases (the folds of
    // an earlier launch) finished at a kernel boundary, so a relaxed store
    // suffices: a peer that sees it can only write after those reads.
    if (DSS_ONESHOT_ACK_RELAXED) {
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(a.ack_peer[threadIdx.x] + a.me), "l"(a.seq) : "memory");
    } else {
      st_release_sys(a.ack_peer[threadIdx.x] + a.me, a.seq);
    }
  }
  // phase 1: step + push
  for (int u = blockIdx.x; u < a.n_items; u += gridDim.x) {
    if (threadIdx.x == 0) {
      it = a.items[u];
      sok = ~0ull;
    }
    __syncthreads();
    if (threadIdx.x < it.ndst) {
      sdst[threadIdx.x] = reinterpret_cast<T*>(static_cast<char*>(a.item_dst[it.dst_beg + threadIdx.x]) + a.stage_shift);
      // the destination must be done with this buffer's previous launch; on
      // a timeout (latched) nothing is pushed into a buffer it may still read
      if (a.seq >= DSS_ONESHOT_BUFFERS &&
          !chain_wait(a.ack_mine + a.item_gpu[it.dst_beg + threadIdx.x], a.seq - DSS_ONESHOT_BUFFERS + 1, a.timeout)) {
        atomicAnd(&sok, ~(1ull << threadIdx.x));
      }
    }
    __syncthreads();
    const unsigned long long dst_ok = sok;
    const long r = static_cast<long>(it.lr) * a.ld;
    const T b1 = static_cast<T>(a.bc1[it.lr]);
    const T b2 = static_cast<T>(a.bc2[it.lr]);
    for (long e = it.lo / VN + threadIdx.x; e < it.hi / VN; e += blockDim.x) {
      const long off = e * VN;
      if constexpr (BSP) {
        const Pack<T> gv = ldv(a.g + r + off);
        for (int q = 0; q < it.ndst; ++q) {
          if ((dst_ok >> q) & 1) stv_cg(sdst[q] + (off - it.lo), gv);
        }
        continue;
      }
      Pack<T> x = ldv(a.w + r + off);
      const Pack<T> gv = ldv(a.g + r + off);
      Pack<T> s1, s2;
      if constexpr (OPT != kSgd) s1 = ldv(a.m1 + r + off);
      if constexpr (OPT == kAdam || OPT == kAdamW) s2 = ldv(a.m2 + r + off);
      step_pack<T, OPT>(x, gv, s1, s2, a.c, b1, b2);
      bool ok = true;
#pragma unroll
      for (int l = 0; l < VN; ++l) ok = ok && finite_(x.v[l]);
      if constexpr (OPT != kSgd) stv(a.m1 + r + off, s1);
      if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r + off, s2);
      if (!ok) {
        const unsigned long long k = err_key(a.t, 0, it.rank);
        bad = k < bad ? k : bad;
      }
      for (int q = 0; q < it.ndst; ++q) {
        if ((dst_ok >> q) & 1) stv_cg(sdst[q] + (off - it.lo), x);
      }
    }
    __syncthreads();
    if (threadIdx.x < it.ndst && ((dst_ok >> threadIdx.x) & 1)) {
      st_release_sys(a.item_flag[it.dst_beg + threadIdx.x] + a.flag_shift, a.epoch);
    }
    __syncthreads();
  }
  // phase 2: ordered fold of owned chunks
  for (int u = blockIdx.x; u < a.n_folds; u += gridDim.x) {
    if (threadIdx.x == 0) fo = a.folds[u];
    __syncthreads();
    // the S row flags are polled in parallel (thread j: row j); a serial
    // poll costs one system-scope load latency per row
    int okj = 1;
    for (int j = threadIdx.x; j < fo.S; j += blockDim.x) {
      okj &= chain_wait(fo.flags + a.flag_shift + j * fo.flag_ld, a.epoch, a.timeout) ? 1 : 0;
    }
    if (__syncthreads_and(okj)) {
      const T inv = static_cast<T>(1.0 / static_cast<double>(fo.S));
      const T* st = reinterpret_cast<const T*>(static_cast<const char*>(fo.stage) + a.stage_shift);
      for (long e = fo.lo / VN + threadIdx.x; e < fo.hi / VN; e += blockDim.x) {
        const long off = e * VN;
        const long so = off - fo.lo;
        Pack<T> acc = ldv_cg(st + so);
        // rows in load batches of 4, added in ascending order
        int j = 1;
        for (; j + 4 <= fo.S; j += 4) {
          Pack<T> x[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) x[b] = ldv_cg(st + (j + b) * fo.stage_ld + so);
#pragma unroll
          for (int b = 0; b < 4; ++b) {
#pragma unroll
            for (int l = 0; l < VN; ++l) acc.v[l] = add_(acc.v[l], x[b].v[l]);
          }
        }
        for (; j < fo.S; ++j) {
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
        if (!ok) {  // collective failure: members[0] (DS phase 1, BSP phase 0)
          const unsigned long long k = err_key(a.t, BSP ? 0 : 1, fo.err_rank);
          bad = k < bad ? k : bad;
        }
        if constexpr (BSP) {
          // every local replica steps with the mean gradient, replicas in
          // load batches of 4 (all loads of a batch before its stores)
          for (int q0 = 0; q0 < fo.n_dst; q0 += 4) {
            const int nb = fo.n_dst - q0 < 4 ? fo.n_dst - q0 : 4;
            Pack<T> x[4], s1[4], s2[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (b < nb) {
                const long r = static_cast<long>(a.dst_lr[fo.dst_beg + q0 + b]) * a.ld + off;
                x[b] = ldv(a.w + r);
                if constexpr (OPT != kSgd) s1[b] = ldv(a.m1 + r);
                if constexpr (OPT == kAdam || OPT == kAdamW) s2[b] = ldv(a.m2 + r);
              }
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (b < nb) {
                const int lr = a.dst_lr[fo.dst_beg + q0 + b];
                const long r = static_cast<long>(lr) * a.ld + off;
                const T b1 = static_cast<T>(a.bc1[lr]);
                const T b2 = static_cast<T>(a.bc2[lr]);
                step_pack<T, OPT>(x[b], acc, s1[b], s2[b], a.c, b1, b2);
                bool oks = true;
#pragma unroll
                for (int l = 0; l < VN; ++l) oks = oks && finite_(x[b].v[l]);
                stv(a.w + r, x[b]);
                if constexpr (OPT != kSgd) stv(a.m1 + r, s1[b]);
                if constexpr (OPT == kAdam || OPT == kAdamW) stv(a.m2 + r, s2[b]);
                if (!oks) {
                  const unsigned long long k = err_key(a.t, 1, a.rank_of[lr]);
                  bad = k < bad ? k : bad;
                }
              }
            }
          }
        } else {
          for (int q = 0; q < fo.n_dst; ++q) stv_cg(a.dst[fo.dst_beg + q] + off, acc);
        }
      }
    }
    __syncthreads();
  }
  if (__any_sync(__activemask(), bad != ~0ull)) latch_error(a.err, bad);
  __threadfence_system();
  if (a.arrive_epoch) {
    // arriving half of the split barrier: every CTA's stores (fenced above)
    // precede its count; the last CTA releases the epoch to every GPU
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(a.arrive_count, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      if (static_cast<int>(threadIdx.x) < a.n_gpus) {
        __threadfence_system();
        st_release_sys(a.arrive_flags[threadIdx.x] + a.me, a.arrive_epoch);
      }
      if (threadIdx.x == 0) atomicExch(a.arrive_count, 0u);
    }
  }
}

}  // namespace dssb
