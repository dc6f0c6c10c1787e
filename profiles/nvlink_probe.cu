// NVLink probe: bandwidth of SM-issued 16-B peer loads / stores between
// GPUs of one box (one process, peer access enabled), to size the two-shot
// fold's design.  Modes, each run concurrently on every GPU g with peer
// (g+1) % n (or all peers for "all"):
//   read      g loads from peer, stores locally
//   write     g loads locally, stores to peer
//   mixed     g loads from peer AND stores to peer (fold-like push)
//   readall   g loads equal slices from every peer (fold-like gather)
//   writeall  g stores equal slices to every peer (fold-like broadcast)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/nvlink_probe profiles/nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                     \
    }                                                                                   \
  } while (0)

__global__ void copy_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long n) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    dst[i] = __ldcg(src + i);
  }
}

// dst_k[i] = src_k[i] for k peers (one launch), i over n/k elements each
struct Multi {
  const float4* src[8];
  float4* dst[8];
  int k;
  long n;  // per pair
};
__global__ void multi_kernel(Multi m) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m.n; i += stride) {
#pragma unroll 8
    for (int q = 0; q < m.k; ++q) m.dst[q][i] = __ldcg(m.src[q] + i);
  }
}

// Two-shot fold shapes: GPU g owns slice g of n rows (one per GPU); it
// folds the slice over all rows (n-1 remote) and stores the result to all.
struct Fold {
  const float4* src[8];
  float4* dst[8];
  int k;
  long lo, hi;  // vector range of the owned slice
};
template <int U>
__global__ void fold_kernel(Fold f) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x * U;
  for (long i = f.lo + (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) * U; i < f.hi; i += stride) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = __ldcg(f.src[0] + i + u);
    for (int q = 1; q < f.k; ++q) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float4 x = __ldcg(f.src[q] + i + u);
        acc[u].x += x.x; acc[u].y += x.y; acc[u].z += x.z; acc[u].w += x.w;
      }
    }
    for (int q = 0; q < f.k; ++q) {
#pragma unroll
      for (int u = 0; u < U; ++u) __stcg(f.dst[q] + i + u, acc[u]);
    }
  }
}
// fold with all loads issued before any add (k <= 8 fixed at 4 here)
__global__ void fold4_kernel(Fold f) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = f.lo + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < f.hi; i += stride) {
    float4 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = __ldcg(f.src[q] + i);
    float4 acc = x[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) { acc.x += x[q].x; acc.y += x[q].y; acc.z += x[q].z; acc.w += x[q].w; }
#pragma unroll
    for (int q = 0; q < 4; ++q) __stcg(f.dst[q] + i, acc);
  }
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  const long bytes = (argc > 1 ? std::atol(argv[1]) : 256L) << 20;  // per buffer
  const long nv = bytes / 16;
  std::printf("gpus=%d buffer=%ld MiB\n", n, bytes >> 20);
  std::vector<float4*> a(n), b(n), c(n);
  std::vector<cudaStream_t> st(n);
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < n; ++p) {
      if (p != g) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, g, p));
        if (ok) CK(cudaDeviceEnablePeerAccess(p, 0));
      }
    }
    CK(cudaMalloc(&a[g], bytes));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMalloc(&c[g], bytes));
    CK(cudaMemset(a[g], 1, bytes));
    CK(cudaMemset(b[g], 0, bytes));
    CK(cudaStreamCreate(&st[g]));
  }
  const char* modes[] = {"local", "read", "write", "mixed", "readall", "writeall", "fold1", "fold2", "fold4", "foldall4"};
  for (const char* mode : modes) {
    for (int blocks_per_sm : {4, 8, 16}) {
      std::vector<cudaEvent_t> e0(n), e1(n);
      for (int rep = 0; rep < 6; ++rep) {
        for (int g = 0; g < n; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < n; ++g) {
          CK(cudaSetDevice(g));
          if (rep == 5) {
            CK(cudaEventCreate(&e0[g]));
            CK(cudaEventCreate(&e1[g]));
            CK(cudaEventRecord(e0[g], st[g]));
          }
          const int peer = (g + 1) % n;
          const int grid = 148 * blocks_per_sm;
          if (!std::strcmp(mode, "local")) {
            copy_kernel<<<grid, 256, 0, st[g]>>>(a[g], b[g], nv);
          } else if (!std::strcmp(mode, "read")) {
            copy_kernel<<<grid, 256, 0, st[g]>>>(a[peer], b[g], nv);
          } else if (!std::strcmp(mode, "write")) {
            copy_kernel<<<grid, 256, 0, st[g]>>>(a[g], c[peer], nv);
          } else if (!std::strcmp(mode, "mixed")) {
            Multi m{};
            m.k = 2;
            m.n = nv / 2;
            m.src[0] = a[peer];
            m.dst[0] = b[g];
            m.src[1] = a[g];
            m.dst[1] = c[peer];
            multi_kernel<<<grid, 256, 0, st[g]>>>(m);
          } else if (!std::strncmp(mode, "fold", 4)) {
            Fold f{};
            f.k = n;
            for (int p = 0; p < n; ++p) {
              f.src[p] = a[p];
              f.dst[p] = b[p];
            }
            f.lo = nv / n * g;
            f.hi = f.lo + nv / n;
            if (!std::strcmp(mode, "fold1")) fold_kernel<1><<<grid, 256, 0, st[g]>>>(f);
            else if (!std::strcmp(mode, "fold2")) fold_kernel<2><<<grid, 256, 0, st[g]>>>(f);
            else if (!std::strcmp(mode, "fold4")) fold_kernel<4><<<grid, 256, 0, st[g]>>>(f);
            else if (n == 4) fold4_kernel<<<grid, 256, 0, st[g]>>>(f);
          } else {
            Multi m{};
            m.k = 0;
            for (int p = 0; p < n; ++p) {
              if (p == g) continue;
              const long off = static_cast<long>(m.k) * (nv / (n - 1));
              if (!std::strcmp(mode, "readall")) {
                m.src[m.k] = a[p] + off;
                m.dst[m.k] = b[g] + off;
              } else {
                m.src[m.k] = a[g] + off;
                m.dst[m.k] = c[p] + off + static_cast<long>(g) * 0;
              }
              ++m.k;
            }
            m.n = nv / (n - 1);
            multi_kernel<<<grid, 256, 0, st[g]>>>(m);
          }
          CK(cudaGetLastError());
          if (rep == 5) CK(cudaEventRecord(e1[g], st[g]));
        }
      }
      double worst = 0;
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      // Every GPU runs the same pattern against its neighbour(s), so each
      // GPU's inbound AND outbound NVLink direction carries `bytes` per
      // launch in every non-local mode (mixed: half reads, half writes each
      // way).  local reports the HBM copy (read + write).
      double gbs = bytes / (worst / 1e3) / 1e9;
      if (!std::strncmp(mode, "fold", 4)) gbs = gbs * (n - 1) / n;  // remote bytes each way per GPU
      std::printf("%-9s blocks/SM=%2d  %8.3f ms  %7.1f GB/s%s\n", mode, blocks_per_sm, worst,
                  !std::strcmp(mode, "local") ? 2 * gbs : gbs,
                  !std::strcmp(mode, "local") ? " (HBM r+w)" : " per direction, both directions loaded");
    }
  }
  return 0;
}
