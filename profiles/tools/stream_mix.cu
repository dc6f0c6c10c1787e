// HBM stream-mix probe: R read rows and Wr write rows per element vector,
// the access pattern of the fused group kernels without their arithmetic
// (grid-stride over 16-B vectors, streaming ld/st.global.cs, 256-thread
// CTAs, 148 x 8 CTAs).  Answers whether a kernel's bandwidth is capped by
// its DRAM stream mix rather than by its instruction stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mix stream_mix.cu
//   ./stream_mix <elements per row> <R> <Wr> [ctas per SM] [threads]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int R, int WR>
__global__ void mix_kernel(const float4* __restrict__ in, float4* __restrict__ out, long nvec, long ld) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < nvec; e += stride) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldcs(in + r * ld + e);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w;
    }
#pragma unroll
    for (int w = 0; w < WR; ++w) __stcs(out + w * ld + e, acc);
  }
}

template <int R, int WR>
float run(long n, int cps, int threads) {
  const long nvec = n / 4;
  float4 *in, *out;
  if (cudaMalloc(&in, sizeof(float4) * nvec * R) || cudaMalloc(&out, sizeof(float4) * nvec * WR)) return -1;
  cudaMemset(in, 0, sizeof(float4) * nvec * R);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * cps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) mix_kernel<R, WR><<<grid, threads>>>(in, out, nvec, nvec);
  cudaEventRecord(a);
  const int K = 10;
  for (int i = 0; i < K; ++i) mix_kernel<R, WR><<<grid, threads>>>(in, out, nvec, nvec);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(in);
  cudaFree(out);
  return static_cast<float>(16.0 * nvec * (R + WR) * K / (ms / 1e3) / 1e9);
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 100000000L;
  const int cps = argc > 2 ? atoi(argv[2]) : 8;
  const int threads = argc > 3 ? atoi(argv[3]) : 256;
  printf("{\"elements_per_row\": %ld, \"ctas_per_sm\": %d, \"threads\": %d, \"gbs\": {", n, cps, threads);
  printf("\"r1w1\": %.1f, ", run<1, 1>(n, cps, threads));
  printf("\"r2w1\": %.1f, ", run<2, 1>(n, cps, threads));
  printf("\"r4w2\": %.1f, ", run<4, 2>(n, cps, threads));
  printf("\"r8w4\": %.1f, ", run<8, 4>(n, cps, threads));
  printf("\"r16w8\": %.1f, ", run<16, 8>(n, cps, threads));
  printf("\"r12w8\": %.1f, ", run<12, 8>(n, cps, threads));
  printf("\"r16w12\": %.1f, ", run<16, 12>(n, cps, threads));
  printf("\"r32w24\": %.1f}}\n", run<32, 24>(n, cps, threads));
  return 0;
}
