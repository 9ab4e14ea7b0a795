// Copy-pattern microbenchmark (B200): which per-warp access order lets a plain
// 16-B LDG/STG copy of a large contiguous region reach the HBM roof?  Trivial address
// math, 256-thread CTAs, 4 CTAs/SM, 8 loads in flight per thread; 4 GiB copied.
//   A  "cta-interleaved": a CTA round covers 32 KiB; iteration u of warp w reads
//      [round + u*4 KiB + w*512, +512)       (round-1 kernel's task order)
//   B  "warp-contiguous": iteration u of warp w reads [round + w*4 KiB + u*512, +512)
//   C  like B with 2 KiB per warp round (4 loads in flight)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/copy_pattern tools/copy_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(void *p, const uint4 &v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int MODE, int U>
__global__ void __launch_bounds__(256, 4) copyk(const char *__restrict__ src, char *__restrict__ dst,
                                                 long long bytes) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long round_bytes = 256LL * 16 * U;   // per CTA per round
  for (long long base = blockIdx.x * round_bytes; base < bytes; base += gridDim.x * round_bytes) {
    uint4 v[U];
    long long off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0)
        off[u] = base + (long long)u * 4096 + w * 512 + lane * 16;
      else
        off[u] = base + (long long)w * (512 * U) + u * 512 + lane * 16;
      v[u] = ldg(src + off[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) stg(dst + off[u], v[u]);
  }
}

int main() {
  const long long bytes = 4LL << 30;
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto kern) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      kern<<<sms * 4, 256>>>(a, b, bytes);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    printf("%-34s %8.3f ms  %7.1f GB/s r+w\n", name, best, 2.0 * bytes / (best * 1e-3) / 1e9);
  };
  run("A cta-interleaved U=8", copyk<0, 8>);
  run("B warp-contiguous U=8", copyk<1, 8>);
  run("C warp-contiguous U=4", copyk<1, 4>);
  run("A cta-interleaved U=4", copyk<0, 4>);
  cudaMemcpy(b, a, 16, cudaMemcpyDeviceToDevice);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
