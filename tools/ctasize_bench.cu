// Diagnostic microbenchmark (not product code): does the CTA size / count of a
// single-wave copy kernel set its ramp on B200?  Copies `mb` MiB contiguously with
// every thread holding 8 x 16 B in flight; the same total resident threads
// (148 SMs x 1024) arranged as 592 x 256, 296 x 512 or 148 x 1024 CTAs.  Also times
// two dependent copies of half the size back to back on one stream against one copy
// of the full size (the per-kernel ramp + tail a decode step pays twice).
// Usage: ctasize_bench [mb=19] [warm(0/1)=1]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int T>
__global__ void __launch_bounds__(T) copyk(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * T;
  for (size_t base = (size_t)blockIdx.x * T + threadIdx.x; base < n; base += stride * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t i = base + u * stride;
      if (i < n)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t i = base + u * stride;
      if (i < n) dst[i] = v[u];
    }
  }
}

__global__ void flush(char *p, size_t n) {
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n;
       i += (size_t)gridDim.x * blockDim.x * 16)
    *reinterpret_cast<uint4 *>(p + i) = make_uint4(1, 2, 3, 4);
}

template <int T>
void launch(int grid, const uint4 *s, uint4 *d, size_t n, cudaStream_t st) {
  copyk<T><<<grid, T, 0, st>>>(s, d, n);
}

int main(int argc, char **argv) {
  const double mb = argc > 1 ? atof(argv[1]) : 19.0;
  const int warm = argc > 2 ? atoi(argv[2]) : 1;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = (size_t)(mb * (1 << 20)) & ~(size_t)15;
  const size_t n = bytes / 16;
  uint4 *src, *dst;
  char *fl;
  const size_t flb = 512ull << 20;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaMalloc(&fl, flb));
  CK(cudaMemset(src, 1, bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int reps = 200;
  struct Cfg { const char *name; int threads, grid; };
  const Cfg cfgs[] = {{"592x256", 256, sms * 4}, {"296x512", 512, sms * 2}, {"148x1024", 1024, sms},
                      {"296x256", 256, sms * 2}, {"1184x128", 128, sms * 8}};
  for (int pass = 0; pass < 2; ++pass) {  // pass 0 warms up everything
    for (const Cfg &c : cfgs) {
      for (int mode = 0; mode < 2; ++mode) {  // 0: one copy of `bytes`; 1: two dependent halves
        float tot = 0;
        for (int r = 0; r < reps; ++r) {
          if (!warm) flush<<<sms * 4, 256, 0, st>>>(fl, flb);
          else launch<256>(sms * 4, src, dst, n, st);  // data in L2 like a decode step
          CK(cudaEventRecord(a, st));
          auto go = [&](const uint4 *s, uint4 *d, size_t m) {
            if (c.threads == 128) launch<128>(c.grid, s, d, m, st);
            if (c.threads == 256) launch<256>(c.grid, s, d, m, st);
            if (c.threads == 512) launch<512>(c.grid, s, d, m, st);
            if (c.threads == 1024) launch<1024>(c.grid, s, d, m, st);
          };
          if (mode == 0) go(src, dst, n);
          else {
            go(src, dst, n / 2);
            go(src + n / 2, dst + n / 2, n - n / 2);
          }
          CK(cudaEventRecord(b, st));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          tot += ms;
        }
        CK(cudaGetLastError());
        if (pass == 1) {
          const double us = tot / reps * 1e3;
          printf("%-9s %s %.1f MiB %s: %7.2f us  %7.1f GB/s (r+w)\n", c.name,
                 mode ? "2 halves" : "1 copy  ", mb, warm ? "warm" : "cold", us,
                 2.0 * bytes / (us * 1e-6) / 1e9);
        }
      }
    }
  }
  return 0;
}
