// Diagnostic microbenchmark (not product code): host cost of one kernel launch
// vs the size of its parameter block (__grid_constant__ struct), B200 + this
// driver.  Empty kernels, 592 x 256, launched 2000 times back to back; reports
// host microseconds per launch call.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct Blob { char b[N]; };

template <int N>
__global__ void k(const __grid_constant__ Blob<N> p) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[N - 1] == 123) printf("x");
}

__global__ void spin(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) break;
  }
}

// GPU-side rate: the launches are queued behind a 30 ms spin kernel, so the device
// drains a full queue; events around the queued launches time the device only.
template <int N>
void run_gpu(cudaStream_t s) {
  Blob<N> p{};
  const int iters = 500;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  spin<<<1, 1, 0, s>>>(30000000ll);
  cudaEventRecord(a, s);
  for (int i = 0; i < iters; ++i) {
    p.b[0] = (char)i;
    k<N><<<592, 256, 0, s>>>(p);
  }
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("params %6d B: device %.2f us/launch (queued)\n", N, ms * 1e3 / iters);
}

template <int N>
void run(cudaStream_t s) {
  Blob<N> p{};
  for (int i = 0; i < 100; ++i) k<N><<<592, 256, 0, s>>>(p);
  cudaStreamSynchronize(s);
  const int iters = 2000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) {
    p.b[0] = (char)i;
    k<N><<<592, 256, 0, s>>>(p);
  }
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  printf("params %6d B: host %.2f us/launch, gpu-drained %.2f us/launch\n", N,
         std::chrono::duration<double>(t1 - t0).count() * 1e6 / iters,
         std::chrono::duration<double>(t2 - t0).count() * 1e6 / iters);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  run<256>(s); run<1024>(s); run<4096>(s); run<8192>(s); run<16384>(s); run<28672>(s); run<32000>(s);
  run_gpu<256>(s); run_gpu<4096>(s); run_gpu<8192>(s); run_gpu<16384>(s); run_gpu<28672>(s);
  return 0;
}
