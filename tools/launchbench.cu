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
  return 0;
}
