// How fast can 592 CTAs pull a ~10 KiB descriptor out of the kernel parameter space
// into shared memory, and what does the host pay for the launch?  (B200)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/param_probe tools/param_probe.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

template <int N>
struct Blob {
  uint4 w[N];
};

// (a) warp-uniform: warp w copies words w, w+8, ...; lane 0 stores
template <int N>
__global__ void __launch_bounds__(256) uni(const __grid_constant__ Blob<N> b, unsigned *out) {
  __shared__ uint4 sm[N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = w; k < N; k += 8) {
    uint4 x = b.w[k];
    if (lane == 0) sm[k] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, sm[N - 1].x);
}
// (b) divergent: thread t copies words t, t+256, ...
template <int N>
__global__ void __launch_bounds__(256) div(const __grid_constant__ Blob<N> b, unsigned *out) {
  __shared__ uint4 sm[N];
  for (int k = threadIdx.x; k < N; k += 256) sm[k] = b.w[k];
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, sm[N - 1].x);
}
// (c) global copy (reference)
template <int N>
__global__ void __launch_bounds__(256) glob(const uint4 *__restrict__ b, unsigned *out) {
  __shared__ uint4 sm[N];
  for (int k = threadIdx.x; k < N; k += 256) sm[k] = b[k];
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, sm[N - 1].x);
}

template <int N>
void run(const char *tag) {
  static Blob<N> hb;
  memset(&hb, 1, sizeof hb);
  unsigned *out;
  cudaMalloc(&out, 4);
  uint4 *g;
  cudaMalloc(&g, sizeof hb);
  cudaMemcpy(g, &hb, sizeof hb, cudaMemcpyHostToDevice);
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  for (int mode = 0; mode < 3; ++mode) {
    // back-to-back launches: device time per launch and host time per launch call
    const int reps = 200;
    cudaDeviceSynchronize();
    auto h0 = std::chrono::steady_clock::now();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) uni<N><<<592, 256>>>(hb, out);
      else if (mode == 1) div<N><<<592, 256>>>(hb, out);
      else glob<N><<<592, 256>>>(g, out);
    }
    cudaEventRecord(e);
    auto h1 = std::chrono::steady_clock::now();
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, a, e);
    double host_us = std::chrono::duration<double, std::micro>(h1 - h0).count() / reps;
    printf("%s %-8s %6d B: device %7.2f us/launch, host %6.2f us/launch call\n", tag,
           mode == 0 ? "uniform" : mode == 1 ? "diverg" : "global", (int)sizeof hb,
           ms * 1e3 / reps, host_us);
  }
  // host cost of a 10 KiB pinned H2D on a second stream
  char *hp;
  cudaHostAlloc((void **)&hp, sizeof hb, 0);
  cudaStream_t s2;
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  auto h0 = std::chrono::steady_clock::now();
  for (int r = 0; r < 200; ++r) cudaMemcpyAsync(g, hp, sizeof hb, cudaMemcpyHostToDevice, s2);
  auto h1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s2);
  printf("%s cudaMemcpyAsync H2D %d B: host %6.2f us/call\n", tag, (int)sizeof hb,
         std::chrono::duration<double, std::micro>(h1 - h0).count() / 200);
  // interleaved with kernel launches on the default stream (the decode loop's pattern)
  cudaDeviceSynchronize();
  h0 = std::chrono::steady_clock::now();
  double tm = 0, tk = 0;
  for (int r = 0; r < 200; ++r) {
    auto x0 = std::chrono::steady_clock::now();
    cudaMemcpyAsync(g, hp, sizeof hb, cudaMemcpyHostToDevice, s2);
    auto x1 = std::chrono::steady_clock::now();
    glob<N><<<592, 256>>>(g, out);
    auto x2 = std::chrono::steady_clock::now();
    tm += std::chrono::duration<double, std::micro>(x1 - x0).count();
    tk += std::chrono::duration<double, std::micro>(x2 - x1).count();
  }
  h1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  printf("%s interleaved: memcpy %6.2f us/call, launch %6.2f us/call, total %6.2f us/pair\n", tag,
         tm / 200, tk / 200, std::chrono::duration<double, std::micro>(h1 - h0).count() / 200);
  // same with a second pinned buffer per iteration (ring of 16 slots of 8 MiB)
  char *ring[16];
  for (int i = 0; i < 16; ++i) cudaHostAlloc((void **)&ring[i], 8 << 20, 0);
  char *gr[16];
  for (int i = 0; i < 16; ++i) cudaMalloc(&gr[i], 8 << 20);
  cudaDeviceSynchronize();
  tm = tk = 0;
  for (int r = 0; r < 200; ++r) {
    auto x0 = std::chrono::steady_clock::now();
    cudaMemcpyAsync(gr[r % 16], ring[r % 16], sizeof hb, cudaMemcpyHostToDevice, s2);
    auto x1 = std::chrono::steady_clock::now();
    glob<N><<<592, 256>>>((const uint4 *)gr[r % 16], out);
    auto x2 = std::chrono::steady_clock::now();
    tm += std::chrono::duration<double, std::micro>(x1 - x0).count();
    tk += std::chrono::duration<double, std::micro>(x2 - x1).count();
  }
  cudaDeviceSynchronize();
  printf("%s ring-16 x 8MiB: memcpy %6.2f us/call, launch %6.2f us/call\n", tag, tm / 200, tk / 200);
}

int main() {
  run<64>("1K ");
  run<256>("4K ");
  run<640>("10K");
  run<1200>("19K");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
