// Diagnostic microbenchmark (not product code): host cost of one kernel launch
// vs the size of its parameter block (__grid_constant__ struct), B200 + this
// driver.  Empty kernels, 592 x 256, launched 2000 times back to back; reports
// host microseconds per launch call.
#include <chrono>
#include <cstdio>
#include <vector>
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

// Device time per kernel when the same launches come from one CUDA graph, and the host
// cost of updating a graph kernel node's parameters (what a per-step graph would pay).
template <int N>
void run_graph(cudaStream_t s) {
  Blob<N> p{};
  const int iters = 200;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < iters; ++i) k<N><<<592, 256, 0, s>>>(p);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  spin<<<1, 1, 0, s>>>(30000000ll);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // host cost of a parameter update of one node
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  std::vector<cudaGraphNode_t> nodes(nn);
  cudaGraphGetNodes(g, nodes.data(), &nn);
  cudaKernelNodeParams kp;
  cudaGraphKernelNodeGetParams(nodes[0], &kp);
  void *args[1] = {&p};
  kp.kernelParams = args;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) {
    p.b[0] = (char)i;
    cudaGraphExecKernelNodeSetParams(ge, nodes[i % nn], &kp);
  }
  auto t1 = std::chrono::steady_clock::now();
  printf("params %6d B: graph device %.2f us/kernel, node update host %.2f us\n", N,
         ms * 1e3 / iters, std::chrono::duration<double>(t1 - t0).count() * 1e6 / 1000);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  run<256>(s); run<1024>(s); run<4096>(s); run<8192>(s); run<16384>(s); run<28672>(s); run<32000>(s);
  run_gpu<256>(s); run_gpu<4096>(s); run_gpu<8192>(s); run_gpu<16384>(s); run_gpu<28672>(s);
  run_graph<256>(s); run_graph<8192>(s); run_graph<16384>(s); run_graph<28672>(s);
  return 0;
}
