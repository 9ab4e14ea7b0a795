// Diagnostic microbenchmark (not product code): cost of the ring-put's
// publication protocol on B200, without any copy.  592 CTAs x 256 threads
// (the decode-step grid); thread 0 of every CTA adds its count to one of 4
// per-pool counters; the CTA that completes a pool publishes seq.
//   mode 0: empty kernel
//   mode 1: atom.add.relaxed.gpu
//   mode 2: atom.add.release.gpu
//   mode 3: mode 2 + completing CTA: fence.acq_rel.gpu + st.release.gpu seq
//   mode 4: mode 3 preceded by 8 x 16-B stores per thread + bar.sync
//   mode 5: mode 4 with fence.acq_rel.gpu + atom.add.relaxed (fence form)
//   mode 6: mode 4 without any fence/atomic (stores only)
//   mode 7: mode 4 with red.release (no completion detection: lower bound)
//   mode 8: empty + griddepcontrol.wait (no PDL attribute on the launch)
//   mode 9: mode 8 + griddepcontrol.launch_dependents
// Usage: pubbench [grid] ; prints avg us per launch (back-to-back) and isolated.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(256, 4) k(unsigned long long *cnt, unsigned long long *seq,
                                            unsigned long long target, uint4 *buf, int grid) {
  if (MODE == 8 || MODE == 9) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (MODE == 9) asm volatile("griddepcontrol.launch_dependents;" :::);
    return;
  }
  if (MODE >= 4) {
    uint4 v = make_uint4(blockIdx.x, threadIdx.x, 1, 2);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(buf + ((size_t)blockIdx.x * 8 + u) * 256 + threadIdx.x),
                   "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    __syncthreads();
  }
  if (MODE == 0 || MODE == 6 || threadIdx.x != 0) return;
  unsigned long long *c = cnt + (blockIdx.x & 3) * 16;
  unsigned long long old = 0;
  if (MODE == 1) asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
  if (MODE == 2 || MODE == 3 || MODE == 4) asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
  if (MODE == 5) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("atom.add.relaxed.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
  }
  if (MODE == 7) { asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(c) : "memory"); return; }
  if (MODE >= 3 && old + 1 == target) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(seq + (blockIdx.x & 3) * 16), "l"(target) : "memory");
  }
}

template <int MODE>
int run(int grid, unsigned long long *cnt, unsigned long long *seq, uint4 *buf) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 200;
  unsigned long long per_pool = grid / 4;
  // back-to-back
  CK(cudaMemset(cnt, 0, 4096));
  for (int i = 0; i < 10; ++i) k<MODE><<<grid, 256>>>(cnt, seq, per_pool * (i + 1), buf, grid);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(cnt, 0, 4096));
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) k<MODE><<<grid, 256>>>(cnt, seq, per_pool * (i + 1), buf, grid);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  // isolated
  float tot = 0;
  CK(cudaMemset(cnt, 0, 4096));
  for (int i = 0; i < 50; ++i) {
    cudaEventRecord(a);
    k<MODE><<<grid, 256>>>(cnt, seq, per_pool * (i + 1), buf, grid);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float m; cudaEventElapsedTime(&m, a, b); tot += m;
  }
  printf("mode %d grid %d: back-to-back %.2f us/launch, isolated %.2f us\n", MODE, grid, ms * 1e3 / iters, tot * 1e3 / 50);
  return 0;
}

int main(int argc, char **argv) {
  int grid = argc > 1 ? atoi(argv[1]) : 592;
  unsigned long long *cnt, *seq; uint4 *buf;
  CK(cudaMalloc(&cnt, 4096)); CK(cudaMalloc(&seq, 4096));
  CK(cudaMalloc(&buf, (size_t)grid * 8 * 256 * 16));
  run<0>(grid, cnt, seq, buf); run<1>(grid, cnt, seq, buf); run<2>(grid, cnt, seq, buf);
  run<3>(grid, cnt, seq, buf); run<4>(grid, cnt, seq, buf); run<5>(grid, cnt, seq, buf);
  run<6>(grid, cnt, seq, buf); run<7>(grid, cnt, seq, buf);
  run<8>(grid, cnt, seq, buf); run<9>(grid, cnt, seq, buf);
  return 0;
}
