// HBM efficiency of the decode step's access patterns at steady state (large copies, so
// launch latency does not count): 256-B (layer, K/V, head) slices of one token per
// 512-KiB block, 4 KiB apart (layout R4), against a contiguous copy of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stride_probe tools/stride_probe.cu
// Patterns (user bytes U per pass; r+w GB/s = 2U / time):
//   contig     read contiguous, write contiguous
//   append     read contiguous (dense token rows), write slices (paged pool)
//   publish    read slices, write slices at the same offsets of another region
//   publish2   as publish, 2 tokens per block (512 B contiguous per 4 KiB)
//   publish16  full blocks (a bulk re-seed: contiguous 512 KiB per block)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr long long kBlock = 512 << 10;  // 8 layers x 2 x 8 heads x 16 tokens x 256 B
constexpr int kSlice = 256, kStride = 4096, kCombos = 128;

// chunk k (16 B) of the pattern's user bytes -> byte offset in the paged layout
__device__ __forceinline__ long long paged_off(long long k, int tok_per_blk) {
  const long long s = k >> 4;                      // slice (tok_per_blk tokens per combo)
  const long long per_blk = (long long)kCombos * tok_per_blk;
  const long long b = s / per_blk;
  const int r = (int)(s - b * per_blk);
  const int c = r / tok_per_blk, t = r - c * tok_per_blk;
  return b * kBlock + (long long)c * kStride + (long long)t * kSlice + ((k & 15) << 4);
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) probe(const char *src, char *dst, long long nchunks,
                                                int tpb) {
  const long long W = (long long)gridDim.x * blockDim.x;
  for (long long k0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; k0 < nchunks; k0 += W * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long k = k0 + u * W;
      if (k < nchunks) {
        const long long so = MODE == 0 || MODE == 1 ? (k << 4) : paged_off(k, tpb);
        v[u] = __ldcs(reinterpret_cast<const uint4 *>(src + so));
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long k = k0 + u * W;
      if (k < nchunks) {
        const long long d = MODE == 0 ? (k << 4) : paged_off(k, tpb);
        __stcs(reinterpret_cast<uint4 *>(dst + d), v[u]);
      }
    }
  }
}

int main() {
  const long long user = 256ll << 20;          // user bytes per pass
  const long long blocks = user / (kCombos * kSlice);  // one token per block
  const long long foot = blocks * kBlock;      // 4 GiB per region at 1 token per block
  char *a, *b;
  CK(cudaMalloc(&a, foot));
  CK(cudaMalloc(&b, foot));
  CK(cudaMemset(a, 1, foot));
  CK(cudaMemset(b, 2, foot));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct P { const char *name; int mode, tpb; } ps[] = {
      {"contig", 0, 1}, {"append", 1, 1}, {"publish", 2, 1}, {"publish2", 2, 2},
      {"publish4", 2, 4}, {"publish16", 2, 16}};
  for (auto &p : ps) {
    const long long n = user >> 4;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (p.mode == 0) probe<0><<<grid, 256>>>(a, b, n, p.tpb);
      else if (p.mode == 1) probe<1><<<grid, 256>>>(a, b, n, p.tpb);
      else probe<2><<<grid, 256>>>(a, b, n, p.tpb);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-10s user %4lld MiB  %8.3f ms  %7.1f GB/s r+w\n", p.name, user >> 20, best,
           2.0 * user / (best * 1e-3) / 1e9);
  }
  // decode-sized passes (one step's publication: ~16 MiB user), back to back in one launch
  // is what the step kernel does; here 16 MiB per launch, 20 launches, to show the
  // per-launch ramp at this size
  for (auto &p : ps) {
    const long long u16 = 16ll << 20, n = u16 >> 4;
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) {
      if (p.mode == 0) probe<0><<<grid, 256>>>(a, b, n, p.tpb);
      else if (p.mode == 1) probe<1><<<grid, 256>>>(a, b, n, p.tpb);
      else probe<2><<<grid, 256>>>(a, b, n, p.tpb);
    }
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-10s 16 MiB x20   %8.2f us/launch  %7.1f GB/s r+w\n", p.name, ms * 1e3 / 20,
           2.0 * u16 * 20 / (ms * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
