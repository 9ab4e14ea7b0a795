// A/B of the data path's copy primitive: 16-B LDG/STG (the step
// kernel's loop) against the bulk-async (TMA) engine, on the access patterns of the
// hot path, in local HBM and over NVLink to a peer GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/tma_probe tools/tma_probe.cu
//   tools/tma_probe [peer]        (peer: destination on GPU 1 through peer access)
//
// Patterns (units of `run` contiguous bytes, source and destination at the same offsets):
//   bulk    C5 re-seed: contiguous, 4 KiB units, 256 MiB
//   decode  C2 decode publication: one 256-B token slice of each of the 128 (layer, K/V,
//           head) rows of a 512-KiB block (4 KiB apart), over many blocks, 16 / 32 MiB
//   (and bulk at 16 MiB: size vs pattern)
// Kernels (each warp moves 4 KiB per round, rounds dealt grid-stride):
//   ldst        8 x 16-B loads in flight per lane, then 8 stores (kvring_step.cu's loop)
//   tma         cp.async.bulk global -> smem (mbarrier complete_tx), then
//               cp.async.bulk smem -> global; two 4-KiB buffers per warp, the next round's
//               load issued before the current round's store
//   ldg+tmast   16-B loads -> st.shared -> fence.proxy.async -> cp.async.bulk store
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

struct Pat {
  int run;           // bytes per unit (256 or 4096)
  int shift;         // log2(run)
  long long units;   // number of units
  int decode;        // 1: unit u = slice (u % 128) of block u / 128 at token (u / 128) % 16
};

__device__ __forceinline__ long long unit_off(const Pat &p, long long u) {
  if (!p.decode) return u * p.run;
  const long long b = u >> 7, c = u & 127;
  return b * (512 << 10) + c * 4096 + ((b * 7) & 15) * 256;
}

constexpr int kWarps = 8;
constexpr int kRound = 4096;  // bytes per warp round

__global__ void __launch_bounds__(256) k_ldst(const char *src, char *dst, Pat p) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const long long W = (long long)gridDim.x * kWarps;
  const long long total = p.units * p.run;
  for (long long r = gw; r * kRound < total; r += W) {
    uint4 v[8];
    long long off[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long c = r * kRound + (long long)(k * 32 + lane) * 16;  // byte in the flat space
      const long long u = c >> p.shift;
      off[k] = unit_off(p, u) + (c & (p.run - 1));
      asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + off[k]));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + off[k]), "r"(v[k].x),
                   "r"(v[k].y), "r"(v[k].z), "r"(v[k].w) : "memory");
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// lane 0 of each warp drives the bulk engine; the round's units are contiguous in the
// warp's smem buffer
__device__ __forceinline__ void tma_load_round(const Pat &p, const char *src, long long r,
                                               uint32_t buf, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kRound)
               : "memory");
  const int n = kRound / p.run;
  for (int k = 0; k < n; ++k) {
    const long long u = r * n + k;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(buf + k * p.run), "l"(src + unit_off(p, u)), "r"(p.run), "r"(bar) : "memory");
  }
}

__device__ __forceinline__ void tma_store_round(const Pat &p, char *dst, long long r, uint32_t buf) {
  const int n = kRound / p.run;
  for (int k = 0; k < n; ++k) {
    const long long u = r * n + k;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst + unit_off(p, u)), "r"(buf + k * p.run), "r"(p.run) : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(256) k_tma(const char *src, char *dst, Pat p) {
  extern __shared__ __align__(128) char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ __align__(8) unsigned long long bars[kWarps][2];
  const uint32_t buf0 = smem_u32(sm + w * 2 * kRound), buf1 = buf0 + kRound;
  const uint32_t bar0 = smem_u32(&bars[w][0]), bar1 = smem_u32(&bars[w][1]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane != 0) return;
  const long long gw = (long long)blockIdx.x * kWarps + w;
  const long long W = (long long)gridDim.x * kWarps;
  const long long total = p.units * p.run;
  const long long R = total / kRound;
  uint32_t ph0 = 0, ph1 = 0;
  long long r = gw;
  int b = 0;
  if (r < R) tma_load_round(p, src, r, buf0, bar0);
  for (; r < R; r += W, b ^= 1) {
    const long long nx = r + W;
    if (nx < R) {
      // the other buffer's previous store (round r - W) must have read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      tma_load_round(p, src, nx, b ? buf0 : buf1, b ? bar0 : bar1);
    }
    if (b == 0) {
      mbar_wait(bar0, ph0);
      ph0 ^= 1;
    } else {
      mbar_wait(bar1, ph1);
      ph1 ^= 1;
    }
    tma_store_round(p, dst, r, b ? buf1 : buf0);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(256) k_ldg_tmast(const char *src, char *dst, Pat p) {
  extern __shared__ __align__(128) char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char *mybuf = sm + w * 2 * kRound;
  const long long gw = (long long)blockIdx.x * kWarps + w;
  const long long W = (long long)gridDim.x * kWarps;
  const long long total = p.units * p.run;
  int b = 0;
  for (long long r = gw; r * kRound < total; r += W, b ^= 1) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long c = r * kRound + (long long)(k * 32 + lane) * 16;
      const long long u = c >> p.shift;
      const long long off = unit_off(p, u) + (c & (p.run - 1));
      asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + off));
    }
    // this buffer was last read by the store group before the previous one
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    char *bb = mybuf + b * kRound;
#pragma unroll
    for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4 *>(bb + (k * 32 + lane) * 16) = v[k];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) tma_store_round(p, dst, r, smem_u32(bb));
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
  const bool peer = argc > 1 && argv[1][0] == 'p';
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (peer && ndev < 2) {
    printf("peer mode needs 2 GPUs\n");
    return 0;
  }
  CK(cudaSetDevice(0));
  const size_t bytes = 600ull << 20;
  char *src, *dst;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMemset(src, 1, bytes));
  if (peer) {
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&dst, bytes));
    CK(cudaSetDevice(0));
  } else {
    CK(cudaMalloc(&dst, bytes));
  }
  const int smem = kWarps * 2 * kRound;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_ldg_tmast, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int occ_l = 0, occ_t = 0, occ_m = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_l, k_ldst, 256, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, k_tma, 256, smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_m, k_ldg_tmast, 256, smem));
  // decode: 128 slices x 256 B per block, 16 MiB of slices (= 512 blocks); bulk: 256 MiB
  const Pat pats[4] = {{4096, 12, (256ll << 20) / 4096, 0}, {256, 8, 512ll * 128, 1},
                       {4096, 12, (16ll << 20) / 4096, 0}, {256, 8, 1024ll * 128, 1}};
  const char *pname[4] = {"bulk 256 MiB", "decode 16 MiB", "bulk 16 MiB", "decode 32 MiB"};
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  printf("%s, %d SMs, resident CTAs/SM: ldst %d, tma %d, ldg+tmast %d\n",
         peer ? "peer (dst on GPU 1)" : "local", sms, occ_l, occ_t, occ_m);
  for (int pi = 0; pi < 4; ++pi) {
    const Pat p = pats[pi];
    const double D = (double)p.units * p.run;
    for (int ki = 0; ki < 3; ++ki) {
      const int occ = ki == 0 ? occ_l : ki == 1 ? occ_t : occ_m;
      const int grid = sms * (occ > 4 ? 4 : occ);
      float best = 1e30f, sum = 0.f;
      const int reps = 20;
      for (int it = 0; it < reps + 3; ++it) {
        CK(cudaEventRecord(a));
        if (ki == 0) k_ldst<<<grid, 256>>>(src, dst, p);
        else if (ki == 1) k_tma<<<grid, 256, smem>>>(src, dst, p);
        else k_ldg_tmast<<<grid, 256, smem>>>(src, dst, p);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it >= 3) {
          sum += ms;
          if (ms < best) best = ms;
        }
      }
      const char *kn[3] = {"ldst", "tma", "ldg+tmast"};
      const double avg = sum / reps;
      printf("%-14s %-10s grid %4d  avg %8.2f us  best %8.2f us  %7.1f GB/s moved (%s %.1f)\n",
             pname[pi], kn[ki], grid, avg * 1e3, best * 1e3, D / (avg * 1e-3) / 1e9,
             peer ? "NVLink" : "r+w", peer ? D / (avg * 1e-3) / 1e9 : 2 * D / (avg * 1e-3) / 1e9);
    }
  }
  // spot check: the destination holds the source's bytes (memset 1) at unit 0
  char hd[64];
  CK(cudaMemcpy(hd, dst, 64, cudaMemcpyDefault));
  printf("check %s\n", hd[0] == 1 && hd[63] == 1 ? "ok" : "MISMATCH");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
