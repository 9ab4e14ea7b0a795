// Diagnostic microbenchmark (not product code): access patterns of the slice
// copy engine on B200.  A "task" moves 128 slices of 256 B (32 KiB).
//   mode 0: src contiguous 32 KiB  -> dst 128 x 256 B at 4 KiB stride   (append-like, decode)
//   mode 1: src 128 x 256 B @4 KiB -> dst 128 x 256 B @4 KiB            (ring-put, decode)
//   mode 2: src contiguous         -> dst contiguous                     (full blocks)
//   mode 3: src 256 B @4 KiB       -> dst contiguous                     (gather-pack)
// Tasks target random 512-KiB blocks of a large pool (like live requests).
// Usage: copybench [n_tasks] [warm(0/1)] [peer(0/1): destination on GPU 1 over NVLink]
//                  [streams(1/2): 2 = two such copies launched concurrently on two streams]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

struct Task { long long src, dst; };

template <int MODE, int U>
__global__ void __launch_bounds__(256, 4) k(const Task *tasks, int n, const char *src, char *dst) {
  for (int t = blockIdx.x; t < n; t += gridDim.x) {
    const Task tk = tasks[t];
    const int nch = 2048;
    for (int base = 0; base < nch; base += 256 * U) {
      uint4 v[U];
      long long doff[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = base + u * 256 + threadIdx.x;
        const int s = c >> 4, lc = (c & 15) << 4;
        long long so, d;
        if (MODE == 0) { so = tk.src + c * 16; d = tk.dst + (long long)s * 4096 + lc; }
        else if (MODE == 1) { so = tk.src + (long long)s * 4096 + lc; d = tk.dst + (long long)s * 4096 + lc; }
        else if (MODE == 2) { so = tk.src + c * 16; d = tk.dst + c * 16; }
        else { so = tk.src + (long long)s * 4096 + lc; d = tk.dst + c * 16; }
        doff[u] = d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + so));
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + doff[u]),
                     "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w) : "memory");
    }
  }
}

__global__ void flush(char *p, size_t n) {
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n;
       i += (size_t)gridDim.x * blockDim.x * 16)
    *reinterpret_cast<uint4 *>(p + i) = make_uint4(1, 2, 3, 4);
}

__global__ void touch(const Task *tasks, int n, const char *src, int mode, unsigned *sink) {
  unsigned acc = 0;
  for (int t = blockIdx.x; t < n; t += gridDim.x) {
    for (int c = threadIdx.x; c < 2048; c += 256) {
      const int s = c >> 4, lc = (c & 15) << 4;
      long long so = (mode == 0 || mode == 2) ? tasks[t].src + c * 16 : tasks[t].src + (long long)s * 4096 + lc;
      acc += *reinterpret_cast<const unsigned *>(src + so);
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 600;
  const int warm = argc > 2 ? atoi(argv[2]) : 1;
  const int peer = argc > 3 ? atoi(argv[3]) : 0;
  const int nstreams = argc > 4 ? atoi(argv[4]) : 1;
  cudaStream_t s2;
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e2a, e2b;
  cudaEventCreate(&e2a);
  cudaEventCreate(&e2b);
  const size_t pool = 6ull << 30, flushb = 512ull << 20;
  char *src, *dst, *fl;
  unsigned *sink;
  CK(cudaMalloc(&src, pool));
  if (peer) {
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&dst, pool));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
  } else {
    CK(cudaMalloc(&dst, pool));
  }
  CK(cudaMalloc(&fl, flushb));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(src, 1, pool));
  CK(cudaMemset(dst, 2, pool));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  srand(7);
  const long long nblk = pool / (512 << 10);
  const char *names[4] = {"append-like contig->scatter", "ring-put scatter->scatter",
                          "block contig->contig", "pack scatter->contig"};
  for (int mode = 0; mode < 4; ++mode) {
    std::vector<Task> h(n);
    for (int i = 0; i < n; ++i) {
      long long b = (rand() % nblk) * (512ll << 10) + (rand() % 16) * 256ll;
      long long b2 = (rand() % nblk) * (512ll << 10) + (rand() % 16) * 256ll;
      if (mode == 0 || mode == 2) b = ((long long)i * 32768) % (pool - 65536);
      if (mode == 2 || mode == 3) b2 = ((long long)i * 32768) % (pool - 65536);
      h[i] = {b, b2};
    }
    Task *d;
    CK(cudaMalloc(&d, n * sizeof(Task)));
    CK(cudaMemcpy(d, h.data(), n * sizeof(Task), cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int variant = 0; variant < 2; ++variant) {
      float best = 1e9, sum = 0;
      const int reps = 20;
      for (int r = 0; r < reps; ++r) {
        flush<<<sms * 4, 256>>>(fl, flushb);
        if (warm) touch<<<sms * 4, 256>>>(d, n, src, mode, sink);
        const int grid = n < sms * 4 ? n : sms * 4;
        cudaEventRecord(a);
        if (nstreams == 2) {  // a second, identical copy on another stream (other bytes)
          cudaEventRecord(e2a, 0);
          cudaStreamWaitEvent(s2, e2a, 0);
          if (mode == 1) k<1, 8><<<grid, 256, 0, s2>>>(d, n, src, dst);  // same bytes: timing only
          cudaEventRecord(e2b, s2);
        }
        if (variant == 0) {
          if (mode == 0) k<0, 8><<<grid, 256>>>(d, n, src, dst);
          if (mode == 1) k<1, 8><<<grid, 256>>>(d, n, src, dst);
          if (mode == 2) k<2, 8><<<grid, 256>>>(d, n, src, dst);
          if (mode == 3) k<3, 8><<<grid, 256>>>(d, n, src, dst);
        } else {
          if (mode == 0) k<0, 4><<<grid, 256>>>(d, n, src, dst);
          if (mode == 1) k<1, 4><<<grid, 256>>>(d, n, src, dst);
          if (mode == 2) k<2, 4><<<grid, 256>>>(d, n, src, dst);
          if (mode == 3) k<3, 4><<<grid, 256>>>(d, n, src, dst);
        }
        if (nstreams == 2) cudaStreamWaitEvent(0, e2b, 0);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 2) { best = ms < best ? ms : best; sum += ms; }
      }
      const double bytes = (peer ? 1.0 : 2.0) * n * 32768 * (mode == 1 ? nstreams : 1);
      printf("%-30s n=%5d x%d warm=%d U=%d peer=%d best %7.2f us  avg %7.2f us  -> %7.1f GB/s (%s, best)\n",
             names[mode], n, mode == 1 ? nstreams : 1, warm, variant == 0 ? 8 : 4, peer, best * 1e3, sum / (reps - 3) * 1e3,
             bytes / (best * 1e-3) / 1e9, peer ? "NVLink payload" : "r+w");
    }
    cudaFree(d);
  }
  return 0;
}
