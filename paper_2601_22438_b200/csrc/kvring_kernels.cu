// sm_100a kernels of libkvring: one task-driven slice-copy engine used by
//   append-scatter  (dense model KV -> paged pool,          SURVEY §8(a) a2)
//   ring-put        (paged pool -> successor replica, fused gather + P2P store
//                    + metadata + release seq flag,          a4+a5, §3.2)
//   gather-pack     (paged pool -> packed buffer,            a4 / a6)
//   unpack          (packed buffer -> replica + publish,     a6)
//   restore-remap   (replica -> pool at new block ids,       a8, §3.2)
//
// Pure data movement: no tensor cores (HBM / NVLink bound, DESIGN.md
// "Rooflines").  Each CTA takes one 32-KiB task at a time; each thread keeps
// 8 independent 16-B loads in flight (L1::no_allocate streaming loads), then
// stores them (16-B stores; peer addresses go over NVLink).  Tasks that finish
// bump a per-pool monotone counter after a system-scope fence; the CTA that
// completes a pool's last task writes the parity metadata and then the seq
// flag with st.release.sys (reading R9: a reader that acquires seq = t sees
// everything of step t).
#include <cuda_runtime.h>

#include "kvring_internal.h"

namespace kvring {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void *p, const uint4 &v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p,
                                                   unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__device__ __forceinline__ long long slice_offset(const KvGeomDev &g, int unit, int s,
                                                  int n_tok, int tok_lo) {
  if (MODE == kPacked) return ((long long)unit + s) * g.seg_bytes;
  const int combo = s / n_tok;
  const int tok = s - combo * n_tok;
  if (MODE == kPaged)
    return (long long)unit * g.block_bytes +
           (long long)(combo * g.block_size + tok_lo + tok) * g.seg_bytes;
  // kTokMajor
  return ((long long)unit + tok) * g.token_bytes + (long long)combo * g.seg_bytes;
}

// Copy one task's slices: thread t handles 16-B chunks t, t+256, ... of the
// task; 16 consecutive lanes cover one 256-B slice (coalesced).
template <int SRC, int DST>
__device__ __forceinline__ void copy_task(const KvTask &tk, const char *__restrict__ src,
                                          char *__restrict__ dst, const KvGeomDev &g) {
  const int nchunks = tk.seg_count << g.cps_shift;
  const int cmask = (1 << g.cps_shift) - 1;
  for (int base = 0; base < nchunks; base += kThreads * kUnroll) {
    uint4 v[kUnroll];
    long long doff[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) {
        const int s = tk.seg_begin + (c >> g.cps_shift);
        const int lc = (c & cmask) << 4;
        const long long so = slice_offset<SRC>(g, tk.src_unit, s, tk.n_tok, tk.tok_lo) + lc;
        doff[u] = slice_offset<DST>(g, tk.dst_unit, s, tk.n_tok, tk.tok_lo) + lc;
        v[u] = ld_stream(src + so);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) st_stream(dst + doff[u], v[u]);
    }
  }
}

// Publication of one pool's step by the CTA that completed its last task.
__device__ void publish(const KvPoolParams &pp) {
  char *meta = pp.meta;
  const int R = pp.max_reqs;
  const int par = (int)(pp.step & 1ull);
  int64_t *mreq = reinterpret_cast<int64_t *>(meta + 32) + (size_t)par * R;
  int32_t *mlen = reinterpret_cast<int32_t *>(meta + 32 + 16 * (size_t)R) + (size_t)par * R;
  for (int s = threadIdx.x; s < R; s += blockDim.x) {
    mreq[s] = pp.slot_req[s];
    mlen[s] = pp.slot_len[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *reinterpret_cast<int32_t *>(meta + 8) = pp.writer_node;
    __threadfence_system();
    st_release_sys_u64(reinterpret_cast<unsigned long long *>(meta), pp.step);
  }
}

// Called by all threads after a task's data stores: bt entry, fence, count, maybe publish.
__device__ __forceinline__ void finish_task(const KvTask &tk, const KvPoolParams &pp,
                                            int *s_last) {
  if (!pp.publish) return;
  if (threadIdx.x == 0 && (tk.flags & kFirst) && tk.slot >= 0) {
    int32_t *bt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)pp.max_reqs);
    bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
  }
  __syncthreads();  // every thread's stores of this task precede thread 0's fence
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned long long old = atomicAdd(pp.counter, 1ull);
    *s_last = (old + 1ull == pp.target);
  }
  __syncthreads();
  if (*s_last) publish(pp);
}

template <int SRC, int DST>
__global__ void __launch_bounds__(kThreads) copy_kernel(const KvTask *__restrict__ tasks,
                                                        int n_tasks,
                                                        const KvPoolParams *__restrict__ params,
                                                        KvGeomDev g) {
  __shared__ int s_last;
  for (int t = blockIdx.x; t < n_tasks; t += gridDim.x) {
    const KvTask tk = tasks[t];
    const KvPoolParams &pp = params[tk.pool];
    copy_task<SRC, DST>(tk, pp.src, pp.dst, g);
    finish_task(tk, pp, &s_last);
  }
}

// Receiver of the NCCL comparison: parameters come from the packed header on
// the device, so the receiving host never reads the buffer.
__global__ void __launch_bounds__(kThreads) unpack_kernel(const char *__restrict__ packed,
                                                          char *replica, char *meta,
                                                          unsigned long long *counter,
                                                          KvGeomDev g) {
  __shared__ KvPoolParams pp;
  __shared__ int s_last;
  __shared__ int n_tasks;
  const KvPackedHeader *h = reinterpret_cast<const KvPackedHeader *>(packed);
  if (threadIdx.x == 0) {
    n_tasks = h->n_tasks;
    pp.src = packed + h->payload_off;
    pp.dst = replica;
    pp.meta = meta;
    pp.slot_req = reinterpret_cast<const int64_t *>(packed + h->slot_off);
    pp.slot_len = reinterpret_cast<const int32_t *>(packed + h->slot_off + 8 * (size_t)h->max_reqs);
    pp.counter = counter;
    pp.target = (unsigned long long)h->n_tasks;
    pp.step = h->step;
    pp.max_reqs = h->max_reqs;
    pp.max_blk = h->max_blk;
    pp.writer_node = h->writer_node;
    pp.publish = 1;
  }
  __syncthreads();
  const KvTask *tasks = reinterpret_cast<const KvTask *>(packed + h->task_off);
  for (int t = blockIdx.x; t < n_tasks; t += gridDim.x) {
    const KvTask tk = tasks[t];
    copy_task<kPacked, kPaged>(tk, pp.src, pp.dst, g);
    finish_task(tk, pp, &s_last);
    if (s_last && threadIdx.x == 0) *counter = 0ull;  // counter is per call, not monotone
  }
}

__global__ void meta_init_kernel(char *meta, int R, int M) {
  const size_t n_req = 2 * (size_t)R, n_bt = (size_t)R * M;
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  if (i0 == 0) {
    *reinterpret_cast<unsigned long long *>(meta) = 0ull;
    int32_t *hdr = reinterpret_cast<int32_t *>(meta + 8);
    hdr[0] = -1;
    hdr[1] = R;
    hdr[2] = M;
    hdr[3] = kMetaMagic;
    *reinterpret_cast<long long *>(meta + 24) = 0;
  }
  int64_t *req = reinterpret_cast<int64_t *>(meta + 32);
  int32_t *len = reinterpret_cast<int32_t *>(meta + 32 + 16 * (size_t)R);
  int32_t *bt = reinterpret_cast<int32_t *>(meta + 32 + 24 * (size_t)R);
  for (size_t i = i0; i < n_req; i += stride) {
    req[i] = -1;
    len[i] = 0;
  }
  for (size_t i = i0; i < n_bt; i += stride) bt[i] = -1;
}

}  // namespace

int copy_grid(int device, int n_tasks) {
  static int sms[64] = {0};
  int d = device < 0 ? 0 : (device & 63);
  if (sms[d] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)
      v = 148;
    sms[d] = v;
  }
  const int cap = sms[d] * 8;  // 8 resident 256-thread CTAs per SM
  return n_tasks < cap ? (n_tasks > 0 ? n_tasks : 1) : cap;
}

cudaError_t launch_copy(int src_mode, int dst_mode, const KvTask *tasks, int n_tasks,
                        const KvPoolParams *params, const KvGeomDev &g, int grid,
                        cudaStream_t stream) {
  if (n_tasks <= 0) return cudaSuccess;
#define KV_LAUNCH(S, D)                                                              \
  if (src_mode == S && dst_mode == D) {                                              \
    copy_kernel<S, D><<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g);     \
    return cudaGetLastError();                                                       \
  }
  KV_LAUNCH(kTokMajor, kPaged)  // append-scatter
  KV_LAUNCH(kPaged, kPaged)     // ring-put, restore-remap
  KV_LAUNCH(kPaged, kPacked)    // gather-pack
  KV_LAUNCH(kPacked, kPaged)    // (host-driven unpack; tests)
#undef KV_LAUNCH
  return cudaErrorInvalidValue;
}

cudaError_t launch_unpack(const char *packed, char *replica, char *meta,
                          unsigned long long *counter, const KvGeomDev &g, int grid,
                          cudaStream_t stream) {
  unpack_kernel<<<grid, kThreads, 0, stream>>>(packed, replica, meta, counter, g);
  return cudaGetLastError();
}

cudaError_t launch_meta_init(char *meta, int R, int M, cudaStream_t stream) {
  const size_t n = (size_t)R * M + 2 * (size_t)R;
  int grid = (int)((n + 255) / 256);
  if (grid > 1024) grid = 1024;
  if (grid < 1) grid = 1;
  meta_init_kernel<<<grid, 256, 0, stream>>>(meta, R, M);
  return cudaGetLastError();
}

}  // namespace kvring
