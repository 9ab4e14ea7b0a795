// sm_100a kernels of libkvring driven by host-built task lists (the decode-step
// engine -- append + device-derived replication -- is kvring_step.cu):
//   restore-remap   (replica -> pool at new block ids,       SURVEY §8(a) a8, §3.2)
//   gather-pack     (paged pool -> packed buffer,            a4 / a6 NCCL comparison)
//   unpack          (packed buffer -> replica + publish,     a6)
//   ring-put        (paged pool -> holder, host tasks: shared-capacity links whose
//                    replica blocks sit at holder-allocated ids, NEXT-3, and the
//                    copy-engine variant's partial blocks + publication, NEXT-4)
//
// Pure data movement: no tensor cores (HBM / NVLink bound, DESIGN.md
// "Rooflines").  Each CTA takes one <= 32-KiB task at a time; each thread keeps
// 8 independent 16-B loads in flight (L1::no_allocate streaming loads), then
// stores them.  Publication runs in a second pass: each CTA adds its per-pool task
// counts to a monotone counter with one release RMW (GPU scope); the CTA that
// completes a pool's count issues an acquire-release fence (system scope for an
// NVLink successor) and stores the seq flag right after it (release pattern;
// reading R9: a reader that acquires seq = t sees everything of step t).
#include <cuda_runtime.h>

#include "kvring_internal.h"

namespace kvring {

namespace {

constexpr int kThreads = 256;
#ifndef KV_UNROLL
#define KV_UNROLL 8
#endif
#ifndef KV_MIN_BLOCKS
#define KV_MIN_BLOCKS 4
#endif
// 8 x 16 B loads in flight per thread, 4 resident 256-thread CTAs per SM (<= 64
// registers, no spills): 128 KB in flight per SM.
constexpr int kUnroll = KV_UNROLL;
constexpr int kMinBlocks = KV_MIN_BLOCKS;

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

// Byte offset of a task's item base (64-bit) and of slice s inside the item
// (32-bit: an item never spans more than one block / B token rows).
template <int MODE>
__device__ __forceinline__ long long item_base(const KvGeomDev &g, int unit, int tok_lo) {
  if (MODE == kPacked) return (long long)unit * g.seg_bytes;
  if (MODE == kPaged) return (long long)unit * g.block_bytes + (long long)tok_lo * g.seg_bytes;
  return (long long)unit * g.token_bytes;  // kTokMajor
}

template <int MODE>
__device__ __forceinline__ unsigned slice_off(const KvGeomDev &g, int s, int n_tok) {
  if (MODE == kPacked) return (unsigned)s * (unsigned)g.seg_bytes;
  const int combo = s / n_tok;
  const int tok = s - combo * n_tok;
  if (MODE == kPaged) return (unsigned)(combo * g.block_size + tok) * (unsigned)g.seg_bytes;
  return (unsigned)tok * (unsigned)g.token_bytes + (unsigned)combo * (unsigned)g.seg_bytes;
}

// Copy one task's slices: thread t handles 16-B chunks t, t+256, ... of the
// task; 16 consecutive lanes cover one 256-B slice (coalesced).  All loads of
// a round are issued before its stores (8 x 16 B in flight per thread).
template <int SRC, int DST, bool RUN>
__device__ __forceinline__ void copy_task(const KvTask &tk, const char *__restrict__ src,
                                          char *__restrict__ dst, const KvGeomDev &g,
                                          unsigned long long src_bytes,
                                          unsigned long long dst_bytes) {
  const char *sb = src + item_base<SRC>(g, tk.src_unit, tk.tok_lo);
  char *db = dst + item_base<DST>(g, tk.dst_unit, tk.tok_lo);
#ifdef KV_BOUNDS_CHECK
  // debug builds: every 16-B access must stay inside its buffer (compute-sanitizer
  // is not available on this pool); a violation traps the kernel
  const long long sbase = item_base<SRC>(g, tk.src_unit, tk.tok_lo);
  const long long dbase = item_base<DST>(g, tk.dst_unit, tk.tok_lo);
  if (tk.seg_count > 0 && threadIdx.x == 0) {
    const int last = tk.seg_begin + tk.seg_count - 1;
    for (int s2 : {tk.seg_begin, last}) {
      if (sbase < 0 || (unsigned long long)(sbase + slice_off<SRC>(g, s2, tk.n_tok) + g.seg_bytes) > src_bytes ||
          dbase < 0 || (unsigned long long)(dbase + slice_off<DST>(g, s2, tk.n_tok) + g.seg_bytes) > dst_bytes ||
          tk.n_tok <= 0 || tk.tok_lo + tk.n_tok > g.block_size)
        __trap();
    }
  }
#else
  (void)src_bytes;
  (void)dst_bytes;
#endif
  const int nchunks = tk.seg_count << g.cps_shift;
  // a task covering whole blocks between paged / packed layouts (bulk re-seed, restore,
  // gather-pack / unpack of full blocks): slice s sits at s * seg on both sides (combo * B
  // + tok = s when n_tok = B), so no division per chunk.  RUN: a loop of its own over the
  // contiguous run (gather-pack 1.82 -> 1.49 ms at C5, unpack 1.53 -> 1.44; in the
  // restore's dynamic-task kernel it spills and costs 15 %, so there the general loop
  // only skips the divisions: pack alone that way 1.74 ms)
  const bool full = SRC != kTokMajor && DST != kTokMajor && tk.n_tok == g.block_size;
  if (RUN && full) {
    const char *sr = sb + (size_t)tk.seg_begin * (unsigned)g.seg_bytes;
    char *dr = db + (size_t)tk.seg_begin * (unsigned)g.seg_bytes;
    for (int base = 0; base < nchunks; base += kThreads * kUnroll) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int c = base + u * kThreads + (int)threadIdx.x;
        if (c < nchunks) v[u] = ld_stream(sr + ((size_t)c << 4));
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int c = base + u * kThreads + (int)threadIdx.x;
        if (c < nchunks) st_stream(dr + ((size_t)c << 4), v[u]);
      }
    }
    return;
  }
  const int cmask = (1 << g.cps_shift) - 1;
  for (int base = 0; base < nchunks; base += kThreads * kUnroll) {
    uint4 v[kUnroll];
    unsigned doff[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) {
        const int s = tk.seg_begin + (c >> g.cps_shift);
        const unsigned lc = (unsigned)(c & cmask) << 4;
        unsigned so;
        if (full) {
          so = (unsigned)s * (unsigned)g.seg_bytes + lc;
          doff[u] = so;
        } else {
          so = slice_off<SRC>(g, s, tk.n_tok) + lc;
          doff[u] = slice_off<DST>(g, s, tk.n_tok) + lc;
        }
        v[u] = ld_stream(sb + so);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) st_stream(db + doff[u], v[u]);
    }
  }
}

// Release-only RMW (every CTA's count); the CTA that completes a pool then
// issues an acquire fence before its release store of seq (synchronises with
// every earlier release in the counter's RMW chain).
__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long *p,
                                                               unsigned long long v, bool sys) {
  unsigned long long old;
  if (sys)
    asm volatile("atom.add.release.sys.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  else
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ void fence_acquire(bool sys) {
  if (sys)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// The store of seq right after fence_acquire: a fence.acq_rel followed by a strong
// (relaxed) store is a release pattern in the PTX memory model, so the store needs no
// second fence (st.release would emit another MEMBAR; at system scope that second
// MEMBAR.SYS costs microseconds per step over NVLink).
__device__ __forceinline__ void st_after_fence(unsigned long long *p, unsigned long long v,
                                               bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Parity-`step` (req_id, len) table of one pool (reading R9).  Written by the
// CTA that owns the pool's first task, BEFORE that CTA's release: a reader
// only trusts parity t once it acquires seq = t, so writing it early is safe.
__device__ void write_parity_table(const KvPoolParams &pp) {
  char *meta = pp.meta;
  const int R = pp.max_reqs;
  const int par = (int)(pp.step & 1ull);
  int64_t *mreq = reinterpret_cast<int64_t *>(meta + 32) + (size_t)par * R;
  int32_t *mlen = reinterpret_cast<int32_t *>(meta + 32 + 16 * (size_t)R) + (size_t)par * R;
  const int n = pp.n_table;
  for (int s = threadIdx.x; s < R; s += blockDim.x) {
    mreq[s] = s < n ? pp.slot_req[s] : -1;
    mlen[s] = s < n ? pp.slot_len[s] : 0;
  }
  if (threadIdx.x == 0) *reinterpret_cast<int32_t *>(meta + 8) = pp.writer_node;
}

constexpr int kMaxPoolsPerLaunch = 64;

// Pass 2 of the ring-put: publication bookkeeping of this CTA's tasks, one task
// per thread: bt entries of first tasks, per-pool task counts, pools whose
// parity table this CTA owns (kPoolFirst).  Readers trust none of it before
// seq = t.  Then __syncthreads() and ONE thread adds the counts with
// release RMWs (GPU scope) -- the bar.sync + single-release pattern of CUTLASS's
// semaphore, no per-thread fences.  The CTA whose RMW completes a pool's count
// issues one acquire-release fence (system scope for an NVLink successor) and
// stores that pool's seq (last-CTA pattern, reading R9).
__device__ __noinline__ void publish_pass(const KvTask *__restrict__ tasks, int n_tasks,
                                          const KvPoolParams *__restrict__ params, int n_pools) {
  __shared__ int s_cnt[kMaxPoolsPerLaunch];
  __shared__ int s_own[kMaxPoolsPerLaunch];
  for (int i = threadIdx.x; i < n_pools; i += blockDim.x) {
    s_cnt[i] = 0;
    s_own[i] = 0;
  }
  __syncthreads();
  // the tasks this CTA copied (task t runs on CTA t mod G), one per thread: counting
  // exactly the CTA's own tasks is what makes its release cover the stores it counts
  const int G = (int)gridDim.x;
  for (int t = (int)blockIdx.x + (int)threadIdx.x * G; t < n_tasks; t += (int)blockDim.x * G) {
    const KvTask tk = tasks[t];
    const KvPoolParams &pp = params[tk.pool];
    if ((tk.flags & kFirst) && tk.slot >= 0) {
      int32_t *bt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)pp.max_reqs);
      bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
    }
    if (tk.flags & kPoolFirst) s_own[tk.pool] = 1;
    atomicAdd(&s_cnt[tk.pool], 1);
  }
  __syncthreads();
  for (int i = 0; i < n_pools; ++i)
    if (s_own[i]) write_parity_table(params[i]);
  __syncthreads();  // every thread's stores precede the single release below
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_pools; ++i) {
      if (s_cnt[i] == 0) continue;
      const KvPoolParams &pp = params[i];
      const bool sys = pp.sys_scope != 0;
      // The count RMW is a release at SYSTEM scope when the successor is an NVLink peer:
      // a GPU-scope release does not wait for this CTA's stores into peer memory (the
      // concurrent reader test caught seq = t ahead of step t's slices with it); the
      // completing CTA then issues one acquire-release fence before its store of seq.
      const unsigned long long old =
          atom_add_release(pp.counter, (unsigned long long)s_cnt[i], sys);
      if (old + (unsigned long long)s_cnt[i] == pp.target) {
        fence_acquire(sys);
        st_after_fence(reinterpret_cast<unsigned long long *>(pp.meta), pp.step, sys);
      }
    }
  }
}

// Grid-stride over tasks.  A CTA counts the tasks it finished per pool in
// shared memory.  After its loop: __syncthreads(), then ONE thread adds the
// counts with acquire-release RMWs (GPU scope, or system scope when the
// successor is an NVLink peer) -- the bar.sync + single-release pattern of
// CUTLASS's semaphore, so no per-thread fences.  The CTA whose RMW completes a
// pool's count stores that pool's seq with a release store (last-CTA
// pattern): readers that acquire seq = t see all of step t.
template <int SRC, int DST, bool PUB, bool DYN>
__device__ __forceinline__ void run_tasks(const KvTask *__restrict__ tasks, int n_tasks,
                                          const KvPoolParams *__restrict__ params,
                                          const KvGeomDev &g, int n_pools) {
  // pass 1: the copies -- identical for every kernel, no publication state live.
  if constexpr (PUB || !DYN) {
    // the ring-put's publication counts each task on the CTA that copied it (task u on
    // CTA u mod G): static grid-stride (gather-pack too: measured no faster dynamic)
    for (int u = blockIdx.x; u < n_tasks; u += gridDim.x) {
      const KvTask tk = tasks[u];
      const KvPoolParams &pp = params[tk.pool];
#ifdef KV_BOUNDS_CHECK
      const unsigned long long sbytes = pp.src_bytes, dbytes = pp.dst_bytes;
#else
      const unsigned long long sbytes = 0, dbytes = 0;
#endif
      copy_task<SRC, DST, !PUB>(tk, pp.src, pp.dst, g, sbytes, dbytes);
    }
    if constexpr (PUB) publish_pass(tasks, n_tasks, params, n_pools);
  } else {
    // restore: the first task of every CTA static, the rest handed out by a
    // counter in the launch's staged parameters (zero as staged): SMs do not move bytes
    // at the same rate, so a static split leaves the slowest CTAs finishing alone.  The
    // next draw is issued before the current task's copy, so its latency hides.
    __shared__ int s_next;
    unsigned int *ctr = reinterpret_cast<unsigned int *>(
        const_cast<int32_t *>(&params[0].pad0));
    for (int u = blockIdx.x; u < n_tasks;) {
      unsigned int nx = 0;
      if (threadIdx.x == 0) nx = atomicAdd(ctr, 1u);
      const KvTask tk = tasks[u];
      const KvPoolParams &pp = params[tk.pool];
#ifdef KV_BOUNDS_CHECK
      const unsigned long long sbytes = pp.src_bytes, dbytes = pp.dst_bytes;
#else
      const unsigned long long sbytes = 0, dbytes = 0;
#endif
      copy_task<SRC, DST, false>(tk, pp.src, pp.dst, g, sbytes, dbytes);
      if (threadIdx.x == 0) s_next = (int)gridDim.x + (int)nx;
      __syncthreads();
      u = s_next;
      __syncthreads();  // before thread 0 writes the next draw
    }
  }
}

// One named kernel per role (ncu / launch lists show what ran).
#define KV_KERNEL(NAME, SRC, DST, PUB, DYN)                                              \
  __global__ void __launch_bounds__(kThreads, kMinBlocks)                                \
      NAME(const KvTask *__restrict__ tasks, int n_tasks,                                \
           const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools) {          \
    run_tasks<SRC, DST, PUB, DYN>(tasks, n_tasks, params, g, n_pools);                   \
  }
KV_KERNEL(kv_restore_remap_kernel, kPaged, kPaged, false, true)   // a8: replica -> new block ids
KV_KERNEL(kv_gather_pack_kernel, kPaged, kPacked, false, false)   // a4: NCCL-variant sender
// host-task ring-put: shared-capacity links (replica blocks at holder-allocated ids)
// and the copy-engine variant's partial blocks + publication
KV_KERNEL(kv_ring_put_kernel, kPaged, kPaged, true, false)
#undef KV_KERNEL

// Receiver of the NCCL comparison: parameters come from the packed header on
// the device, so the receiving host never reads the buffer.  The counter is
// per call (reset by the publishing CTA), not monotone.
__global__ void __launch_bounds__(kThreads) kv_unpack_kernel(const char *__restrict__ packed,
                                                             char *replica, char *meta,
                                                             unsigned long long *counter,
                                                             KvGeomDev g) {
  __shared__ KvPoolParams pp;
  __shared__ int s_cnt, n_tasks;
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
    pp.sys_scope = 1;
    pp.n_table = h->max_reqs;
    s_cnt = 0;
  }
  __syncthreads();
  const KvTask *tasks = reinterpret_cast<const KvTask *>(packed + h->task_off);
  for (int t = blockIdx.x; t < n_tasks; t += gridDim.x) {
    const KvTask tk = tasks[t];
    copy_task<kPacked, kPaged, true>(tk, pp.src, pp.dst, g, ~0ull, ~0ull);
    if (tk.flags & kPoolFirst) write_parity_table(pp);
    if (threadIdx.x == 0) {
      if ((tk.flags & kFirst) && tk.slot >= 0) {
        int32_t *bt = reinterpret_cast<int32_t *>(meta + 32 + 24 * (size_t)pp.max_reqs);
        bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
      }
      s_cnt += 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt > 0) {
    const unsigned long long old = atom_add_release(counter, (unsigned long long)s_cnt, true);
    if (old + (unsigned long long)s_cnt == pp.target) {
      fence_acquire(true);
      st_after_fence(reinterpret_cast<unsigned long long *>(meta), pp.step, true);
      *counter = 0ull;  // per-call counter: the next unpack is stream-ordered after this one
    }
  }
}

__global__ void kv_meta_init_kernel(char *meta, int R, int M) {
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

// kv_restore's read of a holder's metadata (reading R9, reader side): thread 0 of
// every CTA acquires seq (ld.acquire.sys), the CTA synchronises, every thread issues
// an acquire fence, then the CTAs copy header + parity tables + bt rows to `out`.
// The seq written to out[0] is the acquired value, so the tables the host reads are
// at least as new as that step's publication (the failed predecessor writes no more).
__global__ void __launch_bounds__(256) kv_meta_acquire_kernel(const char *__restrict__ meta,
                                                              char *__restrict__ out,
                                                              size_t bytes) {
  __shared__ unsigned long long s_seq;
  if (threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(meta) : "memory");
    s_seq = v;
  }
  __syncthreads();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<unsigned long long *>(out) = s_seq;
  const size_t n16 = bytes / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x)
    if (i > 0)  // word 0..15 holds seq (written above) and the header
      reinterpret_cast<uint4 *>(out)[i] = reinterpret_cast<const uint4 *>(meta)[i];
  if (blockIdx.x == 0 && threadIdx.x == 1)  // header bytes 8..15 (writer, R)
    reinterpret_cast<unsigned long long *>(out)[1] =
        reinterpret_cast<const unsigned long long *>(meta)[1];
}

}  // namespace

// Resident 256-thread CTAs of the copy kernels (kMinBlocks per SM).
// A launch never exceeds this: extra tasks are taken by grid-stride, so a
// decode-sized step is one wave.
int resident_ctas(int device) {
  static int sms[64] = {0};
  const int d = device < 0 ? 0 : (device & 63);
  if (sms[d] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)
      v = 148;
    cudaGetLastError();
    sms[d] = v;
  }
  return sms[d] * kMinBlocks;
}

int copy_grid(int device, int n_tasks) {
  const int cap = resident_ctas(device);
  return n_tasks < cap ? (n_tasks > 0 ? n_tasks : 1) : cap;
}

cudaError_t launch_copy(int kind, const KvTask *tasks, int n_tasks, const KvPoolParams *params,
                        int n_pools, const KvGeomDev &g, int grid, cudaStream_t stream) {
  if (n_tasks <= 0) return cudaSuccess;
  if (n_pools > kMaxPoolsPerLaunch) return cudaErrorInvalidValue;
  switch (kind) {
    case kKindRingPut:
      kv_ring_put_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools);
      break;
    case kKindRestore:
      kv_restore_remap_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools);
      break;
    case kKindPack:
      kv_gather_pack_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack(const char *packed, char *replica, char *meta,
                          unsigned long long *counter, const KvGeomDev &g, int grid,
                          cudaStream_t stream) {
  kv_unpack_kernel<<<grid, kThreads, 0, stream>>>(packed, replica, meta, counter, g);
  return cudaGetLastError();
}

cudaError_t launch_meta_init(char *meta, int R, int M, cudaStream_t stream) {
  const size_t n = (size_t)R * M + 2 * (size_t)R;
  int grid = (int)((n + 255) / 256);
  if (grid > 1024) grid = 1024;
  if (grid < 1) grid = 1;
  kv_meta_init_kernel<<<grid, 256, 0, stream>>>(meta, R, M);
  return cudaGetLastError();
}

cudaError_t launch_meta_acquire(const char *meta, char *out, size_t bytes, cudaStream_t stream) {
  size_t n16 = bytes / 16;
  int grid = (int)((n16 + 255) / 256);
  if (grid > 64) grid = 64;
  if (grid < 1) grid = 1;
  kv_meta_acquire_kernel<<<grid, 256, 0, stream>>>(meta, out, bytes);
  return cudaGetLastError();
}

}  // namespace kvring
