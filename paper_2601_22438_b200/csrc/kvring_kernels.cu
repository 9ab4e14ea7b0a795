// sm_100a kernels of libkvring: one task-driven slice-copy engine used by
//   append-scatter  (dense model KV -> paged pool,          SURVEY §8(a) a2)
//   ring-put        (paged pool -> successor replica, fused gather + P2P store
//                    + metadata + release seq flag,          a4+a5, §3.2)
//   gather-pack     (paged pool -> packed buffer,            a4 / a6)
//   unpack          (packed buffer -> replica + publish,     a6)
//   restore-remap   (replica -> pool at new block ids,       a8, §3.2)
//
// Pure data movement: no tensor cores (HBM / NVLink bound, DESIGN.md
// "Rooflines").  Each CTA takes one <= 32-KiB task at a time; each thread keeps
// 8 independent 16-B loads in flight (L1::no_allocate streaming loads), then
// stores them (16-B stores; peer addresses go over NVLink).  Publication runs in
// a second pass: each CTA adds its per-pool task counts to a monotone counter
// with one release RMW (GPU scope); the CTA that completes a pool's count issues
// an acquire-release fence (system scope for an NVLink successor) and stores the
// seq flag right after it (release pattern; reading R9: a reader that acquires seq = t sees
// everything of step t).  The hot kernels exist twice: with descriptors staged in
// global memory, and "inline" with parameters, tables and tasks in the kernel
// parameter space (KvInlineDescT, 4-28 KiB size classes) for decode-size steps.
#include <cstdlib>

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
template <int SRC, int DST>
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
        doff[u] = slice_off<DST>(g, s, tk.n_tok) + lc;
        v[u] = ld_stream(sb + slice_off<SRC>(g, s, tk.n_tok) + lc);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) st_stream(db + doff[u], v[u]);
    }
  }
}

// Paged destination with a runtime source layout (dense token-major for the
// append part of a fused step, paged for its ring-put part): one loop body, so
// the fused kernel keeps the 64-register budget of the single-role kernels.
__device__ __forceinline__ void copy_task_dyn(const KvTask &tk, const char *__restrict__ src,
                                              char *__restrict__ dst, const KvGeomDev &g,
                                              bool src_tokmajor) {
  const char *sb = src + (src_tokmajor ? item_base<kTokMajor>(g, tk.src_unit, tk.tok_lo)
                                       : item_base<kPaged>(g, tk.src_unit, tk.tok_lo));
  char *db = dst + item_base<kPaged>(g, tk.dst_unit, tk.tok_lo);
  const int nchunks = tk.seg_count << g.cps_shift;
  const int cmask = (1 << g.cps_shift) - 1;
  const unsigned tstride = src_tokmajor ? (unsigned)g.token_bytes : (unsigned)g.seg_bytes;
  const unsigned cstride = src_tokmajor ? (unsigned)g.seg_bytes
                                        : (unsigned)(g.block_size * g.seg_bytes);
  for (int base = 0; base < nchunks; base += kThreads * kUnroll) {
    uint4 v[kUnroll];
    unsigned doff[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * kThreads + (int)threadIdx.x;
      if (c < nchunks) {
        const int s = tk.seg_begin + (c >> g.cps_shift);
        const unsigned lc = (unsigned)(c & cmask) << 4;
        const int combo = s / tk.n_tok;
        const int tok = s - combo * tk.n_tok;
        doff[u] = (unsigned)(combo * g.block_size + tok) * (unsigned)g.seg_bytes + lc;
        v[u] = ld_stream(sb + (unsigned)tok * tstride + (unsigned)combo * cstride + lc);
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
// tbl_base != nullptr: an inline launch, slot_req / slot_len hold offsets into it.
__device__ void write_parity_table(const KvPoolParams &pp, const char *tbl_base) {
  char *meta = pp.meta;
  const int R = pp.max_reqs;
  const int par = (int)(pp.step & 1ull);
  int64_t *mreq = reinterpret_cast<int64_t *>(meta + 32) + (size_t)par * R;
  int32_t *mlen = reinterpret_cast<int32_t *>(meta + 32 + 16 * (size_t)R) + (size_t)par * R;
  const int64_t *sreq = tbl_base ? reinterpret_cast<const int64_t *>(
                                       tbl_base + reinterpret_cast<size_t>(pp.slot_req))
                                 : pp.slot_req;
  const int32_t *slen = tbl_base ? reinterpret_cast<const int32_t *>(
                                       tbl_base + reinterpret_cast<size_t>(pp.slot_len))
                                 : pp.slot_len;
  const int n = pp.n_table;
  for (int s = threadIdx.x; s < R; s += blockDim.x) {
    mreq[s] = s < n ? sreq[s] : -1;
    mlen[s] = s < n ? slen[s] : 0;
  }
  if (threadIdx.x == 0) *reinterpret_cast<int32_t *>(meta + 8) = pp.writer_node;
}

constexpr int kMaxPoolsPerLaunch = 64;

// Pass 2 of the ring-put: publication bookkeeping of this CTA's tasks, one task
// per thread: bt entries of first tasks, per-pool task counts, pools whose
// parity table this CTA owns (kPoolFirst).  Readers trust none of it before
// seq = t.  Then __syncthreads() and ONE thread adds the counts with
// acquire-release RMWs (GPU scope, or system scope when the successor is an
// NVLink peer) -- the bar.sync + single-release pattern of CUTLASS's semaphore,
// no per-thread fences.  The CTA whose RMW completes a pool's count stores
// that pool's seq with a release store (last-CTA pattern, reading R9).
__device__ __noinline__ void publish_pass(const KvTask *__restrict__ tasks, int n_tasks,
                                          const KvPoolParams *__restrict__ params, int n_pools,
                                          const char *tbl_base = nullptr, int split = 1,
                                          int unit_off = 0) {
  __shared__ int s_cnt[kMaxPoolsPerLaunch];
  __shared__ int s_own[kMaxPoolsPerLaunch];
  for (int i = threadIdx.x; i < n_pools; i += blockDim.x) {
    s_cnt[i] = 0;
    s_own[i] = 0;
  }
  __syncthreads();
  // the units this CTA copied, one per thread: global unit ug = blockIdx.x + i * gridDim.x
  // of the copy loop, of which this list holds [unit_off, unit_off + n_units) (the fused
  // kernel's ring-put part follows its append part).  Counting exactly the CTA's own
  // units is what makes its release cover the stores it counts.
  const int G = (int)gridDim.x;
  const int n_units = n_tasks * split;
  int u0 = (int)blockIdx.x;
  if (u0 < unit_off) u0 += (unit_off - u0 + G - 1) / G * G;
  for (int ug = u0 + (int)threadIdx.x * G; ug < unit_off + n_units; ug += (int)blockDim.x * G) {
    const int u = ug - unit_off;
    const KvTask tk = tasks[u / split];
    const bool lead = (u % split) == 0;  // bt entry / table ownership: once per task
    const KvPoolParams &pp = params[tk.pool];
    if (lead && (tk.flags & kFirst) && tk.slot >= 0) {
      int32_t *bt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)pp.max_reqs);
      bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
    }
    if (lead && (tk.flags & kPoolFirst)) s_own[tk.pool] = 1;
    atomicAdd(&s_cnt[tk.pool], 1);
  }
  __syncthreads();
  for (int i = 0; i < n_pools; ++i)
    if (s_own[i]) write_parity_table(params[i], tbl_base);
  __syncthreads();  // every thread's stores precede the single release below
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_pools; ++i) {
      if (s_cnt[i] == 0) continue;
      const KvPoolParams &pp = params[i];
      const bool sys = pp.sys_scope != 0;
      // Every CTA of this launch runs on this GPU, so the count RMW only needs GPU
      // scope even when the stores went to an NVLink peer; the completing CTA then
      // issues ONE system-scope acquire-release fence before its (relaxed) store of
      // seq.  Causality order is transitive (release.gpu -> fence.acq_rel.sys, which
      // acquires the count and releases the seq store that follows it), so a peer that
      // acquires seq = t sees every CTA's stores.
      // KVRING_SYS_PER_CTA=1 (experiments) restores a system-scope RMW per CTA.
      const unsigned long long old = atom_add_release(
          pp.counter, (unsigned long long)s_cnt[i], sys && (pp.pad0 & 1));
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
template <int SRC, int DST, bool PUB>
__device__ __forceinline__ void run_tasks(const KvTask *__restrict__ tasks, int n_tasks,
                                          const KvPoolParams *__restrict__ params,
                                          const KvGeomDev &g, int n_pools,
                                          const KvParamPack *pk = nullptr,
                                          const char *tbl_base = nullptr, int split = 1) {
  // pass 1: the copies -- identical for every kernel, no publication state live.
  // Unit u = task u / split, share u % split of its slices.
  const int n_units = n_tasks * split;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    KvTask tk = tasks[u / split];
    if (split > 1) {
      const int per = (tk.seg_count + split - 1) / split;
      const int b0 = (u % split) * per;
      tk.seg_begin += b0;
      tk.seg_count = max(0, min(per, tk.seg_count - b0));
    }
    const KvPoolParams &pp = params[tk.pool];
#ifdef KV_BOUNDS_CHECK
    const unsigned long long sbytes = pp.src_bytes, dbytes = pp.dst_bytes;
#else
    const unsigned long long sbytes = 0, dbytes = 0;
#endif
    const bool inl = pk && pk->n;
    const char *src = inl ? pk->src[tk.pool] : pp.src;
    char *dst = inl ? pk->dst[tk.pool] : pp.dst;
    copy_task<SRC, DST>(tk, src, dst, g, sbytes, dbytes);
  }
  if constexpr (PUB) publish_pass(tasks, n_tasks, params, n_pools, tbl_base, split);
}

// One named kernel per role (ncu / launch lists show what ran).
// Programmatic dependent launch (PDL, kv_run_steps_pdl): both instructions are
// no-ops for a kernel launched without the programmatic-serialization attribute.
//  - ring-put k : wait for its append (griddepcontrol.wait: the primary grid has
//                 completed and its writes are visible), then let append k+1 launch;
//  - append k+1 : lets ring-put k+1 launch at once (it waits at its start), copies
//                 (concurrently with ring-put k: disjoint slots, reading R7), then
//                 waits for ring-put k before exiting -- so ring-put k+1, which
//                 waits for append k+1, starts after ring-put k: seq stays monotone.
// All CTAs of a primary are resident before its dependent launches (grids never
// exceed the resident CTA count), so a waiting dependent cannot starve it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

#define KV_KERNEL(NAME, SRC, DST, PUB)                                                   \
  __global__ void __launch_bounds__(kThreads, kMinBlocks)                                \
      NAME(const KvTask *__restrict__ tasks, int n_tasks,                                \
           const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools) {          \
    run_tasks<SRC, DST, PUB>(tasks, n_tasks, params, g, n_pools);                        \
  }
KV_KERNEL(kv_restore_remap_kernel, kPaged, kPaged, false)      // a8: replica -> new block ids
KV_KERNEL(kv_gather_pack_kernel, kPaged, kPacked, false)       // a4: NCCL-variant sender
#undef KV_KERNEL

// The hot kernels take the per-pool parameters (<= kInlinePools pools) by value in
// the kernel's constant parameter space: no dependent global load precedes a CTA's
// first data load (only its task descriptor).  More pools: the staged global copy.
// a2: model KV write stand-in (dense -> paged)
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_append_scatter_kernel(const KvTask *__restrict__ tasks, int n_tasks,
                             const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools,
                             const __grid_constant__ KvParamPack pk, int split) {
  pdl_launch_dependents();
  run_tasks<kTokMajor, kPaged, false>(tasks, n_tasks, params, g, n_pools, &pk, nullptr, split);
  pdl_wait();
}

// a4+a5: fused gather + ring hop + publication
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_ring_put_kernel(const KvTask *__restrict__ tasks, int n_tasks,
                       const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools,
                       const __grid_constant__ KvParamPack pk, int split) {
  pdl_wait();
  pdl_launch_dependents();
  run_tasks<kPaged, kPaged, true>(tasks, n_tasks, params, g, n_pools, &pk, nullptr, split);
}

// Inline-descriptor twins of the two hot kernels (KvInlineDesc: parameters, tables
// and tasks in the kernel's parameter space; same PDL protocol as above).
template <int CAP>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_append_scatter_inl_kernel(KvGeomDev g, const __grid_constant__ KvInlineDescT<CAP> d) {
  pdl_launch_dependents();
  run_tasks<kTokMajor, kPaged, false>(reinterpret_cast<const KvTask *>(d.data + d.task_off),
                                      d.n_tasks, d.pools, g, d.n_pools, nullptr, nullptr,
                                      d.split);
  pdl_wait();
}

template <int CAP>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_ring_put_inl_kernel(KvGeomDev g, const __grid_constant__ KvInlineDescT<CAP> d) {
  pdl_wait();
  pdl_launch_dependents();
  run_tasks<kPaged, kPaged, true>(reinterpret_cast<const KvTask *>(d.data + d.task_off),
                                  d.n_tasks, d.pools, g, d.n_pools, nullptr, d.data, d.split);
}

// Split publication (graph loop): the ring-put's copies without the publication pass
// (no per-CTA release RMW, no bar.sync tail), and a separate publication kernel node
// that runs after it -- the kernel boundary orders every copy before the metadata.
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_ring_put_copy_kernel(const KvTask *__restrict__ tasks, int n_tasks,
                            const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools,
                            const __grid_constant__ KvParamPack pk, int split) {
  run_tasks<kPaged, kPaged, false>(tasks, n_tasks, params, g, n_pools, &pk, nullptr, split);
}

// One CTA per pool: the bt entries of its first tasks, its parity table, the task
// counter advanced by its units (kept equal to the host's `issued`), then ONE
// acquire-release fence and the seq store (reading R9).  An aborted launch (target
// all-ones, kv_inject_abort) publishes nothing.
__global__ void __launch_bounds__(kThreads)
    kv_publish_kernel(const KvTask *__restrict__ tasks, int n_tasks,
                      const KvPoolParams *__restrict__ params, KvGeomDev g, int n_pools,
                      const __grid_constant__ KvParamPack pk, int split) {
  (void)g;
  (void)pk;
  const int q = blockIdx.x;
  if (q >= n_pools) return;
  const KvPoolParams &pp = params[q];
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  int32_t *bt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)pp.max_reqs);
  for (int t = threadIdx.x; t < n_tasks; t += blockDim.x) {
    const KvTask tk = tasks[t];
    if (tk.pool != q) continue;
    if ((tk.flags & kFirst) && tk.slot >= 0) bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
    atomicAdd(&s_n, 1);
  }
  write_parity_table(pp, nullptr);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(pp.counter, (unsigned long long)s_n * (unsigned long long)split);
    if (pp.target != ~0ull) {
      const bool sys = pp.sys_scope != 0;
      fence_acquire(sys);
      st_after_fence(reinterpret_cast<unsigned long long *>(pp.meta), pp.step, sys);
    }
  }
}

// Fixed-node graph steps: the launch is described by the step header in the slot.
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_append_scatter_fx_kernel(const char *__restrict__ slot, int i) {
  const KvStepHdr &h = reinterpret_cast<const KvStepHdr *>(slot)[i];
  const int n = h.n_tasks[0];
  if (n <= 0) return;
  run_tasks<kTokMajor, kPaged, false>(reinterpret_cast<const KvTask *>(slot + h.tasks_off[0]), n,
                                      reinterpret_cast<const KvPoolParams *>(slot + h.params_off[0]),
                                      h.g, h.n_pools[0], nullptr, nullptr, h.split[0]);
}

__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_ring_put_copy_fx_kernel(const char *__restrict__ slot, int i) {
  const KvStepHdr &h = reinterpret_cast<const KvStepHdr *>(slot)[i];
  const int n = h.n_tasks[1];
  if (n <= 0) return;
  run_tasks<kPaged, kPaged, false>(reinterpret_cast<const KvTask *>(slot + h.tasks_off[1]), n,
                                   reinterpret_cast<const KvPoolParams *>(slot + h.params_off[1]),
                                   h.g, h.n_pools[1], nullptr, nullptr, h.split[1]);
}

__global__ void __launch_bounds__(kThreads)
    kv_publish_fx_kernel(const char *__restrict__ slot, int i) {
  const KvStepHdr &h = reinterpret_cast<const KvStepHdr *>(slot)[i];
  const int n_tasks = h.n_tasks[1];
  const int q = blockIdx.x;
  if (n_tasks <= 0 || q >= h.n_pools[1]) return;
  const KvTask *tasks = reinterpret_cast<const KvTask *>(slot + h.tasks_off[1]);
  const KvPoolParams &pp = reinterpret_cast<const KvPoolParams *>(slot + h.params_off[1])[q];
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  int32_t *bt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)pp.max_reqs);
  for (int t = threadIdx.x; t < n_tasks; t += blockDim.x) {
    const KvTask tk = tasks[t];
    if (tk.pool != q) continue;
    if ((tk.flags & kFirst) && tk.slot >= 0) bt[(size_t)tk.slot * pp.max_blk + tk.j] = tk.dst_unit;
    atomicAdd(&s_n, 1);
  }
  write_parity_table(pp, nullptr);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(pp.counter, (unsigned long long)s_n * (unsigned long long)h.split[1]);
    if (pp.target != ~0ull) {
      const bool sys = pp.sys_scope != 0;
      fence_acquire(sys);
      st_after_fence(reinterpret_cast<unsigned long long *>(pp.meta), pp.step, sys);
    }
  }
}

// Software-pipelined decode step (kv_run_steps_fused): ONE launch carries the
// append of step k (tasks [0, n_append), pools params[0, n_app_pools)) and the
// publication of step k-1 (tasks [n_append, n_tasks), pools params[n_app_pools..),
// task pool indices local to each part).  The two parts touch disjoint slots
// (positions >= len_{k-1} or blocks quarantined >= 1 step vs dirty positions
// < len_{k-1}, reading R7), so they need no ordering; the task branch is uniform
// per CTA.  The publication pass runs over the ring-put part only.
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_step_fused_kernel(const KvTask *__restrict__ tasks, int n_append, int n_tasks,
                         const KvPoolParams *__restrict__ params, int n_app_pools,
                         KvGeomDev g, int n_rep_pools) {
  const KvPoolParams *rparams = params + n_app_pools;
  for (int t = blockIdx.x; t < n_tasks; t += gridDim.x) {
    const KvTask tk = tasks[t];
    const bool app = t < n_append;
    const KvPoolParams &pp = app ? params[tk.pool] : rparams[tk.pool];
    copy_task_dyn(tk, pp.src, pp.dst, g, app);
  }
  if (n_rep_pools > 0)
    publish_pass(tasks + n_append, n_tasks - n_append, rparams, n_rep_pools, nullptr, 1, n_append);
}

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
    copy_task<kPacked, kPaged>(tk, pp.src, pp.dst, g, ~0ull, ~0ull);
    if (tk.flags & kPoolFirst) write_parity_table(pp, nullptr);
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

}  // namespace

// Resident 256-thread CTAs of the copy kernels (kMinBlocks per SM).
// A launch never exceeds this: extra tasks are taken by grid-stride, so a
// decode-sized step is one wave.  KVRING_CTAS_PER_SM overrides (experiments).
int resident_ctas(int device) {
  static int sms[64] = {0};
  static int per_sm = 0;
  const int d = device < 0 ? 0 : (device & 63);
  if (sms[d] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0)
      v = 148;
    cudaGetLastError();
    sms[d] = v;
  }
  if (per_sm == 0) {
    const char *e = getenv("KVRING_CTAS_PER_SM");
    per_sm = (e && atoi(e) > 0) ? atoi(e) : kMinBlocks;
  }
  return sms[d] * per_sm;
}

int copy_grid(int device, int n_tasks) {
  const int cap = resident_ctas(device);
  return n_tasks < cap ? (n_tasks > 0 ? n_tasks : 1) : cap;
}

void kernel_node_params(int kind, int grid, KvNodeArgs &a, cudaKernelNodeParams &kp) {
  a.ptrs[0] = &a.tasks;
  a.ptrs[1] = &a.n_tasks;
  a.ptrs[2] = &a.params;
  a.ptrs[3] = &a.g;
  a.ptrs[4] = &a.n_pools;
  a.ptrs[5] = &a.pk;
  a.ptrs[6] = &a.split;
  kp.func = kind == kKindAppend ? reinterpret_cast<void *>(kv_append_scatter_kernel)
            : kind == kKindRingPutCopy ? reinterpret_cast<void *>(kv_ring_put_copy_kernel)
            : kind == kKindPublish     ? reinterpret_cast<void *>(kv_publish_kernel)
                                       : reinterpret_cast<void *>(kv_ring_put_kernel);
  kp.gridDim = dim3(grid > 0 ? grid : 1);
  kp.blockDim = dim3(kThreads);
  kp.sharedMemBytes = 0;
  kp.kernelParams = a.ptrs;
  kp.extra = nullptr;
}

void fx_node_params(int kind, int grid, KvFxArgs &a, cudaKernelNodeParams &kp) {
  a.ptrs[0] = &a.slot;
  a.ptrs[1] = &a.step;
  kp.func = kind == kKindAppend        ? reinterpret_cast<void *>(kv_append_scatter_fx_kernel)
            : kind == kKindPublish     ? reinterpret_cast<void *>(kv_publish_fx_kernel)
                                       : reinterpret_cast<void *>(kv_ring_put_copy_fx_kernel);
  kp.gridDim = dim3(grid > 0 ? grid : 1);
  kp.blockDim = dim3(kThreads);
  kp.sharedMemBytes = 0;
  kp.kernelParams = a.ptrs;
  kp.extra = nullptr;
}

cudaError_t launch_copy(int kind, const KvTask *tasks, int n_tasks, const KvPoolParams *params,
                        int n_pools, const KvGeomDev &g, int grid, cudaStream_t stream,
                        const KvPoolParams *host_params, int split) {
  if (n_tasks <= 0) return cudaSuccess;
  if (n_pools > kMaxPoolsPerLaunch) return cudaErrorInvalidValue;
  KvParamPack pk;
  pk.n = 0;
  if (host_params && n_pools <= kInlinePools) {
    pk.n = n_pools;
    for (int i = 0; i < n_pools; ++i) {
      pk.src[i] = host_params[i].src;
      pk.dst[i] = host_params[i].dst;
    }
  }
  switch (kind) {
    case kKindAppend:
      kv_append_scatter_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools,
                                                               pk, split);
      break;
    case kKindRingPut:
      kv_ring_put_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools, pk,
                                                         split);
      break;
    case kKindRestore:
      if (split != 1) return cudaErrorInvalidValue;
      kv_restore_remap_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools);
      break;
    case kKindPack:
      if (split != 1) return cudaErrorInvalidValue;
      kv_gather_pack_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_tasks, params, g, n_pools);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_fused(const KvTask *tasks, int n_append, int n_tasks, const KvPoolParams *params,
                         int n_app_pools, int n_rep_pools, const KvGeomDev &g, int grid,
                         cudaStream_t stream) {
  if (n_tasks <= 0) return cudaSuccess;
  if (n_rep_pools > kMaxPoolsPerLaunch) return cudaErrorInvalidValue;
  kv_step_fused_kernel<<<grid, kThreads, 0, stream>>>(tasks, n_append, n_tasks, params,
                                                       n_app_pools, g, n_rep_pools);
  return cudaGetLastError();
}

cudaError_t launch_copy_inline(int kind, const KvInlineDesc &d, const KvGeomDev &g, int grid,
                               cudaStream_t stream, bool pdl) {
  if (d.n_tasks <= 0) return cudaSuccess;
  if (d.n_pools > kInlinePools) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  // every class is a prefix of the largest (same header, pools and data offset)
#define KV_INL_CLASS(CAP)                                                                 \
  if (d.used <= (CAP)) {                                                                  \
    const auto &ds = *reinterpret_cast<const KvInlineDescT<(CAP)> *>(&d);                 \
    if (kind == kKindAppend)                                                              \
      return cudaLaunchKernelEx(&cfg, kv_append_scatter_inl_kernel<(CAP)>, g, ds);        \
    if (kind == kKindRingPut)                                                             \
      return cudaLaunchKernelEx(&cfg, kv_ring_put_inl_kernel<(CAP)>, g, ds);              \
    return cudaErrorInvalidValue;                                                         \
  }
  KV_INL_CLASS(4 * 1024)
  KV_INL_CLASS(8 * 1024)
  KV_INL_CLASS(16 * 1024)
  KV_INL_CLASS(kInlineBytes)
#undef KV_INL_CLASS
  return cudaErrorInvalidValue;
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

}  // namespace kvring
