// Decode-step engine of libkvring (sm_100a): ONE kernel launch carries
//   - the appends of a step (a2, the harness stand-in for the model's KV write):
//     dense new-token KV -> paged slots, items built by the host allocator; each
//     item also writes its block id into the pool's DEVICE-RESIDENT block table;
//   - and/or the publication of a step to the ring successor (a3 + a4 + a5,
//     P:229 §3.2 "replicate it block-by-block in the background"): the work list
//     is derived ON THE DEVICE from per-slot (req_id, len, pub_len) snapshots and
//     that device block table -- dirty tokens [pub_len, len) of every live slot
//     (completed blocks only in KV_MODE_BLOCKS), split at block boundaries, a
//     prefix sum over slots giving each slot its range of the launch's flat work --
//     then copied with 16-B loads / stores into the successor's replica region at
//     the same block ids (NVLink P2P stores when the successor is a peer), followed
//     by the parity-t (req_id, len) table, the touched bt entries and, from the last
//     CTA, the seq flag (reading R9: one acquire-release fence, system scope for a
//     peer, then the store -- a reader that acquires seq = t sees all of step t).
//
// Balance: the launch's bytes form two flat spaces of 16-B chunks (append and
// replicate); CTA b takes the b-th 1/G share of each, so every CTA moves the same
// bytes whatever the step's mix of prefill, decode and publication (a fused decode
// loop puts append k and the publication of k-1 in one launch; their slots are
// disjoint by reading R7, so they need no ordering inside the kernel).
//
// Pure data movement, HBM / NVLink bound: no tensor cores.  Descriptors (items and
// per-slot tables, <= 24 KiB) travel in the kernel parameter space; each CTA copies
// them to shared memory with warp-uniform loads (the constant bank broadcasts),
// larger launches read a device copy.
#include <cstring>

#include <cuda_runtime.h>

#include "kvring_internal.h"

namespace kvring {

namespace {

constexpr int kThreads = 256;
constexpr int kMinBlocks = 4;
constexpr int kU = 6;  // 16-B chunks in flight per thread (96 KB per SM at 4 CTAs / SM; 56 registers)
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const KvDiv &d) {
  const uint32_t t = __umulhi(d.m, x);
  return (t + ((x - t) >> d.sh1)) >> d.sh2;
}

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

__device__ __forceinline__ unsigned long long atom_add_release_gpu(unsigned long long *p,
                                                                   unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;"
               : "=l"(old)
               : "l"(p), "l"(v)
               : "memory");
  return old;
}

// Shared-memory layout of one CTA: the descriptor blob, then the replicate prefix
// pref[n_ent + 1] (slices) and blk0[n_ent] (block id of each entry's first dirty block).
struct StepSmem {
  const KvAppItem *items;
  const int64_t *req;
  int32_t *hi;   // len snapshot, overwritten with the published length
  const int32_t *lo;
  int32_t *pref;
  int32_t *blk0;
};

__device__ __forceinline__ StepSmem step_smem(const KvStepHdr &h, char *sm) {
  StepSmem s;
  s.items = reinterpret_cast<const KvAppItem *>(sm + h.items_off);
  s.req = reinterpret_cast<const int64_t *>(sm + h.req_off);
  s.hi = reinterpret_cast<int32_t *>(sm + h.len_off);
  s.lo = reinterpret_cast<const int32_t *>(sm + h.pub_off);
  s.pref = reinterpret_cast<int32_t *>(sm + h.data_bytes);
  s.blk0 = s.pref + h.n_ent + 1;
  return s;
}

// Pool of replicate entry e (entries are pool-major).
__device__ __forceinline__ int rep_pool_of(const KvStepHdr &h, int e) {
  int q = 0;
  while (q + 1 < h.n_rep && e >= h.rep[q + 1].ent_off) ++q;
  return q;
}

// Append item walker: slice x (flat, append space) -> source / destination addresses.
struct AppLoc {
  const KvStepHdr &h;
  const KvAppItem *items;
  int i = -1, lo = 0, hi = 0;
  __device__ AppLoc(const KvStepHdr &h_, const KvAppItem *it) : h(h_), items(it) {}
  __device__ __forceinline__ void seek(int x) {
    int a = 0, b = h.n_items - 1;  // last item with off <= x
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (items[m].off <= x) a = m; else b = m - 1;
    }
    i = a;
    lo = items[a].off;
    hi = a + 1 < h.n_items ? items[a + 1].off : h.app_slices;
  }
  __device__ __forceinline__ bool at(int x, const char *&sp, char *&dp) {
    if (i < 0 || x < lo) seek(x);
    while (x >= hi) {
      ++i;
      lo = hi;
      hi = i + 1 < h.n_items ? items[i + 1].off : h.app_slices;
    }
    const KvAppItem &it = items[i];
    const KvStepPool &pp = h.app[it.pool];
    const uint32_t r = (uint32_t)(x - lo);
    const uint32_t t = fdiv(r, h.div_sl);          // token inside the item
    const uint32_t c = r - t * h.div_sl.d;         // (layer, K/V, head)
    const uint32_t j = fdiv((uint32_t)it.p0, h.div_b);
    const uint32_t tok = (uint32_t)it.p0 - j * (uint32_t)h.g.block_size + t;
    sp = pp.src + (long long)(it.row + (int)t) * h.g.token_bytes + (long long)c * h.g.seg_bytes;
    dp = pp.dst + (long long)it.blk * h.g.block_bytes +
         (long long)(c * (uint32_t)h.g.block_size + tok) * h.g.seg_bytes;
    return true;
  }
};

// Replicate entry walker: slice x (flat, replicate space) -> addresses at the same
// block id in this pool and in the successor's replica region (reading R5).
struct RepLoc {
  const KvStepHdr &h;
  const StepSmem &s;
  int e = -1, lo = 0, hi = 0, q = 0, slot = 0, plo = 0;
  int cj = -1, cblk = 0;  // cached (j, block id) of the current entry
  __device__ RepLoc(const KvStepHdr &h_, const StepSmem &s_) : h(h_), s(s_) {}
  __device__ __forceinline__ void enter(int ee) {
    e = ee;
    lo = s.pref[e];
    hi = s.pref[e + 1];
    q = rep_pool_of(h, e);
    slot = e - h.rep[q].ent_off;
    plo = s.lo[e];
    cj = -1;
  }
  __device__ __forceinline__ void seek(int x) {
    int a = 0, b = h.n_ent - 1;  // last entry with pref <= x and a non-empty range
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (s.pref[m] <= x) a = m; else b = m - 1;
    }
    enter(a);
  }
  // false: the chunk is not copied (fault injection cut the pool's step short)
  __device__ __forceinline__ bool at(int x, const char *&sp, char *&dp) {
    if (e < 0 || x < lo) seek(x);
    while (x >= hi) enter(e + 1);
    const KvStepPool &pp = h.rep[q];
    if (h.any_abort && pp.abort_slices >= 0 && x - s.pref[pp.ent_off] >= pp.abort_slices)
      return false;
    const uint32_t r = (uint32_t)(x - lo);
    const uint32_t t = fdiv(r, h.div_sl);
    const uint32_t c = r - t * h.div_sl.d;
    const uint32_t p = (uint32_t)plo + t;           // token position in the request
    const uint32_t j = fdiv(p, h.div_b);
    const uint32_t tok = p - j * (uint32_t)h.g.block_size;
    if ((int)j != cj) {
      cj = (int)j;
      cblk = j == fdiv((uint32_t)plo, h.div_b) ? s.blk0[e] : pp.bt[(size_t)slot * pp.M + j];
    }
    const long long off = (long long)cblk * h.g.block_bytes +
                          (long long)(c * (uint32_t)h.g.block_size + tok) * h.g.seg_bytes;
    sp = pp.src + off;
    dp = pp.dst + off;
    return true;
  }
};

// Copies the chunks [c0, c1) of one flat space: thread t takes chunks c0 + t,
// c0 + t + 256, ... (16 consecutive lanes cover one 256-B slice: coalesced); all
// kU loads of a round are issued before its stores.
template <class Loc>
__device__ __forceinline__ void copy_range(uint32_t c0, uint32_t c1, Loc &loc,
                                           const KvGeomDev &g) {
  const uint32_t cmask = (1u << g.cps_shift) - 1u;
  for (uint32_t base = c0; base < c1; base += (uint32_t)kThreads * kU) {
    uint4 v[kU];
    char *dp[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t y = base + (uint32_t)(u * kThreads) + threadIdx.x;
      dp[u] = nullptr;
      const char *sp;
      char *d;
      if (y < c1 && loc.at((int)(y >> g.cps_shift), sp, d)) {
        const uint32_t lc = (y & cmask) << 4;
        v[u] = ld_stream(sp + lc);
        dp[u] = d + lc;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (dp[u]) st_stream(dp[u], v[u]);
  }
}

// Block-wide exclusive scan of one int per thread; returns the exclusive prefix and
// the total in *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int *total) {
  __shared__ int s_w[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  int wbase = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const int sv = s_w[k];
    if (k < w) wbase += sv;
    tot += sv;
  }
  *total = tot;
  return wbase + x - v;
}

template <bool INL>
__device__ __forceinline__ void step_body(const KvStepHdr &h, const char *__restrict__ data) {
  extern __shared__ __align__(16) char sm[];
  // 1. descriptor blob -> shared memory
  {
    const int n16 = h.data_bytes >> 4;
    if (INL) {
      // parameter space: warp-uniform 16-B loads (constant-bank broadcast)
      const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int k = w; k < n16; k += kWarps) {
        const uint4 x = reinterpret_cast<const uint4 *>(data)[k];
        if (lane == 0) reinterpret_cast<uint4 *>(sm)[k] = x;
      }
    } else {
      for (int k = threadIdx.x; k < n16; k += kThreads)
        reinterpret_cast<uint4 *>(sm)[k] = reinterpret_cast<const uint4 *>(data)[k];
    }
  }
  __syncthreads();
  StepSmem s = step_smem(h, sm);
  const uint32_t SL = h.div_sl.d;
  const int B = h.g.block_size;
  // 2. replicate work list (a3): per-slot dirty slices, prefix sum over slots
  int P = 0;
  if (h.n_rep > 0) {
    const int per = (h.n_ent + kThreads - 1) / kThreads;
    const int e0 = min((int)threadIdx.x * per, h.n_ent), e1 = min(e0 + per, h.n_ent);
    int local = 0;
    int q = e0 < h.n_ent ? rep_pool_of(h, e0) : 0;
    for (int e = e0; e < e1; ++e) {
      while (q + 1 < h.n_rep && e >= h.rep[q + 1].ent_off) ++q;
      const KvStepPool &pp = h.rep[q];
      const int lo = s.lo[e];
      int hi = 0;
      if (s.req[e] >= 0) {
        hi = s.hi[e];
        if (pp.mode == 1) hi = max(lo, hi - hi % B);  // KV_MODE_BLOCKS: completed blocks
      }
      hi = max(hi, lo);
      s.hi[e] = hi;
      const int cnt = (hi - lo) * (int)SL;
      s.pref[e] = cnt;
      local += cnt;
      if (hi > lo) {
        const int slot = e - pp.ent_off;
        s.blk0[e] = pp.bt[(size_t)slot * pp.M + (lo / B)];
      }
    }
    int total;
    int base = block_exclusive_scan(local, &total);
    for (int e = e0; e < e1; ++e) {
      const int c = s.pref[e];
      s.pref[e] = base;
      base += c;
    }
    if (threadIdx.x == 0) s.pref[h.n_ent] = total;
    P = total;
    __syncthreads();
  }
  // 3. copies: this CTA's share of each flat space
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const int cs = h.g.cps_shift;
  if (h.n_items > 0) {
    const unsigned long long T = (unsigned long long)h.app_slices << cs;
    AppLoc loc(h, s.items);
    copy_range((uint32_t)(T * b / G), (uint32_t)(T * (b + 1) / G), loc, h.g);
  }
  if (P > 0) {
    const unsigned long long T = (unsigned long long)P << cs;
    RepLoc loc(h, s);
    copy_range((uint32_t)(T * b / G), (uint32_t)(T * (b + 1) / G), loc, h.g);
  }
  // 4. tables: the appended items' device bt entries; the publication's parity
  //    (req_id, len) table and the bt entries of the blocks it touched.  Readers trust
  //    none of it before seq = step (written below, after every CTA's release).
  const uint32_t gt = b * kThreads + threadIdx.x, stride = G * kThreads;
  for (uint32_t i = gt; i < (uint32_t)h.n_items; i += stride) {
    const KvAppItem &it = s.items[i];
    const KvStepPool &pp = h.app[it.pool];
    pp.bt[(size_t)it.slot * pp.M + fdiv((uint32_t)it.p0, h.div_b)] = it.blk;
  }
  if (h.publish) {
    for (int q = 0; q < h.n_rep; ++q) {
      const KvStepPool &pp = h.rep[q];
      if (pp.abort_slices >= 0) continue;  // aborted: nothing of this step is published
      const int R = pp.R, par = (int)(pp.step & 1ull);
      int64_t *mreq = reinterpret_cast<int64_t *>(pp.meta + 32) + (size_t)par * R;
      int32_t *mlen = reinterpret_cast<int32_t *>(pp.meta + 32 + 16 * (size_t)R) + (size_t)par * R;
      int32_t *mbt = reinterpret_cast<int32_t *>(pp.meta + 32 + 24 * (size_t)R);
      for (uint32_t sl = gt; sl < (uint32_t)R; sl += stride) {
        if ((int)sl < pp.n_slots) {
          const int e = pp.ent_off + (int)sl;
          const int lo = s.lo[e], hi = s.hi[e];
          mreq[sl] = hi > 0 ? s.req[e] : -1;
          mlen[sl] = hi;
          if (hi > lo)
            for (int j = lo / B; j * B < hi; ++j)
              mbt[(size_t)sl * pp.M + j] = j == lo / B ? s.blk0[e] : pp.bt[(size_t)sl * pp.M + j];
        } else {
          mreq[sl] = -1;
          mlen[sl] = 0;
        }
      }
      if (gt == 0) *reinterpret_cast<int32_t *>(pp.meta + 8) = pp.writer_node;
    }
  }
  // 5. completion: bar.sync + one release RMW per CTA; the last CTA issues one
  //    acquire-release fence (system scope if a successor is a peer) and stores every
  //    publishing pool's seq (release pattern), then rearms the counter.
  if (h.publish) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long old = atom_add_release_gpu(h.counter, 1ull);
      if (old == (unsigned long long)G - 1ull) {
        if (h.sys_any)
          asm volatile("fence.acq_rel.sys;" ::: "memory");
        else
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int q = 0; q < h.n_rep; ++q) {
          const KvStepPool &pp = h.rep[q];
          if (pp.abort_slices >= 0) continue;
          unsigned long long *seq = reinterpret_cast<unsigned long long *>(pp.meta);
          if (pp.sys)
            asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(seq), "l"(pp.step) : "memory");
          else
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(seq), "l"(pp.step) : "memory");
        }
        *h.counter = 0ull;  // the next launch on this counter is stream-ordered after this one
      }
    }
  }
}

}  // namespace

// Descriptors in the kernel parameter space (<= kStepInline bytes of data).
template <int CAP>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_step_inl_kernel(const __grid_constant__ KvStepInlT<CAP> d) {
  step_body<true>(d.h, d.data);
}

// Larger launches: the blob is a device copy (staged H2D by the host).
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_step_kernel(const __grid_constant__ KvStepHdr h, const char *__restrict__ gdata) {
  step_body<false>(h, gdata);
}

const void *step_kernel_fn() { return reinterpret_cast<const void *>(kv_step_kernel); }

int step_smem_bytes(const KvStepHdr &h) {
  return h.data_bytes + 4 * (2 * h.n_ent + 1) + 16;
}

namespace {
template <int CAP>
cudaError_t launch_inl(const KvStepHdr &h, const char *host_data, int grid, int smem,
                       cudaStream_t st) {
  static thread_local KvStepInlT<CAP> d;  // argument block (copied by the launch)
  d.h = h;
  memcpy(d.data, host_data, (size_t)h.data_bytes);
  kv_step_inl_kernel<CAP><<<grid, kThreads, smem, st>>>(d);
  return cudaGetLastError();
}

bool g_attr_set = false;
}  // namespace

cudaError_t launch_step(const KvStepHdr &h, const char *host_data, const char *gdata, int grid,
                        cudaStream_t st) {
  const int smem = step_smem_bytes(h);
  if (!g_attr_set) {
    // staged launches may carry up to ~200 KiB of descriptors in shared memory
    cudaFuncSetAttribute(kv_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    g_attr_set = true;
  }
  if (gdata == nullptr) {
    if (h.data_bytes <= 4096) return launch_inl<4096>(h, host_data, grid, smem, st);
    if (h.data_bytes <= 8192) return launch_inl<8192>(h, host_data, grid, smem, st);
    if (h.data_bytes <= 16384) return launch_inl<16384>(h, host_data, grid, smem, st);
    if (h.data_bytes <= kStepInline) return launch_inl<kStepInline>(h, host_data, grid, smem, st);
    return cudaErrorInvalidValue;
  }
  kv_step_kernel<<<grid, kThreads, smem, st>>>(h, gdata);
  return cudaGetLastError();
}

}  // namespace kvring
