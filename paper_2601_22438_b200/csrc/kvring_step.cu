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
// Pure data movement, HBM / NVLink bound: no tensor cores.  The per-launch header
// (pool bases, step, divisors) travels in the kernel parameter space; the descriptor
// blob (items and per-slot tables) is written by the host into pinned memory, pulled
// across PCIe once by the first copying CTA and shared with the other CTAs through device
// memory and a release/acquire flag -- the per-step host cost is one launch.
#include <cstdio>
#include <cstring>

#include <cuda_runtime.h>

#include "kvring_internal.h"

namespace kvring {

namespace {

// A bounded wait that ran out (a launch never completed: a bug, not a slow GPU) traps.
// Debug builds (-DKV_TRAP_PRINT) say which wait first.
#ifdef KV_TRAP_PRINT
#define KV_TRAP(what, a, b)                                                            \
  do {                                                                                 \
    printf("kv_step_kernel trap: %s block %d thread %d: %llu vs %llu\n", what,        \
           (int)blockIdx.x, (int)threadIdx.x, (unsigned long long)(a),                 \
           (unsigned long long)(b));                                                   \
    __trap();                                                                          \
  } while (0)
#else
#define KV_TRAP(what, a, b) __trap()
#endif

constexpr int kThreads = 256;
// 4 resident 256-thread CTAs per SM (32 warps: the address arithmetic of one warp hides
// behind the others) with 8 independent 16-B loads in flight per thread (<= 64
// registers): 128 KB in flight per SM; a decode step's share of a lane (~7 chunks at C2)
// is one round of loads.
constexpr int kMinBlocks = 4;
constexpr int kU = 8;  // 6: -4 % per step; 10: spills, -33 % (profiles/r02/ab/ku_n1.log)
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const KvDiv &d) {
  const uint32_t t = __umulhi(d.m, x);
  return (t + ((x - t) >> d.sh1)) >> d.sh2;
}

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): the tokens an append
// writes into the pool are read again by the next launch's publication, so they are
// stored evict_last; everything else is touched once (dense sources, the publication's
// reads, the replica writes: evict_first).  The 126 MB L2 then keeps a step's appended
// tokens (~30 MB at C2) for the publication that follows: 1 GPU +5.5 % per step (0.70 ->
// 0.74 of the HBM roof over the bench's window), 2 GPUs +1.5 % (profiles/r02/ab).
__device__ __forceinline__ uint4 ld_hint(const void *p, unsigned long long pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_hint(void *p, const uint4 &v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ unsigned long long policy_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long policy_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long *p,
                                                               unsigned long long v, bool sys) {
  unsigned long long old;
  if (sys)
    asm volatile("atom.add.release.sys.global.u64 %0, [%1], %2;"
                 : "=l"(old)
                 : "l"(p), "l"(v)
                 : "memory");
  else
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
  int32_t *bpref;  // prefix over entries of the blocks each publication touches
};

__device__ __forceinline__ StepSmem step_smem(const KvStepHdr &h, char *sm) {
  StepSmem s;
  s.items = reinterpret_cast<const KvAppItem *>(sm + h.items_off);
  s.req = reinterpret_cast<const int64_t *>(sm + h.req_off);
  s.hi = reinterpret_cast<int32_t *>(sm + h.len_off);
  s.lo = reinterpret_cast<const int32_t *>(sm + h.pub_off);
  s.pref = reinterpret_cast<int32_t *>(sm + h.data_bytes);
  s.blk0 = reinterpret_cast<int32_t *>(sm + h.blk0_off);
  s.bpref = s.pref + h.n_ent + 1;
  return s;
}

// Pool of replicate entry e (entries are pool-major).
__device__ __forceinline__ int rep_pool_of(const KvStepHdr &h, int e) {
  int q = 0;
  while (q + 1 < h.n_rep && e >= h.rep[q + 1].ent_off) ++q;
  return q;
}

// q / n for a small divisor n and q < 2^24: float reciprocal estimate, then an exact
// integer correction (the estimate is within one of the quotient).
__device__ __forceinline__ uint32_t div_small(uint32_t q, uint32_t n, float rn) {
  uint32_t d = (uint32_t)((float)q * rn);
  if (d * n > q) --d;
  if ((d + 1) * n <= q) ++d;
  return d;
}

// Work cursor over the launch's ONE flat space of slices: [0, A) are the append
// items' slices, [A, A + P) the publication's.  A warp round moves kU consecutive warp
// iterations; lane l handles 16-B chunk (l mod cps) of slice x + l / cps and each
// iteration advances every lane by d = 32 / cps slices (16 lanes per 256-B slice:
// coalesced).  Appends and publication share the space, so a lane issues its loads of
// both in the same rounds (a decode step is one round of loads in flight per lane).
//
// Inside a piece (an append item, or one block of a publication entry) a slice is an
// (inner, outer) pair; source offset = inner * s_in + outer * s_out, destination offset
// = inner * d_in + outer * d_out, inner runs fastest:
//   append  (token-major: the dense source row is read contiguously)
//           inner = (layer, K/V, head) c < SL, outer = token t:
//           src = row base + t * token_bytes + c * seg; dst = block + (c * B + t0 + t) * seg
//   publish ((layer, K/V, head)-major within a block piece of n tokens: a full block is
//           ONE contiguous run, read from this pool and written at the same offsets of
//           the successor's replica region, reading R5)
//           inner = token t < n, outer = combo c: off = block + (c * B + t0 + t) * seg
// so stepping d slices is pointer += d * stride plus a rare carry; only a piece boundary
// (or the round's end, or a fault-injection cut) starts a new sub-round with a locate.
// blk0 word of a publication entry: block id | kBlkGated when one of the entry's blocks
// with no previously published token was freed one step ago (deferred publication)
constexpr int kBlkGated = 1 << 30;
constexpr int kBlkMask = kBlkGated - 1;

struct Cursor {
  const KvStepHdr &h;
  const StepSmem &s;
  const char *sp = nullptr;   // current slice's source address
  char *dp = nullptr;         // current slice's destination address
  uint32_t in = 0, nin = 1;
  int ds_in = 0, dd_in = 0;   // d * s_in, d * d_in
  int s_wrap = 0, d_wrap = 0; // s_out - nin * s_in, d_out - nin * d_in
  int idx = -1;               // item / entry of the current piece
  int pb = -1;                // end of the piece (flat slice)
  int lim = 0x7fffffff;       // publication cut short by fault injection (flat slice)
  bool in_rep = false;        // idx is a publication entry
  bool gated = false;         // the piece's block holds no previously published token and
                              // the entry's new blocks include one freed one step ago
  bool agated = false;        // append item into a block freed one step ago (kItemGated)
  __device__ Cursor(const KvStepHdr &h_, const StepSmem &s_) : h(h_), s(s_) {}

  __device__ __forceinline__ void locate(int x, uint32_t d) {
    uint32_t out, s_in, s_out, d_in, d_out;
    const uint32_t B = (uint32_t)h.g.block_size, seg = (uint32_t)h.g.seg_bytes;
    if (x < h.app_slices) {
      const KvAppItem *items = s.items;
      int a = !in_rep && idx >= 0 && items[idx].off <= x ? idx : 0, b = h.n_items - 1;
      while (a < b) {                  // last item with off <= x
        const int m = (a + b + 1) >> 1;
        if (items[m].off <= x) a = m; else b = m - 1;
      }
      idx = a;
      in_rep = false;
      gated = false;
      const KvAppItem &it = items[a];
      agated = (it.blk & kItemGated) != 0;
      pb = a + 1 < h.n_items ? items[a + 1].off : h.app_slices;
      lim = 0x7fffffff;
      const uint32_t r = (uint32_t)(x - it.off);
      out = fdiv(r, h.div_sl);
      in = r - out * h.div_sl.d;
      nin = h.div_sl.d;
      const KvStepPool &pp = h.app[it.pool];
      const uint32_t j = fdiv((uint32_t)it.p0, h.div_b);
      s_in = seg;
      s_out = (uint32_t)h.g.token_bytes;
      d_in = B * seg;
      d_out = seg;
      sp = pp.src + (long long)it.row * h.g.token_bytes + (long long)(in * s_in) +
           (long long)out * s_out;
      dp = pp.dst + (long long)(it.blk & kItemBlkMask) * h.g.block_bytes +
           (long long)(it.p0 - j * B) * seg + (long long)(in * d_in) + (long long)out * d_out;
    } else {
      const int xr = x - h.app_slices;
      if (!in_rep || xr < s.pref[idx] || xr >= s.pref[idx + 1]) {
        int a = in_rep && xr >= s.pref[idx] ? idx : 0, b = h.n_ent - 1;
        while (a < b) {                // last entry with pref <= xr
          const int m = (a + b + 1) >> 1;
          if (s.pref[m] <= xr) a = m; else b = m - 1;
        }
        idx = a;
        in_rep = true;
      }
      agated = false;
      const int e = idx;
      const int q = rep_pool_of(h, e);
      const KvStepPool &pp = h.rep[q];
      const int slot = e - pp.ent_off;
      lim = (h.any_abort && pp.abort_slices >= 0)
                ? h.app_slices + s.pref[pp.ent_off] + pp.abort_slices : 0x7fffffff;
      const uint32_t SL = h.div_sl.d;
      const uint32_t plo = (uint32_t)s.lo[e], phi = (uint32_t)s.hi[e];
      const uint32_t j0 = fdiv(plo, h.div_b), t0 = plo - j0 * B;
      const uint32_t n0 = min(B - t0, phi - plo);
      const uint32_t r = (uint32_t)(xr - s.pref[e]);
      uint32_t j, tok0, rr, pa;
      gated = true;
      if (r < n0 * SL) {               // the entry's first (possibly partial) block
        j = j0;
        nin = n0;
        tok0 = t0;
        rr = r;
        pa = 0;
        gated = t0 == 0;
      } else {                         // full blocks, the last one possibly partial
        const uint32_t r2 = r - n0 * SL;
        const uint32_t jj = fdiv(r2, h.div_bs);
        j = j0 + 1 + jj;
        nin = min(B, phi - j * B);
        tok0 = 0;
        rr = r2 - jj * h.div_bs.d;
        pa = n0 * SL + jj * h.div_bs.d;
      }
      pb = h.app_slices + s.pref[e] + (int)(pa + nin * SL);
      out = div_small(rr, nin, __frcp_rn((float)nin));
      in = rr - out * nin;
      const int b0w = s.blk0[e];
      const int blk = j == j0 ? (b0w & kBlkMask) : pp.bt[(size_t)slot * pp.M + j];
      gated = gated && (b0w & kBlkGated);
      const long long off = (long long)blk * h.g.block_bytes + (long long)tok0 * seg +
                            (long long)in * seg + (long long)out * (B * seg);
      s_in = d_in = seg;
      s_out = d_out = B * seg;
      sp = pp.src + off;
      dp = pp.dst + off;
    }
    ds_in = (int)(d * s_in);
    dd_in = (int)(d * d_in);
    s_wrap = (int)s_out - (int)(nin * s_in);
    d_wrap = (int)d_out - (int)(nin * d_in);
  }

  __device__ __forceinline__ void carry_src() {
    while (in >= nin) {
      in -= nin;
      sp += s_wrap;
    }
  }
};

// Copies the flat space [0, T) with every warp of the grid: rounds of kU warp
// iterations (32 x kU chunks of consecutive slices: 4 KiB at 256-B slices) are dealt
// grid-stride, so the whole grid works inside one window of ~(warps x 4 KiB) at a time.
// A lane locates its piece once per (sub-)round and then only adds strides; a round is
// split where a lane's slices leave the piece (rare: pieces are >= 128 slices at C2).
// All loads of a (sub-)round are issued before its stores; the stores replay the
// destination stepping instead of keeping kU pointers live.
//
// Rounds [0, st * W) are dealt statically (round r to warp r mod W); the rest are
// handed out dynamically through kWorkCtrs counters (warp w draws from counter w mod
// kWorkCtrs the rounds st*W + c, st*W + c + kWorkCtrs, ...): SMs do not all move bytes
// at the same rate (GPCs differ in SM count, the two dies), so a static split leaves
// the slowest warps finishing alone.  st = 3/4 of the rounds per warp (at least 1):
// a decode step (fewer rounds than warps) never touches the counters.
constexpr int kWorkCtrs = 8;
constexpr int kBlobBatch = 8;  // descriptor loads in flight per thread
constexpr int kWorkStride = 16;  // u32 words between counters (64 B)

// Waits (one thread) until the launch's publisher CTA opened the gate (deferred
// publication, kvring_internal.h); bounded: a trap beats a hang.
__device__ __forceinline__ void wait_gate(const KvStepHdr &h) {
  unsigned long long v;
  for (long long spin = 0;; ++spin) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(h.gate) : "memory");
    if (v == h.nonce) break;
    if (spin > (1ll << 24)) KV_TRAP("gate", v, h.nonce);
    if (spin > 16) __nanosleep(64);
  }
}

// Waits (one thread) until a launch's completion counter reached `target` (bounded).
__device__ __forceinline__ void wait_count(const unsigned long long *c, unsigned long long target) {
  unsigned long long v;
  for (long long spin = 0;; ++spin) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
    if (v >= target) break;
    if (spin > (1ll << 24)) KV_TRAP("count", v, target);  // that launch never completed
    if (spin > 64) __nanosleep(32);
  }
}

// A warp of an early-started launch that has not yet seen the previous launch arrive
// (wait_prev) acquires its arrival count before the loads of a publication round or of an
// append item into a block freed one step ago.
__device__ __forceinline__ void warp_wait_prev(const KvStepHdr &h, int lane, bool &wait_prev) {
  if (lane == 0) wait_count(h.prev_counter, h.prev_target);
  __syncwarp();
  wait_prev = false;
}

__device__ __forceinline__ void copy_round(int base, int rend, int lane, int cs, uint32_t d,
                                           uint32_t lc, Cursor &cur, bool &gate_shut,
                                           bool pub_round, bool &wait_prev) {
  if (wait_prev && pub_round) warp_wait_prev(cur.h, lane, wait_prev);
  {
    int x = base + (lane >> cs);                // this lane's slice
    while (__any_sync(0xffffffffu, x < rend)) {
      int n = 0;
      if (x < rend) {
        cur.locate(x, d);
        const bool skip = x >= cur.lim;
        const int end = min(min(rend, cur.pb), skip ? cur.pb : cur.lim);
        n = min(kU, (end - x + (int)d - 1) / (int)d);
        if (skip) {                             // fault injection: this stretch is not copied
          x += n * (int)d;
          n = 0;
        }
      }
      if (wait_prev && __any_sync(0xffffffffu, n > 0 && cur.agated))
        warp_wait_prev(cur.h, lane, wait_prev);
      char *const dp0 = cur.dp;
      const uint32_t in0 = cur.in;
      uint4 v[kU];
      const unsigned long long pol_ld = policy_first();
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (u < n) {
          v[u] = ld_hint(cur.sp + lc, pol_ld);
          cur.sp += cur.ds_in;
          cur.in += d;
          cur.carry_src();
        }
      }
      // stores into a block that the last stored seq may still list as another
      // request's wait for the previous publication's seq (deferred publication)
      if (gate_shut && __any_sync(0xffffffffu, n > 0 && cur.gated)) {
        if (lane == 0) wait_gate(cur.h);
        __syncwarp();
        gate_shut = false;
      }
      char *dq = dp0;
      uint32_t in = in0;
      const unsigned long long pol_st = pub_round ? policy_first() : policy_last();
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (u < n) {
          st_hint(dq + lc, v[u], pol_st);
          dq += cur.dd_in;
          in += d;
          while (in >= cur.nin) {
            in -= cur.nin;
            dq += cur.d_wrap;
          }
        }
      }
      x += n * (int)d;
    }
  }
}

//
// Round order.  Over NVLink (h.app_first = 0) append rounds and publication rounds are
// interleaved in proportion (round r is a publication round iff floor((r+1) f) >
// floor(r f), f = Rp / R in 32.32 fixed point, rounded up so that exactly Rp of the R
// rounds are): the publication's peer stores then run all through the launch instead of
// waiting for the appends (2 GPUs: +7 % per step, and 0.68 vs 0.65 of NVLink against
// appends first with the early start, 0.66 with the publication's rounds first).  In one
// GPU's HBM (app_first = 1) the append rounds come first: with the early start
// (wait_prev) the warps that become resident
// while the previous launch drains take append rounds, which need nothing from it
// (+1.5 % per step against interleaved, which loses 2 %: its early warps stall on the
// previous launch's arrival before their publication rounds).
__device__ __forceinline__ void copy_all(int A, int P, int G, int b, Cursor &cur,
                                         const KvGeomDev &g, unsigned int *work, bool wait_prev,
                                         bool app_first) {
  const int lane = threadIdx.x & 31;
  const int gw = b * kWarps + (int)(threadIdx.x >> 5);
  const int W = G * kWarps;
  const int cs = g.cps_shift;
  const uint32_t d = 32u >> cs;                 // slices per warp iteration
  const int span = (int)d * kU;                 // slices per warp round
  const uint32_t lc = ((uint32_t)lane & ((1u << cs) - 1u)) << 4;
  const int Ra = (A + span - 1) / span, Rp = (P + span - 1) / span;
  const int R = Ra + Rp;
  const unsigned long long f =
      Ra == 0 ? (1ull << 32) : (((unsigned long long)Rp << 32) + (unsigned long long)R - 1) / R;
#ifdef KV_AB_STATIC  // A/B builds (tools/ab_bench.sh): every round dealt statically
  const int st = R;
#elif defined(KV_AB_DYN4)
  const int st = R / W >= 4 ? (R / W) * 3 / 4 : R;
#else
  const int st = max(1, (R / W) * 3 / 4);
#endif
  const int Rs = (int)min((long long)R, (long long)st * W);
  const int c = gw % kWorkCtrs;
  unsigned int *const ctr = work + c * kWorkStride;
  // one call site for both phases (two inlined copies of the round spill registers); the
  // draw of the next dynamic round is issued before the current round's copies, so its
  // latency hides behind them
  unsigned int next = 0;
  bool drawn = false;                           // `next` holds a draw (warp-uniform)
  bool gate_shut = cur.h.n_prev > 0;            // warp-uniform
  for (int r = gw;;) {
    if (r >= Rs) {                              // static share done: take a drawn round
      if (Rs >= R) break;
      if (!drawn && lane == 0) next = atomicAdd(ctr, 1u);
      const unsigned int k = __shfl_sync(0xffffffffu, next, 0);
      drawn = false;
      const long long rd = (long long)Rs + c + (long long)k * kWorkCtrs;
      if (rd >= R) break;
      r = (int)rd;
    }
    if (Rs < R && (r >= Rs || r + W >= Rs)) {   // the next round is dynamic: draw it now
      if (lane == 0) next = atomicAdd(ctr, 1u);
      drawn = true;
    }
    int b0, b1;
    bool pub;
    if (app_first) {                            // append rounds first, then the publication's
      pub = r >= Ra;
      b0 = pub ? A + (r - Ra) * span : r * span;
    } else {
      const unsigned int pr = (unsigned int)(((unsigned long long)r * f) >> 32);
      pub = (unsigned int)(((unsigned long long)(r + 1) * f) >> 32) > pr;
      b0 = pub ? A + (int)pr * span : (r - (int)pr) * span;  // publication round pr / append r - pr
    }
    b1 = pub ? min(A + P, b0 + span) : min(A, b0 + span);
    copy_round(b0, b1, lane, cs, d, lc, cur, gate_shut, pub, wait_prev);
    r = r < Rs ? r + W : 0x7fffffff;
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

#ifdef KV_TIMELINE
// Debug builds (-DKV_TIMELINE, tools/step_timeline.py): thread 0 of every CTA stamps
// %globaltimer at each phase boundary of the latest launch.
__device__ unsigned long long g_kv_timeline[32 * 1024 * 8];  // the last 32 launches
#define KV_STAMP(k)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                      \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_kv_timeline[((unsigned)h.pad0 & 31u) * 8192 + blockIdx.x * 8 + (k)] = t_;     \
    }                                                                                 \
  } while (0)
#else
#define KV_STAMP(k) \
  do {              \
  } while (0)
#endif

// Completion (step 5 of step_body; also the publisher CTA's arrival).
__device__ __forceinline__ void step_complete(const KvStepHdr &h) {
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef KV_AB_GPU_RELEASE  // A/B builds only: unsafe for remote readers (bound on the gain)
    const bool sys_rel = false;
#else
    // a deferred launch does not wait for its peer stores here: the next launch's
    // publisher waits for this grid to complete before it stores the seqs
    const bool sys_rel = h.sys_any != 0 && !h.defer;
#endif
    const unsigned long long old = atom_add_release(h.counter, 1ull, sys_rel);
    if (old + 1ull == h.target) {
      if (sys_rel)
        asm volatile("fence.acq_rel.sys;" ::: "memory");
      else
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      // this launch's seqs, and its final count, follow the previous launch's (same
      // seq locations; the next launch's seqs follow ours through our final count)
      if (h.chain) {
        unsigned long long v;
        for (long long spin = 0;; ++spin) {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(h.prev_counter) : "memory");
          if (v > h.prev_target) break;
          if (spin > (1ll << 24)) KV_TRAP("prev final", v, h.prev_target);
        }
      }
      if (h.publish && !h.defer)
        for (int q = 0; q < h.n_rep; ++q) {
          const KvStepPool &pp = h.rep[q];
          if (pp.abort_slices >= 0) continue;
          unsigned long long *seq = reinterpret_cast<unsigned long long *>(pp.meta);
          if (pp.sys)
            asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(seq), "l"(pp.step) : "memory");
          else
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(seq), "l"(pp.step) : "memory");
        }
      // the dynamic round counters are free again (every warp drew its last round)
      for (int c = 0; c < kWorkCtrs; ++c) h.work[c * kWorkStride] = 0u;
      // final count: the next chained launch acquires it (its seq stores follow these)
      atom_add_release(h.counter, 1ull, sys_rel);
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(h.done), "l"(h.nonce) : "memory");
    }
  }
}

__device__ __forceinline__ void step_body(const KvStepHdr &h) {
  extern __shared__ __align__(16) char sm[];
  KV_STAMP(0);
#ifdef KV_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x < 1024)
    g_kv_timeline[((unsigned)h.pad0 & 31u) * 8192 + blockIdx.x * 8 + 7] = (unsigned)h.pad0;
#endif
  // programmatic dependent launch: the next step's grid may start its prologue as soon
  // as this grid's CTAs leave (a no-op for a normally serialised launch)
  if (h.pdl) asm volatile("griddepcontrol.launch_dependents;" :::);
  // the publisher CTA of a launch following a deferred one (kvring_internal.h) is CTA 0
  // (CTA 1 pulls the descriptor): wait for that launch to complete -- every one of its
  // stores, peer stores included, performed -- then store its seqs and open the gate; it
  // moves no data and arrives like the others.  CTA 0 is dispatched first, so the copying
  // CTAs that spin on the gate never hold the slot it needs (as the last CTA it could find
  // every slot taken by them: a 2-GPU bench trapped in that wait 3 times in 5)
  if (h.n_prev > 0 && blockIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int q = 0; q < h.n_prev; ++q) {
        if ((h.prev_sys >> q) & 1)
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(h.prev_seq[q]), "l"(h.prev_step[q]) : "memory");
        else
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(h.prev_seq[q]), "l"(h.prev_step[q]) : "memory");
      }
      // the seqs are stored (system scope): stores that the old seqs forbade may go
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(h.gate), "l"(h.nonce) : "memory");
    }
    step_complete(h);
    return;
  }
  // 1. descriptor blob -> shared memory.  The host writes it into pinned host memory and
  //    launches -- no copy-engine call and no event per step.  The first copying CTA (CTA
  //    0, or CTA 1 behind a publisher CTA) pulls it across PCIe once (zero copy) into a
  //    device buffer and releases a per-buffer flag carrying the launch nonce; every other
  //    CTA acquires the flag (bounded wait: a timeout traps) and copies the buffer from
  //    L2.  (The puller is dispatched before the CTAs that wait for it and waits for none
  //    of them.)
  {
    const int n16 = h.data_bytes >> 4;
    uint4 *smv = reinterpret_cast<uint4 *>(sm);
    if (blockIdx.x == (h.n_prev > 0 ? 1u : 0u)) {  // the puller: the first copying CTA
      const uint4 *src = reinterpret_cast<const uint4 *>(h.hblob);
      uint4 *dst = reinterpret_cast<uint4 *>(h.gblob);
      // kBlobBatch loads in flight per thread before any store: one PCIe round trip per
      // 32 KiB instead of one per 4 KiB
      for (int k0 = 0; k0 < n16; k0 += kThreads * kBlobBatch) {
        uint4 x[kBlobBatch];
#pragma unroll
        for (int u = 0; u < kBlobBatch; ++u) {
          const int k = k0 + u * kThreads + (int)threadIdx.x;
          if (k < n16)
            asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w)
                         : "l"(src + k));
        }
#pragma unroll
        for (int u = 0; u < kBlobBatch; ++u) {
          const int k = k0 + u * kThreads + (int)threadIdx.x;
          if (k < n16) {
            smv[k] = x[u];
            asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + k), "r"(x[u].x),
                         "r"(x[u].y), "r"(x[u].z), "r"(x[u].w) : "memory");
          }
        }
      }
      __syncthreads();  // every thread's stores precede the single release below
      if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(h.flag), "l"(h.nonce) : "memory");
    } else {
      if (threadIdx.x == 0) {
        unsigned long long v;
        for (long long spin = 0;; ++spin) {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(h.flag) : "memory");
          if (v == h.nonce) break;
          if (spin > (1ll << 22)) KV_TRAP("blob flag", v, h.nonce);  // CTA 0 never published it
          __nanosleep(64);
        }
      }
      __syncthreads();
      const uint4 *gsrc = reinterpret_cast<const uint4 *>(h.gblob);
      for (int k0 = 0; k0 < n16; k0 += kThreads * kBlobBatch) {
        uint4 x[kBlobBatch];
#pragma unroll
        for (int u = 0; u < kBlobBatch; ++u) {
          const int k = k0 + u * kThreads + (int)threadIdx.x;
          if (k < n16)
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w)
                         : "l"(gsrc + k));
        }
#pragma unroll
        for (int u = 0; u < kBlobBatch; ++u) {
          const int k = k0 + u * kThreads + (int)threadIdx.x;
          if (k < n16) smv[k] = x[u];
        }
      }
    }
  }
  __syncthreads();
  KV_STAMP(1);
  StepSmem s = step_smem(h, sm);
  const uint32_t SL = h.div_sl.d;
  const int B = h.g.block_size;
  // 2. replicate work list (a3): per-slot dirty slices, prefix sum over slots
  int P = 0;
  if (h.n_rep > 0) {
    const int per = (h.n_ent + kThreads - 1) / kThreads;
    const int e0 = min((int)threadIdx.x * per, h.n_ent), e1 = min(e0 + per, h.n_ent);
    int local = 0, blocal = 0;
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
      const int nb = hi > lo ? (hi + B - 1) / B - lo / B : 0;  // blocks touched (bt entries)
      s.bpref[e] = nb;
      blocal += nb;
    }
    int total, btotal;
    int base = block_exclusive_scan(local, &total);
    __syncthreads();  // the scan's shared scratch is reused below
    int bbase = block_exclusive_scan(blocal, &btotal);
    for (int e = e0; e < e1; ++e) {
      const int c = s.pref[e];
      s.pref[e] = base;
      base += c;
      const int cb = s.bpref[e];
      s.bpref[e] = bbase;
      bbase += cb;
    }
    if (threadIdx.x == 0) {
      s.pref[h.n_ent] = total;
      s.bpref[h.n_ent] = btotal;
    }
    P = total;
    __syncthreads();
  }
  // every read below may touch data the previous step's grid wrote (its appends, its
  // device block-table entries, its seq): wait for it.  A chained launch (the previous
  // kernel on the stream is this library's previous step launch, nothing else between)
  // acquires that launch's arrival count -- reached once every CTA's data is complete
  // (each CTA arrives with a release) -- which returns ~3 us before griddepcontrol.wait
  // would (that waits for the whole grid to retire and flush); only this launch's seq
  // stores also wait for the previous launch's seqs (its final count, step_complete).  No deadlock: a programmatic
  // dependent grid starts only after every CTA of the previous grid has started.
  //
  // Early start (h.early: the previous launch was chained too, so the one before it is
  // this library's launch as well): only that launch's arrival is awaited here -- the
  // previous launch may still be copying.  Appends of this step touch neither its
  // publication's reads (blocks of requests live when it was snapshotted: a block freed
  // since then is flagged kItemGated and waited for) nor its appends (other tokens /
  // blocks); so the append rounds start at once and fill the previous grid's tail, and a
  // warp acquires the previous arrival count only before its first publication round or
  // gated item (copy_round); every CTA does before its tables.
#ifdef KV_AB_NOEARLY
  const bool early = false;
#else
  const bool early = h.chain && h.early;
#endif
  if (early) {
    if (threadIdx.x == 0) wait_count(h.pp_counter, h.pp_target);
    __syncthreads();
  } else if (h.chain) {
    if (threadIdx.x == 0) wait_count(h.prev_counter, h.prev_target);
    __syncthreads();
  } else if (h.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  // 3. copies: the grid's flat space, dealt in warp rounds
  KV_STAMP(2);
  const uint32_t G = gridDim.x - (h.n_prev > 0 ? 1u : 0u);      // copying CTAs
  const uint32_t b = blockIdx.x - (h.n_prev > 0 ? 1u : 0u);       // this one's index
  {
    Cursor cur(h, s);
    copy_all(h.app_slices, P, (int)G, (int)b, cur, h.g, h.work, early, h.app_first != 0);
  }
  if (early) {  // the tables below read / write what the previous launch used
    if (threadIdx.x == 0) wait_count(h.prev_counter, h.prev_target);
    __syncthreads();
  }
  KV_STAMP(3);
  // 4. tables: the appended items' device bt entries; the publication's parity
  //    (req_id, len) table and the bt entries of the blocks it touched.  Readers trust
  //    none of it before seq = step (written below, after every CTA's release).
  //    Entries are spread CTA-major (entry i on CTA i mod G): a decode step has a few
  //    hundred of them, which would otherwise all sit on the first CTAs' threads after
  //    their copies -- the launch's tail.
#ifdef KV_AB_TBLPACK  // A/B builds: entries thread-major (the first CTAs take them all)
  const uint32_t gt = b * kThreads + threadIdx.x, stride = G * kThreads;
#else
  const uint32_t gt = threadIdx.x * G + b, stride = G * kThreads;
#endif
  for (uint32_t i = gt; i < (uint32_t)h.n_items; i += stride) {
    const KvAppItem &it = s.items[i];
    const KvStepPool &pp = h.app[it.pool];
    pp.bt[(size_t)it.slot * pp.M + fdiv((uint32_t)it.p0, h.div_b)] = it.blk & kItemBlkMask;
  }
  if (h.publish) {
    if (h.n_prev > 0) {  // the tables may be listed by the last stored seq: wait for the newer one
      if (threadIdx.x == 0) wait_gate(h);
      __syncthreads();
    }
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
          const int hi = s.hi[e];
          mreq[sl] = hi > 0 ? s.req[e] : -1;
          mlen[sl] = hi;
        } else {
          mreq[sl] = -1;
          mlen[sl] = 0;
        }
      }
      // bt entries of every touched block, one per thread over the whole pool (a bulk
      // re-seed touches thousands of blocks per request)
      const int e_lo = pp.ent_off, e_hi = pp.ent_off + pp.n_slots;
      const int nb_lo = s.bpref[e_lo], nb_hi = s.bpref[e_hi];
      for (uint32_t k = gt; k < (uint32_t)(nb_hi - nb_lo); k += stride) {
        const int gk = nb_lo + (int)k;
        int a = e_lo, z = e_hi - 1;      // last entry with bpref <= gk
        while (a < z) {
          const int m = (a + z + 1) >> 1;
          if (s.bpref[m] <= gk) a = m; else z = m - 1;
        }
        const int sl = a - pp.ent_off;
        const int j = s.lo[a] / B + (gk - s.bpref[a]);
        mbt[(size_t)sl * pp.M + j] =
            gk == s.bpref[a] ? (s.blk0[a] & kBlkMask) : pp.bt[(size_t)sl * pp.M + j];
      }
      if (gt == 0) *reinterpret_cast<int32_t *>(pp.meta + 8) = pp.writer_node;
    }
  }
  KV_STAMP(4);
  // 5. completion: bar.sync + one release RMW per CTA on the launch's counter -- at SYSTEM
  //    scope when a successor is an NVLink peer: a GPU-scope release does not wait for the
  //    CTA's stores into peer memory, and the concurrent reader test (tests/mgpu_worker.py
  //    r9) saw seq = t before step t's slices with it -- then the last CTA issues one
  //    acquire-release fence (system scope if a successor is a peer) and
  //    stores every publishing pool's seq (release pattern; reading R9), then tells the
  //    host the descriptor slot is free (nonce into pinned memory: every CTA read the
  //    slot long before it arrived here).  The slot's counter is monotone: the host passes
  //    the value the last arrival of this launch makes it reach.
  step_complete(h);
  KV_STAMP(5);
}

}  // namespace

// The decode-step kernel: header by value in the parameter space, descriptor blob in
// pinned host memory (pulled in by CTA 0, see step_body).
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    kv_step_kernel(const __grid_constant__ KvStepHdr h) {
  step_body(h);
}

const void *step_kernel_fn() { return reinterpret_cast<const void *>(kv_step_kernel); }

#ifdef KV_TIMELINE
extern "C" __attribute__((visibility("default"))) int kv_debug_timeline(unsigned long long *out,
                                                                       int n) {
  return cudaMemcpyFromSymbol(out, g_kv_timeline, sizeof(unsigned long long) * (size_t)n) ==
                 cudaSuccess ? 0 : -3;
}
#endif

namespace {
// Function attributes of the step kernel, once per device (they are per context): large
// launches may carry up to ~200 KiB of descriptors in shared memory.  (The largest
// shared-memory carveout for every launch measured 4 % slower at 2 GPUs.)
void step_kernel_attrs(int device) {
  static unsigned long long done = 0;
  if (device < 0 || device >= 64 || ((done >> device) & 1ull)) return;
  cudaFuncSetAttribute(kv_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaGetLastError();
  done |= 1ull << device;
}
}  // namespace

// Resident CTAs of the step kernel on `device` for a launch's shared memory.
int step_resident_ctas(int device, int smem) {
  static int cache_dev = -1, cache_smem = -1, cache_val = 0;
  if (device == cache_dev && smem == cache_smem) return cache_val;
  int sms = 148, per = kMinBlocks;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    sms = 148;
  step_kernel_attrs(device);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kv_step_kernel, kThreads, smem) !=
          cudaSuccess || per < 1)
    per = 1;
#ifdef KV_AB_CTAS_PER_SM  // A/B builds (tools/ab_bench.sh): a smaller grid cap
  per = per < KV_AB_CTAS_PER_SM ? per : KV_AB_CTAS_PER_SM;
#endif
  cudaGetLastError();
  cache_dev = device;
  cache_smem = smem;
  cache_val = sms * per;
  return cache_val;
}

// 16-B chunks per CTA the host sizes a launch's grid for (at most every resident CTA).
int step_chunks_per_cta() {
#ifdef KV_AB_CHUNKS  // A/B builds (tools/ab_bench.sh)
  return KV_AB_CHUNKS;
#else
  return 1024;
#endif
}

int step_smem_bytes(const KvStepHdr &h) {
  return h.data_bytes + 4 * (2 * h.n_ent + 2) + 16;
}

cudaError_t launch_step(const KvStepHdr &h, int grid, cudaStream_t st, bool pdl) {
  const int smem = step_smem_bytes(h);
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) step_kernel_attrs(dev);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kv_step_kernel, h);
}

}  // namespace kvring
