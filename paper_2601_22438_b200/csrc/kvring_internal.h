// Internal types shared by the host core (kvring_host.cpp) and the sm_100a
// kernels (kvring_kernels.cu, kvring_step.cu).  Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime_api.h>

namespace kvring {

// Address modes of the one copy engine.  A copy task
// moves `seg_count` (layer, K/V, head, token) slices of seg_bytes each; the
// slice s of an item with n_tok tokens is combo = s / n_tok, tok = s % n_tok.
enum AddrMode : int {
  kPaged = 0,     // base + unit*block_bytes + (combo*B + tok_lo + tok)*seg   (pool / replica)
  kTokMajor = 1,  // base + (unit + tok)*token_bytes + combo*seg              (dense model KV)
  kPacked = 2,    // base + (unit + s)*seg                                     (packed send buffer)
};

// 32-byte copy task (host-built, H2D-staged every step).
struct alignas(16) KvTask {
  int32_t src_unit;   // block id / token row / packed segment offset of the item
  int32_t dst_unit;
  int16_t pool;       // index into the launch's KvPoolParams
  int16_t slot;       // request slot of the item (bt publication), -1 = none
  int16_t j;          // logical block index of the item
  int16_t tok_lo;     // first token slot inside the block
  int16_t n_tok;      // tokens in the item (1..B)
  int16_t flags;      // kFirst: this task writes the item's bt entry
  int32_t seg_begin;  // first slice (item-relative) of this task
  int32_t seg_count;  // slices in this task (0 = publish-only task)
  int32_t pad;
};
static_assert(sizeof(KvTask) == 32, "KvTask must be 32 B");
enum : int16_t { kFirst = 1, kPoolFirst = 2 };  // kPoolFirst: writes the pool's parity table

// Per-pool launch parameters (device copy staged with the tasks).
struct alignas(16) KvPoolParams {
  const char *src;             // source base
  char *dst;                   // destination base
  char *meta;                  // destination metadata (publish), or nullptr
  const int64_t *slot_req;     // staged [R] req ids (publish)
  const int32_t *slot_len;     // staged [R] lengths (publish)
  unsigned long long *counter; // monotone completed-task counter (publish)
  unsigned long long target;   // counter value after the last task of this launch
  unsigned long long step;     // seq to publish
  int32_t max_reqs, max_blk, writer_node, publish;
  int32_t sys_scope;           // successor is an NVLink peer: system-scope fences / release
  int32_t pad0;
  int32_t n_table;             // publish: table entries staged; slots >= n_table publish (-1, 0)
  int32_t pad2;
  unsigned long long src_bytes;  // extent of src / dst (debug bounds checks, KV_BOUNDS_CHECK)
  unsigned long long dst_bytes;
};

struct KvGeomDev {
  long long block_bytes;
  int token_bytes;
  int seg_bytes;
  int block_size;
  int cps_shift;    // log2(seg_bytes / 16): 16-B chunks per slice
};

// Metadata region layout (include/kvring.h).
constexpr int kMetaMagic = 0x4B56524D;
inline size_t meta_off_req(int) { return 32; }
inline size_t meta_off_len(int R) { return 32 + 16 * (size_t)R; }
inline size_t meta_off_bt(int R) { return 32 + 24 * (size_t)R; }
inline size_t meta_bytes(int R, int M) {
  size_t b = 32 + 24 * (size_t)R + 4 * (size_t)R * (size_t)M;
  return (b + 255) & ~(size_t)255;
}

// Packed (NCCL-variant) buffer header.
struct alignas(16) KvPackedHeader {
  int32_t magic;        // 0x4B565042 "KVPB"
  int32_t n_tasks;
  int32_t max_reqs, max_blk;
  int32_t writer_node, seg_bytes;
  unsigned long long step;
  unsigned long long task_off, slot_off, payload_off, payload_bytes, total_bytes;
};
constexpr int kPackedMagic = 0x4B565042;

// Launch wrappers of the host-task kernels (kvring_kernels.cu): restore-remap, the
// NCCL-variant gather-pack, and the host-task ring-put that the shared-capacity
// (holder-allocated replica ids) and copy-engine links use.  All return the
// cudaError_t of the launch.
enum KernelKind : int { kKindRingPut = 1, kKindRestore = 2, kKindPack = 3 };
constexpr int kMaxPoolsPerLaunchHost = 64;
cudaError_t launch_copy(int kind, const KvTask *tasks, int n_tasks, const KvPoolParams *params,
                        int n_pools, const KvGeomDev &g, int grid, cudaStream_t stream);
cudaError_t launch_unpack(const char *packed, char *replica, char *meta,
                          unsigned long long *counter, const KvGeomDev &g, int grid,
                          cudaStream_t stream);
cudaError_t launch_meta_init(char *meta, int R, int M, cudaStream_t stream);
// 1-CTA acquire of a holder's metadata (kv_restore): ld.acquire.sys of seq, then a copy
// of header + tables into `out` (device scratch).
cudaError_t launch_meta_acquire(const char *meta, char *out, size_t bytes, cudaStream_t stream);
int copy_grid(int device, int n_tasks);
int resident_ctas(int device);

// ---------------------------------------------------------------------------
// Decode-step engine (kvring_step.cu): ONE launch carries the appends of a step
// (host-built items: the allocator is the host's) and/or the publication of a
// step whose work list the DEVICE derives (§8(a) a3) from per-slot
// (req_id, len, pub_len) snapshots and the pool's device-resident block table.
// Every byte moved by the launch is one flat space of 16-B chunks split evenly
// over the CTAs (append chunks and replication chunks each), so the launch is
// balanced however the step mixes prefill, decode and publication.

// Unsigned 32-bit division by an invariant d >= 1 (Granlund-Montgomery, Hacker's
// Delight 10-8): l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1,
// t = umulhi(m, x), q = (t + ((x - t) >> sh1)) >> sh2, sh1 = min(l, 1), sh2 = max(l - 1, 0).
struct KvDiv {
  uint32_t d, m, sh1, sh2;
};
inline KvDiv kv_div(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  KvDiv r;
  r.d = d;
  r.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1ull);
  r.sh1 = l < 1 ? l : 1;
  r.sh2 = l > 1 ? l - 1 : 0;
  return r;
}

// One append item: n tokens of one request slot that land in ONE block.  Its slices
// occupy the flat range [off, next item's off) in token-major order (slice x of the
// item = token x / combos, (layer, K/V, head) x % combos).
struct alignas(8) KvAppItem {
  int32_t off;    // first slice (flat, over every item of the launch)
  int32_t row;    // first token row in the pool's dense source
  int32_t blk;    // destination block id (host allocator)
  int32_t p0;     // position of the item's first token (j = p0 / B, slot in block = p0 % B)
  int16_t slot;   // request slot: the item writes bt[slot][j] = blk on the device
  int16_t pool;   // index into KvStepHdr::app
};
static_assert(sizeof(KvAppItem) == 24, "KvAppItem must be 24 B");
// KvAppItem::blk | kItemGated: the block was freed one step ago, so the previous launch's
// publication may still be reading it -- an early-started launch copies into it only
// after that launch's arrival count (KvStepHdr::early)
constexpr int32_t kItemGated = 1 << 30;
constexpr int32_t kItemBlkMask = kItemGated - 1;

struct alignas(16) KvStepPool {
  const char *src;        // append: dense source; replicate: this pool
  char *dst;              // append: this pool; replicate: successor replica region
  char *meta;             // replicate: successor metadata (include/kvring.h layout)
  int32_t *bt;            // device block table [R][M] of the pool (append writes, replicate reads)
  unsigned long long step;  // replicate: seq to publish
  int32_t R, M;
  int32_t n_slots;        // replicate: table entries (slots >= n_slots publish (-1, 0))
  int32_t ent_off;        // replicate: index of the pool's first entry
  int32_t mode;           // KV_MODE_TOKENS / KV_MODE_BLOCKS
  int32_t abort_slices;   // replicate: -1, or copy only the first N slices and never publish
  int32_t writer_node;
  int32_t sys;            // successor is not this GPU's HBM: system-scope publication
};

constexpr int kStepPools = 8;      // pools per launch (each role)
constexpr int kStepMaxEnt = 4096;  // replicate table entries per launch (sum of n_slots)

struct alignas(16) KvStepHdr {
  int32_t n_app, n_rep;             // pools per role
  int32_t n_items, n_ent;           // append items; replicate entries
  int32_t items_off, req_off, len_off, pub_off;  // byte offsets into the data blob
  int32_t blk0_off;                 // per entry: block holding the first dirty token
  int32_t data_bytes;               // bytes of the data blob (a multiple of 16)
  int32_t app_slices;               // total append slices (end of the last item)
  int32_t publish;                  // some replicate pool publishes this launch
  int32_t any_abort;
  int32_t sys_any;
  int32_t pad0;                     // launch nonce (debug timelines)
  int32_t pdl;                      // launched as a programmatic dependent of the previous kernel
  int32_t chain;                    // the previous kernel on the stream is this library's step
                                    // launch: acquire its final count instead of griddepcontrol.wait
  const char *hblob;                // the descriptor blob in pinned host memory (device-mapped)
  char *gblob;                      // its device copy (written by CTA 0)
  unsigned long long *flag;         // = nonce once gblob holds this launch's blob
  unsigned long long nonce;         // launch nonce (monotone per process)
  unsigned long long *counter;      // completion counter of the slot (monotone)
  unsigned long long target;        // its value once every CTA of this launch arrived
  unsigned long long *done;         // pinned host word: = nonce once the launch completed
  unsigned int *work;               // dynamic round counters of the slot (8 x 64 B, zero at rest)
  // deferred publication over NVLink: a launch with `defer` does not wait for its peer
  // stores' acknowledgements (its CTAs arrive with a GPU-scope release) and stores no
  // seq; the next launch on the stream -- chained, so it starts copying at once -- adds
  // one publisher CTA (the last) that waits for that launch to complete
  // (griddepcontrol.wait: every store performed) and stores its seqs (n_prev of them)
  // R7 under deferral: until the publisher has stored the previous seqs, the last
  // stored seq may still list blocks freed one step ago -- so this launch's stores into
  // blocks with no previously published token, and its table writes, wait for `gate`
  // (= nonce, released by the publisher after its seq stores)
  int32_t defer;
  int32_t n_prev;
  int32_t prev_sys;                 // bit q: prev_seq[q] is in a peer's memory
  // early start of a chained launch whose predecessor was chained too: the launch before
  // the previous one (pp_counter) has arrived before any copy; the append rounds then go
  // at once -- except items into blocks freed one step ago (kItemGated) -- while the
  // previous launch drains, and a warp acquires the previous launch's arrival count
  // (prev_counter) before its first publication round / gated item; every CTA before
  // its tables (they read and write the device block table the previous launch used)
  int32_t early;
  int32_t app_first;                // append rounds before publication rounds (no NVLink
                                    // successor), else interleaved (kvring_step.cu copy_all)
  int32_t pad3;
  unsigned long long *gate;
  unsigned long long *prev_seq[kStepPools];
  unsigned long long prev_step[kStepPools];
  unsigned long long *prev_counter; // chain: the previous launch's counter ...
  unsigned long long prev_target;   // ... and its arrival target (every CTA arrived: its data
                                    // is complete; + 1 once its seqs are stored)
  unsigned long long *pp_counter;   // early: the launch before the previous one ...
  unsigned long long pp_target;     // ... and its arrival target
  KvGeomDev g;
  KvDiv div_sl;                     // slices per token (layers x 2 x kv_heads)
  KvDiv div_b;                      // block size
  KvDiv div_bs;                     // slices per block (block size x slices per token)
  KvStepPool app[kStepPools];
  KvStepPool rep[kStepPools];
};

// Launches the step kernel (blob, flag and nonce in the header).  pdl: programmatic
// dependent launch (the previous kernel on the stream may still be draining).
cudaError_t launch_step(const KvStepHdr &h, int grid, cudaStream_t stream, bool pdl);
int step_smem_bytes(const KvStepHdr &h);
int step_chunks_per_cta();
const void *step_kernel_fn();
int step_resident_ctas(int device, int smem);

}  // namespace kvring
