// Internal types shared by the host core (kvring_host.cpp) and the sm_100a
// kernels (kvring_kernels.cu).  Not part of the ABI.
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

// Launch wrappers (kvring_kernels.cu).  All return the cudaError_t of the launch.
enum KernelKind : int { kKindAppend = 0, kKindRingPut = 1, kKindRestore = 2, kKindPack = 3,
                        kKindRingPutCopy = 4, kKindPublish = 5 };
constexpr int kMaxPoolsPerLaunchHost = 64;
// Per-pool source / destination bases passed by value in the kernel parameter
// space (hot kernels): the only parameters on the path to a CTA's first data load.
constexpr int kInlinePools = 8;
struct KvParamPack {
  const char *src[kInlinePools];
  char *dst[kInlinePools];
  int n;  // 0: read them from the staged global copy
};
// split: each task is processed as `split` CTA units (a contiguous share of its
// slices each), so the host emits whole-item tasks (<= 32 KiB) and the device still
// spreads a decode step over every resident CTA; the publication counts units.
cudaError_t launch_copy(int kind, const KvTask *tasks, int n_tasks, const KvPoolParams *params,
                        int n_pools, const KvGeomDev &g, int grid, cudaStream_t stream,
                        const KvPoolParams *host_params = nullptr, int split = 1);
cudaError_t launch_fused(const KvTask *tasks, int n_append, int n_tasks, const KvPoolParams *params,
                         int n_app_pools, int n_rep_pools, const KvGeomDev &g, int grid,
                         cudaStream_t stream);
// A launch carried entirely in the kernel's parameter space (<= 32 KiB since
// CUDA 12.1): per-pool parameters, the ring-put's publication tables and the task
// list.  No H2D staging copy and no dependent global load before a CTA's first
// data load; ring-put pools carry their table offsets (into `data`) in
// slot_req / slot_len.
// Size classes: the launch copies the whole parameter block (the driver's copy
// costs ~0.2 us per KiB on the host), so a launch pays for the smallest class its
// tables + tasks fit: 4, 8, 16 or 28 KiB.
constexpr int kInlineBytes = 28 * 1024;
template <int CAP>
struct KvInlineDescT {
  int32_t n_tasks, n_pools, task_off, used;  // used: bytes of data in use
  int32_t split, pad0, pad1, pad2;           // CTA units per task (see launch_copy)
  KvPoolParams pools[kInlinePools];
  alignas(16) char data[CAP];
};
using KvInlineDesc = KvInlineDescT<kInlineBytes>;
cudaError_t launch_copy_inline(int kind, const KvInlineDesc &d, const KvGeomDev &g, int grid,
                               cudaStream_t stream, bool pdl);
// Self-describing graph steps (kv_run_steps_graph, fixed nodes): step i of a group
// reads its launches from this header at the start of the group's staged slot, so
// the graph's kernel nodes keep fixed parameters (slot base, step index) and the host
// updates nothing per step but the slot contents.  [0] = append, [1] = ring-put.
struct alignas(16) KvStepHdr {
  int32_t n_tasks[2];
  int32_t n_pools[2];
  int32_t split[2];
  int32_t pad[2];
  unsigned long long params_off[2];
  unsigned long long tasks_off[2];
  KvGeomDev g;
};
constexpr int kFxPublishGrid = 64;  // publication node: one CTA per pool, up to 64 pools
// Fills kp for a fixed-node kernel (kKindAppend / kKindRingPutCopy / kKindPublish)
// reading step `i` of the slot at `slot`; a must outlive the call consuming kp.
struct KvFxArgs {
  const char *slot = nullptr;
  int step = 0;
  void *ptrs[2] = {};
};
void fx_node_params(int kind, int grid, KvFxArgs &a, cudaKernelNodeParams &kp);

// Arguments of a staged append / ring-put launch as a CUDA graph kernel node (the
// graph decode loop updates them per step with cudaGraphExecKernelNodeSetParams).
struct KvNodeArgs {
  const KvTask *tasks = nullptr;
  int n_tasks = 0;
  const KvPoolParams *params = nullptr;
  KvGeomDev g{};
  int n_pools = 0;
  KvParamPack pk{};
  int split = 1;
  void *ptrs[7] = {};
};
// Fills kp (function, grid, block, argument pointers into a) for kind
// kKindAppend / kKindRingPut; a must outlive the call that consumes kp.
void kernel_node_params(int kind, int grid, KvNodeArgs &a, cudaKernelNodeParams &kp);
cudaError_t launch_unpack(const char *packed, char *replica, char *meta,
                          unsigned long long *counter, const KvGeomDev &g, int grid,
                          cudaStream_t stream);
cudaError_t launch_meta_init(char *meta, int R, int M, cudaStream_t stream);
int copy_grid(int device, int n_tasks);
int resident_ctas(int device);

}  // namespace kvring
