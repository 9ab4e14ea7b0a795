/*
 * kvring.h -- C ABI of libkvring: ring-shaped KV-cache replication for
 * fault-tolerant pipeline-parallel LLM serving, B200 (sm_100a) native.
 *
 * Method: KevlarFlow (arXiv 2601.22438).  PAPER.md P:223-225 (§3.2):
 *   "KevlarFlow replicates KV cache for each request to the GPU memory of
 *    other nodes in the load balancing group ... When failure occurs ...
 *    in-progress requests will be served continuously on the replication
 *    target from the replicated state, avoiding retries"
 * and P:229 (§3.2): "a block representation of KV cache ... replicate it
 * block-by-block in the background.  A separate CUDA stream is used to
 * overlap the communication with computation."  Ring shape: P:8 (§3.3).
 * Readings of what the paper leaves open (R1-R16) are listed in DESIGN.md;
 * the ones that fix behaviour visible through this ABI are cited per call.
 *
 * Conventions
 *  - Every call returns KV_OK (0) or a negative kv_status_t; the message of the
 *    last failure on the calling thread is kv_last_error().  No C++ exception
 *    crosses this boundary.
 *  - "device" pointers are CUDA device (or NVLink peer-mapped) addresses;
 *    "host" pointers are CPU memory.  Streams are cudaStream_t passed as void*.
 *  - All GPU work is enqueued asynchronously on the stream given; no call ever
 *    waits on a peer GPU.  kv_restore is the one call that synchronises (it
 *    must read the holder's published metadata).
 *  - One host thread per pool handle at a time.  Pools on the same device share
 *    an internal staging context guarded by a mutex.
 *
 * Memory layout (reading R4)
 *  - 16-bit words (fp16/bf16 bit patterns, never interpreted: R13).
 *  - block  = [layers][2 (K,V)][kv_heads][block_size][head_dim] words, so one
 *             (layer, K/V, head, token) slice of head_dim words is contiguous
 *             (256 B for head_dim 128) and a full block is contiguous.
 *  - pool   = [num_blocks] blocks.  replica region = [replica_blocks] blocks,
 *             holding the ring predecessor's blocks AT THE SAME BLOCK IDS (R5).
 *  - dense new-token KV (kv_append source) = [sum n_new][layers][2][kv_heads][head_dim].
 *  - replica metadata (kv_meta_bytes), written only by the predecessor's
 *    replicate kernel, little-endian:
 *        off 0   uint64 seq          last published step, 0 = nothing (R9)
 *        off 8   int32  writer_node  node_id of the predecessor that wrote it
 *        off 12  int32  max_reqs R
 *        off 16  int32  max_blocks_per_req M
 *        off 20  int32  magic 0x4B56524D ("KVRM")
 *        off 24  int64  reserved
 *        off 32  int64  req_id[2][R]  parity (step & 1) buffers, -1 = empty slot
 *        off 32+16R     int32 len[2][R]
 *        off 32+24R     int32 bt[R][M] block ids in the predecessor's pool
 *                       (entries j < ceil(len/B) of a listed slot are valid)
 *    seq is stored last, right after a system-scope acquire-release fence, so a
 *    reader that acquires seq = t sees parity t's lengths, rows and KV slices.
 */
#ifndef KVRING_H
#define KVRING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVRING_ABI_VERSION 1

typedef enum {
  KV_OK = 0,
  KV_EINVAL = -1,      /* bad geometry / argument, unknown request, non-monotone step  */
  KV_ENOMEM = -2,      /* pool blocks or request slots exhausted; all-or-nothing */
  KV_ECUDA = -3,       /* a CUDA call failed or a sticky asynchronous error surfaced       */
  KV_ESTATE = -4,      /* the pool is dead (after kv_fail_stage) or the call is not allowed  */
  KV_ENOREPLICA = -5,  /* holder metadata invalid or nothing published (seq == 0)         */
  KV_EPEER = -6        /* no successor bound                                                */
} kv_status_t;

typedef struct kv_pool kv_pool_t; /* opaque; one per logical node (instance, stage) */

typedef struct {
  int32_t layers;      /* L_s, layers of this pipeline stage                         */
  int32_t kv_heads;    /* H (Llama-3.1-8B: 8)                                         */
  int32_t head_dim;    /* d (128); head_dim * elem_bytes: a power of 2 in [16, 512]    */
  int32_t block_size;  /* B tokens per block (16)                                     */
  int32_t elem_bytes;  /* must be 2 (16-bit words)                                    */
} kv_geom_t;

typedef struct {
  kv_geom_t g;
  int32_t num_blocks;         /* NB of the primary pool                                 */
  int32_t max_reqs;           /* request slots R (>= 2 x live batch: slots quarantine, R7) */
  int32_t max_blocks_per_req; /* M                                                       */
  int32_t device;             /* CUDA ordinal; -1 = tables only (host-logic tests: no
                                 device memory, nothing launched, no bytes moved)        */
  int32_t node_id;            /* logical node id, written into the successor's metadata */
  int32_t replica_blocks;     /* blocks in this node's replica region (= pred's NB)      */
  void *pool;                 /* device, caller-owned, num_blocks * kv_block_bytes        */
  void *replica;              /* device, caller-owned, replica_blocks * kv_block_bytes    */
  void *replica_meta;         /* device, caller-owned, kv_meta_bytes(R, M); initialised
                                 by kv_pool_create (seq 0, empty slots, bt -1)            */
} kv_pool_desc_t;

/* Bytes of one block / one replica metadata region (layout above). */
size_t kv_block_bytes(const kv_geom_t *g);
size_t kv_meta_bytes(int32_t max_reqs, int32_t max_blocks_per_req);
int32_t kv_abi_version(void);

/* Create a pool handle over caller-owned device memory.  Validates geometry,
 * builds the host allocator (R6 lowest-free-id, R7 one-step quarantine) and
 * initialises replica_meta on the device (synchronously).  pool/replica bytes
 * are left untouched (the caller fills its sentinel). */
int kv_pool_create(const kv_pool_desc_t *desc, kv_pool_t **out);
int kv_pool_destroy(kv_pool_t *p);

/* Bind the ring link p -> successor (SPEC S:298-306 apply_plan; ring map is
 * data, reading R1).  succ_replica / succ_meta are the successor's replica
 * region and metadata: local device pointers or NVLink peer pointers (e.g.
 * torch symmetric-memory buffer_ptrs).  succ_replica_blocks must be >= p's NB.
 * NULL succ_replica disables replication.  Any (re)bind re-seeds: every live
 * request is republished from token 0 at the next kv_replicate_step. */
int kv_set_successor(kv_pool_t *p, int32_t succ_node, void *succ_replica,
                     int32_t succ_replica_blocks, void *succ_meta);

/* Shared-capacity link (§8(f) NEXT-3, reading R17): §3.2 "KevlarFlow
 * utilizes such memory headroom to temporarily handle ... the replicated KV
 * cache.  When memory pressure happens, KevlarFlow drops the replicated KV cache
 * and recomputes them if needed".
 *   - holder h keeps p's replica IN ITS OWN POOL: replica blocks come from h's
 *     free list (lowest id, R6) when p publishes; h's metadata bt rows hold h's
 *     block ids (restore: pass h's pool as holder_replica, h's NB as its size);
 *   - when an append on h needs more blocks than are free, h evicts p's
 *     replicas, oldest admission first, until it fits; an append is rejected
 *     (KV_ENOMEM, nothing changes) only if free + all replica blocks cannot
 *     cover it;
 *   - a request whose replica cannot grow (h full) is dropped, as is an evicted
 *     one: it is listed as absent from then on and never re-sent (recompute on
 *     failure);
 *   - freed replica blocks are reusable AT ONCE: the entry that referenced them
 *     is withdrawn from the published table (two memsets, flushed before the
 *     next launch touching h).  Stream order needed: an append on h after the
 *     ring-put of the previous step (kv_run_steps does it; kv_loop_step
 *     reject shared pools, KV_EINVAL).
 * Same device, geometry, max_reqs and max_blocks_per_req; one predecessor per
 * holder (a previous one is unlinked, its replicas freed).  Re-seeds p. */
int kv_set_successor_shared(kv_pool_t *p, kv_pool_t *holder);

/* Holder side: free every replica block held for the predecessor (after a
 * restore has read them -- promotion or fresh -- or on demand); those requests
 * count as dropped.  A dead predecessor is unlinked.  Host-only. */
int kv_drop_replicas(kv_pool_t *holder);

/* Shared capacity across GPUs (NEXT-3 with the holder in another process).  The
 * holder's process creates a MIRROR of the predecessor: a pool on the HOLDER's
 * device whose `pool` pointer is the predecessor's pool as mapped into this process
 * (an NVLink peer address, e.g. from symmetric memory) and whose replica/meta are
 * scratch.  on = 1 (before the mirror's first append): appends and releases on the
 * mirror update its tables only (the owner moves the bytes; src_kv may be NULL), so
 * applying the owner's append calls in the same order keeps identical tables
 * (allocation is deterministic, reading R6); kv_set_successor_shared(mirror, holder)
 * then replicates by PULLING the dirty slices from the owner's pool over NVLink into
 * holder-allocated blocks -- the allocator that must decide them lives here.  The
 * caller orders the pull after the owner's append of the step (e.g. a host barrier)
 * and the owner's append of step t+2 after the pull of step t (R7).  kv_fail_stage on
 * a mirror only marks it dead (the owner poisons its own memory).  KV_ESTATE if the
 * mirror was already used.  The mirror does not choose block ids: the owner's
 * allocator also serves the owner's own holder role, so the owner forwards the ids
 * its append allocated (kv_last_alloc) and the holder queues them
 * (kv_mirror_blocks) before the mirror's append of the same step (KV_ESTATE if
 * fewer are queued than the append needs). */
int kv_pool_set_mirror(kv_pool_t *p, int32_t on);
int kv_mirror_blocks(kv_pool_t *mirror, int32_t n, const int32_t *block_ids);
/* Block ids allocated by p's last append, in allocation order (copies min(n, cap));
 * returns n. */
int kv_last_alloc(kv_pool_t *p, int32_t *out, int32_t cap);

/* Step boundary: blocks and slots quarantined by the
 * previous step become allocatable. */
int kv_begin_step(kv_pool_t *p);

/* Finish requests (§8(c) step 2): their blocks and slot go to quarantine and
 * are not reallocated before the next kv_begin_step (R7).  Host-only. */
int kv_release(kv_pool_t *p, int32_t n, const int64_t *req_ids);

/* Append new-token KV (the model's KV write; harness stand-in, §8(a) a2).
 * Entries are processed in order: a known req_id grows by n_new[i] tokens
 * (a new block = lowest free id whenever len % B == 0); an unknown req_id is an
 * admission (slot = lowest free slot, then ceil(n_new/B) blocks).  src_kv is
 * dense [sum n_new][L][2][H][d] in entry order, on the device, or on the host
 * when flags & KV_SRC_HOST: pinned (page-locked) host memory is read by the
 * scatter kernel directly over PCIe (zero copy; it must stay valid until the
 * kernel has run), pageable host memory is copied into a library staging buffer
 * in the call's stream order.  All-or-nothing: KV_ENOMEM / KV_EINVAL
 * leave the tables unchanged.  Launches one scatter kernel. */
#define KV_SRC_HOST 1
int kv_append(kv_pool_t *p, int32_t n, const int64_t *req_ids, const int32_t *n_new,
              const void *src_kv, int32_t flags, void *stream);

/* Batched form for several pools on ONE device: per pool an optional
 * begin_step, releases, and appends -- one H2D and one kernel launch in total.
 * Validation of every pool happens before any pool changes. */
typedef struct {
  kv_pool_t *pool;
  int32_t begin_step;          /* nonzero: kv_begin_step first                 */
  int32_t n_release;
  const int64_t *release_ids;
  int32_t n;                   /* appends                                      */
  const int64_t *req_ids;
  const int32_t *n_new;
  const void *src_kv;          /* device (or host with KV_SRC_HOST)            */
  int32_t flags;
} kv_append_args_t;
int kv_append_multi(int32_t n_pools, const kv_append_args_t *args, void *stream);

/* Publish step `step` to the successor (§8(c) step 5; R2 dirty tokens; R9).
 * ONE kernel derives the work list on the device (§8(a) a3): from a snapshot of
 * each live slot's (req_id, len, pub_len) and the pool's device-resident block
 * table it splits the dirty tokens [pub_len, len) at block boundaries, sums them
 * over slots, and copies them from this pool to the successor's replica region at
 * the same block ids with 16-B stores (NVLink P2P when the successor is remote);
 * then the bt entries of the touched blocks and the parity (step & 1)
 * (req_id, len) table are written, and the last CTA stores seq = step (release,
 * system scope for a peer).  Shared-capacity links use a host-built work list.  step >= 1 and strictly increasing per
 * pool; KV_EPEER if no successor is bound.  pub_len := len on return (the host
 * never waits for the peer). */
int kv_replicate_step(kv_pool_t *p, uint64_t step, void *stream);
/* Same for several pools of ONE device in a single launch. */
int kv_replicate_step_multi(int32_t n_pools, kv_pool_t *const *pools, uint64_t step, void *stream);

/* Replication granularity (reading R2; §8(f) NEXT-2).  KV_MODE_TOKENS (default):
 * every step publishes all appended tokens (exact replica).  KV_MODE_BLOCKS: only
 * completed blocks ("replicate it block-by-block"): whole 16-token blocks,
 * the replica lags by <= B-1 tokens per request and the published length is a
 * multiple of B (a request with no completed block is listed as empty).  A mode
 * change re-seeds the link. */
#define KV_MODE_TOKENS 0
#define KV_MODE_BLOCKS 1
int kv_set_mode(kv_pool_t *p, int32_t mode);

/* Decode steps.  A step = the appends of step `step` (the model's KV write,
 * kv_append_multi semantics) followed by the publication of the same step by
 * repl_pools (kv_replicate_step_multi semantics).  The
 * optional cudaEvent_t handles are recorded around the launches named below. */
typedef struct {
  int32_t n_append;
  const kv_append_args_t *append;
  int32_t n_repl;              /* 0: no publication this step (e.g. step 0) */
  kv_pool_t *const *repl_pools;
  uint64_t step;
  void *ev_call, *ev_kernel_start, *ev_kernel_end, *ev_done;
  void *ev_append_start, *ev_append_end;
} kv_step_t;

/* Two-stream decode loop, the paper's shape (§3.2: "A separate CUDA stream
 * is used to overlap the communication with computation"): per step ONE append
 * launch on append_stream and, ordered after it by an event, ONE publication
 * launch on repl_stream.  The append of step k also waits (event) for the
 * publication of step k-2 (k-1 for shared-capacity pools): blocks freed by a
 * retiring request are reused one step later (reading R7) and must not be
 * overwritten while a lagging publication still reads them.  Steps are counted
 * across calls on the same stream pair; on a new pair the first append waits for
 * everything already on repl_stream.  Equal streams: plain stream order.
 * ev_append_start/end bracket the append launch, ev_call / ev_done the publication
 * (stream position), ev_kernel_start/end its kernel.  Stops at the first error
 * (steps before it stay applied). */
int kv_run_steps(int32_t n_steps, const kv_step_t *steps, void *append_stream,
                 void *repl_stream);

/* One-launch-per-step decode loop on ONE stream (software pipelined; no lookahead:
 * each call prepares and launches exactly the step it is given).  kv_loop_step
 * launches ONE kernel that carries the appends of `step` AND the publication of
 * the step previously given to this loop (the "pending" publication): the
 * replication of step k-1 overlaps the KV write of step k inside one balanced
 * grid -- their slots are disjoint by reading R7 -- and `step`'s publication
 * becomes pending.  The pending publication is built from the pools' tables as
 * they are when the next kv_loop_step / kv_loop_flush runs (the appends of the new
 * step are applied after it), so calls made in between -- kv_fail_stage, kv_restore,
 * kv_set_successor, a resume kv_append -- act exactly as between the append and the
 * replicate of the sequential protocol; pending pools that died or lost their
 * successor meanwhile publish nothing.  If the appends are rejected (KV_ENOMEM /
 * KV_EINVAL, tables unchanged) the pending publication is still launched and the
 * error returned.  Shared-capacity pools are not accepted (KV_EINVAL).
 * ev_kernel_start / ev_kernel_end bracket the launch; the other events are ignored.
 * kv_loop_flush launches the pending publication alone; kv_loop_run is n_steps
 * kv_loop_step calls.  One host thread per loop; a pool is pending in one loop. */
typedef struct kv_loop kv_loop_t;
int kv_loop_create(kv_loop_t **out);
int kv_loop_destroy(kv_loop_t *loop);
int kv_loop_step(kv_loop_t *loop, const kv_step_t *step, void *stream);
int kv_loop_run(kv_loop_t *loop, int32_t n_steps, const kv_step_t *steps, void *stream);
int kv_loop_flush(kv_loop_t *loop, void *stream);

/* Launch log of the calling thread (measurement): mode 1 clears and starts it;
 * mode 0 stops it and copies min(count, cap) records of 5 uint64 each --
 * [kind (1 append, 2 publication, 3 both), append payload bytes, publication
 * payload bytes, grid, descriptor bytes] -- for every decode-step kernel launched
 * since; returns the count. */
int kv_launch_log(uint64_t *out, int32_t cap, int32_t mode);

/* Re-protection after a failure (§8(f) NEXT-1; §3.2: "replication targets
 * will be automatically adjusted to exclude the nodes under traffic rerouting").
 * succ[n_nodes] is the ring's successor map over logical node ids; excluded
 * (may be NULL) marks failed nodes and nodes under traffic rerouting.  Each
 * non-excluded node's target is the first non-excluded node met by walking the
 * successors (never itself); -1 if there is none, and -1 for excluded nodes (they
 * neither send nor receive).  Host-only; apply with kv_set_successor (re-seed). */
int kv_plan_targets(int32_t n_nodes, const int32_t *succ, const uint8_t *excluded,
                    int32_t *targets);

/* Copy-engine variant (§8(f) NEXT-4, zero-SM bulk copies): like
 * kv_replicate_step_multi, but every FULL block of the dirty set is moved by the
 * copy engines (consecutive block ids coalesced into one cudaMemcpyAsync, peer
 * capable); partial blocks still go through the ring-put kernel, which is
 * stream-ordered after the copies, writes all bt entries and publishes seq.  Same
 * replica bytes and metadata as kv_replicate_step_multi. */
int kv_replicate_step_ce(int32_t n_pools, kv_pool_t *const *pools, uint64_t step, void *stream);

/* Fault injection: the next publication of p copies only the first
 * `slices` (layer, K/V, head, token) slices of its dirty set (in the device's work
 * order) and publishes nothing -- no tables, no seq, and p's host state stays at
 * its previous publication: a stage dying mid-step.  -1 clears. */
int kv_inject_abort(kv_pool_t *p, int32_t slices);

/* Simulated failure (§8(a) a7): p becomes dead; its pool, replica region and
 * replica metadata are overwritten with 0xFF bytes on `stream`. */
int kv_fail_stage(kv_pool_t *p, void *stream);

/* Restore (§8(a) a8): rebuild the requests published in a holder's
 * replica region into pool dst.  Reads seq = t* with a device acquire
 * (ld.acquire.sys in a kernel on dst's device, then a fence; reading R9) and the
 * parity-t* metadata copied after it, allocates in dst by ascending req_id then logical block j (lowest
 * free ids, R6), copies each block's valid slots [0, min(B, len - jB)) from
 * holder_replica (local HBM, or NVLink when it is a peer pointer) and rebuilds
 * dst's tables.  dst may be the holder itself (promotion, R10).  Outputs
 * (req_id, resume_len) ascending into caller arrays of capacity `cap`.
 * Synchronous; restored requests start unpublished.  KV_ENOREPLICA if seq is 0
 * or all-ones (poisoned) or the metadata shape differs; KV_ENOMEM all-or-nothing. */
int kv_restore(kv_pool_t *dst, const void *holder_replica, int32_t holder_replica_blocks,
               const void *holder_meta, void *stream, uint64_t *t_star,
               int64_t *req_ids_out, int32_t *resume_len_out, int32_t cap, int32_t *n_out);

/* NCCL-comparison path (§8(a) a4/a6): gather this step's dirty slices into
 * one contiguous device buffer (header + item list + slot table + payload,
 * see DESIGN.md "Packed format"), without touching the successor.  *bytes_out
 * is the packed size (the 8-B count exchanged before ncclSend/Recv).  Advances
 * pub_len like kv_replicate_step.  kv_pack_bytes gives the size without packing. */
int kv_pack_bytes(kv_pool_t *p, size_t *bytes_out);
int kv_pack_step(kv_pool_t *p, uint64_t step, void *packed, size_t cap, size_t *bytes_out,
                 void *stream);
/* Receiver side: scatter a packed buffer into (replica, replica_meta) and
 * publish its step; one kernel whose grid is sized from max_items (host arg). */
int kv_unpack(const void *packed, size_t packed_bytes, void *replica, int32_t replica_blocks,
              void *replica_meta, const kv_geom_t *g, int32_t max_reqs,
              int32_t max_blocks_per_req, void *stream);

/* Queries (host tables; no device access). */
int kv_query(kv_pool_t *p, int64_t req_id, int32_t *len, int32_t *blocks, int32_t cap,
             int32_t *nblk);
typedef struct {
  int32_t free_blocks, quarantined_blocks, used_blocks;
  int32_t free_slots, quarantined_slots, live_reqs;
  int32_t dead, has_successor;
  uint64_t last_step;
  uint64_t bytes_replicated;   /* algorithmic payload bytes published so far */
  uint64_t tasks_launched;     /* copy tasks issued by replicate kernels      */
  uint64_t kernels_launched;   /* kernels issued by this pool (all kinds)     */
  uint64_t last_step_bytes;    /* payload bytes of the latest replicate       */
  int64_t replica_blocks_held; /* shared capacity: predecessor replica blocks in this pool */
  uint64_t replica_evictions;  /* shared capacity: replicas this holder evicted (requests) */
  uint64_t replica_drops;      /* shared capacity: replicas dropped on growth (requests)   */
  int32_t shared_holder;       /* node id of the shared-capacity holder, -1 if none        */
  int32_t pad0;
} kv_stats_t;
int kv_stats(kv_pool_t *p, kv_stats_t *out);
/* Per-slot tables: req_id (-1 empty), len, pub_len, nblk; arrays of max_reqs. */
int kv_dump_slots(kv_pool_t *p, int64_t *req_id, int32_t *len, int32_t *pub_len,
                  int32_t *nblk);

/* Surface sticky asynchronous CUDA errors of p's device (synchronises it). */
int kv_sync(kv_pool_t *p);
const char *kv_last_error(void);

/* Kernels launched by this process through libkvring, all kinds (evidence
 * counter for bench gpu_launches). */
uint64_t kv_kernel_launch_count(void);

/* Profiling hook: record the given cudaEvent_t handles (either may be NULL)
 * on the launch stream immediately before / after the NEXT kernel this thread
 * launches through libkvring (the descriptor H2D that precedes it is excluded).
 * Used by bench.py to time the ring-put kernel live. */
int kv_time_next_launch(void *ev_before, void *ev_after);

/* Host-side phase counters of the decode path (seconds, cumulative since the last
 * reset; diagnostics, updated without synchronisation): [0] append preparation
 * (validation, allocation, items), [1] publication preparation (snapshot +
 * commit), [2] descriptor staging / host-source staging, [3] launch calls; [4..7] split
 * [2]: packing the descriptor blob, acquiring a staging slot, the H2D call, events.
 * Copies min(n, count) values; returns the count. */
int kv_host_profile(double *out, int32_t n, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* KVRING_H */
