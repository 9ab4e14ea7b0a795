// libkvring host core: C ABI (include/kvring.h), allocator and block tables
// (N2), ring link state, work-list / task builder (N4), staging of the
// per-step descriptors (kernel parameter space for decode-size launches, one H2D
// per launch otherwise) and kernel launches.
//
// Paper: KevlarFlow (arXiv 2601.22438) P:223-229 §3.2 (background replication
// of each request's KV, block representation, separate stream, promotion on
// the replication target).  Readings R1-R16: DESIGN.md.  The allocator and
// the step protocol follow SURVEY §8(c) steps 1-7 exactly; the CPU oracle
// (oracle/) implements the same rules independently and the tests compare the
// two byte for byte.
#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime_api.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (ranges show up under nsys / ncu)

#include "kvring.h"
#include "kvring_internal.h"

#define KV_API extern "C" __attribute__((visibility("default")))

// Host-side phase counters of the decode path (seconds, cumulative; kv_host_profile).
#include <chrono>
namespace {
enum { kPhPrepAppend = 0, kPhPrepRepl, kPhStage, kPhLaunch, kPhPack, kPhAcquire, kPhH2D,
       kPhEvents, kPhN };
std::atomic<long long> g_phase_ns[kPhN];
inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
inline void phase_add(int i, double v) {
  g_phase_ns[i].fetch_add((long long)(v * 1e9), std::memory_order_relaxed);
}
}  // namespace
KV_API int kv_host_profile(double *out, int32_t n, int32_t reset) {
  for (int i = 0; i < n && i < kPhN; ++i) out[i] = g_phase_ns[i].load() * 1e-9;
  if (reset)
    for (auto &x : g_phase_ns) x.store(0);
  return kPhN;
}

using namespace kvring;

namespace {
// NVTX phase range (SURVEY §5 tracing): append / replicate / decode-loop step / restore.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(KV_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                               \
  } while (0)

// RAII current-device switch (restores the caller's device).
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Lowest-free-id set over [0, n) (reading R6): 64-bit words + first-nonzero hint.
class IdSet {
 public:
  void init(int n, bool full) {
    n_ = n;
    words_.assign((n + 63) / 64, 0ull);
    count_ = 0;
    hint_ = 0;
    if (full)
      for (int i = 0; i < n; ++i) insert(i);
  }
  bool contains(int i) const { return (words_[i >> 6] >> (i & 63)) & 1ull; }
  void insert(int i) {
    words_[i >> 6] |= 1ull << (i & 63);
    ++count_;
    if ((i >> 6) < hint_) hint_ = i >> 6;
  }
  int take_min() {  // precondition: count_ > 0
    while (words_[hint_] == 0ull) ++hint_;
    const int b = __builtin_ctzll(words_[hint_]);
    words_[hint_] &= words_[hint_] - 1ull;
    --count_;
    return hint_ * 64 + b;
  }
  int size() const { return count_; }
  void erase(int i) {
    if (!contains(i)) return;
    words_[i >> 6] &= ~(1ull << (i & 63));
    --count_;
  }

 private:
  int n_ = 0, count_ = 0, hint_ = 0;
  std::vector<unsigned long long> words_;
};

// req_id -> slot map: open addressing, linear probing, backward-shift erase
// (no tombstones).  Capacity is a power of two >= 4 x max_reqs, so probes stay short.
class SlotMap {
 public:
  void init(int max_entries) {
    size_t cap = 16;
    while (cap < 4 * (size_t)max_entries) cap <<= 1;
    keys_.assign(cap, kEmpty);
    vals_.assign(cap, -1);
    mask_ = cap - 1;
    size_ = 0;
  }
  int find(int64_t k) const {
    for (size_t i = hash(k);; i = (i + 1) & mask_) {
      if (keys_[i] == k) return vals_[i];
      if (keys_[i] == kEmpty) return -1;
    }
  }
  void insert(int64_t k, int v) {  // k not present
    size_t i = hash(k);
    while (keys_[i] != kEmpty) i = (i + 1) & mask_;
    keys_[i] = k;
    vals_[i] = v;
    ++size_;
  }
  void erase(int64_t k) {
    size_t i = hash(k);
    while (keys_[i] != k) {
      if (keys_[i] == kEmpty) return;
      i = (i + 1) & mask_;
    }
    for (size_t j = (i + 1) & mask_;; j = (j + 1) & mask_) {  // backward shift
      if (keys_[j] == kEmpty) break;
      const size_t h = hash(keys_[j]);
      const bool move = (j > i) ? (h <= i || h > j) : (h <= i && h > j);
      if (move) {
        keys_[i] = keys_[j];
        vals_[i] = vals_[j];
        i = j;
      }
    }
    keys_[i] = kEmpty;
    vals_[i] = -1;
    --size_;
  }
  size_t size() const { return size_; }

 private:
  static constexpr int64_t kEmpty = INT64_MIN;
  size_t hash(int64_t k) const {
    uint64_t x = (uint64_t)k * 0x9E3779B97F4A7C15ull;
    return (size_t)(x >> 32) & mask_;
  }
  std::vector<int64_t> keys_;
  std::vector<int> vals_;
  size_t mask_ = 0, size_ = 0;
};

// Pinned-host + device staging buffer ring, per device (shared by its pools).
struct StageBuf {
  char *host = nullptr;
  char *hmapped = nullptr;    // device-side address of `host` (zero-copy reads)
  char *dev = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;   // recorded on the consuming stream after the last use
  bool pending = false;
};

struct DeviceCtx {
  int device = 0;
  std::mutex mu;
  static constexpr int kRing = 16;
  StageBuf ring[kRing];
  int next = 0;
  StageBuf src[kRing];  // device copies of host-resident append sources (KV_SRC_HOST)
  int next_src = 0;
  unsigned long long *unpack_counter = nullptr;
  // Descriptor slots of the decode-step engine.  A slot is reused once the pinned word
  // done[slot] (written by the launch's last CTA) shows the nonce of its last launch: the
  // host polls memory instead of recording an event per launch, so nothing but kernels
  // sits between two steps on the stream (a programmatic launch overlaps them).
  static constexpr int kBlobRing = 32;
  struct BlobSlot {
    char *host = nullptr, *hmapped = nullptr, *dev = nullptr;
    size_t cap = 0;
    unsigned long long used = 0;      // nonce of the last launch that read this slot
    unsigned long long arrivals = 0;  // CTAs counted so far on the slot's device counter
  };
  BlobSlot blob[kBlobRing];
  int next_blob = 0;
  unsigned long long *flags = nullptr;     // device: per slot, nonce of the blob its buffer holds
  unsigned long long *counters = nullptr;  // device: per slot, completion counter
  unsigned int *work = nullptr;            // device: per slot, 8 dynamic round counters (512 B)
  volatile unsigned long long *done_host = nullptr;  // pinned host: per slot, last completed nonce
  unsigned long long *done_dev = nullptr;       // its device-side address
  // the last decode-step launch on this device: a chained launch (kvring_step.cu) on the
  // same stream acquires its final count
  cudaStream_t last_stream = nullptr;
  unsigned long long *last_counter = nullptr;
  unsigned long long last_final = 0;   // arrival target of the last launch
  // whether the last launch was chained, and its predecessor's counter / arrival target
  // (an early-started launch waits for that one before any copy: kvring_internal.h)
  bool last_chained = false;
  unsigned long long *last_prev_counter = nullptr;
  unsigned long long last_prev_final = 0;
  // seqs of the last launch if it deferred its publication (kvring_internal.h): the next
  // launch on pend_stream stores them from its publisher CTA
  int n_pend_pub = 0;
  unsigned long long *pend_seq[kStepPools] = {};
  unsigned long long pend_step[kStepPools] = {};
  int pend_sys = 0;
  cudaStream_t pend_stream = nullptr;
  int acquire_blob(size_t bytes, BlobSlot **out, int *index) {
    if (!flags) {
      CU(cudaMalloc(reinterpret_cast<void **>(&flags), 128 * (size_t)kBlobRing));
      CU(cudaMemset(flags, 0, 128 * (size_t)kBlobRing));
      CU(cudaMalloc(reinterpret_cast<void **>(&counters), 128 * (size_t)kBlobRing));
      CU(cudaMemset(counters, 0, 128 * (size_t)kBlobRing));
      CU(cudaMalloc(reinterpret_cast<void **>(&work), 512 * (size_t)kBlobRing));
      CU(cudaMemset(work, 0, 512 * (size_t)kBlobRing));
      CU(cudaDeviceSynchronize());  // once: the zeroed words precede any launch on any stream
      void *h = nullptr;
      CU(cudaHostAlloc(&h, 64 * (size_t)kBlobRing, cudaHostAllocMapped));
      std::memset(h, 0, 64 * (size_t)kBlobRing);
      done_host = static_cast<volatile unsigned long long *>(h);
      CU(cudaHostGetDevicePointer(reinterpret_cast<void **>(&done_dev), h, 0));
    }
    const int i = next_blob;
    next_blob = (next_blob + 1) % kBlobRing;
    BlobSlot &b = blob[i];
    // wait for the slot's previous launch (bounded: a launch that never completes is a
    // sticky CUDA error, surfaced instead of spinning forever)
    const double t0 = now_s();
    for (long long k = 0; done_host[8 * i] < b.used; ++k) {
      if ((k & 1023) == 1023) {
        const cudaError_t e = cudaStreamQuery(nullptr);
        if (e != cudaSuccess && e != cudaErrorNotReady)
          return fail(KV_ECUDA, "decode-step launch failed: %s", cudaGetErrorString(e));
        if (now_s() - t0 > 30.0) return fail(KV_ECUDA, "descriptor slot %d never released", i);
      }
    }
    if (b.cap < bytes) {
      const size_t cap = std::max<size_t>((bytes + 4095) & ~(size_t)4095, 64 << 10);
      if (b.host) cudaFreeHost(b.host);
      if (b.dev) cudaFree(b.dev);
      b.host = b.dev = nullptr;
      CU(cudaHostAlloc(reinterpret_cast<void **>(&b.host), cap, cudaHostAllocMapped));
      CU(cudaHostGetDevicePointer(reinterpret_cast<void **>(&b.hmapped), b.host, 0));
      CU(cudaMalloc(reinterpret_cast<void **>(&b.dev), cap));
      b.cap = cap;
    }
    *out = &b;
    *index = i;
    return KV_OK;
  }
  size_t cap_hint = 8u << 20;       // descriptor slots: 8 MiB (growth never hits a hot loop)
  size_t src_cap_hint = 64u << 20;  // host-source slots: 64 MiB (a 2k-token prefill per stage)

  // Returns a buffer of >= bytes whose previous use has completed.  Growth
  // (cudaFree synchronises the device; cudaHostAlloc costs ms) resizes EVERY slot
  // of the ring at once, doubling, so it happens a handful of times per process
  // instead of once per slot and size.
  int acquire(StageBuf *ringv, int &nxt, size_t bytes, bool want_host, StageBuf **out) {
    StageBuf &b = ringv[nxt];
    nxt = (nxt + 1) % kRing;
    if (b.pending) {
      CU(cudaEventSynchronize(b.ev));
      b.pending = false;
    }
    if (b.cap < bytes) {
      size_t cap = std::max(bytes, b.cap * 2);
      cap = std::max(cap, want_host ? cap_hint : src_cap_hint);
      cap = (cap + 4095) & ~(size_t)4095;
      for (int i = 0; i < kRing; ++i) {
        StageBuf &r = ringv[i];
        if (r.cap >= cap) continue;
        if (r.pending) {
          CU(cudaEventSynchronize(r.ev));
          r.pending = false;
        }
        if (r.host) cudaFreeHost(r.host);
        if (r.dev) cudaFree(r.dev);
        r.host = nullptr;
        r.dev = nullptr;
        r.cap = 0;
        if (want_host) {
          CU(cudaHostAlloc(reinterpret_cast<void **>(&r.host), cap, cudaHostAllocMapped));
          CU(cudaHostGetDevicePointer(reinterpret_cast<void **>(&r.hmapped), r.host, 0));
        }
        CU(cudaMalloc(reinterpret_cast<void **>(&r.dev), cap));
        r.cap = cap;
      }
    }
    if (!b.ev) CU(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
    *out = &b;
    return KV_OK;
  }
  int done(StageBuf *b, cudaStream_t s) {
    CU(cudaEventRecord(b->ev, s));
    b->pending = true;
    return KV_OK;
  }
  // kv_restore's device scratch for the holder's metadata (kept: a failover must not
  // cudaMalloc / cudaFree -- cudaFree synchronises the whole device)
  char *meta_scratch = nullptr;
  size_t meta_scratch_cap = 0;
  int reserve_meta_scratch(size_t bytes) {
    if (meta_scratch_cap >= bytes) return KV_OK;
    if (meta_scratch) cudaFree(meta_scratch);
    meta_scratch = nullptr;
    meta_scratch_cap = 0;
    CU(cudaMalloc(reinterpret_cast<void **>(&meta_scratch), bytes));
    meta_scratch_cap = bytes;
    return KV_OK;
  }
  // Setup-time reservation (kv_pool_create): the staging ring the host-task kernels
  // (restore, ring-put) use and the restore scratch, so their first use on a failover
  // path does not pin / allocate memory (cudaHostAlloc of the ring costs ~100 ms)
  int reserve(size_t meta_bytes_needed) {
    std::lock_guard<std::mutex> lk(mu);
    if (ring[0].cap < cap_hint) {
      StageBuf *b = nullptr;
      int save = next;
      int rc = acquire(ring, next, cap_hint, true, &b);
      next = save;
      if (rc) return rc;
    }
    return reserve_meta_scratch(meta_bytes_needed);
  }
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>> g_ctx;

DeviceCtx *ctx_for(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto &p = g_ctx[device];
  if (!p) {
    p.reset(new DeviceCtx());
    p->device = device;
  }
  return p.get();
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Optional CUDA events recorded right around the next kernel this thread
// launches through libkvring (kv_time_next_launch): kernel-only timing for the
// bench's live roofline, excluding the descriptor H2D that precedes it.
thread_local cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;

cudaError_t timed_launch(int kind, const KvTask *tasks, int n_tasks, const KvPoolParams *params,
                         int n_pools, const KvGeomDev &g, int grid, cudaStream_t st) {
  cudaEvent_t b = g_ev_before, a = g_ev_after;
  g_ev_before = g_ev_after = nullptr;
  if (b) {
    cudaError_t e = cudaEventRecord(b, st);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_copy(kind, tasks, n_tasks, params, n_pools, g, grid, st);
  if (e != cudaSuccess) return e;
  if (a) return cudaEventRecord(a, st);
  return cudaSuccess;
}

}  // namespace

// Growable array of POD tasks: no value-initialisation on growth and no
// per-element capacity check on the emission path (push_item reserves once per
// item) -- the host builds ~1k tasks per decode step.
class TaskVec {
 public:
  TaskVec() = default;
  TaskVec(const TaskVec &) = delete;
  TaskVec &operator=(const TaskVec &) = delete;
  ~TaskVec() { std::free(d_); }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  KvTask *data() { return d_; }
  const KvTask *data() const { return d_; }
  KvTask &operator[](size_t i) { return d_[i]; }
  const KvTask &operator[](size_t i) const { return d_[i]; }
  void clear() { n_ = 0; }
  void resize(size_t n) {  // new elements are uninitialised (shrink in practice)
    reserve(n);
    n_ = n;
  }
  void reserve(size_t n) {
    if (n <= cap_) return;
    size_t c = cap_ ? cap_ : 1024;
    while (c < n) c *= 2;
    KvTask *d = static_cast<KvTask *>(std::realloc(d_, c * sizeof(KvTask)));
    if (!d) throw std::bad_alloc();
    d_ = d;
    cap_ = c;
  }
  KvTask *grow(size_t k) {  // k uninitialised slots at the end
    reserve(n_ + k);
    KvTask *p = d_ + n_;
    n_ += k;
    return p;
  }
  void push_back(const KvTask &t) { *grow(1) = t; }
  KvTask *begin() { return d_; }
  KvTask *end() { return d_ + n_; }
  const KvTask *begin() const { return d_; }
  const KvTask *end() const { return d_ + n_; }

 private:
  KvTask *d_ = nullptr;
  size_t n_ = 0, cap_ = 0;
};

struct kv_loop;

struct kv_pool {
  kv_geom_t g{};
  int NB = 0, R = 0, M = 0, device = -1, node_id = 0, replica_blocks = 0;
  char *pool = nullptr, *replica = nullptr, *meta = nullptr;
  // geometry derived
  long long block_bytes = 0;
  int token_bytes = 0, seg_bytes = 0, combos = 0, task_segs = 0, cps_shift = 0;
  // ring link
  int repl_mode = KV_MODE_TOKENS;  // KV_MODE_BLOCKS: completed blocks only (NEXT-2)
  // mirror of a pool owned by another process (kv_pool_set_mirror): appends update the
  // tables only, `pool` is the owner's pool through NVLink, the holder pulls from it
  bool mirror = false;
  std::vector<int> mirror_q;   // the owner's block ids for the mirror's next appends
  size_t mirror_qi = 0;
  std::vector<int> last_alloc; // block ids the last append call allocated, in order
  bool has_succ = false;
  bool succ_sys = true;  // successor memory is not this GPU's HBM (NVLink peer)
  int succ_node = -1, succ_replica_blocks = 0;
  char *succ_replica = nullptr, *succ_meta = nullptr;
  // allocator (R6, R7)
  IdSet free_blocks, free_slots;
  std::vector<int> q_blocks, q_slots;
  // begin_step count and, per block, the count when it was last released: a deferred
  // publication gates stores into blocks freed one step ago (kvring_internal.h)
  int epoch = 0;
  std::vector<int> freed_at;
  std::vector<int64_t> slot_req;
  std::vector<int32_t> slot_len, pub_len;
  int slot_hi = 0;  // 1 + highest live slot (slots are taken lowest first): loop bound
  std::vector<std::vector<int32_t>> slot_bt;
  SlotMap slot_of;
  std::vector<uint32_t> rel_stamp, app_stamp;  // per-slot call stamps (validation)
  uint32_t call_id = 0;
  std::vector<int64_t> scratch_ids;
  std::vector<int> scratch_slot;  // slot of each append entry found by validation (-1: new)
  // shared-capacity mode (§8(f) NEXT-3, reading R17): the successor
  // `holder` keeps this pool's replicas in ITS OWN pool.  Predecessor side: per
  // slot the holder block ids of the replica, whether it was dropped, and the
  // admission order (eviction age).  Holder side: `rep_src`, the predecessor whose
  // replicas it holds, the census of those blocks, and published-table entries to
  // invalidate on the device before freed replica blocks are reused.
  kv_pool *holder = nullptr, *rep_src = nullptr;
  std::vector<std::vector<int32_t>> rep_bt;
  std::vector<uint8_t> dropped;
  std::vector<uint64_t> admit_seq;
  uint64_t admit_ctr = 0;
  long long census = 0;                       // predecessor side: replica blocks in holder
  struct Inval {
    char *meta;
    int par, slot;
  };
  std::vector<Inval> pending_inval;           // holder side
  uint64_t rep_evictions = 0, rep_drops = 0;
  long long scratch_need = 0;                 // blocks the current append needs
  // state
  bool dead = false;
  uint64_t last_step = 0;
  int abort_slices = -1;                  // fault injection (kv_inject_abort)
  unsigned long long *counter = nullptr;  // device, monotone (host-task ring-put)
  unsigned long long issued = 0;          // host mirror of the counter target
  int32_t *d_bt = nullptr;                // device-resident block table [R][M]
  kv_loop *loop = nullptr;                // decode loop holding a pending publication
  uint64_t bytes_replicated = 0, tasks_launched = 0, kernels = 0, last_step_bytes = 0;

  KvGeomDev geom_dev() const {
    KvGeomDev d;
    d.block_bytes = block_bytes;
    d.token_bytes = token_bytes;
    d.seg_bytes = seg_bytes;
    d.block_size = g.block_size;
    d.cps_shift = cps_shift;
    return d;
  }
  bool same_geom(const kv_pool &o) const {
    return g.layers == o.g.layers && g.kv_heads == o.g.kv_heads && g.head_dim == o.g.head_dim &&
           g.block_size == o.g.block_size && g.elem_bytes == o.g.elem_bytes;
  }
};

namespace {

int validate_geom(const kv_geom_t *g) {
  if (!g) return fail(KV_EINVAL, "null geometry");
  if (g->layers <= 0 || g->kv_heads <= 0 || g->head_dim <= 0 || g->block_size <= 0 ||
      g->block_size > 4096)
    return fail(KV_EINVAL, "geometry fields must be positive (block_size <= 4096)");
  if (g->elem_bytes != 2) return fail(KV_EINVAL, "elem_bytes must be 2 (16-bit words)");
  const int seg = g->head_dim * g->elem_bytes;
  if (seg < 16 || seg > 512 || (seg & (seg - 1)) != 0)
    return fail(KV_EINVAL, "head_dim * elem_bytes = %d must be a power of two in [16, 512]", seg);
  if ((long long)g->block_size * g->layers * 2 * g->kv_heads >= (1LL << 24))
    return fail(KV_EINVAL, "a block must hold fewer than 2^24 (layer, K/V, head, token) slices");
  return KV_OK;
}

// Appends the tasks of one item (n_tok tokens x combos slices) split into
// tasks of <= task_segs slices.
inline void push_item(TaskVec &out, int16_t pool, int src_unit, int dst_unit, int slot,
                      int j, int tok_lo, int n_tok, int combos, int task_segs) {
  const int nseg = n_tok * combos;
  KvTask *t = out.grow((size_t)((nseg + task_segs - 1) / task_segs));
  for (int b = 0; b < nseg; b += task_segs, ++t) {
    t->src_unit = src_unit;
    t->dst_unit = dst_unit;
    t->pool = pool;
    t->slot = (int16_t)slot;
    t->j = (int16_t)j;
    t->tok_lo = (int16_t)tok_lo;
    t->n_tok = (int16_t)n_tok;
    t->flags = b == 0 ? kFirst : 0;
    t->seg_begin = b;
    t->seg_count = std::min(task_segs, nseg - b);
    t->pad = 0;
  }
}

inline void push_publish_only(TaskVec &out, int16_t pool) {
  KvTask t{};
  t.pool = pool;
  t.slot = -1;
  t.n_tok = 1;
  t.seg_count = 0;
  out.push_back(t);
}

// ---- shared capacity (NEXT-3, reading R17) ----------------------------------
// A replica block is freed AT ONCE, after its request is withdrawn from the
// holder's published table (the parity of the step last published): the device
// does that with two small memsets, flushed ahead of the next launch that may
// reuse the block (the holder's append, or the predecessor's ring-put).
void free_rep(kv_pool *p, int s) {
  kv_pool *h = p->holder;
  if (!h || p->rep_bt[s].empty()) return;
  if (p->last_step > 0 && !h->dead && h->device >= 0)
    h->pending_inval.push_back({p->succ_meta, (int)(p->last_step & 1), s});
  for (int b : p->rep_bt[s]) h->free_blocks.insert(b);
  p->census -= (long long)p->rep_bt[s].size();
  p->rep_bt[s].clear();
}

void free_all_reps(kv_pool *p) {
  for (int s = 0; s < p->R; ++s) free_rep(p, s);
}

// Holder side: drop the predecessor's replicas, oldest admission first, until
// `need` blocks are free ("drops the replicated KV cache").
void evict_for(kv_pool *h, long long need) {
  kv_pool *pred = h->rep_src;
  if (!pred) return;
  std::vector<std::pair<uint64_t, int>> order;
  for (int s = 0; s < pred->R; ++s)
    if (pred->slot_req[s] >= 0 && !pred->rep_bt[s].empty())
      order.push_back({pred->admit_seq[s], s});
  std::sort(order.begin(), order.end());
  for (auto &o : order) {
    if (h->free_blocks.size() >= need) break;
    free_rep(pred, o.second);
    pred->dropped[o.second] = 1;
    h->rep_evictions++;
  }
}

// Unlinks a shared predecessor from its holder (replicas freed).
void unlink_holder(kv_pool *p) {
  if (!p->holder) return;
  free_all_reps(p);
  if (p->holder->rep_src == p) p->holder->rep_src = nullptr;
  p->holder = nullptr;
}

inline void slot_taken(kv_pool *p, int s) { p->slot_hi = std::max(p->slot_hi, s + 1); }
inline void slot_freed(kv_pool *p) {
  while (p->slot_hi > 0 && p->slot_req[p->slot_hi - 1] < 0) --p->slot_hi;
}

void admitted(kv_pool *p, int s) {
  p->admit_seq[s] = ++p->admit_ctr;
  p->dropped[s] = 0;
  p->census -= (long long)p->rep_bt[s].size();  // (empty: freed at release)
  p->rep_bt[s].clear();
}

// ---- append ---------------------------------------------------------------
// Validates one pool's releases + appends against `free_b` / `free_s` free
// blocks / slots (the counts after the optional begin_step).  No allocation
// on the hot path: duplicate detection uses per-slot call stamps.
int append_validate(kv_pool *p, const kv_append_args_t &a, long long free_b, long long free_s) {
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  if (a.n < 0 || a.n_release < 0) return fail(KV_EINVAL, "negative count");
  if ((a.n > 0 && (!a.req_ids || !a.n_new)) || (a.n_release > 0 && !a.release_ids))
    return fail(KV_EINVAL, "null array");
  const uint32_t cid = ++p->call_id;
  for (int i = 0; i < a.n_release; ++i) {
    const int rs = p->slot_of.find(a.release_ids[i]);
    if (rs < 0)
      return fail(KV_EINVAL, "release of unknown request %lld", (long long)a.release_ids[i]);
    if (p->rel_stamp[rs] == cid) return fail(KV_EINVAL, "request released twice");
    p->rel_stamp[rs] = cid;
  }
  const int B = p->g.block_size;
  long long need_blocks = 0, need_slots = 0, tokens = 0;
  p->scratch_ids.clear();
  p->scratch_slot.resize(a.n > 0 ? a.n : 0);
  for (int i = 0; i < a.n; ++i) {
    const int64_t r = a.req_ids[i];
    const int n = a.n_new[i];
    if (n < 0) return fail(KV_EINVAL, "negative n_new");
    long long cur = 0;
    const int s = p->slot_of.find(r);
    p->scratch_slot[i] = s;
    if (s >= 0) {
      if (p->app_stamp[s] == cid)
        return fail(KV_EINVAL, "request %lld twice in one append", (long long)r);
      if (p->rel_stamp[s] == cid)
        return fail(KV_EINVAL, "request %lld released and appended", (long long)r);
      p->app_stamp[s] = cid;
      cur = p->slot_len[s];
    } else {
      if (r < 0) return fail(KV_EINVAL, "request ids must be >= 0 (-1 marks an empty slot)");
      if (n <= 0) return fail(KV_EINVAL, "admission of %lld with no tokens", (long long)r);
      p->scratch_ids.push_back(r);
      ++need_slots;
    }
    const long long tot = (cur + n + B - 1) / B;
    if (tot > p->M) return fail(KV_ENOMEM, "request %lld exceeds max_blocks_per_req", (long long)r);
    need_blocks += tot - (cur + B - 1) / B;
    tokens += n;
  }
  if (p->scratch_ids.size() > 1) {
    std::sort(p->scratch_ids.begin(), p->scratch_ids.end());
    for (size_t i = 1; i < p->scratch_ids.size(); ++i)
      if (p->scratch_ids[i] == p->scratch_ids[i - 1])
        return fail(KV_EINVAL, "request %lld twice in one append", (long long)p->scratch_ids[i]);
  }
  // a shared-capacity holder may evict its predecessor's replicas to make room
  // (no rejection while the census could cover the need)
  const long long census = p->rep_src ? p->rep_src->census : 0;
  if (need_slots > free_s || need_blocks > free_b + census)
    return fail(KV_ENOMEM, "pool %d exhausted (need %lld blocks / %lld slots, free %lld / %lld)",
                p->node_id, need_blocks, need_slots, free_b, free_s);
  p->scratch_need = need_blocks;
  if (tokens > 0x7fffffffLL) return fail(KV_EINVAL, "too many tokens in one append");
  return KV_OK;
}

void do_begin_step(kv_pool *p) {
  ++p->epoch;
  for (int b : p->q_blocks) p->free_blocks.insert(b);
  for (int s : p->q_slots) p->free_slots.insert(s);
  p->q_blocks.clear();
  p->q_slots.clear();
}

void do_release(kv_pool *p, int n, const int64_t *ids) {
  for (int i = 0; i < n; ++i) {
    const int s = p->slot_of.find(ids[i]);
    p->slot_of.erase(ids[i]);
    if (p->holder) {
      free_rep(p, s);
      p->dropped[s] = 0;
    }
    for (int b : p->slot_bt[s]) {
      p->q_blocks.push_back(b);
      p->freed_at[b] = p->epoch;
    }
    p->slot_bt[s].clear();
    p->q_slots.push_back(s);
    p->slot_req[s] = -1;
    slot_freed(p);
    p->slot_len[s] = 0;
    p->pub_len[s] = 0;
  }
}

// Applies the appends to the tables and emits the launch's append items (one per
// (slot, block) piece; src rows are token rows of the pool's dense source).  Items
// are emitted for device pools only; `slices` is the running end of the launch's
// append space.  Returns the rows appended.
long long do_append(kv_pool *p, const kv_append_args_t &a, int16_t pidx,
                    std::vector<KvAppItem> &items, int32_t &slices) {
  const int B = p->g.block_size;
  p->last_alloc.clear();
  int row = 0;
  for (int i = 0; i < a.n; ++i) {
    const int64_t r = a.req_ids[i];
    int s = p->scratch_slot[i];  // looked up by append_validate (releases cannot alias it)
    if (s < 0) {
      s = p->free_slots.take_min();
      p->slot_of.insert(r, s);
      p->slot_req[s] = r;
      p->slot_len[s] = 0;
      p->pub_len[s] = 0;
      p->slot_bt[s].clear();
      admitted(p, s);
      slot_taken(p, s);
    }
    int len = p->slot_len[s];
    int left = a.n_new[i];
    while (left > 0) {
      if (len % B == 0) {
        int b;
        if (p->mirror) {  // the owner's choice (its allocator also serves its holder role)
          b = p->mirror_q[p->mirror_qi++];
          p->free_blocks.erase(b);
        } else {
          b = p->free_blocks.take_min();
        }
        p->slot_bt[s].push_back(b);
        p->last_alloc.push_back(b);
      }
      const int j = len / B, lo = len % B;
      const int n = std::min(B - lo, left);
      if (p->device >= 0) {
        KvAppItem it;
        it.off = slices;
        it.row = row;
        it.blk = p->slot_bt[s][j];
        it.p0 = len;
        it.slot = (int16_t)s;
        it.pool = pidx;
        items.push_back(it);
        slices += n * p->combos;
      }
      row += n;
      len += n;
      left -= n;
    }
    p->slot_len[s] = len;
  }
  return row;
}

// ---- replicate --------------------------------------------------------------
// Length a publication of slot s reaches: every appended token (KV_MODE_TOKENS,
// reading R2) or the completed blocks only (KV_MODE_BLOCKS, P:229 literal).
inline int pub_hi(const kv_pool *p, int s) {
  if (p->holder && p->dropped[s]) return 0;  // a dropped replica is never re-sent
  const int len = p->slot_len[s];
  if (p->repl_mode == KV_MODE_BLOCKS) return std::max(p->pub_len[s], len - len % p->g.block_size);
  return len;
}

// Parity table of a publication: (req_id, published length); a slot with
// nothing published yet is listed as empty (-1, 0).
void fill_pub_table(const kv_pool *p, char *dst) {
  int64_t *rq = reinterpret_cast<int64_t *>(dst);
  int32_t *ln = reinterpret_cast<int32_t *>(dst + 8 * (size_t)p->R);
  for (int s = 0; s < p->slot_hi; ++s) {
    const int hi = p->slot_req[s] >= 0 ? pub_hi(p, s) : 0;
    rq[s] = hi > 0 ? p->slot_req[s] : -1;
    ln[s] = hi;
  }
  std::fill(rq + p->slot_hi, rq + p->R, (int64_t)-1);
  std::fill(ln + p->slot_hi, ln + p->R, 0);
}

void commit_pub_len(kv_pool *p) {
  for (int s = 0; s < p->slot_hi; ++s) p->pub_len[s] = p->slot_req[s] >= 0 ? pub_hi(p, s) : 0;
}

// Dirty ranges [pub_len, pub_hi) of every live slot split at block boundaries
// (§8(a) a3); returns payload bytes.
uint64_t build_dirty_tasks(kv_pool *p, int16_t pidx, TaskVec &tasks, bool packed,
                           int32_t *packed_unit, int task_segs,
                           std::vector<int> *ce_blocks = nullptr) {
  const int B = p->g.block_size;
  uint64_t bytes = 0;
  kv_pool *h = p->holder;
  for (int s = 0; s < p->slot_hi; ++s) {
    if (p->slot_req[s] < 0) continue;
    int pos = p->pub_len[s];
    const int len = pub_hi(p, s);
    if (h && pos < len) {
      // shared capacity: the replica's blocks come from the holder's free list
      // (lowest id, R6); a request whose replica cannot grow is dropped
      const long long grow = (long long)ceil_div(len, B) - (long long)p->rep_bt[s].size();
      if (grow > h->free_blocks.size()) {
        free_rep(p, s);
        p->dropped[s] = 1;
        p->rep_drops++;
        continue;
      }
      for (long long k = 0; k < grow; ++k) p->rep_bt[s].push_back(h->free_blocks.take_min());
      p->census += grow;
    }
    while (pos < len) {
      const int j = pos / B, lo = pos % B;
      const int n = std::min(B - lo, len - pos);
      const int blk = p->slot_bt[s][j];
      if (h) {
        push_item(tasks, pidx, blk, p->rep_bt[s][j], s, j, lo, n, p->combos, task_segs);
      } else if (ce_blocks && lo == 0 && n == B) {
        // copy-engine variant: the whole block moves by cudaMemcpyAsync; the kernel
        // only writes its bt entry (a zero-slice task) and counts it for publication
        KvTask t{};
        t.src_unit = t.dst_unit = blk;
        t.pool = pidx;
        t.slot = (int16_t)s;
        t.j = (int16_t)j;
        t.n_tok = (int16_t)B;
        t.flags = kFirst;
        tasks.push_back(t);
        ce_blocks->push_back(blk);
      } else if (packed) {
        push_item(tasks, pidx, blk, *packed_unit, s, j, lo, n, p->combos, task_segs);
        *packed_unit += n * p->combos;
      } else {
        push_item(tasks, pidx, blk, blk, s, j, lo, n, p->combos, task_segs);
      }
      bytes += (uint64_t)n * p->token_bytes;
      pos += n;
    }
  }
  return bytes;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
KV_API int32_t kv_abi_version(void) { return KVRING_ABI_VERSION; }

KV_API const char *kv_last_error(void) { return g_err.c_str(); }

KV_API uint64_t kv_kernel_launch_count(void) { return g_launches.load(); }

KV_API int kv_time_next_launch(void *ev_before, void *ev_after) {
  g_ev_before = static_cast<cudaEvent_t>(ev_before);
  g_ev_after = static_cast<cudaEvent_t>(ev_after);
  return KV_OK;
}

KV_API size_t kv_block_bytes(const kv_geom_t *g) {
  if (!g || validate_geom(g) != KV_OK) return 0;
  return (size_t)g->layers * 2 * g->kv_heads * g->block_size * g->head_dim * g->elem_bytes;
}

KV_API size_t kv_meta_bytes(int32_t max_reqs, int32_t max_blocks_per_req) {
  if (max_reqs <= 0 || max_blocks_per_req <= 0) return 0;
  return meta_bytes(max_reqs, max_blocks_per_req);
}

KV_API int kv_pool_create(const kv_pool_desc_t *d, kv_pool_t **out) {
  if (!d || !out) return fail(KV_EINVAL, "null argument");
  *out = nullptr;
  int rc = validate_geom(&d->g);
  if (rc) return rc;
  if (d->num_blocks <= 0 || d->max_reqs <= 0 || d->max_blocks_per_req <= 0)
    return fail(KV_EINVAL, "num_blocks, max_reqs, max_blocks_per_req must be positive");
  if (d->max_reqs > 32767 || d->max_blocks_per_req > 32767)
    return fail(KV_EINVAL, "max_reqs and max_blocks_per_req must be < 32768");
  if (d->device >= 0 && (!d->pool || !d->replica || !d->replica_meta))
    return fail(KV_EINVAL, "pool, replica and replica_meta must be device pointers");
  std::unique_ptr<kv_pool> p(new kv_pool());
  p->g = d->g;
  p->NB = d->num_blocks;
  p->R = d->max_reqs;
  p->M = d->max_blocks_per_req;
  p->device = d->device;
  p->node_id = d->node_id;
  p->replica_blocks = d->replica_blocks > 0 ? d->replica_blocks : d->num_blocks;
  p->pool = static_cast<char *>(d->pool);
  p->replica = static_cast<char *>(d->replica);
  p->meta = static_cast<char *>(d->replica_meta);
  p->seg_bytes = d->g.head_dim * d->g.elem_bytes;
  p->combos = d->g.layers * 2 * d->g.kv_heads;
  p->token_bytes = p->combos * p->seg_bytes;
  p->block_bytes = (long long)p->token_bytes * d->g.block_size;
  p->task_segs = std::max(1, 32768 / p->seg_bytes);
  p->cps_shift = __builtin_ctz(p->seg_bytes / 16);
  p->free_blocks.init(p->NB, true);
  p->freed_at.assign(p->NB, -(1 << 29));
  p->free_slots.init(p->R, true);
  p->slot_req.assign(p->R, -1);
  p->slot_len.assign(p->R, 0);
  p->pub_len.assign(p->R, 0);
  p->slot_bt.assign(p->R, {});
  p->rel_stamp.assign(p->R, 0);
  p->app_stamp.assign(p->R, 0);
  p->slot_of.init(p->R);
  for (auto &v : p->slot_bt) v.reserve(8);
  p->rep_bt.assign(p->R, {});
  p->dropped.assign(p->R, 0);
  p->admit_seq.assign(p->R, 0);
  if (p->device >= 0) {
    DeviceGuard dg(p->device);
    if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice(%d) failed", p->device);
    CU(cudaMalloc(reinterpret_cast<void **>(&p->counter), 2 * sizeof(unsigned long long)));
    CU(cudaMemset(p->counter, 0, 2 * sizeof(unsigned long long)));
    CU(cudaMalloc(reinterpret_cast<void **>(&p->d_bt), sizeof(int32_t) * (size_t)p->R * p->M));
    CU(cudaMemset(p->d_bt, 0xFF, sizeof(int32_t) * (size_t)p->R * p->M));
    CU(launch_meta_init(p->meta, p->R, p->M, 0));
    g_launches++;
    p->kernels++;
    CU(cudaDeviceSynchronize());
    rc = ctx_for(p->device)->reserve(meta_bytes(p->R, p->M));
    if (rc) return rc;
  }
  *out = p.release();
  return KV_OK;
}

namespace {
void loop_forget(kv_loop *L, kv_pool *p);
}  // namespace

KV_API int kv_pool_destroy(kv_pool_t *p) {
  if (!p) return KV_OK;
  if (p->holder) unlink_holder(p);
  if (p->rep_src) {
    p->rep_src->census = 0;
    for (auto &v : p->rep_src->rep_bt) v.clear();
    p->rep_src->holder = nullptr;
    p->rep_src->has_succ = false;
    p->rep_src = nullptr;
  }
  if (p->loop) loop_forget(p->loop, p);
  if (p->counter) {
    DeviceGuard dg(p->device);
    cudaDeviceSynchronize();
    cudaFree(p->counter);
    cudaFree(p->d_bt);
  }
  delete p;
  return KV_OK;
}

KV_API int kv_set_successor(kv_pool_t *p, int32_t succ_node, void *succ_replica,
                            int32_t succ_replica_blocks, void *succ_meta) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  unlink_holder(p);  // leaving shared-capacity mode frees the replicas it held
  std::fill(p->dropped.begin(), p->dropped.end(), 0);
  if (succ_replica == nullptr) {
    p->has_succ = false;
    p->succ_replica = nullptr;
    p->succ_meta = nullptr;
    p->succ_node = -1;
  } else {
    if (!succ_meta) return fail(KV_EINVAL, "successor metadata pointer is null");
    if (succ_replica_blocks < p->NB)
      return fail(KV_EINVAL, "successor replica region (%d blocks) smaller than pool (%d)",
                  succ_replica_blocks, p->NB);
    p->has_succ = true;
    p->succ_sys = true;
    if (p->device >= 0) {
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, succ_replica) == cudaSuccess &&
          at.type == cudaMemoryTypeDevice) {
        if (at.device == p->device) {
          p->succ_sys = false;
        } else {
          // a successor on another GPU of this process (plain cudaMalloc memory, not an
          // IPC / symmetric-memory mapping): the stores need peer access
          DeviceGuard dg(p->device);
          int can = 0;
          if (cudaDeviceCanAccessPeer(&can, p->device, at.device) == cudaSuccess && can)
            cudaDeviceEnablePeerAccess(at.device, 0);  // already enabled: harmless error
        }
      }
      cudaGetLastError();
    }
    p->succ_node = succ_node;
    p->succ_replica = static_cast<char *>(succ_replica);
    p->succ_replica_blocks = succ_replica_blocks;
    p->succ_meta = static_cast<char *>(succ_meta);
  }
  std::fill(p->pub_len.begin(), p->pub_len.end(), 0);  // re-seed the new link
  return KV_OK;
}

KV_API int kv_set_successor_shared(kv_pool_t *p, kv_pool_t *h) {
  if (!p || !h) return fail(KV_EINVAL, "null pool");
  if (p == h) return fail(KV_EINVAL, "a pool cannot hold its own replicas");
  if (p->dead || h->dead) return fail(KV_ESTATE, "pool is dead");
  if (p->device != h->device || !p->same_geom(*h) || p->R != h->R || p->M != h->M)
    return fail(KV_EINVAL, "shared capacity needs the same device, geometry, max_reqs, max_blocks");
  unlink_holder(p);
  if (h->rep_src && h->rep_src != p) unlink_holder(h->rep_src);  // one predecessor per holder
  if (h->rep_src == p) h->rep_src = nullptr;
  p->holder = h;
  h->rep_src = p;
  p->has_succ = true;
  p->succ_sys = false;
  p->succ_node = h->node_id;
  p->succ_replica = h->pool;  // the replica lives in the holder's own pool
  p->succ_replica_blocks = h->NB;
  p->succ_meta = h->meta;
  std::fill(p->pub_len.begin(), p->pub_len.end(), 0);  // re-seed
  std::fill(p->dropped.begin(), p->dropped.end(), 0);
  return KV_OK;
}

KV_API int kv_pool_set_mirror(kv_pool_t *p, int32_t on) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->device < 0) return fail(KV_EINVAL, "a mirror needs a device (the holder's)");
  if (p->slot_hi > 0 || p->last_step > 0 || p->free_blocks.size() != p->NB)
    return fail(KV_ESTATE, "mirror a pool before its first append");
  p->mirror = on != 0;
  return KV_OK;
}

KV_API int kv_mirror_blocks(kv_pool_t *p, int32_t n, const int32_t *block_ids) {
  if (!p || (n > 0 && !block_ids)) return fail(KV_EINVAL, "null argument");
  if (!p->mirror) return fail(KV_EINVAL, "pool %d is not a mirror", p->node_id);
  if (p->mirror_qi == p->mirror_q.size()) {
    p->mirror_q.clear();
    p->mirror_qi = 0;
  }
  for (int i = 0; i < n; ++i) {
    if (block_ids[i] < 0 || block_ids[i] >= p->NB) return fail(KV_EINVAL, "block id out of range");
    p->mirror_q.push_back(block_ids[i]);
  }
  return KV_OK;
}

KV_API int kv_last_alloc(kv_pool_t *p, int32_t *out, int32_t cap) {
  if (!p) return fail(KV_EINVAL, "null pool");
  const int n = (int)p->last_alloc.size();
  if (out)
    for (int i = 0; i < n && i < cap; ++i) out[i] = p->last_alloc[i];
  return n;
}

KV_API int kv_drop_replicas(kv_pool_t *h) {
  if (!h) return fail(KV_EINVAL, "null pool");
  kv_pool *pred = h->rep_src;
  if (!pred) return KV_OK;
  for (int s = 0; s < pred->R; ++s)
    if (!pred->rep_bt[s].empty()) {
      free_rep(pred, s);
      pred->dropped[s] = 1;
    }
  if (pred->dead) {
    pred->holder = nullptr;
    h->rep_src = nullptr;
  }
  return KV_OK;
}

KV_API int kv_begin_step(kv_pool_t *p) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  do_begin_step(p);
  return KV_OK;
}

KV_API int kv_release(kv_pool_t *p, int32_t n, const int64_t *req_ids) {
  if (!p) return fail(KV_EINVAL, "null pool");
  kv_append_args_t a{};
  a.pool = p;
  a.n_release = n;
  a.release_ids = req_ids;
  int rc = append_validate(p, a, p->free_blocks.size(), p->free_slots.size());
  if (rc) return rc;
  do_release(p, n, req_ids);
  return KV_OK;
}

namespace {

// ---- host-task launches (restore, pack, shared-capacity + copy-engine ring-put) ----
inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// One host-task kernel launch prepared on the host.
struct Launch {
  int kind = kKindRingPut;
  int n_pools = 0;
  kv_pool *p0 = nullptr;
  std::vector<KvPoolParams> params;
  std::vector<char> tables;        // replicate: per pool slot_req[R] (8R B) then slot_len[R] (4R B)
  std::vector<size_t> table_off;   // per pool offset into `tables`
  TaskVec tasks;
  std::vector<int> ntask;          // replicate: tasks per pool
  std::vector<uint64_t> bytes;     // replicate: payload bytes per pool
  std::vector<std::vector<int>> ce_blocks;  // copy-engine variant: full blocks per pool
  bool use_ce = false;
  std::vector<kv_pool::Inval> inval;  // shared capacity: published entries to withdraw first
  int max_reqs_inval = 0;
  // filled by stage()
  const KvPoolParams *params_dev = nullptr;
  const KvTask *tasks_dev = nullptr;
  void reset(int kind_, int n) {
    kind = kind_;
    n_pools = n;
    params.assign(n, KvPoolParams{});
    tables.clear();
    table_off.assign(n, 0);
    tasks.clear();
    ntask.assign(n, 0);
    bytes.assign(n, 0);
    if ((int)ce_blocks.size() < n) ce_blocks.resize(n);
    for (auto &v : ce_blocks) v.clear();
    use_ce = false;
    inval.clear();
    params_dev = nullptr;
    tasks_dev = nullptr;
  }
  size_t staged_bytes() const {
    return align16(sizeof(KvPoolParams) * n_pools) + align16(tables.size()) +
           sizeof(KvTask) * tasks.size();
  }
};

// Moves the pending published-entry invalidations of every holder a launch
// touches (its pools, and the holders of its pools) into `out`.
void collect_inval(std::vector<kv_pool::Inval> &out, int &max_reqs, kv_pool *const *pools,
                   int n) {
  auto take = [&](kv_pool *h) {
    if (!h || h->pending_inval.empty()) return;
    max_reqs = h->R;
    out.insert(out.end(), h->pending_inval.begin(), h->pending_inval.end());
    h->pending_inval.clear();
  };
  for (int k = 0; k < n; ++k) {
    take(pools[k]);
    take(pools[k]->holder);
  }
}

int check_same_device(int n, kv_pool *const *pools) {
  kv_pool *p0 = pools[0];
  for (int k = 0; k < n; ++k) {
    kv_pool *p = pools[k];
    if (!p) return fail(KV_EINVAL, "null pool");
    if (p->device != p0->device || !p->same_geom(*p0))
      return fail(KV_EINVAL, "pools of one launch must share device and geometry");
    for (int k2 = 0; k2 < k; ++k2)
      if (pools[k2] == p) return fail(KV_EINVAL, "pool listed twice");
  }
  return KV_OK;
}

// Checks shared by both publication paths (state is not touched).
int validate_replicate(int n_pools, kv_pool *const *pools, uint64_t step) {
  if (n_pools <= 0 || !pools) return fail(KV_EINVAL, "no pools");
  if (n_pools > kMaxPoolsPerLaunchHost)
    return fail(KV_EINVAL, "at most %d pools per launch", kMaxPoolsPerLaunchHost);
  if (!pools[0]) return fail(KV_EINVAL, "null pool");
  int rc = check_same_device(n_pools, pools);
  if (rc) return rc;
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k];
    if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
    if (!p->has_succ) return fail(KV_EPEER, "pool %d has no successor", p->node_id);
    if (step == 0 || step <= p->last_step)
      return fail(KV_EINVAL, "step %llu not > last step %llu of pool %d",
                  (unsigned long long)step, (unsigned long long)p->last_step, p->node_id);
  }
  return KV_OK;
}

// Host-task publication (shared-capacity links: the replica's block ids come from
// the holder's allocator; the copy-engine variant): the host builds the dirty work
// list (build_dirty_tasks); state is committed by commit_replicate once enqueued.
int prepare_replicate(int n_pools, kv_pool *const *pools, uint64_t step, Launch &L,
                      bool use_ce) {
  int rc = validate_replicate(n_pools, pools, step);
  if (rc) return rc;
  L.reset(kKindRingPut, n_pools);
  L.p0 = pools[0];
  L.use_ce = use_ce;
  size_t toff = 0;
  for (int k = 0; k < n_pools; ++k) toff += 12 * (size_t)pools[k]->R;
  L.tables.resize(toff);
  toff = 0;
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k];
    const size_t before = L.tasks.size();
    L.bytes[k] = build_dirty_tasks(p, (int16_t)k, L.tasks, false, nullptr, p->task_segs,
                                   use_ce ? &L.ce_blocks[k] : nullptr);
    if (L.tasks.size() == before) push_publish_only(L.tasks, (int16_t)k);
    L.tasks[before].flags |= kPoolFirst;
    L.ntask[k] = (int)(L.tasks.size() - before);
    const bool aborting = p->abort_slices >= 0;  // a stage dying mid-step: never published
    if (aborting) {
      // the first abort_slices slices of the step (task order) are copied
      long long left = p->abort_slices;
      size_t keep = before;
      while (keep < L.tasks.size() && left > 0) {
        KvTask &t = L.tasks[keep];
        if (t.seg_count > left) t.seg_count = (int32_t)left;
        left -= t.seg_count;
        ++keep;
      }
      L.tasks.resize(keep);
      L.ntask[k] = (int)(keep - before);
    }
    L.table_off[k] = toff;
    fill_pub_table(p, L.tables.data() + toff);
    toff += 12 * (size_t)p->R;
    KvPoolParams &pp = L.params[k];
    pp.src = p->pool;
    pp.dst = p->succ_replica;
    pp.meta = p->succ_meta;
    pp.src_bytes = (unsigned long long)p->NB * p->block_bytes;
    pp.dst_bytes = (unsigned long long)p->succ_replica_blocks * p->block_bytes;
    pp.counter = p->counter;
    pp.target = aborting ? ~0ull : p->issued + (unsigned long long)L.ntask[k];
    pp.step = step;
    pp.max_reqs = p->R;
    pp.max_blk = p->M;
    pp.n_table = p->R;
    pp.writer_node = p->node_id;
    pp.publish = aborting ? 0 : 1;
    pp.sys_scope = p->succ_sys ? 1 : 0;
  }
  collect_inval(L.inval, L.max_reqs_inval, pools, n_pools);
  return KV_OK;
}

// Publication state after an enqueued host-task replicate (aborted pools publish
// nothing: their host state stays at the previous publication).
void commit_replicate(Launch &L, kv_pool *const *pools, uint64_t step) {
  for (int k = 0; k < L.n_pools; ++k) {
    kv_pool *p = pools[k];
    p->issued += (unsigned long long)L.ntask[k];
    p->tasks_launched += L.ntask[k];
    if (p->abort_slices >= 0) {
      p->abort_slices = -1;
      continue;
    }
    p->last_step_bytes = L.bytes[k];
    p->bytes_replicated += L.bytes[k];
    commit_pub_len(p);
    p->last_step = step;
  }
}

// Stages the descriptors of a host-task launch with ONE pinned H2D copy.
int stage(DeviceCtx *ctx, Launch &L, cudaStream_t st, StageBuf **out) {
  StageBuf *b = nullptr;
  const double t0 = now_s();
  int rc = ctx->acquire(ctx->ring, ctx->next, L.staged_bytes(), true, &b);
  if (rc) return rc;
  const size_t pbytes = align16(sizeof(KvPoolParams) * L.n_pools);
  const size_t tbl = align16(L.tables.size());
  char *h = b->host;
  char *d = b->dev;
  for (int k = 0; k < L.n_pools; ++k) {
    if (L.kind == kKindRingPut) {
      const size_t o = pbytes + L.table_off[k];
      L.params[k].slot_req = reinterpret_cast<const int64_t *>(d + o);
      L.params[k].slot_len = reinterpret_cast<const int32_t *>(d + o + 8 * (size_t)L.params[k].max_reqs);
    }
  }
  std::memcpy(h, L.params.data(), sizeof(KvPoolParams) * L.n_pools);
  if (!L.tables.empty()) std::memcpy(h + pbytes, L.tables.data(), L.tables.size());
  std::memcpy(h + pbytes + tbl, L.tasks.data(), sizeof(KvTask) * L.tasks.size());
  L.params_dev = reinterpret_cast<const KvPoolParams *>(d);
  L.tasks_dev = reinterpret_cast<const KvTask *>(d + pbytes + tbl);
  CU(cudaMemcpyAsync(b->dev, b->host, L.staged_bytes(), cudaMemcpyHostToDevice, st));
  phase_add(kPhStage, now_s() - t0);
  *out = b;
  return KV_OK;
}

// Shared capacity: withdraw the freed replicas' published entries (req_id -1,
// len 0 in the published parity) before a launch may reuse their blocks.
int flush_inval(std::vector<kv_pool::Inval> &inval, int R, cudaStream_t st) {
  for (const auto &iv : inval) {
    CU(cudaMemsetAsync(iv.meta + 32 + ((size_t)iv.par * R + iv.slot) * 8, 0xFF, 8, st));
    CU(cudaMemsetAsync(iv.meta + meta_off_len(R) + ((size_t)iv.par * R + iv.slot) * 4, 0, 4, st));
  }
  inval.clear();
  return KV_OK;
}

int enqueue(Launch &L, cudaStream_t st) {
  if (!L.inval.empty() && L.p0 && L.p0->device >= 0) {
    int rc = flush_inval(L.inval, L.max_reqs_inval, st);
    if (rc) return rc;
  }
  if (L.tasks.empty()) return KV_OK;
  CU(timed_launch(L.kind, L.tasks_dev, (int)L.tasks.size(), L.params_dev, L.n_pools,
                  L.p0->geom_dev(), copy_grid(L.p0->device, (int)L.tasks.size()), st));
  g_launches++;
  L.p0->kernels++;
  return KV_OK;
}

// Copy-engine runs of the full blocks of a ring-put launch (consecutive block ids
// coalesced into ONE cudaMemcpyAsync each; the replica mirrors block ids, R5), issued
// before the kernel on the same stream: the kernel's publication is stream-ordered
// after them.
int issue_ce_copies(Launch &L, kv_pool *const *pools, cudaStream_t st) {
  for (int k = 0; k < L.n_pools; ++k) {
    std::vector<int> &v = L.ce_blocks[k];
    if (v.empty()) continue;
    kv_pool *p = pools[k];
    std::sort(v.begin(), v.end());
    size_t i = 0;
    while (i < v.size()) {
      size_t e = i + 1;
      while (e < v.size() && v[e] == v[e - 1] + 1) ++e;
      const size_t off = (size_t)v[i] * (size_t)p->block_bytes;
      CU(cudaMemcpyAsync(p->succ_replica + off, p->pool + off,
                         (e - i) * (size_t)p->block_bytes, cudaMemcpyDefault, st));
      i = e;
    }
  }
  return KV_OK;
}

int replicate_host_tasks(int n_pools, kv_pool *const *pools, uint64_t step, cudaStream_t st,
                         bool use_ce) {
  thread_local Launch L;
  int rc = prepare_replicate(n_pools, pools, step, L, use_ce);
  if (rc) return rc;
  if (L.p0->device < 0) {  // tables only
    commit_replicate(L, pools, step);
    return KV_OK;
  }
  DeviceGuard dg(L.p0->device);
  if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice failed");
  DeviceCtx *ctx = ctx_for(L.p0->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  StageBuf *b = nullptr;
  rc = stage(ctx, L, st, &b);
  if (rc) return rc;
  if (use_ce && (rc = issue_ce_copies(L, pools, st))) return rc;
  rc = enqueue(L, st);
  if (rc) return rc;
  commit_replicate(L, pools, step);
  return ctx->done(b, st);
}

// ---- decode-step engine launches (kvring_step.cu) --------------------------------
// One StepLaunch = one kernel: the appends of a step (items from the host allocator)
// and/or a publication whose work list the device derives from per-slot snapshots.
struct StepLaunch {
  KvStepHdr h{};
  int device = -1;
  kv_pool *app_pool[kStepPools] = {};
  kv_pool *rep_pool[kStepPools] = {};
  std::vector<KvAppItem> items;
  std::vector<int64_t> req;          // replicate snapshots, entry-major (pool, slot)
  std::vector<int32_t> len, pub, blk0;
  bool pdl = false;  // launched as a programmatic dependent of the previous step's grid
  bool chain_ok = false;  // the previous kernel on the stream is this library's step launch
  bool defer_next = false;  // the next launch on the stream is chained (it may publish ours)
  std::vector<char> blob;
  const void *host_src[kStepPools] = {};  // KV_SRC_HOST sources
  size_t host_src_bytes[kStepPools] = {};
  uint64_t app_bytes = 0, rep_bytes = 0;
  uint64_t rep_pool_bytes[kStepPools] = {};
  uint64_t rep_step = 0;
  std::vector<kv_pool::Inval> inval;
  int max_reqs_inval = 0;
  void reset() {
    h = KvStepHdr{};
    device = -1;
    for (int i = 0; i < kStepPools; ++i) {
      app_pool[i] = rep_pool[i] = nullptr;
      host_src[i] = nullptr;
      host_src_bytes[i] = 0;
      rep_pool_bytes[i] = 0;
    }
    items.clear();
    req.clear();
    len.clear();
    pub.clear();
    blk0.clear();
    pdl = false;
    chain_ok = false;
    defer_next = false;
    app_bytes = rep_bytes = 0;
    rep_step = 0;
    inval.clear();
  }
  bool empty() const { return h.n_app == 0 && h.n_rep == 0; }
};

void set_geom(StepLaunch &S, const kv_pool *p) {
  if (S.device >= 0 || S.h.n_app + S.h.n_rep > 0) return;
  S.device = p->device;
  S.h.g = p->geom_dev();
  S.h.div_sl = kv_div((uint32_t)p->combos);
  S.h.div_b = kv_div((uint32_t)p->g.block_size);
  S.h.div_bs = kv_div((uint32_t)(p->g.block_size * p->combos));
}

// Appends a pool's items (do_append) to the launch.  Item slices are token-major:
// the launch's append space is the concatenation of every item's n_tok x combos.
void step_add_append(StepLaunch &S, kv_pool *p, const kv_append_args_t &a) {
  set_geom(S, p);
  const int q = S.h.n_app++;
  S.app_pool[q] = p;
  KvStepPool &pp = S.h.app[q];
  pp.src = static_cast<const char *>(a.src_kv);
  pp.dst = p->pool;
  pp.bt = p->d_bt;
  pp.R = p->R;
  pp.M = p->M;
  pp.abort_slices = -1;
  const size_t i0 = S.items.size();
  long long rows = do_append(p, a, (int16_t)q, S.items, S.h.app_slices);
  S.app_bytes += (uint64_t)rows * p->token_bytes;
  // blocks freed one step ago: the previous launch's publication may still read them
  // while an early-started launch appends (kItemGated)
  for (size_t i = i0; i < S.items.size(); ++i)
    if (p->freed_at[S.items[i].blk] >= p->epoch - 1) S.items[i].blk |= kItemGated;
  if ((a.flags & KV_SRC_HOST) && rows > 0) {
    S.host_src[q] = a.src_kv;
    S.host_src_bytes[q] = (size_t)rows * p->token_bytes;
  }
}

// Snapshots a pool's publication (tables as they are now) into the launch and
// commits it on the host: pub_len := the published length of every live slot.
// The device derives the same dirty ranges from the snapshot (reading R2).
void step_add_replicate(StepLaunch &S, kv_pool *p, uint64_t step) {
  set_geom(S, p);
  const int q = S.h.n_rep++;
  S.rep_pool[q] = p;
  S.rep_step = step;
  KvStepPool &pp = S.h.rep[q];
  pp.src = p->pool;
  pp.dst = p->succ_replica;
  pp.meta = p->succ_meta;
  pp.bt = p->d_bt;
  pp.step = step;
  pp.R = p->R;
  pp.M = p->M;
  pp.n_slots = p->slot_hi;
  pp.ent_off = S.h.n_ent;
  pp.mode = p->repl_mode;
  pp.abort_slices = p->abort_slices;
  pp.writer_node = p->node_id;
  pp.sys = p->succ_sys ? 1 : 0;
  S.h.n_ent += p->slot_hi;
  S.req.insert(S.req.end(), p->slot_req.begin(), p->slot_req.begin() + p->slot_hi);
  S.len.insert(S.len.end(), p->slot_len.begin(), p->slot_len.begin() + p->slot_hi);
  S.pub.insert(S.pub.end(), p->pub_len.begin(), p->pub_len.begin() + p->slot_hi);
  uint64_t bytes = 0;
  const int B = p->g.block_size;
  for (int s = 0; s < p->slot_hi; ++s) {
    int b0 = -1;
    if (p->slot_req[s] >= 0) {
      const int lo = p->pub_len[s], hi = pub_hi(p, s);
      bytes += (uint64_t)(hi - lo);
      if (hi > lo) {
        b0 = p->slot_bt[s][lo / B];  // the block of the first dirty token
        // blocks with no published token that were freed one step ago: the last stored
        // seq may still list them (only matters when this publication is deferred)
        for (int j = (lo + B - 1) / B; j <= (hi - 1) / B; ++j)
          if (p->freed_at[p->slot_bt[s][j]] >= p->epoch - 1) {
            b0 |= 1 << 30;
            break;
          }
      }
    }
    S.blk0.push_back(b0);
  }
  bytes *= (uint64_t)p->token_bytes;
  if (pp.abort_slices >= 0) {  // a stage dying mid-step: partial copy, never published
    const uint64_t cut = (uint64_t)pp.abort_slices * (uint64_t)p->seg_bytes;
    S.rep_pool_bytes[q] = 0;
    S.rep_bytes += std::min(bytes, cut);
    p->abort_slices = -1;
  } else {
    S.h.publish = 1;
    S.h.sys_any |= pp.sys;
    S.rep_pool_bytes[q] = bytes;
    S.rep_bytes += bytes;
    p->last_step_bytes = bytes;
    p->bytes_replicated += bytes;
    commit_pub_len(p);
    p->last_step = step;
  }
  if (pp.abort_slices >= 0) S.h.any_abort = 1;
}

// Prepares the publication part: validation, then snapshot + commit of each pool.
int step_prepare_replicate(StepLaunch &S, int n_pools, kv_pool *const *pools, uint64_t step) {
  int rc = validate_replicate(n_pools, pools, step);
  if (rc) return rc;
  if (S.h.n_app > 0 && S.device != pools[0]->device)
    return fail(KV_EINVAL, "append and publication of one launch must share a device");
  long long ent = S.h.n_ent;
  for (int k = 0; k < n_pools; ++k) {
    if (pools[k]->holder) return fail(KV_EINVAL, "shared-capacity links publish through the host-task path");
    ent += pools[k]->slot_hi;
  }
  if (S.h.n_rep + n_pools > kStepPools || ent > kStepMaxEnt)
    return fail(KV_EINVAL, "too many pools / slots for one launch (%d pools, %lld slots)",
                S.h.n_rep + n_pools, ent);
  for (int k = 0; k < n_pools; ++k) step_add_replicate(S, pools[k], step);
  return KV_OK;
}

// Validates every pool of an append (all-or-nothing: nothing changes on error).
int validate_appends(int n_pools, const kv_append_args_t *args) {
  if (n_pools <= 0 || !args) return fail(KV_EINVAL, "no pools");
  if (n_pools > kMaxPoolsPerLaunchHost)
    return fail(KV_EINVAL, "at most %d pools per append", kMaxPoolsPerLaunchHost);
  kv_pool *pools[kMaxPoolsPerLaunchHost];
  for (int k = 0; k < n_pools; ++k) pools[k] = args[k].pool;
  if (!pools[0]) return fail(KV_EINVAL, "null pool");
  int rc = check_same_device(n_pools, pools);
  if (rc) return rc;
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k];
    if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
    const bool bs = args[k].begin_step != 0;  // validation sees the released quarantine
    rc = append_validate(p, args[k],
                         p->free_blocks.size() + (bs ? (long long)p->q_blocks.size() : 0),
                         p->free_slots.size() + (bs ? (long long)p->q_slots.size() : 0));
    if (rc) return rc;
    long long rows = 0;
    for (int i = 0; i < args[k].n; ++i) rows += args[k].n_new[i];
    if (p->mirror && p->scratch_need > (long long)(p->mirror_q.size() - p->mirror_qi))
      return fail(KV_ESTATE, "mirror %d: %lld new blocks but %lld owner block ids queued",
                  p->node_id, p->scratch_need, (long long)(p->mirror_q.size() - p->mirror_qi));
    if (p->device >= 0 && !p->mirror && rows > 0 && !args[k].src_kv)
      return fail(KV_EINVAL, "null src_kv with tokens to append");
    if (rows * p->combos > (long long)INT32_MAX / 4)
      return fail(KV_EINVAL, "append too large for one launch");
  }
  return KV_OK;
}

// Applies begin_step / releases / appends of <= kStepPools validated pools to the
// host tables, building the launch's append items.
void apply_appends(StepLaunch &S, int n_pools, const kv_append_args_t *args) {
  kv_pool *pools[kStepPools];
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k] = args[k].pool;
    if (args[k].begin_step) do_begin_step(p);
    do_release(p, args[k].n_release, args[k].release_ids);
    if (p->scratch_need > p->free_blocks.size()) evict_for(p, p->scratch_need);
    if (p->mirror) {  // the owner moves the bytes: tables only
      set_geom(S, p);  // the device of withdrawals this append may cause on the holder
      std::vector<KvAppItem> none;
      int32_t sl = 0;
      do_append(p, args[k], 0, none, sl);
      continue;
    }
    step_add_append(S, p, args[k]);
  }
  collect_inval(S.inval, S.max_reqs_inval, pools, n_pools);
}

// Pinned host sources are read by the kernel over PCIe (zero copy); pageable ones
// are copied into a staging buffer in stream order.
int step_stage_host_sources(DeviceCtx *ctx, StepLaunch &S, cudaStream_t st, StageBuf **out) {
  *out = nullptr;
  size_t total = 0;
  for (int k = 0; k < S.h.n_app; ++k) {
    if (!S.host_src_bytes[k]) continue;
    cudaPointerAttributes at;
    void *dptr = nullptr;
    if (cudaPointerGetAttributes(&at, S.host_src[k]) == cudaSuccess &&
        at.type == cudaMemoryTypeHost &&
        cudaHostGetDevicePointer(&dptr, const_cast<void *>(S.host_src[k]), 0) == cudaSuccess &&
        dptr) {
      S.h.app[k].src = static_cast<const char *>(dptr);
      S.host_src_bytes[k] = 0;
      continue;
    }
    cudaGetLastError();
    total += S.host_src_bytes[k];
  }
  if (total == 0) return KV_OK;
  StageBuf *sb = nullptr;
  int rc = ctx->acquire(ctx->src, ctx->next_src, total, false, &sb);
  if (rc) return rc;
  size_t off = 0;
  for (int k = 0; k < S.h.n_app; ++k) {
    if (!S.host_src_bytes[k]) continue;
    CU(cudaMemcpyAsync(sb->dev + off, S.host_src[k], S.host_src_bytes[k], cudaMemcpyHostToDevice,
                       st));
    S.h.app[k].src = sb->dev + off;
    off += S.host_src_bytes[k];
  }
  *out = sb;
  return KV_OK;
}

std::atomic<unsigned long long> g_blob_nonce{0};

// Per-launch record (kv_launch_log): bytes and grid of every decode-step launch.
struct LaunchRec {
  uint64_t kind, app_bytes, rep_bytes, grid, blob_bytes;
};
thread_local bool g_log_on = false;
thread_local std::vector<LaunchRec> g_log;

constexpr size_t kItemsPerLaunch = 2048;  // 48 KiB of append items per launch

// Packs one launch's descriptor blob -- append items [i0, i1) and, if `with_rep`, the
// publication part -- then launches (data inline in the parameter space when it fits,
// else one H2D of the blob first).  Events of kv_time_next_launch honoured.
int step_launch_one(StepLaunch &S, size_t i0, size_t i1, bool with_rep, bool chain,
                    DeviceCtx *ctx, cudaStream_t st) {
  const double t0 = now_s();
  KvStepHdr h = S.h;
  if (!with_rep) {
    h.n_rep = 0;
    h.n_ent = 0;
    h.publish = 0;
    h.any_abort = 0;
    h.sys_any = 0;
  }
  const int32_t base = i0 < S.items.size() ? S.items[i0].off : 0;
  h.n_items = (int32_t)(i1 - i0);
  h.app_slices = i1 < S.items.size() ? S.items[i1].off - base : S.h.app_slices - base;
  if (h.n_items == 0) h.app_slices = 0;
  const size_t nent = with_rep ? S.req.size() : 0;
  // blob: [16-B header: launch nonce] [items] [req_id] [len] [pub_len] [blk0]
  size_t off = 16;
  h.items_off = (int32_t)off;
  off += align16(sizeof(KvAppItem) * h.n_items);
  h.req_off = (int32_t)off;
  off += align16(8 * nent);
  h.len_off = (int32_t)off;
  off += align16(4 * nent);
  h.pub_off = (int32_t)off;
  off += align16(4 * nent);
  h.blk0_off = (int32_t)off;
  off += align16(4 * nent);
  h.data_bytes = (int32_t)off;
  S.blob.assign(off, 0);
  char *b = S.blob.data();
  const unsigned long long nonce = ++g_blob_nonce;
  std::memcpy(b, &nonce, 8);
  if (h.n_items > 0) {
    KvAppItem *it = reinterpret_cast<KvAppItem *>(b + h.items_off);
    std::memcpy(it, S.items.data() + i0, sizeof(KvAppItem) * h.n_items);
    if (base)
      for (int k = 0; k < h.n_items; ++k) it[k].off -= base;
  }
  if (nent) {
    std::memcpy(b + h.req_off, S.req.data(), 8 * nent);
    std::memcpy(b + h.len_off, S.len.data(), 4 * nent);
    std::memcpy(b + h.pub_off, S.pub.data(), 4 * nent);
    std::memcpy(b + h.blk0_off, S.blk0.data(), 4 * nent);
  }
  h.pdl = S.pdl ? 1 : 0;
  h.app_first = h.sys_any ? 0 : 1;  // round order (kvring_step.cu copy_all)
  // grid: enough CTAs for ~1024 16-B chunks each, at most every resident CTA
  const uint64_t rep_slices = with_rep ? S.rep_bytes / (uint64_t)h.g.seg_bytes : 0;
  const unsigned long long chunks = ((unsigned long long)h.app_slices + rep_slices)
                                    << h.g.cps_shift;
  const int cap = step_resident_ctas(S.device, step_smem_bytes(h));
  const unsigned long long per = (unsigned long long)step_chunks_per_cta();
  int grid = (int)std::min<unsigned long long>(cap, std::max(1ull, (chunks + per - 1) / per));
  // a deferred publication of the previous launch: one more CTA stores its seqs
  h.n_prev = 0;
  if (ctx->n_pend_pub > 0) {
    if (ctx->pend_stream != st)
      return fail(KV_ESTATE, "a deferred publication is pending on another stream");
    h.n_prev = ctx->n_pend_pub;
    h.prev_sys = ctx->pend_sys;
    for (int q = 0; q < h.n_prev; ++q) {
      h.prev_seq[q] = ctx->pend_seq[q];
      h.prev_step[q] = ctx->pend_step[q];
    }
    grid = std::min(grid, std::max(1, cap - 1)) + 1;
  }
  // defer this launch's own seqs when a chained launch follows on the stream (a later
  // chunk of this step, or the next step of kv_loop_run) and a successor is a peer: the
  // CTAs then leave without waiting for their NVLink stores' acknowledgements
  h.defer = 0;
  int n_def = 0, def_sys = 0;
  unsigned long long *def_seq[kStepPools];
  unsigned long long def_step[kStepPools];
  if (with_rep && h.publish && h.sys_any && S.pdl && (i1 < S.items.size() || S.defer_next)) {
    for (int q = 0; q < h.n_rep; ++q) {
      if (h.rep[q].abort_slices >= 0) continue;
      def_seq[n_def] = reinterpret_cast<unsigned long long *>(h.rep[q].meta);
      def_step[n_def] = h.rep[q].step;
      if (h.rep[q].sys) def_sys |= 1 << n_def;
      ++n_def;
    }
    h.defer = n_def > 0;
  }
  // the blob goes into a pinned host slot; CTA 0 of the kernel pulls it across PCIe and
  // shares it through the slot's device buffer and flag (no copy-engine call, no event)
  DeviceCtx::BlobSlot *db = nullptr;
  int slot = 0;
  const double ta = now_s();
  phase_add(kPhPack, ta - t0);
  int rc = ctx->acquire_blob((size_t)h.data_bytes, &db, &slot);
  if (rc) return rc;
  std::memcpy(db->host, b, (size_t)h.data_bytes);
  phase_add(kPhAcquire, now_s() - ta);
  h.hblob = db->hmapped;
  h.gblob = db->dev;
  h.flag = ctx->flags + 16 * slot;        // one 128-B line per slot
  h.gate = ctx->flags + 16 * slot + 8;    // its second half: the deferred-publication gate
  h.counter = ctx->counters + 16 * slot;
  h.work = ctx->work + 128 * slot;
  h.target = db->arrivals + (unsigned long long)grid;
  db->arrivals = h.target + 1;            // + the final count after the seq stores
  h.chain = 0;
  h.early = 0;
  if (chain && S.pdl && ctx->last_counter && ctx->last_stream == st) {
    h.chain = 1;
    h.prev_counter = ctx->last_counter;
    h.prev_target = ctx->last_final;
    // early start (kvring_internal.h) when the launch before the previous one is ours as
    // well -- not over NVLink, where it measured neutral to -1.5 % (profiles/r02/ab)
    if (ctx->last_chained && !h.sys_any) {
      h.early = 1;
      h.pp_counter = ctx->last_prev_counter;
      h.pp_target = ctx->last_prev_final;
    }
  }
  ctx->last_chained = h.chain != 0;
  ctx->last_prev_counter = h.prev_counter;
  ctx->last_prev_final = h.prev_target;
  ctx->last_stream = st;
  ctx->last_counter = h.counter;
  ctx->last_final = h.target;             // its arrival target (kvring_internal.h)
  h.done = ctx->done_dev + 8 * slot;      // 64-B apart in pinned memory
  h.nonce = nonce;
  db->used = nonce;
  const double t1 = now_s();
  phase_add(kPhStage, t1 - t0);
  h.pad0 = (int32_t)(nonce & 0x7fffffff);  // launch nonce (debug timelines)
  CU(launch_step(h, grid, st, S.pdl));
  phase_add(kPhLaunch, now_s() - t1);
  // launched: the previous deferred publication is this launch's; this one's is pending
  ctx->n_pend_pub = n_def;
  if (n_def > 0) {
    for (int q = 0; q < n_def; ++q) {
      ctx->pend_seq[q] = def_seq[q];
      ctx->pend_step[q] = def_step[q];
    }
    ctx->pend_sys = def_sys;
    ctx->pend_stream = st;
  }
  g_launches++;
  if (g_log_on) {
    uint64_t app = 0;  // payload bytes of this launch's items
    app = (uint64_t)h.app_slices * (uint64_t)h.g.seg_bytes;
    g_log.push_back({(uint64_t)((h.n_items > 0) | ((with_rep && h.n_rep > 0) << 1)), app,
                     with_rep ? S.rep_bytes : 0, (uint64_t)grid, (uint64_t)h.data_bytes});
  }
  return KV_OK;
}

// Launches a prepared StepLaunch: one kernel (more only when the appends carry more
// than kItemsPerLaunch items, e.g. a 32k-token prefill; the publication rides on the
// first).
int step_enqueue(StepLaunch &S, cudaStream_t st) {
  if (S.device < 0) return KV_OK;
  if (S.empty()) {  // nothing to launch (mirror appends only): still withdraw entries
    if (S.inval.empty()) return KV_OK;
    DeviceGuard dg(S.device);
    if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice(%d) failed", S.device);
    return flush_inval(S.inval, S.max_reqs_inval, st);
  }
  DeviceGuard dg(S.device);
  if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice(%d) failed", S.device);
  if (!S.inval.empty()) {
    int rc = flush_inval(S.inval, S.max_reqs_inval, st);
    if (rc) return rc;
  }
  DeviceCtx *ctx = ctx_for(S.device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  StageBuf *sb = nullptr;
  int rc = step_stage_host_sources(ctx, S, st, &sb);
  if (rc) return rc;
  cudaEvent_t eb = g_ev_before, ea = g_ev_after;
  g_ev_before = g_ev_after = nullptr;
  if (eb) CU(cudaEventRecord(eb, st));
  const size_t n = S.items.size();
  size_t i0 = 0;
  bool first = true;
  do {
    const size_t i1 = std::min(n, i0 + kItemsPerLaunch);
    // a later chunk follows this enqueue's previous launch directly on the stream
    if ((rc = step_launch_one(S, i0, i1, first, first ? S.chain_ok : true, ctx, st))) return rc;
    first = false;
    i0 = i1;
  } while (i0 < n);
  if (ea) CU(cudaEventRecord(ea, st));
  for (int q = 0; q < S.h.n_app; ++q) S.app_pool[q]->kernels++;
  for (int q = 0; q < S.h.n_rep; ++q)
    if (S.h.n_app == 0 || S.rep_pool[q] != S.app_pool[0]) S.rep_pool[q]->kernels++;
  if (sb && (rc = ctx->done(sb, st))) return rc;  // the staged source outlives the kernel
  return KV_OK;
}

}  // namespace

KV_API int kv_append_multi(int32_t n_pools, const kv_append_args_t *args, void *stream) {
  NvtxRange nv("kv_append");
  thread_local StepLaunch S;
  const double t0 = now_s();
  int rc = validate_appends(n_pools, args);
  phase_add(kPhPrepAppend, now_s() - t0);
  if (rc) return rc;
  for (int k0 = 0; k0 < n_pools; k0 += kStepPools) {  // one launch per <= 8 pools
    S.reset();
    const double t1 = now_s();
    apply_appends(S, std::min(kStepPools, n_pools - k0), args + k0);
    phase_add(kPhPrepAppend, now_s() - t1);
    if (S.device >= 0 && (rc = step_enqueue(S, static_cast<cudaStream_t>(stream)))) return rc;
  }
  return KV_OK;
}

KV_API int kv_append(kv_pool_t *p, int32_t n, const int64_t *req_ids, const int32_t *n_new,
                     const void *src_kv, int32_t flags, void *stream) {
  kv_append_args_t a{};
  a.pool = p;
  a.n = n;
  a.req_ids = req_ids;
  a.n_new = n_new;
  a.src_kv = src_kv;
  a.flags = flags;
  return kv_append_multi(1, &a, stream);
}

namespace {
// Publication of several pools of one device: the device-derived step engine for
// plain links, the host-task ring-put for shared-capacity links (one launch each).
int replicate_any(int32_t n_pools, kv_pool_t *const *pools, uint64_t step, cudaStream_t st) {
  NvtxRange nv("kv_replicate_step");
  int rc = validate_replicate(n_pools, pools, step);
  if (rc) return rc;
  kv_pool *plain[kMaxPoolsPerLaunchHost], *shared[kMaxPoolsPerLaunchHost];
  int np = 0, ns = 0;
  for (int k = 0; k < n_pools; ++k) (pools[k]->holder ? shared[ns++] : plain[np++]) = pools[k];
  if (ns > 0 && (rc = replicate_host_tasks(ns, shared, step, st, false))) return rc;
  thread_local StepLaunch S;
  for (int k0 = 0; k0 < np;) {  // launches of <= kStepPools pools / kStepMaxEnt slots
    S.reset();
    int k1 = k0;
    long long ent = 0;
    while (k1 < np && k1 - k0 < kStepPools && ent + plain[k1]->slot_hi <= kStepMaxEnt)
      ent += plain[k1++]->slot_hi;
    if (k1 == k0) return fail(KV_EINVAL, "pool %d has too many slots for one launch", plain[k0]->node_id);
    const double t0 = now_s();
    if ((rc = step_prepare_replicate(S, k1 - k0, plain + k0, step))) return rc;
    phase_add(kPhPrepRepl, now_s() - t0);
    if (S.device >= 0 && (rc = step_enqueue(S, st))) return rc;
    k0 = k1;
  }
  return KV_OK;
}
}  // namespace

KV_API int kv_replicate_step(kv_pool_t *p, uint64_t step, void *stream) {
  return replicate_any(1, &p, step, static_cast<cudaStream_t>(stream));
}

KV_API int kv_replicate_step_multi(int32_t n_pools, kv_pool_t *const *pools, uint64_t step,
                                   void *stream) {
  return replicate_any(n_pools, pools, step, static_cast<cudaStream_t>(stream));
}

KV_API int kv_replicate_step_ce(int32_t n_pools, kv_pool_t *const *pools, uint64_t step,
                                void *stream) {
  return replicate_host_tasks(n_pools, pools, step, static_cast<cudaStream_t>(stream), true);
}

KV_API int kv_set_mode(kv_pool_t *p, int32_t mode) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (mode != KV_MODE_TOKENS && mode != KV_MODE_BLOCKS) return fail(KV_EINVAL, "unknown mode");
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  p->repl_mode = mode;
  std::fill(p->pub_len.begin(), p->pub_len.end(), 0);  // a mode switch re-seeds the link
  return KV_OK;
}

KV_API int kv_inject_abort(kv_pool_t *p, int32_t slices) {
  if (!p) return fail(KV_EINVAL, "null pool");
  p->abort_slices = slices < 0 ? -1 : slices;
  return KV_OK;
}

KV_API int kv_fail_stage(kv_pool_t *p, void *stream) {
  NvtxRange nv("kv_fail_stage");
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->dead) return fail(KV_ESTATE, "pool %d already dead", p->node_id);
  p->dead = true;
  p->has_succ = false;
  if (p->device < 0 || p->mirror) return KV_OK;  // a mirror's bytes are its owner's
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU(cudaMemsetAsync(p->pool, 0xFF, (size_t)p->NB * p->block_bytes, st));
  CU(cudaMemsetAsync(p->replica, 0xFF, (size_t)p->replica_blocks * p->block_bytes, st));
  CU(cudaMemsetAsync(p->meta, 0xFF, meta_bytes(p->R, p->M), st));
  return KV_OK;
}

KV_API int kv_restore(kv_pool_t *dst, const void *holder_replica, int32_t holder_replica_blocks,
                      const void *holder_meta, void *stream, uint64_t *t_star,
                      int64_t *req_ids_out, int32_t *resume_len_out, int32_t cap,
                      int32_t *n_out) {
  NvtxRange nv("kv_restore");
  if (!dst || !holder_replica || !holder_meta) return fail(KV_EINVAL, "null argument");
  if (dst->dead) return fail(KV_ESTATE, "restore target %d is dead", dst->node_id);
  if (dst->device < 0) return fail(KV_ESTATE, "restore needs a device pool");
  DeviceGuard dg(dst->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int R = dst->R, M = dst->M, B = dst->g.block_size;
  {  // a holder on another GPU of this process: the kernels read it over NVLink
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, holder_meta) == cudaSuccess &&
        at.type == cudaMemoryTypeDevice && at.device != dst->device) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, dst->device, at.device) == cudaSuccess && can)
        cudaDeviceEnablePeerAccess(at.device, 0);  // already enabled: harmless error
    }
    cudaGetLastError();
  }
  // 1. acquire the holder's seq and the parity metadata (reading R9, reader side): a
  //    kernel loads seq with ld.acquire.sys, fences, then copies header + tables into a
  //    device scratch that is read back -- first the 32-B header (shape check), then
  //    the whole region.  Synchronous: restore needs the tables on the host.
  std::vector<char> meta(meta_bytes(R, M));
  DeviceCtx *ctx = ctx_for(dst->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  int rc = ctx->reserve_meta_scratch(meta.size());
  if (rc) return rc;
  char *scratch = ctx->meta_scratch;
  uint64_t seq;
  int32_t hdr[4];
  CU(launch_meta_acquire(static_cast<const char *>(holder_meta), scratch, 32, st));
  CU(cudaMemcpyAsync(meta.data(), scratch, 32, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  std::memcpy(&seq, meta.data(), 8);
  std::memcpy(hdr, meta.data() + 8, 16);
  if (hdr[3] != kMetaMagic || hdr[1] != R || hdr[2] != M)
    return fail(KV_ENOREPLICA, "holder metadata invalid (magic %x, R %d, M %d)", hdr[3], hdr[1],
                hdr[2]);
  if (seq == 0 || seq == ~0ull) return fail(KV_ENOREPLICA, "holder published nothing (seq %llu)",
                                            (unsigned long long)seq);
  CU(launch_meta_acquire(static_cast<const char *>(holder_meta), scratch, meta.size(), st));
  CU(cudaMemcpyAsync(meta.data(), scratch, meta.size(), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  g_launches += 2;
  dst->kernels += 2;
  std::memcpy(&seq, meta.data(), 8);
  const int par = (int)(seq & 1);
  const int64_t *mreq = reinterpret_cast<const int64_t *>(meta.data() + 32) + (size_t)par * R;
  const int32_t *mlen =
      reinterpret_cast<const int32_t *>(meta.data() + meta_off_len(R)) + (size_t)par * R;
  const int32_t *mbt = reinterpret_cast<const int32_t *>(meta.data() + meta_off_bt(R));
  struct Ent {
    int64_t req;
    int len, slot;
  };
  std::vector<Ent> ents;
  long long need_blocks = 0;
  for (int s = 0; s < R; ++s)
    if (mreq[s] >= 0) {
      if (mlen[s] < 0 || ceil_div(mlen[s], B) > M)
        return fail(KV_ENOREPLICA, "holder metadata slot %d corrupt", s);
      ents.push_back({mreq[s], mlen[s], s});
      need_blocks += ceil_div(mlen[s], B);
    }
  std::sort(ents.begin(), ents.end(), [](const Ent &a, const Ent &b) { return a.req < b.req; });
  if ((int)ents.size() > cap) return fail(KV_EINVAL, "output capacity %d < %zu", cap, ents.size());
  if ((long long)ents.size() > dst->free_slots.size() || need_blocks > dst->free_blocks.size())
    return fail(KV_ENOMEM, "restore target too small");
  for (auto &e : ents) {
    if (dst->slot_of.find(e.req) >= 0)
      return fail(KV_EINVAL, "request %lld already in restore target", (long long)e.req);
    for (int j = 0; j < ceil_div(e.len, B); ++j) {
      const int b = mbt[(size_t)e.slot * M + j];
      if (b < 0 || b >= holder_replica_blocks)
        return fail(KV_ENOREPLICA, "holder bt entry out of range");
    }
  }
  // 2. allocate (req_id asc, j asc, lowest free ids) and build the remap tasks.
  TaskVec tasks;
  for (auto &e : ents) {
    const int s = dst->free_slots.take_min();
    dst->slot_of.insert(e.req, s);
    dst->slot_req[s] = e.req;
    slot_taken(dst, s);
    dst->slot_len[s] = e.len;
    dst->pub_len[s] = 0;
    dst->slot_bt[s].clear();
    admitted(dst, s);
    for (int j = 0; j < ceil_div(e.len, B); ++j) {
      const int nb = dst->free_blocks.take_min();
      dst->slot_bt[s].push_back(nb);
      const int valid = std::min(B, e.len - j * B);
      push_item(tasks, 0, mbt[(size_t)e.slot * M + j], nb, -1, j, 0, valid, dst->combos,
                dst->task_segs);
    }
  }
  // 3. one pinned staging buffer: [params][remap tasks][dst's device block table rows]
  //    -> one H2D; then copy valid slots (local HBM, or NVLink reads when the holder is
  //    remote).  The device-resident block table is read by the step engine's publications.
  {
    KvPoolParams pp;
    std::memset(&pp, 0, sizeof pp);
    pp.src = static_cast<const char *>(holder_replica);
    pp.dst = dst->pool;
    pp.src_bytes = (unsigned long long)holder_replica_blocks * dst->block_bytes;
    pp.dst_bytes = (unsigned long long)dst->NB * dst->block_bytes;
    const size_t pbytes = sizeof pp, tbytes = sizeof(KvTask) * tasks.size();
    const size_t roff = (pbytes + tbytes + 15) & ~(size_t)15, rbytes = sizeof(int32_t) * (size_t)R * M;
    StageBuf *b = nullptr;
    rc = ctx->acquire(ctx->ring, ctx->next, roff + rbytes, true, &b);
    if (rc) return rc;
    std::memcpy(b->host, &pp, pbytes);
    if (tbytes) std::memcpy(b->host + pbytes, tasks.data(), tbytes);
    int32_t *rows = reinterpret_cast<int32_t *>(b->host + roff);
    std::fill(rows, rows + (size_t)R * M, -1);
    for (int s = 0; s < dst->slot_hi; ++s)
      for (size_t j = 0; j < dst->slot_bt[s].size(); ++j) rows[(size_t)s * M + j] = dst->slot_bt[s][j];
    CU(cudaMemcpyAsync(b->dev, b->host, roff + rbytes, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dst->d_bt, b->dev + roff, rbytes, cudaMemcpyDeviceToDevice, st));
    if (!tasks.empty()) {
      CU(timed_launch(kKindRestore, reinterpret_cast<const KvTask *>(b->dev + pbytes),
                     (int)tasks.size(), reinterpret_cast<const KvPoolParams *>(b->dev), 1,
                     dst->geom_dev(), copy_grid(dst->device, (int)tasks.size()), st));
      g_launches++;
      dst->kernels++;
    }
    rc = ctx->done(b, st);
    if (rc) return rc;
  }
  // 4. outputs
  if (t_star) *t_star = seq;
  for (size_t i = 0; i < ents.size(); ++i) {
    if (req_ids_out) req_ids_out[i] = ents[i].req;
    if (resume_len_out) resume_len_out[i] = ents[i].len;
  }
  if (n_out) *n_out = (int32_t)ents.size();
  return KV_OK;
}

// ---- NCCL-comparison pack / unpack -------------------------------------------
namespace {
size_t packed_layout(kv_pool *p, size_t n_tasks, uint64_t payload_bytes, KvPackedHeader *h) {
  size_t off = sizeof(KvPackedHeader);
  off = (off + 31) & ~(size_t)31;
  h->task_off = off;
  off += sizeof(KvTask) * n_tasks;
  off = (off + 15) & ~(size_t)15;
  h->slot_off = off;
  off += 12 * (size_t)p->R;
  off = (off + 255) & ~(size_t)255;
  h->payload_off = off;
  h->payload_bytes = payload_bytes;
  off += payload_bytes;
  h->total_bytes = off;
  return off;
}
}  // namespace

KV_API int kv_pack_bytes(kv_pool_t *p, size_t *bytes_out) {
  if (!p || !bytes_out) return fail(KV_EINVAL, "null argument");
  TaskVec tasks;
  int32_t unit = 0;
  const uint64_t bytes = build_dirty_tasks(p, 0, tasks, true, &unit, p->task_segs);
  if (tasks.empty()) push_publish_only(tasks, 0);
  KvPackedHeader h{};
  *bytes_out = packed_layout(p, tasks.size(), bytes, &h);
  return KV_OK;
}

KV_API int kv_pack_step(kv_pool_t *p, uint64_t step, void *packed, size_t cap, size_t *bytes_out,
                        void *stream) {
  if (p && p->holder) return fail(KV_EINVAL, "kv_pack_step does not support shared-capacity links");
  if (!p || !packed) return fail(KV_EINVAL, "null argument");
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  if (p->device < 0) return fail(KV_ESTATE, "pack needs a device pool");
  if (step == 0 || step <= p->last_step) return fail(KV_EINVAL, "step not increasing");
  TaskVec tasks;
  int32_t unit = 0;
  const uint64_t bytes = build_dirty_tasks(p, 0, tasks, true, &unit, p->task_segs);
  if (tasks.empty()) push_publish_only(tasks, 0);
  tasks[0].flags |= kPoolFirst;
  KvPackedHeader h{};
  const size_t total = packed_layout(p, tasks.size(), bytes, &h);
  if (total > cap) return fail(KV_ENOMEM, "packed buffer too small (%zu > %zu)", total, cap);
  h.magic = kPackedMagic;
  h.n_tasks = (int32_t)tasks.size();
  h.max_reqs = p->R;
  h.max_blk = p->M;
  h.writer_node = p->node_id;
  h.seg_bytes = p->seg_bytes;
  h.step = step;
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceCtx *ctx = ctx_for(p->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  // head of the packed buffer: header + receiver-form tasks + slot table
  const size_t head = h.payload_off;
  KvPoolParams pp;
  std::memset(&pp, 0, sizeof pp);
  StageBuf *b = nullptr;
  const size_t pbytes = sizeof pp, tbytes = sizeof(KvTask) * tasks.size();
  int rc = ctx->acquire(ctx->ring, ctx->next, head + pbytes + tbytes, true, &b);
  if (rc) return rc;
  char *hb = b->host;
  std::memset(hb, 0, head);
  std::memcpy(hb, &h, sizeof h);
  KvTask *rt = reinterpret_cast<KvTask *>(hb + h.task_off);
  for (size_t i = 0; i < tasks.size(); ++i) {  // receiver: packed -> paged at the same ids
    rt[i] = tasks[i];
    rt[i].src_unit = tasks[i].dst_unit;
    rt[i].dst_unit = tasks[i].src_unit;
  }
  fill_pub_table(p, hb + h.slot_off);
  pp.src = p->pool;
  pp.dst = static_cast<char *>(packed) + h.payload_off;
  pp.src_bytes = (unsigned long long)p->NB * p->block_bytes;
  pp.dst_bytes = h.payload_bytes;
  std::memcpy(hb + head, &pp, pbytes);
  std::memcpy(hb + head + pbytes, tasks.data(), tbytes);
  CU(cudaMemcpyAsync(packed, hb, head, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(b->dev, hb + head, pbytes + tbytes, cudaMemcpyHostToDevice, st));
  int real = 0;
  for (auto &t : tasks) real += t.seg_count > 0;
  if (real > 0) {
    CU(timed_launch(kKindPack, reinterpret_cast<const KvTask *>(b->dev + pbytes),
                   (int)tasks.size(), reinterpret_cast<const KvPoolParams *>(b->dev), 1,
                   p->geom_dev(), copy_grid(p->device, (int)tasks.size()), st));
    g_launches++;
    p->kernels++;
  }
  rc = ctx->done(b, st);
  if (rc) return rc;
  p->last_step_bytes = bytes;
  p->bytes_replicated += bytes;
  commit_pub_len(p);
  p->last_step = step;
  if (bytes_out) *bytes_out = total;
  return KV_OK;
}

KV_API int kv_unpack(const void *packed, size_t packed_bytes, void *replica,
                     int32_t replica_blocks, void *replica_meta, const kv_geom_t *g,
                     int32_t max_reqs, int32_t max_blocks_per_req, void *stream) {
  if (!packed || !replica || !replica_meta || !g) return fail(KV_EINVAL, "null argument");
  int rc = validate_geom(g);
  if (rc) return rc;
  if (packed_bytes < sizeof(KvPackedHeader)) return fail(KV_EINVAL, "packed buffer too small");
  (void)replica_blocks;
  (void)max_reqs;
  (void)max_blocks_per_req;
  int dev = 0;
  CU(cudaGetDevice(&dev));
  DeviceCtx *ctx = ctx_for(dev);
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!ctx->unpack_counter) {
    CU(cudaMalloc(reinterpret_cast<void **>(&ctx->unpack_counter), sizeof(unsigned long long)));
    CU(cudaMemset(ctx->unpack_counter, 0, sizeof(unsigned long long)));
  }
  KvGeomDev gd;
  const int seg = g->head_dim * g->elem_bytes;
  gd.seg_bytes = seg;
  gd.token_bytes = g->layers * 2 * g->kv_heads * seg;
  gd.block_bytes = (long long)gd.token_bytes * g->block_size;
  gd.block_size = g->block_size;
  gd.cps_shift = __builtin_ctz(seg / 16);
  const int grid = copy_grid(dev, (int)std::max<size_t>(1, packed_bytes / 32768 + 1));
  cudaStream_t ust = static_cast<cudaStream_t>(stream);
  cudaEvent_t eb = g_ev_before, ea = g_ev_after;  // kv_time_next_launch applies here too
  g_ev_before = g_ev_after = nullptr;
  if (eb) CU(cudaEventRecord(eb, ust));
  CU(launch_unpack(static_cast<const char *>(packed), static_cast<char *>(replica),
                   static_cast<char *>(replica_meta), ctx->unpack_counter, gd, grid, ust));
  if (ea) CU(cudaEventRecord(ea, ust));
  g_launches++;
  return KV_OK;
}

KV_API int kv_query(kv_pool_t *p, int64_t req_id, int32_t *len, int32_t *blocks, int32_t cap,
                    int32_t *nblk) {
  if (!p) return fail(KV_EINVAL, "null pool");
  const int s = p->slot_of.find(req_id);
  if (s < 0) return fail(KV_EINVAL, "unknown request %lld", (long long)req_id);
  if (len) *len = p->slot_len[s];
  const int n = (int)p->slot_bt[s].size();
  if (nblk) *nblk = n;
  if (blocks)
    for (int j = 0; j < std::min(n, cap); ++j) blocks[j] = p->slot_bt[s][j];
  return KV_OK;
}

KV_API int kv_stats(kv_pool_t *p, kv_stats_t *o) {
  if (!p || !o) return fail(KV_EINVAL, "null argument");
  o->free_blocks = p->free_blocks.size();
  o->quarantined_blocks = (int32_t)p->q_blocks.size();
  o->used_blocks = p->NB - o->free_blocks - o->quarantined_blocks;
  o->free_slots = p->free_slots.size();
  o->quarantined_slots = (int32_t)p->q_slots.size();
  o->live_reqs = (int32_t)p->slot_of.size();
  o->dead = p->dead;
  o->has_successor = p->has_succ;
  o->last_step = p->last_step;
  o->bytes_replicated = p->bytes_replicated;
  o->tasks_launched = p->tasks_launched;
  o->kernels_launched = p->kernels;
  o->last_step_bytes = p->last_step_bytes;
  o->replica_blocks_held = p->rep_src ? p->rep_src->census : 0;
  o->replica_evictions = p->rep_evictions;
  o->replica_drops = p->rep_drops;
  o->shared_holder = p->holder ? p->holder->node_id : -1;
  return KV_OK;
}

KV_API int kv_dump_slots(kv_pool_t *p, int64_t *req_id, int32_t *len, int32_t *pub_len,
                         int32_t *nblk) {
  if (!p) return fail(KV_EINVAL, "null pool");
  for (int s = 0; s < p->R; ++s) {
    if (req_id) req_id[s] = p->slot_req[s];
    if (len) len[s] = p->slot_len[s];
    if (pub_len) pub_len[s] = p->pub_len[s];
    if (nblk) nblk[s] = (int32_t)p->slot_bt[s].size();
  }
  return KV_OK;
}

KV_API int kv_sync(kv_pool_t *p) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->device < 0) return KV_OK;
  DeviceGuard dg(p->device);
  CU(cudaDeviceSynchronize());
  CU(cudaGetLastError());
  return KV_OK;
}

// ---- decode loops ------------------------------------------------------------------
namespace {

bool step_has_shared(const kv_step_t &st) {
  for (int i = 0; i < st.n_append; ++i) {
    const kv_pool *p = st.append[i].pool;
    if (p && (p->holder || p->rep_src)) return true;
  }
  for (int i = 0; i < st.n_repl; ++i) {
    const kv_pool *p = st.repl_pools[i];
    if (p && (p->holder || p->rep_src)) return true;
  }
  return false;
}

int step_device(const kv_step_t &st) {
  if (st.n_append > 0 && st.append[0].pool) return st.append[0].pool->device;
  if (st.n_repl > 0 && st.repl_pools[0]) return st.repl_pools[0]->device;
  return -1;
}

int record(void *ev, cudaStream_t s) {
  if (ev) CU(cudaEventRecord(static_cast<cudaEvent_t>(ev), s));
  return KV_OK;
}

// Cross-stream order of the two-stream loop: the publication of step k after append
// k (event `aready`), and append k after the publication of step k-2 -- blocks a
// retiring request frees in step k-1 are reused from step k on (quarantine, reading
// R7), and the publication that last read them is k-2's, which may otherwise still
// lag on its stream (k-1 with shared capacity: a freed replica block is reusable at once).
struct StreamOrder {
  static constexpr int kN = 4;
  cudaEvent_t aready[kN] = {};
  cudaEvent_t rdone[kN] = {};
  long long astep[kN] = {-1, -1, -1, -1};
  long long rstep[kN] = {-1, -1, -1, -1};
  long long n = 0;  // steps issued on this stream pair (continues across calls)
  cudaStream_t sa = nullptr, sr = nullptr;
  int dev = -1;
  int ensure(int device, cudaStream_t a, cudaStream_t r) {
    if (dev != device) {
      for (auto &e : aready)
        if (e) cudaEventDestroy(e);
      for (auto &e : rdone)
        if (e) cudaEventDestroy(e);
      for (auto &e : aready) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      for (auto &e : rdone) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      dev = device;
      sa = sr = nullptr;
    }
    if (a != sa || r != sr) {  // a new stream pair: its first append waits for repl_stream
      for (int i = 0; i < kN; ++i) astep[i] = rstep[i] = -1;
      n = 0;
      sa = a;
      sr = r;
      CU(cudaEventRecord(rdone[0], r));
      CU(cudaStreamWaitEvent(a, rdone[0], 0));
    }
    return KV_OK;
  }
};

}  // namespace

KV_API int kv_run_steps(int32_t n_steps, const kv_step_t *steps, void *append_stream,
                        void *repl_stream) {
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  cudaStream_t sa = static_cast<cudaStream_t>(append_stream);
  cudaStream_t sr = static_cast<cudaStream_t>(repl_stream);
  thread_local StreamOrder so;
  thread_local StepLaunch S;
  const int N = StreamOrder::kN;
  for (int i = 0; i < n_steps; ++i) {
    const kv_step_t &st = steps[i];
    const int dev = step_device(st);
    DeviceGuard dg(dev);
    const bool two = dev >= 0 && sa != sr;
    int rc = KV_OK;
    if (two && (rc = so.ensure(dev, sa, sr))) return rc;
    const long long k = two ? so.n++ : i;
    // the appends of step k (the model's KV write) on the append stream
    if (st.n_append > 0) {
      const double t0 = now_s();
      rc = validate_appends(st.n_append, st.append);
      phase_add(kPhPrepAppend, now_s() - t0);
      if (rc) return rc;
      if (dev >= 0) {
        const int lag = step_has_shared(st) ? 1 : 2;
        if (two && k >= lag && so.rstep[(k - lag) % N] == k - lag)
          CU(cudaStreamWaitEvent(sa, so.rdone[(k - lag) % N], 0));
      }
      for (int k0 = 0; k0 < st.n_append; k0 += kStepPools) {
        S.reset();
        const double t1 = now_s();
        const int n = std::min(kStepPools, st.n_append - k0);
        apply_appends(S, n, st.append + k0);
        phase_add(kPhPrepAppend, now_s() - t1);
        if (dev < 0) continue;
        g_ev_before = k0 == 0 ? static_cast<cudaEvent_t>(st.ev_append_start) : nullptr;
        g_ev_after = k0 + n == st.n_append ? static_cast<cudaEvent_t>(st.ev_append_end) : nullptr;
        rc = step_enqueue(S, sa);
        g_ev_before = g_ev_after = nullptr;
        if (rc) return rc;
      }
    }
    // the publication of step k on the replication stream (§3.2)
    if (st.n_repl > 0) {
      if (two) {
        CU(cudaEventRecord(so.aready[k % N], sa));
        so.astep[k % N] = k;
        CU(cudaStreamWaitEvent(sr, so.aready[k % N], 0));
      }
      if (dev >= 0 && (rc = record(st.ev_call, sr))) return rc;
      g_ev_before = static_cast<cudaEvent_t>(st.ev_kernel_start);
      g_ev_after = static_cast<cudaEvent_t>(st.ev_kernel_end);
      rc = replicate_any(st.n_repl, st.repl_pools, st.step, sr);
      g_ev_before = g_ev_after = nullptr;
      if (rc) return rc;
      if (dev >= 0 && (rc = record(st.ev_done, sr))) return rc;
      if (two) {
        CU(cudaEventRecord(so.rdone[k % N], sr));
        so.rstep[k % N] = k;
      }
    }
  }
  return KV_OK;
}

// ---- one launch per decode step (software pipelined) -------------------------------
struct kv_loop {
  std::vector<kv_pool *> pend;  // pools whose publication of pend_step is pending
  uint64_t pend_step = 0;
  std::vector<std::unique_ptr<StepLaunch>> S;  // launches of one step (<= 8 pools each)
  StepLaunch &at(size_t i) {
    while (S.size() <= i) S.emplace_back(new StepLaunch());
    return *S[i];
  }
};

namespace {
void loop_forget(kv_loop *L, kv_pool *p) {
  auto &v = L->pend;
  v.erase(std::remove(v.begin(), v.end(), p), v.end());
}

// The pending publication, built from the pools' CURRENT tables: everything the
// harness did since the previous step (a failure, a restore, a relink, a resume
// re-append) is reflected exactly as in the sequential protocol (append t, then
// replicate t).  Pools that died or lost their successor meanwhile publish nothing.
// Fills launches 0..(*n_out - 1) (<= kStepPools pools / kStepMaxEnt slots each).
int loop_take_pending(kv_loop *L, int *n_out) {
  *n_out = 0;
  if (L->pend.empty()) return KV_OK;
  kv_pool *ps[kMaxPoolsPerLaunchHost];
  int n = 0;
  for (kv_pool *p : L->pend) {
    p->loop = nullptr;
    if (!p->dead && p->has_succ) ps[n++] = p;
  }
  L->pend.clear();
  if (n == 0) return KV_OK;
  const double t0 = now_s();
  int rc = validate_replicate(n, ps, L->pend_step);
  int nl = 0;
  for (int k0 = 0; !rc && k0 < n; ++nl) {
    int k1 = k0;
    long long ent = 0;
    while (k1 < n && k1 - k0 < kStepPools && ent + ps[k1]->slot_hi <= kStepMaxEnt)
      ent += ps[k1++]->slot_hi;
    if (k1 == k0) return fail(KV_EINVAL, "pool %d has too many slots for one launch", ps[k0]->node_id);
    StepLaunch &S = L->at(nl);
    S.reset();
    rc = step_prepare_replicate(S, k1 - k0, ps + k0, L->pend_step);
    k0 = k1;
  }
  phase_add(kPhPrepRepl, now_s() - t0);
  *n_out = nl;
  return rc;
}
}  // namespace

KV_API int kv_loop_create(kv_loop_t **out) {
  if (!out) return fail(KV_EINVAL, "null argument");
  *out = new kv_loop();
  return KV_OK;
}

KV_API int kv_loop_destroy(kv_loop_t *L) {
  if (!L) return KV_OK;
  for (kv_pool *p : L->pend) p->loop = nullptr;
  delete L;
  return KV_OK;
}

namespace {
// chain_first: the previous kernel on `stream` is this loop's previous launch (inside
// kv_loop_run, which enqueues nothing else between its steps)
// defer_last: a chained launch follows this step's last launch on the stream (the next
// step of kv_loop_run), so a publication over NVLink may hand its seq stores to it
int loop_step(kv_loop_t *L, const kv_step_t *st, void *stream, bool chain_first,
              bool defer_last) {
  NvtxRange nv("kv_loop_step");
  if (!L || !st) return fail(KV_EINVAL, "null argument");
  if (st->n_repl > kMaxPoolsPerLaunchHost) return fail(KV_EINVAL, "too many pools");
  for (int i = 0; i < st->n_repl; ++i) {
    kv_pool *p = st->repl_pools[i];
    if (!p) return fail(KV_EINVAL, "null pool");
    if (p->holder || p->rep_src)
      return fail(KV_EINVAL, "shared-capacity pools need kv_run_steps (two streams)");
    if (p->loop && p->loop != L) return fail(KV_ESTATE, "pool %d is pending in another loop", p->node_id);
  }
  for (int i = 0; i < st->n_append; ++i)
    if (st->append[i].pool && (st->append[i].pool->holder || st->append[i].pool->rep_src))
      return fail(KV_EINVAL, "shared-capacity pools need kv_run_steps (two streams)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // 1. the previous step's publication (snapshots + host commit, before any append)
  int n_rep = 0;
  int rc = loop_take_pending(L, &n_rep);
  if (rc) return rc;
  for (int i = n_rep; i < (int)L->S.size(); ++i) L->S[i]->reset();
  // 2. this step's appends; if they are rejected the publication still launches
  int rc_app = KV_OK, n_app = 0;
  if (st->n_append > 0) {
    const double t0 = now_s();
    rc_app = validate_appends(st->n_append, st->append);
    if (!rc_app)
      for (int k0 = 0; k0 < st->n_append; k0 += kStepPools, ++n_app)
        apply_appends(L->at(n_app), std::min(kStepPools, st->n_append - k0), st->append + k0);
    phase_add(kPhPrepAppend, now_s() - t0);
  }
  // 3. one launch (more only beyond 8 pools per role)
  const int nl = std::max(n_rep, n_app);
  for (int i = 0; i < nl; ++i) {
    g_ev_before = i == 0 ? static_cast<cudaEvent_t>(st->ev_kernel_start) : nullptr;
    g_ev_after = i == nl - 1 ? static_cast<cudaEvent_t>(st->ev_kernel_end) : nullptr;
    // consecutive steps of the loop overlap: a launch's prologue (descriptor, work list)
    // runs while the previous step's grid drains (timed launches are serialised)
    L->S[i]->pdl = !st->ev_kernel_start && !st->ev_kernel_end;
    L->S[i]->chain_ok = i > 0 || chain_first;
    L->S[i]->defer_next = i < nl - 1 || defer_last;
    rc = step_enqueue(*L->S[i], s);
    g_ev_before = g_ev_after = nullptr;
    if (rc) return rc;
  }
  if (rc_app) return rc_app;
  // 4. this step's publication rides on the next launch
  if (st->n_repl > 0) {
    L->pend.assign(st->repl_pools, st->repl_pools + st->n_repl);
    L->pend_step = st->step;
    for (kv_pool *p : L->pend) p->loop = L;
  }
  return KV_OK;
}

}  // namespace

KV_API int kv_loop_step(kv_loop_t *L, const kv_step_t *st, void *stream) {
  return loop_step(L, st, stream, false, false);
}

namespace {
// A launch deferred its seq stores but no launch followed on `stream` (an error stopped
// the loop): one launch with nothing to move but the publisher CTA stores them.
int flush_deferred(void *stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<DeviceCtx *> ctxs;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto &kv : g_ctx) ctxs.push_back(kv.second.get());
  }
  for (DeviceCtx *ctx : ctxs) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->n_pend_pub == 0 || ctx->pend_stream != st) continue;
    DeviceGuard dg(ctx->device);
    if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice(%d) failed", ctx->device);
    StepLaunch S;
    S.device = ctx->device;
    S.pdl = true;
    int rc = step_launch_one(S, 0, 0, false, true, ctx, st);
    if (rc) return rc;
  }
  return KV_OK;
}
}  // namespace

KV_API int kv_loop_run(kv_loop_t *L, int32_t n_steps, const kv_step_t *steps, void *stream) {
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  for (int i = 0; i < n_steps; ++i) {
    // the next step launches (its appends, or this step's publication) and is chained
    const bool next = i + 1 < n_steps && (steps[i + 1].n_append > 0 || steps[i].n_repl > 0);
    int rc = loop_step(L, &steps[i], stream, i > 0, next);
    if (rc) {
      flush_deferred(stream);
      return rc;
    }
  }
  return flush_deferred(stream);
}

KV_API int kv_loop_flush(kv_loop_t *L, void *stream) {
  if (!L) return fail(KV_EINVAL, "null loop");
  int n = 0;
  int rc = loop_take_pending(L, &n);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    L->S[i]->pdl = true;
    if ((rc = step_enqueue(*L->S[i], static_cast<cudaStream_t>(stream)))) return rc;
  }
  return KV_OK;
}

KV_API int kv_launch_log(uint64_t *out, int32_t cap, int32_t mode) {
  if (mode == 1) {
    g_log.clear();
    g_log_on = true;
    return 0;
  }
  g_log_on = false;
  const int n = (int)g_log.size();
  if (out)
    for (int i = 0; i < n && i < cap; ++i) {
      out[5 * i + 0] = g_log[i].kind;
      out[5 * i + 1] = g_log[i].app_bytes;
      out[5 * i + 2] = g_log[i].rep_bytes;
      out[5 * i + 3] = g_log[i].grid;
      out[5 * i + 4] = g_log[i].blob_bytes;
    }
  return n;
}

// ---- re-protection (§8(f) NEXT-1; §3.2) --------------------
// Each non-excluded node's replication target is the first non-excluded node met
// by walking its ring successors; never itself; -1 when none exists (the node is
// unprotected: "replication-disabled").  Excluded nodes (failed, or under traffic
// rerouting) neither send nor receive: -1.
KV_API int kv_plan_targets(int32_t n_nodes, const int32_t *succ, const uint8_t *excluded,
                           int32_t *targets) {
  if (n_nodes <= 0 || !succ || !targets) return fail(KV_EINVAL, "bad arguments");
  for (int i = 0; i < n_nodes; ++i)
    if (succ[i] < 0 || succ[i] >= n_nodes) return fail(KV_EINVAL, "successor out of range");
  for (int i = 0; i < n_nodes; ++i) {
    targets[i] = -1;
    if (excluded && excluded[i]) continue;
    int j = succ[i];
    for (int hops = 0; hops < n_nodes && j != i; ++hops, j = succ[j]) {
      if (!(excluded && excluded[j])) {
        targets[i] = j;
        break;
      }
    }
  }
  return KV_OK;
}
