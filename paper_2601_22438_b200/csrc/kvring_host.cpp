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

#include "kvring.h"
#include "kvring_internal.h"

#define KV_API extern "C" __attribute__((visibility("default")))

// Host-side phase counters of kv_run_steps (seconds, cumulative; kv_host_profile).
#include <chrono>
namespace {
enum { kPhPrepare = 0, kPhWaitPrep, kPhStage, kPhEnqA, kPhEnqP, kPhEvents, kPhWaitIssue,
       kPhAcquire, kPhHostCopy, kPhH2DCall, kPhPrepAppend, kPhPrepRepl, kPhCommit,
       kPhPubStage, kPhInlineLaunches, kPhStagedLaunches, kPhN };
// Two threads (helper + issue) add to them: relaxed atomics, integer nanoseconds.
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
  char *dev = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
};

struct DeviceCtx {
  int device = 0;
  std::mutex mu;
  static constexpr int kRing = 8;
  StageBuf ring[kRing];
  int next = 0;
  StageBuf src[kRing];  // device copies of host-resident append sources (KV_SRC_HOST)
  int next_src = 0;
  unsigned long long *unpack_counter = nullptr;
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
        if (want_host) CU(cudaHostAlloc(reinterpret_cast<void **>(&r.host), cap, cudaHostAllocDefault));
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
                         int n_pools, const KvGeomDev &g, int grid, cudaStream_t st,
                         const KvPoolParams *host_params = nullptr, int split = 1) {
  cudaEvent_t b = g_ev_before, a = g_ev_after;
  g_ev_before = g_ev_after = nullptr;
  if (b) {
    cudaError_t e = cudaEventRecord(b, st);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_copy(kind, tasks, n_tasks, params, n_pools, g, grid, st, host_params,
                              split);
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

struct kv_pool {
  kv_geom_t g{};
  int NB = 0, R = 0, M = 0, device = -1, node_id = 0, replica_blocks = 0;
  char *pool = nullptr, *replica = nullptr, *meta = nullptr;
  // geometry derived
  long long block_bytes = 0;
  int token_bytes = 0, seg_bytes = 0, combos = 0, task_segs = 0, cps_shift = 0;
  // ring link
  int repl_mode = KV_MODE_TOKENS;  // KV_MODE_BLOCKS: completed blocks only (NEXT-2)
  bool has_succ = false;
  bool succ_sys = true;  // successor memory is not this GPU's HBM (NVLink peer)
  int succ_node = -1, succ_replica_blocks = 0;
  char *succ_replica = nullptr, *succ_meta = nullptr;
  // allocator (R6, R7)
  IdSet free_blocks, free_slots;
  std::vector<int> q_blocks, q_slots;
  std::vector<int64_t> slot_req;
  std::vector<int32_t> slot_len, pub_len;
  int slot_hi = 0;  // 1 + highest live slot (slots are taken lowest first): loop bound
  std::vector<std::vector<int32_t>> slot_bt;
  SlotMap slot_of;
  std::vector<uint32_t> rel_stamp, app_stamp;  // per-slot call stamps (validation)
  uint32_t call_id = 0;
  std::vector<int64_t> scratch_ids;
  std::vector<int> scratch_slot;  // slot of each append entry found by validation (-1: new)
  TaskVec scratch_tasks;
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
  int abort_after = -1;
  unsigned long long *counter = nullptr;  // device, monotone
  unsigned long long issued = 0;          // host mirror of the counter target
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
  if (seg < 16 || (seg & (seg - 1)) != 0)
    return fail(KV_EINVAL, "head_dim * elem_bytes = %d must be a power of two >= 16", seg);
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
    for (int b : p->slot_bt[s]) p->q_blocks.push_back(b);
    p->slot_bt[s].clear();
    p->q_slots.push_back(s);
    p->slot_req[s] = -1;
    slot_freed(p);
    p->slot_len[s] = 0;
    p->pub_len[s] = 0;
  }
}

// Applies the appends to the tables and emits the scatter tasks (src rows are
// token rows of the dense source, `row_base` added).
void do_append(kv_pool *p, const kv_append_args_t &a, int16_t pidx, TaskVec &tasks,
               int task_segs) {
  const int B = p->g.block_size;
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
      if (len % B == 0) p->slot_bt[s].push_back(p->free_blocks.take_min());
      const int j = len / B, lo = len % B;
      const int n = std::min(B - lo, left);
      if (p->device >= 0)
        push_item(tasks, pidx, row, p->slot_bt[s][j], -1, j, lo, n, p->combos, task_segs);
      row += n;
      len += n;
      left -= n;
    }
    p->slot_len[s] = len;
  }
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
    CU(cudaMalloc(reinterpret_cast<void **>(&p->counter), sizeof(unsigned long long)));
    CU(cudaMemset(p->counter, 0, sizeof(unsigned long long)));
    CU(launch_meta_init(p->meta, p->R, p->M, 0));
    g_launches++;
    p->kernels++;
    CU(cudaDeviceSynchronize());
    ctx_for(p->device);
  }
  *out = p.release();
  return KV_OK;
}

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
  if (p->counter) {
    DeviceGuard dg(p->device);
    cudaDeviceSynchronize();
    cudaFree(p->counter);
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

// ---- launches: prepare on the host, stage descriptors with ONE H2D, enqueue ----
inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// One kernel launch prepared on the host.
struct Launch {
  int kind = kKindAppend;
  int n_pools = 0;
  kv_pool *p0 = nullptr;
  std::vector<KvPoolParams> params;
  std::vector<char> tables;        // replicate: per pool slot_req[R] (8R B) then slot_len[R] (4R B)
  std::vector<size_t> table_off;   // per pool offset into `tables`
  TaskVec tasks;
  std::vector<int> ntask;          // replicate: tasks per pool
  std::vector<uint64_t> bytes;     // replicate: payload bytes per pool
  std::vector<const void *> host_src;  // append: host sources (KV_SRC_HOST), per pool
  std::vector<size_t> host_src_bytes;
  std::vector<std::vector<int>> ce_blocks;  // copy-engine variant: full blocks per pool
  bool use_ce = false;
  std::vector<kv_pool::Inval> inval;  // shared capacity: published entries to withdraw first
  int max_reqs_inval = 0;
  int split = 1;                      // CTA units per task (whole-item tasks)
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
    host_src.assign(n, nullptr);
    host_src_bytes.assign(n, 0);
    if ((int)ce_blocks.size() < n) ce_blocks.resize(n);
    for (auto &v : ce_blocks) v.clear();
    use_ce = false;
    inval.clear();
    split = 1;
    params_dev = nullptr;
    tasks_dev = nullptr;
  }
  size_t staged_bytes() const {
    return align16(sizeof(KvPoolParams) * n_pools) + align16(tables.size()) +
           sizeof(KvTask) * tasks.size();
  }
};

// Moves the pending published-entry invalidations of every holder this launch
// touches (its pools, and the holders of its pools) into the launch.
void collect_inval(Launch &L, kv_pool *const *pools, int n) {
  auto take = [&](kv_pool *h) {
    if (!h || h->pending_inval.empty()) return;
    L.max_reqs_inval = h->R;
    L.inval.insert(L.inval.end(), h->pending_inval.begin(), h->pending_inval.end());
    h->pending_inval.clear();
  };
  for (int k = 0; k < n; ++k) {
    take(pools[k]);
    take(pools[k]->holder);
  }
}

// Task size for one launch: spread the launch's slices over every resident CTA
// (SMs x 4) so a decode-sized step runs in one wave, capped at 32 KiB per task.
int choose_task_segs(const kv_pool *p, long long total_segs) {
  const int maxs = std::max(1, 32768 / p->seg_bytes);
  const long long slots = (long long)resident_ctas(p->device < 0 ? 0 : p->device);
  static int min_segs = -1;  // experiment knob KVRING_MIN_TASK_SEGS (default 16)
  if (min_segs < 0) {
    const char *e = getenv("KVRING_MIN_TASK_SEGS");
    min_segs = (e && atoi(e) > 0) ? atoi(e) : 16;
  }
  long long t = (total_segs + slots - 1) / std::max(1LL, slots);
  t = (t + 15) & ~15LL;
  t = std::max<long long>(std::min(maxs, min_segs), t);
  return (int)std::min<long long>(maxs, t);
}

// Whole-item tasks (<= 32 KiB each, fewer descriptors to stage or carry in the
// parameter space) split on the device into `split` CTA units so a decode step still
// spreads over every resident CTA (KVRING_MIN_TASK_SEGS > 0: the old sizing, split 1).
int whole_item_segs(const kv_pool *p) { return std::max(1, 32768 / p->seg_bytes); }

int choose_split(const kv_pool *p, size_t n_tasks) {
  if (n_tasks == 0) return 1;
  const long long slots = (long long)resident_ctas(p->device < 0 ? 0 : p->device);
  return (int)std::max(1LL, std::min(8LL, slots / (long long)n_tasks));
}

bool legacy_task_sizing() {
  static const bool legacy = getenv("KVRING_MIN_TASK_SEGS") != nullptr;
  return legacy;
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

// Validates every pool (all-or-nothing), applies begin_step / releases / appends
// to the host tables and builds the scatter tasks.
int prepare_append(int n_pools, const kv_append_args_t *args, Launch &L, bool allow_split = true) {
  if (n_pools <= 0 || !args) return fail(KV_EINVAL, "no pools");
  if (n_pools > kMaxPoolsPerLaunchHost)
    return fail(KV_EINVAL, "at most %d pools per launch", kMaxPoolsPerLaunchHost);
  kv_pool *pools[kMaxPoolsPerLaunchHost];
  for (int k = 0; k < n_pools; ++k) pools[k] = args[k].pool;
  if (!pools[0]) return fail(KV_EINVAL, "null pool");
  int rc = check_same_device(n_pools, pools);
  if (rc) return rc;
  long long tokens = 0;
  {
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = args[k].pool;
    if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
    const bool bs = args[k].begin_step != 0;  // validation sees the released quarantine
    rc = append_validate(p, args[k],
                         p->free_blocks.size() + (bs ? (long long)p->q_blocks.size() : 0),
                         p->free_slots.size() + (bs ? (long long)p->q_slots.size() : 0));
    if (rc) return rc;
    long long rows = 0;
    for (int i = 0; i < args[k].n; ++i) rows += args[k].n_new[i];
    if (p->device >= 0 && rows > 0 && !args[k].src_kv)
      return fail(KV_EINVAL, "null src_kv with tokens to append");
    tokens += rows;
  }
  }
  L.reset(kKindAppend, n_pools);
  L.p0 = pools[0];
  const bool whole = allow_split && !legacy_task_sizing();
  const int task_segs =
      whole ? whole_item_segs(L.p0) : choose_task_segs(L.p0, tokens * L.p0->combos);
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = args[k].pool;
    if (args[k].begin_step) do_begin_step(p);
    do_release(p, args[k].n_release, args[k].release_ids);
    if (p->scratch_need > p->free_blocks.size()) evict_for(p, p->scratch_need);
    const size_t before = L.tasks.size();
    do_append(p, args[k], (int16_t)k, L.tasks, task_segs);
    L.ntask[k] = (int)(L.tasks.size() - before);
    long long rows = 0;
    for (int i = 0; i < args[k].n; ++i) rows += args[k].n_new[i];
    KvPoolParams &pp = L.params[k];
    pp.src = static_cast<const char *>(args[k].src_kv);
    pp.dst = p->pool;
    pp.src_bytes = (unsigned long long)rows * p->token_bytes;
    pp.dst_bytes = (unsigned long long)p->NB * p->block_bytes;
    if ((args[k].flags & KV_SRC_HOST) && rows > 0) {
      L.host_src[k] = args[k].src_kv;
      L.host_src_bytes[k] = (size_t)rows * p->token_bytes;
    }
  }
  collect_inval(L, pools, n_pools);
  if (whole) L.split = choose_split(L.p0, L.tasks.size());
  return KV_OK;
}

// Validates the pools and builds the dirty work list (§8(a) a3); state is
// committed by commit_replicate once the launch is enqueued.
int prepare_replicate(int n_pools, kv_pool *const *pools, uint64_t step, Launch &L,
                      bool use_ce = false, bool allow_split = true) {
  if (n_pools <= 0 || !pools) return fail(KV_EINVAL, "no pools");
  if (n_pools > kMaxPoolsPerLaunchHost)
    return fail(KV_EINVAL, "at most %d pools per launch", kMaxPoolsPerLaunchHost);
  if (!pools[0]) return fail(KV_EINVAL, "null pool");
  int rc = check_same_device(n_pools, pools);
  if (rc) return rc;
  const bool whole = allow_split && !legacy_task_sizing();
  long long dirty = 0;  // only the legacy task sizing needs it before building
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k];
    if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
    if (!p->has_succ) return fail(KV_EPEER, "pool %d has no successor", p->node_id);
    if (step == 0 || step <= p->last_step)
      return fail(KV_EINVAL, "step %llu not > last step %llu of pool %d",
                  (unsigned long long)step, (unsigned long long)p->last_step, p->node_id);
    if (!whole)
      for (int s = 0; s < p->slot_hi; ++s)
        if (p->slot_req[s] >= 0) dirty += pub_hi(p, s) - p->pub_len[s];
  }
  L.reset(kKindRingPut, n_pools);
  L.p0 = pools[0];
  L.use_ce = use_ce;
  const int task_segs =
      whole ? whole_item_segs(L.p0) : choose_task_segs(L.p0, dirty * L.p0->combos);
  size_t toff = 0;
  for (int k = 0; k < n_pools; ++k) toff += 12 * (size_t)pools[k]->R;
  L.tables.resize(toff);
  toff = 0;
  for (int k = 0; k < n_pools; ++k) {
    kv_pool *p = pools[k];
    const size_t before = L.tasks.size();
    L.bytes[k] = build_dirty_tasks(p, (int16_t)k, L.tasks, false, nullptr, task_segs,
                                   use_ce ? &L.ce_blocks[k] : nullptr);
    if (L.tasks.size() == before) push_publish_only(L.tasks, (int16_t)k);
    L.tasks[before].flags |= kPoolFirst;
    L.ntask[k] = (int)(L.tasks.size() - before);
    const bool aborting = p->abort_after >= 0 && p->abort_after < L.ntask[k];
    if (aborting) {  // fault injection: partial step, never published
      L.tasks.resize(before + p->abort_after);
      L.ntask[k] = p->abort_after;
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
    pp.target = aborting || p->abort_after >= 0 ? ~0ull : 0ull;  // + units, set below
    pp.step = step;
    pp.max_reqs = p->R;
    pp.max_blk = p->M;
    pp.n_table = p->R;  // staged tables carry every slot (inline launches trim them)
    pp.writer_node = p->node_id;
    pp.publish = 1;
    // KVRING_DEBUG_GPU_SCOPE=1 (experiments only: measures the cost of the system-scope
    // publication; a remote reader could then see seq before the data)
    static const bool dbg_gpu_scope = getenv("KVRING_DEBUG_GPU_SCOPE") != nullptr;
    pp.sys_scope = p->succ_sys && !dbg_gpu_scope ? 1 : 0;
    static const int sys_per_cta = getenv("KVRING_SYS_PER_CTA") ? 1 : 0;  // experiments
    pp.pad0 = sys_per_cta;
  }
  collect_inval(L, pools, n_pools);
  if (whole) L.split = choose_split(L.p0, L.tasks.size());
  for (int k = 0; k < n_pools; ++k)  // the counter counts CTA units: tasks x split
    if (L.params[k].target == 0ull)
      L.params[k].target = pools[k]->issued + (unsigned long long)L.ntask[k] * L.split;
  static const bool dbg_nocopy = getenv("KVRING_DEBUG_RINGPUT_NOCOPY") != nullptr;
  if (dbg_nocopy)  // experiment knob: publication only (timing breakdown, breaks parity)
    for (size_t i = 0; i < L.tasks.size(); ++i) L.tasks[i].seg_count = 0;
  return KV_OK;
}

void commit_replicate(Launch &L, kv_pool *const *pools, uint64_t step) {
  for (int k = 0; k < L.n_pools; ++k) {
    kv_pool *p = pools[k];
    p->issued += (unsigned long long)L.ntask[k] * L.split;
    p->last_step_bytes = L.bytes[k];
    p->bytes_replicated += L.bytes[k];
    p->tasks_launched += L.ntask[k];
    commit_pub_len(p);
    p->last_step = step;
    p->abort_after = -1;
  }
}

// Copies host-resident append sources into one device staging buffer (data,
// not descriptors) and points the launch at it.
int stage_host_sources(DeviceCtx *ctx, Launch &L, cudaStream_t st, StageBuf **out) {
  *out = nullptr;
  size_t total = 0;
  for (int k = 0; k < L.n_pools; ++k) {
    if (!L.host_src_bytes[k]) continue;
    // pinned (page-locked, hence mapped under UVA) host memory: the append kernel reads
    // it directly over PCIe -- no staging copy and no staging buffer to grow
    cudaPointerAttributes at;
    void *dptr = nullptr;
    if (cudaPointerGetAttributes(&at, L.host_src[k]) == cudaSuccess &&
        at.type == cudaMemoryTypeHost &&
        cudaHostGetDevicePointer(&dptr, const_cast<void *>(L.host_src[k]), 0) == cudaSuccess &&
        dptr) {
      L.params[k].src = static_cast<const char *>(dptr);
      L.host_src_bytes[k] = 0;
      continue;
    }
    cudaGetLastError();
    total += L.host_src_bytes[k];
  }
  if (total == 0) return KV_OK;
  StageBuf *sb = nullptr;
  int rc = ctx->acquire(ctx->src, ctx->next_src, total, false, &sb);
  if (rc) return rc;
  size_t off = 0;
  for (int k = 0; k < L.n_pools; ++k) {
    if (!L.host_src_bytes[k]) continue;
    CU(cudaMemcpyAsync(sb->dev + off, L.host_src[k], L.host_src_bytes[k], cudaMemcpyHostToDevice,
                       st));
    L.params[k].src = sb->dev + off;
    off += L.host_src_bytes[k];
  }
  *out = sb;
  return KV_OK;
}

// Stages the descriptors of up to two launches with ONE pinned H2D copy (launches that
// do not carry them inline in the kernel parameter space).
int stage(DeviceCtx *ctx, Launch *const *ls, int nl, cudaStream_t st, StageBuf **out) {
  size_t total = 0;
  for (int i = 0; i < nl; ++i) total += align16(ls[i]->staged_bytes());
  StageBuf *b = nullptr;
  const double ta = now_s();
  int rc = ctx->acquire(ctx->ring, ctx->next, total, true, &b);
  if (rc) return rc;
  const double tb = now_s();
  phase_add(kPhAcquire, tb - ta);
  size_t off = 0;
  for (int i = 0; i < nl; ++i) {
    Launch &L = *ls[i];
    const size_t pbytes = align16(sizeof(KvPoolParams) * L.n_pools);
    const size_t tbl = align16(L.tables.size());
    char *h = b->host + off;
    char *d = b->dev + off;
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
    off += align16(L.staged_bytes());
  }
  const double tc = now_s();
  phase_add(kPhHostCopy, tc - tb);
  CU(cudaMemcpyAsync(b->dev, b->host, total, cudaMemcpyHostToDevice, st));
  phase_add(kPhH2DCall, now_s() - tc);
  *out = b;
  return KV_OK;
}

// Grid of a copy launch: one CTA per task up to the resident CTA count (capping the
// append's grid so the concurrent ring-put finds free CTA slots was measured: no
// gain, profiles/r01/exp25.log).
int launch_grid(const Launch &L) {
  return copy_grid(L.p0->device, (int)L.tasks.size() * L.split);
}

// Shared capacity: withdraw the freed replicas' published entries (req_id -1,
// len 0 in the published parity) before this launch may reuse their blocks.
int flush_inval(Launch &L, cudaStream_t st) {
  for (const auto &iv : L.inval) {
    const int R = L.max_reqs_inval;
    CU(cudaMemsetAsync(iv.meta + 32 + ((size_t)iv.par * R + iv.slot) * 8, 0xFF, 8, st));
    CU(cudaMemsetAsync(iv.meta + meta_off_len(R) + ((size_t)iv.par * R + iv.slot) * 4, 0, 4, st));
  }
  L.inval.clear();
  return KV_OK;
}

int enqueue(Launch &L, cudaStream_t st) {
  if (!L.inval.empty() && L.p0 && L.p0->device >= 0) {
    int rc = flush_inval(L, st);
    if (rc) return rc;
  }
  if (L.tasks.empty()) return KV_OK;
  CU(timed_launch(L.kind, L.tasks_dev, (int)L.tasks.size(), L.params_dev, L.n_pools,
                  L.p0->geom_dev(), launch_grid(L), st, L.params.data(), L.split));
  phase_add(kPhStagedLaunches, 1.0);
  g_launches++;
  L.p0->kernels++;
  return KV_OK;
}

thread_local Launch g_append_launch, g_repl_launch;

// Copy-engine runs of the full blocks of a ring-put launch (consecutive block ids
// coalesced; the replica mirrors block ids, R5), issued before the kernel on the
// same stream: the kernel's publication is stream-ordered after them.
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

int replicate_impl(int n_pools, kv_pool *const *pools, uint64_t step, cudaStream_t st,
                   bool use_ce = false) {
  Launch &L = g_repl_launch;
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
  Launch *ls[1] = {&L};
  rc = stage(ctx, ls, 1, st, &b);
  if (rc) return rc;
  if (use_ce && (rc = issue_ce_copies(L, pools, st))) return rc;
  rc = enqueue(L, st);
  if (rc) return rc;
  commit_replicate(L, pools, step);
  return ctx->done(b, st);
}

}  // namespace

KV_API int kv_append_multi(int32_t n_pools, const kv_append_args_t *args, void *stream) {
  Launch &L = g_append_launch;
  int rc = prepare_append(n_pools, args, L);
  if (rc) return rc;
  if (L.p0->device < 0) return KV_OK;
  if (L.tasks.empty()) {
    if (L.inval.empty()) return KV_OK;
    DeviceGuard dg(L.p0->device);
    return flush_inval(L, static_cast<cudaStream_t>(stream));
  }
  DeviceGuard dg(L.p0->device);
  if (!dg.ok) return fail(KV_ECUDA, "cudaSetDevice failed");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceCtx *ctx = ctx_for(L.p0->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  StageBuf *sb = nullptr, *b = nullptr;
  rc = stage_host_sources(ctx, L, st, &sb);
  if (rc) return rc;
  Launch *ls[1] = {&L};
  rc = stage(ctx, ls, 1, st, &b);
  if (rc) return rc;
  rc = enqueue(L, st);
  if (rc) return rc;
  if (sb && (rc = ctx->done(sb, st))) return rc;  // the staged source outlives the kernel
  return ctx->done(b, st);
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

KV_API int kv_replicate_step(kv_pool_t *p, uint64_t step, void *stream) {
  return replicate_impl(1, &p, step, static_cast<cudaStream_t>(stream));
}

KV_API int kv_replicate_step_multi(int32_t n_pools, kv_pool_t *const *pools, uint64_t step,
                                   void *stream) {
  return replicate_impl(n_pools, pools, step, static_cast<cudaStream_t>(stream));
}

KV_API int kv_replicate_step_ce(int32_t n_pools, kv_pool_t *const *pools, uint64_t step,
                                void *stream) {
  return replicate_impl(n_pools, pools, step, static_cast<cudaStream_t>(stream), true);
}

KV_API int kv_set_mode(kv_pool_t *p, int32_t mode) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (mode != KV_MODE_TOKENS && mode != KV_MODE_BLOCKS) return fail(KV_EINVAL, "unknown mode");
  if (p->dead) return fail(KV_ESTATE, "pool %d is dead", p->node_id);
  p->repl_mode = mode;
  std::fill(p->pub_len.begin(), p->pub_len.end(), 0);  // a mode switch re-seeds the link
  return KV_OK;
}

KV_API int kv_inject_abort(kv_pool_t *p, int32_t tasks) {
  if (!p) return fail(KV_EINVAL, "null pool");
  p->abort_after = tasks < 0 ? -1 : tasks;
  return KV_OK;
}

KV_API int kv_fail_stage(kv_pool_t *p, void *stream) {
  if (!p) return fail(KV_EINVAL, "null pool");
  if (p->dead) return fail(KV_ESTATE, "pool %d already dead", p->node_id);
  p->dead = true;
  p->has_succ = false;
  if (p->device < 0) return KV_OK;
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
  if (!dst || !holder_replica || !holder_meta) return fail(KV_EINVAL, "null argument");
  if (dst->dead) return fail(KV_ESTATE, "restore target %d is dead", dst->node_id);
  if (dst->device < 0) return fail(KV_ESTATE, "restore needs a device pool");
  DeviceGuard dg(dst->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int R = dst->R, M = dst->M, B = dst->g.block_size;
  // 1. acquire the holder's seq and the parity metadata (synchronous read).
  std::vector<char> meta(meta_bytes(R, M));
  CU(cudaStreamSynchronize(st));
  CU(cudaMemcpy(meta.data(), holder_meta, 32, cudaMemcpyDefault));
  uint64_t seq;
  int32_t hdr[4];
  std::memcpy(&seq, meta.data(), 8);
  std::memcpy(hdr, meta.data() + 8, 16);
  if (hdr[3] != kMetaMagic || hdr[1] != R || hdr[2] != M)
    return fail(KV_ENOREPLICA, "holder metadata invalid (magic %x, R %d, M %d)", hdr[3], hdr[1],
                hdr[2]);
  if (seq == 0 || seq == ~0ull) return fail(KV_ENOREPLICA, "holder published nothing (seq %llu)",
                                            (unsigned long long)seq);
  CU(cudaMemcpy(meta.data(), holder_meta, meta.size(), cudaMemcpyDefault));
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
  // 3. copy valid slots (local HBM, or NVLink reads when the holder is remote).
  if (!tasks.empty()) {
    DeviceCtx *ctx = ctx_for(dst->device);
    std::lock_guard<std::mutex> lk(ctx->mu);
    KvPoolParams pp;
    std::memset(&pp, 0, sizeof pp);
    pp.src = static_cast<const char *>(holder_replica);
    pp.dst = dst->pool;
    pp.src_bytes = (unsigned long long)holder_replica_blocks * dst->block_bytes;
    pp.dst_bytes = (unsigned long long)dst->NB * dst->block_bytes;
    const size_t pbytes = sizeof pp, tbytes = sizeof(KvTask) * tasks.size();
    StageBuf *b = nullptr;
    int rc = ctx->acquire(ctx->ring, ctx->next, pbytes + tbytes, true, &b);
    if (rc) return rc;
    std::memcpy(b->host, &pp, pbytes);
    std::memcpy(b->host + pbytes, tasks.data(), tbytes);
    CU(cudaMemcpyAsync(b->dev, b->host, pbytes + tbytes, cudaMemcpyHostToDevice, st));
    CU(timed_launch(kKindRestore, reinterpret_cast<const KvTask *>(b->dev + pbytes),
                   (int)tasks.size(), reinterpret_cast<const KvPoolParams *>(b->dev), 1,
                   dst->geom_dev(), copy_grid(dst->device, (int)tasks.size()), st));
    g_launches++;
    dst->kernels++;
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

namespace {

// Inline descriptors (KvInlineDesc): a launch whose tables + tasks fit the kernel
// parameter space travels with the launch itself (KVRING_INLINE=0 disables).
// Published-table entries of pool q a ring-put launch must carry: up to the last
// slot listed (later slots publish (-1, 0), written by the kernel).
int table_hi(const Launch &L, int q) {
  const int R = L.params[q].max_reqs;
  const int64_t *rq = reinterpret_cast<const int64_t *>(L.tables.data() + L.table_off[q]);
  int hi = R;
  while (hi > 0 && rq[hi - 1] < 0) --hi;
  return hi;
}

size_t inline_table_bytes(const Launch &L) {
  if (L.kind != kKindRingPut) return 0;
  size_t b = 0;
  for (int q = 0; q < L.n_pools; ++q) b += align16(12 * (size_t)table_hi(L, q));
  return b;
}

bool inline_fits(const Launch &L) {
  static const int enabled = [] {
    const char *e = getenv("KVRING_INLINE");
    return e ? atoi(e) : 1;
  }();
  return enabled && L.n_pools <= kInlinePools &&
         inline_table_bytes(L) + sizeof(KvTask) * L.tasks.size() <= (size_t)kInlineBytes;
}

void fill_inline(const Launch &L, KvInlineDesc &d) {
  size_t off = 0;
  for (int q = 0; q < L.n_pools; ++q) {
    d.pools[q] = L.params[q];
    if (L.kind != kKindRingPut) continue;
    const int R = L.params[q].max_reqs, hi = table_hi(L, q);
    const char *t = L.tables.data() + L.table_off[q];
    std::memcpy(d.data + off, t, 8 * (size_t)hi);                       // req ids
    std::memcpy(d.data + off + 8 * (size_t)hi, t + 8 * (size_t)R, 4 * (size_t)hi);  // lens
    d.pools[q].slot_req = reinterpret_cast<const int64_t *>(off);
    d.pools[q].slot_len = reinterpret_cast<const int32_t *>(off + 8 * (size_t)hi);
    d.pools[q].n_table = hi;
    off += align16(12 * (size_t)hi);
  }
  d.n_tasks = (int32_t)L.tasks.size();
  d.n_pools = L.n_pools;
  d.task_off = (int32_t)off;
  d.split = L.split;
  std::memcpy(d.data + off, L.tasks.data(), sizeof(KvTask) * L.tasks.size());
  d.used = (int32_t)(off + sizeof(KvTask) * L.tasks.size());
}

}  // namespace

// ---- decode-loop driver -------------------------------------------------------
// For each step: appends on the compute stream, then (after an event) the
// publication on the replication stream -- the paper's "separate CUDA stream
// ... to overlap the communication with computation" (§3.2).
namespace {

// Host side of one decode step, prepared ahead of its CUDA calls.
struct StepPrep {
  Launch A, P;
  bool has_a = false, has_p = false;
  bool shared = false;  // a pool of this step is in shared-capacity mode (NEXT-3)
  // inline descriptors (kernel parameter space), filled on the helper thread
  bool inl_a = false, inl_p = false;
  bool no_inline = false;  // the graph loop stages every step's descriptors
  std::unique_ptr<KvInlineDesc> da, dp;
  int rc = KV_OK;
  std::string err;
};

// Tables, work lists and (already) committed publication state of step k.
// Commit happens here, before the launch: the next step's dirty ranges start
// where this one ends; a launch error is sticky and ends the run anyway.
bool any_shared(const kv_step_t &st) {
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

void prepare_step(const kv_step_t &st, StepPrep &sp) {
  sp.has_a = st.n_append > 0;
  sp.has_p = st.n_repl > 0;
  sp.rc = KV_OK;
  sp.shared = any_shared(st);
  const double t0 = now_s();
  if (sp.has_a && (sp.rc = prepare_append(st.n_append, st.append, sp.A))) {
    sp.err = g_err;
    return;
  }
  const double t1 = now_s();
  phase_add(kPhPrepAppend, t1 - t0);
  if (sp.has_p) {
    if ((sp.rc = prepare_replicate(st.n_repl, st.repl_pools, st.step, sp.P))) {
      sp.err = g_err;
      return;
    }
    const double t2 = now_s();
    phase_add(kPhPrepRepl, t2 - t1);
    commit_replicate(sp.P, st.repl_pools, st.step);
    phase_add(kPhCommit, now_s() - t2);
  }
  kv_pool *p0 = sp.has_a ? sp.A.p0 : (sp.has_p ? sp.P.p0 : nullptr);
  if (p0 && sp.has_a && sp.has_p && sp.P.p0->device != p0->device) {
    sp.rc = fail(KV_EINVAL, "append and publication of one step must share a device");
    sp.err = g_err;
    return;
  }
  // descriptors that fit the kernel parameter space travel with the launch (no
  // staging copy, no H2D, no dependent descriptor load); host-source appends and
  // large (prefill / bulk) steps are staged
  sp.inl_a = sp.inl_p = false;
  if (!p0 || p0->device < 0 || sp.no_inline) return;
  bool host_src = false;
  if (sp.has_a)
    for (size_t q = 0; q < sp.A.host_src_bytes.size(); ++q) host_src |= sp.A.host_src_bytes[q] != 0;
  if (sp.has_a && !host_src && !sp.A.tasks.empty() && inline_fits(sp.A)) {
    if (!sp.da) sp.da.reset(new KvInlineDesc());
    fill_inline(sp.A, *sp.da);
    sp.inl_a = true;
  }
  if (sp.has_p && !sp.P.tasks.empty() && inline_fits(sp.P)) {
    if (!sp.dp) sp.dp.reset(new KvInlineDesc());
    fill_inline(sp.P, *sp.dp);
    sp.inl_p = true;
  }
}

// Launch of a prepared inline launch (events of kv_time_next_launch honoured).
int enqueue_inline(Launch &L, const KvInlineDesc &d, cudaStream_t st, bool pdl) {
  if (!L.inval.empty()) {
    int rc = flush_inval(L, st);
    if (rc) return rc;
  }
  if (L.tasks.empty()) return KV_OK;
  cudaEvent_t b = g_ev_before, a = g_ev_after;
  g_ev_before = g_ev_after = nullptr;
  if (b) CU(cudaEventRecord(b, st));
  CU(launch_copy_inline(L.kind, d, L.p0->geom_dev(), launch_grid(L), st, pdl));
  phase_add(kPhInlineLaunches, 1.0);  // a count (kv_host_profile divides like the times)
  if (a) CU(cudaEventRecord(a, st));
  g_launches++;
  L.p0->kernels++;
  return KV_OK;
}

// Cross-stream order of the two-stream loop: ring-put k after append k (event
// `ready`), and append k after ring-put k-2 -- blocks a retiring request frees in
// step k-1 are reused from step k on (quarantine, reading R7), and the ring-put
// that last read them is k-2's, which may otherwise still lag on its stream.
struct StreamOrder {
  static constexpr int kN = 4;
  cudaEvent_t aready[kN] = {};  // recorded on the append stream after append k
  cudaEvent_t rdone[kN] = {};   // recorded on the replication stream after ring-put k
  long long astep[kN] = {-1, -1, -1, -1};
  long long rstep[kN] = {-1, -1, -1, -1};
  long long n = 0;  // steps issued on this stream pair (continues across calls)
  cudaStream_t sa = nullptr, sr = nullptr;
  int dev = -1;
  int ensure(int device) {
    if (dev == device) return KV_OK;
    for (auto &e : aready)
      if (e) cudaEventDestroy(e);
    for (auto &e : rdone)
      if (e) cudaEventDestroy(e);
    for (int i = 0; i < kN; ++i) {
      aready[i] = rdone[i] = nullptr;
      astep[i] = rstep[i] = -1;
    }
    sa = sr = nullptr;
    for (auto &e : aready) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : rdone) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    dev = device;
    return KV_OK;
  }
};

// CUDA side of one prepared step, in two halves that may run on two host threads
// (kv_run_steps pipelines them): the append on sa (after the ring-put of step
// k - lag, see StreamOrder), then the publication on sr (the paper's separate
// replication stream) after an event on sa.  Inline launches need no
// staging; a staged launch gets its own H2D on its own stream.
int issue_append(const kv_step_t &st, long long k, StepPrep &sp, cudaStream_t sa,
                 cudaStream_t sr, StreamOrder &so) {
  kv_pool *p0 = sp.has_a ? sp.A.p0 : (sp.has_p ? sp.P.p0 : nullptr);
  if (!p0 || p0->device < 0) return KV_OK;  // nothing to launch / tables-only pools
  DeviceGuard dg(p0->device);
  int rc = KV_OK;
  if (sa != sr && (rc = so.ensure(p0->device))) return rc;
  const int N = StreamOrder::kN;
  if (sp.has_a && (!sp.A.tasks.empty() || !sp.A.inval.empty())) {
    DeviceCtx *ctx = ctx_for(p0->device);
    std::lock_guard<std::mutex> lk(ctx->mu);
    StageBuf *sb = nullptr, *b = nullptr;
    const double t0 = now_s();
    if ((rc = stage_host_sources(ctx, sp.A, sa, &sb))) return rc;
    Launch *ls[1] = {&sp.A};
    if (!sp.inl_a && !sp.A.tasks.empty() && (rc = stage(ctx, ls, 1, sa, &b))) return rc;
    const double t1 = now_s();
    phase_add(kPhStage, t1 - t0);
    // shared capacity: a freed replica block may be reused by this very append, so
    // the ring-put that last wrote it (k-1) must be complete
    const int lag = sp.shared ? 1 : 2;
    if (sa != sr && k >= lag && so.rstep[(k - lag) % N] == k - lag)
      CU(cudaStreamWaitEvent(sa, so.rdone[(k - lag) % N], 0));
    g_ev_before = static_cast<cudaEvent_t>(st.ev_append_start);
    g_ev_after = static_cast<cudaEvent_t>(st.ev_append_end);
    rc = sp.inl_a ? enqueue_inline(sp.A, *sp.da, sa, false) : enqueue(sp.A, sa);
    g_ev_before = g_ev_after = nullptr;
    if (rc) return rc;
    if (sb && (rc = ctx->done(sb, sa))) return rc;  // the staged source outlives the kernel
    if (b && (rc = ctx->done(b, sa))) return rc;
    phase_add(kPhEnqA, now_s() - t1);
  }
  if (sa != sr && sp.has_p) {  // the publication of step k follows this append
    CU(cudaEventRecord(so.aready[k % N], sa));
    so.astep[k % N] = k;
  }
  return KV_OK;
}

int issue_publish(const kv_step_t &st, long long k, StepPrep &sp, cudaStream_t sa,
                  cudaStream_t sr, StreamOrder &so) {
  kv_pool *p0 = sp.has_a ? sp.A.p0 : (sp.has_p ? sp.P.p0 : nullptr);
  if (!p0 || p0->device < 0 || !sp.has_p) return KV_OK;
  DeviceGuard dg(p0->device);
  const int N = StreamOrder::kN;
  const double t0 = now_s();
  if (sa != sr && so.astep[k % N] == k) CU(cudaStreamWaitEvent(sr, so.aready[k % N], 0));
  if (st.ev_call) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_call), sr));
  const double t1 = now_s();
  phase_add(kPhEvents, t1 - t0);
  DeviceCtx *ctx = ctx_for(p0->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  StageBuf *b = nullptr;
  int rc = KV_OK;
  Launch *ls[1] = {&sp.P};
  if (!sp.inl_p && !sp.P.tasks.empty() && (rc = stage(ctx, ls, 1, sr, &b))) return rc;
  phase_add(kPhPubStage, now_s() - t1);
  g_ev_before = static_cast<cudaEvent_t>(st.ev_kernel_start);
  g_ev_after = static_cast<cudaEvent_t>(st.ev_kernel_end);
  rc = sp.inl_p ? enqueue_inline(sp.P, *sp.dp, sr, false) : enqueue(sp.P, sr);
  g_ev_before = g_ev_after = nullptr;
  if (rc) return rc;
  if (st.ev_done) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_done), sr));
  if (sa != sr) {
    CU(cudaEventRecord(so.rdone[k % N], sr));
    so.rstep[k % N] = k;
  }
  if (b && (rc = ctx->done(b, sr))) return rc;
  phase_add(kPhEnqP, now_s() - t1);
  return KV_OK;
}

}  // namespace

// Decode-loop driver.  For runs of >= 8 steps a helper thread prepares step
// k+1 (allocation, tables, work lists) while this thread issues step k's CUDA
// calls; the two meet through a 2-deep ring of StepPrep.
KV_API int kv_run_steps(int32_t n_steps, const kv_step_t *steps, void *append_stream,
                        void *repl_stream) {
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  cudaStream_t sa = static_cast<cudaStream_t>(append_stream);
  cudaStream_t sr = static_cast<cudaStream_t>(repl_stream);
  thread_local StreamOrder so;
  if (sa != sr && n_steps > 0) {
    const kv_step_t &s0 = steps[0];
    kv_pool *q = s0.n_append > 0 ? s0.append[0].pool : (s0.n_repl > 0 ? s0.repl_pools[0] : nullptr);
    if (q && q->device >= 0 && (so.sa != sa || so.sr != sr || so.dev != q->device)) {
      // a new stream pair: everything already on sr precedes this call's appends
      DeviceGuard dg(q->device);
      int rc = so.ensure(q->device);
      if (rc) return rc;
      for (int i = 0; i < StreamOrder::kN; ++i) so.rstep[i] = so.astep[i] = -1;
      CU(cudaEventRecord(so.rdone[0], sr));
      CU(cudaStreamWaitEvent(sa, so.rdone[0], 0));
      so.sa = sa;
      so.sr = sr;
    }
  }
  if (n_steps < 8) {
    thread_local StepPrep sp;
    for (int k = 0; k < n_steps; ++k) {
      prepare_step(steps[k], sp);
      if (sp.rc) return sp.rc;
      const long long kk = so.n++;
      int rc = issue_append(steps[k], kk, sp, sa, sr, so);
      if (!rc) rc = issue_publish(steps[k], kk, sp, sa, sr, so);
      if (rc) return rc;
    }
    return KV_OK;
  }
  // A helper thread prepares step k+1 (allocation, tables, work lists, inline
  // descriptors) while this thread issues step k's CUDA calls; a 2-deep ring of
  // StepPrep.  (Issuing the appends from the helper too was measured slower:
  // concurrent launches from two threads contend in the driver.)
  StepPrep ring[2];  // shared with the worker (per call: reentrant across threads)
  std::atomic<int> produced{0}, consumed{0};
  std::atomic<bool> stop{false};
  std::thread worker([&]() {
    for (int k = 0; k < n_steps && !stop.load(std::memory_order_acquire); ++k) {
      const double w0 = now_s();
      while (k - consumed.load(std::memory_order_acquire) >= 2) {
        if (stop.load(std::memory_order_acquire)) return;
        std::this_thread::yield();
      }
      phase_add(kPhWaitIssue, now_s() - w0);
      StepPrep &sp = ring[k & 1];
      const double t0 = now_s();
      prepare_step(steps[k], sp);
      phase_add(kPhPrepare, now_s() - t0);
      produced.store(k + 1, std::memory_order_release);
      if (sp.rc) return;
    }
  });
  int rc = KV_OK;
  for (int k = 0; k < n_steps; ++k) {
    const double w0 = now_s();
    while (produced.load(std::memory_order_acquire) <= k) std::this_thread::yield();
    phase_add(kPhWaitPrep, now_s() - w0);
    StepPrep &sp = ring[k & 1];
    if (sp.rc) {
      rc = sp.rc;
      g_err = sp.err;
      break;
    }
    const long long kk = so.n++;
    rc = issue_append(steps[k], kk, sp, sa, sr, so);
    if (!rc) rc = issue_publish(steps[k], kk, sp, sa, sr, so);
    consumed.store(k + 1, std::memory_order_release);
    if (rc) break;
  }
  stop.store(true, std::memory_order_release);
  worker.join();
  return rc;
}

// ---- CUDA-graph decode loop ---------------------------------------------------
// The same work as kv_run_steps, issued as one CUDA graph per group of graph_steps() (8)
// steps: per step an append kernel node and a ring-put kernel node with the
// stream-order constraints of kv_run_steps as graph edges (append k after append
// k-1 and after ring-put k-2 -- R7 --, ring-put k after append k and after ring-put
// k-1), all descriptors of the group staged by ONE H2D memcpy node.  A kernel node
// costs the device < 1 us instead of 2-4 us for a stream launch and the host a
// ~0.3 us parameter update instead of a 3-6 us launch (tools/launchbench.cu).
// Consecutive groups run on the two streams and are chained by event-wait nodes,
// so group g+1 overlaps the tail of group g exactly like consecutive steps do.
namespace {

constexpr int kGraphMax = 32;  // node arrays; the group size itself: graph_steps()
// Steps per graph (KVRING_GRAPH_STEPS, 2..32, default 8), read once per process.
int graph_steps() {
  static const int n = [] {
    const char *e = getenv("KVRING_GRAPH_STEPS");
    const int v = e ? atoi(e) : 8;
    return std::max(2, std::min(kGraphMax, v));
  }();
  return n;
}

struct GraphLoop {
  static constexpr int kEv = 4, kSlots = 4;
  int device = -1;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge[kSlots] = {};  // 2 used (parity), or one per slot in fixed mode
  bool fixed = false;  // self-describing steps: kernel nodes never updated per step
  KvFxArgs fx[3 * kGraphMax];
  cudaGraphNode_t mc = nullptr, wait_a = nullptr, wait_r2 = nullptr, wait_r1 = nullptr;
  cudaGraphNode_t an[kGraphMax] = {}, rn[kGraphMax] = {}, pn[kGraphMax] = {};
  cudaGraphNode_t es[kGraphMax] = {}, ee[kGraphMax] = {};
  cudaGraphNode_t rec_a = nullptr, rec_r2 = nullptr, rec_r1 = nullptr, rec_p = nullptr;
  cudaGraphNode_t wait_p = nullptr;
  cudaEvent_t ev_a[kEv] = {}, ev_r2[kEv] = {}, ev_r1[kEv] = {}, ev_p[kEv] = {};
  bool split_pub = false;  // ring-put = copy node + separate publication node
  bool lean = false;       // no timing event nodes (KVRING_GRAPH_LEAN=1, experiments)
  cudaEvent_t start_a = nullptr, start_r = nullptr, join = nullptr;
  cudaEvent_t dummy[2 * kGraphMax] = {};
  StageBuf slot[kSlots];
  KvNodeArgs args[3 * kGraphMax];
  int steps = 8;  // group size of this graph
  // last values set per exec instance: skip redundant update calls (each ~0.3 us)
  signed char enabled[kSlots][3 * kGraphMax];
  cudaEvent_t ev_set[kSlots][2 * kGraphMax] = {};
  long long group = 0;
  std::mutex mu;  // one call at a time per device (the graph and its slots are shared)

  int make_event(cudaEvent_t *e) {
    CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return KV_OK;
  }
  // Fixed mode: point exec e's kernel nodes at slot e (once, and after a slot grows).
  int bind_slot(int e) {
    const int fx_grid = resident_ctas(device);
    for (int k = 0; k < steps; ++k) {
      cudaKernelNodeParams kp{};
      KvFxArgs a{slot[e].dev, k};
      fx_node_params(kKindAppend, fx_grid, a, kp);
      CU(cudaGraphExecKernelNodeSetParams(ge[e], an[k], &kp));
      fx_node_params(kKindRingPutCopy, fx_grid, a, kp);
      CU(cudaGraphExecKernelNodeSetParams(ge[e], rn[k], &kp));
      fx_node_params(kKindPublish, kFxPublishGrid, a, kp);
      CU(cudaGraphExecKernelNodeSetParams(ge[e], pn[k], &kp));
    }
    return KV_OK;
  }
  int build(int dev) {
    device = dev;
    for (int i = 0; i < kEv; ++i) {
      int rc = make_event(&ev_a[i]);
      if (!rc) rc = make_event(&ev_r2[i]);
      if (!rc) rc = make_event(&ev_r1[i]);
      if (!rc) rc = make_event(&ev_p[i]);
      if (rc) return rc;
    }
    for (auto &e : dummy)
      if (int rc = make_event(&e)) return rc;
    if (int rc = make_event(&start_a)) return rc;
    if (int rc = make_event(&start_r)) return rc;
    if (int rc = make_event(&join)) return rc;
    for (auto &sl : slot) {
      const size_t cap = 32u << 20;
      CU(cudaHostAlloc(reinterpret_cast<void **>(&sl.host), cap, cudaHostAllocDefault));
      CU(cudaMalloc(reinterpret_cast<void **>(&sl.dev), cap));
      sl.cap = cap;
      CU(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
    }
    CU(cudaGraphCreate(&g, 0));
    CU(cudaGraphAddMemcpyNode1D(&mc, g, nullptr, 0, slot[0].dev, slot[0].host, 16,
                                cudaMemcpyHostToDevice));
    CU(cudaGraphAddEventWaitNode(&wait_a, g, nullptr, 0, start_a));
    CU(cudaGraphAddEventWaitNode(&wait_r2, g, nullptr, 0, start_r));
    CU(cudaGraphAddEventWaitNode(&wait_r1, g, nullptr, 0, start_r));
    // the publication as its own node (KVRING_GRAPH_SPLIT_PUB=0: inside the ring-put):
    // the copies lose the per-CTA release RMW and bar.sync tail (ring-put node 10.7 vs
    // 14.3 us median, +5 % steps/s, profiles/r01/exp43.log)
    split_pub = [] {
      const char *e = getenv("KVRING_GRAPH_SPLIT_PUB");
      return e ? atoi(e) != 0 : true;
    }();
    if (split_pub) CU(cudaGraphAddEventWaitNode(&wait_p, g, nullptr, 0, start_r));
    // self-describing steps (KVRING_GRAPH_FIXED=1, needs the split publication): each
    // kernel node reads its launch from the step header in the group's slot
    fixed = split_pub && [] {
      const char *e = getenv("KVRING_GRAPH_FIXED");
      return e ? atoi(e) != 0 : false;
    }();
    const int fx_grid = resident_ctas(dev);
    // experiment knob KVRING_GRAPH_LAG=1: append k waits for ring-put k-1 (no overlap of
    // an append with the previous publication); default 2 (reading R7's minimum)
    static const int lag = [] {
      const char *e = getenv("KVRING_GRAPH_LAG");
      return e && atoi(e) == 1 ? 1 : 2;
    }();
    steps = graph_steps();
    // Timing event nodes sit beside the chain (es(k) has R(k)'s dependencies, ee(k)
    // follows R(k)); no kernel waits on them unless KVRING_GRAPH_EVENTS_IN_CHAIN=1.
    static const bool in_chain = getenv("KVRING_GRAPH_EVENTS_IN_CHAIN") != nullptr;
    lean = !in_chain && getenv("KVRING_GRAPH_LEAN") != nullptr;  // experiment knob
    for (int k = 0; k < steps; ++k) {
      cudaKernelNodeParams kp{};
      if (fixed) {
        fx[3 * k] = KvFxArgs{slot[0].dev, k};
        fx_node_params(kKindAppend, fx_grid, fx[3 * k], kp);
      } else {
        kernel_node_params(kKindAppend, 1, args[2 * k], kp);
      }
      cudaGraphNode_t rprev = k > 0 ? (in_chain ? ee[k - 1] : rn[k - 1]) : wait_r1;
      cudaGraphNode_t lagdep =
          lag == 2 ? (k >= 2 ? (in_chain ? ee[k - 2] : rn[k - 2]) : (k == 0 ? wait_r2 : wait_r1))
                   : rprev;
      // append k also follows the LAUNCH of ring-put k-1 (the node that becomes ready with
      // it, its start event): the publication then gets the free CTA slots first
      // (+2-10 % measured, profiles/r01/exp39.log)
      cudaGraphNode_t da[4] = {mc, k > 0 ? an[k - 1] : wait_a, lagdep,
                               k > 0 ? es[k - 1] : nullptr};
      CU(cudaGraphAddKernelNode(&an[k], g, da, k > 0 ? 4 : 3, &kp));
      cudaGraphNode_t ds[2] = {an[k], rprev};
      if (lean)  // experiment: no timing nodes (an empty node keeps the ordering role)
        CU(cudaGraphAddEmptyNode(&es[k], g, ds, 2));
      else
        CU(cudaGraphAddEventRecordNode(&es[k], g, ds, 2, dummy[2 * k]));
      if (fixed) {
        fx[3 * k + 1] = KvFxArgs{slot[0].dev, k};
        fx_node_params(kKindRingPutCopy, fx_grid, fx[3 * k + 1], kp);
      } else {
        kernel_node_params(split_pub ? kKindRingPutCopy : kKindRingPut, 1, args[2 * k + 1], kp);
      }
      if (in_chain)
        CU(cudaGraphAddKernelNode(&rn[k], g, &es[k], 1, &kp));
      else
        CU(cudaGraphAddKernelNode(&rn[k], g, ds, 2, &kp));
      if (!lean) CU(cudaGraphAddEventRecordNode(&ee[k], g, &rn[k], 1, dummy[2 * k + 1]));
      if (split_pub) {  // publication k after copies k and publication k-1 (seq order)
        if (fixed) {
          fx[3 * k + 2] = KvFxArgs{slot[0].dev, k};
          fx_node_params(kKindPublish, kFxPublishGrid, fx[3 * k + 2], kp);
        } else {
          kernel_node_params(kKindPublish, 1, args[2 * kGraphMax + k], kp);
        }
        cudaGraphNode_t dp[2] = {rn[k], k > 0 ? pn[k - 1] : wait_p};
        CU(cudaGraphAddKernelNode(&pn[k], g, dp, 2, &kp));
      }
    }
    CU(cudaGraphAddEventRecordNode(&rec_a, g, &an[steps - 1], 1, ev_a[0]));
    CU(cudaGraphAddEventRecordNode(&rec_r2, g, &rn[steps - 2], 1, ev_r2[0]));
    CU(cudaGraphAddEventRecordNode(&rec_r1, g, &rn[steps - 1], 1, ev_r1[0]));
    if (split_pub) CU(cudaGraphAddEventRecordNode(&rec_p, g, &pn[steps - 1], 1, ev_p[0]));
    for (int e = 0; e < (fixed ? kSlots : 2); ++e) {
      CU(cudaGraphInstantiate(&ge[e], g, 0));
      if (fixed) {
        int rc = bind_slot(e);
        if (rc) return rc;
      }
    }
    std::memset(enabled, -1, sizeof enabled);
    return KV_OK;
  }
};

std::mutex g_graph_mu;
std::map<int, std::unique_ptr<GraphLoop>> g_graph;

// Packs one launch's descriptors (params, publication tables, tasks) into a group
// slot at `off` and points the launch at the device copy.
void pack_launch(Launch &L, char *h, char *d, size_t &off) {
  const size_t pbytes = align16(sizeof(KvPoolParams) * L.n_pools);
  const size_t tbl = align16(L.tables.size());
  for (int k = 0; k < L.n_pools; ++k)
    if (L.kind == kKindRingPut) {
      const size_t o = off + pbytes + L.table_off[k];
      L.params[k].slot_req = reinterpret_cast<const int64_t *>(d + o);
      L.params[k].slot_len = reinterpret_cast<const int32_t *>(d + o + 8 * (size_t)L.params[k].max_reqs);
    }
  std::memcpy(h + off, L.params.data(), sizeof(KvPoolParams) * L.n_pools);
  if (!L.tables.empty()) std::memcpy(h + off + pbytes, L.tables.data(), L.tables.size());
  std::memcpy(h + off + pbytes + tbl, L.tasks.data(), sizeof(KvTask) * L.tasks.size());
  L.params_dev = reinterpret_cast<const KvPoolParams *>(d + off);
  L.tasks_dev = reinterpret_cast<const KvTask *>(d + off + pbytes + tbl);
  off += align16(L.staged_bytes());
}

int set_kernel_node(cudaGraphExec_t ge, cudaGraphNode_t node, Launch *L, bool present,
                    KvNodeArgs &a, int kind, signed char &enabled) {
  cudaKernelNodeParams kp{};
  a = KvNodeArgs{};
  int grid = 1;
  if (present && L && !L->tasks.empty()) {
    a.tasks = L->tasks_dev;
    a.n_tasks = (int)L->tasks.size();
    a.params = L->params_dev;
    a.g = L->p0->geom_dev();
    a.n_pools = L->n_pools;
    a.split = L->split;
    if (L->n_pools <= kInlinePools) {
      a.pk.n = L->n_pools;
      for (int q = 0; q < L->n_pools; ++q) {
        a.pk.src[q] = L->params[q].src;
        a.pk.dst[q] = L->params[q].dst;
      }
    }
    grid = kind == kKindPublish ? L->n_pools : launch_grid(*L);  // publication: CTA per pool
  }
  kernel_node_params(kind, grid, a, kp);
  CU(cudaGraphExecKernelNodeSetParams(ge, node, &kp));
  if (enabled != (present ? 1 : 0)) {
    CU(cudaGraphNodeSetEnabled(ge, node, present ? 1 : 0));
    enabled = present ? 1 : 0;
  }
  return KV_OK;
}

// Issues group [k0, k0 + n) of prepared steps (n <= G.steps).
int issue_group(GraphLoop &G, const kv_step_t *steps, StepPrep *const *sp, int n,
                cudaStream_t sa, cudaStream_t sr, bool first) {
  const int N = GraphLoop::kEv;
  const long long gi = G.group++;
  const int se = (int)(gi % GraphLoop::kSlots);
  StageBuf &sl = G.slot[se];
  const size_t hdr_bytes = G.fixed ? align16(sizeof(KvStepHdr) * G.steps) : 0;
  const double t0 = now_s();
  if (sl.pending) {
    CU(cudaEventSynchronize(sl.ev));
    sl.pending = false;
  }
  phase_add(kPhAcquire, now_s() - t0);
  size_t need = hdr_bytes;
  for (int i = 0; i < n; ++i) {
    if (sp[i]->has_a) need += align16(sp[i]->A.staged_bytes());
    if (sp[i]->has_p) need += align16(sp[i]->P.staged_bytes());
  }
  if (need > sl.cap) {  // rare (bulk steps): grow this slot
    if (sl.host) cudaFreeHost(sl.host);
    if (sl.dev) cudaFree(sl.dev);
    const size_t cap = std::max(need * 2, sl.cap);
    CU(cudaHostAlloc(reinterpret_cast<void **>(&sl.host), cap, cudaHostAllocDefault));
    CU(cudaMalloc(reinterpret_cast<void **>(&sl.dev), cap));
    sl.cap = cap;
    if (G.fixed) {
      int rc = G.bind_slot(se);
      if (rc) return rc;
    }
  }
  const double t1 = now_s();
  size_t off = hdr_bytes;
  KvStepHdr *hdr = reinterpret_cast<KvStepHdr *>(sl.host);
  for (int i = 0; i < (G.fixed ? G.steps : n); ++i) {
    KvStepHdr h{};
    if (i < n) {
      Launch *ls2[2] = {sp[i]->has_a && !sp[i]->A.tasks.empty() ? &sp[i]->A : nullptr,
                        sp[i]->has_p && !sp[i]->P.tasks.empty() ? &sp[i]->P : nullptr};
      for (int w = 0; w < 2; ++w) {
        Launch *L = ls2[w];
        if (!L) continue;
        pack_launch(*L, sl.host, sl.dev, off);
        h.n_tasks[w] = (int32_t)L->tasks.size();
        h.n_pools[w] = L->n_pools;
        h.split[w] = L->split;
        h.params_off[w] = (unsigned long long)(reinterpret_cast<const char *>(L->params_dev) - sl.dev);
        h.tasks_off[w] = (unsigned long long)(reinterpret_cast<const char *>(L->tasks_dev) - sl.dev);
        h.g = L->p0->geom_dev();
      }
    }
    if (G.fixed) hdr[i] = h;
  }
  phase_add(kPhHostCopy, now_s() - t1);
  const double tu = now_s();
  const int par = (int)(gi & 1);
  const int xi = G.fixed ? se : par;  // exec instance (and its update caches)
  cudaGraphExec_t ge = G.ge[xi];
  cudaStream_t st = par ? sr : sa;
  CU(cudaGraphExecMemcpyNodeSetParams1D(ge, G.mc, sl.dev, sl.host, off > 0 ? off : 16,
                                        cudaMemcpyHostToDevice));
  const int pe = (int)((gi + N - 1) % N);
  CU(cudaGraphExecEventWaitNodeSetEvent(ge, G.wait_a, first ? G.start_a : G.ev_a[pe]));
  CU(cudaGraphExecEventWaitNodeSetEvent(ge, G.wait_r2, first ? G.start_r : G.ev_r2[pe]));
  CU(cudaGraphExecEventWaitNodeSetEvent(ge, G.wait_r1, first ? G.start_r : G.ev_r1[pe]));
  if (G.split_pub)
    CU(cudaGraphExecEventWaitNodeSetEvent(ge, G.wait_p, first ? G.start_r : G.ev_p[pe]));
  for (int k = 0; k < G.steps; ++k) {
    const bool on = k < n;
    StepPrep *s = on ? sp[k] : nullptr;
    if (!G.fixed) {  // fixed mode: the step header in the slot describes the launches
      signed char *en = G.enabled[xi];
      int rc = set_kernel_node(ge, G.an[k], s ? &s->A : nullptr, on && s->has_a, G.args[2 * k],
                               kKindAppend, en[3 * k]);
      if (!rc)
        rc = set_kernel_node(ge, G.rn[k], s ? &s->P : nullptr, on && s->has_p,
                             G.args[2 * k + 1], G.split_pub ? kKindRingPutCopy : kKindRingPut,
                             en[3 * k + 1]);
      if (!rc && G.split_pub)
        rc = set_kernel_node(ge, G.pn[k], s ? &s->P : nullptr, on && s->has_p,
                             G.args[2 * kGraphMax + k], kKindPublish, en[3 * k + 2]);
      if (rc) return rc;
    }
    cudaEvent_t e0 = G.dummy[2 * k], e1 = G.dummy[2 * k + 1];
    if (on && steps[k].ev_kernel_start) e0 = static_cast<cudaEvent_t>(steps[k].ev_kernel_start);
    if (on && steps[k].ev_kernel_end) e1 = static_cast<cudaEvent_t>(steps[k].ev_kernel_end);
    if (G.lean) e0 = e1 = nullptr;
    if (e0 && G.ev_set[xi][2 * k] != e0) {
      CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.es[k], e0));
      G.ev_set[xi][2 * k] = e0;
    }
    if (e1 && G.ev_set[xi][2 * k + 1] != e1) {
      CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.ee[k], e1));
      G.ev_set[xi][2 * k + 1] = e1;
    }
    if (on) {
      if (s->has_a && !s->A.tasks.empty()) {
        g_launches++;
        s->A.p0->kernels++;
      }
      if (s->has_p && !s->P.tasks.empty()) {
        g_launches++;
        s->P.p0->kernels++;
      }
    }
  }
  CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.rec_a, G.ev_a[gi % N]));
  CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.rec_r2, G.ev_r2[gi % N]));
  CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.rec_r1, G.ev_r1[gi % N]));
  if (G.split_pub) CU(cudaGraphExecEventRecordNodeSetEvent(ge, G.rec_p, G.ev_p[gi % N]));
  const double t2 = now_s();
  phase_add(kPhEvents, t2 - tu);  // graph node updates (reported as "events")
  CU(cudaGraphLaunch(ge, st));
  CU(cudaEventRecord(sl.ev, st));
  sl.pending = true;
  phase_add(kPhEnqP, now_s() - t2);
  return KV_OK;
}

}  // namespace

KV_API int kv_run_steps_graph(int32_t n_steps, const kv_step_t *steps, void *append_stream,
                              void *repl_stream) {
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  if (n_steps == 0) return KV_OK;
  cudaStream_t sa = static_cast<cudaStream_t>(append_stream);
  cudaStream_t sr = static_cast<cudaStream_t>(repl_stream);
  if (sa == sr) return fail(KV_EINVAL, "kv_run_steps_graph needs two distinct streams");
  kv_pool *p0 = nullptr;
  for (int k = 0; k < n_steps; ++k) {
    if (any_shared(steps[k]))
      return fail(KV_EINVAL, "shared-capacity pools need kv_run_steps");
    for (int i = 0; i < steps[k].n_append; ++i) {
      if (steps[k].append[i].flags & KV_SRC_HOST)
        return fail(KV_EINVAL, "KV_SRC_HOST is not supported by kv_run_steps_graph");
      if (!p0) p0 = steps[k].append[i].pool;
    }
    if (!p0 && steps[k].n_repl > 0) p0 = steps[k].repl_pools[0];
  }
  if (!p0) return fail(KV_EINVAL, "no pools");
  if (p0->device < 0) return fail(KV_ESTATE, "kv_run_steps_graph needs device pools");
  DeviceGuard dg(p0->device);
  GraphLoop *G;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto &up = g_graph[p0->device];
    if (!up) {
      up.reset(new GraphLoop());
      if (int rc = up->build(p0->device)) {
        up.reset();
        return rc;
      }
    }
    G = up.get();
  }
  std::lock_guard<std::mutex> call_lock(G->mu);
  // earlier work on both streams precedes the first group
  CU(cudaEventRecord(G->start_a, sa));
  CU(cudaEventRecord(G->start_r, sr));
  const int GS = G->steps;
  const int R = 2 * GS;  // prepared-step ring shared with the helper
  std::vector<StepPrep> ring(R);
  for (auto &x : ring) x.no_inline = true;
  std::atomic<int> produced{0}, consumed{0};
  std::atomic<bool> stop{false};
  std::thread worker([&]() {
    for (int k = 0; k < n_steps && !stop.load(std::memory_order_acquire); ++k) {
      const double w0 = now_s();
      while (k - consumed.load(std::memory_order_acquire) >= R) {
        if (stop.load(std::memory_order_acquire)) return;
        std::this_thread::yield();
      }
      phase_add(kPhWaitIssue, now_s() - w0);
      const double t0 = now_s();
      prepare_step(steps[k], ring[k % R]);
      phase_add(kPhPrepare, now_s() - t0);
      produced.store(k + 1, std::memory_order_release);
      if (ring[k % R].rc) return;
    }
  });
  int rc = KV_OK;
  cudaStream_t last = sa;
  for (int k0 = 0; k0 < n_steps && !rc; k0 += GS) {
    const int n = std::min(GS, n_steps - k0);
    const double w0 = now_s();
    while (produced.load(std::memory_order_acquire) < k0 + n) {
      if (ring[(produced.load() + R - 1) % R].rc && produced.load() > 0) break;
      std::this_thread::yield();
    }
    phase_add(kPhWaitPrep, now_s() - w0);
    StepPrep *sp[kGraphMax];
    for (int i = 0; i < n; ++i) {
      sp[i] = &ring[(k0 + i) % R];
      if (produced.load(std::memory_order_acquire) <= k0 + i || sp[i]->rc) {
        rc = sp[i]->rc ? sp[i]->rc : KV_EINVAL;
        g_err = sp[i]->err;
        break;
      }
    }
    if (rc) break;
    rc = issue_group(*G, steps + k0, sp, n, sa, sr, k0 == 0);
    last = (G->group - 1) & 1 ? sr : sa;
    consumed.store(k0 + n, std::memory_order_release);
  }
  stop.store(true, std::memory_order_release);
  worker.join();
  if (!rc) {  // both streams end after the last group
    cudaStream_t other = last == sa ? sr : sa;
    CU(cudaEventRecord(G->join, last));
    CU(cudaStreamWaitEvent(other, G->join, 0));
  }
  return rc;
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

// ---- software-pipelined decode loop (single stream) --------------------------
namespace {

struct FusedPrep {
  Launch A, P;        // append of step k, publication of step k-1
  bool has_a = false, has_p = false;
  int rc = KV_OK;
  std::string err;
};

// Prepare launch k: the publication of step k-1 FIRST (its dirty ranges end at
// len_{k-1}), then the append of step k (which moves len on).
void prepare_fused(const kv_step_t *steps, int n_steps, int k, FusedPrep &fp) {
  fp.rc = KV_OK;
  fp.has_p = k >= 1 && steps[k - 1].n_repl > 0;
  fp.has_a = k < n_steps && steps[k].n_append > 0;
  if (fp.has_p) {
    const kv_step_t &pv = steps[k - 1];
    if ((fp.rc = prepare_replicate(pv.n_repl, pv.repl_pools, pv.step, fp.P, false, false))) {
      fp.err = g_err;
      return;
    }
    commit_replicate(fp.P, pv.repl_pools, pv.step);
  }
  if (fp.has_a && (fp.rc = prepare_append(steps[k].n_append, steps[k].append, fp.A, false))) {
    fp.err = g_err;
    return;
  }
  if (fp.has_a && fp.has_p && fp.A.p0->device != fp.P.p0->device) {
    fp.rc = fail(KV_EINVAL, "append and publication of one launch must share a device");
    fp.err = g_err;
  }
}

// One H2D: [A params | P params] [P tables] [A tasks | P tasks]; P tasks keep
// pool indices local to P (the kernel offsets its params pointer).
int stage_fused(DeviceCtx *ctx, FusedPrep &fp, cudaStream_t st, StageBuf **out,
                const KvPoolParams **params_dev, const KvTask **tasks_dev) {
  Launch &A = fp.A, &P = fp.P;
  const int na = fp.has_a ? A.n_pools : 0, np = fp.has_p ? P.n_pools : 0;
  const size_t pbytes = align16(sizeof(KvPoolParams) * (size_t)(na + np));
  const size_t tbl = fp.has_p ? align16(P.tables.size()) : 0;
  const size_t nta = fp.has_a ? A.tasks.size() : 0, ntp = fp.has_p ? P.tasks.size() : 0;
  const size_t total = pbytes + tbl + sizeof(KvTask) * (nta + ntp);
  StageBuf *b = nullptr;
  const double ta = now_s();
  int rc = ctx->acquire(ctx->ring, ctx->next, total, true, &b);
  if (rc) return rc;
  const double tb = now_s();
  phase_add(kPhAcquire, tb - ta);
  char *h = b->host, *d = b->dev;
  for (int k = 0; k < np; ++k) {
    P.params[k].slot_req = reinterpret_cast<const int64_t *>(d + pbytes + P.table_off[k]);
    P.params[k].slot_len =
        reinterpret_cast<const int32_t *>(d + pbytes + P.table_off[k] + 8 * (size_t)P.params[k].max_reqs);
  }
  if (na) std::memcpy(h, A.params.data(), sizeof(KvPoolParams) * na);
  if (np) std::memcpy(h + sizeof(KvPoolParams) * na, P.params.data(), sizeof(KvPoolParams) * np);
  if (tbl) std::memcpy(h + pbytes, P.tables.data(), P.tables.size());
  if (nta) std::memcpy(h + pbytes + tbl, A.tasks.data(), sizeof(KvTask) * nta);
  if (ntp) std::memcpy(h + pbytes + tbl + sizeof(KvTask) * nta, P.tasks.data(), sizeof(KvTask) * ntp);
  const double tc = now_s();
  phase_add(kPhHostCopy, tc - tb);
  CU(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, st));
  phase_add(kPhH2DCall, now_s() - tc);
  *params_dev = reinterpret_cast<const KvPoolParams *>(d);
  *tasks_dev = reinterpret_cast<const KvTask *>(d + pbytes + tbl);
  *out = b;
  return KV_OK;
}

int issue_fused(const kv_step_t *ev_step, FusedPrep &fp, cudaStream_t st) {
  kv_pool *p0 = fp.has_a ? fp.A.p0 : (fp.has_p ? fp.P.p0 : nullptr);
  if (!p0 || p0->device < 0) return KV_OK;
  DeviceGuard dg(p0->device);
  DeviceCtx *ctx = ctx_for(p0->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  StageBuf *sb = nullptr, *b = nullptr;
  int rc = KV_OK;
  double t0 = now_s();
  if (fp.has_a && (rc = stage_host_sources(ctx, fp.A, st, &sb))) return rc;
  const KvPoolParams *pd = nullptr;
  const KvTask *td = nullptr;
  if ((rc = stage_fused(ctx, fp, st, &b, &pd, &td))) return rc;
  double t1 = now_s();
  phase_add(kPhStage, t1 - t0);
  const int na = fp.has_a ? fp.A.n_pools : 0, np = fp.has_p ? fp.P.n_pools : 0;
  const int nta = fp.has_a ? (int)fp.A.tasks.size() : 0;
  const int ntot = nta + (fp.has_p ? (int)fp.P.tasks.size() : 0);
  if (ntot > 0) {
    if (ev_step && ev_step->ev_kernel_start)
      CU(cudaEventRecord(static_cast<cudaEvent_t>(ev_step->ev_kernel_start), st));
    CU(launch_fused(td, nta, ntot, pd, na, np, p0->geom_dev(), copy_grid(p0->device, ntot), st));
    if (ev_step && ev_step->ev_kernel_end)
      CU(cudaEventRecord(static_cast<cudaEvent_t>(ev_step->ev_kernel_end), st));
    g_launches++;
    p0->kernels++;
  }
  if (sb && (rc = ctx->done(sb, st))) return rc;
  rc = ctx->done(b, st);
  phase_add(kPhEnqA, now_s() - t1);
  return rc;
}

}  // namespace

// Single-stream, software-pipelined decode loop: launch k carries the append of
// step k AND the publication of step k-1 (disjoint slots, see kv_step_fused_kernel),
// a last launch publishes step n-1.  Same work as kv_run_steps, half the launches,
// no cross-stream event; the publication of a step trails its append by one launch
// -- the overlap of replication with the next step's compute of P:229.
KV_API int kv_run_steps_fused(int32_t n_steps, const kv_step_t *steps, void *stream) {
  for (int k = 0; k < n_steps && steps; ++k)
    if (any_shared(steps[k]))
      return fail(KV_EINVAL, "shared-capacity pools need kv_run_steps (append after ring-put k-1)");
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n_launch = n_steps + 1;  // + the flush of the last publication
  if (n_steps < 8) {
    thread_local FusedPrep fp;
    for (int k = 0; k < n_launch; ++k) {
      prepare_fused(steps, n_steps, k, fp);
      if (fp.rc) return fp.rc;
      int rc = issue_fused(k < n_steps ? &steps[k] : nullptr, fp, st);
      if (rc) return rc;
    }
    return KV_OK;
  }
  FusedPrep ring[2];
  std::atomic<int> produced{0}, consumed{0};
  std::atomic<bool> stop{false};
  std::thread worker([&]() {
    for (int k = 0; k < n_launch && !stop.load(std::memory_order_acquire); ++k) {
      const double w0 = now_s();
      while (k - consumed.load(std::memory_order_acquire) >= 2) {
        if (stop.load(std::memory_order_acquire)) return;
        std::this_thread::yield();
      }
      phase_add(kPhWaitIssue, now_s() - w0);
      const double t0 = now_s();
      prepare_fused(steps, n_steps, k, ring[k & 1]);
      phase_add(kPhPrepare, now_s() - t0);
      produced.store(k + 1, std::memory_order_release);
      if (ring[k & 1].rc) return;
    }
  });
  int rc = KV_OK;
  for (int k = 0; k < n_launch; ++k) {
    const double w0 = now_s();
    while (produced.load(std::memory_order_acquire) <= k) std::this_thread::yield();
    phase_add(kPhWaitPrep, now_s() - w0);
    FusedPrep &fp = ring[k & 1];
    if (fp.rc) {
      rc = fp.rc;
      g_err = fp.err;
      break;
    }
    rc = issue_fused(k < n_steps ? &steps[k] : nullptr, fp, st);
    consumed.store(k + 1, std::memory_order_release);
    if (rc) break;
  }
  stop.store(true, std::memory_order_release);
  worker.join();
  return rc;
}

// ---- single-stream decode loop with programmatic dependent launch ----------------
namespace {

// One step of the PDL loop: launches whose descriptors fit the parameter space go
// inline with the PDL attribute (no copy node between kernels); larger ones (bulk
// prefill steps) are staged by one H2D and launched normally -- that step
// serialises, the kernels' griddepcontrol calls are then no-ops.
int issue_step_pdl(const kv_step_t &st, int k, StepPrep &sp, cudaStream_t s) {
  (void)k;
  kv_pool *p0 = sp.has_a ? sp.A.p0 : (sp.has_p ? sp.P.p0 : nullptr);
  if (!p0 || p0->device < 0) return KV_OK;
  DeviceGuard dg(p0->device);
  const bool has_a = sp.has_a && !sp.A.tasks.empty(), has_p = sp.has_p && !sp.P.tasks.empty();
  if (sp.has_a)
    for (size_t q = 0; q < sp.A.host_src_bytes.size(); ++q)
      if (sp.A.host_src_bytes[q])
        return fail(KV_EINVAL, "KV_SRC_HOST is not supported by kv_run_steps_pdl");
  const bool inl_a = has_a && sp.inl_a, inl_p = has_p && sp.inl_p;  // filled by prepare_step
  const double t0 = now_s();
  DeviceCtx *ctx = ctx_for(p0->device);
  std::lock_guard<std::mutex> lk(ctx->mu);
  Launch *ls[2];
  int nl = 0;
  if (has_a && !inl_a) ls[nl++] = &sp.A;
  if (has_p && !inl_p) ls[nl++] = &sp.P;
  StageBuf *b = nullptr;
  int rc = KV_OK;
  if (nl && (rc = stage(ctx, ls, nl, s, &b))) return rc;
  const double t1 = now_s();
  phase_add(kPhStage, t1 - t0);
  if (has_a) {
    if (st.ev_append_start) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_append_start), s));
    if (inl_a) {
      if ((rc = enqueue_inline(sp.A, *sp.da, s, true))) return rc;
    } else if ((rc = enqueue(sp.A, s))) {
      return rc;
    }
    if (st.ev_append_end) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_append_end), s));
  }
  const double t2 = now_s();
  phase_add(kPhEnqA, t2 - t1);
  if (has_p) {
    if (st.ev_kernel_start) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_kernel_start), s));
    if (inl_p) {
      if ((rc = enqueue_inline(sp.P, *sp.dp, s, true))) return rc;
    } else if ((rc = enqueue(sp.P, s))) {
      return rc;
    }
    if (st.ev_kernel_end) CU(cudaEventRecord(static_cast<cudaEvent_t>(st.ev_kernel_end), s));
  }
  if (b && (rc = ctx->done(b, s))) return rc;
  phase_add(kPhEnqP, now_s() - t2);
  return KV_OK;
}

}  // namespace

// Single-stream decode loop with programmatic dependent launch: per step the
// append and the publication are launched back to back on ONE stream with the
// PDL attribute, descriptors travel in the kernel parameter space (inline), and the
// kernels order themselves with griddepcontrol (see kvring_kernels.cu): the
// publication of step k starts as soon as append k completes and runs while append
// k+1 copies -- the overlap the paper gets from a separate stream, without
// a cross-stream event per step.  A helper thread prepares step k+1 meanwhile.
KV_API int kv_run_steps_pdl(int32_t n_steps, const kv_step_t *steps, void *stream) {
  if (n_steps < 0 || (n_steps > 0 && !steps)) return fail(KV_EINVAL, "bad steps");
  for (int k = 0; k < n_steps; ++k)
    if (any_shared(steps[k]))
      return fail(KV_EINVAL, "shared-capacity pools need kv_run_steps (append after ring-put k-1)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  StepPrep ring[2];
  std::atomic<int> produced{0}, consumed{0};
  std::atomic<bool> stop{false};
  std::thread worker([&]() {
    for (int k = 0; k < n_steps && !stop.load(std::memory_order_acquire); ++k) {
      const double w0 = now_s();
      while (k - consumed.load(std::memory_order_acquire) >= 2) {
        if (stop.load(std::memory_order_acquire)) return;
        std::this_thread::yield();
      }
      phase_add(kPhWaitIssue, now_s() - w0);
      const double t0 = now_s();
      prepare_step(steps[k], ring[k & 1]);
      phase_add(kPhPrepare, now_s() - t0);
      produced.store(k + 1, std::memory_order_release);
      if (ring[k & 1].rc) return;
    }
  });
  int rc = KV_OK;
  for (int k = 0; k < n_steps; ++k) {
    const double w0 = now_s();
    while (produced.load(std::memory_order_acquire) <= k) std::this_thread::yield();
    phase_add(kPhWaitPrep, now_s() - w0);
    StepPrep &sp = ring[k & 1];
    if (sp.rc) {
      rc = sp.rc;
      g_err = sp.err;
      break;
    }
    rc = issue_step_pdl(steps[k], k, sp, s);
    consumed.store(k + 1, std::memory_order_release);
    if (rc) break;
  }
  stop.store(true, std::memory_order_release);
  worker.join();
  return rc;
}
