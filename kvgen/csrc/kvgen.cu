// CUDA twin of kvgen/content.py (input generator; no replication arithmetic).
//
//   content(seed, req, l, kv, h, pos, dim) = T[l,kv,h,dim] ^ word16(K(seed,req,pos), dim % 4)
//   K(seed, req, pos) = sm(sm(sm(seed) ^ req) ^ pos)
//   T[idx]            = sm(sm(seed ^ TABLE_SALT) ^ idx) & 0xFFFF,
//                       idx = ((l*2 + kv)*H + h)*d + dim   (l = global layer)
// with sm = splitmix64.  tests/test_kvgen_cuda.py pins it byte-for-byte to the
// numpy generator.  Output layout: dense [n][L][2][H][d] uint16 (the layout
// kv_append consumes).
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kTableSalt = 0x4B565441424C45ull;

__host__ __device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One thread = 8 consecutive words (16 B) of one token's dense row.
__global__ void content_kernel(unsigned long long seed_mix, unsigned long long salt_mix,
                               const int64_t *__restrict__ req, const int32_t *__restrict__ pos,
                               long long n, int layer0, int L, int H, int d,
                               uint16_t *__restrict__ out) {
  const long long words_per_tok = (long long)L * 2 * H * d;
  const long long chunks = n * (words_per_tok / 8);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < chunks;
       c += (long long)gridDim.x * blockDim.x) {
    const long long w0 = c * 8;
    const long long tok = w0 / words_per_tok;
    const long long within = w0 - tok * words_per_tok;  // index in [L][2][H][d]
    const unsigned long long key =
        sm64(sm64(seed_mix ^ (unsigned long long)req[tok]) ^ (unsigned long long)(long long)pos[tok]);
    const long long lkvh = within / d;
    const int dim0 = (int)(within - lkvh * d);
    const long long l_local = lkvh / (2 * H);
    const long long rest = lkvh - l_local * 2 * H;  // kv*H + h
    const unsigned long long base =
        ((unsigned long long)((layer0 + l_local) * 2 * H + rest)) * (unsigned long long)d;
    uint16_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int dim = dim0 + k;
      const uint16_t t = (uint16_t)(sm64(salt_mix ^ (base + dim)) & 0xFFFFull);
      const uint16_t wd = (uint16_t)((key >> (16 * (dim & 3))) & 0xFFFFull);
      v[k] = t ^ wd;
    }
    uint4 pk;
    pk.x = v[0] | ((uint32_t)v[1] << 16);
    pk.y = v[2] | ((uint32_t)v[3] << 16);
    pk.z = v[4] | ((uint32_t)v[5] << 16);
    pk.w = v[6] | ((uint32_t)v[7] << 16);
    *reinterpret_cast<uint4 *>(out + w0) = pk;
  }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int kvgen_content(
    unsigned long long seed, const int64_t *req_dev, const int32_t *pos_dev, long long n,
    int layer0, int L, int H, int d, uint16_t *out_dev, void *stream) {
  if (n <= 0) return 0;
  if (d % 8 != 0) return -1;
  const unsigned long long seed_mix = sm64(seed);
  const unsigned long long salt_mix = sm64(seed ^ kTableSalt);
  const long long chunks = n * ((long long)L * 2 * H * d / 8);
  long long grid = (chunks + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  content_kernel<<<(int)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed_mix, salt_mix, req_dev, pos_dev, n, layer0, L, H, d, out_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---- test support: concurrent reader of a replica's publication (reading R9) ----------
// One CTA spins on a replica metadata's seq with ld.acquire.sys while the predecessor
// (another GPU) keeps publishing.  For every new seq it snapshots the parity (seq & 1)
// (req_id, len) table and, for each listed slot, the first 256-B slice of its last valid
// token (layer 0, K, head 0), then re-reads seq (acquire) so the host can drop snapshots
// whose parity buffer was overwritten meanwhile (seq advanced by >= 2); stops at
// `last_seq` (the writer's final step) or after `max_spin` polls without news.  Records:
//   out[k] = { u64 seq, u64 seq_after, i64 req[R], i32 len[R], u16 slice[R][d] }
// Bounded: gives up after `max_spin` polls without a new seq.  Test infrastructure.
namespace {
__global__ void r9_observe_kernel(const char *meta, const char *replica, int R, int M, int B,
                                  long long block_bytes, int seg_bytes, int n_obs,
                                  long long max_spin, unsigned long long last_seq, char *out,
                                  long long rec_bytes, int *n_done) {
  __shared__ unsigned long long s_seq;
  __shared__ int s_stop;
  unsigned long long last = 0;
  int k = 0;
  while (k < n_obs) {
    if (threadIdx.x == 0) {
      unsigned long long v = last;
      long long spin = 0;
      while (v == last && spin < max_spin) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(meta) : "memory");
        ++spin;
      }
      s_seq = v;
      s_stop = (v == last);
    }
    __syncthreads();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (s_stop) break;
    const unsigned long long seq = s_seq;
    last = seq;
    char *rec = out + (long long)k * rec_bytes;
    const int par = (int)(seq & 1ull);
    const long long *mreq = reinterpret_cast<const long long *>(meta + 32) + (long long)par * R;
    const int *mlen = reinterpret_cast<const int *>(meta + 32 + 16LL * R) + (long long)par * R;
    const int *mbt = reinterpret_cast<const int *>(meta + 32 + 24LL * R);
    long long *oreq = reinterpret_cast<long long *>(rec + 16);
    int *olen = reinterpret_cast<int *>(rec + 16 + 8LL * R);
    char *oslice = rec + 16 + 12LL * R;
    for (int s = threadIdx.x; s < R; s += blockDim.x) {
      const long long r = *(volatile const long long *)(mreq + s);
      const int ln = *(volatile const int *)(mlen + s);
      oreq[s] = r;
      olen[s] = ln;
      if (r >= 0 && ln > 0) {
        const int pos = ln - 1;
        const int blk = *(volatile const int *)(mbt + (long long)s * M + pos / B);
        const char *src = replica + (long long)blk * block_bytes + (long long)(pos % B) * seg_bytes;
        for (int b = 0; b < seg_bytes; b += 4)
          *reinterpret_cast<int *>(oslice + (long long)s * seg_bytes + b) =
              *(volatile const int *)(src + b);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(meta) : "memory");
      reinterpret_cast<unsigned long long *>(rec)[0] = seq;
      reinterpret_cast<unsigned long long *>(rec)[1] = v;
    }
    __syncthreads();
    ++k;
    if (seq >= last_seq) break;  // the writer's final step
  }
  if (threadIdx.x == 0) *n_done = k;
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int kvgen_r9_observe(
    const void *meta, const void *replica, int R, int M, int B, long long block_bytes,
    int seg_bytes, int n_obs, long long max_spin, unsigned long long last_seq, void *out,
    long long rec_bytes, int *n_done, void *stream) {
  r9_observe_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char *>(meta), static_cast<const char *>(replica), R, M, B, block_bytes,
      seg_bytes, n_obs, max_spin, last_seq, static_cast<char *>(out), rec_bytes, n_done);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---- workload proxy: paged decode attention over the live KV (bench interference leg) --
// The model-side consumer replication competes with for HBM: for
// every (request, layer, KV head) one warp streams the request's K and V slices out of the
// paged pool (layout [blk][L][2][H][B][d], bf16) and computes softmax(q.K / sqrt(d)) V for
// the GQA group's `qpk` query heads with an online softmax.  Reads every valid KV slot once
// per step, as a decode step's attention does.  Workload proxy, not part of the method.
namespace {
__device__ __forceinline__ float bf16f(uint16_t x) { return __uint_as_float((uint32_t)x << 16); }

__global__ void attn_proxy_kernel(const char *const *pools, const int *req_pool,
                                  const int *req_len, const int *req_bt_off, const int *bt,
                                  int n_req, int L, int H, int B, int d, int qpk,
                                  const float *q, float *out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int per_req = L * H;
  if (warp >= n_req * per_req) return;
  const int r = warp / per_req, lh = warp % per_req, l = lh / H, h = lh % H;
  const char *pool = pools[req_pool[r]];
  const long long blk_bytes = (long long)L * 2 * H * B * d * 2;
  const int dv = d / 32;  // dims per lane (d = 128: 4)
  float qv[4][4], acc[4][4], m[4], ssum[4];
  for (int g = 0; g < qpk && g < 4; ++g) {
    for (int k = 0; k < dv && k < 4; ++k) {
      qv[g][k] = q[((long long)(lh * qpk + g)) * d + lane * dv + k];
      acc[g][k] = 0.f;
    }
    m[g] = -1e30f;
    ssum[g] = 0.f;
  }
  const float scale = rsqrtf((float)d);
  const int len = req_len[r];
  for (int t = 0; t < len; ++t) {
    const int blk = bt[req_bt_off[r] + t / B];
    const char *base = pool + (long long)blk * blk_bytes;
    const uint16_t *kp = reinterpret_cast<const uint16_t *>(
        base + ((((long long)l * 2 + 0) * H + h) * B + (t % B)) * d * 2);
    const uint16_t *vp = reinterpret_cast<const uint16_t *>(
        base + ((((long long)l * 2 + 1) * H + h) * B + (t % B)) * d * 2);
    float kf[4], vf[4];
    for (int k = 0; k < dv && k < 4; ++k) {
      kf[k] = bf16f(kp[lane * dv + k]);
      vf[k] = bf16f(vp[lane * dv + k]);
    }
    for (int g = 0; g < qpk && g < 4; ++g) {
      float s = 0.f;
      for (int k = 0; k < dv && k < 4; ++k) s += qv[g][k] * kf[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      s *= scale;
      if (!(s == s) || s > 1e30f || s < -1e30f) s = 0.f;  // the words are arbitrary bits
      const float mn = fmaxf(m[g], s), c = __expf(m[g] - mn), p = __expf(s - mn);
      ssum[g] = ssum[g] * c + p;
      for (int k = 0; k < dv && k < 4; ++k) {
        const float v = (vf[k] == vf[k] && fabsf(vf[k]) < 1e30f) ? vf[k] : 0.f;
        acc[g][k] = acc[g][k] * c + p * v;
      }
      m[g] = mn;
    }
  }
  for (int g = 0; g < qpk && g < 4; ++g)
    for (int k = 0; k < dv && k < 4; ++k)
      out[((long long)(warp * qpk + g)) * d + lane * dv + k] = acc[g][k] / fmaxf(ssum[g], 1e-30f);
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int kvgen_attn_proxy(
    const void *pools_dev, const int *req_pool, const int *req_len, const int *req_bt_off,
    const int *bt, int n_req, int L, int H, int B, int d, int qpk, const float *q, float *out,
    void *stream) {
  if (d % 32 != 0 || d > 128 || qpk > 4) return -1;
  const long long warps = (long long)n_req * L * H;
  const int threads = 256;
  const long long grid = (warps * 32 + threads - 1) / threads;
  attn_proxy_kernel<<<(int)grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char *const *>(pools_dev), req_pool, req_len, req_bt_off, bt, n_req, L,
      H, B, d, qpk, q, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
