// libkvnccl: a thin native driver of NCCL send/recv for the MEASURED COMPARISON transport
// (the paper's transport, P:8 §3.3: "NCCL ... direct GPU-to-GPU").
// It issues the grouped ncclSend / ncclRecv of a replication step's packed buffers on the
// caller's stream with no Python in between (a communicator of one rank sends to itself:
// the N = 1 loopback runs through NCCL too).  Links against the NCCL 2.28 that ships with
// the torch venv.  Plain C ABI: include/kvnccl.h.
#include <cstdio>
#include <cstring>

#include <cuda_runtime_api.h>
#include <nccl.h>

#include "kvnccl.h"

#define KVN_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local char g_msg[256];
int fail(ncclResult_t r, const char *what) {
  snprintf(g_msg, sizeof g_msg, "%s: %s", what, ncclGetErrorString(r));
  return -1;
}
}  // namespace

KVN_API const char *kvn_last_error(void) { return g_msg; }

KVN_API int kvn_unique_id_bytes(void) { return NCCL_UNIQUE_ID_BYTES; }

KVN_API int kvn_get_unique_id(void *out) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
  return 0;
}

KVN_API int kvn_comm_init(int nranks, int rank, const void *unique_id, int device,
                          void **comm_out) {
  if (cudaSetDevice(device) != cudaSuccess) {
    snprintf(g_msg, sizeof g_msg, "cudaSetDevice(%d) failed", device);
    return -1;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return fail(r, "ncclCommInitRank");
  *comm_out = c;
  return 0;
}

KVN_API int kvn_comm_destroy(void *comm) {
  if (!comm) return 0;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? 0 : fail(r, "ncclCommDestroy");
}

// One group: n_send sends (buffer, bytes, peer rank) and n_recv receives, all on `stream`.
// Byte counts must match pairwise (NCCL point-to-point semantics).
KVN_API int kvn_sendrecv(void *comm, int n_send, const void *const *sbuf, const size_t *sbytes,
                         const int *speer, int n_recv, void *const *rbuf, const size_t *rbytes,
                         const int *rpeer, void *stream) {
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return fail(r, "ncclGroupStart");
  for (int i = 0; i < n_send && r == ncclSuccess; ++i)
    r = ncclSend(sbuf[i], sbytes[i], ncclUint8, speer[i], c, st);
  for (int i = 0; i < n_recv && r == ncclSuccess; ++i)
    r = ncclRecv(rbuf[i], rbytes[i], ncclUint8, rpeer[i], c, st);
  ncclResult_t e = ncclGroupEnd();
  if (r != ncclSuccess) return fail(r, "ncclSend/ncclRecv");
  if (e != ncclSuccess) return fail(e, "ncclGroupEnd");
  return 0;
}
