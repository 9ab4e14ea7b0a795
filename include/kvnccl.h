/*
 * kvnccl.h -- C ABI of libkvnccl: NCCL send/recv driver of the COMPARISON transport of
 * ring KV-cache replication.  KevlarFlow replicates KV blocks with NCCL
 * send/recv (§3.3); this build's transport is one-sided NVLink stores
 * (kvring.h), and this library exists so that the paper's transport can be measured on
 * the same packed payload (kv_pack_step -> send/recv -> kv_unpack).
 *
 * Every call returns 0 or -1 (message: kvn_last_error(), thread-local).  Buffers are
 * device pointers owned by the caller; streams are cudaStream_t passed as void*.
 */
#ifndef KVNCCL_H
#define KVNCCL_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *kvn_last_error(void);
/* Size of an ncclUniqueId (128). */
int kvn_unique_id_bytes(void);
/* Writes a fresh ncclUniqueId (rank 0 creates it, the caller distributes it). */
int kvn_get_unique_id(void *out);
/* Joins communicator `unique_id` as `rank` of `nranks` on CUDA device `device`
 * (synchronises with the other ranks).  nranks = 1 is allowed: the rank then sends to
 * and receives from itself (the N = 1 loopback through NCCL). */
int kvn_comm_init(int nranks, int rank, const void *unique_id, int device, void **comm_out);
int kvn_comm_destroy(void *comm);
/* ONE ncclGroupStart/ncclGroupEnd group on `stream`: n_send ncclSend of sbytes[i] bytes
 * from sbuf[i] to rank speer[i], and n_recv ncclRecv of rbytes[i] bytes into rbuf[i] from
 * rank rpeer[i].  Counts must match the peer's (point-to-point semantics). */
int kvn_sendrecv(void *comm, int n_send, const void *const *sbuf, const size_t *sbytes,
                 const int *speer, int n_recv, void *const *rbuf, const size_t *rbytes,
                 const int *rpeer, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KVNCCL_H */
