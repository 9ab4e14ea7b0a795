"""NCCL send/recv transport for the ring hop -- the MEASURED COMPARISON only
(§8(a) a6).  The paper replicates with NCCL send/recv (P:8 §3.3); here that path is:
gather-pack the dirty slices of each local node into one contiguous device buffer
(kv_pack_step), learn the packed byte count of every incoming link (a receive must name
the sender's count: one host-side exchange per step over a gloo group, no GPU sync),
then ONE grouped ncclSend/ncclRecv (libkvnccl: include/kvnccl.h, NCCL 2.28 from the
torch venv), then kv_unpack on the receiver (scatter into the replica region + publish
the seq flag).  HBM traffic is 2D (pack) + 2D (unpack) on top of the D that crosses
NVLink, versus D read + D remote write for the one-sided ring-put.

Every link goes through NCCL, the successor on the same GPU included: at world size 1
the communicator has one rank and NCCL sends to itself.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import kvring as K

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def kvn():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libkvnccl.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build()")
        L = ctypes.CDLL(path)
        P, I, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        for name, res, args in (
                ("kvn_last_error", ctypes.c_char_p, []),
                ("kvn_unique_id_bytes", I, []),
                ("kvn_get_unique_id", I, [P]),
                ("kvn_comm_init", I, [I, I, P, I, ctypes.POINTER(P)]),
                ("kvn_comm_destroy", I, [P]),
                ("kvn_sendrecv", I, [P, I, P, P, P, I, P, P, P, P])):
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("libkvnccl: " + kvn().kvn_last_error().decode(errors="replace"))


class NcclRing:
    def __init__(self, rt, max_packed_bytes: int):
        self.rt = rt
        self.dev = rt.dev
        self.send_bufs = {}
        self.recv_bufs = {}
        self.cap = max_packed_bytes
        nb = kvn().kvn_unique_id_bytes()
        uid = ctypes.create_string_buffer(nb)
        if rt.rank == 0:
            _check(kvn().kvn_get_unique_id(uid))
        if rt.world > 1:
            obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=0, group=rt.group)
            uid = ctypes.create_string_buffer(obj[0], nb)
            # host-side count exchange: a gloo group (CPU), so no GPU synchronisation
            self.gloo = dist.new_group(backend="gloo")
        comm = ctypes.c_void_p()
        _check(kvn().kvn_comm_init(rt.world, rt.rank, uid, rt.device, ctypes.byref(comm)))
        self.comm = comm.value

    def destroy(self) -> None:
        if self.comm:
            _check(kvn().kvn_comm_destroy(self.comm))
            self.comm = None

    def _buf(self, table, key, need: int = 0):
        """Per-link buffer of at least max(cap, need) bytes (grown on demand)."""
        b = table.get(key)
        if b is None or b.numel() < need:
            b = torch.empty(max(self.cap, need), dtype=torch.uint8, device=self.dev)
            table[key] = b
        return b

    def step(self, t: int, stream=None, events=None) -> int:
        """Replicate step t of every local node through NCCL; returns the packed bytes sent.
        events: optional (before_send, after_recv) CUDA events around the NCCL group."""
        rt = self.rt
        s = torch.cuda.current_stream(self.dev) if stream is None else stream
        out_nodes = [n for n in rt.alive_local() if rt.succ.get(n) is not None]
        sizes = {}
        with torch.cuda.stream(s):
            for n in out_nodes:
                buf = self._buf(self.send_bufs, n, K.kv_pack_bytes(rt.handle(n)))
                sizes[n] = K.kv_pack_step(rt.handle(n), t, buf, buf.numel(), s.cuda_stream)
            # the packed size of every link, known on its sender's host: one host exchange
            n_ids = max(rt.placement) + 1
            if rt.world > 1:
                vec = torch.zeros(n_ids, dtype=torch.int64)
                for n in out_nodes:
                    vec[n] = sizes[n]
                dist.all_reduce(vec, group=self.gloo)
                all_sizes = {n: int(vec[n]) for n in range(n_ids) if int(vec[n]) > 0}
            else:
                all_sizes = dict(sizes)
            sends, recvs = [], []
            for n in out_nodes:
                m = rt.succ[n]
                sends.append((self.send_bufs[n], sizes[n], rt.placement[m]))
            incoming = []
            for n, sz in all_sizes.items():
                m = rt.succ.get(n)
                if m is not None and m in rt.local and m not in rt.dead and n not in rt.dead:
                    rb = self._buf(self.recv_bufs, m, sz)
                    recvs.append((rb, sz, rt.placement[n]))
                    incoming.append((m, rb, sz))
            P = ctypes.c_void_p
            sb = (P * max(1, len(sends)))(*[x[0].data_ptr() for x in sends])
            ss = (ctypes.c_size_t * max(1, len(sends)))(*[x[1] for x in sends])
            sp = (ctypes.c_int * max(1, len(sends)))(*[x[2] for x in sends])
            rbp = (P * max(1, len(recvs)))(*[x[0].data_ptr() for x in recvs])
            rs = (ctypes.c_size_t * max(1, len(recvs)))(*[x[1] for x in recvs])
            rp = (ctypes.c_int * max(1, len(recvs)))(*[x[2] for x in recvs])
            if events:
                events[0].record(s)
            _check(kvn().kvn_sendrecv(self.comm, len(sends), sb, ss, sp, len(recvs), rbp, rs, rp,
                                      s.cuda_stream))
            if events:
                events[1].record(s)
            for m, rb, sz in incoming:
                dst = rt.local[m]
                K.kv_unpack(rb, sz, dst.replica, rt.NB, dst.meta, rt.kg, rt.R, rt.M,
                            s.cuda_stream)
        return sum(sizes.values())
