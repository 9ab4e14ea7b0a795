"""NCCL send/recv transport for the ring hop -- the MEASURED COMPARISON only
(§8(a) a6).  The paper replicates with NCCL send/recv (P:8 §3.3); here that
path is: gather-pack the dirty slices of each local node into one contiguous
device buffer (kv_pack_step), exchange the packed byte count (a receive needs
the sender's count, so the receiver synchronises on it: one extra round trip),
then grouped ncclSend/ncclRecv of the payload, then kv_unpack on the receiver
(scatter into the replica region + publish the seq flag).  HBM traffic is 2D
(pack) + 2D (unpack) on top of the D that crosses NVLink, versus D read + D
remote write for the fused ring-put.

At world size 1 (loopback) the payload does not leave the GPU: pack, then
unpack into the local successor.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import kvring as K


class NcclRing:
    def __init__(self, rt, max_packed_bytes: int):
        self.rt = rt
        self.dev = rt.dev
        self.send_bufs = {}
        self.recv_bufs = {}
        self.cap = max_packed_bytes

    def _buf(self, table, key, need: int = 0):
        """Per-link buffer of at least max(cap, need) bytes (grown on demand)."""
        b = table.get(key)
        if b is None or b.numel() < need:
            b = torch.empty(max(self.cap, need), dtype=torch.uint8, device=self.dev)
            table[key] = b
        return b

    def step(self, t: int, stream=None) -> int:
        """Replicate step t of every local node through NCCL; returns payload-incl. bytes sent."""
        rt = self.rt
        s = torch.cuda.current_stream(self.dev) if stream is None else stream
        out_nodes = [n for n in rt.alive_local() if rt.succ.get(n) is not None]
        in_nodes = [m for m in sorted(rt.local) if m not in rt.dead]
        sizes = {}
        with torch.cuda.stream(s):
            for n in out_nodes:
                buf = self._buf(self.send_bufs, n, K.kv_pack_bytes(rt.handle(n)))
                sizes[n] = K.kv_pack_step(rt.handle(n), t, buf, buf.numel(), s.cuda_stream)
            # links whose successor lives on this GPU never leave it: unpack directly
            for n in out_nodes:
                m = rt.succ[n]
                if m in rt.local:
                    dst = rt.local[m]
                    K.kv_unpack(self.send_bufs[n], sizes[n], dst.replica, rt.NB, dst.meta, rt.kg,
                                rt.R, rt.M, s.cuda_stream)
            remote_out = sorted((n for n in out_nodes if rt.succ[n] not in rt.local),
                                key=lambda n: rt.succ[n])
            preds = {m: [n for n in rt.placement if rt.succ.get(n) == m and n not in rt.dead
                         and n not in rt.local] for m in in_nodes}
            remote_in = [m for m in in_nodes if preds[m]]
            if rt.world == 1 or (not remote_out and not remote_in):
                return sum(sizes.values())
            # count exchange (8 B per remote link), then the payloads, grouped by peer
            ops, cnt_out, cnt_in = [], {}, {}
            for n in remote_out:
                m = rt.succ[n]
                cnt_out[n] = torch.tensor([sizes[n]], dtype=torch.int64, device=self.dev)
                ops.append(dist.P2POp(dist.isend, cnt_out[n], rt.placement[m]))
            for m in remote_in:
                (n,) = preds[m]
                cnt_in[m] = torch.empty(1, dtype=torch.int64, device=self.dev)
                ops.append(dist.P2POp(dist.irecv, cnt_in[m], rt.placement[n]))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            counts = {m: int(cnt_in[m].item()) for m in remote_in}   # host sync: the round trip
            ops = []
            for n in remote_out:
                m = rt.succ[n]
                ops.append(dist.P2POp(dist.isend, self.send_bufs[n][:sizes[n]], rt.placement[m]))
            for m in remote_in:
                (n,) = preds[m]
                rb = self._buf(self.recv_bufs, m, counts[m])
                ops.append(dist.P2POp(dist.irecv, rb[:counts[m]], rt.placement[n]))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for m in remote_in:
                dst = rt.local[m]
                K.kv_unpack(self.recv_bufs[m], counts[m], dst.replica, rt.NB, dst.meta, rt.kg,
                            rt.R, rt.M, s.cuda_stream)
        return sum(sizes.values())
