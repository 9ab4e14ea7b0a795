"""Shared helpers for the GPU parity tests: run the CUDA path (RingRuntime +
ScheduleDriver over libkvring) and the CPU oracle on the same seeded inputs
and compare them.  Test infrastructure: imports both sides, which never import
each other."""
from __future__ import annotations

import numpy as np
import torch

from kvgen.content import CONTENT_SEED
from kvgen.cuda import content_tokens_cuda
from oracle.ring import instance_ring, stage_ring
from oracle.simulate import OracleRing


def make_gpu(cfg, ring="stage", device=0, spares=1, schedules=None, restore_mode=None,
             mode="tokens", shared=False):
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    from kvgen.configs import build_schedules
    I, S = cfg.pipelines, cfg.stages
    coords = {(i, s): i * S + s for i in range(I) for s in range(S)}
    fn = instance_ring if ring == "instance" else stage_ring
    succ = {coords[c]: coords[fn(c, I, S)] for c in coords}
    placement = {n: 0 for n in coords.values()}
    torch.cuda.set_device(device)
    from paper_2601_22438_b200 import kvring as K
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=0, world=1, device=device, spares=spares,
                     mode=K.KV_MODE_BLOCKS if mode == "blocks" else K.KV_MODE_TOKENS,
                     shared=shared)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=device)

    sched = schedules if schedules is not None else build_schedules(cfg)
    mode = restore_mode or ("promote" if ring == "instance" else "fresh")
    drv = ScheduleDriver(rt, sched, coords, content, restore_mode=mode)
    return rt, drv


def node_map(rt, drv, oring: OracleRing) -> dict:
    """GPU node id -> oracle node (original coords, then fresh restore pools in order)."""
    m = {drv.coords[c]: oring.nodes[c] for c in oring.coords}
    extra = sorted(n for n in rt.local if n not in m)
    for n, o in zip(extra, oring.extra_nodes):
        m[n] = o
    return m


def compare_state(rt, drv, oring: OracleRing, content: bool = True, tag="", only=None) -> None:
    """Byte-for-byte comparison of every local node (or the node ids in ``only``)."""
    torch.cuda.synchronize()
    from paper_2601_22438_b200 import kvring as K
    for gid, on in node_map(rt, drv, oring).items():
        if gid not in rt.local or (only is not None and gid not in only):
            continue
        slot = rt.local[gid]
        if content:
            prim = slot.pool.cpu().numpy().view(np.uint16)
            rep = slot.replica.cpu().numpy().view(np.uint16)
            if not np.array_equal(prim, on.primary):
                bad = np.argwhere(prim != on.primary)[:5]
                raise AssertionError(f"{tag} node {gid}: primary differs at {bad.tolist()}")
            if not np.array_equal(rep, on.replica):
                bad = np.argwhere(rep != on.replica)[:5]
                raise AssertionError(f"{tag} node {gid}: replica differs at {bad.tolist()}")
        meta = rt.read_meta(gid)
        assert meta["seq"] == on.rseq, (tag, gid, meta["seq"], on.rseq)
        assert np.array_equal(meta["req"], on.rreq), (tag, gid)
        assert np.array_equal(meta["len"], on.rlen), (tag, gid)
        assert np.array_equal(meta["bt"], on.rbt), (tag, gid)
        if not on.dead:
            req, ln, pub, nb = K.kv_dump_slots(rt.handle(gid), rt.R)
            live = {}
            for s in range(rt.R):
                if req[s] >= 0:
                    live[int(req[s])] = (s, int(ln[s]), K.kv_query(rt.handle(gid), int(req[s]))[1])
            assert live == on.live(), (tag, gid)
            # a shared link to a holder on another rank is driven by that rank's mirror
            # of this node: the publication state (pub_len, drops) lives there
            pulled = getattr(rt, "shared", False) and \
                rt.succ.get(gid) is not None and rt.succ[gid] not in rt.local
            if not pulled:
                assert np.array_equal(pub, on.pub_len), (tag, gid)
            st = K.kv_stats(rt.handle(gid))
            assert st["free_blocks"] == len(on.free_blocks), (tag, gid)
            assert st["quarantined_blocks"] == len(on.q_blocks), (tag, gid)
            # shared capacity (NEXT-3): evictions, drops and the held-replica census
            assert st["replica_evictions"] == on.evictions, (tag, gid)
            if not pulled:
                assert st["replica_drops"] == on.drops, (tag, gid)
            held = on.rep_src.census() if on.rep_src is not None else 0
            assert st["replica_blocks_held"] == held, (tag, gid, st["replica_blocks_held"], held)


def compare_mirrors(rt, drv, oring: OracleRing, tag="") -> int:
    """NEXT-3 across GPUs: every live mirror on this rank (a remote predecessor whose
    replica this rank's holder pulls) has the owner's tables, and the publication state
    of the link (pub_len, drops) == the oracle's node.  Returns the mirrors checked."""
    from paper_2601_22438_b200 import kvring as K
    m = {drv.coords[c]: oring.nodes[c] for c in oring.coords}
    n = 0
    for gid, (h, _) in sorted(getattr(rt, "mirrors", {}).items()):
        if gid in rt.dead or gid not in m or rt.succ.get(gid) not in rt.local:
            continue
        on = m[gid]
        req, ln, pub, nb = K.kv_dump_slots(h, rt.R)
        live = {}
        for s in range(rt.R):
            if req[s] >= 0:
                live[int(req[s])] = (s, int(ln[s]), K.kv_query(h, int(req[s]))[1])
        assert live == on.live(), (tag, "mirror tables", gid, live, on.live())
        assert np.array_equal(pub, on.pub_len), (tag, "mirror pub_len", gid, pub, on.pub_len)
        st = K.kv_stats(h)   # (its free list is not the owner's: the owner's ids are given)
        assert st["replica_drops"] == on.drops, (tag, "mirror drops", gid, st["replica_drops"],
                                                 on.drops)
        n += 1
    return n
