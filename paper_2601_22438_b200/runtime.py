"""Ring runtime: device memory, pool handles and ring links for the logical
nodes one process (one GPU) hosts, plus the per-step driver that feeds them a
request schedule.  PyTorch is used only for device memory, streams and the
process group / symmetric-memory rendezvous that yields NVLink peer pointers;
every byte of KV is moved by libkvring's kernels.

Harness protocol (identical to the oracle's):
for each step t, for each serving node: begin_step, release the retiring
requests of every pipeline it serves, ONE append (decodes of all its requests
in ascending req_id, then admissions in pipeline order, FCFS); on a failure
at t: fail(f) after the appends, unlink pred(f), restore into a fresh pool or
promote into the holder (R10), re-append what the replica lacks,
relink; if t >= 1 every alive linked node replicates with seq = t.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kvring as K

SENTINEL_WORD = 0x5A5A


class StreamOrder:
    """Cross-stream order of a hand-written two-stream decode loop, the same rule
    kv_run_steps applies natively: the publication of step k after append k, and
    append k after the publication of step k-2 (blocks a retiring request frees
    are reused one step later, reading R7, and must not be overwritten while a
    lagging publication still reads them)."""

    def __init__(self, comp, repl):
        self.comp, self.repl = comp, repl
        self.done: list = []

    def before_append(self) -> None:
        if len(self.done) >= 2:
            self.comp.wait_event(self.done[-2])

    def before_publish(self) -> None:
        ev = torch.cuda.Event()
        ev.record(self.comp)
        self.repl.wait_event(ev)

    def after_publish(self) -> None:
        ev = torch.cuda.Event()
        ev.record(self.repl)
        self.done = self.done[-1:] + [ev]


def _meta_stride(R: int, M: int) -> int:
    return (K.kv_meta_bytes(R, M) + 4095) // 4096 * 4096


@dataclass
class NodeSlot:
    """Memory of one logical node slot on this rank."""
    index: int                     # slot index inside this rank's arena
    pool: torch.Tensor             # int16 [NB][L][2][H][B][d]
    replica: torch.Tensor          # int16 view into the arena
    meta: torch.Tensor             # uint8 view into the arena
    handle: int | None = None
    node: int | None = None        # logical node id bound to this slot


class RingRuntime:
    """Pools of the logical nodes placed on this rank, linked into a ring.

    ``placement[node] -> rank``; ``succ[node] -> node``.  ``spares`` extra
    slots per rank host fresh pools created by restores.  With world > 1 the
    replica regions and metadata live in one symmetric-memory arena per rank,
    so a successor on another GPU is addressed through NVLink peer pointers.
    """

    def __init__(self, geom, num_blocks: int, max_reqs: int, max_blocks_per_req: int,
                 placement: dict[int, int], succ: dict[int, int], rank: int = 0, world: int = 1,
                 device: int | None = None, spares: int = 1, group=None,
                 sentinel: int | None = SENTINEL_WORD, dtype_words=torch.int16,
                 mode: int = K.KV_MODE_TOKENS, shared: bool = False):
        self.g = geom
        # shared capacity (NEXT-3): the successor keeps the replica in its own pool
        # (kv_set_successor_shared); the replica regions stay unused.  A successor on
        # another rank PULLS: its rank keeps a mirror of the predecessor (tables only,
        # pool = the predecessor's pool through NVLink, kv_pool_set_mirror) linked to
        # the local holder -- the holder's allocator decides the replica blocks
        self.shared = shared
        self.mirrors: dict[int, tuple[int, torch.Tensor]] = {}
        self.NB, self.R, self.M = num_blocks, max_reqs, max_blocks_per_req
        self.placement = dict(placement)
        self.succ = dict(succ)
        self.rank, self.world = rank, world
        self.mode = mode
        self.copy_engine = False   # replicate_all through kv_replicate_step_ce (NEXT-4)
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        self.kg = K.geom(geom.layers, geom.kv_heads, geom.head_dim, geom.block_size, geom.elem_bytes)
        self.block_bytes = K.kv_block_bytes(self.kg)
        self.block_words = self.block_bytes // 2
        self.shape = (num_blocks, geom.layers, 2, geom.kv_heads, geom.block_size, geom.head_dim)
        per_rank = {}
        for n, r in placement.items():
            per_rank[r] = per_rank.get(r, 0) + 1
        self.n_slots = max(per_rank.values()) + spares
        self.replica_bytes = num_blocks * self.block_bytes
        self.meta_stride = _meta_stride(max_reqs, max_blocks_per_req)
        self.slot_stride = self.replica_bytes + self.meta_stride
        arena_bytes = self.n_slots * self.slot_stride
        self.group = group
        if world > 1:
            import torch.distributed._symmetric_memory as symm_mem
            self.arena = symm_mem.empty(arena_bytes, dtype=torch.uint8, device=self.dev)
            gname = group.group_name if group is not None else torch.distributed.group.WORLD.group_name
            self.symm = symm_mem.rendezvous(self.arena, gname)
            self.peer_base = [int(p) for p in self.symm.buffer_ptrs]
        else:
            self.arena = torch.empty(arena_bytes, dtype=torch.uint8, device=self.dev)
            self.symm = None
            self.peer_base = [self.arena.data_ptr()]
        self.pool_bytes = num_blocks * self.block_bytes
        self.pool_peer_base = None
        if world > 1 and shared:   # pools in symmetric memory: a remote holder pulls from them
            import torch.distributed._symmetric_memory as symm_mem
            self.pool_arena = symm_mem.empty(self.n_slots * self.pool_bytes, dtype=torch.uint8,
                                             device=self.dev)
            self.pool_symm = symm_mem.rendezvous(self.pool_arena, gname)
            self.pool_peer_base = [int(p) for p in self.pool_symm.buffer_ptrs]
        self.slots: list[NodeSlot] = []
        for k in range(self.n_slots):
            base = k * self.slot_stride
            rep = self.arena[base: base + self.replica_bytes].view(dtype_words).view(self.shape)
            meta = self.arena[base + self.replica_bytes: base + self.slot_stride]
            if self.pool_peer_base is not None:
                pool = self.pool_arena[k * self.pool_bytes:(k + 1) * self.pool_bytes] \
                    .view(dtype_words).view(self.shape)
            else:
                pool = torch.empty(self.shape, dtype=dtype_words, device=self.dev)
            if sentinel is not None:
                w = sentinel if sentinel < 0x8000 else sentinel - 0x10000
                pool.fill_(w)
                rep.fill_(w)
            self.slots.append(NodeSlot(k, pool, rep, meta))
        self.local: dict[int, NodeSlot] = {}
        self.slot_of_node: dict[int, tuple[int, int]] = {}   # node -> (rank, slot index)
        # deterministic slot assignment on every rank: ascending node id
        counters = {r: 0 for r in range(world)}
        for n in sorted(placement):
            r = placement[n]
            self.slot_of_node[n] = (r, counters[r])
            counters[r] += 1
        self.next_spare = {r: counters[r] for r in range(world)}
        self.dead: set[int] = set()
        torch.cuda.synchronize(self.dev)
        if world > 1:
            torch.distributed.barrier(group=group)
        for n in sorted(placement):
            if placement[n] == rank:
                self._create(n, self.slots[self.slot_of_node[n][1]])
        if self.pool_peer_base is not None:
            # a mirror of EVERY remote node (every rank receives every owner's block ids),
            # so a link re-formed after a failure finds its mirror up to date
            for n in sorted(placement):
                if placement[n] != rank:
                    self._create_mirror(n)
        for n in sorted(self.local):
            self._link(n)
        for n in sorted(self.mirrors):
            self._link_mirror(n)

    # ----------------------------------------------------------------- memory
    def _create(self, node: int, slot: NodeSlot) -> int:
        d = K.kv_pool_desc_t(self.kg, self.NB, self.R, self.M, self.device, node, self.NB,
                             slot.pool.data_ptr(), slot.replica.data_ptr(), slot.meta.data_ptr())
        slot.handle = K.kv_pool_create(d)
        if self.mode != K.KV_MODE_TOKENS:
            K.kv_set_mode(slot.handle, self.mode)
        slot.node = node
        self.local[node] = slot
        return slot.handle

    def pool_ptr(self, node: int) -> int:
        r, k = self.slot_of_node[node]
        return self.pool_peer_base[r] + k * self.pool_bytes

    def _create_mirror(self, node: int) -> None:
        """Tables-only mirror of remote ``node`` on this rank's device, its pool pointer
        the node's pool through NVLink (NEXT-3 across GPUs)."""
        scratch = torch.zeros(self.block_bytes + self.meta_stride, dtype=torch.uint8,
                              device=self.dev)
        d = K.kv_pool_desc_t(self.kg, self.NB, self.R, self.M, self.device, node, 1,
                             self.pool_ptr(node), scratch.data_ptr(),
                             scratch.data_ptr() + self.block_bytes)
        h = K.kv_pool_create(d)
        K.kv_pool_set_mirror(h, True)
        self.mirrors[node] = (h, scratch)

    def replica_ptr(self, node: int) -> int:
        r, k = self.slot_of_node[node]
        return self.peer_base[r] + k * self.slot_stride

    def meta_ptr(self, node: int) -> int:
        return self.replica_ptr(node) + self.replica_bytes

    def _link(self, node: int) -> None:
        m = self.succ.get(node)
        h = self.local[node].handle
        if m is None or m in self.dead:
            K.kv_set_successor(h, -1, None, 0, None)
        elif self.shared:
            if m not in self.local:
                if self.pool_peer_base is None or self.placement.get(m) is None:
                    raise RuntimeError("shared-capacity links need the successor on this rank")
                # the holder's rank pulls through its mirror of this node: no link here
                K.kv_set_successor(h, -1, None, 0, None)
            else:
                K.kv_set_successor_shared(h, self.local[m].handle)
        else:
            K.kv_set_successor(h, m, self.replica_ptr(m), self.NB, self.meta_ptr(m))

    def _link_mirror(self, node: int) -> None:
        """A mirror replicates into a holder on this rank; otherwise it is unlinked."""
        h = self.mirrors[node][0]
        m = self.succ.get(node)
        if node in self.dead:
            return
        if m is not None and m in self.local and m not in self.dead:
            K.kv_set_successor_shared(h, self.local[m].handle)
        else:
            K.kv_set_successor(h, -1, None, 0, None)

    def handle(self, node: int) -> int:
        return self.local[node].handle

    def alive_local(self) -> list[int]:
        return [n for n in sorted(self.local) if n not in self.dead]

    # ------------------------------------------------------------------ steps
    def append_all(self, entries: list[dict], stream=None) -> None:
        """entries: per local node dict(node, begin_step, release, req_ids, n_new, src)."""
        if not entries:
            return
        s = self._stream(stream)
        K.kv_append_multi([dict(e, pool=self.mirrors[e["node"]][0] if e["node"] in self.mirrors
                                else self.handle(e["node"])) for e in entries], s)

    def replicate_all(self, step: int, nodes: list[int] | None = None, stream=None) -> None:
        def linked_here(n):   # shared links to a remote holder are pulled by its rank
            m = self.succ.get(n)
            return m is not None and (not self.shared or m in self.local)
        nodes = [n for n in (self.alive_local() if nodes is None else nodes) if linked_here(n)]
        hs = [self.handle(n) for n in nodes]
        # mirrors of remote predecessors: the local holder pulls their dirty slices
        hs += [h for n, (h, _) in sorted(self.mirrors.items())
               if n not in self.dead and self.succ.get(n) in self.local]
        if hs:
            fn = K.kv_replicate_step_ce if self.copy_engine else K.kv_replicate_step_multi
            fn(hs, step, self._stream(stream))

    def _stream(self, stream) -> int:
        if stream is None:
            return torch.cuda.current_stream(self.dev).cuda_stream
        return stream if isinstance(stream, int) else stream.cuda_stream

    # ------------------------------------------------------ failure / restore
    def fail(self, node: int, stream=None) -> None:
        """Simulated failure of ``node``; every rank calls it (owner poisons, others unlink)."""
        self.dead.add(node)
        if node in self.local:
            K.kv_fail_stage(self.handle(node), self._stream(stream))
        if node in self.mirrors:   # marks the mirror dead (its owner poisons the memory)
            K.kv_fail_stage(self.mirrors[node][0], self._stream(stream))
        for n, m in list(self.succ.items()):
            if m == node:
                self.succ[n] = None
                if n in self.local and n not in self.dead:
                    self._link(n)
                if n in self.mirrors:
                    self._link_mirror(n)

    def new_node(self, node: int, rank: int) -> None:
        """Bind a spare slot on ``rank`` to a fresh logical node id (every rank calls it)."""
        k = self.next_spare[rank]
        if k >= self.n_slots:
            raise RuntimeError("no spare slot left for a fresh pool")
        self.next_spare[rank] = k + 1
        self.placement[node] = rank
        self.slot_of_node[node] = (rank, k)
        if rank == self.rank:
            self._create(node, self.slots[k])

    def restore(self, dst: int, holder: int, stream=None):
        """kv_restore into local pool ``dst`` from ``holder``'s replica (local or peer).
        Shared capacity: the replica is read from the holder's own pool, whose
        replica blocks are then freed (kv_drop_replicas)."""
        if self.shared:
            out = K.kv_restore(self.handle(dst), self.local[holder].pool.data_ptr(), self.NB,
                               self.meta_ptr(holder), self._stream(stream))
            K.kv_drop_replicas(self.handle(holder))
            return out
        return K.kv_restore(self.handle(dst), self.replica_ptr(holder), self.NB,
                            self.meta_ptr(holder), self._stream(stream))

    def set_succ(self, node: int, succ: int | None) -> None:
        self.succ[node] = succ
        if node in self.local and node not in self.dead:
            self._link(node)
        if node in self.mirrors:
            self._link_mirror(node)

    # ---------------------------------------------------------------- readout
    def read_meta(self, node: int) -> dict:
        """Decode the replica metadata of local node ``node`` (layout: include/kvring.h)."""
        raw = self.local[node].meta.cpu().numpy()
        R, M = self.R, self.M
        seq = int(raw[0:8].view(np.uint64)[0])
        hdr = raw[8:24].view(np.int32)
        req = raw[32:32 + 16 * R].view(np.int64).reshape(2, R)
        ln = raw[32 + 16 * R:32 + 24 * R].view(np.int32).reshape(2, R)
        bt = raw[32 + 24 * R:32 + 24 * R + 4 * R * M].view(np.int32).reshape(R, M)
        return {"seq": seq, "writer": int(hdr[0]), "R": int(hdr[1]), "M": int(hdr[2]),
                "magic": int(hdr[3]), "req": req, "len": ln, "bt": bt}

    def destroy(self) -> None:
        torch.cuda.synchronize(self.dev)
        for s in self.slots:
            if s.handle is not None:
                K.kv_pool_destroy(s.handle)
                s.handle = None
        for n, (h, _) in list(self.mirrors.items()):
            K.kv_pool_destroy(h)
        self.mirrors.clear()


@dataclass
class DriverEvent:
    kind: str
    step: int
    data: dict = field(default_factory=dict)


class ScheduleDriver:
    """Feeds per-pipeline schedules (kvgen) through a RingRuntime, step by step.

    ``coords`` maps logical (pipeline, stage) -> node id.  ``content(stage,
    ids, positions)`` returns the dense device source for the given tokens
    (the caller decides how it is generated: kvgen's CUDA twin in tests and
    bench).  Only nodes local to this rank are stepped.
    """

    def __init__(self, rt: RingRuntime, schedules, coords: dict[tuple[int, int], int], content,
                 restore_mode: str = "fresh"):
        self.rt = rt
        self.sched = schedules
        self.coords = dict(coords)
        self.serving = dict(coords)            # (p, s) -> node currently serving it
        self.content = content
        self.restore_mode = restore_mode
        self.events: list[DriverEvent] = []
        self.next_node = max(rt.placement) + 1
        self.orig_succ = dict(rt.succ)          # ring map over the original nodes

    def stage_of_node(self, node: int) -> int:
        for (p, s), n in self.serving.items():
            if n == node:
                return s
        raise KeyError(node)

    def plan(self, t: int) -> dict[int, dict]:
        """Per serving node: release ids, append ids, n_new and token positions."""
        groups: dict[int, list[tuple[int, int]]] = {}
        for key in sorted(self.serving):
            groups.setdefault(self.serving[key], []).append(key)
        out = {}
        for node, keys in groups.items():
            if node in self.rt.dead:
                continue
            rel, dec, adm = [], [], []
            for (p, s) in keys:
                ev = self.sched[p].steps[t]
                rel.extend(ev.retire)
                dec.extend((r, p) for r in ev.decode)
                adm.extend((r, pp) for r, pp in ev.admit)
            dec.sort()
            ids = [r for r, _ in dec] + [r for r, _ in adm]
            n_new = [1] * len(dec) + [pp for _, pp in adm]
            pos = [self.sched[p].length_at(r, t - 1) for r, p in dec] + [0] * len(adm)
            out[node] = dict(stage=keys[0][1], release=rel, req_ids=ids, n_new=n_new, start=pos)
        return out

    def tokens(self, req_ids, n_new, start):
        ids, pos = [], []
        for r, n, p0 in zip(req_ids, n_new, start):
            ids.extend([r] * n)
            pos.extend(range(p0, p0 + n))
        return ids, pos

    def append_step(self, t: int, stream=None, sources: dict | None = None,
                    plan: dict | None = None) -> None:
        if getattr(self.rt, "pool_peer_base", None) is not None:
            return self._append_step_pulled(t, stream, sources, plan)
        entries = []
        for node, e in (self.plan(t) if plan is None else plan).items():
            if node not in self.rt.local:
                continue
            if sources is not None and node in sources:
                src = sources[node]
            else:
                ids, pos = self.tokens(e["req_ids"], e["n_new"], e["start"])
                src = self.content(e["stage"], ids, pos) if ids else None
            entries.append(dict(node=node, begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        self.rt.append_all(entries, stream)
        self._keep = entries   # sources must outlive the async kernel launch

    def _append_step_pulled(self, t, stream, sources, plan):
        """Shared capacity across ranks (NEXT-3): nodes append in serving order, each
        owner forwards the block ids its append allocated and a holder's rank applies the
        same append to its mirror with those ids -- a holder's own append (which may
        evict its predecessor's replicas) then sees the predecessor's tables of this step
        exactly as in the one-process protocol."""
        import torch.distributed as dist
        rt = self.rt
        keep = []
        for node, e in (self.plan(t) if plan is None else plan).items():
            allocs = None
            if node in rt.local:
                if sources is not None and node in sources:
                    src = sources[node]
                else:
                    ids, pos = self.tokens(e["req_ids"], e["n_new"], e["start"])
                    src = self.content(e["stage"], ids, pos) if ids else None
                keep.append(src)
                rt.append_all([dict(node=node, begin_step=1, release=e["release"],
                                    req_ids=e["req_ids"], n_new=e["n_new"], src=src)], stream)
                allocs = K.kv_last_alloc(rt.handle(node))
            obj = [allocs]
            dist.broadcast_object_list(obj, src=rt.placement[node], group=rt.group)
            if node in rt.mirrors:
                K.kv_mirror_blocks(rt.mirrors[node][0], obj[0])
                rt.append_all([dict(node=node, begin_step=1, release=e["release"],
                                    req_ids=e["req_ids"], n_new=e["n_new"], src=None)], stream)
        self._keep = keep

    def fail_and_restore(self, t: int, coord: tuple[int, int], stream=None):
        """Fail the node serving ``coord`` after the appends of step t and restore it."""
        rt = self.rt
        f = self.serving[coord]
        holder = rt.succ[f]
        rt.fail(f, stream)
        if self.restore_mode == "fresh":
            dst = self.next_node
            self.next_node += 1
            rt.new_node(dst, rt.placement[holder])
        else:
            dst = holder
        result = None
        if dst in rt.local:
            result = rt.restore(dst, holder, stream)
        keys = [k for k, n in self.serving.items() if n == f]
        for k in keys:
            self.serving[k] = dst
        if dst in rt.local:
            t_star, restored = result
            got = dict(restored)
            ext, adm = [], []
            for (p, s) in keys:
                sch = self.sched[p]
                for r in sorted(sch.requests):
                    cur = sch.length_at(r, t)
                    if cur == 0 or sch.admitted_at[r] + sch.requests[r].output + 1 <= t:
                        continue
                    if r in got:
                        if cur > got[r]:
                            ext.append((r, cur - got[r], got[r]))
                    else:
                        adm.append((r, cur, 0))
            todo = ext + adm
            if todo:
                ids = [x[0] for x in todo]
                n_new = [x[1] for x in todo]
                start = [x[2] for x in todo]
                tid, tpos = self.tokens(ids, n_new, start)
                src = self.content(coord[1], tid, tpos)
                rt.append_all([dict(node=dst, begin_step=0, release=[], req_ids=ids,
                                    n_new=n_new, src=src)], stream)
                self._keep_restore = src
            self.events.append(DriverEvent("restore", t, dict(coord=coord, t_star=t_star,
                                                              restored=restored, dst=dst,
                                                              resume=todo)))
        if self.restore_mode == "fresh":
            for n, m in self.orig_succ.items():
                if m == f and n != f and n not in rt.dead:
                    rt.set_succ(n, dst)
            rt.set_succ(dst, holder)
        return dst, result

    def reprotect(self, excluded_coords) -> dict:
        """Re-protection after a failure (§8(f) NEXT-1): walk the ORIGINAL ring
        over logical coordinates skipping excluded ones (failed nodes and nodes under
        traffic rerouting) with kv_plan_targets; rebind (re-seed) every link whose
        target node changed; excluded nodes stop replicating.  Returns {coord: coord}."""
        coords = sorted(self.coords)
        idx = {c: k for k, c in enumerate(coords)}
        node_coord = {n: c for c, n in self.coords.items()}
        succ = [idx[node_coord[self.orig_succ[self.coords[c]]]] for c in coords]
        excl = [idx[c] for c in excluded_coords]
        tgt = K.kv_plan_targets(succ, excl)
        plan = {}
        for c in coords:
            n = self.serving[c]
            if n in self.rt.dead:
                continue
            t = tgt[idx[c]]
            want = None if t < 0 else self.serving[coords[t]]
            plan[c] = None if t < 0 else coords[t]
            if self.rt.succ.get(n) != want:
                self.rt.set_succ(n, want)
        return plan

    def run(self, n_steps: int, fail_step: int | None = None, fail_coord=None, on_step=None,
            stream=None):
        for t in range(n_steps):
            self.append_step(t, stream)
            if fail_step is not None and t == fail_step:
                self.fail_and_restore(t, fail_coord, stream)
            if t >= 1:
                self.rt.replicate_all(t, stream=stream)
            if on_step is not None:
                on_step(self, t)
        return self


class TablesRuntime:
    """RingRuntime's interface over tables-only pools (kv_pool_desc_t.device = -1):
    the C++ allocator, quarantine and work-list builder run, nothing is launched
    and no KV byte moves.  Used by the CPU tests of the multi-rank host logic."""

    FAKE = 0x1000

    def __init__(self, geom, num_blocks, max_reqs, max_blocks_per_req, placement, succ,
                 rank=0, world=1):
        self.g = geom
        self.NB, self.R, self.M = num_blocks, max_reqs, max_blocks_per_req
        self.placement, self.succ = dict(placement), dict(succ)
        self.rank, self.world = rank, world
        self.kg = K.geom(geom.layers, geom.kv_heads, geom.head_dim, geom.block_size,
                         geom.elem_bytes)
        self.dead: set[int] = set()
        self.mirrors: dict = {}   # no cross-rank shared links in tables-only runs
        self.handles: dict[int, int] = {}
        self.local = self.handles
        for n in sorted(placement):
            if placement[n] == rank:
                self._create(n)
        for n in sorted(self.handles):
            self._link(n)

    def _create(self, node):
        d = K.kv_pool_desc_t(self.kg, self.NB, self.R, self.M, -1, node, self.NB, None, None, None)
        self.handles[node] = K.kv_pool_create(d)

    def _link(self, node):
        m = self.succ.get(node)
        if m is None or m in self.dead:
            K.kv_set_successor(self.handles[node], -1, None, 0, None)
        else:
            K.kv_set_successor(self.handles[node], m, self.FAKE + m, self.NB, self.FAKE + m)

    def handle(self, node):
        return self.handles[node]

    def alive_local(self):
        return [n for n in sorted(self.handles) if n not in self.dead]

    def append_all(self, entries, stream=None):
        if entries:
            K.kv_append_multi([dict(e, pool=self.handle(e["node"]), src=None) for e in entries])

    def replicate_all(self, step, nodes=None, stream=None):
        nodes = [n for n in (self.alive_local() if nodes is None else nodes)
                 if self.succ.get(n) is not None]
        if nodes:
            K.kv_replicate_step_multi([self.handle(n) for n in nodes], step)

    def fail(self, node, stream=None):
        self.dead.add(node)
        if node in self.handles:
            K.kv_fail_stage(self.handles[node])
        for n, m in list(self.succ.items()):
            if m == node:
                self.succ[n] = None
                if n in self.handles and n not in self.dead:
                    self._link(n)

    def set_succ(self, node, succ):
        self.succ[node] = succ
        if node in self.handles and node not in self.dead:
            self._link(node)

    def destroy(self):
        for h in self.handles.values():
            K.kv_pool_destroy(h)
        self.handles.clear()
