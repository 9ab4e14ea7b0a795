"""Oracle ring driver and invariant checks.  TEST INFRASTRUCTURE ONLY.

Drives every logical node of a config through the step protocol of SURVEY
§8(c) (steps 1-7):

for each step t:
  per serving node, in serving order (by the first logical coordinate it
  serves): begin_step; release the retiring requests
  of every pipeline it serves; ONE append with the decodes of all its
  requests in ascending req_id, then the admissions (pipeline order, FCFS);
  [failure at t: fail(f) after the appends, unlink pred(f), then restore:
   "fresh" -> a new pool replaces f, "promote" -> the holder succ(f) takes f's
   requests (reading R10); re-append positions [resume_len, len_t) and
   re-admit requests absent from the replica; relink the ring (re-seed)]
  if t >= 1: every alive, linked node replicates with seq = t (node order).

Checks are plain functions over the nodes.
"""
from __future__ import annotations

import numpy as np

from kvgen.configs import Config, build_schedules
from kvgen.content import CONTENT_SEED, SENTINEL_WORD, content_tokens, content_segment_table
from .kvring_oracle import OracleNode, ceil_div
from .ring import instance_ring, stage_ring


class OracleRing:
    def __init__(self, cfg: Config, content: bool = True, ring: str | None = None,
                 restore_mode: str | None = None, seed: int = CONTENT_SEED,
                 schedules=None, mode: str = "tokens", shared: bool = False):
        self.cfg = cfg
        self.g = cfg.geom
        self.seed = seed
        self.content = content
        ring = ring or cfg.ring
        self.ring_fn = instance_ring if ring == "instance" else stage_ring
        self.restore_mode = restore_mode or ("promote" if ring == "instance" else "fresh")
        I, S = cfg.pipelines, cfg.stages
        self.coords = [(i, s) for i in range(I) for s in range(S)]
        self.nodes = {c: OracleNode(self.g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                                    node_id=k, content=content)
                      for k, c in enumerate(self.coords)}
        self.mode = mode
        self.shared = shared      # NEXT-3: replicas inside the holder's own pool (R17)
        for c in self.coords:
            self.nodes[c].set_mode(mode)
            self.nodes[c].set_successor(self.nodes[self.ring_fn(c, I, S)], shared=shared)
        self.serving = dict(self.nodes)         # logical (pipeline, stage) -> node serving it
        self.extra_nodes: list[OracleNode] = []
        self.sched = schedules if schedules is not None else build_schedules(cfg)
        self.tables = {s: content_segment_table(seed, s * self.g.layers, self.g.layers,
                                                self.g.kv_heads, self.g.head_dim)
                       for s in range(S)}
        self.moved = 0
        self.events: list[tuple] = []

    # ----------------------------------------------------------------- helpers
    def stage_of(self, node: OracleNode) -> int:
        for (p, s), n in self.serving.items():
            if n is node:
                return s
        raise KeyError("node serves nothing")

    def src_for(self, stage: int, req_ids, n_new, start_lens) -> np.ndarray | None:
        if not self.content:
            return None
        ids, pos = [], []
        for r, n, l0 in zip(req_ids, n_new, start_lens):
            ids.extend([r] * n)
            pos.extend(range(l0, l0 + n))
        g = self.g
        return content_tokens(self.seed, ids, pos, stage * g.layers, g.layers, g.kv_heads,
                              g.head_dim, table=self.tables[stage])

    def all_nodes(self) -> list[OracleNode]:
        return [self.nodes[c] for c in self.coords] + self.extra_nodes

    def served_by(self) -> dict[int, list[tuple[int, int]]]:
        out: dict[int, list[tuple[int, int]]] = {}
        for key, n in sorted(self.serving.items()):
            out.setdefault(id(n), []).append(key)
        return out

    # -------------------------------------------------------------------- step
    def appends(self, t: int):
        """Per serving node: begin_step, releases, one append (harness protocol)."""
        groups = self.served_by()
        # serving order: by the first logical coordinate a node serves (a fresh
        # restore pool takes the failed node's place); the order matters only
        # between a shared-capacity holder and its predecessor (NEXT-3)
        order = []
        for key in sorted(self.serving):
            n = self.serving[key]
            if all(n is not m for m in order):
                order.append(n)
        for node in order:
            if node.dead or id(node) not in groups:
                continue
            keys = groups[id(node)]
            node.begin_step()
            for (p, s) in keys:
                node.release(self.sched[p].steps[t].retire)
            dec, adm = [], []
            for (p, s) in keys:
                ev = self.sched[p].steps[t]
                dec.extend(ev.decode)
                adm.extend(ev.admit)
            ids = sorted(dec) + [r for r, _ in adm]
            n_new = [1] * len(dec) + [pp for _, pp in adm]
            live = node.live()
            starts = [live[r][1] if r in live else 0 for r in ids]
            stage = keys[0][1]
            node.append(ids, n_new, self.src_for(stage, ids, n_new, starts))

    def replicate(self, t: int) -> None:
        for node in self.all_nodes():
            if node.dead or node.succ is None:
                continue
            self.moved += node.replicate(t)

    def fail_and_restore(self, t: int, coord: tuple[int, int]):
        """Fail logical node ``coord`` after the appends of step t, then restore it."""
        I, S = self.cfg.pipelines, self.cfg.stages
        f = self.serving[coord]
        holder = f.succ
        f.fail()
        for n in self.all_nodes():
            if n is not f and not n.dead and n.succ is f:
                n.set_successor(None)
        if self.restore_mode == "fresh":
            dst = OracleNode(self.g, self.cfg.num_blocks, self.cfg.max_reqs,
                             self.cfg.max_blocks_per_req, node_id=len(self.coords) + len(self.extra_nodes),
                             content=self.content)
            dst.set_mode(self.mode)
            self.extra_nodes.append(dst)
        else:
            dst = holder
        t_star, restored = dst.restore_from(holder)
        if self.shared:
            holder.drop_replicas()    # the restore has read them; f is dead
        # resume: re-append what the replica lacks (<= 1 token per request, R3) and
        # re-admit requests absent from it (admitted in the unpublished step)
        keys = [k for k, n in self.serving.items() if n is f]
        for k in keys:
            self.serving[k] = dst
        stage = coord[1]
        got = dict(restored)
        ext_ids, ext_n, ext_start, adm_ids, adm_n = [], [], [], [], []
        for (p, s) in keys:
            sch = self.sched[p]
            for r in sorted(sch.requests):
                cur = sch.length_at(r, t)
                if cur == 0 or sch.admitted_at[r] + sch.requests[r].output + 1 <= t:
                    continue            # not live at step t
                if r in got:
                    if cur > got[r]:
                        ext_ids.append(r); ext_n.append(cur - got[r]); ext_start.append(got[r])
                else:
                    adm_ids.append(r); adm_n.append(cur)
        ids = ext_ids + adm_ids
        n_new = ext_n + adm_n
        starts = ext_start + [0] * len(adm_ids)
        if ids:
            dst.append(ids, n_new, self.src_for(stage, ids, n_new, starts))
        if self.restore_mode == "fresh":
            for n in self.all_nodes():
                if n is not dst and not n.dead and self.ring_fn_target(n) is f:
                    n.set_successor(dst, shared=self.shared)
            dst.set_successor(holder, shared=self.shared)
        self.events.append(("restore", t, coord, t_star, restored, ids, n_new))
        return t_star, restored, dst

    def reprotect(self, excluded_coords) -> dict:
        """P:227 §3.2 re-protection: targets from the ring walk skipping the excluded
        nodes (oracle/ring.py plan_replication_targets); a link is rebound (re-seeded)
        iff its target node changes; excluded nodes stop replicating."""
        from .ring import plan_replication_targets
        plan = plan_replication_targets(self.cfg.pipelines, self.cfg.stages, set(excluded_coords),
                                        ring=self.ring_fn)
        for c in self.coords:
            n = self.serving[c]
            if n.dead:
                continue
            t = plan.get(c)
            want = None if t is None else self.serving[t]
            if n.succ is not want:
                n.set_successor(want, shared=self.shared and want is not None)
        return plan

    def ring_fn_target(self, node: OracleNode):
        """The node ``node`` was originally linked to (ring map over logical coords)."""
        I, S = self.cfg.pipelines, self.cfg.stages
        for c, n in self.nodes.items():
            if n is node:
                return self.nodes[self.ring_fn(c, I, S)]
        return None

    def run(self, n_steps: int | None = None, check_every: int = 0, on_step=None):
        n_steps = self.cfg.n_steps if n_steps is None else n_steps
        for t in range(n_steps):
            self.appends(t)
            if self.cfg.fail_step is not None and t == self.cfg.fail_step:
                self.fail_and_restore(t, self.cfg.fail_node)
            if t >= 1:
                self.replicate(t)
            if on_step is not None:
                on_step(self, t)
            if check_every and t % check_every == 0:
                check_all(self)
        return self


def run_config(cfg: Config, **kw) -> OracleRing:
    return OracleRing(cfg, **kw).run()


# ------------------------------------------------------------------------ checks
def check_replica_equals_primary(n: OracleNode) -> None:
    """I1: succ(n)'s replica equals n's primary on every valid slot; metadata matches."""
    m = n.succ
    if m is None or n.dead or m.dead or n.last_step == 0:
        return
    B = n.g.block_size
    pub = m.published()
    live = n.live()
    assert m.rseq == n.last_step, (m.rseq, n.last_step)
    # published = the primary's tables cut at the published length of each slot
    # (all tokens, or completed blocks only in "blocks" mode)
    want = {}
    for r, (s, ln, bt) in live.items():
        hi = n.published_len(s)
        if hi > 0:
            want[r] = (s, hi, bt[:ceil_div(hi, B)])
    if n.holder is not None:
        # shared capacity (NEXT-3): the replica lives in the holder's pool at its own
        # block ids; dropped requests are absent
        want = {r: (s, hi, n.rep_bt[s][:ceil_div(hi, B)]) for r, (s, hi, _) in want.items()
                if not n.dropped[s]}
    assert pub == want, "published metadata != primary tables"
    if n.content:
        store = m.primary if n.holder is not None else m.replica
        for r, (s, ln, bt) in want.items():
            for j, blk in enumerate(bt):
                v = min(B, ln - j * B)
                src = n.slot_bt[s][j]
                assert np.array_equal(store[blk, :, :, :, :v], n.primary[src, :, :, :, :v]), (r, j)


def check_content(ring: OracleRing, node: OracleNode, stage: int, sample: int | None = None,
                  rng=None) -> None:
    """I2: every valid slot equals the closed-form content of (req, layer, kv, h, pos, dim)."""
    if not node.content or node.dead:
        return
    g = node.g
    B = g.block_size
    items = []
    for r, (s, ln, bt) in node.live().items():
        for pos in range(ln):
            items.append((r, pos, bt[pos // B]))
    if sample is not None and len(items) > sample:
        rng = rng or np.random.default_rng(0)
        items = [items[i] for i in rng.choice(len(items), sample, replace=False)]
    if not items:
        return
    exp = content_tokens(ring.seed, [i[0] for i in items], [i[1] for i in items],
                         stage * g.layers, g.layers, g.kv_heads, g.head_dim)
    for k, (r, pos, blk) in enumerate(items):
        assert np.array_equal(node.primary[blk, :, :, :, pos % B], exp[k]), (r, pos)


def check_tables(n: OracleNode) -> None:
    """I3: bt injective; free / quarantined / used partition [0, NB); nblk == ceil(len/B)."""
    if n.dead:
        return
    B = n.g.block_size
    used = [b for s in range(n.R) for b in n.slot_bt[s]]
    if n.rep_src is not None:      # shared capacity: the predecessor's replica blocks
        used += [b for s in range(n.rep_src.R) for b in n.rep_src.rep_bt[s]]
    assert len(used) == len(set(used)), "block used twice"
    parts = [set(used), set(n.free_blocks), set(n.q_blocks)]
    assert sum(len(p) for p in parts) == n.NB and set().union(*parts) == set(range(n.NB))
    for r, s in n.slot_of.items():
        assert len(n.slot_bt[s]) == ceil_div(int(n.slot_len[s]), B)
        assert n.slot_req[s] == r
    slots = [set(n.slot_of.values()), set(n.free_slots), set(n.q_slots)]
    assert sum(len(p) for p in slots) == n.R and set().union(*slots) == set(range(n.R))


def check_all(ring: OracleRing) -> None:
    for n in ring.all_nodes():
        check_tables(n)
        check_replica_equals_primary(n)
    for (p, s), n in ring.serving.items():
        check_content(ring, n, s, sample=256)


def full_copy_replay(cfg: Config, n_steps: int, **kw) -> dict:
    """I6 brute force: replicas rebuilt by copying ALL valid slots at every published step.

    Runs the oracle ring with replication disabled for content and, after each
    step t >= 1, copies every valid slot of each primary into its successor's
    brute-force replica (no pub_len bookkeeping).  ``brute`` is keyed by the
    HOLDER's coordinate (the node whose replica region it models).
    """
    ring = OracleRing(cfg, **kw)
    brute = {c: np.full_like(ring.nodes[c].replica, SENTINEL_WORD) for c in ring.coords}
    I, S = cfg.pipelines, cfg.stages
    B = cfg.geom.block_size
    for t in range(n_steps):
        ring.appends(t)
        if t >= 1:
            for c in ring.coords:
                n = ring.nodes[c]
                m = ring.ring_fn(c, I, S)
                for r, (s, ln, bt) in n.live().items():
                    for j, blk in enumerate(bt):
                        v = min(B, ln - j * B)
                        brute[m][blk, :, :, :, :v] = n.primary[blk, :, :, :, :v]
            ring.replicate(t)
    return {"ring": ring, "brute": brute}
