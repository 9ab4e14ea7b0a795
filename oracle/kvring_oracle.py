"""Oracle logical node: paged KV pool, block tables, replica region (numpy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper passages this follows:
* P:223-225 §3.2 -- "replicates KV cache for each request to the GPU memory of
  other nodes ... In-progress requests will be served continuously on the
  replication target from the replicated state."
* P:229 §3.2 -- "a block representation of KV cache ... replicate it
  block-by-block in the background" (granularity reading R2: the dirty tokens
  of each block, every step).
* SURVEY §8(c) "Algorithm" steps 1-7 and readings R4-R12.

Layout (reading R4): a block is uint16 [L][2][H][B][d]; the pool is
[NB][L][2][H][B][d].  The replica region of node m mirrors the block ids of
its ring predecessor (R5).  Shared-capacity mode (§8(f) NEXT-3
§3.2, SPEC S:152/S:158/S:312, reading R17): the holder keeps its predecessor's
replica blocks inside its OWN pool, allocated from its own free list, and drops
them (oldest request first) when its primary needs the memory.  Replica metadata (R9): ``seq`` (0 = nothing
published), parity double-buffered (req_id, len) per request slot, and one bt
row per slot.
"""
from __future__ import annotations

import numpy as np

from kvgen.content import SENTINEL_WORD, POISON_WORD

ENOMEM, EINVAL, ESTATE, ENOREPLICA = "KV_ENOMEM", "KV_EINVAL", "KV_ESTATE", "KV_ENOREPLICA"
POISON_U64 = (1 << 64) - 1


class OracleError(Exception):
    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class OracleNode:
    """One logical node (instance, stage): primary pool + replica of its predecessor.

    ``content=False`` keeps tables only (metadata-only mode for full-size
    configs, where valid KV is checked against the closed form instead).
    """

    def __init__(self, geom, num_blocks: int, max_reqs: int, max_blocks_per_req: int,
                 node_id: int, pred_num_blocks: int | None = None, content: bool = True):
        self.g = geom
        self.NB = num_blocks
        self.R = max_reqs
        self.M = max_blocks_per_req
        self.node_id = node_id
        self.content = content
        B = geom.block_size
        shape = (geom.layers, 2, geom.kv_heads, B, geom.head_dim)
        nb_pred = num_blocks if pred_num_blocks is None else pred_num_blocks
        if content:
            self.primary = np.full((num_blocks,) + shape, SENTINEL_WORD, dtype=np.uint16)
            self.replica = np.full((nb_pred,) + shape, SENTINEL_WORD, dtype=np.uint16)
        else:
            self.primary = self.replica = None
        # replica metadata written by the predecessor (R9); initial = nothing published
        self.rseq = 0
        self.rreq = np.full((2, max_reqs), -1, dtype=np.int64)
        self.rlen = np.zeros((2, max_reqs), dtype=np.int32)
        self.rbt = np.full((max_reqs, max_blocks_per_req), -1, dtype=np.int32)
        # host tables of the primary pool (R6: lowest free id; R7: one-step quarantine)
        self.free_blocks = set(range(num_blocks))
        self.q_blocks: list[int] = []
        self.free_slots = set(range(max_reqs))
        self.q_slots: list[int] = []
        self.slot_req = np.full(max_reqs, -1, dtype=np.int64)
        self.slot_len = np.zeros(max_reqs, dtype=np.int32)
        self.slot_bt: list[list[int]] = [[] for _ in range(max_reqs)]
        self.pub_len = np.zeros(max_reqs, dtype=np.int32)
        self.slot_of: dict[int, int] = {}
        self.succ: OracleNode | None = None
        self.last_step = 0
        self.dead = False
        self.mode = "tokens"     # "blocks": completed blocks only (P:229 literal; NEXT-2)
        # shared-capacity mode (NEXT-3, reading R17).  Predecessor side: the holder
        # and, per slot, the holder block ids of the request's replica, whether
        # its replica was dropped, and its admission order (eviction age).
        self.holder: OracleNode | None = None
        self.rep_bt: list[list[int]] = [[] for _ in range(max_reqs)]
        self.dropped = np.zeros(max_reqs, dtype=bool)
        self.admit_seq = np.zeros(max_reqs, dtype=np.int64)
        self.admit_ctr = 0
        # holder side: the predecessor whose replicas live in this pool
        self.rep_src: OracleNode | None = None
        self.evictions = 0       # requests whose replica this holder evicted
        self.drops = 0           # requests whose replica could not grow (predecessor side)

    # ------------------------------------------------------------------ allocator
    def begin_step(self) -> None:
        """§8(c) step 1: ``free U= quarantine; quarantine = {}`` (R7)."""
        self._alive()
        self.free_blocks.update(self.q_blocks)
        self.free_slots.update(self.q_slots)
        self.q_blocks, self.q_slots = [], []

    def release(self, req_ids) -> None:
        """§8(c) step 2 (retire): blocks and slot go to quarantine, not to the free list (R7)."""
        self._alive()
        for r in req_ids:
            if r not in self.slot_of:
                raise OracleError(EINVAL, f"unknown request {r}")
        for r in req_ids:
            s = self.slot_of.pop(r)
            if self.holder is not None:
                self._free_rep(s)
                self.dropped[s] = False
            self.q_blocks.extend(self.slot_bt[s])
            self.q_slots.append(s)
            self.slot_bt[s] = []
            self.slot_req[s] = -1
            self.slot_len[s] = 0
            self.pub_len[s] = 0

    def _take_block(self) -> int:
        b = min(self.free_blocks)            # R6: lowest free block id
        self.free_blocks.remove(b)
        return b

    def append(self, req_ids, n_new, src: np.ndarray | None) -> None:
        """§8(c) steps 3-4: decode appends and admissions, in the given entry order.

        ``src`` is dense uint16 [sum(n_new)][L][2][H][d] (entry order).  An
        unknown req_id is an admission: slot = min(free slots), then its
        blocks.  For every token: ``if len % B == 0: bt.append(min(free))``,
        write the token at (bt[len // B], len % B), ``len += 1``.  All or
        nothing: on exhaustion nothing changes and KV_ENOMEM is raised.
        """
        self._alive()
        B = self.g.block_size
        if len(req_ids) != len(n_new) or any(n < 0 for n in n_new):
            raise OracleError(EINVAL, "bad append arguments")
        need_blocks, need_slots, seen = 0, 0, set()
        for r, n in zip(req_ids, n_new):
            if r in seen:
                raise OracleError(EINVAL, f"request {r} twice in one append")
            seen.add(r)
            if r in self.slot_of:
                s = self.slot_of[r]
                cur = int(self.slot_len[s])
            else:
                if n <= 0:
                    raise OracleError(EINVAL, "admission with no tokens (S:129)")
                need_slots += 1
                cur = 0
            new_total = ceil_div(cur + n, B)
            if new_total > self.M:
                raise OracleError(ENOMEM, f"request {r} exceeds max_blocks_per_req")
            need_blocks += new_total - ceil_div(cur, B)
        census = self.rep_src.census() if self.rep_src is not None else 0
        if need_slots > len(self.free_slots) or need_blocks > len(self.free_blocks) + census:
            raise OracleError(ENOMEM, "pool or slots exhausted")
        if need_blocks > len(self.free_blocks):
            self._evict_for(need_blocks)        # drop replicated KV under pressure
        row = 0
        for r, n in zip(req_ids, n_new):
            if r not in self.slot_of:
                s = min(self.free_slots)        # R6: lowest free slot
                self.free_slots.remove(s)
                self.slot_of[r] = s
                self.slot_req[s] = r
                self.slot_len[s] = 0
                self.pub_len[s] = 0
                self._admitted(s)
            s = self.slot_of[r]
            for _ in range(n):
                ln = int(self.slot_len[s])
                if ln % B == 0:
                    self.slot_bt[s].append(self._take_block())
                if self.content:
                    blk = self.slot_bt[s][ln // B]
                    self.primary[blk, :, :, :, ln % B, :] = src[row]
                self.slot_len[s] = ln + 1
                row += 1

    # ---------------------------------------------------------------- replication
    def set_mode(self, mode: str) -> None:
        """Granularity reading R2: "tokens" (every step, exact) or "blocks" (P:229
        "block-by-block": only completed blocks; the replica lags < B tokens).
        A switch re-seeds the link."""
        assert mode in ("tokens", "blocks")
        self.mode = mode
        self.pub_len[:] = 0

    def published_len(self, s: int) -> int:
        """Length a publication of slot s reaches (all tokens, or completed blocks)."""
        if self.holder is not None and self.dropped[s]:
            return 0                            # dropped replica: never published again
        ln = int(self.slot_len[s])
        if self.mode == "blocks":
            return max(int(self.pub_len[s]), ln - ln % self.g.block_size)
        return ln

    def set_successor(self, succ: OracleNode | None, shared: bool = False) -> None:
        """Bind the ring link (SPEC S:298-306 apply_plan); a new link re-seeds: pub_len = 0.

        ``shared``: the successor keeps the replica in its own pool (NEXT-3, R17).
        Replicas held by a previous shared successor are freed first; a holder
        serves one predecessor, so another predecessor's replicas in ``succ`` are
        dropped and that predecessor unlinked from it."""
        self._alive()
        if self.holder is not None:
            self._free_all_reps()
            self.holder.rep_src = None
            self.holder = None
        self.succ = succ
        self.pub_len[:] = 0
        self.dropped[:] = False
        if shared:
            if succ is None or succ is self:
                raise OracleError(EINVAL, "shared mode needs another successor")
            old = succ.rep_src
            if old is not None and old is not self:
                old._free_all_reps()
                old.holder = None
                old.succ = None
            self.holder = succ
            succ.rep_src = self

    # ------------------------------------------------ shared capacity (NEXT-3, R17)
    # P:233-235 §3.2: "KevlarFlow utilizes such memory headroom to temporarily
    # handle rerouted traffic and the replicated KV cache.  When memory pressure
    # happens, KevlarFlow drops the replicated KV cache and recomputes them if
    # needed."  SPEC S:158 (replica blocks go first, oldest request first; primary
    # blocks are never evicted), S:312 (no admission is rejected while evicting
    # replicas could make room).
    def census(self) -> int:
        """Replica blocks this node's replicas occupy in its holder (predecessor side)."""
        return sum(len(b) for b in self.rep_bt)

    def _admitted(self, s: int) -> None:
        self.admit_ctr += 1
        self.admit_seq[s] = self.admit_ctr
        self.dropped[s] = False
        self.rep_bt[s] = []

    def _free_rep(self, s: int) -> None:
        """Free slot s's replica blocks in the holder AT ONCE, after removing the
        request from the holder's published table (parity of the published step):
        a restore can then never read the reused blocks (the device does the same
        with two small memsets ordered before any reuse)."""
        h = self.holder
        if h is None or not self.rep_bt[s]:
            return
        if self.last_step > 0 and not h.dead:
            par = self.last_step & 1
            h.rreq[par, s] = -1
            h.rlen[par, s] = 0
        h.free_blocks.update(self.rep_bt[s])
        self.rep_bt[s] = []

    def _free_all_reps(self) -> None:
        for s in range(self.R):
            self._free_rep(s)

    def _evict_for(self, need_blocks: int) -> None:
        """Holder side: drop the predecessor's replicas, oldest request first, until
        ``need_blocks`` blocks are free."""
        pred = self.rep_src
        order = sorted((int(pred.admit_seq[s]), s) for s in range(pred.R)
                       if pred.slot_req[s] >= 0 and pred.rep_bt[s])
        for _, s in order:
            if len(self.free_blocks) >= need_blocks:
                break
            pred._free_rep(s)
            pred.dropped[s] = True
            self.evictions += 1

    def drop_replicas(self) -> None:
        """Holder side: free every replica block held for the predecessor (after a
        restore read them, or on demand); a dead predecessor is unlinked."""
        pred = self.rep_src
        if pred is None:
            return
        for s in range(pred.R):
            if pred.rep_bt[s]:
                pred._free_rep(s)
                pred.dropped[s] = True
        if pred.dead:
            pred.holder = None
            self.rep_src = None

    def replicate(self, step: int) -> int:
        """§8(c) step 5: copy tokens [pub_len, len) of every live slot to succ's replica.

        Same block ids on the successor (R5), then (req_id, len) into parity
        buffer ``step & 1``, the bt rows, and ``seq = step`` (R9).  Returns the
        payload bytes D moved (D = n_tok * L * 2 * H * d * 2).
        """
        self._alive()
        if step <= self.last_step:
            raise OracleError(EINVAL, "step must be strictly increasing")
        m = self.succ
        if m is None:
            raise OracleError("KV_EPEER", "no successor bound")
        B = self.g.block_size
        moved = 0
        if m.dead:
            raise OracleError(ESTATE, "successor is dead; the harness must unlink it first")
        hi_all = np.zeros(self.R, dtype=np.int32)
        shared = self.holder is not None
        for s in range(self.R):
            if self.slot_req[s] < 0:
                continue
            lo, hi = int(self.pub_len[s]), self.published_len(s)
            if shared and hi > lo:
                # replica blocks come from the holder's own free list (R6 order);
                # if it cannot hold the growth, this request's replica is dropped
                grow = ceil_div(hi, B) - len(self.rep_bt[s])
                if grow > len(m.free_blocks):
                    self._free_rep(s)
                    self.dropped[s] = True
                    self.drops += 1
                    continue
                for _ in range(grow):
                    self.rep_bt[s].append(m._take_block())
            hi_all[s] = hi
            if self.content:
                for pos in range(lo, hi):
                    blk = self.slot_bt[s][pos // B]
                    if shared:
                        dst = self.rep_bt[s][pos // B]
                        m.primary[dst, :, :, :, pos % B, :] = self.primary[blk, :, :, :, pos % B, :]
                    else:
                        m.replica[blk, :, :, :, pos % B, :] = self.primary[blk, :, :, :, pos % B, :]
            moved += (hi - lo) * self.g.token_bytes
        par = step & 1
        m.rreq[par, :] = np.where(hi_all > 0, self.slot_req, -1)
        m.rlen[par, :] = hi_all
        for s in range(self.R):
            if self.slot_req[s] >= 0:
                nb = ceil_div(int(hi_all[s]), B)
                m.rbt[s, :nb] = (self.rep_bt[s] if shared else self.slot_bt[s])[:nb]
        m.rseq = step
        self.pub_len[:] = hi_all
        self.last_step = step
        return moved

    # ------------------------------------------------------------ failure / restore
    def fail(self) -> None:
        """§8(c) step 6: the node's memory is lost -- poison pool, replica and metadata (a7)."""
        self.dead = True
        if self.content:
            self.primary[...] = POISON_WORD
            self.replica[...] = POISON_WORD
        self.rseq = POISON_U64
        self.rreq[...] = -1
        self.rlen[...] = -1
        self.rbt[...] = -1

    def restore_from(self, holder: OracleNode) -> tuple[int, list[tuple[int, int]]]:
        """§8(c) step 7: rebuild the failed predecessor's requests into THIS pool.

        Reads holder's ``seq = t*`` and parity ``t* & 1`` metadata; for req_id
        ascending, for logical block j ascending: ``new = min(free)``, copy the
        valid slots [0, min(B, len - jB)) of replica block bt[slot][j], and
        rebuild bt.  Returns (t*, [(req_id, resume_len)]).  The restored
        requests start unpublished (pub_len = 0).  ``holder`` may be this very
        node (promotion on the replication target, P:225 / reading R10): the
        copy then runs from its replica region into its own primary pool.  A
        shared-capacity holder (NEXT-3) keeps the replica in its own pool; the
        copy reads it there (the caller frees it afterwards: drop_replicas).
        """
        self._alive()
        if holder.dead or holder.rseq == 0:
            raise OracleError(ENOREPLICA, "holder dead or nothing published")
        t_star = int(holder.rseq)
        par = t_star & 1
        entries = sorted((int(holder.rreq[par, s]), int(holder.rlen[par, s]), s)
                         for s in range(holder.R) if holder.rreq[par, s] >= 0)
        B = self.g.block_size
        need_b = sum(ceil_div(ln, B) for _, ln, _ in entries)
        if len(entries) > len(self.free_slots) or need_b > len(self.free_blocks):
            raise OracleError(ENOMEM, "restore target too small")
        for r, _, _ in entries:
            if r in self.slot_of:
                raise OracleError(EINVAL, f"request {r} already present in restore target")
        out = []
        store = holder.primary if holder.rep_src is not None else holder.replica
        for r, ln, hs in entries:
            s = min(self.free_slots)
            self.free_slots.remove(s)
            self.slot_of[r] = s
            self.slot_req[s] = r
            self.slot_len[s] = ln
            self.pub_len[s] = 0
            self._admitted(s)
            for j in range(ceil_div(ln, B)):
                new = self._take_block()
                self.slot_bt[s].append(new)
                if self.content:
                    src_blk = int(holder.rbt[hs, j])
                    valid = min(B, ln - j * B)
                    self.primary[new, :, :, :, :valid, :] = store[src_blk, :, :, :, :valid, :]
            out.append((r, ln))
        return t_star, out

    # ------------------------------------------------------------------- queries
    def query(self, req_id: int) -> tuple[int, list[int]]:
        s = self.slot_of.get(req_id)
        if s is None:
            raise OracleError(EINVAL, f"unknown request {req_id}")
        return int(self.slot_len[s]), list(self.slot_bt[s])

    def live(self) -> dict[int, tuple[int, int, list[int]]]:
        """{req_id: (slot, len, bt)} of the primary pool."""
        return {r: (s, int(self.slot_len[s]), list(self.slot_bt[s])) for r, s in self.slot_of.items()}

    def published(self) -> dict[int, tuple[int, int, list[int]]]:
        """{req_id: (slot, len, bt[:nblk])} in this node's replica metadata at seq."""
        if self.dead or self.rseq == 0:
            return {}
        par = self.rseq & 1
        B = self.g.block_size
        out = {}
        for s in range(self.R):
            r = int(self.rreq[par, s])
            if r >= 0:
                ln = int(self.rlen[par, s])
                out[r] = (s, ln, [int(x) for x in self.rbt[s, :ceil_div(ln, B)]])
        return out

    def _alive(self) -> None:
        if self.dead:
            raise OracleError(ESTATE, f"node {self.node_id} is dead")
