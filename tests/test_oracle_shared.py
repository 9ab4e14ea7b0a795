"""Pins for the shared-capacity mode of the oracle (§8(f) NEXT-3, reading R17):
replicas live in the holder's own pool and are dropped under memory pressure.

* P:233-235 §3.2 -- "utilizes such memory headroom to temporarily handle ... the
  replicated KV cache.  When memory pressure happens, KevlarFlow drops the
  replicated KV cache and recomputes them if needed."
* SPEC S:152 (blocks_held <= capacity; replica blocks evicted strictly before
  primary blocks), S:158 (replica blocks, oldest request first, then reject new
  admissions), S:311 (dropping replicas never changes results, only latency),
  S:312 (no admission is rejected while the replica census could make room).

The first test is a hand-derived trace (ids written out below, not produced by
the oracle); the others check invariants that hold at any size.
"""
import numpy as np
import pytest

from kvgen import configs
from kvgen.configs import Geometry
from kvgen.content import content_tokens
from kvgen.schedule import closed_loop_schedule
from oracle import OracleNode, OracleError
from oracle.simulate import OracleRing, check_all, check_tables

G = Geometry(layers=1, kv_heads=1, head_dim=8, block_size=2)


def _src(req, n, start, stage=0):
    return content_tokens(2601, [req] * n, list(range(start, start + n)), stage, 1, 1, 8)


def _pub(n):
    return {r: (ln, bt) for r, (s, ln, bt) in n.published().items()}


def test_hand_trace_eviction_order_drop_and_rejection():
    a = OracleNode(G, 6, 4, 4, node_id=0)          # predecessor
    h = OracleNode(G, 6, 4, 4, node_id=1)          # holder (shared capacity)
    a.set_successor(h, shared=True)
    # step 0: a admits r1 (3 tok -> blocks 0,1) and r2 (2 tok -> block 2); h admits q1 (block 0)
    a.begin_step(); a.append([1, 2], [3, 2], np.concatenate([_src(1, 3, 0), _src(2, 2, 0)]))
    h.begin_step(); h.append([101], [2], _src(101, 2, 0))
    # step 1: replicas from h's free list, lowest id first: r1 -> [1, 2], r2 -> [3]
    a.replicate(1)
    assert _pub(h) == {1: (3, [1, 2]), 2: (2, [3])}
    assert a.census() == 3 and sorted(h.free_blocks) == [4, 5]
    assert np.array_equal(h.primary[1, :, :, :, :2], a.primary[0, :, :, :, :2])
    assert np.array_equal(h.primary[2, :, :, :, :1], a.primary[1, :, :, :, :1])
    # step 2: h admits q2 (6 tok = 3 blocks); free 2 < 3 <= free + census 5: evict the
    # OLDEST replica (r1) only -> free {1, 2, 4, 5}; q2 takes 1, 2, 4
    h.begin_step(); h.append([102], [6], _src(102, 6, 0))
    assert h.evictions == 1 and a.dropped[0] and not a.dropped[1]
    assert h.live()[102][2] == [1, 2, 4]
    assert _pub(h) == {2: (2, [3])}                 # r1 left the published table at once
    a.replicate(2)
    assert _pub(h) == {2: (2, [3])}                 # a dropped replica is never re-sent
    # step 3: h admits q3 (4 tok = 2 blocks): free {5} + census 1 -> evict r2; q3 takes 3, 5
    h.begin_step(); h.append([103], [4], _src(103, 4, 0))
    assert h.evictions == 2 and a.census() == 0 and h.live()[103][2] == [3, 5]
    # step 4: q4 needs 1 block, free 0 + census 0 -> rejected (only now), no change
    h.begin_step()
    with pytest.raises(OracleError, match="ENOMEM"):
        h.append([104], [2], _src(104, 2, 0))
    assert 104 not in h.live() and h.evictions == 2
    # a new request of a: its replica cannot get a block -> dropped, not queued
    a.begin_step(); a.append([5], [2], _src(5, 2, 0))
    a.replicate(4)
    assert a.drops == 1 and _pub(h) == {}
    check_tables(h)
    check_tables(a)


def test_release_frees_replica_blocks_immediately():
    a = OracleNode(G, 8, 4, 4, node_id=0)
    h = OracleNode(G, 8, 4, 4, node_id=1)
    a.set_successor(h, shared=True)
    a.begin_step(); a.append([7], [4], _src(7, 4, 0))
    a.replicate(1)
    assert _pub(h) == {7: (4, [0, 1])}
    a.begin_step(); a.release([7])
    # primary blocks are quarantined (R7); the replica blocks are free at once because
    # the published entry that referenced them is withdrawn first
    assert sorted(a.q_blocks) == [0, 1] and {0, 1} <= h.free_blocks and _pub(h) == {}
    check_tables(h)


def _pressure_cfg(**kw):
    base = dict(num_blocks=40, max_reqs=12, max_blocks_per_req=12, batch_cap=5,
                n_requests=60, n_steps=40, fixed_prompt=None, fail_node=(0, 1), fail_step=23)
    base.update(kw)
    return configs.scaled(configs.C1, **base)


def _sched(cfg, seed):
    rng = np.random.default_rng(seed)
    p = rng.integers(1, 70, size=cfg.n_requests)
    o = rng.integers(1, 30, size=cfg.n_requests)
    return [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap, pipeline=i)
            for i in range(cfg.pipelines)]


# (seed, ring, restore, blocks, batch cap, slots): sized so that evictions AND drops occur
PRESSURE = [(0, "stage", "fresh", 32, 5, 12), (1, "stage", "fresh", 28, 5, 12),
            (4, "instance", "promote", 48, 5, 24)]


def pressure_ring(seed, ring, restore_mode, nb, cap, slots):
    cfg = _pressure_cfg(num_blocks=nb, batch_cap=cap, max_reqs=slots,
                        pipelines=2 if ring == "instance" else 1, ring=ring,
                        fail_node=(0, 2) if ring == "instance" else (0, 1))
    return cfg, _sched(cfg, seed)


@pytest.mark.parametrize("seed,ring,restore_mode,nb,cap,slots", PRESSURE)
def test_shared_pressure_run_invariants(seed, ring, restore_mode, nb, cap, slots):
    """Churn under pressure with a failure: tables partition every pool (primary +
    held replica + free + quarantine), every published replica equals its primary
    (I1), every valid slot equals the closed form (I2, I4 after the restore), and
    evictions / drops actually happened."""
    cfg, sch = pressure_ring(seed, ring, restore_mode, nb, cap, slots)
    r = OracleRing(cfg, shared=True, restore_mode=restore_mode, ring=ring, schedules=sch)
    r.run(check_every=1)
    check_all(r)
    assert sum(n.evictions for n in r.all_nodes()) > 0
    assert sum(n.drops for n in r.all_nodes()) > 0


def test_dropping_replicas_never_changes_primary_content():
    """the same schedule with and without the shared holder (and its drops)
    ends with identical primary pools and tables on every node (no failure)."""
    cfg = _pressure_cfg(fail_node=None, fail_step=None)
    sch = _sched(cfg, 3)
    a = OracleRing(cfg, shared=True, schedules=sch).run()
    b = OracleRing(cfg, shared=False, schedules=sch).run()
    for c in a.coords:
        la, lb = a.nodes[c].live(), b.nodes[c].live()
        assert {r: v[:2] for r, v in la.items()} == {r: v[:2] for r, v in lb.items()}
        used = sorted(x for _, _, bt in a.nodes[c].live().values() for x in bt)
        # same live content; block ids may differ (replicas share the free list)
        for rr, (s, ln, bt) in a.nodes[c].live().items():
            sb = b.nodes[c].live()[rr][2]
            for j in range(len(bt)):
                v = min(cfg.geom.block_size, ln - j * cfg.geom.block_size)
                assert np.array_equal(a.nodes[c].primary[bt[j], :, :, :, :v],
                                      b.nodes[c].primary[sb[j], :, :, :, :v])
        assert len(used) == len(set(used))


def test_admission_rejected_only_when_census_cannot_cover_it():
    """S:312 as a property: for random pressure, an append is rejected iff its
    block need exceeds free + census; when it succeeds it evicted the minimum
    prefix of replicas in admission order."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        a = OracleNode(G, 10, 6, 6, node_id=0)
        h = OracleNode(G, 10, 6, 6, node_id=1)
        a.set_successor(h, shared=True)
        ids = list(range(1, 1 + int(rng.integers(1, 5))))
        lens = [int(x) for x in rng.integers(1, 5, size=len(ids))]
        a.begin_step()
        a.append(ids, lens, np.concatenate([_src(r, n, 0) for r, n in zip(ids, lens)]))
        h.begin_step()
        h.append([900], [1], _src(900, 1, 0))
        a.replicate(1)
        free, census = len(h.free_blocks), a.census()
        ages = [s for _, s in sorted((int(a.admit_seq[s]), s) for s in range(a.R) if a.rep_bt[s])]
        need_tok = int(rng.integers(1, 13))
        need = -(-need_tok // 2)
        h.begin_step()
        if need > free + census:
            with pytest.raises(OracleError, match="ENOMEM"):
                h.append([901], [need_tok], _src(901, need_tok, 0))
            assert a.census() == census
        else:
            before = [list(b) for b in a.rep_bt]
            h.append([901], [need_tok], _src(901, need_tok, 0))
            evicted = [s for s in range(a.R) if before[s] and not a.rep_bt[s]]
            assert evicted == ages[:len(evicted)]          # oldest first, a prefix
            got = free + sum(len(before[s]) for s in evicted)
            assert got >= need and (not evicted or got - len(before[evicted[-1]]) < need)
        check_tables(h)
