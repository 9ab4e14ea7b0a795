"""Pins for the CPU oracle against things other than itself (SURVEY §8(c) "What pins").

* hand-derived C1 tables (tests/golden/c1_tables.json);
* the paper's own worked example P:215 / P:225 / P:227 (ring walk);
* SPEC S:51-53, S:60-62 examples and exhaustive brute force;
* brute-force full-copy replay (I6) and library special cases (index_copy, memcpy);
* closed-form byte counts and block arithmetic, resume point;
* the R7 quarantine rule, with a naive variant that must break it.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch

from kvgen import configs
from kvgen.content import SENTINEL_WORD, POISON_WORD, content_tokens
from kvgen.schedule import closed_loop_schedule
from oracle import OracleNode, OracleError, instance_ring, stage_ring, plan_replication_targets
from oracle.simulate import OracleRing, check_all, check_content, full_copy_replay

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_tables.json")))


def _bt(live):
    return {str(r): bt for r, (s, ln, bt) in live.items()}


def test_c1_golden_tables_and_restore():
    snaps, moved = {}, {}

    def on_step(ring, t):
        snaps[t] = {k: n.live() for k, n in ring.serving.items()}
        moved[t] = ring.moved

    ring = OracleRing(configs.C1).run(on_step=on_step, check_every=1)
    for s in range(4):
        assert _bt(snaps[0][(0, s)]) == GOLD["after_prefill_bt"]
        if s != 2:
            for t in range(1, 9):
                assert _bt(snaps[t][(0, s)]) == GOLD["after_step1_bt"]
        assert all(ln == GOLD["final_len"] for _, ln, _ in snaps[8][(0, s)].values())
    # dirty bytes: 4 stages x 32 KiB per decode step in a failure-free step
    assert moved[3] - moved[2] == 4 * GOLD["decode_bytes_per_step_per_stage"]
    (_, t, coord, t_star, restored, ids, n_new) = ring.events[0]
    assert (t, coord, t_star) == (5, (0, 2), GOLD["t_star"])
    assert restored == [(r, GOLD["restored_len"]) for r in range(4)]
    assert ids == [0, 1, 2, 3] and n_new == [1, 1, 1, 1]       # <= 1 token re-appended (R3)
    assert _bt(snaps[5][(0, 2)]) == GOLD["restore_fresh_bt"]
    assert _bt(snaps[8][(0, 2)]) == GOLD["restore_fresh_bt"]
    check_content(ring, ring.serving[(0, 2)], 2)               # I4: restored == failure-free content


def test_c1_promotion_into_donor():
    cfg = configs.scaled(configs.C1, pipelines=2, num_blocks=48, max_reqs=8, ring="instance")
    ring = OracleRing(cfg)
    for t in range(5):
        ring.appends(t)
        if t >= 1:
            ring.replicate(t)
    ring.appends(5)
    donor = ring.nodes[(1, 2)]
    assert sorted(b for _, _, bt in donor.live().values() for b in bt) == list(range(20))
    t_star, restored, dst = ring.fail_and_restore(5, (0, 2))
    assert dst is donor and t_star == 4
    lo, hi = GOLD["promote_donor_ids"]
    got = sorted(b for r, (_, _, bt) in donor.live().items() if r < 1_000_000 for b in bt)
    assert got == list(range(lo, hi + 1))
    check_content(ring, donor, 2)


def test_paper_ring_example_p215_p227():
    # P:215 / P:225: (0,2) fails -> replacement and replication target (1,2)
    assert instance_ring((0, 2), 4, 4) == (1, 2)
    excl = {(0, 2), (1, 2), (2, 1), (3, 1)}
    base = plan_replication_targets(4, 4, set())
    plan = plan_replication_targets(4, 4, excl)
    changed = {n for n in plan if plan[n] != base[n]}
    assert changed == {(1, 1), (3, 2)}                       # exactly these two
    assert plan[(1, 1)] == (0, 1) and plan[(3, 2)] == (2, 2)
    # the stage ring would adjust different nodes: the paper's ring is the instance ring
    sbase = plan_replication_targets(4, 4, set(), ring=stage_ring)
    splan = plan_replication_targets(4, 4, excl, ring=stage_ring)
    assert {n for n in splan if splan[n] != sbase[n]} == {(0, 1), (1, 1), (2, 0), (3, 0)}


def test_ring_successor_spec_examples():
    assert instance_ring((0, 2), 4, 4) == (1, 2)
    assert instance_ring((3, 2), 4, 4) == (0, 2)
    assert instance_ring((0, 0), 2, 1) == (1, 0)
    assert stage_ring((0, 3), 1, 4) == (0, 0)
    for I, S in [(2, 3), (4, 4), (5, 2)]:
        for n in itertools.product(range(I), range(S)):
            x = n
            for _ in range(I):
                x = instance_ring(x, I, S)
            assert x == n                                    # S:74 cycle property
    assert plan_replication_targets(2, 1, {(1, 0)}) == {(0, 0): None}
    with pytest.raises(ValueError):
        instance_ring((4, 0), 4, 4)


def test_plan_matches_exhaustive_bruteforce():
    # S:75 / S:609: brute force = nearest non-excluded same-stage node by instance distance
    for I in range(2, 5):
        for S in range(1, 4):
            nodes = list(itertools.product(range(I), range(S)))
            for k in range(0, 3):
                for excl in itertools.combinations(nodes, k):
                    plan = plan_replication_targets(I, S, set(excl))
                    for (i, s) in nodes:
                        if (i, s) in excl:
                            assert (i, s) not in plan
                            continue
                        cands = [((i + dd) % I, s) for dd in range(1, I) if ((i + dd) % I, s) not in excl]
                        assert plan[(i, s)] == (cands[0] if cands else None)


def test_block_arithmetic_spec_s128_s137():
    g = configs.Geometry(layers=1, kv_heads=1, head_dim=8)
    n = OracleNode(g, 8, 2, 4, 0)
    src = content_tokens(1, [5] * 17, range(17), 0, 1, 1, 8)
    n.begin_step()
    n.append([5], [17], src)
    ln, bt = n.query(5)
    assert ln == 17 and bt == [0, 1]                    # 2 blocks, the second holds 1 token
    n.append([5], [15], content_tokens(1, [5] * 15, range(17, 32), 0, 1, 1, 8))
    assert n.query(5) == (32, [0, 1])                   # block 1 full at len 32
    n.append([5], [1], content_tokens(1, [5], [32], 0, 1, 1, 8))
    assert n.query(5) == (33, [0, 1, 2])                # rollover when len % B == 0
    with pytest.raises(OracleError) as e:
        n.append([6], [0], None)
    assert e.value.code == "KV_EINVAL"                  # S:129 empty prompt


def test_dirty_bytes_closed_form():
    g = configs.Geometry(layers=8)
    assert g.token_bytes == 8 * 2 * 8 * 128 * 2 == 32 * 1024
    assert g.block_bytes == 512 * 1024
    assert configs.Geometry(layers=4).block_bytes == 256 * 1024


def test_enomem_all_or_nothing():
    g = configs.Geometry(layers=1, kv_heads=1, head_dim=8)
    n = OracleNode(g, 4, 2, 4, 0)
    n.begin_step()
    n.append([1], [40], content_tokens(1, [1] * 40, range(40), 0, 1, 1, 8))   # 3 blocks
    before = (n.live(), set(n.free_blocks))
    with pytest.raises(OracleError) as e:
        n.append([1, 2], [9, 20], content_tokens(1, [1] * 9 + [2] * 20, list(range(40, 49)) + list(range(20)), 0, 1, 1, 8))
    assert e.value.code == "KV_ENOMEM"
    assert (n.live(), set(n.free_blocks)) == before


def _random_cfg(seed, NB=96, R=6, steps=40):
    return configs.scaled(configs.C1, num_blocks=NB, max_reqs=2 * R, max_blocks_per_req=12,
                          batch_cap=R, n_requests=60, n_steps=steps, fail_node=None, fail_step=None,
                          fixed_prompt=None, trace_seed=1000 + seed)


def _small_sched(cfg, seed):
    rng = np.random.default_rng(seed)
    p = rng.integers(1, 70, size=cfg.n_requests)
    o = rng.integers(1, 30, size=cfg.n_requests)
    return [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap)]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_incremental_equals_bruteforce_full_copy(seed):
    """I6: incremental replicas == full-copy replay, byte for byte, whole arrays (churn included)."""
    cfg = _random_cfg(seed)
    out = full_copy_replay(cfg, cfg.n_steps, schedules=_small_sched(cfg, seed))
    ring = out["ring"]
    for c in ring.coords:                                   # brute is keyed by holder
        assert np.array_equal(ring.nodes[c].replica, out["brute"][c])
    check_all(ring)


def test_full_block_loopback_is_index_copy():
    # special case: requests made of full blocks only; the replica is index_copy_ of block rows
    g = configs.Geometry(layers=2)
    a, b = OracleNode(g, 16, 4, 8, 0), OracleNode(g, 16, 4, 8, 1)
    a.set_successor(b)
    a.begin_step()
    ids, n_new = [3, 9], [32, 48]
    pos = list(range(32)) + list(range(48))
    a.append(ids, n_new, content_tokens(7, [3] * 32 + [9] * 48, pos, 0, 2, 8, 128))
    a.replicate(1)
    used = torch.tensor([blk for r in ids for blk in a.query(r)[1]])
    want = torch.full(tuple(b.replica.shape), SENTINEL_WORD, dtype=torch.int32)
    prim = torch.from_numpy(a.primary.astype(np.int32))
    want.index_copy_(0, used, prim.index_select(0, used))
    assert np.array_equal(b.replica.astype(np.int32), want.numpy())


def test_single_request_restore_is_memcpy():
    g = configs.Geometry(layers=2)
    f, h, dst = (OracleNode(g, 8, 2, 8, k) for k in range(3))
    f.set_successor(h)
    f.begin_step()
    f.append([11], [64], content_tokens(3, [11] * 64, range(64), 0, 2, 8, 128))
    f.replicate(1)
    before = f.primary.copy()
    f.fail()
    assert (f.primary == POISON_WORD).all()
    t_star, restored = dst.restore_from(h)
    assert t_star == 1 and restored == [(11, 64)]
    assert np.array_equal(dst.primary, before)         # identity remap == memcpy of the pool


def test_resume_point_spec_s295():
    g = configs.Geometry(layers=1, kv_heads=1, head_dim=8)
    f, h, dst = (OracleNode(g, 8, 2, 8, k) for k in range(3))
    f.set_successor(h)
    f.begin_step()
    f.append([4], [48], content_tokens(1, [4] * 48, range(48), 0, 1, 1, 8))
    f.replicate(1)
    f.begin_step()
    f.append([4], [1], content_tokens(1, [4], [48], 0, 1, 1, 8))   # unpublished token 48
    f.fail()
    assert dst.restore_from(h) == (1, [(4, 48)])                    # resume at 48
    with pytest.raises(OracleError) as e:
        OracleNode(g, 8, 2, 8, 9).restore_from(OracleNode(g, 8, 2, 8, 10))
    assert e.value.code == "KV_ENOREPLICA"                          # seq == 0


def _valid_positions(meta):
    out = set()
    B = 16
    for r, (s, ln, bt) in meta.items():
        for pos in range(ln):
            out.add((bt[pos // B], pos % B))
    return out


@pytest.mark.parametrize("naive", [False, True])
def test_quarantine_rule_r7(naive):
    """R7: no write of step t lands in a slot valid at published t-1 (and naive reuse breaks it)."""
    hits = 0
    for seed in range(6):
        cfg = _random_cfg(seed, NB=64, R=4, steps=60)
        ring = OracleRing(cfg, schedules=_small_sched(cfg, seed + 50))
        if naive:
            for n in ring.nodes.values():
                orig = n.release

                def rel(req_ids, n=n, orig=orig):
                    orig(req_ids)
                    n.free_blocks.update(n.q_blocks)
                    n.free_slots.update(n.q_slots)
                    n.q_blocks, n.q_slots = [], []
                n.release = rel
        for t in range(cfg.n_steps):
            ring.appends(t)
            if t >= 1:
                for c in ring.coords:
                    n = ring.nodes[c]
                    m = n.succ
                    prev_valid = _valid_positions(m.published())
                    before = m.replica.copy()
                    ring.moved += n.replicate(t)
                    diff = np.argwhere((before != m.replica).any(axis=(1, 2, 3, 5)))
                    hits += sum((int(b), int(s)) in prev_valid for b, s in diff)
    if naive:
        assert hits > 0
    else:
        assert hits == 0


def test_invariants_random_run_with_failure():
    cfg = configs.scaled(_random_cfg(4, NB=96, R=6, steps=30), fail_node=(0, 1), fail_step=17)
    ring = OracleRing(cfg, schedules=_small_sched(cfg, 99))
    ring.run(check_every=1)
    check_all(ring)
    (_, t, coord, t_star, restored, ids, n_new) = ring.events[0]
    assert t_star == 16
    for (p, s), n in ring.serving.items():
        check_content(ring, n, s)          # I2 / I4 on every live slot, restored stage included


@pytest.mark.parametrize("seed", [0, 1])
def test_block_mode_equals_completed_block_copy(seed):
    """NEXT-2 ("block-by-block", P:229 literal): the replica equals a brute-force copy
    of every COMPLETED block of every live request, published lengths are multiples
    of B, and the replica lags the primary by < B tokens per request."""
    cfg = _random_cfg(seed, steps=35)
    ring = OracleRing(cfg, schedules=_small_sched(cfg, seed), mode="blocks")
    B = cfg.geom.block_size
    brute = {c: np.full_like(ring.nodes[c].replica, SENTINEL_WORD) for c in ring.coords}
    for t in range(cfg.n_steps):
        ring.appends(t)
        if t >= 1:
            for c in ring.coords:
                n = ring.nodes[c]
                m = stage_ring(c, 1, 4)
                for r, (s, ln, bt) in n.live().items():
                    for j in range(ln // B):
                        brute[m][bt[j]] = n.primary[bt[j]]
            ring.replicate(t)
            for c in ring.coords:
                n = ring.nodes[c]
                pub = n.succ.published()
                for r, (s, ln, bt) in n.live().items():
                    hi = pub.get(r, (s, 0, []))[1]
                    assert hi % B == 0 and 0 <= ln - hi < B
        check_all(ring)
    for c in ring.coords:
        assert np.array_equal(ring.nodes[c].replica, brute[c])


def test_block_mode_restore_resumes_at_block_boundary():
    cfg = configs.scaled(_random_cfg(7, NB=96, R=6, steps=30), fail_node=(0, 1), fail_step=19)
    ring = OracleRing(cfg, schedules=_small_sched(cfg, 70), mode="blocks")
    ring.run(check_every=1)
    (_, t, coord, t_star, restored, ids, n_new) = ring.events[0]
    assert t_star == 18 and all(ln % 16 == 0 for _, ln in restored)
    for (p, s), n in ring.serving.items():
        check_content(ring, n, s)          # I4: resumed stage == failure-free content


def _brute_i1(n, holder):
    """I1 written out independently of the oracle's link bookkeeping: every valid slot
    of n's primary equals the holder's replica region at the same block id."""
    B = n.g.block_size
    for r, (s, ln, bt) in n.live().items():
        for j, blk in enumerate(bt):
            v = min(B, ln - j * B)
            if not np.array_equal(holder.replica[blk, :, :, :, :v], n.primary[blk, :, :, :, :v]):
                return False
    return True


def test_reprotect_applies_p227_plan_reseeds_and_freezes_excluded():
    """OracleRing.reprotect (NEXT-1, §3.2) pinned against the paper's own example
    rather than against the product: 4 instances x 3 stages on the paper's instance ring,
    (0,2) fails and is promoted onto (1,2); the exclusion set
    {(0,2),(1,2),(2,1),(3,1)} of P:227 must re-target exactly (1,1)->(0,1) and
    (3,2)->(2,2).  Applying the plan must (a) re-seed the re-targeted links -- the new
    holders did not hold those predecessors before, so only a full re-seed makes I1 hold at
    the next step, (b) leave the other links untouched (no re-seed: their holders' seq
    keeps advancing without a republication of old tokens), and (c) stop the excluded
    nodes: (2,1)'s and (3,1)'s old holders stay frozen at the last step published before
    the plan.  check_all (I1-I3) runs after every step."""
    cfg = configs.scaled(configs.C1, pipelines=4, stages=3, num_blocks=128, max_reqs=16,
                         max_blocks_per_req=12, batch_cap=3, n_requests=60, n_steps=30,
                         fixed_prompt=None, fail_node=(0, 2), fail_step=12, ring="instance")
    rng = np.random.default_rng(227)
    sched = [closed_loop_schedule(rng.integers(1, 60, 60), rng.integers(1, 25, 60),
                                  cfg.n_steps, cfg.batch_cap, pipeline=p) for p in range(4)]
    ring = OracleRing(cfg, ring="instance", schedules=sched)
    N = ring.nodes
    excluded = {(0, 2), (1, 2), (2, 1), (3, 1)}
    plan_t = 14
    frozen = {}
    for t in range(cfg.n_steps):
        ring.appends(t)
        if t == cfg.fail_step:
            ring.fail_and_restore(t, cfg.fail_node)
            assert ring.serving[(0, 2)] is N[(1, 2)]          # promotion onto (1,2)
        if t == plan_t:
            before = {c: N[c].succ for c in ring.coords}
            plan = ring.reprotect(excluded)
            # the paper's example: exactly these two adjusted targets
            changed = {c for c in ring.coords if c not in excluded
                       and plan[c] != instance_ring(c, 4, 3)}
            assert changed == {(1, 1), (3, 2)}
            assert plan[(1, 1)] == (0, 1) and plan[(3, 2)] == (2, 2)
            assert N[(1, 1)].succ is N[(0, 1)] and N[(3, 2)].succ is N[(2, 2)]
            for c in ((2, 1), (3, 1), (1, 2)):                # excluded: send nothing
                assert N[c].succ is None
            for c in ring.coords:                             # untouched links keep their holder
                if c not in excluded and c not in changed:
                    assert N[c].succ is before[c]
            # old holders of the excluded senders freeze at the last published step
            frozen = {(3, 1): N[(3, 1)].rseq, (0, 1): N[(0, 1)].rseq}
            assert frozen[(3, 1)] == t - 1 and frozen[(0, 1)] == t - 1
            # the new holders have not seen these predecessors yet
            assert not _brute_i1(N[(1, 1)], N[(0, 1)]) or not N[(1, 1)].live()
        if t >= 1:
            ring.replicate(t)
        check_all(ring)
        if t >= plan_t:
            assert N[(3, 1)].rseq == frozen[(3, 1)]      # (2,1) excluded: (3,1) frozen
            assert N[(0, 1)].rseq == t                    # now written by (1,1)
            assert N[(2, 2)].rseq == t
            assert _brute_i1(N[(1, 1)], N[(0, 1)]) and _brute_i1(N[(3, 2)], N[(2, 2)])
            for c in ring.coords:
                n = N[c]
                if c not in excluded and not n.dead and n.succ is not None:
                    assert _brute_i1(n, n.succ), c
