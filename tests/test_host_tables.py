"""CPU tests of libkvring's host logic (no GPU): the library loads and exports
every symbol include/kvring.h declares, and the C++ allocator / step protocol
(tables-only pools, device = -1: nothing is launched, no KV byte moves) matches
the CPU oracle's tables step by step -- at full C2 / C4 geometry."""
import os
import re

import pytest

from kvgen import configs
from oracle.simulate import OracleRing
from paper_2601_22438_b200 import kvring as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE_PTR = 0x1000   # never dereferenced by a tables-only pool


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "kvring.h")).read()
    declared = set(re.findall(r"\b(kv_[a-z_]+)\s*\(", hdr))
    lib = K.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(K.EXPORTED)
    assert K.kv_abi_version() == 1
    g = K.geom(8)
    assert K.kv_block_bytes(g) == 512 * 1024
    assert K.kv_meta_bytes(64, 192) % 256 == 0
    assert K.kv_meta_bytes(64, 192) >= 32 + 24 * 64 + 4 * 64 * 192


def _pool(cfg, node_id, device=-1):
    g = cfg.geom
    d = K.kv_pool_desc_t(K.geom(g.layers, g.kv_heads, g.head_dim, g.block_size, g.elem_bytes),
                         cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, device, node_id,
                         cfg.num_blocks, None, None, None)
    return K.kv_pool_create(d)


def _tables(h, R):
    req, ln, pub, nb = K.kv_dump_slots(h, R)
    out = {}
    for s in range(R):
        if req[s] >= 0:
            out[int(req[s])] = (s, int(ln[s]), K.kv_query(h, int(req[s]))[1])
    return out


@pytest.mark.parametrize("name,steps,ce", [("c1_tiny", 9, False), ("c2_pp4_b64", 260, False),
                                           ("c4_failover_16", 60, False),
                                           ("c2_pp4_b64", 120, True)])
def test_tables_match_oracle(name, steps, ce):
    """Slots, lengths, block ids and per-step payload bytes == oracle (metadata mode);
    ce: the copy-engine variant's work-list split (NEXT-4) keeps the same tables/bytes."""
    cfg = configs.ALL[name]
    cfg = configs.scaled(cfg, fail_step=None, fail_node=None)
    ring = OracleRing(cfg, content=False)
    sched = ring.sched
    coords = ring.coords
    hs = {c: _pool(cfg, k) for k, c in enumerate(coords)}
    for c in coords:
        K.kv_set_successor(hs[c], 0, FAKE_PTR, cfg.num_blocks, FAKE_PTR)
    try:
        for t in range(steps):
            ring.appends(t)
            entries = []
            for c in coords:
                p = c[0]
                ev = sched[p].steps[t]
                ids, n_new = ev.appends()
                entries.append(dict(pool=hs[c], begin_step=1, release=ev.retire,
                                    req_ids=sorted(ev.decode) + [r for r, _ in ev.admit],
                                    n_new=[1] * len(ev.decode) + [pp for _, pp in ev.admit], src=None))
            K.kv_append_multi(entries)
            if t >= 1:
                before = {c: ring.nodes[c].pub_len.copy() for c in coords}
                moved0 = ring.moved
                ring.replicate(t)
                (K.kv_replicate_step_ce if ce else K.kv_replicate_step_multi)(
                    [hs[c] for c in coords], t)
                total = sum(K.kv_stats(hs[c])["last_step_bytes"] for c in coords)
                assert total == ring.moved - moved0
            for c in coords:
                assert _tables(hs[c], cfg.max_reqs) == ring.nodes[c].live(), (t, c)
                st = K.kv_stats(hs[c])
                n = ring.nodes[c]
                assert st["free_blocks"] == len(n.free_blocks)
                assert st["quarantined_blocks"] == len(n.q_blocks)
    finally:
        for h in hs.values():
            K.kv_pool_destroy(h)


def test_errors_and_all_or_nothing():
    cfg = configs.scaled(configs.C1, num_blocks=4, max_reqs=2, max_blocks_per_req=4)
    h = _pool(cfg, 0)
    try:
        K.kv_append(h, [1], [40], None)                         # 3 blocks
        before = _tables(h, 2)
        with pytest.raises(K.KvError) as e:
            K.kv_append(h, [1, 2], [9, 20], None)               # needs 3 more, 1 free
        assert e.value.code == K.KV_ENOMEM
        assert _tables(h, 2) == before
        with pytest.raises(K.KvError) as e:
            K.kv_append(h, [5], [0], None)
        assert e.value.code == K.KV_EINVAL                       # empty admission
        with pytest.raises(K.KvError) as e:
            K.kv_append(h, [-1], [3], None)
        assert e.value.code == K.KV_EINVAL                       # -1 marks an empty slot (R9)
        with pytest.raises(K.KvError) as e:
            K.kv_append(h, [7, 7], [1, 1], None)
        assert e.value.code == K.KV_EINVAL
        with pytest.raises(K.KvError) as e:
            K.kv_release(h, [99])
        assert e.value.code == K.KV_EINVAL
        with pytest.raises(K.KvError) as e:
            K.kv_replicate_step(h, 1)
        assert e.value.code == K.KV_EPEER
        K.kv_set_successor(h, 1, FAKE_PTR, 4, FAKE_PTR)
        with pytest.raises(K.KvError) as e:
            K.kv_replicate_step(h, 0)
        assert e.value.code == K.KV_EINVAL                       # steps start at 1
        K.kv_replicate_step(h, 3)
        with pytest.raises(K.KvError) as e:
            K.kv_replicate_step(h, 3)
        assert e.value.code == K.KV_EINVAL                       # strictly increasing
        with pytest.raises(K.KvError):
            K.kv_set_successor(h, 1, FAKE_PTR, 3, FAKE_PTR)      # replica region too small
        # release -> quarantine: not reusable before begin_step (R7)
        K.kv_release(h, [1])
        assert K.kv_stats(h)["quarantined_blocks"] == 3
        with pytest.raises(K.KvError) as e:
            K.kv_append(h, [2], [20], None)
        assert e.value.code == K.KV_ENOMEM
        K.kv_begin_step(h)
        K.kv_append(h, [2], [20], None)
        assert K.kv_query(h, 2) == (20, [0, 1])
    finally:
        K.kv_pool_destroy(h)


def test_bad_geometry_rejected():
    for kw in (dict(layers=0), dict(head_dim=100), dict(elem_bytes=4), dict(block_size=0)):
        g = dict(layers=2, kv_heads=8, head_dim=128, block_size=16, elem_bytes=2)
        g.update(kw)
        d = K.kv_pool_desc_t(K.geom(**g), 8, 2, 4, -1, 0, 8, None, None, None)
        with pytest.raises(K.KvError) as e:
            K.kv_pool_create(d)
        assert e.value.code == K.KV_EINVAL


def test_plan_targets_matches_oracle_ring_walk():
    """kv_plan_targets (C++) == the oracle's ring walk, exhaustively."""
    import itertools
    from oracle.ring import instance_ring, plan_replication_targets, stage_ring
    for ring in (instance_ring, stage_ring):
        for I in range(1, 5):
            for S in range(1, 4):
                coords = [(i, s) for i in range(I) for s in range(S)]
                idx = {c: k for k, c in enumerate(coords)}
                succ = [idx[ring(c, I, S)] for c in coords]
                for k in range(0, 4):
                    for excl in itertools.combinations(coords, k):
                        got = K.kv_plan_targets(succ, [idx[c] for c in excl])
                        want = plan_replication_targets(I, S, set(excl), ring=ring)
                        for c in coords:
                            w = want.get(c)
                            assert got[idx[c]] == (-1 if w is None else idx[w]), (I, S, excl, c)
    # the paper's example through the C ABI
    coords = [(i, s) for i in range(4) for s in range(4)]
    idx = {c: k for k, c in enumerate(coords)}
    succ = [idx[instance_ring(c, 4, 4)] for c in coords]
    excl = [(0, 2), (1, 2), (2, 1), (3, 1)]
    base = K.kv_plan_targets(succ)
    got = K.kv_plan_targets(succ, [idx[c] for c in excl])
    changed = {coords[k] for k in range(16) if got[k] != base[k] and coords[k] not in excl}
    assert changed == {(1, 1), (3, 2)}
    assert got[idx[(1, 1)]] == idx[(0, 1)] and got[idx[(3, 2)]] == idx[(2, 2)]


def test_loop_tables_match_oracle():
    """The one-launch-per-step loop's host side (tables-only pools): after the final
    flush every table and the payload byte count equal the oracle's at C2 size."""
    cfg = configs.C2
    ring = OracleRing(cfg, content=False)
    sched = ring.sched
    hs = {c: _pool(cfg, k) for k, c in enumerate(ring.coords)}
    for c in ring.coords:
        K.kv_set_successor(hs[c], 0, FAKE_PTR, cfg.num_blocks, FAKE_PTR)
    loop = K.KvLoop()
    try:
        steps = []
        for t in range(150):
            ring.appends(t)
            if t >= 1:
                ring.replicate(t)
            ev = sched[0].steps[t]
            app = [dict(pool=hs[c], begin_step=1, release=ev.retire,
                        req_ids=sorted(ev.decode) + [r for r, _ in ev.admit],
                        n_new=[1] * len(ev.decode) + [pp for _, pp in ev.admit], src=None)
                   for c in ring.coords]
            steps.append(dict(append=app, repl_pools=[hs[c] for c in ring.coords] if t >= 1 else [],
                              step=t))
        loop.run(K.PreparedSteps(steps))
        for c in ring.coords:               # step 149's publication is still pending
            assert K.kv_stats(hs[c])["last_step"] == 148
        loop.flush()
        for c in ring.coords:
            assert _tables(hs[c], cfg.max_reqs) == ring.nodes[c].live()
            assert K.kv_stats(hs[c])["last_step"] == 149
            req, ln, pub, nb = K.kv_dump_slots(hs[c], cfg.max_reqs)
            assert (pub == ln).all()
        assert sum(K.kv_stats(hs[c])["bytes_replicated"] for c in ring.coords) == ring.moved
    finally:
        loop.destroy()
        for h in hs.values():
            K.kv_pool_destroy(h)


def test_loop_rejected_append_still_publishes_pending_step():
    """when the appends of step k are rejected (KV_ENOMEM, all-or-nothing),
    the publication of step k-1 that rides on the same launch still goes out, and the
    host state matches the sequential protocol (publish k-1, append k rejected)."""
    cfg = configs.scaled(configs.C1, num_blocks=6, max_reqs=4, max_blocks_per_req=8)
    a = _pool(cfg, 0)
    K.kv_set_successor(a, 1, FAKE_PTR, cfg.num_blocks, FAKE_PTR)
    loop = K.KvLoop()
    try:
        ok = [dict(append=[dict(pool=a, begin_step=1, release=[], req_ids=[7], n_new=[40],
                                src=None)], repl_pools=[a], step=1)]
        loop.run(K.PreparedSteps(ok))                      # 3 blocks; step 1 pending
        assert K.kv_stats(a)["last_step"] == 0
        big = [dict(append=[dict(pool=a, begin_step=1, release=[], req_ids=[8], n_new=[60],
                                 src=None)], repl_pools=[a], step=2)]
        with pytest.raises(K.KvError) as e:                # needs 4 blocks, 3 free
            loop.run(K.PreparedSteps(big))
        assert e.value.code == K.KV_ENOMEM
        st = K.kv_stats(a)
        assert st["last_step"] == 1                        # step 1 was published anyway
        assert st["bytes_replicated"] == 40 * 2 * 2 * 8 * 128 * 2
        assert _tables(a, cfg.max_reqs) == {7: (0, 40, [0, 1, 2])}
        req, ln, pub, nb = K.kv_dump_slots(a, cfg.max_reqs)
        assert pub[0] == 40
        loop.flush()                                       # nothing pending: no-op
        assert K.kv_stats(a)["last_step"] == 1
    finally:
        loop.destroy()
        K.kv_pool_destroy(a)


@pytest.mark.parametrize("seed,nb,mode", [(0, 32, "tokens"), (1, 28, "tokens"), (3, 24, "tokens"),
                                          (0, 28, "blocks")])
def test_shared_capacity_tables_match_oracle(seed, nb, mode):
    """NEXT-3 (reading R17) on tables-only pools: the C++ allocator, eviction
    (oldest admission first), drops on growth and the held-replica census equal
    the oracle's step by step under memory pressure (stage ring, no failure); also
    combined with the block-granular mode (NEXT-2)."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_shared import _pressure_cfg, _sched
    cfg = _pressure_cfg(num_blocks=nb, fail_node=None, fail_step=None)
    sch = _sched(cfg, seed)
    ring = OracleRing(cfg, content=False, shared=True, schedules=sch, mode=mode)
    coords = ring.coords
    hs = {c: _pool(cfg, k) for k, c in enumerate(coords)}
    S = cfg.stages
    for c in coords:
        if mode == "blocks":
            K.kv_set_mode(hs[c], K.KV_MODE_BLOCKS)
        K.kv_set_successor_shared(hs[c], hs[(c[0], (c[1] + 1) % S)])
    try:
        for t in range(cfg.n_steps):
            ring.appends(t)
            for c in coords:       # one call per node, node order (the harness protocol)
                ev = sch[c[0]].steps[t]
                K.kv_append_multi([dict(pool=hs[c], begin_step=1, release=ev.retire,
                                        req_ids=sorted(ev.decode) + [r for r, _ in ev.admit],
                                        n_new=[1] * len(ev.decode) + [pp for _, pp in ev.admit],
                                        src=None)])
            if t >= 1:
                ring.replicate(t)
                for c in coords:
                    K.kv_replicate_step(hs[c], t)
            for c in coords:
                n = ring.nodes[c]
                st = K.kv_stats(hs[c])
                assert _tables(hs[c], cfg.max_reqs) == n.live(), (t, c)
                assert st["free_blocks"] == len(n.free_blocks), (t, c)
                assert st["quarantined_blocks"] == len(n.q_blocks), (t, c)
                assert st["replica_evictions"] == n.evictions, (t, c)
                assert st["replica_drops"] == n.drops, (t, c)
                assert st["replica_blocks_held"] == n.rep_src.census(), (t, c)
        assert sum(n.evictions for n in ring.nodes.values()) > 0
        if mode == "tokens":
            assert sum(n.drops for n in ring.nodes.values()) > 0
    finally:
        for h in hs.values():
            K.kv_pool_destroy(h)


def test_decode_loop_argument_errors():
    """The one-launch loop rejects shared-capacity pools (they need kv_run_steps'
    append-after-previous-publication order) before touching any pool; a pool can be
    pending in one loop only."""
    cfg = configs.scaled(configs.C1, num_blocks=16, max_reqs=4, max_blocks_per_req=4)
    a, b = _pool(cfg, 0), _pool(cfg, 1)
    l1, l2 = K.KvLoop(), K.KvLoop()
    try:
        K.kv_set_successor(a, 1, FAKE_PTR, cfg.num_blocks, FAKE_PTR)
        step = [dict(append=[dict(pool=a, begin_step=1, release=[], req_ids=[1], n_new=[3],
                                  src=None)], repl_pools=[a], step=1)]
        l1.run(K.PreparedSteps(step))
        step2 = [dict(append=[], repl_pools=[a], step=2)]
        with pytest.raises(K.KvError) as e:
            l2.run(K.PreparedSteps(step2))
        assert e.value.code == K.KV_ESTATE
        l1.flush()
        assert K.kv_stats(a)["last_step"] == 1
        K.kv_set_successor_shared(a, b)
        with pytest.raises(K.KvError) as e:
            l1.run(K.PreparedSteps([dict(append=[dict(pool=a, begin_step=1, release=[],
                                                      req_ids=[2], n_new=[3], src=None)],
                                         repl_pools=[a], step=2)]))
        assert e.value.code == K.KV_EINVAL
        assert set(_tables(a, cfg.max_reqs)) == {1}
    finally:
        l1.destroy()
        l2.destroy()
        K.kv_pool_destroy(a)
        K.kv_pool_destroy(b)


def test_last_alloc_and_mirror_arguments():
    """kv_last_alloc lists the block ids the last append allocated, in allocation order
    (what an owner forwards to a remote holder's mirror, NEXT-3 across GPUs); a mirror
    needs a device and an unused pool; kv_mirror_blocks only takes a mirror."""
    cfg = configs.scaled(configs.C1, num_blocks=16, max_reqs=4, max_blocks_per_req=8)
    h = _pool(cfg, 0)
    try:
        K.kv_append(h, [1, 2], [20, 40], None)                  # 2 + 3 blocks, lowest first
        assert K.kv_last_alloc(h) == [0, 1, 2, 3, 4]
        assert K.kv_query(h, 1)[1] + K.kv_query(h, 2)[1] == [0, 1, 2, 3, 4]
        K.kv_append(h, [1, 2], [13, 1], None)                   # 20+13 = 33 -> one more block
        assert K.kv_last_alloc(h) == [5]
        K.kv_append(h, [2], [1], None)                          # no new block
        assert K.kv_last_alloc(h) == []
        with pytest.raises(K.KvError) as e:
            K.kv_pool_set_mirror(h, True)                        # tables-only pool: no device
        assert e.value.code == K.KV_EINVAL
        with pytest.raises(K.KvError) as e:
            K.kv_mirror_blocks(h, [1, 2])                        # not a mirror
        assert e.value.code == K.KV_EINVAL
    finally:
        K.kv_pool_destroy(h)
