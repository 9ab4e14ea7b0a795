"""GPU parity: the CUDA path (libkvring through its C ABI) equals the CPU
oracle byte for byte -- whole pools, whole replica regions, metadata, tables --
on the same seeded inputs.  All work is copying, so the bar
is bit-exact (north_star: "bit-exact replicas and restores")."""
import numpy as np
import pytest
import torch

from kvgen import configs
from kvgen.content import CONTENT_SEED, content_tokens
from kvgen.schedule import closed_loop_schedule
from oracle.simulate import OracleRing

pytestmark = pytest.mark.gpu

from gpu_harness import compare_state, make_gpu  # noqa: E402


def _run_both(cfg, ring="stage", schedules=None, every=1, fail=True, restore_mode=None,
              copy_engine=False, shared=False):
    rt, drv = make_gpu(cfg, ring=ring, schedules=schedules, restore_mode=restore_mode,
                       shared=shared)
    rt.copy_engine = copy_engine
    oring = OracleRing(cfg, ring=ring, schedules=drv.sched, restore_mode=restore_mode,
                       shared=shared)
    try:
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if fail and cfg.fail_step == t:
                drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
            if t >= 1:
                drv.rt.replicate_all(t)
                oring.replicate(t)
            if every and (t % every == 0 or t == cfg.n_steps - 1):
                compare_state(rt, drv, oring, tag=f"step {t}")
        return rt, drv, oring
    except Exception:
        rt.destroy()
        raise


def test_c1_bit_exact_every_step():
    rt, drv, oring = _run_both(configs.C1)
    try:
        ev = drv.events[0].data
        assert ev["t_star"] == 4 and ev["restored"] == [(r, 68) for r in range(4)]
        from paper_2601_22438_b200 import kvring as K
        assert [K.kv_query(rt.handle(ev["dst"]), r)[1] for r in range(4)] == \
            [[5 * r + k for k in range(5)] for r in range(4)]
    finally:
        rt.destroy()


def _churn_sched(cfg, seed):
    rng = np.random.default_rng(seed)
    p = rng.integers(1, 70, size=cfg.n_requests)
    o = rng.integers(1, 30, size=cfg.n_requests)
    return [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap, pipeline=i)
            for i in range(cfg.pipelines)]


@pytest.mark.parametrize("seed", [0, 1])
def test_churn_with_failure_bit_exact(seed):
    cfg = configs.scaled(configs.C1, num_blocks=96, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=40, fixed_prompt=None,
                         fail_node=(0, 1), fail_step=23)
    rt, drv, oring = _run_both(cfg, schedules=_churn_sched(cfg, seed))
    rt.destroy()


def test_promotion_instance_ring_bit_exact():
    cfg = configs.scaled(configs.C1, pipelines=2, num_blocks=128, max_reqs=16,
                         max_blocks_per_req=12, batch_cap=4, n_requests=40, n_steps=30,
                         fixed_prompt=None, fail_node=(0, 2), fail_step=17, ring="instance")
    rt, drv, oring = _run_both(cfg, ring="instance", schedules=_churn_sched(cfg, 5))
    try:
        assert drv.events[0].data["dst"] == drv.coords[(1, 2)]   # promoted into the holder
    finally:
        rt.destroy()


def test_ragged_geometry_and_big_prefill():
    # L_s = 3, B = 8 (tasks cut mid-block), a 700-token prefill, ragged tails
    cfg = configs.scaled(configs.C1, geom=configs.Geometry(layers=3, block_size=8),
                         num_blocks=400, max_reqs=8, max_blocks_per_req=120, batch_cap=3,
                         n_requests=10, n_steps=12, fixed_prompt=None, fail_node=(0, 3),
                         fail_step=7)
    p = np.array([700, 1, 9, 17, 33, 64, 5, 8, 100, 2])
    o = np.array([20, 3, 1, 6, 2, 9, 4, 4, 4, 4])
    sched = [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap)]
    rt, drv, oring = _run_both(cfg, schedules=sched)
    rt.destroy()


@pytest.mark.parametrize("heads,head_dim,block", [(4, 64, 16), (2, 256, 32), (1, 8, 4)])
def test_other_head_geometries_bit_exact(heads, head_dim, block):
    """Slice sizes other than 256 B (128 B, 512 B, 16 B: other 16-B chunk counts per
    slice), other KV-head counts and block sizes, through churn and a failure."""
    cfg = configs.scaled(configs.C1, geom=configs.Geometry(layers=2, kv_heads=heads,
                                                           head_dim=head_dim,
                                                           block_size=block),
                         num_blocks=600 if block == 4 else 160, max_reqs=12,
                         max_blocks_per_req=64 if block == 4 else 16, batch_cap=5,
                         n_requests=40, n_steps=24, fixed_prompt=None, fail_node=(0, 2),
                         fail_step=15)
    rt, drv, oring = _run_both(cfg, schedules=_churn_sched(cfg, 9))
    rt.destroy()


@pytest.mark.parametrize("loop", ["direct", "loop"])
def test_abort_mid_step_keeps_last_published_replica(loop):
    """A stage dying mid-replicate leaves its successor's replica at the last
    published step (R7/R9): restore == oracle restore of the previous step.  loop:
    the steps run through the one-launch-per-step loop (kv_loop_*), the aborted
    publication being the pending one launched by kv_loop_flush."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, num_blocks=96, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=30, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    sched = _churn_sched(cfg, 11)
    rt, drv = make_gpu(cfg, schedules=sched)
    keep = []

    def loop_run(kl, t0, t1):
        sts = []
        for t in range(t0, t1):
            app = []
            for node, e in drv.plan(t).items():
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                src = drv.content(e["stage"], ids, pos) if ids else None
                keep.append(src)
                app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=src))
            pools = [rt.handle(n) for n in rt.alive_local()]
            sts.append(dict(append=app, repl_pools=pools if t >= 1 else [], step=t))
        kl.run(K.PreparedSteps(sts), torch.cuda.current_stream().cuda_stream)

    try:
        T = 20
        if loop == "loop":
            kl = K.KvLoop()
            loop_run(kl, 0, T)                                    # step T-1 pending
            K.kv_inject_abort(rt.handle(drv.coords[(0, 1)]), 300)  # 300 slices, no publish
            kl.flush(torch.cuda.current_stream().cuda_stream)
            kl.destroy()
        else:
            for t in range(T):
                drv.append_step(t)
                if t >= 1:
                    if t == T - 1:
                        K.kv_inject_abort(rt.handle(drv.coords[(0, 1)]), 300)   # no publish
                    rt.replicate_all(t)
        torch.cuda.synchronize()
        holder = drv.coords[(0, 2)]
        meta = rt.read_meta(holder)
        assert meta["seq"] == T - 2                           # stage 1's step T-1 never published
        # restore from the holder == the oracle's published state at T-2
        oref = OracleRing(cfg, schedules=sched)
        for t in range(T - 1):
            oref.appends(t)
            if t >= 1:
                oref.replicate(t)
        pub = oref.nodes[(0, 2)].published()
        f = drv.coords[(0, 1)]
        rt.fail(f)
        dst = drv.next_node
        rt.new_node(dst, 0)
        t_star, restored = rt.restore(dst, holder)
        assert t_star == T - 2
        assert restored == sorted((r, ln) for r, (s, ln, bt) in pub.items())
        torch.cuda.synchronize()
        g = cfg.geom
        pool = rt.local[dst].pool.cpu().numpy().view(np.uint16)
        for r, ln in restored:
            _, bt = K.kv_query(rt.handle(dst), r)
            want = content_tokens(CONTENT_SEED, [r] * ln, range(ln), 1 * g.layers, g.layers,
                                  g.kv_heads, g.head_dim)
            for pos in range(ln):
                assert np.array_equal(pool[bt[pos // 16], :, :, :, pos % 16], want[pos]), (r, pos)
    finally:
        rt.destroy()


def test_host_source_append_equals_device_source():
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, stages=2, n_steps=1)
    rt, drv = make_gpu(cfg)
    try:
        g = cfg.geom
        src = content_tokens(CONTENT_SEED, [1] * 70 + [2] * 33, list(range(70)) + list(range(33)),
                             0, g.layers, g.kv_heads, g.head_dim)
        host = torch.from_numpy(src.view(np.int16)).pin_memory()
        dev = host.cuda()
        K.kv_append(rt.handle(0), [1, 2], [70, 33], dev)
        K.kv_append(rt.handle(1), [1, 2], [70, 33], host, flags=K.KV_SRC_HOST)
        torch.cuda.synchronize()
        assert torch.equal(rt.local[0].pool, rt.local[1].pool)
    finally:
        rt.destroy()


def test_pack_unpack_equals_ring_put():
    """NCCL-comparison path (gather-pack -> buffer -> unpack) == fused ring-put, byte for byte."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, num_blocks=96, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=25, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    sched = _churn_sched(cfg, 3)
    rt, drv = make_gpu(cfg, schedules=sched, spares=1)
    try:
        # node 0 -> node 1 by ring-put; a shadow copy of node 0's stream via pack/unpack
        shadow = rt.slots[4]
        shadow.meta.fill_(255)   # a spare slot has no pool handle: its bt rows start at -1
        buf = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        n0 = rt.handle(0)
        for t in range(cfg.n_steps):
            drv.append_step(t)
            if t >= 1:
                nodes = [n for n in rt.alive_local() if n != 0]
                rt.replicate_all(t, nodes=nodes)
                need = K.kv_pack_bytes(n0)
                used = K.kv_pack_step(n0, t, buf, buf.numel())
                assert used == need
                K.kv_unpack(buf, used, shadow.replica, rt.NB, shadow.meta, rt.kg, rt.R, rt.M)
        torch.cuda.synchronize()
        # rebuild the ring-put result: replay with plain ring-put from scratch
        rt2, drv2 = make_gpu(cfg, schedules=sched)
        for t in range(cfg.n_steps):
            drv2.append_step(t)
            if t >= 1:
                rt2.replicate_all(t)
        torch.cuda.synchronize()
        assert torch.equal(shadow.replica, rt2.local[1].replica)
        m1 = rt2.read_meta(1)
        raw = shadow.meta.cpu().numpy()
        R, M = rt.R, rt.M
        assert int(raw[0:8].view(np.uint64)[0]) == m1["seq"] == cfg.n_steps - 1
        assert np.array_equal(raw[32:32 + 16 * R].view(np.int64).reshape(2, R), m1["req"])
        assert np.array_equal(raw[32 + 16 * R:32 + 24 * R].view(np.int32).reshape(2, R), m1["len"])
        assert np.array_equal(raw[32 + 24 * R:32 + 24 * R + 4 * R * M].view(np.int32).reshape(R, M),
                              m1["bt"])
        rt2.destroy()
    finally:
        rt.destroy()


def test_c2_full_size_sampled():
    """C2 at full size on one GPU (4 pools, the bench launch configuration):
    tables and device metadata == oracle (metadata mode) every 25 steps;
    sampled valid slots of every primary and replica == closed form."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.C2
    steps = 260
    rt, drv = make_gpu(cfg)
    oring = OracleRing(cfg, content=False, schedules=drv.sched)
    rng = np.random.default_rng(7)
    g = cfg.geom
    try:
        for t in range(steps):
            drv.append_step(t)
            oring.appends(t)
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            if t % 25 == 0 or t == steps - 1:
                compare_state(rt, drv, oring, content=False, tag=f"step {t}")
        torch.cuda.synchronize()
        for c, gid in drv.coords.items():
            on = oring.nodes[c]
            succ = rt.succ[gid]
            live = on.live()
            items = [(r, pos, bt[pos // 16]) for r, (s, ln, bt) in live.items()
                     for pos in rng.choice(ln, size=min(ln, 3), replace=False)]
            want = content_tokens(CONTENT_SEED, [i[0] for i in items], [i[1] for i in items],
                                  c[1] * g.layers, g.layers, g.kv_heads, g.head_dim)
            idx = torch.tensor([i[2] for i in items], device="cuda")
            slot = torch.tensor([i[1] % 16 for i in items], device="cuda")
            prim = rt.local[gid].pool[idx, :, :, :, slot].cpu().numpy().view(np.uint16)
            rep = rt.local[succ].replica[idx, :, :, :, slot].cpu().numpy().view(np.uint16)
            assert np.array_equal(prim, want)
            assert np.array_equal(rep, want)
    finally:
        rt.destroy()


@pytest.mark.parametrize("shared", [False, True])
def test_run_steps_two_streams_bit_exact(shared):
    """kv_run_steps (the native decode loop the bench times: append on one stream,
    publish on a second stream after an event) == oracle, whole arrays; shared:
    the NEXT-3 shared-capacity links under memory pressure (evictions + drops)."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, num_blocks=28 if shared else 96, max_reqs=12,
                         max_blocks_per_req=12, batch_cap=5 if shared else 6, n_requests=60,
                         n_steps=40 if shared else 30, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    sched = _churn_sched(cfg, 1 if shared else 21)
    rt, drv = make_gpu(cfg, schedules=sched, shared=shared)
    oring = OracleRing(cfg, schedules=sched, shared=shared)
    try:
        comp = torch.cuda.current_stream()
        repl = torch.cuda.Stream()
        steps, keep = [], []
        for t in range(cfg.n_steps):
            app = []
            for node, e in drv.plan(t).items():
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                src = drv.content(e["stage"], ids, pos) if ids else None
                keep.append(src)
                app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=src))
            pools = [rt.handle(n) for n in rt.alive_local()] if t >= 1 else []
            steps.append(dict(append=app, repl_pools=pools, step=t))
            oring.appends(t)
            if t >= 1:
                oring.replicate(t)
        prep = K.PreparedSteps(steps)
        torch.cuda.synchronize()
        K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
        torch.cuda.synchronize()
        compare_state(rt, drv, oring, tag="run_steps")
        if shared:
            assert sum(n.evictions for n in oring.nodes.values()) > 0
            assert sum(n.drops for n in oring.nodes.values()) > 0
            kl = K.KvLoop()
            with pytest.raises(K.KvError):     # the one-launch loop refuses shared pools
                kl.run(K.PreparedSteps(steps[:1]), comp.cuda_stream)
            kl.destroy()
    finally:
        rt.destroy()


def test_nccl_loopback_transport_bit_exact():
    """The comparison transport at world size 1 (pack -> unpack into the local
    successor) keeps every replica == oracle, whole arrays."""
    from paper_2601_22438_b200.nccl_compare import NcclRing
    cfg = configs.scaled(configs.C1, num_blocks=96, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=25, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    sched = _churn_sched(cfg, 9)
    rt, drv = make_gpu(cfg, schedules=sched)
    oring = OracleRing(cfg, schedules=sched)
    ring = NcclRing(rt, 32 << 20)
    try:
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if t >= 1:
                ring.step(t)
                oring.replicate(t)
            if t % 6 == 0:
                compare_state(rt, drv, oring, tag=f"nccl-loopback {t}")
        compare_state(rt, drv, oring, tag="nccl-loopback end")
    finally:
        rt.destroy()


def test_reprotect_after_promotion_bit_exact():
    """NEXT-1: paper ring, (0,2) fails and is promoted onto (1,2); the failed node and
    the rerouting donor are excluded, (3,2) is re-targeted to (2,2) and
    re-seeded; every array stays == oracle for the rest of the run."""
    cfg = configs.scaled(configs.C1, pipelines=4, num_blocks=128, max_reqs=16,
                         max_blocks_per_req=12, batch_cap=3, n_requests=40, n_steps=34,
                         fixed_prompt=None, fail_node=(0, 2), fail_step=15, ring="instance")
    sched = _churn_sched(cfg, 17)
    rt, drv = make_gpu(cfg, ring="instance", schedules=sched)
    oring = OracleRing(cfg, ring="instance", schedules=sched)
    try:
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if t == cfg.fail_step:
                drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
                plan_g = drv.reprotect([(0, 2), (1, 2)])
                plan_o = oring.reprotect([(0, 2), (1, 2)])
                assert {c: plan_g[c] for c in plan_o} == plan_o
                assert plan_g[(3, 2)] == (2, 2)
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            if t % 3 == 0 or t >= cfg.fail_step:
                compare_state(rt, drv, oring, tag=f"reprotect step {t}")
    finally:
        rt.destroy()


@pytest.mark.parametrize("seed,shared", [(2, False), (3, False), (0, True)])
def test_block_mode_with_failure_bit_exact(seed, shared):
    """NEXT-2 block-granular mode (completed blocks only): whole arrays == oracle,
    including a failure, a restore at a block boundary and the resume; shared: combined
    with shared-capacity replicas under pressure (NEXT-3)."""
    cfg = configs.scaled(configs.C1, num_blocks=28 if shared else 96, max_reqs=12,
                         max_blocks_per_req=12, batch_cap=5 if shared else 6, n_requests=60,
                         n_steps=40, fixed_prompt=None, fail_node=(0, 1), fail_step=26)
    sched = _churn_sched(cfg, seed)
    rt, drv = make_gpu(cfg, schedules=sched, mode="blocks", shared=shared)
    oring = OracleRing(cfg, schedules=sched, mode="blocks", shared=shared)
    try:
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if cfg.fail_step == t:
                drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            if t % 2 == 0 or t >= cfg.fail_step:
                compare_state(rt, drv, oring, tag=f"blocks step {t}")
        assert all(ln % 16 == 0 for _, ln in drv.events[0].data["restored"])
    finally:
        rt.destroy()


def test_restore_errors_and_edge_cases():
    """KV_ENOREPLICA for a holder that published nothing (seq 0) or whose memory is
    poisoned (seq all-ones); KV_ENOMEM (all-or-nothing) for a too-small target;
    empty and zero-token appends; publish-only steps keep seq moving."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, stages=3, n_steps=1)
    rt, drv = make_gpu(cfg, spares=2)
    try:
        h0, h1, h2 = rt.handle(0), rt.handle(1), rt.handle(2)
        # nothing published yet: node 1 holds node 0's (empty) replica with seq 0
        with pytest.raises(K.KvError) as e:
            rt.restore(2, 1)
        assert e.value.code == K.KV_ENOREPLICA
        g = cfg.geom
        src = torch.from_numpy(content_tokens(CONTENT_SEED, [5] * 40, range(40), 0, g.layers,
                                              g.kv_heads, g.head_dim).view(np.int16)).cuda()
        K.kv_append(h0, [], [], None)                       # empty append: no-op
        K.kv_append(h0, [5], [40], src)
        K.kv_append(h0, [5], [0], None)                     # zero tokens for a live request
        assert K.kv_query(h0, 5) == (40, [0, 1, 2])
        K.kv_replicate_step(h0, 1)
        K.kv_replicate_step(h0, 2)                          # nothing dirty: publish-only
        torch.cuda.synchronize()
        assert rt.read_meta(1)["seq"] == 2
        # restore into a pool too small for the 3 blocks: all-or-nothing ENOMEM
        small = K.kv_pool_create(K.kv_pool_desc_t(rt.kg, 2, 4, 8, 0, 99, 2,
                                                  rt.slots[3].pool.data_ptr(),
                                                  rt.slots[3].replica.data_ptr(),
                                                  rt.slots[3].meta.data_ptr()))
        with pytest.raises(K.KvError) as e:
            K.kv_restore(small, rt.replica_ptr(1), rt.NB, rt.meta_ptr(1))
        assert e.value.code == K.KV_ENOMEM
        assert K.kv_stats(small)["live_reqs"] == 0 and K.kv_stats(small)["free_blocks"] == 2
        K.kv_pool_destroy(small)
        # a poisoned holder (its memory is lost): ENOREPLICA
        rt.fail(1)
        torch.cuda.synchronize()
        with pytest.raises(K.KvError) as e:
            K.kv_restore(h2, rt.replica_ptr(1), rt.NB, rt.meta_ptr(1))
        assert e.value.code == K.KV_ENOREPLICA
        with pytest.raises(K.KvError) as e:
            K.kv_append(h0, [5], [1], src)                   # h0 still alive: fine ...
            K.kv_replicate_step(rt.handle(1), 3)            # ... but the dead pool refuses
        assert e.value.code == K.KV_ESTATE
    finally:
        rt.destroy()


def _loop_steps(rt, drv, t0, t1, keep):
    from paper_2601_22438_b200 import kvring as K
    sts = []
    for t in range(t0, t1):
        app = []
        for node, e in drv.plan(t).items():
            if node not in rt.local:
                continue
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            src = drv.content(e["stage"], ids, pos) if ids else None
            keep.append(src)
            app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                            req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        pools = [rt.handle(n) for n in rt.alive_local() if rt.succ.get(n) is not None]
        sts.append(dict(append=app, repl_pools=pools if t >= 1 else [], step=t))
    return K.PreparedSteps(sts)


@pytest.mark.parametrize("n_steps,fail,every", [(6, False, 0), (40, False, 7), (41, True, 0),
                                                (33, True, 5)])
def test_loop_bit_exact(n_steps, fail, every):
    """The one-launch-per-step loop (kv_loop_step: appends of step k + the publication
    of step k-1 in ONE kernel, per-step calls, no lookahead) == oracle, whole arrays,
    churn.  `every`: flush and compare every few steps.  With `fail` a stage fails after
    the appends of step 19 while step 19's publication is pending: fail, restore and
    relink run between two kv_loop_step calls and the pending publication follows the
    sequential protocol (dead pool dropped, predecessor re-seeded into the fresh pool,
    which publishes step 19 itself)."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, num_blocks=96, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=n_steps, fixed_prompt=None,
                         fail_node=(0, 2) if fail else None, fail_step=19 if fail else None)
    sched = _churn_sched(cfg, 33)
    rt, drv = make_gpu(cfg, schedules=sched)
    oring = OracleRing(cfg, schedules=sched)
    st = torch.cuda.current_stream().cuda_stream
    kl = K.KvLoop()
    keep = []
    try:
        for t in range(n_steps):
            prep = _loop_steps(rt, drv, t, t + 1, keep)
            kl.step(prep, 0, st)
            oring.appends(t)
            if fail and t == cfg.fail_step:
                dst, _ = drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
                # the fresh pool is not in the loop's pending list: it publishes step t
                # directly, like every alive linked node of the sequential protocol
                rt.replicate_all(t, nodes=[dst])
            if t >= 1:
                oring.replicate(t)
            if every and t % every == every - 1:
                kl.flush(st)
                torch.cuda.synchronize()
                compare_state(rt, drv, oring, tag=f"loop step {t}")
        kl.flush(st)
        torch.cuda.synchronize()
        compare_state(rt, drv, oring, tag="loop end")
    finally:
        kl.destroy()
        rt.destroy()


@pytest.mark.parametrize("n_steps", [12, 90])
def test_loop_batched_run_bit_exact(n_steps):
    """kv_loop_run (the bench's native loop over marshalled steps) == oracle; the
    pending publication survives between two calls."""
    from paper_2601_22438_b200 import kvring as K
    cfg = configs.scaled(configs.C1, num_blocks=160, max_reqs=16, max_blocks_per_req=12,
                         batch_cap=8, n_requests=200, n_steps=n_steps, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    sched = _churn_sched(cfg, 41)
    rt, drv = make_gpu(cfg, schedules=sched)
    oring = OracleRing(cfg, schedules=sched)
    kl = K.KvLoop()
    keep = []
    try:
        for t in range(n_steps):
            oring.appends(t)
            if t >= 1:
                oring.replicate(t)
        half = n_steps // 2
        st = torch.cuda.current_stream().cuda_stream
        kl.run(_loop_steps(rt, drv, 0, half, keep), st)
        kl.run(_loop_steps(rt, drv, half, n_steps, keep), st)
        kl.flush(st)
        torch.cuda.synchronize()
        compare_state(rt, drv, oring, tag="loop run")
    finally:
        kl.destroy()
        rt.destroy()


def test_self_loop_ring_and_max_length_requests():
    """Degenerate cases: a one-stage ring (the pool's successor is itself, so it
    replicates into its own replica region) and requests that fill exactly
    max_blocks_per_req blocks (one more token is KV_ENOMEM, all-or-nothing)."""
    from paper_2601_22438_b200 import kvring as K
    M = 6
    cfg = configs.scaled(configs.C1, stages=1, num_blocks=40, max_reqs=8, max_blocks_per_req=M,
                         batch_cap=3, n_requests=6, n_steps=20, fixed_prompt=None,
                         fail_node=None, fail_step=None)
    p = np.array([M * 16 - 8, 5, M * 16 - 12, 17, 30, 2])
    o = np.array([8, 30, 12, 3, 5, 9])              # requests 0 and 2 end at exactly M blocks
    sched = [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap)]
    rt, drv = make_gpu(cfg, schedules=sched)
    oring = OracleRing(cfg, schedules=sched)
    try:
        assert rt.succ[0] == 0
        lens = []
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            compare_state(rt, drv, oring, tag=f"self-loop {t}")
            lens.extend(ln for _, ln, _ in oring.nodes[(0, 0)].live().values())
        assert max(lens) == M * 16
        h = rt.handle(0)
        live = oring.nodes[(0, 0)].live()
        full = [r for r, (_, ln, _) in live.items() if ln == M * 16]
        if full:
            with pytest.raises(K.KvError) as e:
                K.kv_append(h, [full[0]], [1], torch.zeros(1, 2, 2, 8, 128, dtype=torch.int16,
                                                           device="cuda"))
            assert e.value.code == K.KV_ENOMEM
    finally:
        rt.destroy()


@pytest.mark.parametrize("seed", [0, 4])
def test_copy_engine_variant_bit_exact(seed):
    """NEXT-4: full blocks by cudaMemcpyAsync runs, partial blocks + bt entries +
    publication by the ring-put kernel -- same replicas and metadata as the oracle,
    through churn (prefills of many full blocks, retire/admit) and a restore."""
    cfg = configs.scaled(configs.C1, num_blocks=160, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=6, n_requests=60, n_steps=40, fixed_prompt=None,
                         fail_node=(0, 2), fail_step=21)
    rt, drv, oring = _run_both(cfg, schedules=_churn_sched(cfg, seed), copy_engine=True)
    rt.destroy()


# (seed, ring, restore, blocks, batch cap, slots): evictions AND drops occur (oracle pins)
SHARED_PRESSURE = [(0, "stage", "fresh", 32, 5, 12), (1, "stage", "fresh", 28, 5, 12),
                   (4, "instance", "promote", 48, 5, 24)]


@pytest.mark.parametrize("seed,ring,restore_mode,nb,cap,slots", SHARED_PRESSURE)
def test_shared_capacity_pressure_bit_exact(seed, ring, restore_mode, nb, cap, slots):
    """NEXT-3 (reading R17): replicas in the holder's own pool, evicted oldest-first
    when the holder's appends need the memory, dropped when they cannot grow; a
    failure restored from the shared holder (fresh pool, or promotion onto the
    holder).  Whole pools, metadata, tables, evictions, drops and census == oracle
    at every step."""
    cfg = configs.scaled(configs.C1, num_blocks=nb, max_reqs=slots, max_blocks_per_req=12,
                         batch_cap=cap, n_requests=60, n_steps=40, fixed_prompt=None,
                         pipelines=2 if ring == "instance" else 1, ring=ring,
                         fail_node=(0, 2) if ring == "instance" else (0, 1), fail_step=23)
    rt, drv, oring = _run_both(cfg, ring=ring, schedules=_churn_sched(cfg, seed),
                               restore_mode=restore_mode, shared=True)
    try:
        assert sum(n.evictions for n in oring.all_nodes()) > 0
        assert sum(n.drops for n in oring.all_nodes()) > 0
    finally:
        rt.destroy()
