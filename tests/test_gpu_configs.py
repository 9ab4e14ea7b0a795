"""GPU parity on the BASELINE workloads at (near) full scale on one B200:
C3 (Poisson arrivals, two pipelines), C4 (16 logical nodes, batch 128, failure
of (0,2) at step 300 and restore -- stage ring into a fresh pool, and the
paper's instance ring with promotion onto the holder), C5 (32k-token prefill
per stage: bulk full-block replication and a bulk restore).  Tables and device
metadata are compared with the oracle in metadata mode; EVERY valid KV slot of every
primary and replica is checked against the closed form on the GPU (the full arrays do
not fit the oracle's host memory), and blocks above the run's high-water id must still
hold the sentinel.  Pools are sized to the workload's peak block use
(measured with the oracle), not the 6-12 GiB worst case."""
import numpy as np
import pytest
import torch

from kvgen import configs
from kvgen.content import CONTENT_SEED, content_tokens
from oracle.simulate import OracleRing

from gpu_harness import compare_state, make_gpu, node_map

pytestmark = pytest.mark.gpu


def _gather_positions(arr, bt_of_pos, B, items, dev):
    """arr[bt[pos // B], :, :, :, pos % B, :] for items (req, pos) -> [n][L][2][H][d]."""
    blk = torch.tensor([bt_of_pos[i] for i in range(len(items))], device=dev)
    slot = torch.tensor([p % B for _, p in items], device=dev)
    return arr[blk, :, :, :, slot]


def _full_check(rt, drv, oring, hw, chunk=1 << 16):
    """Every valid slot of every live node's primary AND of its successor's replica (at
    the published length) equals the closed-form content (I2, I1 through the closed form;
    the expected words come from kvgen's CUDA twin of the numpy generator, pinned byte for
    byte by tests/test_kvgen_cuda.py); every block at or above the run's high-water block
    id still holds the sentinel in every pool and replica region (I5: no stray writes).
    Tables come from the oracle (metadata mode), independent of the GPU path."""
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200.runtime import SENTINEL_WORD
    torch.cuda.synchronize()
    g = rt.g
    B = g.block_size
    nm = node_map(rt, drv, oring)
    inv = {n: c for c, n in drv.serving.items()}
    checked = 0
    for gid, on in nm.items():
        if on.dead or gid not in inv or gid not in rt.local:
            continue
        stage = inv[gid][1]
        targets = [("primary", rt.local[gid].pool, on.live())]
        succ = rt.succ.get(gid)
        if succ is not None and succ in rt.local and on.succ is not None and not on.succ.dead:
            pub = on.succ.published()
            targets.append(("replica", rt.local[succ].replica, pub))
        for name, arr, table in targets:
            items, bts = [], []
            for r, (s, ln, bt) in sorted(table.items()):
                for pos in range(ln):
                    items.append((r, pos))
                    bts.append(bt[pos // B])
            for c0 in range(0, len(items), chunk):
                it = items[c0:c0 + chunk]
                want = content_tokens_cuda(CONTENT_SEED, [x[0] for x in it], [x[1] for x in it],
                                           stage * g.layers, g.layers, g.kv_heads, g.head_dim,
                                           device=rt.device)
                got = _gather_positions(arr, bts[c0:c0 + chunk], B, it, rt.dev)
                if not torch.equal(got, want):
                    bad = (got != want).reshape(len(it), -1).any(1).nonzero()[:3].flatten().tolist()
                    raise AssertionError(f"node {gid} {name}: slots {[it[k] for k in bad]} differ")
                checked += len(it)
    w = SENTINEL_WORD if SENTINEL_WORD < 0x8000 else SENTINEL_WORD - 0x10000
    for gid, slot in rt.local.items():
        if gid in rt.dead:            # a failed node's memory is poisoned (a7)
            continue
        for name, arr in (("pool", slot.pool), ("replica", slot.replica)):
            if hw < arr.shape[0]:
                assert bool((arr[hw:] == w).all().item()), f"node {gid} {name}: stray write above block {hw}"
    return checked


def _high_water(oring):
    return max([b for n in oring.all_nodes() if not n.dead for s in range(n.R) for b in n.slot_bt[s]]
               + [-1]) + 1


def _run(cfg, steps, ring="stage", check_every=50, restore_mode=None, copy_engine=False):
    rt, drv = make_gpu(cfg, ring=ring, restore_mode=restore_mode)
    rt.copy_engine = copy_engine
    oring = OracleRing(cfg, content=False, ring=ring, schedules=drv.sched,
                       restore_mode=restore_mode)
    hw = 0
    try:
        for t in range(steps):
            drv.append_step(t)
            oring.appends(t)
            if cfg.fail_step == t:
                drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
                compare_state(rt, drv, oring, content=False, tag=f"after restore {t}")
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            if t % check_every == 0 or t == steps - 1:
                compare_state(rt, drv, oring, content=False, tag=f"step {t}")
            hw = max(hw, _high_water(oring))
            if cfg.fail_step == t:
                _full_check(rt, drv, oring, hw)      # right after the restore (I4)
        n = _full_check(rt, drv, oring, hw)          # the end of the run
        assert n > 0
        return rt, drv, oring
    except Exception:
        rt.destroy()
        raise


def test_c4_failover_stage_ring_fresh_restore():
    cfg = configs.scaled(configs.C4, num_blocks=4096, max_reqs=256)
    rt, drv, oring = _run(cfg, 320)
    try:
        ev = drv.events[0].data
        assert ev["t_star"] == 299 and len(ev["restored"]) == 128
        assert ev["restored"] == oring.events[0][4]
    finally:
        rt.destroy()


def test_c4_paper_ring_promotion_onto_holder():
    # the paper's ring: (0,2)'s replication target and replacement is (1,2)
    cfg = configs.scaled(configs.C4, pipelines=2, num_blocks=8192, max_reqs=512, ring="instance")
    rt, drv, oring = _run(cfg, 315, ring="instance")
    try:
        ev = drv.events[0].data
        assert ev["dst"] == drv.coords[(1, 2)] and len(ev["restored"]) == 128
    finally:
        rt.destroy()


def test_c3_poisson_two_pipelines():
    cfg = configs.scaled(configs.C3, rps=16.0, num_blocks=2048, max_reqs=256)
    rt, drv, oring = _run(cfg, 400, check_every=100)
    rt.destroy()


@pytest.mark.parametrize("copy_engine", [False, True])
def test_c5_bulk_replication_and_restore(copy_engine):
    """One 32,768-token request per stage: 2,048 full blocks of 256 KiB replicated in
    one step (bulk; kernel or copy-engine variant), then stage 3 fails and is restored
    from stage 4's replica."""
    from paper_2601_22438_b200 import kvring as K
    # step 0 admits the 32k prompt, step 1 appends one token and publishes the whole
    # request (bulk seed), step 2: stage 3 fails after its append -> t* = 1
    cfg = configs.scaled(configs.C5, n_steps=3, fixed_output=4, fail_node=(0, 3), fail_step=2,
                         max_reqs=2, num_blocks=2050, max_blocks_per_req=2050)
    rt, drv, oring = _run(cfg, 3, check_every=1, copy_engine=copy_engine)
    try:
        g = cfg.geom
        ev = drv.events[0].data
        assert ev["t_star"] == 1 and ev["restored"] == [(0, 32769)]
        for s in range(cfg.stages):
            n = drv.serving[(0, s)]
            assert K.kv_stats(rt.handle(n))["last_step"] == 2
        # the restored stage holds the request at fresh block ids 0..2048
        dst = ev["dst"]
        ln, bt = K.kv_query(rt.handle(dst), 0)
        assert ln == 32770 and bt == list(range(2049))
        pos = np.random.default_rng(1).choice(32770, 64, replace=False)
        want = content_tokens(CONTENT_SEED, [0] * 64, pos, 3 * g.layers, g.layers, g.kv_heads,
                              g.head_dim)
        idx = torch.tensor([bt[p // 16] for p in pos], device=rt.dev)
        sl = torch.tensor([p % 16 for p in pos], device=rt.dev)
        got = rt.local[dst].pool[idx, :, :, :, sl].cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want)
    finally:
        rt.destroy()


@pytest.mark.parametrize("loop", ["loop", "streams"])
def test_c2_full_geometry_whole_arrays(loop):
    """C2 at BASELINE's full geometry in the bench's launch configurations (4 pools of
    12,288 x 512 KiB blocks on one GPU; the one-launch-per-step kv_loop -- the bench
    default -- and kv_run_steps with two streams), 160 steps:
    whole pools, whole replica regions and metadata == the oracle in content mode.
    The oracle holds the first 2,048 blocks (lowest-free-id allocation gives the same
    block ids while use stays below that; asserted) and every GPU block beyond them
    must still hold the sentinel -- no stray write anywhere in 48 GiB."""
    from paper_2601_22438_b200 import kvring as K
    full = configs.C2
    steps = 160
    small = configs.scaled(full, num_blocks=2048)
    rt, drv = make_gpu(full)
    oring = OracleRing(small, schedules=drv.sched)
    try:
        comp = torch.cuda.current_stream()
        repl = torch.cuda.Stream()
        sts, keep = [], []
        for t in range(steps):
            app = []
            for node, e in drv.plan(t).items():
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                src = drv.content(e["stage"], ids, pos) if ids else None
                keep.append(src)
                app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=src))
            sts.append(dict(append=app, repl_pools=[rt.handle(n) for n in rt.alive_local()]
                            if t >= 1 else [], step=t))
            oring.appends(t)
            if t >= 1:
                oring.replicate(t)
        for n in oring.nodes.values():
            assert max([b for s in range(n.R) for b in n.slot_bt[s]] + [0]) < 2048
        K.kv_host_profile(reset=True)
        K.kv_launch_log(True)
        if loop == "loop":
            kl = K.KvLoop()
            kl.run(K.PreparedSteps(sts), comp.cuda_stream)
            kl.flush(comp.cuda_stream)
            kl.destroy()
        else:
            K.kv_run_steps(K.PreparedSteps(sts), comp.cuda_stream, repl.cuda_stream)
        torch.cuda.synchronize()
        log = K.kv_launch_log(False)
        # both descriptor paths ran: decode steps in the kernel parameter space,
        # prefill-heavy steps (the admissions of step 0) from a device copy
        assert any(r["blob_bytes"] <= 24576 for r in log) and \
            any(r["blob_bytes"] > 24576 for r in log), [r["blob_bytes"] for r in log[:4]]
        sentinel = np.int16(np.uint16(0x5A5A).view(np.int16))
        for c, gid in drv.coords.items():
            on = oring.nodes[c]
            slot = rt.local[gid]
            for name, dev_arr, ora in (("primary", slot.pool, on.primary),
                                       ("replica", slot.replica, on.replica)):
                head = dev_arr[:2048].cpu().numpy().view(np.uint16)
                assert np.array_equal(head, ora), f"{c} {name} differs"
                tail_ok = bool((dev_arr[2048:] == int(sentinel)).all().item())
                assert tail_ok, f"{c} {name}: a block beyond the used range was written"
            meta = rt.read_meta(gid)
            assert meta["seq"] == on.rseq
            assert np.array_equal(meta["req"], on.rreq) and np.array_equal(meta["len"], on.rlen)
            assert np.array_equal(meta["bt"], on.rbt)
    finally:
        rt.destroy()
