"""Multi-GPU parity worker (launched by tests/test_multigpu.py under torchrun).

N pipelines x 4 stages, node (p, s) on rank (p + s) mod N, stage ring inside each
pipeline: every ring hop is a one-sided NVLink store into the successor GPU's
symmetric-memory replica region.  Every rank runs the CPU oracle on the same
inputs (tiny config) and compares its own nodes byte for byte, every few steps;
a stage fails mid-run and is restored into a fresh pool on its holder's GPU,
and a second failure is restored REMOTELY (dst on another GPU, replica read over
NVLink).  Exit code 0 = parity on every rank.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from kvgen.schedule import closed_loop_schedule
    from oracle.simulate import OracleRing
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    from gpu_harness import compare_state

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    from datetime import timedelta
    dist.init_process_group("nccl", device_id=dev, timeout=timedelta(seconds=120))
    if os.environ.get("KV_TRANSPORT") == "r9":
        return r9_main(rank, world, lr, dev)
    if os.environ.get("KV_TRANSPORT") == "shared":
        return shared_main(rank, world, lr, dev)
    N, S = world, 4
    cfg = configs.scaled(configs.C1, pipelines=N, num_blocks=96, max_reqs=12,
                         max_blocks_per_req=12, batch_cap=6, n_requests=60, n_steps=30,
                         fixed_prompt=None, fail_node=(0, 1), fail_step=13)
    rng = np.random.default_rng(77)
    scheds = [closed_loop_schedule(rng.integers(1, 70, size=60), rng.integers(1, 30, size=60),
                                   cfg.n_steps, cfg.batch_cap, pipeline=p) for p in range(N)]
    coords = {(p, s): p * S + s for p in range(N) for s in range(S)}
    placement = {coords[(p, s)]: (p + s) % N for (p, s) in coords}
    succ = {coords[(p, s)]: coords[(p, (s + 1) % S)] for (p, s) in coords}
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=rank, world=world, device=lr, spares=2, group=dist.group.WORLD)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=lr)

    drv = ScheduleDriver(rt, scheds, coords, content)
    oring = OracleRing(cfg, schedules=scheds)
    transport = os.environ.get("KV_TRANSPORT", "p2p")
    nccl = None
    if transport == "nccl":
        from paper_2601_22438_b200.nccl_compare import NcclRing
        nccl = NcclRing(rt, 64 << 20)
    if transport in ("runsteps", "loop"):
        # the bench's launch path: kv_run_steps on two streams (helper-thread prepare,
        # inline descriptors, system-scope publication over NVLink), in chunks around
        # the failure step
        comp = torch.cuda.current_stream(dev)
        repl = torch.cuda.Stream(dev)
        kl = K.KvLoop()
        keep = []

        def chunk(t0, t1):
            sts = []
            for tt in range(t0, t1):
                app = []
                for node, e in drv.plan(tt).items():
                    if node not in rt.local:
                        continue
                    ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                    src = content(e["stage"], ids, pos) if ids else None
                    keep.append(src)
                    app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                    req_ids=e["req_ids"], n_new=e["n_new"], src=src))
                pools = [rt.handle(n) for n in rt.alive_local() if rt.succ.get(n) is not None]
                sts.append(dict(append=app, repl_pools=pools if tt >= 1 else [], step=tt))
                oring.appends(tt)
                if tt >= 1:
                    oring.replicate(tt)
            if transport == "loop":
                kl.run(K.PreparedSteps(sts), comp.cuda_stream)
                kl.flush(comp.cuda_stream)
            else:
                K.kv_run_steps(K.PreparedSteps(sts), comp.cuda_stream, repl.cuda_stream)
            torch.cuda.synchronize(dev)
            dist.barrier()
            compare_state(rt, drv, oring, tag=f"rank {rank} run_steps {t0}..{t1 - 1}")
            dist.barrier()

        chunk(0, cfg.fail_step)
        t = cfg.fail_step
        drv.append_step(t)
        oring.appends(t)
        drv.fail_and_restore(t, cfg.fail_node)
        oring.fail_and_restore(t, cfg.fail_node)
        rt.replicate_all(t)
        oring.replicate(t)
        torch.cuda.synchronize(dev)
        dist.barrier()
        chunk(cfg.fail_step + 1, cfg.n_steps)
    for t in range(cfg.n_steps if transport not in ("runsteps", "loop") else 0):
        drv.append_step(t)
        oring.appends(t)
        if t == cfg.fail_step:
            drv.fail_and_restore(t, cfg.fail_node)
            oring.fail_and_restore(t, cfg.fail_node)
        if t >= 1:
            if nccl is None:
                rt.replicate_all(t)
            else:
                nccl.step(t)
            oring.replicate(t)
        torch.cuda.synchronize(dev)
        dist.barrier()           # every rank's stores into peers are complete
        if t % 4 == 0 or t == cfg.n_steps - 1:
            compare_state(rt, drv, oring, tag=f"rank {rank} step {t}")
        dist.barrier()
    # remote restore: a fresh pool on rank (holder_rank + 1) % N reads the holder's
    # replica region over NVLink.  Fail stage 2 of pipeline 0 after the last step.
    torch.cuda.synchronize(dev)
    dist.barrier()
    f = drv.serving[(0, 2)]
    holder = rt.succ[f]
    rt.fail(f)
    dst_rank = (rt.placement[holder] + 1) % N
    dst = drv.next_node
    drv.next_node += 1
    rt.new_node(dst, dst_rank)
    ok = 1
    if rank == dst_rank:
        t_star, restored = rt.restore(dst, holder)
        torch.cuda.synchronize(dev)
        # expected: the oracle's published state of f at its holder
        hold_o = oring.serving[(0, 2)].succ
        exp = sorted((r, ln) for r, (s, ln, bt) in hold_o.published().items())
        if restored != exp or t_star != cfg.n_steps - 1:
            print(f"rank {rank}: remote restore mismatch {restored} vs {exp}", flush=True)
            ok = 0
        from kvgen.content import content_tokens
        pool = rt.local[dst].pool.cpu().numpy().view(np.uint16)
        for r, ln in restored:
            _, bt = K.kv_query(rt.handle(dst), r)
            want = content_tokens(CONTENT_SEED, [r] * ln, range(ln), 2 * g.layers, g.layers,
                                  g.kv_heads, g.head_dim)
            got = np.stack([pool[bt[p // 16], :, :, :, p % 16] for p in range(ln)])
            if not np.array_equal(got, want):
                print(f"rank {rank}: remote restore content mismatch for {r}", flush=True)
                ok = 0
    okt = torch.tensor([ok], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    rt.destroy()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_PARITY_OK" if int(okt) == 1 else "MGPU_PARITY_FAIL", flush=True)
    sys.exit(0 if int(okt) == 1 else 1)


def shared_main(rank, world, lr, dev):
    """NEXT-3 across GPUs (reading R17 with the holder on another rank): one 4-stage
    pipeline, stage s on rank s mod N, so every successor is remote; pools small enough
    that holders evict and drop replicas.  Each holder's rank keeps a mirror of its
    predecessor (tables only, pool through NVLink) and PULLS the dirty slices into
    blocks its own allocator picks.  Stage 1 fails at step 23 and is restored into a
    fresh pool on its holder's rank.  Every step: whole pools, metadata, tables,
    evictions, census == oracle on every rank, and every mirror's tables and
    publication state (pub_len, drops) == the oracle's node."""
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from kvgen.schedule import closed_loop_schedule
    from oracle.simulate import OracleRing
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    from gpu_harness import compare_mirrors, compare_state
    cfg = configs.scaled(configs.C1, num_blocks=32, max_reqs=12, max_blocks_per_req=12,
                         batch_cap=5, n_requests=60, n_steps=40, fixed_prompt=None,
                         pipelines=1, fail_node=(0, 1), fail_step=23)
    rng = np.random.default_rng(0)
    sched = [closed_loop_schedule(rng.integers(1, 70, size=cfg.n_requests),
                                  rng.integers(1, 30, size=cfg.n_requests), cfg.n_steps,
                                  cfg.batch_cap, pipeline=0)]
    S = cfg.stages
    coords = {(0, s): s for s in range(S)}
    placement = {s: s % world for s in range(S)}
    succ = {s: (s + 1) % S for s in range(S)}
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=rank, world=world, device=lr, spares=1, group=dist.group.WORLD,
                     shared=True)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=lr)

    drv = ScheduleDriver(rt, sched, coords, content, restore_mode="fresh")
    oring = OracleRing(cfg, schedules=sched, restore_mode="fresh", shared=True)
    ok, mirrors_checked = 1, 0
    try:
        for t in range(cfg.n_steps):
            drv.append_step(t)
            oring.appends(t)
            if t == cfg.fail_step:
                drv.fail_and_restore(t, cfg.fail_node)
                oring.fail_and_restore(t, cfg.fail_node)
            torch.cuda.synchronize(dev)
            dist.barrier()       # every owner's appends are in its HBM before a holder pulls
            if t >= 1:
                rt.replicate_all(t)
                oring.replicate(t)
            torch.cuda.synchronize(dev)
            dist.barrier()       # pulls complete before an owner reuses freed blocks (R7)
            compare_state(rt, drv, oring, tag=f"rank {rank} shared step {t}")
            mirrors_checked += compare_mirrors(rt, drv, oring, tag=f"rank {rank} step {t}")
            dist.barrier()
        ev = sum(n.evictions for n in oring.all_nodes())
        dr = sum(n.drops for n in oring.all_nodes())
        print(f"shared rank {rank}: {mirrors_checked} mirror checks, oracle evictions {ev}, "
              f"drops {dr}, mirrors {sorted(rt.mirrors)}", flush=True)
        if ev == 0 or dr == 0 or mirrors_checked == 0:
            ok = 0
    except AssertionError as e:
        print(f"rank {rank}: {e}", flush=True)
        ok = 0
    okt = torch.tensor([ok], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    rt.destroy()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_PARITY_OK" if int(okt) == 1 else "MGPU_PARITY_FAIL", flush=True)
    sys.exit(0 if int(okt) == 1 else 1)


def r9_main(rank, world, lr, dev):
    """Reading R9 observed concurrently: node A (rank 0) publishes every step over NVLink
    into node B's replica region (rank 1) through the one-launch loop, with no barrier or
    synchronize between steps; meanwhile a reader kernel on rank 1 acquires B's seq and,
    for every new value t, snapshots the parity-t table and the newest token slice of every
    listed request.  Each snapshot not overwritten meanwhile must equal the oracle's
    published table of step t and the closed-form words of those tokens: a reader that
    acquires seq = t sees all of step t."""
    from kvgen import configs
    from kvgen.content import CONTENT_SEED, content_tokens
    from kvgen.cuda import content_tokens_cuda, r9_observe
    from kvgen.schedule import closed_loop_schedule
    from oracle.simulate import OracleRing
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    assert world >= 2
    T = 400
    cfg = configs.scaled(configs.C1, stages=2, num_blocks=256, max_reqs=32,
                         max_blocks_per_req=16, batch_cap=12, n_requests=400, n_steps=T,
                         fixed_prompt=None, fail_node=None, fail_step=None)
    rng = np.random.default_rng(909)
    sched = [closed_loop_schedule(rng.integers(1, 90, size=400), rng.integers(1, 60, size=400),
                                  T + 1, cfg.batch_cap)]
    coords = {(0, 0): 0, (0, 1): 1}
    placement = {0: 0, 1: 1 % world}
    succ = {0: 1, 1: None}
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=rank, world=world, device=lr, spares=0, group=dist.group.WORLD)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=lr)

    drv = ScheduleDriver(rt, sched, coords, content)
    # expected published tables of A, step by step (oracle, metadata mode)
    oring = OracleRing(cfg, content=False, schedules=sched)
    expect = {}
    for t in range(T + 1):
        oring.appends(t)
        if t >= 1:
            oring.replicate(t)
            expect[t] = oring.nodes[(0, 1)].published()
    ok = 1
    if rank == 0:
        keep, sts = [], []
        for t in range(T):
            e = drv.plan(t).get(0)
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            src = content(0, ids, pos) if ids else None
            keep.append(src)
            sts.append(dict(append=[dict(pool=rt.handle(0), begin_step=1, release=e["release"],
                                         req_ids=e["req_ids"], n_new=e["n_new"], src=src)],
                            repl_pools=[rt.handle(0)] if t >= 1 else [], step=t))
        prep = K.PreparedSteps(sts)
        kl = K.KvLoop()
        torch.cuda.synchronize(dev)
        dist.barrier()                       # the reader is running
        kl.run(prep, torch.cuda.current_stream(dev).cuda_stream)
        kl.flush(torch.cuda.current_stream(dev).cuda_stream)
        torch.cuda.synchronize(dev)
        kl.destroy()
    elif rank == 1:
        side = torch.cuda.Stream(dev)
        R, M, B = cfg.max_reqs, cfg.max_blocks_per_req, g.block_size
        with torch.cuda.stream(side):
            recs, n_done, rec_bytes = r9_observe(rt.meta_ptr(1), rt.replica_ptr(1), R, M, B,
                                                 rt.block_bytes, g.head_dim * 2, 256,
                                                 last_seq=T - 1, device=lr,
                                                 stream=side.cuda_stream)
        dist.barrier()
        side.synchronize()
        n = int(n_done.item())
        raw = recs.cpu().numpy()
        valid = 0
        for k in range(n):
            rec = raw[k]
            seq, after = (int(x) for x in rec[:16].view(np.uint64))
            if after > seq + 1:              # parity buffer reused while copying
                continue
            req = rec[16:16 + 8 * R].view(np.int64)
            ln = rec[16 + 8 * R:16 + 12 * R].view(np.int32)
            sl = rec[16 + 12 * R:16 + 12 * R + R * g.head_dim * 2].view(np.uint16).reshape(R, -1)
            pub = expect[seq]
            got = {int(req[s]): (s, int(ln[s])) for s in range(R) if req[s] >= 0}
            want = {r: (s, l) for r, (s, l, bt) in pub.items()}
            if got != want:
                print(f"r9: seq {seq}: table {got} != {want}", flush=True)
                ok = 0
                continue
            # a request that retires at t+1 frees its blocks, and step t+2's copies may
            # refill them before seq moves past t+1: check the requests still published at
            # t+1 (their blocks stay theirs until step t+2's retirement, R7)
            nxt = expect.get(seq + 1, {})
            for r, (s, l) in got.items():
                if r not in nxt:
                    continue
                w = content_tokens(CONTENT_SEED, [r], [l - 1], 0, g.layers, g.kv_heads,
                                   g.head_dim)[0, 0, 0, 0]
                if not np.array_equal(sl[s], w):
                    print(f"r9: seq {seq}: request {r} token {l - 1} not visible", flush=True)
                    ok = 0
            valid += 1
        print(f"r9: {n} observations, {valid} checked (distinct seqs seen while publishing)",
              flush=True)
        if valid < 5:
            print("r9: too few concurrent observations", flush=True)
            ok = 0
    else:
        dist.barrier()
    okt = torch.tensor([ok], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    rt.destroy()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_PARITY_OK" if int(okt) == 1 else "MGPU_PARITY_FAIL", flush=True)
    sys.exit(0 if int(okt) == 1 else 1)


if __name__ == "__main__":
    main()
