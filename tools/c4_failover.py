"""C4 failover at scale on N GPUs (BASELINE.json configs[3]): 16 logical nodes
(4 pipelines x 4 stages), the paper's ring (same stage, next instance: P:215,
P:225), node (i, s) on GPU (4i + s) mod N so every hop crosses GPUs, closed-loop
batch 128 per pipeline.  At step 300 (0,2) fails after its append; its 128
requests are promoted onto its replication target (1,2) (restore: the holder's
replica region -> its own pool, local HBM), the failed node and the rerouting
donor are excluded from replication and the ring is re-protected; the
run resumes for 100 steps.  Every rank checks its nodes' tables against the CPU
oracle (metadata mode) after the failure and at the end, and samples valid
slots against the closed form.

    python -m torch.distributed.run --nproc-per-node N tools/c4_failover.py

Rank 0 prints one JSON line (restore ms / GB/s and the parity verdict; the loop
itself runs the oracle and content generation per step, so it is not timed).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from datetime import timedelta
    from kvgen import configs
    from kvgen.content import CONTENT_SEED, content_tokens
    from kvgen.cuda import content_tokens_cuda
    from oracle.simulate import OracleRing
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver, StreamOrder
    from gpu_harness import compare_state

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev, timeout=timedelta(seconds=300))
    steps = int(os.environ.get("C4_STEPS", 401))
    cfg = configs.scaled(configs.C4, num_blocks=8192, max_reqs=512, ring="instance",
                         n_steps=steps)
    I, S = cfg.pipelines, cfg.stages
    coords = {(i, s): i * S + s for i in range(I) for s in range(S)}
    placement = {coords[(i, s)]: (4 * i + s) % world for (i, s) in coords}
    succ = {coords[(i, s)]: coords[((i + 1) % I, s)] for (i, s) in coords}
    scheds = configs.build_schedules(cfg)
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=rank, world=world, device=lr, spares=0,
                     group=dist.group.WORLD if world > 1 else None, sentinel=None)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=lr)

    drv = ScheduleDriver(rt, scheds, coords, content, restore_mode="promote")
    oring = OracleRing(cfg, content=False, ring="instance", schedules=scheds,
                       restore_mode="promote")
    comp = torch.cuda.current_stream(dev)
    repl = torch.cuda.Stream(dev)
    order = StreamOrder(comp, repl)
    step_us = {"before": [], "after": []}
    restore = {}
    ok = 1
    for t in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(comp)
        order.before_append()
        drv.append_step(t, stream=comp)
        oring.appends(t)
        if t == cfg.fail_step:
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            ra, rb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K.kv_time_next_launch(ra, rb)
            w0 = time.perf_counter()
            drv.fail_and_restore(t, cfg.fail_node, stream=comp)
            torch.cuda.synchronize(dev)
            wall = (time.perf_counter() - w0) * 1e3
            oring.fail_and_restore(t, cfg.fail_node)
            if drv.events:
                ev = drv.events[0].data
                tok = sum(ln for _, ln in ev["restored"])
                R = tok * g.token_bytes
                km = ra.elapsed_time(rb)
                restore = {"t_star": ev["t_star"], "requests": len(ev["restored"]),
                           "restored_bytes": R, "ms_wall_incl_resume": round(wall, 3),
                           "kernel_ms": round(km, 3),
                           "kernel_gb_s_rw": round(2 * R / (km * 1e-3) / 1e9, 1),
                           "dst": "holder (1,2): promotion, replica region -> own pool"}
            drv.reprotect([(0, 2), (1, 2)])
            oring.reprotect([(0, 2), (1, 2)])
        if t >= 1:
            order.before_publish()
            rt.replicate_all(t, stream=repl)
            order.after_publish()
        done = torch.cuda.Event()
        done.record(repl)
        comp.wait_event(done)
        b.record(comp)
        if t >= 1:
            oring.replicate(t)
        if 200 <= t < cfg.fail_step or t > cfg.fail_step + 10:
            step_us["before" if t < cfg.fail_step else "after"].append((a, b))
        if t in (cfg.fail_step, steps - 1):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            try:
                compare_state(rt, drv, oring, content=False, tag=f"rank {rank} step {t}")
            except AssertionError as e:
                print(f"rank {rank}: PARITY FAIL {e}", flush=True)
                ok = 0
            if world > 1:
                dist.barrier()
    torch.cuda.synchronize(dev)
    # sampled content of every local live node (primary) against the closed form
    rng = np.random.default_rng(rank)
    inv = {}
    for c, n in drv.serving.items():
        inv.setdefault(n, c)
    for n in rt.alive_local():
        c = inv.get(n)
        if c is None:
            continue
        live = {}
        req, ln, pub, nb = K.kv_dump_slots(rt.handle(n), rt.R)
        items = []
        for sidx in np.nonzero(req >= 0)[0][:16]:
            r, L = int(req[sidx]), int(ln[sidx])
            _, bt = K.kv_query(rt.handle(n), r)
            pos = int(rng.integers(0, L))
            items.append((r, pos, bt[pos // 16]))
        if not items:
            continue
        stage = c[1]
        want = content_tokens(CONTENT_SEED, [i[0] for i in items], [i[1] for i in items],
                              stage * g.layers, g.layers, g.kv_heads, g.head_dim)
        idx = torch.tensor([i[2] for i in items], device=dev)
        sl = torch.tensor([i[1] % 16 for i in items], device=dev)
        got = rt.local[n].pool[idx, :, :, :, sl].cpu().numpy().view(np.uint16)
        if not np.array_equal(got, want):
            print(f"rank {rank}: content mismatch on node {n}", flush=True)
            ok = 0
    med = {k: (float(np.median([x.elapsed_time(y) * 1e3 for x, y in v])) if v else None)
           for k, v in step_us.items()}
    vec = torch.tensor([float(ok), med["before"] or 0.0, med["after"] or 0.0,
                        restore.get("kernel_ms", 0.0)], dtype=torch.float64, device=dev)
    if world > 1:
        mn = vec.clone()
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        ok_all, before, after = int(mn[0]), float(mx[1]), float(mx[2])
        blob = [None] * world
        dist.all_gather_object(blob, restore)
        restore = next((r for r in blob if r), {})
    else:
        ok_all, before, after = ok, med["before"], med["after"]
    rt.destroy()
    if rank == 0:
        print(json.dumps({"workload": "c4_failover_16 (paper instance ring, promotion)",
                          "n_gpus": world, "placement": "(4i+s) mod N", "batch_per_pipeline": 128,
                          "steps": steps, "fail": "(0,2) at step 300 after its append",
                          "parity_tables_and_samples": bool(ok_all),
                          "restore": restore}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok_all else 1)


if __name__ == "__main__":
    main()
