"""C3 (BASELINE.json configs[2]) replication cost vs load: two 4-stage Llama-3.1-8B
pipelines, open-loop Poisson arrivals on a 20 ms logical decode step (§4
"Poisson distribution under different parameters of request rate"), cap 128 per
pipeline, ring within each pipeline.  For each RPS the decode loop runs 200 prelude
steps then 300 steps through kv_run_steps; reported per RPS: mean live requests,
replicated MB per step, ring-put kernel time and replication-stream time per step
(CUDA events), against the 400 us budget (2 % of a 20 ms TPOT).  One GPU (8 logical
nodes), or N GPUs under torchrun with node (p, s) on GPU (p + s) mod N (every hop
crosses NVLink for N > 1; per-step times are the max over ranks, bytes the sum).

    python tools/c3_sweep.py [--rps 1,2,4,8,16,32] [--steps 300]
    python -m torch.distributed.run --nproc-per-node N tools/c3_sweep.py
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def run(rps, steps, prelude, dev, rank=0, world=1, group=None):
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver, StreamOrder
    cfg = configs.scaled(configs.C3, rps=rps, num_blocks=6144, max_reqs=256)
    I, S = cfg.pipelines, cfg.stages
    g = cfg.geom
    coords = {(p, s): p * S + s for p in range(I) for s in range(S)}
    placement = {coords[(p, s)]: (p + s) % world for (p, s) in coords}
    succ = {coords[(p, s)]: coords[(p, (s + 1) % S)] for (p, s) in coords}
    scheds = configs.build_schedules(cfg, n_steps=prelude + steps + 2)
    rt = RingRuntime(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement, succ,
                     rank=rank, world=world, device=dev.index, spares=0, sentinel=None,
                     group=group)

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=dev.index)

    drv = ScheduleDriver(rt, scheds, coords, content)
    comp = torch.cuda.current_stream(dev)
    repl = torch.cuda.Stream(dev)
    order = StreamOrder(comp, repl)
    for t in range(prelude):
        order.before_append()
        drv.append_step(t, stream=comp)
        if t >= 1:
            order.before_publish()
            rt.replicate_all(t, stream=repl)
            order.after_publish()
    torch.cuda.synchronize(dev)
    handles = [rt.handle(n) for n in rt.alive_local()]
    steps_l, evs, live = [], [], []
    for t in range(prelude, prelude + steps):
        plan = drv.plan(t)
        app = []
        for node, e in plan.items():
            if node not in rt.local:
                continue
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                            req_ids=e["req_ids"], n_new=e["n_new"],
                            src=content(e["stage"], ids, pos) if ids else None))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        evs.append(ev)
        steps_l.append(dict(append=app, repl_pools=handles, step=t, ev_call=ev[0],
                            ev_kernel_start=ev[1], ev_kernel_end=ev[2]))
        live.append(sum(len(sc.steps[t].decode) + len(sc.steps[t].admit) for sc in scheds))
    prep = K.PreparedSteps(steps_l)
    b0 = sum(K.kv_stats(h)["bytes_replicated"] for h in handles)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
    torch.cuda.synchronize(dev)
    by = sum(K.kv_stats(h)["bytes_replicated"] for h in handles) - b0
    kern = [b.elapsed_time(c) * 1e3 for a, b, c in evs]
    call = [a.elapsed_time(c) * 1e3 for a, b, c in evs]
    if world > 1:   # per step: max over ranks; bytes: sum
        kt = torch.tensor([kern, call], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(kt, op=torch.distributed.ReduceOp.MAX)
        kern, call = kt[0].tolist(), kt[1].tolist()
        bt = torch.tensor([float(by)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(bt)
        by = float(bt[0])
        torch.distributed.barrier()
    rt.destroy()
    return {"rps": rps, "live_requests_mean": round(float(np.mean(live)), 1),
            "replicated_mb_per_step": round(by / steps / 2**20, 3),
            "ring_put_us": {"median": round(statistics.median(kern), 2),
                            "p99": round(float(np.percentile(kern, 99)), 2)},
            "replication_stream_us_per_step": {"median": round(statistics.median(call), 2),
                                               "p99": round(float(np.percentile(call, 99)), 2)},
            "budget_us": 400.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rps", default="1,2,4,8,16,32")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--prelude", type=int, default=200)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
        group = torch.distributed.group.WORLD
    out = [run(float(r), a.steps, a.prelude, dev, rank, world, group) for r in a.rps.split(",")]
    if rank == 0:
        print(json.dumps({"workload": "c3_2x4_poisson (2 pipelines x 4 stages, 20 ms logical "
                                      "step, cap 128)", "n_gpus": world,
                          "placement": "(p+s) mod N", "sweep": out}))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
