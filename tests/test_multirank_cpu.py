"""World-size-2 gloo test of the multi-rank host path on CPU: the bench placement
(node (p, s) on rank (p + s) mod N), per-rank ScheduleDriver stepping only local
nodes, C++ tables-only pools.  Every rank's tables equal the oracle (metadata
mode) at C2 geometry; the replicated payload bytes summed over ranks (the
bench's `value` numerator) equal the oracle's."""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, steps, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from kvgen import configs
    from oracle.simulate import OracleRing
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import ScheduleDriver, TablesRuntime
    N, S = world, 4
    cfg = configs.scaled(configs.C2, pipelines=N)
    scheds = configs.build_schedules(cfg, n_steps=steps)
    coords = {(p, s): p * S + s for p in range(N) for s in range(S)}
    placement = {coords[(p, s)]: (p + s) % N for (p, s) in coords}
    succ = {coords[(p, s)]: coords[(p, (s + 1) % S)] for (p, s) in coords}
    rt = TablesRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                       placement, succ, rank=rank, world=world)
    drv = ScheduleDriver(rt, scheds, coords, content=lambda *a: None)
    oring = OracleRing(cfg, content=False, schedules=scheds)
    bad = 0
    for t in range(steps):
        drv.append_step(t)
        oring.appends(t)
        if t >= 1:
            rt.replicate_all(t)
            oring.replicate(t)
    for c, n in coords.items():
        if n in rt.local:
            req, ln, pub, nb = K.kv_dump_slots(rt.handle(n), cfg.max_reqs)
            live = {int(req[s]): (s, int(ln[s]), K.kv_query(rt.handle(n), int(req[s]))[1])
                    for s in range(cfg.max_reqs) if req[s] >= 0}
            bad += live != oring.nodes[c].live()
    mine = sum(K.kv_stats(rt.handle(n))["bytes_replicated"] for n in rt.local)
    tot = torch.tensor([float(mine), float(bad), float(len(rt.local))], dtype=torch.float64)
    dist.all_reduce(tot)
    if rank == 0:
        q.put((tot.tolist(), oring.moved))
    rt.destroy()
    dist.destroy_process_group()


def test_two_ranks_tables_and_bytes():
    world, steps = 2, 120
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, 29711, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    (tot, moved) = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    mine, bad, nloc = tot
    assert bad == 0
    assert nloc == 4 * world                 # every GPU hosts 4 stages (weak scaling)
    assert mine == moved                     # bench numerator == oracle's payload bytes
