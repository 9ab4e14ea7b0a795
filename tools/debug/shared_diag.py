"""Diagnostic (not a test): run the shared-capacity pressure case step by step on
the GPU against the oracle and explain the first content mismatch."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from kvgen import configs
from kvgen.content import content_tokens
from kvgen.schedule import closed_loop_schedule
from oracle.simulate import OracleRing
from gpu_harness import make_gpu, node_map
from paper_2601_22438_b200 import kvring as K

def sched(cfg, seed):
    rng = np.random.default_rng(seed)
    p = rng.integers(1, 70, size=cfg.n_requests); o = rng.integers(1, 30, size=cfg.n_requests)
    return [closed_loop_schedule(p, o, cfg.n_steps, cfg.batch_cap, pipeline=i) for i in range(cfg.pipelines)]

cfg = configs.scaled(configs.C1, num_blocks=32, max_reqs=12, max_blocks_per_req=12, batch_cap=5,
                     n_requests=60, n_steps=40, fixed_prompt=None, fail_node=(0, 1), fail_step=23)
rt, drv = make_gpu(cfg, schedules=sched(cfg, 0), restore_mode="fresh", shared=True)
orng = OracleRing(cfg, schedules=drv.sched, restore_mode="fresh", shared=True)
g = cfg.geom
def ident(vec):
    for st in range(4):
        for r in range(60):
            x = content_tokens(2601, [r] * 200, list(range(200)), st * g.layers, g.layers, g.kv_heads, g.head_dim)
            hit = np.nonzero((x[:, 0, 0, 0, :] == vec).all(axis=1))[0]
            if hit.size: return (st, r, int(hit[0]))
    return None
for t in range(cfg.n_steps):
    drv.append_step(t); orng.appends(t)
    if t == cfg.fail_step:
        drv.fail_and_restore(t, cfg.fail_node); orng.fail_and_restore(t, cfg.fail_node)
    if t >= 1:
        rt.replicate_all(t); orng.replicate(t)
    torch.cuda.synchronize()
    bad = False
    for gid, on in node_map(rt, drv, orng).items():
        if gid not in rt.local or on.dead: continue
        prim = rt.local[gid].pool.cpu().numpy().view(np.uint16)
        d = np.argwhere((prim != on.primary).any(axis=-1))
        st = K.kv_stats(rt.handle(gid))
        tabs_ok = st["free_blocks"] == len(on.free_blocks) and st["replica_blocks_held"] == (on.rep_src.census() if on.rep_src else 0)
        if d.size or not tabs_ok:
            print("step", t, "node", gid, "tables_ok", tabs_ok, st, len(on.free_blocks), sorted(on.free_blocks)[:20])
            for b in d[:6]:
                b = tuple(int(x) for x in b)
                print("  diff at", b, "gpu is", ident(prim[b[0], 0, 0, 0, b[4]]), "oracle is", ident(on.primary[b[0], 0, 0, 0, b[4]]))
            src = on.rep_src
            if src is not None:
                print("  oracle rep_bt of pred", src.node_id, {int(src.slot_req[s]): src.rep_bt[s] for s in range(src.R) if src.rep_bt[s]})
            bad = True
    meta_ok = True
    if bad:
        break
print("done at", t)
rt.destroy()
