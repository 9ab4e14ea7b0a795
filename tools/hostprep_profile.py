"""Host-side cost of the decode loop on CPU (no GPU): C2 on tables-only pools
(kv_pool_desc_t.device = -1), so kv_run_steps runs allocation, tables, work lists
and publication bookkeeping exactly as on the GPU box and launches nothing.

    python tools/hostprep_profile.py [steps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from kvgen import configs  # noqa: E402
from paper_2601_22438_b200 import kvring as K  # noqa: E402

FAKE = 0x1000


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    cfg = configs.C2
    g = cfg.geom
    (sch,) = configs.build_schedules(configs.scaled(cfg, n_steps=200 + n))
    kg = K.geom(g.layers, g.kv_heads, g.head_dim, g.block_size, g.elem_bytes)
    hs = [K.kv_pool_create(K.kv_pool_desc_t(kg, cfg.num_blocks, cfg.max_reqs,
                                            cfg.max_blocks_per_req, -1, s, cfg.num_blocks,
                                            None, None, None)) for s in range(cfg.stages)]
    for h in hs:
        K.kv_set_successor(h, 0, FAKE, cfg.num_blocks, FAKE)

    def entries(t):
        ev = sch.steps[t]
        ids = sorted(ev.decode) + [r for r, _ in ev.admit]
        nn = [1] * len(ev.decode) + [p for _, p in ev.admit]
        return [dict(pool=h, begin_step=1, release=ev.retire, req_ids=ids, n_new=nn, src=None)
                for h in hs]

    steps = [dict(append=entries(t), repl_pools=hs if t >= 1 else [], step=t)
             for t in range(200 + n)]
    K.kv_run_steps(K.PreparedSteps(steps[:200]))
    timed = K.PreparedSteps(steps[200:])
    K.kv_host_profile()
    t0 = time.perf_counter()
    K.kv_run_steps(timed)
    dt = time.perf_counter() - t0
    prof = K.kv_host_profile()
    print(f"{n} steps: {dt / n * 1e6:.2f} us/step host (tables only)")
    print({k: round(v / n * 1e6, 2) for k, v in prof.items() if v})
    for h in hs:
        K.kv_pool_destroy(h)


if __name__ == "__main__":
    main()
