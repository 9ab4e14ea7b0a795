"""Diagnostic (not a test): C2 decode steps through kv_run_steps_graph WITHOUT timing
events, wall/device time per step -- for A/B of graph-structure knobs whose variants
cannot record the bench's per-kernel events.

    python tools/graph_ab.py [--steps 400]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--prelude", type=int, default=200)
    a = ap.parse_args()
    cfg = configs.C2
    g = cfg.geom
    S = cfg.stages
    coords = {(0, s): s for s in range(S)}
    scheds = configs.build_schedules(cfg, n_steps=a.prelude + a.steps + 2)
    rt = RingRuntime(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                     {s: 0 for s in range(S)}, {s: (s + 1) % S for s in range(S)},
                     device=0, spares=0, sentinel=None)

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=0)

    drv = ScheduleDriver(rt, scheds, coords, content)
    comp = torch.cuda.current_stream()
    repl = torch.cuda.Stream()
    for t in range(a.prelude):
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
    torch.cuda.synchronize()
    handles = [rt.handle(n) for n in rt.alive_local()]
    sts, keep = [], []
    for t in range(a.prelude, a.prelude + a.steps):
        app = []
        for nd, e in drv.plan(t).items():
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            src = content(e["stage"], ids, pos) if ids else None
            keep.append(src)
            app.append(dict(pool=rt.handle(nd), begin_step=1, release=e["release"],
                            req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        sts.append(dict(append=app, repl_pools=handles, step=t))
    W = 16   # warm-up call: builds and instantiates the graphs outside the timed region
    K.kv_run_steps_graph(K.PreparedSteps(sts[:W]), comp.cuda_stream, repl.cuda_stream)
    prep = K.PreparedSteps(sts[W:])
    torch.cuda.synchronize()
    b0 = sum(K.kv_stats(h)["bytes_replicated"] for h in handles)
    K.kv_host_profile(reset=True)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record(comp)
    K.kv_run_steps_graph(prep, comp.cuda_stream, repl.cuda_stream)
    en.record(comp)
    torch.cuda.synchronize()
    ms = st.elapsed_time(en)
    by = sum(K.kv_stats(h)["bytes_replicated"] for h in handles) - b0
    n = a.steps - W
    print(json.dumps({"value": round(by / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms / n, 4),
                      "host_us_per_step": {k: round(v / n * (1 if k.startswith("n_") else 1e6), 2)
                                           for k, v in K.kv_host_profile(reset=True).items() if v}}))
    rt.destroy()


if __name__ == "__main__":
    main()
