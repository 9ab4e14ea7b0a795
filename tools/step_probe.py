"""Profiling probe for the decode-step kernel (kvring_step.cu), one GPU.

  python tools/step_probe.py decode [steps]   C2 (4 pools, batch 64) through kv_loop: the
                                              prelude to step 200 runs first (untimed), then
                                              `steps` loop launches (append k + publish k-1)
  python tools/step_probe.py bulk [reps]      C5 bulk re-seed: 8 pools x 512 MiB (full blocks)

Prints per-launch CUDA-event times and the algorithmic bytes; meant to run alone and
then under `ncu -k regex:kv_step` (the last launches are the measured ones).
"""
import json
import os
import statistics
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
    what = sys.argv[1] if len(sys.argv) > 1 else "decode"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = torch.device("cuda", 0)
    comp = torch.cuda.current_stream(dev)
    if what == "bulk":
        cfg = configs.C5
        g = cfg.geom
        S = cfg.stages
        rt = RingRuntime(g, cfg.num_blocks, 2, cfg.max_blocks_per_req, {s: 0 for s in range(S)},
                         {s: (s + 1) % S for s in range(S)}, device=0, spares=0, sentinel=None)
        P = cfg.fixed_prompt
        for s in range(S):
            src = content_tokens_cuda(CONTENT_SEED, [s] * P, range(P), s * g.layers, g.layers,
                                      g.kv_heads, g.head_dim, device=0)
            K.kv_append(rt.handle(s), [s], [P], src, 0, comp.cuda_stream)
            torch.cuda.synchronize()
            del src
        hs = [rt.handle(s) for s in range(S)]
        ms = []
        for rep in range(n):
            for s in range(S):
                rt.set_succ(s, (s + 1) % S)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K.kv_time_next_launch(a, b)
            K.kv_replicate_step_multi(hs, rep + 1, comp.cuda_stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        D = S * P * g.token_bytes
        print(json.dumps({"probe": "bulk", "ms": [round(x, 4) for x in ms],
                          "gb_s_rw": round(2 * D / (statistics.median(ms[1:] or ms) * 1e-3) / 1e9, 1)}))
        rt.destroy()
        return
    cfg = configs.C2
    g = cfg.geom
    S = cfg.stages
    coords = {(0, s): s for s in range(S)}
    succ = {s: (s + 1) % S for s in range(S)}
    scheds = configs.build_schedules(cfg, n_steps=200 + n + 2)
    rt = RingRuntime(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                     {s: 0 for s in range(S)}, succ, device=0, spares=0, sentinel=None)

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=0)

    drv = ScheduleDriver(rt, scheds, coords, content)
    for t in range(200):
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
    torch.cuda.synchronize()
    steps, evs, keep = [], [], []
    for t in range(200, 200 + n):
        app = []
        for node, e in drv.plan(t).items():
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            src = content(e["stage"], ids, pos) if ids else None
            keep.append(src)
            app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                            req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        evs.append(ev)
        st = dict(append=app, repl_pools=[rt.handle(s) for s in range(S)], step=t)
        if os.environ.get("STEP_PROBE_NOEVENTS") is None:
            st.update(ev_kernel_start=ev[0], ev_kernel_end=ev[1])
        steps.append(st)
    kl = K.KvLoop()
    torch.cuda.synchronize()
    K.kv_launch_log(True)
    prep = K.PreparedSteps(steps)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    K.kv_host_profile(reset=True)
    t0.record(comp)
    w0 = time.perf_counter()
    kl.run(prep, comp.cuda_stream)
    wall_us = (time.perf_counter() - w0) * 1e6
    t1.record(comp)
    torch.cuda.synchronize()
    loop_us = t0.elapsed_time(t1) * 1e3
    log = K.kv_launch_log(False)
    if os.environ.get("STEP_PROBE_NOFLUSH") is None:
        kl.flush(comp.cuda_stream)
    torch.cuda.synchronize()
    out = []
    prev = None
    noev = os.environ.get("STEP_PROBE_NOEVENTS") is not None
    if noev:  # per-launch bytes and grid (the timeline tool pairs them with its stamps)
        out = [{"rw_mb": round(2 * (r["app_bytes"] + r["rep_bytes"]) / 1e6, 2),
                "grid": r["grid"], "blob": r["blob_bytes"]} for r in log]
    for r, ev in zip(log, evs if not noev else []):
        us = ev[0].elapsed_time(ev[1]) * 1e3
        gap = prev[1].elapsed_time(ev[0]) * 1e3 if prev is not None else None
        prev = ev
        by = 2 * (r["app_bytes"] + r["rep_bytes"])
        out.append({"us": round(us, 2), "gap_us": None if gap is None else round(gap, 2),
                    "rw_mb": round(by / 1e6, 2),
                    "gb_s": round(by / (us * 1e-6) / 1e9, 1), "grid": r["grid"],
                    "blob": r["blob_bytes"]})
    rw = sum(2 * (r["app_bytes"] + r["rep_bytes"]) for r in log)
    host = {k: round(v / n * 1e6, 2) for k, v in K.kv_host_profile(reset=True).items()}
    print(json.dumps({"probe": "decode", "launches": out, "loop_us": round(loop_us, 1),
                      "host_wall_us_per_step": round(wall_us / n, 2), "host": host,
                      "us_per_step": round(loop_us / n, 2),
                      "gb_s_rw": round(rw / (loop_us * 1e-6) / 1e9, 1)}))
    kl.destroy()
    rt.destroy()


if __name__ == "__main__":
    main()
