"""Phase timeline of the decode-step kernel when every hop crosses NVLink, in ONE process
(debug build: KVRING_NVCC_DEFS=-DKV_TIMELINE): the 4 stages of a C2 pipeline on GPU 0,
their successors' replica regions and metadata on GPU 1, driven through kv_loop_run as
in the bench (chained launches, deferred publication).  Prints, per launch, when its CTAs
pass each phase boundary (tools/step_timeline.py's table), then rebuilds the product.

    python tools/step_timeline_nvl.py [steps]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    env = dict(os.environ, KVRING_NVCC_DEFS="-DKV_TIMELINE")
    subprocess.run([sys.executable, "-m", "paper_2601_22438_b200.build", "--force"], env=env,
                   check=True, cwd=ROOT, stdout=subprocess.DEVNULL)
    import ctypes

    import numpy as np
    import torch
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    prelude = 200
    cfg = configs.scaled(configs.C2, num_blocks=4096)
    g = cfg.geom
    S = cfg.stages
    (sch,) = configs.build_schedules(cfg, n_steps=prelude + 2 * n_steps + 2)
    kg = K.geom(g.layers, g.kv_heads, g.head_dim, g.block_size, g.elem_bytes)
    bb = K.kv_block_bytes(kg)
    mb = K.kv_meta_bytes(cfg.max_reqs, cfg.max_blocks_per_req)
    keep = []

    def pool_on(dev, node):
        pool = torch.empty(cfg.num_blocks * bb // 2, dtype=torch.int16, device=dev)
        rep = torch.empty(cfg.num_blocks * bb // 2, dtype=torch.int16, device=dev)
        meta = torch.empty(mb, dtype=torch.uint8, device=dev)
        keep.extend([pool, rep, meta])
        d = K.kv_pool_desc_t(kg, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                             dev.index, node, cfg.num_blocks, pool.data_ptr(), rep.data_ptr(),
                             meta.data_ptr())
        return K.kv_pool_create(d), rep, meta

    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    holders = [pool_on(d1, 100 + s) for s in range(S)]
    torch.cuda.set_device(d0)
    prim = [pool_on(d0, s) for s in range(S)]
    for s in range(S):
        _, rep, meta = holders[(s + 1) % S]
        K.kv_set_successor(prim[s][0], 100 + (s + 1) % S, rep.data_ptr(), cfg.num_blocks,
                           meta.data_ptr())
    handles = [p[0] for p in prim]

    def steps(t0, n):
        out = []
        for t in range(t0, t0 + n):
            ev = sch.steps[t]
            ids = sorted(ev.decode) + [r for r, _ in ev.admit]
            nn = [1] * len(ev.decode) + [p for _, p in ev.admit]
            starts = [sch.length_at(r, t - 1) for r in sorted(ev.decode)] + [0] * len(ev.admit)
            tid, tpos = [], []
            for r, k, p0 in zip(ids, nn, starts):
                tid.extend([r] * k)
                tpos.extend(range(p0, p0 + k))
            app = []
            for s in range(S):
                src = (content_tokens_cuda(CONTENT_SEED, tid, tpos, s * g.layers, g.layers,
                                           g.kv_heads, g.head_dim, device=0) if tid else None)
                keep.append(src)
                app.append(dict(pool=handles[s], begin_step=1, release=ev.retire, req_ids=ids,
                                n_new=nn, src=src))
            out.append(dict(append=app, repl_pools=handles if t >= 1 else [], step=t))
        return out

    comp = torch.cuda.current_stream(d0)
    kl = K.KvLoop()
    kl.run(K.PreparedSteps(steps(0, prelude)), comp.cuda_stream)
    torch.cuda.synchronize(d0)
    prep = K.PreparedSteps(steps(prelude, n_steps))
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(d0)
    b0 = sum(K.kv_stats(h)["bytes_replicated"] for h in handles)
    st.record(comp)
    kl.run(prep, comp.cuda_stream)
    en.record(comp)
    torch.cuda.synchronize(d0)
    by = sum(K.kv_stats(h)["bytes_replicated"] for h in handles) - b0
    ms = st.elapsed_time(en)
    print(json.dumps({"what": "C2 pipeline on GPU 0, successors on GPU 1, kv_loop_run",
                      "steps": n_steps, "bytes_per_step": int(by / n_steps),
                      "us_per_step": round(ms * 1e3 / n_steps, 2),
                      "nvlink_gb_s": round(by / (ms * 1e-3) / 1e9, 1)}), flush=True)
    f = K.lib().kv_debug_timeline
    f.restype = ctypes.c_int
    NL = 32
    buf = np.zeros(NL * 1024 * 8, dtype=np.uint64)
    f(buf.ctypes.data, buf.size)
    t = buf.reshape(NL, 1024, 8)
    launches = []
    for k in range(NL):
        x = t[k].astype(np.float64)
        # CTAs of this launch; the publisher CTA (deferred seqs) stamps only its start
        ok = (t[k][:, 7] != 0) & (x[:, 1:6] >= x[:, [0]]).all(axis=1) & \
             (x[:, 5] - x[:, 0] < 1e6)
        if ok.any():
            launches.append((int(t[k][ok][0, 7]), x[ok]))
    launches.sort()
    names = ["start", "blob", "wait", "copies", "tables", "done"]
    t0 = min(x[:, 0].min() for _, x in launches[-4:])
    for nonce, x in launches[-4:]:
        print("launch %d (%d CTAs):" % (nonce, len(x)))
        for k, name in enumerate(names):
            col = (x[:, k] - t0) / 1e3
            print("   %-7s min %8.2f  median %8.2f  max %8.2f us" % (name, col.min(),
                                                                     np.median(col), col.max()))
    print("\nlaunch  CTAs  period | blob.med wait.med wait.max | copies.med copies.max | "
          "done.med done.max | prev.done.max->wait.min")
    prev = None
    for nonce, x in launches:
        s0 = x[:, 0].min()
        r = lambda k, fn: (fn(x[:, k]) - s0) / 1e3
        period = (s0 - prev[:, 0].min()) / 1e3 if prev is not None else float("nan")
        gap = (x[:, 2].min() - prev[:, 5].max()) / 1e3 if prev is not None else float("nan")
        print("%6d %5d %7.2f | %8.2f %8.2f %8.2f | %10.2f %10.2f | %8.2f %8.2f | %6.2f" % (
            nonce, len(x), period, r(1, np.median), r(2, np.median), r(2, np.max),
            r(3, np.median), r(3, np.max), r(5, np.median), r(5, np.max), gap))
        prev = x
    kl.destroy()
    for h in handles + [p[0] for p in holders]:
        K.kv_pool_destroy(h)


if __name__ == "__main__":
    try:
        main()
    finally:  # back to the product build
        subprocess.run([sys.executable, "-m", "paper_2601_22438_b200.build", "--force"],
                       cwd=ROOT, stdout=subprocess.DEVNULL)
