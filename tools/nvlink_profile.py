"""NVLink evidence for the ring hop, in ONE process (ncu must not wrap a multi-rank
command): the 4 stages of a C2 pipeline live on GPU 0, their ring successors' replica
regions and metadata on GPU 1 (holder pools created there), so every ring-put stores
over NVLink exactly as in the multi-rank bench.  Runs the C2 decode loop through
kv_run_steps (prelude, then timed steps); under `ncu --metrics
nvltx__bytes.sum,nvltx__bytes_data_user.sum,...` the ring-put launches give the NVLink
bytes per launch vs the algorithmic D.

    python tools/nvlink_profile.py [--steps 60]
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--prelude", type=int, default=200)
    ap.add_argument("--steps", type=int, default=60)
    a = ap.parse_args()
    cfg = configs.scaled(configs.C2, num_blocks=4096)
    g = cfg.geom
    S = cfg.stages
    (sch,) = configs.build_schedules(cfg, n_steps=a.prelude + a.steps + 2)
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
    holders = [pool_on(d1, 100 + s) for s in range(S)]      # stage s's successor, on GPU 1
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
    repl = torch.cuda.Stream(d0)
    K.kv_run_steps(K.PreparedSteps(steps(0, a.prelude)), comp.cuda_stream, repl.cuda_stream)
    torch.cuda.synchronize(d0)
    b0 = sum(K.kv_stats(h)["bytes_replicated"] for h in handles)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prep = K.PreparedSteps(steps(a.prelude, a.steps))
    torch.cuda.synchronize(d0)
    st.record(comp)
    K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
    fin = torch.cuda.Event()
    fin.record(repl)
    comp.wait_event(fin)
    en.record(comp)
    torch.cuda.synchronize(d0)
    by = sum(K.kv_stats(h)["bytes_replicated"] for h in handles) - b0
    ms = st.elapsed_time(en)
    print(json.dumps({"what": "C2 pipeline on GPU 0, successors on GPU 1 (one process)",
                      "steps": a.steps, "replicated_bytes": int(by),
                      "bytes_per_step": int(by / a.steps), "ms_per_step": round(ms / a.steps, 4),
                      "gb_s": round(by / (ms * 1e-3) / 1e9, 1)}), flush=True)
    for h in handles + [p[0] for p in holders]:
        K.kv_pool_destroy(h)


if __name__ == "__main__":
    main()
