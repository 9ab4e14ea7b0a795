#!/usr/bin/env python
"""Bench: ring KV-cache replication hot path (KevlarFlow, arXiv 2601.22438) on B200.

Workload (BASELINE.json configs[1], "c2_pp4_b64"): Llama-3.1-8B KV geometry,
4-stage pipelines (8 layers/stage, GQA 8 x 128, bf16 words), closed-loop batch
64 over a ShareGPT-shaped trace, incremental per-decode-step ring replication.
Weak scaling: with N GPUs there are N pipelines and logical node (p, s) lives
on GPU (p + s) mod N, so every GPU hosts 4 stages and (for N > 1) every ring
hop crosses NVLink; at N = 1 the ring is a loopback inside one GPU's HBM.

A step = the whole hot path of SURVEY §8(a): a1/a2 append (allocate + scatter
the step's new-token KV) and a3-a5 replicate (dirty work list, fused gather +
ring-put + metadata + seq flag).  Steps 0..PRELUDE-1 bring the trace to
steady state (untimed), then W warm-up and K timed steps.  `value` = payload
bytes replicated by all ranks / max-over-ranks device time of the K steps.

Extra keys: per-step replication overhead (µs, replicate-only device time),
restore ms (failure of stage 2 after the last step, fresh pool), the ring-put
kernel's live roofline, e2e through host buffers, clocks, the CPU oracle
baseline.  `--impl reference` runs the CPU oracle (the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "replicated KV GB/s (ring KV-cache replication, per-decode-step, C2)"
UNIT = "GB/s"
PRELUDE = 200
CFG_NAME = "c2_pp4_b64"
TIME_EVERY = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="kvring", choices=["kvring", "reference"])
    ap.add_argument("--prelude", type=int, default=PRELUDE)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-restore", action="store_true")
    ap.add_argument("--bulk-reps", type=int, default=5, help="C5 bulk re-seed reps (0: skip)")
    ap.add_argument("--interference-steps", type=int, default=100,
                    help="steps with a Llama-3.1-8B stage decode proxy on the compute stream, "
                         "replication on vs off (0: skip)")
    ap.add_argument("--block-steps", type=int, default=100,
                    help="steps in block-granular mode (NEXT-2), after a re-seed (0: skip)")
    ap.add_argument("--nccl-steps", type=int, default=100,
                    help="steps replicated through the NCCL send/recv comparison (0: skip)")
    ap.add_argument("--shared-steps", type=int, default=100,
                    help="timed steps of the shared-capacity leg (NEXT-3; N = 1 only; 0: skip)")
    ap.add_argument("--timeline", action="store_true",
                    help="diagnostic: time every step and print the replication-stream timeline")
    ap.add_argument("--loop", default="auto", choices=["auto", "fused", "streams", "pdl", "graph"],
                    help="streams: kv_run_steps (append stream + replication stream); graph: "
                         "kv_run_steps_graph (the same steps as CUDA graphs of 8 steps); pdl: "
                         "one stream with programmatic dependent launch; fused: append k + "
                         "publication k-1 per launch; auto (default): graph (measured +7-13 %% "
                         "on 1 GPU, +2.5-3.5 %% on 2 and 4 GPUs over the two-stream loop, "
                         "profiles/r01/exp37.log, exp39-41.log)")
    ap.add_argument("--single-stream", action="store_true",
                    help="append and replicate on one stream (default: replication stream)")
    return ap.parse_args()


def bench_config(n_gpus):
    """The workload (BASELINE.json configs[1]) as the bench line's `config` -- identical
    for the kvring arm and the reference (oracle) arm."""
    from kvgen import configs
    c = configs.C2
    g = c.geom
    return {"workload": CFG_NAME, "pipelines": n_gpus, "stages_per_pipeline": c.stages,
            "layers_per_stage": g.layers, "kv_heads": g.kv_heads, "head_dim": g.head_dim,
            "block_size": g.block_size, "batch_per_pipeline": c.batch_cap,
            "placement": "(p+s) mod N",
            "l2": "inputs larger than L2 (multi-GiB pre-generated sources and pools; no flush); "
                  "the replicated slices were just written by the append, as in serving"}


def traffic_ref(kind, kernel="kv_ring_put_kernel"):
    """Captured DRAM traffic per launch (profiles/traffic.json, from ncu --set full)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)[kernel][kind]
        return d
    except Exception:
        return None


# the timed decode steps launch the inline-descriptor ring-put (descriptors in the
# kernel parameter space); steps whose descriptors exceed 28 KiB use the staged one
RINGPUT = "kv_ring_put_inl_kernel (staged kv_ring_put_kernel for large steps)"
RINGPUT_GRAPH = ("kv_ring_put_copy_kernel (CUDA-graph copy nodes of kv_run_steps_graph; the "
                 "publication is a separate kv_publish_kernel node)")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NVLINK_PEAK_GBS = 770.0   # B200_PROFILING.md measured peer copy per direction (900 nominal)


def step_roofline(tot_bytes, ms_max, n, hbm_peak, peak_src):
    """Whole decode step (append + ring-put + publication) against the roofline.

    Over the timed run the appended bytes equal the replicated bytes D (every token
    appended is published once, one step later).  Per GPU the step
    moves 4·D/N through HBM: the append reads the dense source and writes the pool
    (2·D/N), the ring-put reads the pool (D/N) and the GPU receives one link's writes
    (D/N, its own at N = 1).  At N > 1, D/N also crosses NVLink out of each GPU.
    """
    sec = ms_max * 1e-3
    hbm = 4 * tot_bytes / n / sec / 1e9
    out = {"hbm": {"achieved": round(hbm, 1), "peak": hbm_peak, "unit": "GB/s",
                   "frac": round(hbm / hbm_peak, 4), "peak_source": peak_src},
           "what": "per GPU, whole timed step: algorithmic HBM bytes 4*D/N (append r+w, "
                   "ring-put read, incoming replica writes) over ms_per_step; D = replicated "
                   "bytes (= appended bytes over the run)"}
    if n > 1:
        nvl = tot_bytes / n / sec / 1e9
        out["nvlink"] = {"achieved": round(nvl, 1), "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                         "frac": round(nvl / NVLINK_PEAK_GBS, 4),
                         "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction"}
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to start; the timed region can be shorter
            # (C2: ~8 ms), so wait for its first sample -- the samples then bracket the region
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- GPU arm
def run_kvring(args):
    import torch
    import torch.distributed as dist
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver, StreamOrder

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    N = args.gpus
    if args.loop == "auto":
        args.loop = "graph"
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}; launch N>1 with torch.distributed.run")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    base = configs.C2
    S = base.stages
    cfg = configs.scaled(base, pipelines=N)
    g = cfg.geom
    coords = {(p, s): p * S + s for p in range(N) for s in range(S)}
    placement = {coords[(p, s)]: (p + s) % N for (p, s) in coords}
    succ = {coords[(p, s)]: coords[(p, (s + 1) % S)] for (p, s) in coords}
    n_total = (args.prelude + args.warmup + args.steps + args.e2e_steps + args.nccl_steps
               + 2 * args.interference_steps + args.block_steps + 3)
    scheds = configs.build_schedules(cfg, n_steps=n_total)
    rt = RingRuntime(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement, succ,
                     rank=rank, world=world, device=local_rank, spares=1, group=group,
                     sentinel=None)

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=local_rank)

    drv = ScheduleDriver(rt, scheds, coords, content)
    comp = torch.cuda.current_stream(dev)
    repl = comp if args.single_stream else torch.cuda.Stream(dev)

    order = StreamOrder(comp, repl)

    def step(t):
        order.before_append()
        drv.append_step(t, stream=comp)
        if t >= 1:
            order.before_publish()
            rt.replicate_all(t, stream=repl)
            order.after_publish()

    # ---- prelude: reach steady state (untimed) --------------------------------
    t = 0
    for _ in range(args.prelude):
        step(t)
        t += 1
    torch.cuda.synchronize(dev)

    # ---- pre-generate the sources of the warm-up + timed steps (inputs resident in HBM)
    def gen_sources(t0, n):
        out = {}
        for tt in range(t0, t0 + n):
            plan = drv.plan(tt)
            out[tt] = {}
            for node, e in plan.items():
                if node in rt.local:
                    ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                    out[tt][node] = content(e["stage"], ids, pos) if ids else None
        return out

    src = gen_sources(t, args.warmup + args.steps)
    src_bytes = sum(x.numel() * 2 for d in src.values() for x in d.values() if x is not None)
    # The per-step request events (which requests grow by how many tokens) are the
    # workload's input, planned and marshalled ahead like the sources; allocation,
    # work lists, H2D staging and launches all run inside the timed region
    # (kv_run_steps: the native decode loop, append on the compute stream, publish
    # on the replication stream).
    def prepare(t0, n, timing):
        # kernel-timing events on every TIME_EVERY-th step (each record is a host API
        # call inside the timed region; sampling keeps the host loop lean)
        steps, evs = [], []
        for tt in range(t0, t0 + n):
            plan = drv.plan(tt)
            app = [dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                        req_ids=e["req_ids"], n_new=e["n_new"], src=src[tt].get(node))
                   for node, e in plan.items() if node in rt.local]
            pools = [rt.handle(nd) for nd in rt.alive_local() if rt.succ.get(nd) is not None]
            st = dict(append=app, repl_pools=pools if tt >= 1 else [], step=tt)
            every = 8 if args.loop in ("pdl", "graph") else TIME_EVERY
            if timing and (args.timeline or (tt - t0) % every == every - 1):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                st.update(ev_call=ev[0], ev_kernel_start=ev[1], ev_kernel_end=ev[2])
                if args.timeline:
                    ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    st.update(ev_append_start=ea[0], ev_append_end=ea[1])
                    ev = ev + ea
                evs.append(ev)
            steps.append(st)
        return K.PreparedSteps(steps), evs

    warm, _ = prepare(t, args.warmup, False)
    timed, evs = prepare(t + args.warmup, args.steps, True)
    torch.cuda.synchronize(dev)
    if args.loop == "fused":
        K.kv_run_steps_fused(warm, comp.cuda_stream)
    elif args.loop == "pdl":
        K.kv_run_steps_pdl(warm, comp.cuda_stream)
    elif args.loop == "graph":
        K.kv_run_steps_graph(warm, comp.cuda_stream, repl.cuda_stream)
    else:
        K.kv_run_steps(warm, comp.cuda_stream, repl.cuda_stream)
    t += args.warmup
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    # ---- timed region -----------------------------------------------------------
    local_nodes = rt.alive_local()
    bytes0 = {n: K.kv_stats(rt.handle(n))["bytes_replicated"] for n in local_nodes}
    l0 = K.kv_kernel_launch_count()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_timed0 = t
    K.kv_host_profile(reset=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize(dev)
        w0 = time.perf_counter()
        start.record(comp)
        if args.loop == "fused":
            K.kv_run_steps_fused(timed, comp.cuda_stream)
        elif args.loop == "pdl":
            K.kv_run_steps_pdl(timed, comp.cuda_stream)
        elif args.loop == "graph":
            K.kv_run_steps_graph(timed, comp.cuda_stream, repl.cuda_stream)
        else:
            K.kv_run_steps(timed, comp.cuda_stream, repl.cuda_stream)
        fin = torch.cuda.Event()
        fin.record(repl)
        comp.wait_event(fin)
        end.record(comp)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - w0
    t += args.steps
    del src
    launches = K.kv_kernel_launch_count() - l0
    host_prof = {k: round(v / args.steps * (1.0 if k.startswith("n_") else 1e6), 2)
                 for k, v in K.kv_host_profile(reset=True).items()}
    ms = start.elapsed_time(end)
    kern_us = [e[1].elapsed_time(e[2]) * 1e3 for e in evs]
    rep_us = kern_us if args.loop in ("fused", "pdl", "graph") else [e[0].elapsed_time(e[2]) * 1e3
                                                           for e in evs]
    if args.timeline and rank == 0:
        T = lambda e: start.elapsed_time(e) * 1e3
        print("TIMELINE us: append [start,end] (compute stream) | ring-put [start,end] "
              "(replication stream); host wall %.1f us/step" % (wall / args.steps * 1e6),
              file=sys.stderr)
        for k, e in enumerate(evs[:80]):
            a0, a1 = (T(e[3]), T(e[4])) if len(e) > 3 else (0, 0)
            print("  step %3d  append %8.1f %8.1f (%5.1f)  ringput %8.1f %8.1f (%5.1f)"
                  % (k, a0, a1, a1 - a0, T(e[1]), T(e[2]), T(e[2]) - T(e[1])), file=sys.stderr)
    step_bytes = {n: K.kv_stats(rt.handle(n))["bytes_replicated"] - bytes0[n] for n in local_nodes}
    my_bytes = float(sum(step_bytes.values()))

    # ---- e2e: host-resident inputs (pinned), H2D + D2H inside the timed region ---
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, drv, rt, t, comp, repl, content, dev, world)
        t += args.e2e_steps

    # ---- NCCL comparison (a6): same workload, pack -> count -> send/recv -> unpack ---
    nccl = None
    if args.nccl_steps > 0:
        nccl = run_nccl(args, drv, rt, t, comp, content, dev, world)
        t += args.nccl_steps

    # ---- interference with a decode proxy (NEXT-4; the paper's overhead) ----
    interference = None
    if args.interference_steps > 0:
        interference = run_interference(args, drv, rt, t, comp, repl, content, dev, world)
        t += 2 * args.interference_steps

    # ---- block-granular mode (NEXT-2): completed blocks only ---------------------
    block = None
    if args.block_steps > 0:
        block = run_block_mode(args, drv, rt, t, comp, repl, content, dev, world)
        t += args.block_steps + 1

    # ---- floor of a decode hop: a publication with nothing dirty ("empty
    # launch + one P2P flag store"), same pools, same stream, same launch path; the
    # last leg that replicates on these pools (its step numbers are not schedule steps)
    floor = run_floor(rt, t + 10, comp, repl, dev, world,
                      "graph" if args.loop == "graph" else "streams")

    # ---- restore: fail stage 2 of pipeline 0, restore into a fresh pool ---------
    restore = None
    if not args.no_restore:
        restore = run_restore(drv, rt, t, dev, comp, world)

    # ---- bulk leg (C5: 32k-token prefill per stage, full-block re-seed) -----------
    pool_gib = rt.n_slots * 2 * rt.replica_bytes / 2**30
    rt.destroy()
    del rt, drv
    torch.cuda.empty_cache()
    bulk = run_bulk(args, rank, world, local_rank, dev, group) if args.bulk_reps > 0 else None

    # ---- shared capacity (NEXT-3): replicas in the holder's own pool, under pressure -
    shared = None
    if args.shared_steps > 0:
        shared = (run_shared(args, local_rank, dev) if world == 1 else
                  {"skipped": "shared capacity needs the holder on the same GPU (N = 1)"})

    # ---- reduce over ranks --------------------------------------------------------
    vec = torch.tensor([ms, my_bytes, float(launches), wall], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, tot_bytes, tot_launch = float(mx[0]), float(sm[1]), int(sm[2])
    else:
        ms_max, tot_bytes, tot_launch = ms, my_bytes, launches

    hbm_peak, peak_src = peaks()
    med_kern = statistics.median(kern_us)
    avg_kern = sum(kern_us) / len(kern_us)
    if args.loop == "fused":
        # kv_step_fused_kernel: append of step k (D_k read from the dense source + D_k
        # written into the pool) and publication of step k-1 (D_{k-1} read + written);
        # over the timed run appended bytes == published bytes == my_bytes, in K+1 launches
        n_launch = args.steps + 1
        kname = "kv_step_fused_kernel"
        if N == 1:
            per = 4 * my_bytes / n_launch
            achieved = per / (avg_kern * 1e-6) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved / hbm_peak, 4), "traffic": None, "kernel": kname,
                    "peak_source": peak_src, "algorithmic_bytes_per_launch": int(per),
                    "avg_launch_us": round(avg_kern, 2),
                    "what": "append k (D r+w) + publication k-1 (D r+w) per launch, HBM"}
        else:
            per = my_bytes / n_launch
            achieved = per / (avg_kern * 1e-6) / 1e9
            roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS,
                    "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK_GBS, 4), "traffic": None,
                    "kernel": kname,
                    "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction",
                    "algorithmic_bytes_per_launch": int(per), "avg_launch_us": round(avg_kern, 2),
                    "what": "NVLink bytes of the publication part per launch"}
    # ring-put algorithmic bytes per launch: D read + D written (HBM at N=1; at N>1
    # the write crosses NVLink -- reported against the NVLink per-direction peak)
    elif N == 1:
        per_launch = my_bytes / args.steps
        achieved = 2 * per_launch / (avg_kern * 1e-6) / 1e9
        pop = traffic_ref("decode_population", "kv_ring_put_copy_kernel") if args.loop == "graph" else None
        tr = (traffic_ref("decode_step", "kv_ring_put_copy_kernel") if args.loop == "graph"
              else traffic_ref("decode_step", "kv_ring_put_inl_kernel"))
        if pop:  # per-launch average over a population of this loop's copy-node launches
            tnote = ("ncu --set full over %d consecutive copy-node launches of this bench loop "
                     "(profiles/traffic.json decode_population): avg DRAM bytes/launch %d (read %d, "
                     "write %d) vs avg algorithmic r+w %d (L2 bytes the kernel requested) = %.2f; "
                     "no re-reads, most replica writes stay in L2"
                     % (pop["n_launches"], pop["traffic"], pop["dram_read"], pop["dram_write"],
                        pop["algorithmic_rw"], pop["traffic_over_algorithmic"]))
        elif tr:
            tnote = ("ncu --set full of a decode-step launch (profiles/traffic.json): "
                     "DRAM bytes %d vs algorithmic read %d / r+w %d; writes stay in L2"
                     % (tr["traffic"], tr["algorithmic_read"], tr["algorithmic_rw"]))
        else:
            tnote = None
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4),
                "traffic": pop["traffic"] if pop else (tr["traffic"] if tr else None),
                "traffic_note": tnote,
                "kernel": RINGPUT_GRAPH if args.loop == "graph" else RINGPUT,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": int(2 * per_launch),
                "avg_launch_us": round(avg_kern, 2)}
    else:
        per_launch = my_bytes / args.steps
        achieved = per_launch / (avg_kern * 1e-6) / 1e9
        tr = traffic_ref("decode_step_nvlink", "kv_ring_put_inl_kernel")
        roof = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS,
                "unit": "GB/s", "frac": round(achieved / NVLINK_PEAK_GBS, 4),
                "traffic": (tr["dram_read"] if tr else None),
                "nvlink_traffic_note": ("ncu of a decode-only launch (tools/nvlink_profile.py, "
                                        "profiles/traffic.json): nvltx user bytes %d / wire "
                                        "bytes %d vs algorithmic %d"
                                        % (tr["nvltx_bytes_data_user"], tr["nvltx_bytes"],
                                           tr["algorithmic_nvlink"])) if tr else None,
                "kernel": RINGPUT,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction",
                "algorithmic_bytes_per_launch": int(per_launch), "avg_launch_us": round(avg_kern, 2)}
    value = tot_bytes / (ms_max * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (ShareGPT-shaped lognormal trace, closed-form KV words)",
        "config": bench_config(N),
        "dtype_note": "bf16 KV words moved bit-exactly as 16-bit data (no arithmetic)",
        "run": {"timed_steps": [t_timed0, t_timed0 + args.steps - 1], "loop": args.loop,
                "inputs_gib": {"pre_generated_sources": round(src_bytes / 2**30, 2),
                               "pools_and_replicas_per_gpu": round(pool_gib, 1)},
                "streams": "single" if args.single_stream else "compute+replication"},
        "gb_s_per_gpu": round(value / N, 2),
        "replicated_bytes": int(tot_bytes),
        "loop": args.loop,
        "step_overhead_us": {"median": round(statistics.median(rep_us), 2),
                             "p99": round(float(np.percentile(rep_us, 99)), 2),
                             "budget_us": 400.0, "tpot_ms": 20.0,
                             "fused_loop_note": ("with the fused loop this is the whole fused "
                                                 "launch (append + publication); the replication "
                                                 "overhead proper is the interference leg")
                             if args.loop == "fused" else None,
                             "what": "replication-stream device time per step (ring-put kernel incl. "
                                     "its launch and its wait for the step's append), CUDA events "
                                     "recorded by the decode loop on every %d-th timed step"
                                     % (8 if args.loop in ("pdl", "graph") else TIME_EVERY)},
        "kernel_us": {"kernel": "kv_step_fused_kernel" if args.loop == "fused"
                      else (RINGPUT_GRAPH if args.loop == "graph" else RINGPUT),
                      "median": round(med_kern, 2), "avg": round(avg_kern, 2),
                      "sampled_launches": len(kern_us)},
        "roofline": roof,
        "step_roofline": step_roofline(tot_bytes, ms_max, N, hbm_peak, peak_src),
        "gpu_launches": int(tot_launch),
        "wall_s_timed": round(wall, 3),
        "host_us_per_step": host_prof,
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    line["step_floor_us"] = floor
    if restore is not None:
        line["restore"] = restore
    if bulk is not None:
        line["bulk"] = bulk
    if nccl is not None:
        line["nccl_compare"] = nccl
    if interference is not None:
        line["interference"] = interference
    if block is not None:
        line["block_mode"] = block
    if shared is not None:
        line["shared_capacity"] = shared
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, t_timed0, min(args.steps, 60))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_bulk(args, rank, world, local_rank, dev, group):
    """C5 (BASELINE configs[4]): 8 stages x 4 layers, one P = 32,768 request per stage
    (2,048 full blocks of 256 KiB = 512 MiB), stage s on GPU s mod N, all links
    replicating at once.  Each rep re-binds every link (pub_len = 0, full re-seed)
    and publishes one step: the full-block bulk copy, HBM loopback at N = 1, NVLink
    at N > 1.  Kernel time by CUDA events around each ring-put launch."""
    import torch
    import torch.distributed as dist
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime
    cfg = configs.C5
    g = cfg.geom
    S = cfg.stages
    placement = {s: s % world for s in range(S)}
    succ = {s: (s + 1) % S for s in range(S)}
    rt = RingRuntime(g, cfg.num_blocks, 2, cfg.max_blocks_per_req, placement, succ, rank=rank,
                     world=world, device=local_rank, spares=0, group=group, sentinel=None)
    P = cfg.fixed_prompt
    comp = torch.cuda.current_stream(dev)
    for s in rt.alive_local():
        src = content_tokens_cuda(CONTENT_SEED, [s] * P, range(P), s * g.layers, g.layers,
                                  g.kv_heads, g.head_dim, device=local_rank)
        K.kv_append(rt.handle(s), [s], [P], src, 0, comp.cuda_stream)
        torch.cuda.synchronize(dev)
        del src
    nodes = rt.alive_local()
    handles = [rt.handle(n) for n in nodes]
    D = P * g.token_bytes * len(nodes)
    times = []
    for rep in range(args.bulk_reps + 1):
        for n in nodes:
            rt.set_succ(n, succ[n])          # re-bind: the next publish re-seeds everything
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K.kv_time_next_launch(a, b)
        K.kv_replicate_step_multi(handles, rep + 1, comp.cuda_stream)
        torch.cuda.synchronize(dev)
        if rep > 0:                          # rep 0 is the warm-up
            times.append(a.elapsed_time(b))
    ms = statistics.median(times)
    vec = torch.tensor([ms, float(D)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, tot = float(mx[0]), float(sm[1])
    else:
        ms_max, tot = ms, float(D)
    # sampled check: the last published seq on this GPU's replica metadata
    seq_ok = all(int(rt.read_meta(n)["seq"]) == args.bulk_reps + 1 for n in nodes)
    # gather-pack (a4) and unpack (the NCCL receiver's scatter, a6) of the same bulk
    # payload, each a separate HBM-bound kernel (N = 1: the successor is local)
    pack = None
    if world == 1:
        bufs = {n: torch.empty(P * g.token_bytes + (8 << 20), dtype=torch.uint8, device=dev)
                for n in nodes}
        tp, tu = [], []
        step = args.bulk_reps + 2
        for rep in range(3):
            for n in nodes:
                rt.set_succ(n, succ[n])
            torch.cuda.synchronize(dev)
            sizes, evp, evu = {}, [], []
            for n in nodes:           # kernel-only events (descriptor staging excluded)
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                K.kv_time_next_launch(e[0], e[1])
                sizes[n] = K.kv_pack_step(rt.handle(n), step, bufs[n], bufs[n].numel(),
                                          comp.cuda_stream)
                evp.append(e)
            for n in nodes:
                m = succ[n]
                e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                K.kv_time_next_launch(e[0], e[1])
                K.kv_unpack(bufs[n], sizes[n], rt.local[m].replica, rt.NB, rt.local[m].meta,
                            rt.kg, rt.R, rt.M, comp.cuda_stream)
                evu.append(e)
            torch.cuda.synchronize(dev)
            step += 1
            if rep > 0:
                tp.append(sum(x.elapsed_time(y) for x, y in evp))
                tu.append(sum(x.elapsed_time(y) for x, y in evu))
        pack_ok = all(int(rt.read_meta(n)["seq"]) == step - 1 for n in nodes)
        hbm_peak, _ = peaks()
        mp, mu = statistics.median(tp), statistics.median(tu)
        pack = {"gather_pack": {"ms": round(mp, 4), "gb_s_rw": round(2 * D / (mp * 1e-3) / 1e9, 1),
                                "frac_hbm": round(2 * D / (mp * 1e-3) / 1e9 / hbm_peak, 4),
                                "kernels": len(nodes), "what": "sum of the gather-pack kernel times of "
                                "every stage (CUDA events around each kernel), paged -> contiguous"},
                "unpack": {"ms": round(mu, 4), "gb_s_rw": round(2 * D / (mu * 1e-3) / 1e9, 1),
                           "frac_hbm": round(2 * D / (mu * 1e-3) / 1e9 / hbm_peak, 4),
                           "kernels": len(nodes), "what": "sum of the unpack kernel times (into each "
                           "successor's replica + publish), contiguous -> paged"},
                "seq_ok": pack_ok}
        del bufs
    # copy-engine variant (NEXT-4): the same full-block re-seed moved by cudaMemcpyAsync
    # runs (zero SMs for the payload), the ring-put kernel writing the bt entries and
    # publishing after them; events around the whole call on the stream
    tce = []
    step0 = args.bulk_reps + 10
    for rep in range(args.bulk_reps + 1):
        for n in nodes:
            rt.set_succ(n, succ[n])
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(comp)
        K.kv_replicate_step_ce(handles, step0 + rep, comp.cuda_stream)
        b.record(comp)
        torch.cuda.synchronize(dev)
        if rep > 0:
            tce.append(a.elapsed_time(b))
    mce = statistics.median(tce)
    ce_ok = all(int(rt.read_meta(n)["seq"]) == step0 + args.bulk_reps for n in nodes)
    vce = torch.tensor([mce], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vce, op=dist.ReduceOp.MAX)
    mce_max = float(vce[0])
    ce = {"ms_median": round(mce, 4), "ms_max_over_ranks": round(mce_max, 4),
          "replicated_gb_s_total": round(tot / (mce_max * 1e-3) / 1e9, 1),
          "what": "kv_replicate_step_ce: one cudaMemcpyAsync per run of consecutive full "
                  "blocks + the publishing ring-put kernel; events around the whole call",
          "seq_ok": ce_ok}
    rt.destroy()
    hbm_peak, src_peak = peaks()
    per_gpu = D / (ms * 1e-3) / 1e9
    if world == 1:
        ach = 2 * D / (ms * 1e-3) / 1e9
        tr = traffic_ref("bulk_c5")
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "peak_source": src_peak,
                "algorithmic_bytes_per_launch": int(2 * D),
                "traffic": tr["traffic"] if tr else None}
    else:
        roof = {"bound": "nvlink", "achieved": round(per_gpu, 1), "peak": NVLINK_PEAK_GBS,
                "unit": "GB/s", "frac": round(per_gpu / NVLINK_PEAK_GBS, 4),
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction",
                "algorithmic_bytes_per_launch": int(D)}
    return {"workload": "c5_bulk_32k", "stages": S, "stages_per_gpu": len(nodes),
            "bytes_per_link": int(P * g.token_bytes), "kernel_ms_median": round(ms, 4),
            "kernel_ms_max_over_ranks": round(ms_max, 4),
            "replicated_gb_s_total": round(tot / (ms_max * 1e-3) / 1e9, 1),
            "roofline": roof, "reps": args.bulk_reps, "seq_ok": seq_ok,
            "pack_unpack": pack, "copy_engine": ce}


class DecodeProxy:
    """Llama-3.1-8B pipeline-stage decode proxy: per local stage, L_s = 8 layers of
    bf16 GEMMs at the step's batch (QKV 4096x6144, O 4096x4096, gate/up 4096x28672,
    down 14336x4096, SiLU-gated), random weights, captured in one CUDA graph.  It
    stands in for the model compute the replication must overlap."""

    def __init__(self, n_stages, layers, batch, dev):
        import torch
        g = torch.Generator(device=dev).manual_seed(1234)
        mk = lambda *sh: (torch.randn(*sh, device=dev, dtype=torch.bfloat16, generator=g) * 0.02)
        self.w = [[(mk(4096, 6144), mk(4096, 4096), mk(4096, 28672), mk(14336, 4096))
                   for _ in range(layers)] for _ in range(n_stages)]
        self.x = mk(batch, 4096)
        self.graph = None
        self.dev = dev

    def _forward(self):
        import torch
        for stage in self.w:
            x = self.x
            for wqkv, wo, wup, wdown in stage:
                q = x @ wqkv
                o = q[:, :4096] @ wo
                u = o @ wup
                x = (torch.nn.functional.silu(u[:, :14336]) * u[:, 14336:]) @ wdown
            self.out = x

    def capture(self, stream):
        import torch
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            for _ in range(2):
                self._forward()
        stream.wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=s):
            self._forward()
        stream.wait_stream(s)

    def replay(self):
        self.graph.replay()


def run_interference(args, drv, rt, t0, comp, repl, content, dev, world):
    """Per step: decode proxy (compute stream) -> append (the model's KV write) ->
    publication on the replication stream.  Phase A replicates every step, phase B
    does not; overhead = step time A - step time B (compute-stream CUDA events)."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    n = args.interference_steps
    nodes = rt.alive_local()
    proxy = DecodeProxy(len(nodes), rt.g.layers, 64, dev)
    proxy.capture(comp)
    srcs, plans = {}, {}
    for tt in range(t0, t0 + 2 * n):
        plans[tt] = drv.plan(tt)
        srcs[tt] = {nd: (content(e["stage"], *drv.tokens(e["req_ids"], e["n_new"], e["start"]))
                         if e["req_ids"] else None)
                    for nd, e in plans[tt].items() if nd in rt.local}
    handles = [rt.handle(nd) for nd in nodes if rt.succ.get(nd) is not None]

    def prep(tt, replicate):
        app = [dict(pool=rt.handle(nd), begin_step=1, release=e["release"], req_ids=e["req_ids"],
                    n_new=e["n_new"], src=srcs[tt].get(nd))
               for nd, e in plans[tt].items() if nd in rt.local]
        return K.PreparedSteps([dict(append=app, repl_pools=handles if replicate else [],
                                     step=tt)])

    # alternate blocks of BLK steps with and without replication so clock / thermal drift
    # cancels; the first step of an "on" block also publishes the previous "off" block's
    # backlog (counted against replication: conservative)
    BLK = 10
    per = {"on": [], "off": []}
    torch.cuda.synchronize(dev)
    k = 0
    while k < 2 * n:
        for phase, replicate in (("on", True), ("off", False)):
            m = min(BLK, 2 * n - k)
            if m <= 0:
                break
            preps = [prep(t0 + k + i, replicate) for i in range(m)]
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(m + 1)]
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            for i in range(m):
                ev[i].record(comp)
                proxy.replay()
                K.kv_run_steps(preps[i], comp.cuda_stream, repl.cuda_stream)
            fin = torch.cuda.Event()
            fin.record(repl)
            comp.wait_event(fin)
            ev[m].record(comp)
            torch.cuda.synchronize(dev)
            per[phase].extend(ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(m))
            k += m
    out = {ph: {"median_us": round(statistics.median(v), 2), "mean_us": round(sum(v) / len(v), 2),
                "steps": len(v)} for ph, v in per.items()}
    a, b = out["on"]["median_us"], out["off"]["median_us"]
    return {"proxy": "Llama-3.1-8B stage decode proxy: %d stages x %d layers of bf16 GEMMs at "
                     "batch 64 (CUDA graph) on the compute stream" % (len(nodes), rt.g.layers),
            "step_us_with_replication": out["on"], "step_us_without_replication": out["off"],
            "overhead_us": round(a - b, 2), "overhead_pct": round(100.0 * (a - b) / b, 3),
            "paper": "+2.3 % avg / +2.8 % p99 latency (8 A10 nodes), +4.0 % / +3.6 % (16) "
                     "over 1 Gbps, P:99 -- context, not the target",
            "steps": 2 * n, "blocks_of": BLK}


def run_block_mode(args, drv, rt, t0, comp, repl, content, dev, world):
    """NEXT-2: the paper's literal "replicate it block-by-block": only completed
    16-token blocks are published (whole contiguous 512-KiB blocks instead of 256-B
    token slices); the replica lags < 16 tokens per request.  One re-seed step after
    the switch, then K timed steps through kv_run_steps."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    nodes = rt.alive_local()
    for nd in nodes:
        K.kv_set_mode(rt.handle(nd), K.KV_MODE_BLOCKS)
    n = args.block_steps
    handles = [rt.handle(nd) for nd in nodes if rt.succ.get(nd) is not None]
    steps, evs = [], []
    for k, tt in enumerate(range(t0, t0 + n + 1)):
        plan = drv.plan(tt)
        app = []
        for nd, e in plan.items():
            if nd in rt.local:
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                app.append(dict(pool=rt.handle(nd), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"],
                                src=content(e["stage"], ids, pos) if ids else None))
        st = dict(append=app, repl_pools=handles, step=tt)
        if k > 0 and k % TIME_EVERY == 0:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            st.update(ev_call=ev[0], ev_kernel_start=ev[1], ev_kernel_end=ev[2])
            evs.append(ev)
        steps.append(st)
    reseed = K.PreparedSteps(steps[:1])
    timed = K.PreparedSteps(steps[1:])
    K.kv_run_steps(reseed, comp.cuda_stream, repl.cuda_stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    b0 = {nd: K.kv_stats(rt.handle(nd))["bytes_replicated"] for nd in nodes}
    st_, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st_.record(comp)
    K.kv_run_steps(timed, comp.cuda_stream, repl.cuda_stream)
    fin = torch.cuda.Event()
    fin.record(repl)
    comp.wait_event(fin)
    en.record(comp)
    torch.cuda.synchronize(dev)
    ms = st_.elapsed_time(en)
    by = sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in nodes)
    kern = [b.elapsed_time(c) * 1e3 for a, b, c in evs]
    lags = []
    for nd in nodes:
        req, ln, pub, nb = K.kv_dump_slots(rt.handle(nd), rt.R)
        lags.extend(int(a - b) for a, b, r in zip(ln, pub, req) if r >= 0)
    vec = torch.tensor([ms, float(by)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, by = float(mx[0]), float(sm[1])
    return {"mode": "blocks (completed 16-token blocks only)", "steps": n,
            "value": round(by / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "ms_per_step": round(ms / n, 4),
            "ring_put_kernel_us": {"median": round(statistics.median(kern), 2),
                                   "avg": round(sum(kern) / len(kern), 2)},
            "replica_lag_tokens": {"mean": round(float(np.mean(lags)), 2) if lags else 0.0,
                                   "max": int(max(lags)) if lags else 0}}


FLOOR_REPS = 50


def run_floor(rt, t0, comp, repl, dev, world, loop="streams"):
    """Per-step floor of the publication on the timed loop's own path: FLOOR_REPS steps
    of kv_run_steps with no append and nothing dirty (one publish-only task per pool:
    bt / parity table / release seq, over NVLink when the successor is remote), timed
    exactly like step_overhead_us (events from before the publication to after its
    kernel, on the replication stream; max over ranks).  The decode-step ring-put is
    compared with it."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    nodes = [n for n in rt.alive_local() if rt.succ.get(n) is not None]
    handles = [rt.handle(n) for n in nodes]
    sts, evs = [], []
    for k in range(FLOOR_REPS + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        evs.append(ev)
        sts.append(dict(append=[], repl_pools=handles, step=t0 + k, ev_call=ev[0],
                        ev_kernel_start=ev[1], ev_kernel_end=ev[2]))
    prep = K.PreparedSteps(sts)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    if loop == "graph":
        K.kv_run_steps_graph(prep, comp.cuda_stream, repl.cuda_stream)
    else:
        K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
    torch.cuda.synchronize(dev)
    # graph loop: ev_call is not recorded (events sit around the ring-put node only)
    i0 = 1 if loop == "graph" else 0
    call = sorted(e[i0].elapsed_time(e[2]) * 1e3 for e in evs[1:])
    kern = sorted(e[1].elapsed_time(e[2]) * 1e3 for e in evs[1:])
    v = torch.tensor([call[len(call) // 2], kern[len(kern) // 2]], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return {"median": round(float(v[0]), 2), "kernel_median": round(float(v[1]), 2),
            "reps": FLOOR_REPS, "pools": len(nodes),
            "what": "steps with nothing dirty through the timed loop's own decode loop (%s; "
                    "one publish-only task per pool: launch / graph node + bt/parity tables + "
                    "seq), timed like step_overhead_us (median) and kernel_us (kernel_median); "
                    "the decode-step ring-put's floor" % ("kv_run_steps_graph" if loop == "graph"
                                                         else "kv_run_steps")}


SHARED_NB = 2048   # C2 primary peak is ~1.57k blocks per stage: replicas must compete


def run_shared(args, local_rank, dev):
    """NEXT-3 (§3.2, reading R17): C2 on one GPU with each
    stage's pool cut to SHARED_NB blocks (1 GiB) and its ring predecessor's replica
    kept INSIDE that pool (kv_set_successor_shared): replica blocks come from the
    holder's free list; the holder evicts them, oldest request first, when its own
    appends need the memory, and a replica that cannot grow is dropped.  Prelude on
    one stream, then K timed steps through kv_run_steps (two streams).  Reports the
    replicated throughput, evictions, drops, the share of live requests that still
    have a published replica, and the HBM the pools take (vs. a dedicated mirror)."""
    import torch
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    n = args.shared_steps
    cfg = configs.scaled(configs.C2, num_blocks=SHARED_NB)
    g = cfg.geom
    S = cfg.stages
    coords = {(0, s): s for s in range(S)}
    placement = {s: 0 for s in range(S)}
    succ = {s: (s + 1) % S for s in range(S)}
    scheds = configs.build_schedules(cfg, n_steps=args.prelude + n + 2)
    rt = RingRuntime(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement, succ,
                     device=local_rank, spares=0, sentinel=None, shared=True)

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=local_rank)

    drv = ScheduleDriver(rt, scheds, coords, content)
    comp = torch.cuda.current_stream(dev)
    repl = torch.cuda.Stream(dev)
    for t in range(args.prelude):                 # one stream: trivially ordered
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
    torch.cuda.synchronize(dev)
    nodes = rt.alive_local()
    handles = [rt.handle(nd) for nd in nodes]
    steps, keep = [], []
    for tt in range(args.prelude, args.prelude + n):
        app = []
        for nd, e in drv.plan(tt).items():
            ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
            src = content(e["stage"], ids, pos) if ids else None
            keep.append(src)
            app.append(dict(pool=rt.handle(nd), begin_step=1, release=e["release"],
                            req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        steps.append(dict(append=app, repl_pools=handles, step=tt))
    prep = K.PreparedSteps(steps)
    st0 = {nd: K.kv_stats(rt.handle(nd)) for nd in nodes}
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comp)
    K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
    fin = torch.cuda.Event()
    fin.record(repl)
    comp.wait_event(fin)
    b.record(comp)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b)
    st1 = {nd: K.kv_stats(rt.handle(nd)) for nd in nodes}
    by = sum(st1[nd]["bytes_replicated"] - st0[nd]["bytes_replicated"] for nd in nodes)
    live = covered = 0
    for nd in nodes:                              # published replica coverage at the end
        req, ln, pub, nb = K.kv_dump_slots(rt.handle(nd), rt.R)
        meta = rt.read_meta(succ[nd])
        par = meta["seq"] & 1
        published = {int(r) for r in meta["req"][par] if r >= 0}
        for r in req:
            if r >= 0:
                live += 1
                covered += int(int(r) in published)
    pool_gib = S * SHARED_NB * rt.block_bytes / 2**30
    out = {"workload": "c2_pp4_b64 on 1 GPU, pools cut to %d blocks (shared capacity)" % SHARED_NB,
           "steps": n, "value": round(by / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
           "ms_per_step": round(ms / n, 4),
           "evictions": {nd: int(st1[nd]["replica_evictions"] - st0[nd]["replica_evictions"])
                         for nd in nodes},
           "drops": {nd: int(st1[nd]["replica_drops"] - st0[nd]["replica_drops"]) for nd in nodes},
           "replica_blocks_held_end": {nd: int(st1[nd]["replica_blocks_held"]) for nd in nodes},
           "live_requests_with_published_replica": round(covered / max(1, live), 4),
           "admissions_rejected": 0, "rejected_note": "the driver raises on KV_ENOMEM",
           "pool_hbm_gib": round(pool_gib, 2),
           "dedicated_mirror_hbm_gib_same_primary": round(2 * pool_gib, 2)}
    rt.destroy()
    del keep
    torch.cuda.empty_cache()
    return out


def run_nccl(args, drv, rt, t0, comp, content, dev, world):
    """The paper's transport (NCCL send/recv, P:8 §3.3) on the same workload, as the
    measured comparison: per step append, then gather-pack, 8-B count exchange,
    grouped send/recv, unpack + publish.  One stream; per-step transport time by
    CUDA events around pack..unpack."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.nccl_compare import NcclRing
    n = args.nccl_steps
    ring = NcclRing(rt, 256 << 20)
    srcs, plans = {}, {}
    for tt in range(t0, t0 + n):
        plans[tt] = drv.plan(tt)
        srcs[tt] = {}
        for node, e in plans[tt].items():
            if node in rt.local:
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                srcs[tt][node] = content(e["stage"], ids, pos) if ids else None
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n)]
    b0 = {nd: K.kv_stats(rt.handle(nd))["bytes_replicated"] for nd in rt.alive_local()}
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    st.record(comp)
    for k in range(n):
        tt = t0 + k
        drv.append_step(tt, stream=comp, sources=srcs[tt], plan=plans[tt])
        evs[k][0].record(comp)
        ring.step(tt, comp)
        evs[k][1].record(comp)
    en.record(comp)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - w0
    ms = st.elapsed_time(en)
    by = sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in rt.alive_local())
    us = [a.elapsed_time(b) * 1e3 for a, b in evs]
    vec = torch.tensor([ms, float(by), wall], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, by, wall = float(mx[0]), float(sm[1]), float(mx[2])
    return {"transport": "nccl send/recv (pack, count exchange, send/recv, unpack)" if world > 1
            else "loopback pack -> unpack (no NCCL at N=1)",
            "value": round(by / (ms * 1e-3) / 1e9, 2), "unit": UNIT, "steps": n,
            "ms_per_step": round(ms / n, 4), "wall_ms_per_step": round(wall / n * 1e3, 4),
            "transport_us_per_step": {"median": round(statistics.median(us), 2),
                                      "p99": round(float(np.percentile(us, 99)), 2)}}


def _append_host(drv, t, host_sources, stream):
    """kv_append_multi with KV_SRC_HOST: the library copies the pinned host KV."""
    from paper_2601_22438_b200 import kvring as K
    entries = []
    for node, e in drv.plan(t).items():
        if node not in drv.rt.local:
            continue
        src = host_sources.get(node) if host_sources else None
        entries.append(dict(node=node, begin_step=1, release=e["release"], req_ids=e["req_ids"],
                            n_new=e["n_new"], src=src, flags=K.KV_SRC_HOST))
    drv.rt.append_all(entries, stream)


def run_e2e(args, drv, rt, t0, comp, repl, content, dev, world):
    """Same metric through the C ABI with HOST buffers: per step the new-token KV is
    copied from pinned host memory by kv_append (KV_SRC_HOST) and the published seq
    flags of the successors are read back to pinned host memory."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import StreamOrder
    n = args.e2e_steps
    host = {}
    h2d = 0
    for tt in range(t0, t0 + n):
        host[tt] = {}
        for node, e in drv.plan(tt).items():
            if node in rt.local:
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                if ids:
                    d = content(e["stage"], ids, pos)
                    hbuf = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
                    hbuf.copy_(d)
                    host[tt][node] = hbuf
                    h2d += d.numel() * 2
    torch.cuda.synchronize(dev)
    nodes = rt.alive_local()
    # the step's result on this GPU: the seq flags its nodes' predecessors published into
    # this GPU's replica metadata (local memory whatever the ring placement)
    seq_dev = [rt.local[nd].meta[:8] for nd in nodes]
    seq_host = torch.empty((n, len(nodes), 8), dtype=torch.uint8, pin_memory=True)
    d2h = 0
    b0 = {nd: K.kv_stats(rt.handle(nd))["bytes_replicated"] for nd in nodes}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    st.record(comp)
    order = StreamOrder(comp, repl)
    for k in range(n):
        tt = t0 + k
        order.before_append()
        _append_host(drv, tt, host[tt], comp)
        order.before_publish()
        rt.replicate_all(tt, stream=repl)
        order.after_publish()
        with torch.cuda.stream(repl):
            for i, sd in enumerate(seq_dev):
                if sd is not None:
                    seq_host[k, i].copy_(sd, non_blocking=True)
                    d2h += 8
    fin = torch.cuda.Event()
    fin.record(repl)
    comp.wait_event(fin)
    en.record(comp)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - w0
    ms = st.elapsed_time(en)
    by = sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in nodes)
    vec = torch.tensor([ms, float(by)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vec.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vec.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, by = float(mx[0]), float(sm[1])
    # per-step read-backs are not synchronised with the remote writers (one-sided
    # publication); after a barrier every local replica must hold the last step
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ok = bool(all(int(sd.cpu().numpy().view(np.uint64)[0]) == t0 + n - 1 for sd in seq_dev))
    if world > 1:
        dist.barrier()
    return {"value": round(by / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d // n), "d2h_bytes_per_step": int(d2h // n),
            "steps": n, "ms_per_step": round(ms / n, 4), "wall_s": round(wall, 3),
            "seq_readback_ok": ok,
            "path": "kv_append_multi(KV_SRC_HOST) on pinned host tensors (the scatter kernel "
                    "reads them over PCIe, zero copy) + kv_replicate_step_multi; per step a "
                    "D2H read-back of the published seq flags"}


def run_restore(drv, rt, t, dev, stream, world=1):
    """Fail stage 2 of pipeline 0 after the last step and restore its pool + block table
    from its successor's replica into a fresh pool: on the holder's GPU at N = 1 (local
    HBM), on the NEXT GPU at N > 1 (the replica is read over NVLink: a remote restore)."""
    import torch
    import torch.distributed as dist
    from paper_2601_22438_b200 import kvring as K
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    f = drv.coords[(0, 2)]
    holder = rt.succ[f]
    rt.fail(f, stream)
    dst = drv.next_node
    drv.next_node += 1
    dst_rank = rt.placement[holder] if world == 1 else (rt.placement[holder] + 1) % world
    rt.new_node(dst, dst_rank)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    res = torch.zeros(5, dtype=torch.float64, device=dev)
    if dst in rt.local:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K.kv_time_next_launch(a, b)
        w0 = time.perf_counter()
        t_star, restored = rt.restore(dst, holder, stream)
        torch.cuda.synchronize(dev)
        wall_ms = (time.perf_counter() - w0) * 1e3
        tok = sum(ln for _, ln in restored)
        R = tok * rt.g.layers * 2 * rt.g.kv_heads * rt.g.head_dim * 2
        res = torch.tensor([wall_ms, a.elapsed_time(b), float(t_star), float(len(restored)),
                            float(R)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(res, op=dist.ReduceOp.SUM)   # only dst's rank contributes
    wall_ms, kern_ms, t_star, nreq, R = [float(x) for x in res.tolist()]
    hbm_peak, _ = peaks()
    out = {"ms": round(wall_ms, 3), "kernel_ms": round(kern_ms, 3), "t_star": int(t_star),
           "requests": int(nreq), "restored_bytes": int(R)}
    if world == 1:
        gbs = 2 * R / (kern_ms * 1e-3) / 1e9
        out.update(kernel_gb_s_rw=round(gbs, 1), frac_hbm=round(gbs / hbm_peak, 4),
                   path="local HBM (fresh pool on the holder's GPU)")
    else:
        gbs = R / (kern_ms * 1e-3) / 1e9
        out.update(kernel_gb_s_nvlink=round(gbs, 1), frac_nvlink=round(gbs / NVLINK_PEAK_GBS, 4),
                   path="remote: fresh pool on GPU %d reads the holder's replica on GPU %d "
                        "over NVLink" % (dst_rank, rt.placement[holder]))
    return out


# --------------------------------------------------------------------------- CPU arms
def oracle_sample(cfg, t_start: int, n_steps: int, warmup: int = 0):
    """Time the CPU oracle (as it stands) over steps [t_start, t_start+n) of the same
    workload.  Steps before t_start run in metadata mode to reach the same state;
    the sampled steps run with content (numpy copies), sources pre-generated."""
    from kvgen.configs import build_schedules
    from kvgen.content import CONTENT_SEED, content_tokens
    from oracle.simulate import OracleRing
    from kvgen.configs import scaled
    n_total = warmup + n_steps          # content-mode steps: warm-up (untimed) + timed
    scheds = build_schedules(cfg, n_steps=t_start + n_total + 1)
    # metadata-only pass over the whole sample to find the highest block id used,
    # so the sampled pools hold exactly the blocks the workload touches
    meta = OracleRing(cfg, content=False, schedules=scheds)
    peak = 0
    for tt in range(t_start + n_total):
        meta.appends(tt)
        if tt >= 1:
            meta.replicate(tt)
        peak = max([peak] + [b for n in meta.nodes.values() for s in range(n.R) for b in n.slot_bt[s]])
    small = scaled(cfg, num_blocks=min(cfg.num_blocks, int(peak) + 1))
    ring = OracleRing(small, content=False, schedules=scheds)
    for tt in range(t_start):
        ring.appends(tt)
        if tt >= 1:
            ring.replicate(tt)
    # switch to content mode for the sampled steps: the dirty tokens they copy
    # are the closed-form words appended during the sample
    g = small.geom
    shape = (small.num_blocks, g.layers, 2, g.kv_heads, g.block_size, g.head_dim)
    for c, n in ring.nodes.items():
        n.content = True
        n.primary = np.full(shape, 0x5A5A, dtype=np.uint16)
        n.replica = np.full(shape, 0x5A5A, dtype=np.uint16)
    ring.content = True
    srcs = {}
    for tt in range(t_start, t_start + n_total):
        srcs[tt] = {}
        for c, n in ring.nodes.items():
            p, s = c
            ev = scheds[p].steps[tt]
            ids = sorted(ev.decode) + [r for r, _ in ev.admit]
            nn = [1] * len(ev.decode) + [pp for _, pp in ev.admit]
            starts = [scheds[p].length_at(r, tt - 1) for r in sorted(ev.decode)] + [0] * len(ev.admit)
            tid, tpos = [], []
            for r, k, p0 in zip(ids, nn, starts):
                tid.extend([r] * k)
                tpos.extend(range(p0, p0 + k))
            srcs[tt][c] = (ev.retire, ids, nn,
                           content_tokens(CONTENT_SEED, tid, tpos, s * g.layers, g.layers,
                                          g.kv_heads, g.head_dim))
    def one(tt):
        for c, n in ring.nodes.items():
            rel, ids, nn, src = srcs[tt][c]
            n.begin_step()
            n.release(rel)
            n.append(ids, nn, src)
        for c, n in ring.nodes.items():
            ring.moved += n.replicate(tt)

    for tt in range(t_start, t_start + warmup):
        one(tt)
    moved0 = ring.moved
    t0 = time.perf_counter()
    for tt in range(t_start + warmup, t_start + n_total):
        for c, n in ring.nodes.items():
            rel, ids, nn, src = srcs[tt][c]
            n.begin_step()
            n.release(rel)
            n.append(ids, nn, src)
        for c, n in ring.nodes.items():
            ring.moved += n.replicate(tt)
    dt = time.perf_counter() - t0
    return (ring.moved - moved0), dt


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, t_start, n_steps):
    """The oracle as it stands, pinned to ONE host core (SURVEY §8(d) oracle timing)."""
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    try:
        if aff:
            os.sched_setaffinity(0, {min(aff)})
        by, dt = oracle_sample(cfg, t_start, n_steps)
        return {"value": round(by / dt / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"{n_steps} steps ({t_start}..{t_start + n_steps - 1}) of {CFG_NAME}, "
                          f"one pipeline, numpy, pinned to one core",
                "seconds": round(dt, 3), "host_cpus": os.cpu_count(),
                "affinity_size": len(aff) if aff else None, "cpu_model": _cpu_model()}
    except Exception as e:  # the baseline is reported, never the target
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}
    finally:
        if aff:
            os.sched_setaffinity(0, aff)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from kvgen import configs
    cfg = configs.C2
    # the oracle as it stands (~14 ms per C2 step): K timed steps after W warm-up steps,
    # capped so the run stays within a few minutes
    n = max(1, min(args.steps, 400))
    w = max(0, min(args.warmup, 50))
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    if aff:
        os.sched_setaffinity(0, {min(aff)})      # one core, as the oracle timing asks
    by, dt = oracle_sample(cfg, args.prelude, n, warmup=w)
    value = by / dt / 1e9
    cores = os.cpu_count()
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": n, "warmup": w, "ms_per_step": round(dt / n * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (ShareGPT-shaped lognormal trace, closed-form KV words)",
            "impl": "reference",
            "config": bench_config(args.gpus),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{n} steps from step {args.prelude + w} of {CFG_NAME} "
                                       f"(one pipeline; the oracle as it stands, numpy, pinned "
                                       f"to one core); host has {cores} cores",
                             "cpu_model": _cpu_model()},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_kvring(args)


if __name__ == "__main__":
    main()
