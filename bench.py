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
    ap.add_argument("--bulk-reps", type=int, default=20, help="C5 bulk re-seed reps (0: skip)")
    ap.add_argument("--c4-restores", type=int, default=10,
                    help="C4 failover restores (configs[3]; 0: skip)")
    ap.add_argument("--interference-steps", type=int, default=100,
                    help="steps with a Llama-3.1-8B stage decode proxy on the compute stream, "
                         "replication on vs off (0: skip)")
    ap.add_argument("--block-steps", type=int, default=100,
                    help="steps in block-granular mode (NEXT-2), after a re-seed (0: skip)")
    ap.add_argument("--nccl-steps", type=int, default=100,
                    help="steps replicated through the NCCL send/recv comparison (0: skip)")
    ap.add_argument("--shared-steps", type=int, default=100,
                    help="timed steps of the shared-capacity leg (NEXT-3; N = 1 only; 0: skip)")
    ap.add_argument("--no-survey-layout", dest="survey_layout", action="store_false",
                    help="skip the SURVEY §8(e) one-stage-per-GPU layout leg at N > 1")
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

    def align(self, timeout: float = 0.5):
        """Returns right after the next sample arrives: a sub-ms timed region then starts
        just after nvidia-smi's query and ends long before the next one (-lms 100), so
        the query's driver work never lands inside it (samples still bracket it)."""
        if self.proc is None:
            return
        n = len(self.samples)
        t0 = time.perf_counter()
        while len(self.samples) == n and time.perf_counter() - t0 < timeout:
            time.sleep(0.0005)

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
def layout_map(kind, N, S):
    """Logical nodes -> GPUs.  weak (default): N pipelines of S stages, node (p, s) on GPU
    (p + s) mod N -- every GPU hosts S stages and, for N > 1, every ring hop crosses
    NVLink (per-GPU work fixed).  survey: C2 with ONE stage per GPU --
    one pipeline up to N = 4 (stage s on GPU s mod N), N / 4 pipelines beyond (C3's two
    4-stage pipelines on 8 GPUs); total work fixed up to N = 4."""
    P = N if kind == "weak" else max(1, N // S)
    coords = {(p, s): p * S + s for p in range(P) for s in range(S)}
    if kind == "weak":
        placement = {coords[(p, s)]: (p + s) % N for (p, s) in coords}
    else:
        placement = {coords[(p, s)]: (p * S + s) % N for (p, s) in coords}
    succ = {coords[(p, s)]: coords[(p, (s + 1) % S)] for (p, s) in coords}
    return P, coords, placement, succ


def timed_loop(args, K, kl, drv, rt, t, comp, content, dev, world, instrument=False,
               publish=True):
    """Runs W warm-up and K timed decode steps of the schedule from step t through the
    one-launch-per-step loop (kv_loop_run: each step prepared and launched in order, no
    lookahead).  Sources are pre-generated in HBM (> L2).  Not instrumented, consecutive
    launches overlap (programmatic dependent launch: a launch's prologue runs while the
    previous step's grid drains); `instrument` brackets every launch with CUDA events
    (which serialises them) to time each kernel alone.  Returns the timing record."""
    import torch
    import torch.distributed as dist

    def gen_sources(t0, n):
        out = {}
        for tt in range(t0, t0 + n):
            out[tt] = {}
            for node, e in drv.plan(tt).items():
                if node in rt.local:
                    ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                    out[tt][node] = content(e["stage"], ids, pos) if ids else None
        return out

    src = gen_sources(t, args.warmup + args.steps)
    src_bytes = sum(x.numel() * 2 for d in src.values() for x in d.values() if x is not None)

    def prepare(t0, n, timing):
        steps, evs = [], []
        for k, tt in enumerate(range(t0, t0 + n)):
            app = [dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                        req_ids=e["req_ids"], n_new=e["n_new"], src=src[tt].get(node))
                   for node, e in drv.plan(tt).items() if node in rt.local]
            pools = [rt.handle(nd) for nd in rt.alive_local() if rt.succ.get(nd) is not None]
            st = dict(append=app, repl_pools=pools if (tt >= 1 and publish) else [], step=tt)
            if timing:
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                st.update(ev_kernel_start=ev[0], ev_kernel_end=ev[1])
                evs.append((k, ev))
            steps.append(st)
        return K.PreparedSteps(steps), evs

    warm, _ = prepare(t, args.warmup, False)
    timed, evs = prepare(t + args.warmup, args.steps, instrument)
    torch.cuda.synchronize(dev)
    kl.run(warm, comp.cuda_stream)
    torch.cuda.synchronize(dev)
    nodes = rt.alive_local()
    bytes0 = {n: K.kv_stats(rt.handle(n))["bytes_replicated"] for n in nodes}
    l0 = K.kv_kernel_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K.kv_host_profile(reset=True)
    K.kv_launch_log(True)
    heat = torch.empty(2, 256 << 20, dtype=torch.uint8, device=dev)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        torch.cuda.synchronize(dev)
        clk.align()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize(dev)
        # the GPU idled while the sampler started: ~4 ms of HBM copies right before the
        # region (same stream, no sync) so it starts at full clocks, not on a ramp
        for _ in range(24):
            heat[1].copy_(heat[0])
        w0 = time.perf_counter()
        start.record(comp)
        kl.run(timed, comp.cuda_stream)
        end.record(comp)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - w0
    del heat
    log = K.kv_launch_log(False)
    launches = K.kv_kernel_launch_count() - l0
    host = {k: round(v / args.steps * 1e6, 2) for k, v in K.kv_host_profile(reset=True).items()}
    kl.flush(comp.cuda_stream)         # the last timed step's publication (untimed)
    torch.cuda.synchronize(dev)
    by = float(sum(K.kv_stats(rt.handle(n))["bytes_replicated"] - bytes0[n] for n in nodes))
    del src
    return {"ms": start.elapsed_time(end), "bytes": by, "launches": launches, "wall": wall,
            "log": log, "evs": evs, "host": host, "clocks": clk.summary(),
            "src_gib": src_bytes / 2**30}


def launch_bytes(r, N):
    """Algorithmic bytes of one decode-step launch: (HBM, NVLink).  N = 1: append (read the
    dense source + write the pool) + publication (read the pool + write the local replica)
    = 2 (app + rep) through HBM.  N > 1: the publication's writes go to the peer over
    NVLink, so HBM carries 2 app + rep and NVLink rep."""
    if N == 1:
        return 2 * r["app_bytes"] + 2 * r["rep_bytes"], 0
    return 2 * r["app_bytes"] + r["rep_bytes"], r["rep_bytes"]


def timed_roofline(rec, N, hbm_peak, peak_src):
    """Roofline of the decode-step kernel over the timed region: every launch in it (the
    launch log of the same region) with its algorithmic bytes, divided by the region's
    CUDA-event duration -- the kernel's average launch duration in the pipelined loop is
    region / launches.  N = 1: HBM-bound; N > 1: the NVLink hop (publication bytes) against
    the NVLink peak, the HBM figure beside it."""
    log = rec["log"]
    T = rec["ms"] * 1e-3
    hb = sum(launch_bytes(r, N)[0] for r in log)
    nb = sum(launch_bytes(r, N)[1] for r in log)
    n = max(1, len(log))
    out = {"kernel": "kv_step_kernel (one launch per step: append k + publication k-1)",
           "launches": len(log), "avg_launch_us": round(T / n * 1e6, 2),
           "algorithmic_bytes_per_launch": int((hb if N == 1 else nb) / n),
           "hbm_bytes_per_launch": int(hb / n),
           "append_bytes_per_launch": int(sum(r["app_bytes"] for r in log) / n),
           "replicate_bytes_per_launch": int(sum(r["rep_bytes"] for r in log) / n),
           "what": "sum over the timed region's launches (kv_launch_log) of their algorithmic "
                   "bytes / the region's CUDA-event duration (= bytes per launch / average "
                   "launch duration; launches overlap by programmatic dependent launch)"}
    hbm = hb / T / 1e9
    if N == 1:
        out.update(bound="hbm", achieved=round(hbm, 1), peak=hbm_peak, unit="GB/s",
                   frac=round(hbm / hbm_peak, 4), peak_source=peak_src)
    else:
        nvl = nb / T / 1e9
        out.update(bound="nvlink", achieved=round(nvl, 1), peak=NVLINK_PEAK_GBS, unit="GB/s",
                   frac=round(nvl / NVLINK_PEAK_GBS, 4),
                   peak_source="B200_PROFILING.md measured peer copy 770 GB/s/direction",
                   hbm={"achieved": round(hbm, 1), "peak": hbm_peak,
                        "frac": round(hbm / hbm_peak, 4)})
    return out


def isolated_launches(rec, N, hbm_peak):
    """The instrumented pass: each launch bracketed by its own CUDA events (serialised, no
    overlap), paired with its own bytes from the launch log."""
    log, evs = rec["log"], rec["evs"]
    if len(log) != len(evs):
        return {"paired": False, "note": "launch log has %d records for %d timed steps"
                                         % (len(log), len(evs))}
    durs = [ev[0].elapsed_time(ev[1]) * 1e-3 for _, ev in evs]
    hb = sum(launch_bytes(r, N)[0] for r in log)
    nb = sum(launch_bytes(r, N)[1] for r in log)
    T = sum(durs)
    out = {"launches": len(durs), "median_us": round(statistics.median(durs) * 1e6, 2),
           "avg_us": round(T / len(durs) * 1e6, 2),
           "p99_us": round(float(np.percentile(durs, 99)) * 1e6, 2),
           "hbm_gb_s": round(hb / T / 1e9, 1), "hbm_frac": round(hb / T / 1e9 / hbm_peak, 4),
           "what": "each launch alone between its own CUDA events (no overlap), paired with "
                   "its own algorithmic bytes"}
    if N > 1:
        out["nvlink_gb_s"] = round(nb / T / 1e9, 1)
    return out


def reduce_max_sum(vals, dev, world):
    """[max..., sum...] of a float vector over ranks."""
    import torch
    import torch.distributed as dist
    v = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world == 1:
        return [float(x) for x in v], [float(x) for x in v]
    mx, sm = v.clone(), v.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return [float(x) for x in mx], [float(x) for x in sm]


def run_kvring(args):
    import torch
    import torch.distributed as dist
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}; launch N>1 with torch.distributed.run")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    hbm_peak, peak_src = peaks()

    def build(kind, n_extra):
        base = configs.C2
        S = base.stages
        P, coords, placement, succ = layout_map(kind, N, S)
        cfg = configs.scaled(base, pipelines=P)
        scheds = configs.build_schedules(cfg, n_steps=args.prelude + args.warmup + args.steps
                                         + n_extra + 3)
        rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req,
                         placement, succ, rank=rank, world=world, device=local_rank, spares=1,
                         group=group, sentinel=None)
        g = cfg.geom

        def content(stage, ids, pos):
            return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                       g.kv_heads, g.head_dim, device=local_rank)

        return cfg, rt, ScheduleDriver(rt, scheds, coords, content), content

    comp = torch.cuda.current_stream(dev)
    repl = torch.cuda.Stream(dev)
    # legs after the headline: appends-only (W + K), two-stream (K), e2e, NCCL,
    # interference (2x), block mode (+1 re-seed), slack
    n_extra = (args.e2e_steps + args.nccl_steps + 2 * args.interference_steps + args.block_steps
               + 4 * (args.warmup + args.steps) + 40)
    cfg, rt, drv, content = build("weak", n_extra)

    # ---- prelude: reach steady state (untimed; sequential protocol on one stream) ----
    t = 0
    for _ in range(args.prelude):
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
        t += 1
    torch.cuda.synchronize(dev)

    # ---- headline: one launch per decode step (kv_loop), W warm-up + K timed ----------
    kl = K.KvLoop()
    t_timed0 = t + args.warmup
    rec = timed_loop(args, K, kl, drv, rt, t, comp, content, dev, world)
    t += args.warmup + args.steps
    mx, sm = reduce_max_sum([rec["ms"], rec["bytes"], float(rec["launches"])], dev, world)
    ms_max, tot_bytes, tot_launch = mx[0], sm[1], sm[2]
    roof = timed_roofline(rec, N, hbm_peak, peak_src)
    # the committed ncu capture is of this command at N = 1 (ncu replays one process);
    # at N > 1 the launches differ (peer stores, fewer stages per GPU): not captured
    traffic = traffic_ref("decode_population", "kv_step_kernel") if N == 1 else None
    roof["traffic"] = traffic["traffic"] if traffic else None
    if traffic:
        roof["traffic_note"] = traffic.get("note")
    elif N > 1:
        roof["traffic_note"] = ("no ncu capture at N > 1 (ncu profiles one process; the "
                                "1-GPU capture's population differs)")

    # ---- the same loop, every launch timed alone (events serialise the launches) -------
    inst = timed_loop(args, K, kl, drv, rt, t, comp, content, dev, world, instrument=True)
    t += args.warmup + args.steps
    iso = isolated_launches(inst, N, hbm_peak)

    # ---- the same steps' appends alone: the per-step cost of replication --------------
    base_rec = timed_loop(args, K, kl, drv, rt, t, comp, content, dev, world, publish=False)
    t += args.warmup + args.steps
    ms_app = reduce_max_sum([base_rec["ms"]], dev, world)[0][0]
    # re-seed the backlog the append-only steps left (untimed)
    drv.append_step(t, stream=comp)
    rt.replicate_all(t, stream=comp)
    t += 1
    torch.cuda.synchronize(dev)

    # ---- two-stream loop (P:229's shape): append stream + replication stream ----------
    two = run_two_stream(args, K, drv, rt, t, comp, repl, content, dev, world)
    t += args.steps

    # ---- e2e: host-resident inputs (pinned), H2D + D2H inside the timed region ---
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, K, kl, drv, rt, t, comp, content, dev, world)
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

    # ---- floor of a decode hop: a publication with nothing dirty ----------------------
    floor = run_floor(K, kl, rt, t + 10, comp, dev, world)

    # ---- restore: fail stage 2 of pipeline 0, restore into a fresh pool ---------
    restore = None
    if not args.no_restore:
        restore = run_restore(drv, rt, t, dev, comp, world)

    pool_gib = rt.n_slots * 2 * rt.replica_bytes / 2**30
    kl.destroy()
    rt.destroy()
    del rt, drv
    torch.cuda.empty_cache()

    # ---- SURVEY §8(e) layout at N > 1: one C2 stage per GPU ----------------------------
    survey = None
    if N > 1 and args.survey_layout:
        survey = run_survey_layout(args, build, dev, world, comp)
        torch.cuda.empty_cache()

    # ---- C4 failover (configs[3]): 16 logical nodes, batch 128, kill (0,2) at step 300 --
    c4 = None
    if args.c4_restores > 0:
        c4 = run_c4(args, rank, world, local_rank, dev, group)
        torch.cuda.empty_cache()

    # ---- bulk leg (C5: 32k-token prefill per stage, full-block re-seed) -----------
    bulk = run_bulk(args, rank, world, local_rank, dev, group) if args.bulk_reps > 0 else None

    # ---- shared capacity (NEXT-3): replicas in the holder's own pool, under pressure -
    shared = None
    if args.shared_steps > 0:
        shared = (run_shared(args, local_rank, dev) if world == 1 else
                  {"skipped": "shared capacity needs the holder on the same GPU (N = 1)"})

    value = tot_bytes / (ms_max * 1e-3) / 1e9
    ms_step = ms_max / args.steps
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (ShareGPT-shaped lognormal trace, closed-form KV words)",
        "config": bench_config(N),
        "dtype_note": "bf16 KV words moved bit-exactly as 16-bit data (no arithmetic)",
        "run": {"timed_steps": [t_timed0, t_timed0 + args.steps - 1],
                "loop": "kv_loop_run: per step ONE launch = appends of step k + publication of "
                        "step k-1; each step prepared and launched in order (no lookahead)",
                "inputs_gib": {"pre_generated_sources": round(rec["src_gib"], 2),
                               "pools_and_replicas_per_gpu": round(pool_gib, 1)}},
        "gb_s_per_gpu": round(value / N, 2),
        "replicated_bytes": int(tot_bytes),
        "step_overhead_us": {
            "median": round((ms_max - ms_app) / args.steps * 1e3, 2),
            "step_us_with_replication": round(ms_step * 1e3, 2),
            "step_us_appends_only": round(ms_app / args.steps * 1e3, 2),
            "budget_us": 400.0, "tpot_ms": 20.0,
            "what": "per decode step: the same loop with and without the publications (K steps "
                    "each, max over ranks); the harness has no model compute, so this is the "
                    "whole device cost replication adds to a step (interference: with a model)"},
        "kernel_us": iso,
        "roofline": roof,
        "step_roofline": step_roofline(tot_bytes, ms_max, N, hbm_peak, peak_src),
        "gpu_launches": int(tot_launch),
        "wall_s_timed": round(rec["wall"], 4),
        "host_us_per_step": rec["host"],
        "clocks": rec["clocks"],
        "two_stream": two,
        "step_floor_us": floor,
    }
    if e2e is not None:
        line["e2e"] = e2e
    for k, v in (("restore", restore), ("c4_failover", c4), ("bulk", bulk), ("nccl_compare", nccl),
                 ("interference", interference), ("block_mode", block),
                 ("shared_capacity", shared), ("survey_layout", survey)):
        if v is not None:
            line[k] = v
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, t_timed0, min(args.steps, 60))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_two_stream(args, K, drv, rt, t0, comp, repl, content, dev, world):
    """The same workload through kv_run_steps: per step one append launch on the compute
    stream and one publication launch on a separate replication stream after an event
    ("A separate CUDA stream is used to overlap the communication with
    computation"); append k waits for the publication of k-2 (R7)."""
    import torch
    import torch.distributed as dist
    n = args.steps
    steps, keep = [], []
    for tt in range(t0, t0 + n):
        app = []
        for node, e in drv.plan(tt).items():
            if node in rt.local:
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                src = content(e["stage"], ids, pos) if ids else None
                keep.append(src)
                app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=src))
        pools = [rt.handle(nd) for nd in rt.alive_local() if rt.succ.get(nd) is not None]
        steps.append(dict(append=app, repl_pools=pools, step=tt))
    prep = K.PreparedSteps(steps)
    nodes = rt.alive_local()
    b0 = {nd: K.kv_stats(rt.handle(nd))["bytes_replicated"] for nd in nodes}
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comp)
    K.kv_run_steps(prep, comp.cuda_stream, repl.cuda_stream)
    fin = torch.cuda.Event()
    fin.record(repl)
    comp.wait_event(fin)
    b.record(comp)
    torch.cuda.synchronize(dev)
    by = float(sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in nodes))
    mx, sm = reduce_max_sum([a.elapsed_time(b), by], dev, world)
    ms, tot = mx[0], sm[1]
    return {"value": round(tot / (ms * 1e-3) / 1e9, 2), "unit": UNIT, "steps": n,
            "ms_per_step": round(ms / n, 4),
            "what": "kv_run_steps: append launch on the compute stream, publication launch on a "
                    "replication stream after an event (2 launches per step)"}


def run_survey_layout(args, build, dev, world, comp):
    """C2 with one stage per GPU (1 pipeline at N <= 4, N / 4 pipelines
    beyond); same loop, warm-up and timing as the headline."""
    import torch
    from paper_2601_22438_b200 import kvring as K
    cfg, rt, drv, content = build("survey", 0)
    t = 0
    for _ in range(args.prelude):
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
        t += 1
    torch.cuda.synchronize(dev)
    kl = K.KvLoop()
    rec = timed_loop(args, K, kl, drv, rt, t, comp, content, dev, world)
    mx, sm = reduce_max_sum([rec["ms"], rec["bytes"]], dev, world)
    ms, tot = mx[0], sm[1]
    hbm_peak, peak_src = peaks()
    roof = timed_roofline(rec, world, hbm_peak, peak_src)
    stages = len(rt.alive_local())
    kl.destroy()
    rt.destroy()
    return {"layout": "one C2 stage per GPU (%d pipeline(s) x %d stages, stage s of pipeline p on "
                      "GPU (4p + s) mod N)" % (cfg.pipelines, cfg.stages),
            "stages_per_gpu": stages, "value": round(tot / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "ms_per_step": round(ms / args.steps, 4), "roofline": roof,
            "scaling": "strong (C2's total work fixed)" if world <= 4 else "C3 layout (2 pipelines)"}


C4_NB = 4096   # C4's resident peak is ~3.2k blocks per node (batch 128): pools sized to it


def run_c4(args, rank, world, local_rank, dev, group):
    """BASELINE configs[3] / SURVEY §8(d) C4: 16 logical nodes (4 pipelines x 4 stages,
    north_star's stage ring), node (i, s) on GPU (4i + s) mod N, closed-loop batch 128 per
    pipeline.  Steps 0..299 run the sequential protocol; at step 300 node (0,2) fails
    after its append (before its publication: t* = 299).  Its pool and block table are
    then restored from its successor's replica `c4_restores` times into a fresh pool
    (re-created each time; local HBM at N = 1, over NVLink from the next GPU at N > 1);
    promotion onto the holder runs the same kernel and is covered by the parity tests
    (the paper's instance ring, tests/test_gpu_configs.py).  Kernel time by
    CUDA events around the restore kernel, wall time around the whole kv_restore call
    (metadata acquire + read-back + allocation + kernel)."""
    import torch
    import torch.distributed as dist
    from kvgen import configs
    from kvgen.content import CONTENT_SEED
    from kvgen.cuda import content_tokens_cuda
    from paper_2601_22438_b200 import kvring as K
    from paper_2601_22438_b200.runtime import RingRuntime, ScheduleDriver
    cfg = configs.scaled(configs.C4, num_blocks=C4_NB)
    I, S = cfg.pipelines, cfg.stages
    coords = {(i, s): i * S + s for i in range(I) for s in range(S)}
    placement = {coords[(i, s)]: (4 * i + s) % world for (i, s) in coords}
    succ = {coords[(i, s)]: coords[(i, (s + 1) % S)] for (i, s) in coords}
    scheds = configs.build_schedules(cfg, n_steps=cfg.fail_step + 2)
    rt = RingRuntime(cfg.geom, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, placement,
                     succ, rank=rank, world=world, device=local_rank, spares=1, group=group,
                     sentinel=None)
    g = cfg.geom

    def content(stage, ids, pos):
        return content_tokens_cuda(CONTENT_SEED, ids, pos, stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim, device=local_rank)

    drv = ScheduleDriver(rt, scheds, coords, content)
    comp = torch.cuda.current_stream(dev)
    T = cfg.fail_step
    for t in range(T):
        drv.append_step(t, stream=comp)
        if t >= 1:
            rt.replicate_all(t, stream=comp)
    drv.append_step(T, stream=comp)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    f = coords[cfg.fail_node]
    holder = succ[f]
    rt.fail(f, comp)
    dst = drv.next_node
    drv.next_node += 1
    dst_rank = rt.placement[holder] if world == 1 else (rt.placement[holder] + 1) % world
    rt.new_node(dst, dst_rank)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    kern, wall, info = [], [], [0.0, 0.0, 0.0]
    for rep in range(args.c4_restores + 1):
        if rank == dst_rank:
            slot = rt.local[dst]
            K.kv_pool_destroy(slot.handle)
            rt._create(dst, slot)                     # a fresh pool on the same memory
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K.kv_time_next_launch(a, b)
            w0 = time.perf_counter()
            t_star, restored = rt.restore(dst, holder, comp)
            torch.cuda.synchronize(dev)
            w = (time.perf_counter() - w0) * 1e3
            if rep > 0:
                kern.append(a.elapsed_time(b))
                wall.append(w)
            tok = sum(ln for _, ln in restored)
            info = [float(t_star), float(len(restored)), float(tok * g.token_bytes)]
    res = torch.tensor([statistics.median(kern) if kern else 0.0,
                        statistics.median(wall) if wall else 0.0,
                        float(np.percentile(kern, 99)) if kern else 0.0] + info,
                       dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(res, op=dist.ReduceOp.SUM)      # one rank contributes
    rt.destroy()
    kms, wms, k99, t_star, nreq, R = [float(x) for x in res.tolist()]
    hbm_peak, peak_src = peaks()
    out = {"workload": "c4_failover_16 (16 logical nodes, batch 128 per pipeline, stage ring, "
                       "node (i,s) on GPU (4i+s) mod N, pools of %d blocks)" % C4_NB,
           "failed": list(cfg.fail_node), "fail_step": T, "t_star": int(t_star),
           "requests": int(nreq), "restored_bytes": int(R), "restores": args.c4_restores,
           "kernel_ms_median": round(kms, 4), "kernel_ms_p99": round(k99, 4),
           "wall_ms_median": round(wms, 3)}
    if world == 1:
        gbs = 2 * R / (kms * 1e-3) / 1e9
        out["roofline"] = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                           "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                           "peak_source": peak_src, "algorithmic_bytes_per_launch": int(2 * R),
                           "path": "local HBM: fresh pool on the holder's GPU"}
    else:
        gbs = R / (kms * 1e-3) / 1e9
        out["roofline"] = {"bound": "nvlink", "achieved": round(gbs, 1), "peak": NVLINK_PEAK_GBS,
                           "unit": "GB/s", "frac": round(gbs / NVLINK_PEAK_GBS, 4),
                           "algorithmic_bytes_per_launch": int(R),
                           "path": "remote: fresh pool on GPU %d reads GPU %d's replica over "
                                   "NVLink" % (dst_rank, rt.placement[holder])}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["oracle"] = oracle_c4_restore(cfg, scheds)
    return out


def oracle_c4_restore(cfg, scheds):
    """The oracle's restore of the same failure, as it stands, on ONE core: the ring runs
    to step 300 in metadata mode; the holder's published replica slots are filled with
    their closed-form words (setup, untimed); then OracleNode.restore_from copies them
    into a fresh node (timed).  Peak RSS of the process reported beside it."""
    import resource
    from kvgen.content import CONTENT_SEED, content_tokens
    from oracle.kvring_oracle import OracleNode
    from oracle.simulate import OracleRing
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    try:
        if aff:
            os.sched_setaffinity(0, {min(aff)})
        ring = OracleRing(cfg, content=False, schedules=scheds)
        T = cfg.fail_step
        for t in range(T + 1):
            ring.appends(t)
            if t < T and t >= 1:
                ring.replicate(t)
        f = ring.serving[cfg.fail_node]
        holder = f.succ
        f.fail()
        g = cfg.geom
        shape = (cfg.num_blocks, g.layers, 2, g.kv_heads, g.block_size, g.head_dim)
        holder.content = True
        holder.replica = np.zeros(shape, dtype=np.uint16)
        stage = cfg.fail_node[1]
        B = g.block_size
        for r, (s, ln, bt) in holder.published().items():
            words = content_tokens(CONTENT_SEED, [r] * ln, range(ln), stage * g.layers, g.layers,
                                   g.kv_heads, g.head_dim)
            for j, blk in enumerate(bt):
                v = min(B, ln - j * B)
                holder.replica[blk, :, :, :, :v] = words[j * B:j * B + v].transpose(1, 2, 3, 0, 4)
        dst = OracleNode(g, cfg.num_blocks, cfg.max_reqs, cfg.max_blocks_per_req, node_id=99,
                         content=True)
        t0 = time.perf_counter()
        t_star, restored = dst.restore_from(holder)
        dt = time.perf_counter() - t0
        tok = sum(ln for _, ln in restored)
        return {"restore_ms": round(dt * 1e3, 1), "t_star": int(t_star), "requests": len(restored),
                "restored_bytes": int(tok * g.token_bytes), "cores": 1,
                "peak_rss_gib": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20, 2),
                "what": "OracleNode.restore_from (numpy, one core) of the same failure; peak RSS "
                        "of the bench process (GPU arm + oracle)"}
    except Exception as e:
        return {"restore_ms": None, "error": str(e)[:200]}
    finally:
        if aff:
            os.sched_setaffinity(0, aff)


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
        tr = traffic_ref("bulk_c5", "kv_step_kernel")
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
    down 14336x4096, SiLU-gated), random weights, plus a paged decode-attention read of
    every live request's KV out of the stage pools (kvgen.cuda.AttnProxy: GQA 4 query
    heads per KV head, online softmax) -- the HBM consumer replication competes with --
    captured in one CUDA graph.  It stands in for the model step the replication must
    overlap."""

    def __init__(self, n_stages, layers, batch, dev, attn=None):
        self.attn = attn
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
        if self.attn is not None:
            self.attn.run(torch.cuda.current_stream(self.dev).cuda_stream)
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
    from kvgen.cuda import AttnProxy
    n = args.interference_steps
    nodes = rt.alive_local()
    # the live requests' KV as the window starts (block tables of every local stage)
    pools, tables = [], []
    for i, nd in enumerate(nodes):
        pools.append(rt.local[nd].pool)
        req, ln, pub, nb = K.kv_dump_slots(rt.handle(nd), rt.R)
        for r, l_ in zip(req, ln):
            if r >= 0 and l_ > 0:
                tables.append((i, int(l_), K.kv_query(rt.handle(nd), int(r))[1]))
    attn = AttnProxy(pools, tables, rt.g.layers, rt.g.kv_heads, rt.g.block_size, rt.g.head_dim,
                     qpk=4, device=dev.index)
    proxy = DecodeProxy(len(nodes), rt.g.layers, 64, dev, attn=attn)
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
                     "batch 64 + paged decode attention reading %d live tokens' KV (%.0f MB) "
                     "(CUDA graph) on the compute stream"
                     % (len(nodes), rt.g.layers, attn.tokens, attn.tokens * rt.g.layers * 2
                        * rt.g.kv_heads * rt.g.head_dim * 2 / 1e6),
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


def run_floor(K, kl, rt, t0, comp, dev, world):
    """Per-step floor of the publication on the timed loop's own path: FLOOR_REPS loop
    steps with no append and nothing dirty (a launch that only writes the parity table
    and the seq flag of every pool, over NVLink when the successor is remote), each
    launch bracketed by CUDA events like the headline's kernel_us; max over ranks."""
    import torch
    import torch.distributed as dist
    nodes = [n for n in rt.alive_local() if rt.succ.get(n) is not None]
    handles = [rt.handle(n) for n in nodes]
    sts, evs = [], []
    for k in range(FLOOR_REPS + 2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        evs.append(ev)
        sts.append(dict(append=[], repl_pools=handles, step=t0 + k, ev_kernel_start=ev[0],
                        ev_kernel_end=ev[1]))
    prep = K.PreparedSteps(sts)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    kl.run(prep, comp.cuda_stream)
    kl.flush(comp.cuda_stream)
    torch.cuda.synchronize(dev)
    kern = sorted(e[0].elapsed_time(e[1]) * 1e3 for e in evs[2:])   # launches 2.. publish
    v = torch.tensor([kern[len(kern) // 2]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return {"kernel_median": round(float(v[0]), 2), "reps": FLOOR_REPS, "pools": len(nodes),
            "what": "loop steps with nothing dirty (kv_loop_step: one launch writing every "
                    "pool's parity table and seq), CUDA events around each launch; the "
                    "decode-step launch's floor"}


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


NCCL_WARMUP = 5


def run_nccl(args, drv, rt, t0, comp, content, dev, world):
    """The paper's transport (NCCL send/recv, P:8 §3.3) on the same workload, as the
    measured comparison: per step append, then gather-pack, the packed sizes exchanged on
    the host (gloo; no GPU sync), ONE grouped ncclSend/ncclRecv (libkvnccl; at N = 1 the
    single rank sends to itself), unpack + publish.  One stream; CUDA events around
    pack..unpack and around the NCCL group."""
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
    evn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n)]
    # untimed warm-up steps: NCCL connects a peer pair on its first send/recv (~1 s at
    # N = 2, which would otherwise sit inside the first timed step)
    nw = min(NCCL_WARMUP, n - 1)
    for k in range(nw):
        tt = t0 + k
        drv.append_step(tt, stream=comp, sources=srcs[tt], plan=plans[tt])
        ring.step(tt, comp)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    b0 = {nd: K.kv_stats(rt.handle(nd))["bytes_replicated"] for nd in rt.alive_local()}
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    st.record(comp)
    for k in range(nw, n):
        tt = t0 + k
        drv.append_step(tt, stream=comp, sources=srcs[tt], plan=plans[tt])
        evs[k][0].record(comp)
        ring.step(tt, comp, events=evn[k])
        evs[k][1].record(comp)
    en.record(comp)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - w0
    ms = st.elapsed_time(en)
    by = sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in rt.alive_local())
    us = [a.elapsed_time(b) * 1e3 for a, b in evs[nw:]]
    us_n = [a.elapsed_time(b) * 1e3 for a, b in evn[nw:]]
    n -= nw
    ring.destroy()
    busy_ms = sum(us) * 1e-3          # device time of pack .. unpack, summed over the steps
    mx, sm = reduce_max_sum([ms, float(by), wall, busy_ms], dev, world)
    ms, by, wall, busy_ms = mx[0], sm[1], mx[2], mx[3]
    return {"transport": "NCCL 2.28 grouped ncclSend/ncclRecv (libkvnccl): pack, host count "
                         "exchange (gloo, N > 1), send/recv, unpack"
                         + (" -- one rank sending to itself" if world == 1 else ""),
            "value": round(by / (busy_ms * 1e-3) / 1e9, 2), "unit": UNIT, "steps": n,
            "warmup_steps": nw,
            "what": "replicated bytes / device time of the replication (CUDA events around "
                    "pack .. unpack of every step, summed; max over ranks)",
            "ms_per_step": round(busy_ms / n, 4),
            "loop": {"value": round(by / (ms * 1e-3) / 1e9, 2), "ms_per_step": round(ms / n, 4),
                     "wall_ms_per_step": round(wall / n * 1e3, 4),
                     "what": "the whole Python loop on the device clock: the per-step host "
                             "work (append planning in Python, pack bookkeeping, the gloo "
                             "size exchange) leaves the GPU idle between steps"},
            "step_us": {"median": round(statistics.median(us), 2),
                        "p99": round(float(np.percentile(us, 99)), 2),
                        "what": "pack + count exchange + NCCL group + unpack"},
            "nccl_group_us": {"median": round(statistics.median(us_n), 2),
                              "p99": round(float(np.percentile(us_n, 99)), 2),
                              "what": "the ncclSend/ncclRecv group alone"}}


def run_e2e(args, K, kl, drv, rt, t0, comp, content, dev, world):
    """Same metric through the public API with HOST buffers: per step one kv_loop_step
    (the Python binding's call) whose appends read the step's new-token KV from pinned
    host memory (KV_SRC_HOST: the kernel reads it over PCIe), and a D2H read-back of
    the seq flags the predecessors published into this GPU's replica metadata."""
    import torch
    import torch.distributed as dist
    n = args.e2e_steps
    host, preps = {}, []
    h2d = 0
    for tt in range(t0, t0 + n):
        app = []
        for node, e in drv.plan(tt).items():
            if node in rt.local:
                ids, pos = drv.tokens(e["req_ids"], e["n_new"], e["start"])
                hbuf = None
                if ids:
                    d = content(e["stage"], ids, pos)
                    hbuf = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
                    hbuf.copy_(d)
                    h2d += d.numel() * 2
                host[(tt, node)] = hbuf
                app.append(dict(pool=rt.handle(node), begin_step=1, release=e["release"],
                                req_ids=e["req_ids"], n_new=e["n_new"], src=hbuf,
                                flags=K.KV_SRC_HOST))
        pools = [rt.handle(nd) for nd in rt.alive_local() if rt.succ.get(nd) is not None]
        preps.append(K.PreparedSteps([dict(append=app, repl_pools=pools, step=tt)]))
    torch.cuda.synchronize(dev)
    nodes = rt.alive_local()
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
    for k in range(n):
        kl.step(preps[k], 0, comp.cuda_stream)
        for i, sd in enumerate(seq_dev):
            seq_host[k, i].copy_(sd, non_blocking=True)
            d2h += 8
    kl.flush(comp.cuda_stream)
    en.record(comp)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - w0
    by = float(sum(K.kv_stats(rt.handle(nd))["bytes_replicated"] - b0[nd] for nd in nodes))
    mx, sm = reduce_max_sum([st.elapsed_time(en), by, wall], dev, world)
    ms, by, wall = mx[0], sm[1], mx[2]
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
            "path": "per step one kv_loop_step call from Python (appends read pinned host KV "
                    "over PCIe, zero copy; the previous step's publication in the same launch) "
                    "+ a D2H read-back of the published seq flags"}


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
