"""The five BASELINE.json configurations as plain data.

Geometry is Llama-3.1-8B KV (GQA 8 KV heads x head_dim 128, 32 layers split
over pipeline stages), block size B = 16 tokens (reading R4).
Everything here is an input description; nothing here allocates or copies.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

from .trace import TRACE_SEED_BASE


@dataclass(frozen=True)
class Geometry:
    layers: int            # L_s, layers per stage
    kv_heads: int = 8
    head_dim: int = 128
    block_size: int = 16
    elem_bytes: int = 2    # fp16 / bf16 words (bits only, R13)

    @property
    def seg_bytes(self) -> int:          # one (layer, K/V, head, token) slice
        return self.head_dim * self.elem_bytes

    @property
    def combos(self) -> int:             # (layer, K/V, head) triples per token
        return self.layers * 2 * self.kv_heads

    @property
    def token_bytes(self) -> int:        # bytes per token per stage
        return self.combos * self.seg_bytes

    @property
    def block_bytes(self) -> int:
        return self.token_bytes * self.block_size

    @property
    def block_words(self) -> int:
        return self.block_bytes // self.elem_bytes


@dataclass(frozen=True)
class Config:
    name: str
    geom: Geometry
    stages: int                     # S, stages per pipeline
    pipelines: int                  # I, pipelines (instances)
    num_blocks: int                 # NB per logical node
    max_reqs: int                   # request slots per logical node (>= 2 x batch_cap:
                                    # a retired slot is quarantined one step, R7)
    max_blocks_per_req: int
    batch_cap: int                  # live requests per pipeline
    n_requests: int                 # trace length per pipeline
    n_steps: int
    trace_seed: int
    dtype: str = "bf16"
    fixed_prompt: int | None = None  # C1/C5: every request has this prompt length
    fixed_output: int | None = None
    rps: float | None = None         # C3: open-loop Poisson; None = closed loop
    step_s: float = 0.020            # logical decode step (north_star: 20 ms)
    fail_node: tuple[int, int] | None = None   # (instance, stage)
    fail_step: int | None = None               # fail after the appends of this step
    ring: str = "stage"             # "stage": (i,s)->(i,(s+1)%S); "instance": (i,s)->((i+1)%I,s)
    extra: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return self.stages * self.pipelines


# C1 tiny: 4 stages x 2 layers, fp16, NB 32, 4 requests x 64 tokens admitted at
# step 0, decode steps 1..8, fail stage 2 after the append of step 5 (t* = 4).
C1 = Config(name="c1_tiny", geom=Geometry(layers=2), stages=4, pipelines=1, num_blocks=32,
            max_reqs=4, max_blocks_per_req=8, batch_cap=4, n_requests=4, n_steps=9,
            trace_seed=TRACE_SEED_BASE + 1, dtype="fp16", fixed_prompt=64, fixed_output=16,
            fail_node=(0, 2), fail_step=5)

# C2: 4-stage PP, 8 layers/stage, bf16, closed-loop batch 64 over a 2000-request trace.
# Worst case 64 requests x ceil(3072/16)=192 blocks = 12,288 blocks (6 GiB) per pool.
C2 = Config(name="c2_pp4_b64", geom=Geometry(layers=8), stages=4, pipelines=1,
            num_blocks=12288, max_reqs=128, max_blocks_per_req=192, batch_cap=64,
            n_requests=2000, n_steps=1300, trace_seed=TRACE_SEED_BASE + 2)

# C3: two 4-stage pipelines, Poisson arrivals (RPS sweep), cap 128 per pipeline, 20 ms steps.
C3 = Config(name="c3_2x4_poisson", geom=Geometry(layers=8), stages=4, pipelines=2,
            num_blocks=24576, max_reqs=256, max_blocks_per_req=192, batch_cap=128,
            n_requests=4000, n_steps=3000, trace_seed=TRACE_SEED_BASE + 3, rps=4.0)

# C4: 16 logical nodes (4 pipelines x 4 stages), closed-loop batch 128 per pipeline,
# kill (0,2) at step 300 after its append, restore, resume 100 steps.
C4 = Config(name="c4_failover_16", geom=Geometry(layers=8), stages=4, pipelines=4,
            num_blocks=24576, max_reqs=512, max_blocks_per_req=192, batch_cap=128,
            n_requests=2000, n_steps=401, trace_seed=TRACE_SEED_BASE + 4,
            fail_node=(0, 2), fail_step=300)

# C5: 8 stages x 4 layers, one P = 32,768 request per stage: 2,048 full blocks of 256 KiB.
C5 = Config(name="c5_bulk_32k", geom=Geometry(layers=4), stages=8, pipelines=1,
            num_blocks=2048, max_reqs=1, max_blocks_per_req=2048, batch_cap=1,
            n_requests=1, n_steps=2, trace_seed=TRACE_SEED_BASE + 5,
            fixed_prompt=32768, fixed_output=1)

ALL = {c.name: c for c in (C1, C2, C3, C4, C5)}


def scaled(cfg: Config, **kw) -> Config:
    """A copy of ``cfg`` with some fields replaced (parity tests use small variants)."""
    return replace(cfg, **kw)


def build_schedules(cfg: Config, n_steps: int | None = None):
    """One request schedule per pipeline, seeded from ``cfg.trace_seed`` + pipeline."""
    import numpy as np
    from .schedule import closed_loop_schedule, open_loop_schedule
    from .trace import synth_trace, poisson_arrivals
    steps = cfg.n_steps if n_steps is None else n_steps
    out = []
    for p in range(cfg.pipelines):
        seed = cfg.trace_seed * 1000 + p
        if cfg.fixed_prompt is not None:
            prompts = np.full(cfg.n_requests, cfg.fixed_prompt, dtype=np.int64)
            outputs = np.full(cfg.n_requests, cfg.fixed_output, dtype=np.int64)
        else:
            prompts, outputs = synth_trace(cfg.n_requests, seed)
        if cfg.rps is None:
            out.append(closed_loop_schedule(prompts, outputs, steps, cfg.batch_cap, pipeline=p))
        else:
            arr = poisson_arrivals(cfg.rps / cfg.pipelines, cfg.n_requests, seed + 7)
            out.append(open_loop_schedule(prompts, outputs, arr, steps, cfg.batch_cap,
                                          cfg.step_s, pipeline=p))
    return out
