"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This package holds NONE of the replication method's arithmetic (no allocator,
no block tables, no copies).  It produces only what both sides consume as
input:

* ``content``  -- the closed-form 16-bit KV words a model would have written
  for (request, global layer, K/V, head, position, dim)  (SURVEY §8(c) pins);
* ``trace``    -- ShareGPT-shaped prompt/output lengths and
  Poisson arrivals (§4);
* ``schedule`` -- the per-step request events (retire / decode / admit) of a
  closed-loop batch or an open-loop Poisson stream, per pipeline;
* ``configs``  -- the five BASELINE.json configurations as plain data.
"""
from .content import (SENTINEL_WORD, POISON_WORD, CONTENT_SEED, splitmix64,
                      content_tokens, content_segment_table)
from .trace import synth_trace, poisson_arrivals, TRACE_SEED_BASE
from .schedule import Request, StepEvents, closed_loop_schedule, open_loop_schedule, Schedule
from . import configs

__all__ = [
    "SENTINEL_WORD", "POISON_WORD", "CONTENT_SEED", "splitmix64", "content_tokens",
    "content_segment_table", "synth_trace", "poisson_arrivals", "TRACE_SEED_BASE",
    "Request", "StepEvents", "closed_loop_schedule", "open_loop_schedule", "Schedule",
    "configs",
]
