"""Per-step request events of one pipeline (input generator).

A pipeline's S stages all see the same requests; each stage stores the KV of
its own layers.  This module decides only WHEN requests arrive, grow and
finish -- the serving-side workload -- never where their KV goes (that is the
method: allocator, block tables, replication).

Step semantics (SURVEY §8(c) "Algorithm", readings R3/R16):

* a request (P, O) admitted at step ``a`` appends its P prompt tokens at step
  ``a`` and one decode token at each of steps a+1 .. a+O;
* it retires at step a+O+1 ("requests whose last token was appended in t-1");
* within a step the order is: retire, decode appends (ascending req_id),
  admissions (FCFS arrival order, tie-break req_id) up to the batch cap.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

REQ_STRIDE = 1_000_000   # req_id = pipeline * REQ_STRIDE + k: unique across pipelines


@dataclass(frozen=True)
class Request:
    req_id: int
    prompt: int
    output: int
    arrival: float = 0.0


@dataclass
class StepEvents:
    retire: list[int] = field(default_factory=list)          # req ids, ascending
    decode: list[int] = field(default_factory=list)          # req ids, ascending, +1 token each
    admit: list[tuple[int, int]] = field(default_factory=list)  # (req_id, prompt) FCFS

    def appends(self) -> tuple[list[int], list[int]]:
        """(req_ids, n_new) in the order kv_append processes them."""
        ids = list(self.decode) + [r for r, _ in self.admit]
        n = [1] * len(self.decode) + [p for _, p in self.admit]
        return ids, n


@dataclass
class Schedule:
    requests: dict[int, Request]
    steps: list[StepEvents]
    admitted_at: dict[int, int]

    def length_at(self, req_id: int, step: int) -> int:
        """KV length of a request after the appends of ``step`` (0 if not admitted)."""
        a = self.admitted_at.get(req_id)
        if a is None or step < a:
            return 0
        r = self.requests[req_id]
        return r.prompt + min(step - a, r.output)


def _run(requests: list[Request], n_steps: int, cap: int, step_s: float | None) -> Schedule:
    by_id = {r.req_id: r for r in requests}
    queue = sorted(requests, key=lambda r: (r.arrival, r.req_id))
    qi = 0
    live: dict[int, int] = {}        # req_id -> admitted step
    admitted_at: dict[int, int] = {}
    steps: list[StepEvents] = []
    for t in range(n_steps):
        ev = StepEvents()
        for rid in sorted(live):
            a = live[rid]
            if a + by_id[rid].output + 1 == t:
                ev.retire.append(rid)
        for rid in ev.retire:
            del live[rid]
        ev.decode = sorted(rid for rid, a in live.items() if a < t)
        while qi < len(queue) and len(live) < cap:
            r = queue[qi]
            if step_s is not None and r.arrival > t * step_s:
                break
            live[r.req_id] = t
            admitted_at[r.req_id] = t
            ev.admit.append((r.req_id, r.prompt))
            qi += 1
        steps.append(ev)
    return Schedule(by_id, steps, admitted_at)


def closed_loop_schedule(prompts, outputs, n_steps: int, cap: int, pipeline: int = 0,
                         id_base: int | None = None) -> Schedule:
    """Keep ``cap`` requests live; admit the next trace entry when one finishes (R16)."""
    base = pipeline * REQ_STRIDE if id_base is None else id_base
    reqs = [Request(base + k, int(p), int(o), 0.0) for k, (p, o) in enumerate(zip(prompts, outputs))]
    return _run(reqs, n_steps, cap, None)


def open_loop_schedule(prompts, outputs, arrivals, n_steps: int, cap: int, step_s: float,
                       pipeline: int = 0) -> Schedule:
    """Poisson arrivals on a logical step clock of ``step_s`` seconds, FCFS, cap per pipeline."""
    base = pipeline * REQ_STRIDE
    reqs = [Request(base + k, int(p), int(o), float(a))
            for k, (p, o, a) in enumerate(zip(prompts, outputs, np.asarray(arrivals)))]
    return _run(reqs, n_steps, cap, step_s)
