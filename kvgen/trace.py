"""ShareGPT-shaped request lengths and Poisson arrivals (input generator).

PAPER P:17 §4 names ShareGPT and Poisson arrivals but gives no shape
parameters.  DESIGN.md reading R14 adopts SPEC S:466: prompt_len ~ lognormal
(median 128, sigma_log 1.0) clamped to [1, 2048]; max_new_tokens ~ lognormal
(median 128, sigma_log 0.8) clamped to [1, 1024].  Arrivals: i.i.d.
Exponential(rate = rps) gaps.  numpy PCG64 with fixed seeds; both
the oracle and the CUDA path consume the SAME arrays, so no cross-language
PRNG identity is needed.
"""
from __future__ import annotations

import numpy as np

TRACE_SEED_BASE = 22438      # trace seed 22438 + k
PROMPT_MEDIAN, PROMPT_SIGMA, PROMPT_MAX = 128.0, 1.0, 2048
OUTPUT_MEDIAN, OUTPUT_SIGMA, OUTPUT_MAX = 128.0, 0.8, 1024


def synth_trace(n: int, seed: int, prompt_max: int = PROMPT_MAX,
                output_max: int = OUTPUT_MAX) -> tuple[np.ndarray, np.ndarray]:
    """Return (prompt_len[n], max_new_tokens[n]) as int64 arrays."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = np.exp(np.log(PROMPT_MEDIAN) + PROMPT_SIGMA * rng.standard_normal(n))
    o = np.exp(np.log(OUTPUT_MEDIAN) + OUTPUT_SIGMA * rng.standard_normal(n))
    p = np.clip(np.rint(p), 1, prompt_max).astype(np.int64)
    o = np.clip(np.rint(o), 1, output_max).astype(np.int64)
    return p, o


def poisson_arrivals(rps: float, n: int, seed: int) -> np.ndarray:
    """Arrival times (seconds) of n requests with Exponential(rps) gaps."""
    if rps < 0:
        raise ValueError("negative rps")
    if rps == 0 or n == 0:
        return np.zeros(0, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.cumsum(rng.exponential(1.0 / rps, size=n))
