"""Closed-form synthetic KV content (input generator; no replication arithmetic).

SURVEY §8(c) "What pins each part": every valid KV slot holds

    content(seed, req, l, kv, h, pos, dim) = T[l, kv, h, dim] XOR word16(K(seed, req, pos), dim mod 4)

where ``l`` is the GLOBAL layer index (stage * L_s + local layer), ``T`` is a
splitmix64-derived 16-bit table and ``K`` a splitmix64 key of (seed, req, pos).
The values are bit patterns only (PAPER is silent on dtype; DESIGN.md reading
R13): no floating point is ever applied to them, so NaN / -0 / subnormal
patterns are carried like any other word.

The CUDA twin of this generator (``kvgen/csrc/kvgen.cu``) implements the same
counter-based function; ``tests/test_kvgen.py`` pins the two byte-for-byte.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
TABLE_SALT = 0x4B565441424C45  # "KVTABLE"

CONTENT_SEED = 2601          # content seed 2601
SENTINEL_WORD = 0x5A5A       # never-written slots (I5 "no stray writes")
POISON_WORD = 0xFFFF         # a failed stage's memory (0xFF bytes)


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 (Steele/Lea/Flood), python ints."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def content_keys(seed: int, req_ids, positions) -> np.ndarray:
    """K(seed, req, pos) = sm(sm(sm(seed) ^ req) ^ pos), one uint64 per token."""
    req = np.asarray(req_ids, dtype=np.int64).astype(np.uint64)
    pos = np.asarray(positions, dtype=np.int64).astype(np.uint64)
    s = np.uint64(splitmix64_int(seed & MASK64))
    return splitmix64(splitmix64(s ^ req) ^ pos)


def content_segment_table(seed: int, layer0: int, layers: int, kv_heads: int,
                          head_dim: int) -> np.ndarray:
    """T[l, kv, h, dim] for global layers [layer0, layer0+layers): uint16 [L][2][H][d]."""
    l = np.arange(layer0, layer0 + layers, dtype=np.uint64)[:, None, None, None]
    kv = np.arange(2, dtype=np.uint64)[None, :, None, None]
    h = np.arange(kv_heads, dtype=np.uint64)[None, None, :, None]
    dim = np.arange(head_dim, dtype=np.uint64)[None, None, None, :]
    idx = ((l * np.uint64(2) + kv) * np.uint64(kv_heads) + h) * np.uint64(head_dim) + dim
    salt = np.uint64(splitmix64_int((seed ^ TABLE_SALT) & MASK64))
    return (splitmix64(salt ^ idx) & np.uint64(0xFFFF)).astype(np.uint16)


def content_tokens(seed: int, req_ids, positions, layer0: int, layers: int,
                   kv_heads: int, head_dim: int, table: np.ndarray | None = None) -> np.ndarray:
    """Dense KV of n tokens: uint16 [n][L][2][H][d] (the layout ``kv_append`` takes)."""
    keys = content_keys(seed, req_ids, positions)
    n = keys.shape[0]
    if table is None:
        table = content_segment_table(seed, layer0, layers, kv_heads, head_dim)
    shifts = (np.uint64(16) * (np.arange(head_dim, dtype=np.uint64) % np.uint64(4)))
    words = ((keys[:, None] >> shifts[None, :]) & np.uint64(0xFFFF)).astype(np.uint16)  # [n][d]
    out = np.empty((n, layers, 2, kv_heads, head_dim), dtype=np.uint16)
    np.bitwise_xor(table[None], words[:, None, None, None, :], out=out)
    return out
