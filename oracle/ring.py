"""Oracle ring maps over logical nodes (instance i, stage s).  TEST INFRASTRUCTURE ONLY.

* ``instance_ring`` -- the paper's ring: same stage, next instance,
  (i, s) -> ((i+1) mod I, s).  Pinned by P:215 / P:225 §3.2 ("When node (0, 2)
  fails ... another healthy node (1, 2) ... replication target (e.g., node
  (1, 2))") and SPEC S:48-53.
* ``stage_ring`` -- BASELINE.json north_star's ring inside one pipeline,
  stage i -> (i+1) mod N (reading R1: the ring is data; kernels do not care).
* ``plan_replication_targets`` -- P:227 §3.2: "replication targets will be
  automatically adjusted to exclude the nodes under traffic rerouting";
  SPEC S:54-62: each non-excluded node maps to the first non-excluded node met
  by repeatedly applying the ring successor, never itself; a node with no
  such peer is replication-disabled (None).
"""
from __future__ import annotations

Node = tuple[int, int]


def instance_ring(node: Node, I: int, S: int) -> Node:
    i, s = node
    if not (0 <= i < I and 0 <= s < S):
        raise ValueError(f"invalid node {node}")
    return ((i + 1) % I, s)


def stage_ring(node: Node, I: int, S: int) -> Node:
    i, s = node
    if not (0 <= i < I and 0 <= s < S):
        raise ValueError(f"invalid node {node}")
    return (i, (s + 1) % S)


def plan_replication_targets(I: int, S: int, excluded, ring=instance_ring) -> dict[Node, Node | None]:
    """Walk the ring from each non-excluded node, skipping excluded ones."""
    if I * S == 0:
        raise ValueError("empty cluster")
    excluded = set(excluded)
    plan: dict[Node, Node | None] = {}
    for i in range(I):
        for s in range(S):
            n = (i, s)
            if n in excluded:
                continue
            cur, target = n, None
            for _ in range(I * S):
                cur = ring(cur, I, S)
                if cur == n:
                    break
                if cur not in excluded:
                    target = cur
                    break
            plan[n] = target
    return plan
