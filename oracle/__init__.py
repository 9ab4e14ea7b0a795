"""CPU oracle for ring KV-cache replication (KevlarFlow, arXiv 2601.22438).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2601_22438_b200``) never imports it, and
this package never imports the product: the two share no code, only the
seeded inputs of ``kvgen``.

Plain, slow, obviously correct numpy: 16-bit words, no blocking, no fusion.
Every function cites the passage it follows: ``P:n`` is PAPER.md line n,
``S:n`` SPEC.md line n, and SURVEY §8(c) restates the algorithm (steps 1-7)
together with the readings R1-R16 listed in DESIGN.md.

Parity pins (tests/test_oracle_*.py): hand-derived C1 tables
(tests/golden/c1_tables.json), the P:227 ring-walk example, splitmix64
published vectors, brute-force full-copy replay (I6), ``index_copy`` special
case, closed-form byte counts, resume point.  No function
here is "parity unpinned".
"""
from .kvring_oracle import OracleNode, OracleError, ENOMEM, EINVAL, ESTATE, ENOREPLICA
from .ring import stage_ring, instance_ring, plan_replication_targets
from .simulate import OracleRing, run_config

__all__ = ["OracleNode", "OracleError", "ENOMEM", "EINVAL", "ESTATE", "ENOREPLICA",
           "stage_ring", "instance_ring", "plan_replication_targets",
           "OracleRing", "run_config"]
