"""CPU oracle of the KFVM-WENO stage update — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker /
reported CPU baseline, never as the measured or shipped path.

Pinning status: the reference ships no golden vectors or tests for this path
(SURVEY.md §8(c)); the oracle is pinned by the SPEC's inline known-answer
examples (tests/golden/spec_examples.json), the SPEC invariants and PAPER.md
Table 1 convergence orders — see tests/test_oracle_*.py and DESIGN.md §3.
"""
from .kfvm_oracle import Oracle, point_api  # noqa: F401
