r"""CPU oracle for segmental-refinement FAS-FMG (arXiv 1406.7808).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this package.  The product path
(`paper_1406_7808_b200`) never imports it, and it never imports the product path: the two
share no code.  Only `workloads.py` (seeded input generators, no method arithmetic) serves
both.

Plain, slow, obviously-correct numpy in fp64: every function cites the PAPER.md passage it
transcribes.  Pins: tests/test_oracle_*.py.  Parity status per function:
  fill_bc_ghosts, apply_A, cheb, restrict_avg8, prolong, exact_solve  -> pinned
  Oracle.vconv / fmg_conventional / vsolve                            -> pinned
  Oracle.vsr / solve (SR)                                             -> pinned by
      equivalences (huge buffer, one segment), region brute force, symmetry, O(h^2),
      GSR-freeze invariants, the FASMGVSR fixed point at u_h*, the GSR increment by
      every correction (R17) and the tau's zero residual on C \ F (R18); the paper's e_r
      table values are for a different stencil, so the e_r VALUES are "parity unpinned"
      (context only).
"""
from .grid import Box, Field
from .ops import (apply_A, cheb, cheb_constants, dense_operator, exact_solve, fill_bc_ghosts,
                  prolong, residual, restrict_avg8)
from .solver import Config, Oracle, solve, vcycle_iterate, vsolve

__all__ = [
    "Box", "Field", "apply_A", "cheb", "cheb_constants", "dense_operator", "exact_solve",
    "fill_bc_ghosts", "prolong", "residual", "restrict_avg8", "Config", "Oracle", "solve",
    "vcycle_iterate", "vsolve",
]
