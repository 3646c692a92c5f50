"""CPU oracle for arXiv 2312.12771 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2312_12771_b200``) never imports it and shares no code with it.
See ``oracle/hom_oracle.c`` for what is computed and which PAPER.md passages
each function follows.

Parity status per function:
  rve_condense_linear / condense_batch_linear  pinned (closed forms, bounds, brute force)
  condense_batch_nh                            pinned (FD of the averaged stress, brute force)
  macro_solve                                  pinned (affine patch test, brute force, energy)
"""
from .oracle import *  # noqa: F401,F403
