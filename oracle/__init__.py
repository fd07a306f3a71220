"""CPU oracle for the FPSAttention hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the algorithm of the reference package
``fp8sta`` (``/root/reference/pkg/src/fp8sta``) for the path named by
``BASELINE.json:north_star``: tile layout, FP8 codec, per-tile / per-channel
quantisation, sliding-tile window lists, the step schedule and the quantised
sparse attention forward.  Every function cites the reference file:line it
follows.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` -- as the checker
or the timed CPU baseline, never as the product path.  The product package
``paper_2506_04648_b200`` never imports this module.

Parity pinning: the restatement is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports ``fp8sta`` from
``/root/reference`` in the build container and freezes its outputs into
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""

from .fpsa_oracle import *  # noqa: F401,F403
