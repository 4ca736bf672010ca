"""CPU oracle for the REXI hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(``swerexi``, arXiv 1805.06557, mounted read-only at /root/reference) for
the REXI pole-sum path and the spherical-harmonic N-term around it.  Every
function cites the reference file:line it follows.

Rules:
  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it, and only as
    the checker or as the timed CPU baseline -- never as the product path;
  * it is pinned against golden vectors produced by the reference itself
    (``tests/golden/make_golden.py``, run in the build container where the
    reference is importable) -- see ``tests/test_oracle_golden.py``.
"""

from . import layout, rexi, sht, stepping  # noqa: F401
