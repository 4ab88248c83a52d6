"""PRISM oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation of the PRISM
Newton–Schulz iterations of arXiv 2601.22137, written from the paper
(`/root/reference/PAPER.md`, cited as ``P:<line>``) and used to prove the
CUDA path right.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package ``paper_2601_22137_b200`` never imports it, and this
package never imports the product package: the two share no code (only the
seeded input generators of ``paper_2601_22137_b200.workloads``, which hold
none of the method's arithmetic, feed both sides from the tests).

Modules
-------
``philox``   counter-based Philox4x32-10 + portable fp64 Box–Muller that
             draws the Gaussian sketch S_k bit-for-bit the same
             way the device does (reading R8).
``prism``    the iterations (Table 1; Appendix A.1):
             residual, sketched trace table t_i, the paper's
             coefficient formulas, the quartic argmin,
             polar and coupled square-root drivers.

Parity status of every function is listed in DESIGN.md §"Oracle pins";
all oracle functions are pinned (no "parity unpinned" entries).
"""

from . import philox, prism  # noqa: F401
