"""CPU oracle for the GPU-SLS solver core — TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference ``scanmpc``
algorithm (``/root/reference/pkg/src/scanmpc``), written from its behaviour,
and used in exactly three places:

* ``tests/`` — as the checker the CUDA path is compared against;
* ``__graft_entry__.smoke()`` — one small check of the CUDA path;
* ``bench.py`` — the ``cpu_baseline`` leg and ``--impl reference`` arm.

Nothing in ``paper_2604_07644_b200`` (the product) imports this package; the
product path fails loudly when its CUDA library is missing and never falls
back to this code.

Parity status: PINNED.  ``tests/golden/*.npz`` hold outputs of the real
reference (generated in the build container by
``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks this
restatement against every fixture.
"""

from . import tree, lqr, admm, sls, sqp  # noqa: F401
from .lqr import relative_error  # noqa: F401
