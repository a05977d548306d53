"""CPU oracle for the parallel-in-time Newton path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / the timed CPU reference.  The product package
``paper_2409_20027_b200`` never imports it: its solver path is the CUDA
library and fails loudly when that library is missing.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference (``/root/reference/pkg/src/pintoc``) in the build container, runs
it on seeded cases and commits the outputs as ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .pintoc_oracle import *  # noqa: F401,F403
