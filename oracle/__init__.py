"""CPU oracle for the kernel-OT SSN hot path — TEST INFRASTRUCTURE ONLY.

This package is a NumPy restatement of the reference algorithm
(``/root/reference/pkg/src/kot``), used exclusively as the *checker* by
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py``.  The product path
(``paper_2310_14087_b200``) never imports it and has no CPU fallback.

Pinning: ``tests/test_oracle_golden.py`` checks this port against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``
imports ``kot`` from ``/root/reference/pkg/src`` in the build container and
writes ``tests/golden/*.npz``) and against the reference's own known-answer
tests (``pkg/tests/test_linalg.py``, ``pkg/tests/test_psdcone.py``).
"""

from oracle.kot_port import *  # noqa: F401,F403
