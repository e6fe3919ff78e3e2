"""CPU oracle for the Jenga attention-carving hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package ``paper_2505_16864_b200`` never
imports it; there is no CPU fallback in the product path.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against fixtures in ``tests/golden/`` that were produced by running the real
reference package (``tokencarve`` 0.1.0 from ``/root/reference/pkg/src``) via
``tests/golden/make_golden.py``.
"""

from .port import *  # noqa: F401,F403
