"""CPU oracle for the ADER-DG time step -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference algorithm
(`/root/reference/pkg/src/aderdg`, arXiv:1808.03788 desk implementation).
Every function cites the reference file:line it follows.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
`--impl reference` legs may import it, and only as the checker or as the
timed CPU baseline.  The product package `paper_1808_03788_b200` never
imports it; the GPU path fails loudly if its CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced
by running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`), see
`tests/test_oracle_golden.py`.
"""

from .basis import OracleTables, oracle_tables, time_operators  # noqa: F401
from .euler import EulerOracle  # noqa: F401
from .sim import OracleMesh, OracleSimulation  # noqa: F401
