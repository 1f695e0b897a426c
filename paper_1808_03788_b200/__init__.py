"""B200-native (sm_100a) ADER-DG time step for the compressible Euler
equations -- a drop-in for the reference `aderdg` solver API
(/root/reference/pkg/src/aderdg/__init__.py:3-11).

    from paper_1808_03788_b200 import CartesianMesh, Simulation, make_system

The hot path (predictor, corrector, limiter, CFL reduction) runs in the
hand-written CUDA library `libaderdg_b200.so` through a ctypes C-ABI
(include/aderdg_b200.h); PyTorch only provides device memory and streams.
"""

from .basis import BasisTables, basis_tables
from .mesh import CartesianMesh
from .problems import build_problem
from .systems import make_system

__all__ = ["BasisTables", "CartesianMesh", "DEFAULT_CFL", "Simulation",
           "basis_tables", "build_problem", "default_cfl", "make_system"]
__version__ = "0.1.0"


def __getattr__(name):
    # the driver imports torch; keep `import paper_1808_03788_b200` light
    if name in ("Simulation", "DEFAULT_CFL", "default_cfl"):
        from . import driver

        return getattr(driver, name)
    raise AttributeError(name)
