"""Shared plumbing of the module-level shims (corrector.py, limiter.py):
device tensors in the reference layouts and a flattened-grid adg_grid."""

import numpy as np
import torch

from . import _lib


def as_device(a, device=None):
    """fp64 contiguous CUDA tensor (numpy arrays are uploaded)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1808_03788_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to(device or torch.cuda.current_device())
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64),
                            device=device or torch.cuda.current_device())
    return t.to(dtype=torch.float64).contiguous()


def require_euler(system):
    if getattr(system, "name", None) != "euler":
        raise NotImplementedError(
            f"system '{getattr(system, 'name', system)}' has no B200 kernels (Euler only)")


def flat_grid(system, degree, n_elem, spacings=None, mode="conservative"):
    """adg_grid of E = n_elem elements along axis 0 (element-local calls)."""
    g = _lib.Grid()
    d = system.dim
    g.dim, g.degree, g.nvars = d, int(degree), system.n_vars
    g.mode = _lib.MODE_CODES[mode]
    for j in range(3):
        g.cells[j] = int(max(n_elem, 1)) if j == 0 else 1
        g.dx[j] = float(spacings[j]) if (spacings is not None and j < d) else 1.0
    _lib.fill_system(g, system)
    return g


def handle_for(t, tables=None):
    h = _lib.Handle.get(t.device.index)
    if tables is not None:
        h.ensure_tables(tables)
    return h


def scalar(x, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).reshape(1).contiguous()
    return torch.full((1,), float(x), dtype=torch.float64, device=device)
