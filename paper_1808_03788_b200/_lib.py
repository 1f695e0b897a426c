"""ctypes binding of libaderdg_b200.so (the C-ABI in include/aderdg_b200.h).

The shared library is built in-tree by `__graft_entry__.build()`
(`make -C paper_1808_03788_b200/csrc`) (nvcc, -gencode arch=compute_100a,code=sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
entry point raises.
"""

import ctypes
import os

LIB_NAME = "libaderdg_b200.so"
LIB_PATH = os.environ.get("ADG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

ADG_OK = 0
ADG_ERR_INVALID = 1
ADG_ERR_RUNTIME = 2
ADG_ERR_CUDA = 3
ADG_ERR_UNSUPPORTED = 4

BC_CODES = {"periodic": 0, "outflow": 1, "wall": 2, "exact": 3, "ghost": 3}
MODE_CODES = {"conservative": 0, "primitive": 1}   # adg_grid.mode (ADG_MODE_*)
GRID_FOLD_STATE = 1   # adg_grid.flags (ADG_GRID_FOLD_STATE)
SYSTEM_CODES = {"euler": 0, "advection": 1, "elasticity-di": 2}        # adg_grid.system (ADG_SYS_*)


def fill_system(g, system):
    """adg_grid plugin fields from a systems.* descriptor."""
    g.system = SYSTEM_CODES[system.name]
    g.gamma = float(getattr(system, "gamma", 1.4))
    vel = getattr(system, "velocity", None)
    for j in range(3):
        g.velocity[j] = float(vel[j]) if vel is not None and j < len(vel) else 0.0

STATUS_NO_ADMISSIBLE = 1
STATUS_NONFINITE = 2

# every symbol declared in include/aderdg_b200.h (checked by the CPU tests)
EXPORTS = (
    "adg_create", "adg_destroy", "adg_last_error", "adg_version", "adg_set_tables",
    "adg_wavespeed", "adg_timestep", "adg_advance_time", "adg_predict", "adg_face_flux", "adg_update",
    "adg_update_blocks", "adg_trace_block", "adg_totals_finalize", "adg_totals", "adg_state_record", "adg_fold_supported", "adg_minmod", "adg_relaxed_bounds", "adg_detect_cells", "adg_gather_windows", "adg_project_subcells",
    "adg_detect", "adg_rescue", "adg_flatten_ic", "adg_face_fluxes", "adg_volume_integral",
    "adg_face_integral", "adg_element_update", "adg_muscl_windows", "adg_recover_subcells",
    "adg_flatten_cells", "adg_log_step", "adg_predict_range", "adg_predict_range_supported",
    "adg_predict_ex", "adg_extract_traces", "adg_spacetime_rate", "adg_riemann_points",
    "adg_comm_unique_id", "adg_comm_init", "adg_comm_destroy", "adg_halo_exchange",
    "adg_allreduce_reduce", "adg_allreduce_sum",
)

COMM_ID_BYTES = 128

PRED_NOT_CONVERGED = 1   # pred_bad bits (ADG_PRED_*)
PRED_INADMISSIBLE = 2
PRED_STARTUP_ONLY = 1    # adg_predict_ex flags


class Grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("nvars", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("cells", ctypes.c_int64 * 3), ("dx", ctypes.c_double * 3),
                ("gamma", ctypes.c_double), ("bc", (ctypes.c_int32 * 2) * 3),
                ("system", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("velocity", ctypes.c_double * 3)]


class Reduce(ctypes.Structure):
    _fields_ = [("lam_bits", ctypes.c_uint64 * 3), ("n_admissible", ctypes.c_uint64),
                ("n_nonfinite", ctypes.c_uint64), ("reserved", ctypes.c_uint64 * 3)]


class SubcellGhosts(ctypes.Structure):
    """adg_subcell_ghosts: exterior subcell slabs of exact faces."""
    _fields_ = [("slab", (ctypes.c_void_p * 2) * 3), ("layers", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


REDUCE_WORDS = ctypes.sizeof(Reduce) // 8

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double

_SIGS = {
    "adg_create": (_I, [_I, ctypes.POINTER(_P)]),
    "adg_destroy": (_I, [_P]),
    "adg_last_error": (ctypes.c_char_p, [_P]),
    "adg_version": (_I, []),
    "adg_set_tables": (_I, [_P, _I, _P, _I64]),
    "adg_wavespeed": (_I, [_P, _P, _P, _P, _P]),
    "adg_timestep": (_I, [_P, _P, _P, _D, _P, _D, _P, _P, _P]),
    "adg_advance_time": (_I, [_P, _P, _P, _P, _P]),
    "adg_log_step": (_I, [_P, _P, _I64, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "adg_predict": (_I, [_P, _P, _P, _P, _D, _I, _I, _P, _P, _P, _P, _P, _P]),
    "adg_predict_range": (_I, [_P, _P, _I64, _I64, _P, _P, _D, _I, _I, _P, _P, _P, _P, _P, _P]),
    "adg_predict_range_supported": (_I, [_P]),
    "adg_predict_ex": (_I, [_P, _P, _P, _P, _P, _D, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "adg_extract_traces": (_I, [_P, _P, _P, _P, _P]),
    "adg_riemann_points": (_I, [_P, _P, _I64, _P, _I, _P, _P, _P, _P, _P, _P]),
    "adg_comm_unique_id": (_I, [_P]),
    "adg_comm_init": (_I, [_P, _P, _I, _I, ctypes.POINTER(_P)]),
    "adg_comm_destroy": (_I, [_P]),
    "adg_halo_exchange": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "adg_allreduce_reduce": (_I, [_P, _P, _P, _P]),
    "adg_allreduce_sum": (_I, [_P, _P, _P, _I64, _P]),
    "adg_spacetime_rate": (_I, [_P, _P, _P, _P, _P]),
    "adg_face_flux": (_I, [_P, _P, _I, _P, _P, _P, _P, _P]),
    "adg_update": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "adg_update_blocks": (_I64, [_P]),
    "adg_trace_block": (_I64, [_P]),
    "adg_totals_finalize": (_I, [_P, _P, _P, _I64, _P, _P]),
    "adg_totals": (_I, [_P, _P, _P, _P, _P, _P]),
    "adg_state_record": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "adg_fold_supported": (_I, [_P]),
    "adg_minmod": (_I, [_P, _I64, _P, _P, _P, _P]),
    "adg_relaxed_bounds": (_I, [_P, _I, _I, _P, _I, _P, _D, _D, _P, _P, _P, _P, _P]),
    "adg_detect_cells": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "adg_gather_windows": (_I, [_P, _I, _I, _P, _P, _P, _I64, _I, _P, _P]),
    "adg_project_subcells": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "adg_detect": (_I, [_P, _P, _P, _P, _P, _P, _P, _D, _D, _I, _P, _P, _P, _P, _P, _P, _P,
                        _P]),
    "adg_rescue": (_I, [_P, _P, _P, _P, _P, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "adg_flatten_ic": (_I, [_P, _P, _P, _P, _P]),
    "adg_face_fluxes": (_I, [_P, _P, _I, _I64, _P, _P, _P, _P, _P]),
    "adg_volume_integral": (_I, [_P, _P, _P, _P, _P, _P]),
    "adg_face_integral": (_I, [_P, _P, _I, _I, _P, _P, _P, _P]),
    "adg_element_update": (_I, [_P, _P, _P, _P, _P, _I, _P, _P]),
    "adg_muscl_windows": (_I, [_P, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "adg_recover_subcells": (_I, [_P, _P, _P, _P, _P]),
    "adg_flatten_cells": (_I, [_P, _P, _P, _P, _P, _P]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path=LIB_PATH):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(handle, rc, what):
    if rc == ADG_OK:
        return
    lib = load()
    msg = lib.adg_last_error(handle)
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg}"
    if rc == ADG_ERR_INVALID:
        raise ValueError(text)
    if rc == ADG_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise RuntimeError(text)


class Handle:
    """An adg_handle bound to one CUDA device; tables are uploaded on demand.

    `Handle.get(dev)` is the shared per-device handle of the module-level
    functions; every `Simulation` owns a private one (its predictor
    workspace is then never shared or reallocated under another
    Simulation's captured CUDA graphs)."""

    _per_device = {}

    def __init__(self, device_index):
        lib = load()
        h = _P()
        rc = lib.adg_create(int(device_index), ctypes.byref(h))
        if rc != ADG_OK:
            raise RuntimeError(f"adg_create failed on device {device_index} (rc={rc})")
        self.ptr = h
        self.device_index = device_index
        self.lib = lib
        self._degrees = set()

    @classmethod
    def get(cls, device_index):
        if device_index not in cls._per_device:
            cls._per_device[device_index] = Handle(device_index)
        return cls._per_device[device_index]

    def ensure_tables(self, tables):
        if tables.degree in self._degrees:
            return
        import numpy as np

        blob = np.ascontiguousarray(tables.device_blob(), dtype=np.float64)
        rc = self.lib.adg_set_tables(self.ptr, tables.degree, blob.ctypes.data, blob.size)
        check(self.ptr, rc, "adg_set_tables")
        self._degrees.add(tables.degree)

    def call(self, name, *args):
        rc = getattr(self.lib, name)(self.ptr, *args)
        check(self.ptr, rc, name)

    def stream(self):
        """cudaStream_t of torch's current stream on this handle's device."""
        import torch

        return torch.cuda.current_stream(self.device_index).cuda_stream

    def __del__(self):
        ptr, self.ptr = getattr(self, "ptr", None), None
        if ptr and getattr(self, "lib", None) is not None:
            try:
                self.lib.adg_destroy(ptr)
            except Exception:
                pass
