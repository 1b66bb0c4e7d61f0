"""ctypes binding of the C ABI in ``include/pppm_b200.h`` (``libpppm_b200.so``).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the library is missing or no CUDA device is present, every entry
point raises.  Status codes map onto the reference's exception types
(model.py:21-31): PPPM_ERR_CONFIG -> ConfigurationError, PPPM_ERR_VALUE ->
ValueError, everything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_NAME = "libpppm_b200.so"
LIB_PATH = os.environ.get("PPPM_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OK, ERR_CONFIG, ERR_VALUE, ERR_RUNTIME, ERR_CUDA, ERR_CUFFT, ERR_STATE, ERR_NCCL, ERR_SINGULAR = range(9)
MODE_IK, MODE_AD = 0, 1
PREC_FP64, PREC_MIXED = 0, 1
F64, F32 = 0, 1
HOST, DEVICE = 0, 1
INFLUENCE_PME, INFLUENCE_OPTIMAL = 0, 1
PHASE_MAKE_RHO, PHASE_POISSON, PHASE_FIELDFORCE, PHASE_ALL = 1, 2, 4, 7

_c_int = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip32 = ctypes.POINTER(ctypes.c_int32)

# name -> (restype, argtypes); mirrors include/pppm_b200.h
PROTOTYPES = {
    "pppm_abi_version": (_c_int, []),
    "pppm_last_error": (ctypes.c_char_p, []),
    "pppm_device_count": (_c_int, [ctypes.POINTER(_c_int)]),
    "pppm_host_alloc": (_vp, [ctypes.c_size_t]),
    "pppm_host_free": (None, [_vp]),
    "pppm_weight_rows": (_c_int, [_c_int, _c_int, _vp, _c_i64, _vp, _vp]),
    "pppm_table_rows": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp]),
    "pppm_ctx_create": (_c_int, [ctypes.POINTER(_vp), _c_int, _c_int, _c_int, _c_int, _c_dbl, _c_dbl,
                                 _c_dbl, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl]),
    "pppm_ctx_destroy": (_c_int, [_vp]),
    "pppm_ctx_set_table": (_c_int, [_vp, _c_int, _vp, _vp]),
    "pppm_ctx_build_table": (_c_int, [_vp, _c_int]),
    "pppm_ctx_build_influence": (_c_int, [_vp, _c_int, _c_dbl]),
    "pppm_ctx_set_influence": (_c_int, [_vp, _vp]),
    "pppm_ctx_get_influence": (_c_int, [_vp, _vp]),
    "pppm_ctx_get_ik": (_c_int, [_vp, _vp, _vp, _vp]),
    "pppm_particle_map": (_c_int, [_vp, _vp, _c_i64, _c_int, _c_int, _vp]),
    "pppm_make_rho": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _vp]),
    "pppm_set_rho": (_c_int, [_vp, _vp]),
    "pppm_get_rho": (_c_int, [_vp, _vp]),
    "pppm_poisson": (_c_int, [_vp, _c_int, _dp]),
    "pppm_get_fields": (_c_int, [_vp, _vp, _vp, _vp]),
    "pppm_set_fields": (_c_int, [_vp, _vp, _vp, _vp]),
    "pppm_fieldforce": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _vp]),
    "pppm_compute": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _vp, _dp]),
    "pppm_compute_ex": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _vp, _c_int, _dp]),
    "pppm_ctx_load_atoms": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int]),
    "pppm_ctx_step": (_c_int, [_vp, _c_int]),
    "pppm_ctx_synchronize": (_c_int, [_vp]),
    "pppm_ctx_get_forces": (_c_int, [_vp, _vp]),
    "pppm_ctx_update_positions": (_c_int, [_vp, _vp, _c_int, _c_int]),
    "pppm_ctx_update_positions_async": (_c_int, [_vp, _vp, _c_int, _c_int]),
    "pppm_ctx_set_resort": (_c_int, [_vp, _c_dbl]),
    "pppm_ctx_resident_info": (_c_int, [_vp, ctypes.POINTER(_c_i64)]),
    "pppm_ctx_get_energy": (_c_int, [_vp, _dp]),
    "pppm_ctx_time_steps": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp]),
    "pppm_ctx_launches_per_step": (_c_int, [_vp, ctypes.POINTER(_c_int)]),
    "pppm_ctx_set_variant": (_c_int, [_vp, _c_int, _c_int]),
    "pppm_ctx_create_slab": (_c_int, [ctypes.POINTER(_vp), _c_int, _c_int, _c_int, _c_int, _c_dbl, _c_dbl,
                                      _c_dbl, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl, _c_int, _c_int]),
    "pppm_ctx_stream": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "pppm_ctx_launch_count": (_c_int, [_vp, ctypes.POINTER(_c_i64)]),
    "pppm_slab_info": (_c_int, [_vp, ctypes.POINTER(_c_int)]),
    "pppm_slab_buffer": (_c_int, [_vp, _c_int, _c_int, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t)]),
    "pppm_slab_make_rho": (_c_int, [_vp]),
    "pppm_slab_add_ghosts": (_c_int, [_vp]),
    "pppm_slab_fft_fwd": (_c_int, [_vp]),
    "pppm_slab_green": (_c_int, [_vp]),
    "pppm_slab_fft_bwd": (_c_int, [_vp]),
    "pppm_slab_fieldforce": (_c_int, [_vp]),
    "pppm_ctx_pair_forces": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _c_dbl, _c_dbl, _vp, _vp, _dp,
                                      _vp]),
    "pppm_singular_pair": (_c_int, [ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong), _dp]),
    "pppm_ctx_compute_forces": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _c_int, _c_dbl, _vp, _vp, _vp, _vp,
                                         _vp]),
    "pppm_nccl_unique_id": (_c_int, [ctypes.c_char_p]),
    "pppm_slab_attach_nccl": (_c_int, [_vp, ctypes.c_char_p, _c_dbl]),
    "pppm_fftn": (_c_int, [_c_int, _c_int, _vp, _vp, _vp, _c_int]),
    "pppm_get_imag_residue": (_c_int, [_vp, _dp]),
    "pppm_spectrum_apply": (_c_int, [_vp, _vp, _c_int, _vp, _dp]),
    "pppm_ctx_integrate_nve": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int, _c_dbl, _vp, _vp, _vp,
                                        _vp, _vp, _vp]),
}


class _ErrorTypes:
    """Exception classes raised for status codes; install() may swap in the reference's."""

    def __init__(self):
        from .model import ConfigurationError

        self.config = ConfigurationError
        self.value = ValueError
        self.runtime = RuntimeError
        self.singular = None  # SingularityError class (model.SingularityError unless install() swaps it)


ERRORS = _ErrorTypes()

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return LIB_PATH


def load(path: str | None = None):
    """Load (once) and return the native library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"{p} is missing: build the CUDA library first (python -c "
                "'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        lib = ctypes.CDLL(p)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pppm_abi_version() != 1:
            raise RuntimeError("libpppm_b200 ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().pppm_last_error()
    return msg.decode() if msg else ""


def check(status: int):
    """Raise the exception type mapped to ``status``."""
    if status == OK:
        return
    msg = last_error()
    if status == ERR_CONFIG:
        raise ERRORS.config(msg)
    if status == ERR_VALUE:
        raise ERRORS.value(msg)
    if status == ERR_SINGULAR:
        i, j, r = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_double()
        load().pppm_singular_pair(ctypes.byref(i), ctypes.byref(j), ctypes.byref(r))
        from .model import SingularityError

        cls = ERRORS.singular or SingularityError
        exc = cls(i.value, j.value, r.value)
        if msg.startswith("step "):  # integrate_nve's step prefix (driver.py:345-347)
            exc.args = (msg,)
        raise exc
    if status == ERR_RUNTIME:
        raise ERRORS.runtime(msg)
    raise ERRORS.runtime(f"pppm_b200 error {status}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = ctypes.c_int(0)
    st = load().pppm_device_count(ctypes.byref(n))
    if st != OK:
        return 0
    return n.value


def require_device(device: int = 0):
    n = device_count()
    if n <= device:
        raise RuntimeError(
            f"pppm_b200 needs CUDA device {device} but {n} device(s) are visible; "
            "there is no CPU fallback")


class Context:
    """Owning handle of one ``pppm_ctx`` (one mesh geometry on one device)."""

    def __init__(self, device, dims, lengths, order, mode, precision, alpha,
                 coulomb_constant=1.0, dielectric=1.0):
        require_device(device)
        self.device = int(device)
        self.dims = tuple(int(d) for d in dims)
        self.lengths = tuple(float(v) for v in lengths)
        self.order = int(order)
        self.mode = int(mode)
        self.precision = int(precision)
        self.alpha = float(alpha)
        h = ctypes.c_void_p()
        nx, ny, nz = self.dims
        lx, ly, lz = self.lengths
        call("pppm_ctx_create", ctypes.byref(h), self.device, nx, ny, nz, lx, ly, lz, self.order,
             self.mode, self.precision, self.alpha, float(coulomb_constant), float(dielectric))
        self.handle = h
        self.table_key = None
        self.green_key = None
        self.lock = threading.Lock()

    @property
    def mesh_shape(self):
        nx, ny, nz = self.dims
        return (nz, ny, nx)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib = _lib
            if lib is not None:
                lib.pppm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __call__(self, name, *args):
        call(name, self.handle, *args)
