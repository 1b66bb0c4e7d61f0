"""Device-resident PPPM context: the performance path.

Atoms are uploaded once; make_rho -> Poisson -> fieldforce then run on the
context stream with every mesh, spectrum and field buffer resident in HBM
(SURVEY §8b "performance note").  This is what ``bench.py`` times, and what a
time-stepping caller (driver.integrate_nve, driver.py:310-376) would hold
across steps.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import _runtime as rt


class PppmContext:
    """One mesh geometry on one device with resident atoms.

    Parameters mirror ``PppmParams`` plus ``precision`` ("fp64" | "mixed").
    """

    def __init__(self, dims, lengths, order=5, mode="ik", precision="mixed", alpha=0.3,
                 coulomb_constant=1.0, dielectric=1.0, table_points=0, influence="pme",
                 device=None, deconv_floor=1e-10):
        device = rt.get_device() if device is None else int(device)
        self.precision = "mixed" if precision == "fp32" else precision
        self.mode = mode
        self.order = int(order)
        self.dims = tuple(int(d) for d in dims)
        self.ctx = nat.Context(device, self.dims, lengths, self.order, rt.mode_code(mode),
                               rt.prec_code(self.precision), alpha, coulomb_constant, dielectric)
        kind = nat.INFLUENCE_PME if influence == "pme" else nat.INFLUENCE_OPTIMAL
        self.ctx("pppm_ctx_build_influence", kind, float(deconv_floor))
        self.ctx("pppm_ctx_build_table", int(table_points))
        self.n_atoms = 0

    def load_atoms(self, positions, charges):
        """Copy atoms to the device once.  fp32 arrays are used as-is; fp64
        arrays are rounded on the device in mixed precision."""
        pos = np.ascontiguousarray(positions)
        q = np.ascontiguousarray(charges)
        if pos.dtype == np.float32 and q.dtype != np.float32:
            q = q.astype(np.float32)
        if pos.dtype != np.float32:
            pos = pos.astype(np.float64, copy=False)
            q = q.astype(np.float64, copy=False)
        dtype = nat.F32 if pos.dtype == np.float32 else nat.F64
        self.ctx("pppm_ctx_load_atoms", nat.ptr(pos), nat.ptr(q), pos.shape[0], dtype)
        self.n_atoms = pos.shape[0]

    def update_positions(self, positions):
        """Move the resident atoms (caller's order) without re-sorting them."""
        pos = np.ascontiguousarray(positions)
        if pos.dtype != np.float32:
            pos = pos.astype(np.float64, copy=False)
        dtype = nat.F32 if pos.dtype == np.float32 else nat.F64
        self.ctx("pppm_ctx_update_positions", nat.ptr(pos), dtype, nat.HOST)

    def update_positions_async(self, positions, mem=nat.HOST):
        """MD position update without waiting (device pointers: ``mem=DEVICE``
        with an integer address); errors surface at the next synchronize."""
        if mem == nat.DEVICE:
            self.ctx("pppm_ctx_update_positions_async", ctypes.c_void_p(int(positions)), nat.F32, nat.DEVICE)
            return
        pos = np.ascontiguousarray(positions)
        dtype = nat.F32 if pos.dtype == np.float32 else nat.F64
        self._pending = pos  # keep the host buffer alive until the copy ran
        self.ctx("pppm_ctx_update_positions_async", nat.ptr(pos), dtype, nat.HOST)

    def set_resort(self, fraction):
        """Re-sort the residents when more than ``fraction`` of them left their brick."""
        self.ctx("pppm_ctx_set_resort", float(fraction))

    def resident_info(self):
        info = (ctypes.c_int64 * 4)()
        self.ctx("pppm_ctx_resident_info", info)
        return dict(zip(("movers", "resorts", "max_brick", "n"), list(info)))

    def set_variant(self, kernel, variant):
        self.ctx("pppm_ctx_set_variant", int(kernel), int(variant))

    def step(self, phases=nat.PHASE_ALL):
        self.ctx("pppm_ctx_step", int(phases))

    def synchronize(self):
        self.ctx("pppm_ctx_synchronize")

    def forces(self):
        out = np.empty((self.n_atoms, 3))
        self.ctx("pppm_ctx_get_forces", nat.ptr(out))
        return out

    def energy(self):
        e = np.zeros(1)
        self.ctx("pppm_ctx_get_energy", e.ctypes.data_as(nat._dp))
        return float(e[0])

    def rho(self):
        out = np.empty(self.ctx.mesh_shape)
        self.ctx("pppm_get_rho", nat.ptr(out))
        return out

    def fields(self):
        nf = 3 if self.mode == "ik" else 1
        outs = [np.empty(self.ctx.mesh_shape) for _ in range(nf)]
        ptrs = [nat.ptr(a) for a in outs] + [None] * (3 - nf)
        self.ctx("pppm_get_fields", *ptrs)
        return outs

    def time_steps(self, steps, warmup, flush_l2=True):
        """CUDA-event phase times in ms summed over ``steps``:
        dict(bin, spread, poisson, gather, total)."""
        ms = np.zeros(5)
        self.ctx("pppm_ctx_time_steps", int(steps), int(warmup), int(bool(flush_l2)), nat.ptr(ms))
        keys = ("bin", "spread", "poisson", "gather", "total")
        return dict(zip(keys, (float(v) for v in ms)))

    def launches_per_step(self):
        n = ctypes.c_int(0)
        self.ctx("pppm_ctx_launches_per_step", ctypes.byref(n))
        return n.value

    def compute(self, positions, charges, mem=nat.HOST, out=None):
        """One full evaluation through the C ABI with host buffers (H2D, step, D2H).
        ``out``: optional (n, 3) float64 destination (e.g. a pinned PinnedArray
        view), or float32 on a mixed-precision context (the path's own precision)."""
        pos = np.ascontiguousarray(positions)
        q = np.ascontiguousarray(charges)
        dtype = nat.F32 if pos.dtype == np.float32 else nat.F64
        if out is None:
            forces = np.empty((pos.shape[0], 3))
        else:
            forces = out
            if (forces.shape != (pos.shape[0], 3) or forces.dtype not in (np.float64, np.float32)
                    or not forces.flags.c_contiguous):
                raise ValueError("out must be a C-contiguous (n, 3) float64 or float32 array")
        e = np.zeros(1)
        fdt = nat.F64 if forces.dtype == np.float64 else nat.F32
        self.ctx("pppm_compute_ex", nat.ptr(pos), nat.ptr(q), pos.shape[0], dtype, mem, nat.ptr(forces), fdt,
                 e.ctypes.data_as(nat._dp))
        return forces, float(e[0])

    def close(self):
        self.ctx.close()


class PinnedArray:
    """numpy view over pinned host memory from ``pppm_host_alloc``."""

    def __init__(self, shape, dtype):
        self.dtype = np.dtype(dtype)
        self.shape = tuple(shape)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        self._p = nat.load().pppm_host_alloc(max(nbytes, 1))
        if not self._p:
            raise RuntimeError("pinned host allocation failed")
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def free(self):
        if self._p:
            self.array = None
            nat.load().pppm_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
