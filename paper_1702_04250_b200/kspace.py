"""Drop-in Poisson solver: build_plan, poisson_ik, poisson_ad, kspace_energy.

Mirrors kspace.py:99-337 of the reference.  The transforms are cuFFT R2C/C2R
on the device (the reference uses full complex numpy FFTs and keeps the real
part; for the Hermitian spectra involved the two agree).  The influence-function
multiply, the ik gradient and the energy reduction are one hand-written
kernel (``k_green``); the influence function itself is evaluated on the
device (``k_influence``).  Forward transforms are unnormalised and the 1/M of
the backward transform is folded into the Green multiply, as in the
reference's convention (kspace.py:1-6).

``imag_residue`` (kspace.py:264-268) is measured on the device: the Green / ik
half spectra are expanded to the full grid through Hermitian symmetry and
transformed back with a complex inverse FFT (k_spectral.cu).

The plan's ``forward`` / ``backward`` pair (kspace.py:244) defaults to device
transforms with numpy ``fftn`` / ``ifftn`` semantics (``DeviceFFT``).  A
caller-supplied pair (``build_plan(fft=(fwd, bwd))``, the reference's
pluggable-transform hook) is honoured: the solve then runs the caller's
transforms and does the influence / ik multiply and the energy sum on the
device (``pppm_spectrum_apply``).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from . import _runtime as rt
from .model import ConfigurationError

DECONV_FLOOR = 1e-10


class DeviceFFT:
    """numpy ``fftn`` (forward, unnormalised) / ``ifftn`` (backward, 1/N)
    semantics on the device (cuFFT Z2Z, ``pppm_fftn``); 1-3 dimensional
    real or complex input, complex128 output."""

    def __init__(self, inverse: bool):
        self.inverse = bool(inverse)
        self.__name__ = "ifftn" if inverse else "fftn"

    def __call__(self, a):
        x = np.ascontiguousarray(a, dtype=np.complex128)
        if x.ndim < 1 or x.ndim > 3:
            raise ValueError("the device transform supports 1 to 3 dimensions")
        out = np.empty_like(x)
        if x.size == 0:
            raise ValueError("Invalid number of FFT data points (0) specified.")
        shape = np.array(x.shape, dtype=np.int64)
        nat.require_device(rt.get_device())
        nat.call("pppm_fftn", rt.get_device(), x.ndim, nat.ptr(shape), nat.ptr(x), nat.ptr(out),
                 1 if self.inverse else 0)
        return out

    def __repr__(self):
        return f"DeviceFFT({self.__name__})"


DEVICE_FFT = (DeviceFFT(False), DeviceFFT(True))


def _is_default_fft(forward, backward) -> bool:
    """The device pair, or numpy's own fftn / ifftn (the reference default,
    kspace.py:244): the same transforms as the device solve."""
    if isinstance(forward, DeviceFFT) and isinstance(backward, DeviceFFT):
        return True
    return forward is np.fft.fftn and backward is np.fft.ifftn


class KSpacePlan:
    """Solve plan: geometry, influence variant; G lives on the device.

    ``influence`` / ``ik_x`` / ``ik_y`` / ``ik_z`` are computed on the device
    and copied to the host only when read (read-only arrays, as in
    kspace.py:104-132).  ``forward`` / ``backward`` are the device transforms
    (``DEVICE_FFT``) unless the caller supplied its own ``fft`` pair, which the
    solve then runs (module docstring).
    """

    def __init__(self, dims, box_lengths, alpha, order, variant="pme", deconv_floor=DECONV_FLOOR,
                 fft=None):
        self.dims = tuple(int(d) for d in dims)
        self.box_lengths = np.array(box_lengths, dtype=np.float64)
        self.box_lengths.flags.writeable = False
        self.alpha = float(alpha)
        self.order = int(order)
        self.variant = variant
        self.deconv_floor = float(deconv_floor)
        self.forward, self.backward = fft if fft is not None else DEVICE_FFT
        self._influence = None
        self._ik = None

    @property
    def volume(self) -> float:
        return float(np.prod(self.box_lengths))

    @property
    def cell_volume(self) -> float:
        nx, ny, nz = self.dims
        return self.volume / (nx * ny * nz)

    def _ctx(self, mode_code, precision):
        ctx = rt.context(self.dims, self.box_lengths, self.order, mode_code, rt.prec_code(precision),
                         self.alpha)
        key = ("device", self.variant, self.deconv_floor)
        if ctx.green_key != key:
            kind = nat.INFLUENCE_PME if self.variant == "pme" else nat.INFLUENCE_OPTIMAL
            ctx("pppm_ctx_build_influence", kind, self.deconv_floor)
            ctx.green_key = key
        return ctx

    @property
    def influence(self):
        if self._influence is None:
            ctx = self._ctx(nat.MODE_AD, "fp64")
            nx, ny, nz = self.dims
            g = np.empty((nz, ny, nx))
            ctx("pppm_ctx_get_influence", nat.ptr(g))
            g.flags.writeable = False
            self._influence = g
        return self._influence

    def _ik_vectors(self):
        if self._ik is None:
            ctx = self._ctx(nat.MODE_AD, "fp64")
            nx, ny, nz = self.dims
            vx, vy, vz = np.empty(nx), np.empty(ny), np.empty(nz)
            ctx("pppm_ctx_get_ik", nat.ptr(vx), nat.ptr(vy), nat.ptr(vz))
            for v in (vx, vy, vz):
                v.flags.writeable = False
            self._ik = (vx, vy, vz)
        return self._ik

    @property
    def ik_x(self):
        return self._ik_vectors()[0]

    @property
    def ik_y(self):
        return self._ik_vectors()[1]

    @property
    def ik_z(self):
        return self._ik_vectors()[2]


def build_plan(dims, box, alpha, order, *, influence="pme", deconv_floor=DECONV_FLOOR, fft=None):
    """Plan for ``dims`` (kspace.py:199-256); validation identical to the reference."""
    dims = tuple(int(d) for d in dims)
    if any(d <= 0 for d in dims):
        raise ConfigurationError("grid dimensions must be positive")
    if any(d < order for d in dims):
        raise ConfigurationError("grid dimensions must be >= the stencil order")
    if alpha <= 0.0:
        raise ConfigurationError("alpha must be positive")
    if influence not in ("pme", "optimal"):
        raise ConfigurationError(f"unknown influence variant {influence!r}")
    plan = KSpacePlan(dims, box.lengths, alpha, order, influence, deconv_floor, fft)
    ref_plan = rt.types().KSpacePlan
    if ref_plan is None:
        return plan
    # installed into the reference: hand back its own (frozen) plan type
    return ref_plan(dims=dims, box_lengths=np.asarray(box.lengths), alpha=float(alpha),
                    order=int(order), influence=plan.influence, ik_x=plan.ik_x, ik_y=plan.ik_y,
                    ik_z=plan.ik_z, forward=plan.forward, backward=plan.backward)


def _plan_ctx(plan, mode_code, precision):
    if isinstance(plan, KSpacePlan):
        return plan._ctx(mode_code, precision)
    # a foreign plan (e.g. the reference's KSpacePlan): upload its influence grid
    ctx = rt.context(plan.dims, plan.box_lengths, plan.order, mode_code, rt.prec_code(precision),
                     plan.alpha)
    g = np.ascontiguousarray(plan.influence, dtype=np.float64)
    key = ("host", id(plan.influence), g.ctypes.data)
    if ctx.green_key != key:
        ctx("pppm_ctx_set_influence", nat.ptr(g))
        ctx.green_key = key
        ctx._green_ref = g
    return ctx


def _check_grid(grid, plan):
    if tuple(grid.dims) != tuple(plan.dims):
        raise ValueError(f"grid dims {grid.dims} do not match plan dims {plan.dims}")


def _residue(e, real):
    """kspace.py:264-268 on the caller's complex back transform."""
    scale = float(np.max(np.abs(real)))
    if scale == 0.0:
        return 0.0
    return float(np.max(np.abs(np.asarray(e).imag))) / scale


def _solve_custom(rho, plan, ctx, mode_code):
    """Caller-supplied transforms: forward / backward are the caller's, the
    influence and ik multiply run on the device (kspace.py:278-312)."""
    rho_hat = np.ascontiguousarray(plan.forward(rho.values), dtype=np.complex128)
    if rho_hat.shape != ctx.mesh_shape:
        raise ValueError(f"forward transform returned shape {rho_hat.shape}, expected {ctx.mesh_shape}")
    comps = (0, 1, 2) if mode_code == nat.MODE_IK else (-1,)
    outs, residue = [], 0.0
    for comp in comps:
        spec = np.empty_like(rho_hat)
        ctx("pppm_spectrum_apply", nat.ptr(rho_hat), comp, nat.ptr(spec), None)
        e = plan.backward(spec)
        real = np.ascontiguousarray(np.real(e), dtype=np.float64)
        residue = max(residue, _residue(e, real))
        real.flags.writeable = False
        outs.append(real)
    return outs, residue


def _solve(rho, plan, mode_code):
    _check_grid(rho, plan)
    ctx = _plan_ctx(plan, mode_code, rt.get_precision())
    if not _is_default_fft(plan.forward, plan.backward):
        return _solve_custom(rho, plan, ctx, mode_code)
    values = np.ascontiguousarray(rho.values, dtype=np.float64)
    ctx("pppm_set_rho", nat.ptr(values))
    energy = np.zeros(1)
    ctx("pppm_poisson", 2, energy.ctypes.data_as(nat._dp))  # fields + measured imag_residue
    outs = [np.empty(ctx.mesh_shape) for _ in range(3 if mode_code == nat.MODE_IK else 1)]
    ptrs = [nat.ptr(a) for a in outs] + [None] * (3 - len(outs))
    ctx("pppm_get_fields", *ptrs)
    for a in outs:
        a.flags.writeable = False
    residue = np.zeros(1)
    ctx("pppm_get_imag_residue", residue.ctypes.data_as(nat._dp))
    return outs, float(residue[0])


def poisson_ik(rho, plan):
    """E_d = -i k_d G rho^ transformed back, three grids (kspace.py:271-300)."""
    (ex, ey, ez), residue = _solve(rho, plan, nat.MODE_IK)
    T = rt.types()
    return T.FieldGrids(mode=T.DiffMode.IK, dims=rho.dims, spacing=rho.spacing, ex=ex, ey=ey, ez=ez,
                        imag_residue=residue)


def poisson_ad(rho, plan):
    """phi = G rho^ transformed back, one grid (kspace.py:303-317)."""
    (phi,), residue = _solve(rho, plan, nat.MODE_AD)
    T = rt.types()
    return T.FieldGrids(mode=T.DiffMode.AD, dims=rho.dims, spacing=rho.spacing, phi=phi,
                        imag_residue=residue)


def kspace_energy(rho, plan, *, coulomb_constant=1.0, dielectric=1.0):
    """C/eps * Vc^2/(2V) * sum_k G |rho^|^2 (kspace.py:320-337), reduced in fp64 on the device."""
    _check_grid(rho, plan)
    ctx = _plan_ctx(plan, nat.MODE_AD, rt.get_precision())
    scale = coulomb_constant / dielectric
    if not _is_default_fft(plan.forward, plan.backward):
        rho_hat = np.ascontiguousarray(plan.forward(rho.values), dtype=np.complex128)
        total = np.zeros(1)
        ctx("pppm_spectrum_apply", nat.ptr(rho_hat), -1, None, total.ctypes.data_as(nat._dp))
        nx, ny, nz = plan.dims
        volume = float(np.prod(plan.box_lengths))
        vcell = volume / (nx * ny * nz)
        return scale * vcell ** 2 / (2.0 * volume) * float(total[0])
    values = np.ascontiguousarray(rho.values, dtype=np.float64)
    ctx("pppm_set_rho", nat.ptr(values))
    energy = np.zeros(1)
    ctx("pppm_poisson", 0, energy.ctypes.data_as(nat._dp))
    return float(energy[0]) * scale
