"""CPU oracle for the PPPM particle-mesh hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The shipped package
``paper_1702_04250_b200`` never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

It is a numpy restatement of the reference algorithm of
``arxiv/paper_1702_04250`` (package ``pppm`` 0.1.0, pure Python/numpy), written
against plain arrays instead of the reference's dataclasses.  Every function
cites the reference ``file:line`` (paths relative to ``pkg/src/pppm/``) whose
behaviour it restates.

Parity pin: ``tests/golden/*.npz`` hold outputs of the real reference run in
the build container by ``tests/golden/make_golden.py``; the CPU test suite
(``tests/test_oracle_golden.py``) checks this oracle against every one of
them, bit-exact where the reference arithmetic is reproduced op-for-op
(stencil rows, table rows, node indices) and to 1e-12 elsewhere.

Extension not in the reference (parity UNPINNED by the reference): even
orders S = 4 and 6 (BASELINE config 4).  The reference rejects them
(model.py:18 SUPPORTED_ORDERS).  The registration used here puts the atom
between nodes floor(u) and floor(u)+1: node = floor(u), t = frac(u) - 1/2,
lowest stencil node = node - (S-1)//2.  For odd S the reference rule
(gridmap.py:105-109) is kept exactly.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROW_PAD = 8            # stencil.py:23 (rows are zero-padded to 8)
DECONV_FLOOR = 1e-10   # kspace.py:36
ODD_ORDERS = (3, 5, 7)
ALL_ORDERS = (3, 4, 5, 6, 7)


# --------------------------------------------------------------------------
# compute_rho1d / compute_drho1d


def bspline_rows(t, order):
    """Assignment and derivative rows at offsets ``t`` (stencil.py:38-77).

    Triangular recurrence on the cardinal B-spline samples M_m(w + k),
    w = t + 1/2, m = 2..order; the derivative row is taken from the order-1
    samples (M_S'(x) = M_{S-1}(x) - M_{S-1}(x-1)).  The arithmetic is the
    reference's op for op (no fused multiply-add), so rows are bitwise equal
    to the reference's.  Returns two arrays of shape ``t.shape + (8,)``,
    lowest grid node first.
    """
    t = np.asarray(t, dtype=np.float64)
    w = t + 0.5
    cols = [np.ones_like(w)]                      # M_1 samples
    dcols = None
    for m in range(2, order + 1):
        if m == order:
            # derivative from the M_{S-1} samples (stencil.py:58-64)
            dcols = [cols[0]]
            dcols += [cols[k] - cols[k - 1] for k in range(1, order - 1)]
            dcols.append(-cols[order - 2])
        den = m - 1
        nxt = [w * cols[0] / den]
        for k in range(1, m - 1):
            nxt.append(((w + k) * cols[k] + (m - w - k) * cols[k - 1]) / den)
        nxt.append((m - w - (m - 1)) * cols[m - 2] / den)
        cols = nxt
    assign = np.zeros(t.shape + (ROW_PAD,))
    deriv = np.zeros(t.shape + (ROW_PAD,))
    for i in range(order):                       # node i <- sample order-1-i
        assign[..., i] = cols[order - 1 - i]
        deriv[..., i] = dcols[order - 1 - i]
    return assign, deriv


def table_centers(n_points):
    """Bin-centre offsets of the lookup table (stencil.py:135)."""
    return -0.5 + (np.arange(n_points) + 0.5) / n_points


def table_rows(order, n_points):
    """(n_points, 8) assignment / derivative rows at bin centres (stencil.py:129-139)."""
    return bspline_rows(table_centers(int(n_points)), order)


def table_bin(t, n_points):
    """Half-open bin of offset ``t``, clipped (stencil.py:123-126)."""
    k = np.floor((np.asarray(t, dtype=np.float64) + 0.5) * n_points).astype(np.int64)
    return np.clip(k, 0, n_points - 1)


# --------------------------------------------------------------------------
# particle_map


def spacing(lengths, dims):
    """h_d = L_d / n_d in fp64 (gridmap.py:81-89)."""
    return tuple(float(lengths[d]) / int(dims[d]) for d in range(3))


def particle_map(pos, lengths, dims, order):
    """Per-dimension nearest node (pre-wrap) and clipped offset (gridmap.py:103-109).

    Returns ``nodes`` (3, N) int64 and ``t`` (3, N) float64, dimension order
    x, y, z.  Odd orders follow the reference exactly: u = x / h,
    node = floor(u + 1/2), t = clip(u - node, -1/2, nextafter(1/2, 0)); the
    node may equal n_d before wrapping.  Even orders use the extension rule
    described in the module docstring.
    """
    pos = np.asarray(pos, dtype=np.float64)
    h = spacing(lengths, dims)
    top = np.nextafter(0.5, 0.0)
    nodes = np.empty((3, pos.shape[0]), dtype=np.int64)
    offs = np.empty((3, pos.shape[0]))
    for d in range(3):
        u = pos[:, d] / h[d]
        if order % 2:
            node = np.floor(u + 0.5)
            t = u - node
        else:
            node = np.floor(u)
            t = (u - node) - 0.5
        offs[d] = np.clip(t, -0.5, top)
        nodes[d] = node.astype(np.int64)
    return nodes, offs


def check_positions(pos, lengths, dims, order):
    """Domain checks of gridmap.py:85-88 (raises like the reference)."""
    if any(int(dims[d]) < order for d in range(3)):
        raise ValueError("grid dimensions must be >= the stencil order")
    pos = np.asarray(pos, dtype=np.float64)
    if np.any(pos < 0.0) or np.any(pos >= np.asarray(lengths, dtype=np.float64)):
        raise RuntimeError("positions must be wrapped into the box before mapping")


def stencil_weights(pos, lengths, dims, order, table=None):
    """Nodes plus per-dimension rows (gridmap.py:92-119).

    ``table`` is ``None`` (exact rows) or a tuple ``(assign, deriv)`` of
    (n_points, 8) arrays (table mode).  Returns ``nodes`` (3, N) and two
    lists of three (N, 8) arrays (x, y, z).
    """
    nodes, offs = particle_map(pos, lengths, dims, order)
    arows, drows = [], []
    for d in range(3):
        if table is not None:
            ta, td = table
            k = table_bin(offs[d], ta.shape[0])
            arows.append(ta[k])
            drows.append(td[k])
        else:
            a, b = bspline_rows(offs[d], order)
            arows.append(a)
            drows.append(b)
    return nodes, arows, drows


def stencil_indices(nodes, dims, order):
    """Periodic grid index of every stencil entry, (N, order) per dim (gridmap.py:122-129)."""
    lo = (order - 1) // 2
    steps = np.arange(order) - lo
    return [(nodes[d][:, None] + steps[None, :]) % int(dims[d]) for d in range(3)]


# --------------------------------------------------------------------------
# make_rho


def _spread(acc, q, ix, iy, iz, wx, wy, wz):
    """Atom-major scatter of ((q wz) wy) wx (gridmap.py:141-153)."""
    c = q[:, None, None, None] * wz[:, :, None, None]
    c = c * wy[:, None, :, None]
    c = c * wx[:, None, None, :]
    np.add.at(acc, (iz[:, :, None, None], iy[:, None, :, None], ix[:, None, None, :]), c)


def map_charge(pos, q, lengths, dims, order, table=None, *, workers=1, chunk=1 << 16):
    """Charge density on the (nz, ny, nx) mesh (gridmap.py:156-213).

    ``workers`` > 1 scatters contiguous atom subsets into private replicas
    that are summed in replica order (gridmap.py:186-207).  Chunking is the
    same scatter sequence as one pass (np.add.at is sequential), so results
    are bitwise independent of ``chunk``.
    """
    check_positions(pos, lengths, dims, order)
    pos = np.asarray(pos, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    nx, ny, nz = (int(d) for d in dims)
    h = spacing(lengths, dims)

    def scatter(lo_i, hi_i, acc):
        for s in range(lo_i, hi_i, chunk):
            e = min(hi_i, s + chunk)
            nodes, arows, _ = stencil_weights(pos[s:e], lengths, dims, order, table)
            ix, iy, iz = stencil_indices(nodes, dims, order)
            wx, wy, wz = (r[:, :order] for r in arows)
            _spread(acc, q[s:e], ix, iy, iz, wx, wy, wz)
        return acc

    n = pos.shape[0]
    workers = max(1, int(workers))
    if workers == 1:
        grid = scatter(0, n, np.zeros((nz, ny, nx)))
    else:
        # np.array_split boundaries: first (n % workers) parts get one extra
        sizes = [n // workers + (1 if i < n % workers else 0) for i in range(workers)]
        bounds = np.concatenate([[0], np.cumsum(sizes)])
        with ThreadPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(
                lambda i: scatter(bounds[i], bounds[i + 1], np.zeros((nz, ny, nx))),
                range(workers)))
        grid = parts[0]
        for p in parts[1:]:
            grid += p
    grid /= h[0] * h[1] * h[2]
    return grid


# --------------------------------------------------------------------------
# Poisson solve


def mode_numbers(n):
    """FFT-layout integer modes (kspace.py:135-136)."""
    return np.fft.fftfreq(n, d=1.0 / n)


def sinc_pow(m, n, order):
    """sinc(m/n)^S (kspace.py:99-101)."""
    return np.sinc(np.asarray(m, dtype=np.float64) / n) ** order


def influence_pme(dims, lengths, alpha, order, floor=DECONV_FLOOR):
    """Smooth-splitting influence function on the full (nz, ny, nx) grid (kspace.py:139-159)."""
    nx, ny, nz = (int(d) for d in dims)
    lx, ly, lz = (float(v) for v in lengths)
    mx, my, mz = mode_numbers(nx), mode_numbers(ny), mode_numbers(nz)
    two_pi = 2.0 * np.pi
    kx, ky, kz = two_pi * mx / lx, two_pi * my / ly, two_pi * mz / lz
    k2 = kz[:, None, None] ** 2 + ky[None, :, None] ** 2 + kx[None, None, :] ** 2
    d = (sinc_pow(mz, nz, order)[:, None, None] * sinc_pow(my, ny, order)[None, :, None]
         * sinc_pow(mx, nx, order)[None, None, :])
    with np.errstate(divide="ignore", invalid="ignore"):
        g = 4.0 * np.pi * np.exp(-k2 / (4.0 * alpha * alpha)) / k2
        g = g / d ** 2
    g[0, 0, 0] = 0.0
    g[np.abs(d) < floor] = 0.0
    return g


def influence_optimal(dims, lengths, alpha, order, floor=DECONV_FLOOR, images=2):
    """Alias-summed influence function (kspace.py:162-196)."""
    nx, ny, nz = (int(d) for d in dims)
    lx, ly, lz = (float(v) for v in lengths)
    mx, my, mz = mode_numbers(nx), mode_numbers(ny), mode_numbers(nz)
    two_pi = 2.0 * np.pi
    kx = (two_pi * mx / lx)[None, None, :]
    ky = (two_pi * my / ly)[None, :, None]
    kz = (two_pi * mz / lz)[:, None, None]
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    num = np.zeros((nz, ny, nx))
    den = np.zeros((nz, ny, nx))
    rng = range(-images, images + 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        for bz in rng:
            wz = sinc_pow(mz + bz * nz, nz, order)[:, None, None]
            kzb = kz + two_pi * bz * nz / lz
            for by in rng:
                wy = sinc_pow(my + by * ny, ny, order)[None, :, None]
                kyb = ky + two_pi * by * ny / ly
                for bx in rng:
                    wx = sinc_pow(mx + bx * nx, nx, order)[None, None, :]
                    kxb = kx + two_pi * bx * nx / lx
                    w2 = (wx * wy * wz) ** 2
                    kb2 = kxb ** 2 + kyb ** 2 + kzb ** 2
                    gb = 4.0 * np.pi * np.exp(-kb2 / (4.0 * alpha * alpha)) / kb2
                    num += w2 * gb * (kx * kxb + ky * kyb + kz * kzb)
                    den += w2
        g = num / (k2 * den ** 2)
    g[0, 0, 0] = 0.0
    g[den < floor] = 0.0
    np.maximum(g, 0.0, out=g)
    return g


def ik_vectors(dims, lengths):
    """Reciprocal differentiation vectors with zeroed Nyquist (kspace.py:232-242)."""
    out = []
    for n, length in zip((int(d) for d in dims), (float(v) for v in lengths)):
        m = mode_numbers(n).copy()
        if n % 2 == 0:
            m[n // 2] = 0.0
        out.append(2.0 * np.pi * m / length)
    return out


def poisson_ik(rho, g, ik):
    """E_d = Re ifftn(-i k_d G fftn(rho)) (kspace.py:271-300).  Returns (ex, ey, ez)."""
    rho_hat = np.fft.fftn(rho)
    phi_hat = g * rho_hat
    out = []
    for vec, axis in zip(ik, (2, 1, 0)):
        shape = [1, 1, 1]
        shape[axis] = vec.size
        out.append(np.ascontiguousarray(np.fft.ifftn(-1j * vec.reshape(shape) * phi_hat).real))
    return tuple(out)


def poisson_ad(rho, g):
    """phi = Re ifftn(G fftn(rho)) (kspace.py:303-317)."""
    return np.ascontiguousarray(np.fft.ifftn(g * np.fft.fftn(rho)).real)


def kspace_energy(rho, g, lengths, coulomb_constant=1.0, dielectric=1.0):
    """C/eps * Vc^2/(2V) * sum G |rho_hat|^2 over the full spectrum (kspace.py:320-337)."""
    rho_hat = np.fft.fftn(rho)
    total = float(np.sum(g * (rho_hat.real ** 2 + rho_hat.imag ** 2)))
    vol = float(np.prod(np.asarray(lengths, dtype=np.float64)))
    vcell = vol / rho.size
    return coulomb_constant / dielectric * vcell ** 2 / (2.0 * vol) * total


# --------------------------------------------------------------------------
# fieldforce


def _row_sum(block):
    """Left-to-right reduction innermost axis first (gridmap.py:216-229)."""
    out = block
    for _ in range(3):
        acc = out[..., 0]
        for k in range(1, out.shape[-1]):
            acc = acc + out[..., k]
        out = acc
    return out


def _gather(grid, ix, iy, iz):
    return grid[iz[:, :, None, None], iy[:, None, :, None], ix[:, None, None, :]]


def fieldforce_ik(fields, pos, q, lengths, dims, order, table=None, force_scale=1.0,
                  *, chunk=1 << 15):
    """F_d = (C/eps) q sum_stencil wz wy wx E_d (gridmap.py:236-267).  Returns (N, 3)."""
    check_positions(pos, lengths, dims, order)
    pos = np.asarray(pos, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    n = pos.shape[0]
    out = np.empty((n, 3))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        nodes, arows, _ = stencil_weights(pos[s:e], lengths, dims, order, table)
        ix, iy, iz = stencil_indices(nodes, dims, order)
        wx, wy, wz = (r[:, :order] for r in arows)
        wgt = wz[:, :, None, None] * wy[:, None, :, None] * wx[:, None, None, :]
        sc = force_scale * q[s:e]
        for d in range(3):
            out[s:e, d] = sc * _row_sum(wgt * _gather(fields[d], ix, iy, iz))
    return out


def fieldforce_ad(phi, pos, q, lengths, dims, order, table=None, force_scale=1.0,
                  *, chunk=1 << 15):
    """Split-atom ad gather F_d = -(C/eps) q sum_d / h_d (gridmap.py:270-312)."""
    check_positions(pos, lengths, dims, order)
    pos = np.asarray(pos, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    h = spacing(lengths, dims)
    n = pos.shape[0]
    out = np.empty((n, 3))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        nodes, arows, drows = stencil_weights(pos[s:e], lengths, dims, order, table)
        ix, iy, iz = stencil_indices(nodes, dims, order)
        ax, ay, az = (r[:, :order] for r in arows)
        dx, dy, dz = (r[:, :order] for r in drows)
        p = _gather(phi, ix, iy, iz)
        sx = _row_sum(az[:, :, None, None] * ay[:, None, :, None] * dx[:, None, None, :] * p)
        sy = _row_sum(az[:, :, None, None] * dy[:, None, :, None] * ax[:, None, None, :] * p)
        sz = _row_sum(dz[:, :, None, None] * ay[:, None, :, None] * ax[:, None, None, :] * p)
        sc = force_scale * q[s:e]
        out[s:e, 0] = -sc * sx / h[0]
        out[s:e, 1] = -sc * sy / h[1]
        out[s:e, 2] = -sc * sz / h[2]
    return out


# --------------------------------------------------------------------------
# whole PPPM step and the parity metric


def pppm_step(pos, q, lengths, dims, order, alpha, mode="ik", table=None,
              coulomb_constant=1.0, dielectric=1.0, influence="pme"):
    """make_rho -> Poisson -> fieldforce, as driver.compute_forces does (driver.py:269-289).

    Returns (forces (N,3), kspace energy, rho).
    """
    rho = map_charge(pos, q, lengths, dims, order, table)
    if influence == "pme":
        g = influence_pme(dims, lengths, alpha, order)
    else:
        g = influence_optimal(dims, lengths, alpha, order)
    scale = coulomb_constant / dielectric
    energy = kspace_energy(rho, g, lengths, coulomb_constant, dielectric)
    if mode == "ik":
        fields = poisson_ik(rho, g, ik_vectors(dims, lengths))
        f = fieldforce_ik(fields, pos, q, lengths, dims, order, table, scale)
    else:
        phi = poisson_ad(rho, g)
        f = fieldforce_ad(phi, pos, q, lengths, dims, order, table, scale)
    return f, energy, rho


# ---------------------------------------------------------------------------
# either side of the mesh path: pair forces, full force
# evaluation, velocity-Verlet NVE.  Brute force over all pairs (small N only).

def minimum_image(d, lengths):
    """model.minimum_image (model.py:98-110)."""
    out = d - np.round(d / lengths) * lengths
    half = 0.5 * lengths
    out = np.where(out >= half, out - lengths, out)
    return np.where(out < -half, out + lengths, out)


def wrap(pos, lengths):
    """model.wrap (model.py:81-95)."""
    out = pos - np.floor(pos / lengths) * lengths
    out = np.where(out >= lengths, out - lengths, out)
    return np.where(out < 0.0, out + lengths, out)


def pair_forces(pos, q, lengths, alpha, cutoff, lj=None, coulomb_constant=1.0, dielectric=1.0):
    """shortrange.pair_forces (shortrange.py:201-267) over all i < j pairs.

    ``lj``: (epsilon, sigma, lj_cutoff) or None.  Returns (forces, energy,
    pairs within the cutoff).  Raises ValueError on overlapping atoms."""
    from math import erfc as _erfc

    pos = np.asarray(pos, dtype=np.float64)
    n = pos.shape[0]
    i, j = np.triu_indices(n, k=1)
    disp = minimum_image(pos[i] - pos[j], lengths)
    r2 = np.sum(disp * disp, axis=1)
    m = r2 < cutoff * cutoff
    i, j, disp, r2 = i[m], j[m], disp[m], r2[m]
    r = np.sqrt(r2)
    if r.size and float(r.min()) < 1e-10:
        raise ValueError("overlapping atoms")
    scale = coulomb_constant / dielectric
    qq = scale * q[i] * q[j]
    scr = np.array([_erfc(alpha * v) for v in r])
    e = qq * scr / r
    fm = qq * (scr / r2 + 2.0 / np.sqrt(np.pi) * alpha * np.exp(-alpha * alpha * r2) / r)
    if lj is not None:
        eps, sig, rc = lj
        lm = r < rc
        sr6 = (sig / r[lm]) ** 6
        e = e.copy()
        e[lm] += 4.0 * eps * (sr6 * sr6 - sr6)
        fa = np.zeros_like(fm)
        fa[lm] = 24.0 * eps * (2.0 * sr6 * sr6 - sr6) / r[lm]
        fm = fm + fa
    fv = (fm / r)[:, None] * disp
    f = np.zeros((n, 3))
    np.add.at(f, i, fv)
    np.add.at(f, j, -fv)
    return f, float(e.sum()), int(r.size)


def self_energy(q, alpha, coulomb_constant=1.0, dielectric=1.0):
    """shortrange.self_energy (shortrange.py:270-278)."""
    return -(coulomb_constant / dielectric) * alpha / np.sqrt(np.pi) * float(np.sum(np.asarray(q) ** 2))


def compute_forces(pos, q, lengths, dims, order, alpha, cutoff, mode="ik", table=None, lj=None,
                   coulomb_constant=1.0, dielectric=1.0):
    """driver.compute_forces (driver.py:232-307): pair + mesh + self.
    Returns (forces, (pair, kspace, self))."""
    fp, ep, _ = pair_forces(pos, q, lengths, alpha, cutoff, lj, coulomb_constant, dielectric)
    fm, ek, _ = pppm_step(pos, q, lengths, dims, order, alpha, mode, table, coulomb_constant, dielectric)
    return fp + fm, (ep, ek, self_energy(q, alpha, coulomb_constant, dielectric))


def integrate_nve(pos, vel, masses, q, lengths, dims, order, alpha, cutoff, dt, steps, mode="ik", table=None):
    """driver.integrate_nve (driver.py:310-376): velocity Verlet.
    Returns (series (steps+1, 7) [total, kinetic, potential, T, px, py, pz], pos, vel)."""
    pos = np.array(pos, dtype=np.float64)
    vel = np.array(vel, dtype=np.float64)
    m = np.asarray(masses, dtype=np.float64)[:, None]
    n = pos.shape[0]
    ser = np.empty((steps + 1, 7))
    f, e = compute_forces(pos, q, lengths, dims, order, alpha, cutoff, mode, table)
    for step in range(steps + 1):
        kin = 0.5 * float(np.sum(m * vel ** 2))
        pot = e[0] + e[1] + e[2]
        ser[step] = [kin + pot, kin, pot, float(np.sum(m * vel ** 2)) / (3.0 * n), *(m * vel).sum(axis=0)]
        if step == steps:
            break
        vel = vel + 0.5 * dt / m * f
        pos = wrap(pos + dt * vel, lengths)
        f, e = compute_forces(pos, q, lengths, dims, order, alpha, cutoff, mode, table)
        vel = vel + 0.5 * dt / m * f
    return ser, pos, vel


def rms_rel_error(f, f_ref):
    """Relative RMS force error (ewald.py:155-171)."""
    f = np.asarray(f, dtype=np.float64)
    f_ref = np.asarray(f_ref, dtype=np.float64)
    num = np.sqrt(np.sum((f - f_ref) ** 2) / f.shape[0])
    den = np.sqrt(np.sum(f_ref ** 2) / f.shape[0])
    return num / den if den > 0 else num
