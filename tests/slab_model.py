"""numpy model of one z-slab's device steps (test infrastructure only).

It mirrors the buffer layout and the semantics of the ``pppm_slab_*`` C-ABI
calls (padded slab mesh with ghost planes, ky-chunk transposes, packing order
of the all-to-all buffers) in fp64, so the exchange schedule of
``paper_1702_04250_b200.slab.SlabStep`` can run over gloo on CPU (world size 2)
and be checked against the CPU oracle without a GPU.
"""

import numpy as np

from oracle import pppm_oracle as orc


class NumpySlab:
    def __init__(self, dims, lengths, order, mode, alpha, nslabs, rank):
        self.dims = tuple(int(d) for d in dims)
        self.lengths = np.asarray(lengths, dtype=np.float64)
        self.order, self.mode, self.alpha = int(order), mode, float(alpha)
        self.P, self.rank = int(nslabs), int(rank)
        self.nfields = 3 if mode == "ik" else 1
        nx, ny, nz = self.dims
        self.nzl, self.nyl = nz // self.P, ny // self.P
        self.z0, self.y0 = rank * self.nzl, rank * self.nyl
        self.lo = (order - 1) // 2
        hi = order - 1 - self.lo
        self.H = max(self.lo, hi)
        H = self.H
        self.pz, self.py, self.px = self.nzl + 2 * H, ny + 2 * H, nx + 2 * H
        self.nxh = nx // 2 + 1
        self.rho = np.zeros((self.pz, self.py, self.px))
        self.fields = np.zeros((self.nfields, self.pz, self.py, self.px))
        self.recv_lo = np.zeros((H, self.py, self.px))
        self.recv_hi = np.zeros((H, self.py, self.px))
        half = nz * self.nyl * self.nxh
        self.send = np.zeros(2 * half)
        self.recv = np.zeros(2 * half)
        self.send_f = np.zeros(2 * half * self.nfields)
        self.recv_f = np.zeros(2 * half * self.nfields)
        self.energy_buf = np.zeros(1)
        g = orc.influence_pme(self.dims, self.lengths, self.alpha, order)
        self.green_chunk = g[:, self.y0:self.y0 + self.nyl, :self.nxh]
        ik = orc.ik_vectors(self.dims, self.lengths)
        self.ikx, self.iky, self.ikz = ik[0][:self.nxh], ik[1][self.y0:self.y0 + self.nyl], ik[2]
        self.pos = np.zeros((0, 3))
        self.q = np.zeros(0)

    def host_buffer(self, name, field=0):
        H, nzl = self.H, self.nzl
        views = {
            "RHO_GHOST_LO": self.rho[:H], "RHO_GHOST_HI": self.rho[H + nzl:],
            "RECV_LO": self.recv_lo, "RECV_HI": self.recv_hi,
            "A2A_SEND": self.send, "A2A_RECV": self.recv, "A2A_SEND_F": self.send_f, "A2A_RECV_F": self.recv_f,
            "ENERGY": self.energy_buf,
            "FIELD_BOTTOM": self.fields[field, H:2 * H], "FIELD_TOP": self.fields[field, nzl:nzl + H],
            "FIELD_GHOST_LO": self.fields[field, :H], "FIELD_GHOST_HI": self.fields[field, H + nzl:],
        }
        v = views[name].reshape(-1)
        assert np.shares_memory(v, views[name]) or v.size == 0
        return v

    def load_atoms(self, pos, q):
        self.pos = np.asarray(pos, dtype=np.float64)
        self.q = np.asarray(q, dtype=np.float64)

    def _stencil(self):
        nodes, arows, drows = orc.stencil_weights(self.pos, self.lengths, self.dims, self.order)
        nx, ny, nz = self.dims
        n0, n1, n2 = nodes[0] % nx, nodes[1] % ny, nodes[2] % nz - self.z0
        assert np.all((n2 >= 0) & (n2 < self.nzl))
        S, H = self.order, self.H
        ix = n0[:, None] - self.lo + np.arange(S)[None, :] + H
        iy = n1[:, None] - self.lo + np.arange(S)[None, :] + H
        iz = n2[:, None] - self.lo + np.arange(S)[None, :] + H
        return ix, iy, iz, [r[:, :S] for r in arows], [r[:, :S] for r in drows]

    def _fold_xy(self, a):
        H = self.H
        nx, ny = self.dims[0], self.dims[1]
        a[..., :, H:2 * H] += a[..., :, nx + H:nx + 2 * H]
        a[..., :, nx:nx + H] += a[..., :, :H]
        a[..., :, :H] = 0
        a[..., :, nx + H:] = 0
        a[..., H:2 * H, :] += a[..., ny + H:ny + 2 * H, :]
        a[..., ny:ny + H, :] += a[..., :H, :]
        a[..., :H, :] = 0
        a[..., ny + H:, :] = 0

    def _fill_xy(self, a):
        H = self.H
        nx, ny = self.dims[0], self.dims[1]
        a[..., :, :H] = a[..., :, nx:nx + H]
        a[..., :, nx + H:] = a[..., :, H:2 * H]
        a[..., :H, :] = a[..., ny:ny + H, :]
        a[..., ny + H:, :] = a[..., H:2 * H, :]

    def make_rho(self):
        self.rho[...] = 0
        ix, iy, iz, (wx, wy, wz), _ = self._stencil()
        c = self.q[:, None, None, None] * wz[:, :, None, None] * wy[:, None, :, None] * wx[:, None, None, :]
        np.add.at(self.rho, (iz[:, :, None, None], iy[:, None, :, None], ix[:, None, None, :]), c)
        h = self.lengths / np.array(self.dims)
        self.rho /= h[0] * h[1] * h[2]
        self._fold_xy(self.rho)

    def add_ghosts(self):
        H, nzl = self.H, self.nzl
        self.rho[H:2 * H] += self.recv_lo
        self.rho[nzl:nzl + H] += self.recv_hi

    def fft_fwd(self):
        H, nzl = self.H, self.nzl
        nx, ny = self.dims[0], self.dims[1]
        spec = np.fft.rfft2(self.rho[H:H + nzl, H:H + ny, H:H + nx], axes=(1, 2))  # (nzl, ny, nxh)
        packed = spec.reshape(nzl, self.P, self.nyl, self.nxh).transpose(1, 0, 2, 3)  # [c][zl][kyl][kx]
        self.send[:] = np.ascontiguousarray(packed).view(np.float64).reshape(-1)

    def green(self):
        nz = self.dims[2]
        spec = self.recv.view(np.complex128).reshape(nz, self.nyl, self.nxh)
        spec = np.fft.fft(spec, axis=0)
        g = self.green_chunk
        nx = self.dims[0]
        w = np.full(self.nxh, 2.0)
        w[0] = 1.0
        if nx % 2 == 0:
            w[nx // 2] = 1.0
        vol = float(np.prod(self.lengths))
        vcell = vol / np.prod(self.dims)
        self.energy_buf[0] = vcell * vcell / (2.0 * vol) * float(np.sum(w[None, None, :] * g * np.abs(spec) ** 2))
        phi = g * spec
        if self.mode == "ik":
            ew = [-1j * self.ikx[None, None, :] * phi, -1j * self.iky[None, :, None] * phi,
                  -1j * self.ikz[:, None, None] * phi]
        else:
            ew = [phi]
        ew = np.stack([np.fft.ifft(e, axis=0) for e in ew])  # (nf, nz, nyl, nxh)
        nf = self.nfields
        packed = ew.reshape(nf, self.P, self.nzl, self.nyl, self.nxh).transpose(1, 0, 2, 3, 4)  # [s][f][zl]..
        self.send_f[:] = np.ascontiguousarray(packed).view(np.float64).reshape(-1)

    def fft_bwd(self):
        nf, H, nzl = self.nfields, self.H, self.nzl
        nx, ny = self.dims[0], self.dims[1]
        rec = self.recv_f.view(np.complex128).reshape(self.P, nf, nzl, self.nyl, self.nxh)
        spec = rec.transpose(1, 2, 0, 3, 4).reshape(nf, nzl, ny, self.nxh)
        real = np.fft.irfft2(spec, s=(ny, nx), axes=(2, 3))
        self.fields[:, H:H + nzl, H:H + ny, H:H + nx] = real
        self._fill_xy(self.fields)

    def fieldforce(self):
        ix, iy, iz, (ax, ay, az), (dx, dy, dz) = self._stencil()

        def gather(f):
            return self.fields[f][iz[:, :, None, None], iy[:, None, :, None], ix[:, None, None, :]]

        if self.mode == "ik":
            wgt = az[:, :, None, None] * ay[:, None, :, None] * ax[:, None, None, :]
            self.forces = np.stack([self.q * np.sum(wgt * gather(f), axis=(1, 2, 3)) for f in range(3)], axis=1)
        else:
            p = gather(0)
            h = self.lengths / np.array(self.dims)
            sx = np.sum(az[:, :, None, None] * ay[:, None, :, None] * dx[:, None, None, :] * p, axis=(1, 2, 3))
            sy = np.sum(az[:, :, None, None] * dy[:, None, :, None] * ax[:, None, None, :] * p, axis=(1, 2, 3))
            sz = np.sum(dz[:, :, None, None] * ay[:, None, :, None] * ax[:, None, None, :] * p, axis=(1, 2, 3))
            self.forces = np.stack([-self.q * sx / h[0], -self.q * sy / h[1], -self.q * sz / h[2]], axis=1)
