"""z-slab decomposition of the PPPM mesh path over P GPUs.

The reference is single-process (its SPEC puts the distributed FFT out of
scope); this is new.  Slab r owns global mesh planes [r*nz/P, (r+1)*nz/P) and
the atoms whose wrapped node_z falls in them; after the forward transpose it
holds ky rows [r*ny/P, (r+1)*ny/P) of the half spectrum for every kz.  One step:

    make_rho (bin, spread, x/y halo fold)                      device
    ghost planes reverse-summed with slab r-1 / r+1            send/recv
    add_ghosts; 2D R2C of the local planes; pack by ky chunk   device
    transpose                                                  all-to-all
    z FFT, Green / ik multiply + energy partial, inverse z FFT device
    energy                                                     all-reduce
    transpose back                                             all-to-all
    unpack, 2D C2R into the padded fields, x/y halo fill       device
    boundary planes forward-copied into the neighbours' ghosts send/recv
    fieldforce                                                 device

The device halves are the ``pppm_slab_*`` C-ABI calls; the exchanges are
issued here over ``torch.distributed`` (NCCL with CUDA tensors that alias the
context's device buffers, ordered on the context's stream), or by
``LoopbackSlabs`` as device copies between P slab contexts on one GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from . import _runtime as rt

BUF = dict(RHO_GHOST_LO=0, RHO_GHOST_HI=1, RECV_LO=2, RECV_HI=3, A2A_SEND=4, A2A_RECV=5, A2A_SEND_F=6,
           A2A_RECV_F=7, ENERGY=8, FIELD_BOTTOM=9, FIELD_TOP=10, FIELD_GHOST_LO=11, FIELD_GHOST_HI=12)


def owner_of_nodes(nodes_z, nz, nslabs):
    """Slab owning each atom from its pre-wrap node_z (particle_map output)."""
    nodes_z = np.asarray(nodes_z, dtype=np.int64)
    return (nodes_z % nz) // (nz // nslabs)


def migrate_atoms(owner, arrays, group=None):
    """Atom migration between slabs (an all-to-all-v of atoms).

    ``owner`` (n,) int: the slab each of this rank's atoms belongs to after
    the move (``owner_of_nodes`` of the bit-exact node_z; SlabContext.owners
    computes it on the device).  ``arrays``: per-atom numpy arrays (positions,
    charges, velocities, global ids, ...), first axis n.  Every rank calls it
    (collective over ``group``).  Returns the rank's new arrays: the atoms it
    kept, in their order, followed by the atoms received from slab 0, 1, ...
    in the senders' order (deterministic).  Counts travel with all_gather,
    the payload with point-to-point sends / receives (NCCL on CUDA, gloo on
    CPU)."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    owner = np.asarray(owner, dtype=np.int64)
    if owner.size and (owner.min() < 0 or owner.max() >= world):
        raise ValueError("owner slab out of range")
    counts = np.bincount(owner, minlength=world).astype(np.int64)
    allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, torch.from_numpy(counts), group=group)
    recv_counts = [int(allc[src][rank]) for src in range(world)]
    out = []
    for a in arrays:
        a = np.ascontiguousarray(a)
        keep = a[owner == rank]
        flat = a.reshape(a.shape[0], -1)
        width = flat.shape[1]
        ops, recv_bufs = [], {}
        for dst in range(world):
            if dst != rank and counts[dst]:
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(flat[owner == dst])),
                                      dst, group))
        for src in range(world):
            if src != rank and recv_counts[src]:
                buf = torch.empty((recv_counts[src], width), dtype=torch.from_numpy(flat[:0]).dtype)
                recv_bufs[src] = buf
                ops.append(dist.P2POp(dist.irecv, buf, src, group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        parts = [keep.reshape(-1, *a.shape[1:])]
        parts += [recv_bufs[src].numpy().reshape(-1, *a.shape[1:]) for src in range(world) if src in recv_bufs]
        out.append(np.concatenate(parts) if parts else keep)
    return out


class _CudaView:
    """__cuda_array_interface__ over a raw device pointer (no ownership)."""

    def __init__(self, ptr, nbytes, typestr):
        item = int(typestr[-1])
        self.__cuda_array_interface__ = {
            "shape": (nbytes // item,), "typestr": typestr, "data": (int(ptr), False), "version": 3,
            "strides": None,
        }


def nccl_unique_id() -> bytes:
    """An NCCL unique id (128 bytes) for pppm_slab_attach_nccl; made on rank 0
    and broadcast by the caller."""
    buf = ctypes.create_string_buffer(128)
    nat.call("pppm_nccl_unique_id", buf)
    return buf.raw


class SlabContext:
    """One slab of the decomposed mesh on one device (mixed precision)."""

    def __init__(self, dims, lengths, order, mode, alpha, nslabs, rank, device=None, coulomb_constant=1.0,
                 dielectric=1.0, table_points=0, influence="pme"):
        device = rt.get_device() if device is None else int(device)
        nat.require_device(device)
        self.device, self.nslabs, self.rank = device, int(nslabs), int(rank)
        self.dims = tuple(int(d) for d in dims)
        self.mode = mode
        self.nfields = 3 if mode == "ik" else 1
        h = ctypes.c_void_p()
        nx, ny, nz = self.dims
        lx, ly, lz = (float(v) for v in lengths)
        nat.call("pppm_ctx_create_slab", ctypes.byref(h), device, nx, ny, nz, lx, ly, lz, int(order),
                 rt.mode_code(mode), nat.PREC_MIXED, float(alpha), float(coulomb_constant), float(dielectric),
                 self.nslabs, self.rank)
        self.handle = h
        self("pppm_ctx_build_influence", nat.INFLUENCE_PME if influence == "pme" else nat.INFLUENCE_OPTIMAL, 1e-10)
        self("pppm_ctx_build_table", int(table_points))
        info = (ctypes.c_int * 10)()
        self("pppm_slab_info", info)
        (self.P, self.rank, self.z0, self.nzl, self.y0, self.nyl, self.H, self.px, self.py, self.pz) = list(info)
        s = ctypes.c_void_p()
        self("pppm_ctx_stream", ctypes.byref(s))
        self.stream_ptr = s.value or 0
        self.n_atoms = 0

    def __call__(self, name, *args):
        nat.call(name, self.handle, *args)

    def buffer(self, name, field=0):
        """(device pointer, bytes) of one exchange buffer."""
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        self("pppm_slab_buffer", BUF[name], int(field), ctypes.byref(p), ctypes.byref(n))
        return p.value, n.value

    def view(self, name, field=0, typestr="<f4"):
        ptr, nbytes = self.buffer(name, field)
        return _CudaView(ptr, nbytes, typestr)

    def load_atoms(self, positions, charges):
        pos = np.ascontiguousarray(positions, dtype=np.float32)
        q = np.ascontiguousarray(charges, dtype=np.float32)
        self("pppm_ctx_load_atoms", nat.ptr(pos), nat.ptr(q), pos.shape[0], nat.F32)
        self.n_atoms = pos.shape[0]

    # device halves of the step
    def make_rho(self):
        self("pppm_slab_make_rho")

    def add_ghosts(self):
        self("pppm_slab_add_ghosts")

    def fft_fwd(self):
        self("pppm_slab_fft_fwd")

    def green(self):
        self("pppm_slab_green")

    def fft_bwd(self):
        self("pppm_slab_fft_bwd")

    def fieldforce(self):
        self("pppm_slab_fieldforce")

    def synchronize(self):
        self("pppm_ctx_synchronize")

    # the whole step inside the library (NCCL on the context stream, CUDA graphs)
    def attach_nccl(self, unique_id: bytes, timeout_s: float = 600.0):
        """Join the P-slab NCCL communicator (collective over the slabs)."""
        if len(unique_id) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        self("pppm_slab_attach_nccl", unique_id, float(timeout_s))

    def step(self, phases=nat.PHASE_ALL):
        self("pppm_ctx_step", int(phases))

    def time_steps(self, steps, warmup, flush_l2=True):
        """CUDA-event phase times in ms summed over ``steps`` (make_rho includes
        the ghost reverse sum, poisson the transposes and the energy all-reduce)."""
        ms = np.zeros(5)
        self("pppm_ctx_time_steps", int(steps), int(warmup), int(bool(flush_l2)), nat.ptr(ms))
        return dict(zip(("bin", "spread", "poisson", "gather", "total"), (float(v) for v in ms)))

    def launches_per_step(self):
        n = ctypes.c_int(0)
        self("pppm_ctx_launches_per_step", ctypes.byref(n))
        return n.value

    def owners(self, positions):
        """Owning slab of each position (bit-exact particle_map on the device)."""
        pos = np.ascontiguousarray(positions, dtype=np.float32)
        nodes = np.empty((3, pos.shape[0]), dtype=np.int32)
        self("pppm_particle_map", nat.ptr(pos), pos.shape[0], nat.F32, nat.HOST, nat.ptr(nodes))
        return owner_of_nodes(nodes[2], self.dims[2], self.P)

    def update_positions(self, positions):
        """New positions of this slab's atoms (its load order).  Raises when an
        atom left the slab: exchange them with ``migrate_atoms`` and reload."""
        pos = np.ascontiguousarray(positions, dtype=np.float32)
        self("pppm_ctx_update_positions", nat.ptr(pos), nat.F32, nat.HOST)

    def forces(self):
        out = np.empty((self.n_atoms, 3))
        self("pppm_ctx_get_forces", nat.ptr(out))
        return out

    def energy(self):
        e = np.zeros(1)
        self("pppm_ctx_get_energy", e.ctypes.data_as(nat._dp))
        return float(e[0])

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            nat.load().pppm_ctx_destroy(self.handle)
            self.handle = None


class SlabStep:
    """The exchange schedule of one step over a ``comm`` (see module doc).

    ``comm`` provides sendrecv(pairs), all_to_all(recv, send), all_reduce(t)
    on tensors obtained from ``comm.tensor(slab, name, field)``, and
    ``comm.stream()`` (a context manager ordering the exchanges after the
    slab's kernels).  The same schedule runs over NCCL, gloo (tests) or the
    single-GPU loopback.
    """

    def __init__(self, slab, comm):
        self.slab, self.comm = slab, comm
        r, P = slab.rank, slab.P
        self.prev, self.next = (r - 1) % P, (r + 1) % P
        t = lambda n, f=0: comm.tensor(slab, n, f)  # noqa: E731
        self.rho_lo, self.rho_hi = t("RHO_GHOST_LO"), t("RHO_GHOST_HI")
        self.recv_lo, self.recv_hi = t("RECV_LO"), t("RECV_HI")
        self.send, self.recv = t("A2A_SEND"), t("A2A_RECV")
        self.send_f, self.recv_f = t("A2A_SEND_F"), t("A2A_RECV_F")
        self.energy = comm.tensor(slab, "ENERGY", 0, typestr="<f8")
        nf = slab.nfields
        self.f_bottom = [t("FIELD_BOTTOM", f) for f in range(nf)]
        self.f_top = [t("FIELD_TOP", f) for f in range(nf)]
        self.f_glo = [t("FIELD_GHOST_LO", f) for f in range(nf)]
        self.f_ghi = [t("FIELD_GHOST_HI", f) for f in range(nf)]

    def ghost_reverse_sum(self):
        # my lower ghosts belong to the slab below (its top planes: its RECV_HI), upper to the slab above
        self.comm.sendrecv(sends=[(self.rho_lo, self.prev), (self.rho_hi, self.next)],
                           recvs=[(self.recv_hi, self.next), (self.recv_lo, self.prev)])

    def ghost_forward_copy(self):
        sends, recvs = [], []
        for f in range(len(self.f_top)):
            sends += [(self.f_top[f], self.next), (self.f_bottom[f], self.prev)]
            recvs += [(self.f_glo[f], self.prev), (self.f_ghi[f], self.next)]
        self.comm.sendrecv(sends=sends, recvs=recvs)

    def make_rho(self):
        self.slab.make_rho()
        with self.comm.stream(self.slab):
            self.ghost_reverse_sum()
        self.slab.add_ghosts()

    def poisson(self):
        s = self.slab
        s.fft_fwd()
        with self.comm.stream(s):
            self.comm.all_to_all(self.recv, self.send)
        s.green()
        with self.comm.stream(s):
            self.comm.all_reduce(self.energy)
            self.comm.all_to_all(self.recv_f, self.send_f)
        s.fft_bwd()
        with self.comm.stream(s):
            self.ghost_forward_copy()

    def fieldforce(self):
        self.slab.fieldforce()

    def __call__(self):
        self.make_rho()
        self.poisson()
        self.fieldforce()


class TorchComm:
    """Exchanges over a torch.distributed process group (NCCL on CUDA tensors
    aliasing the slab buffers, issued on the slab's stream; gloo on CPU tensors
    in the CPU tests)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group

    def tensor(self, slab, name, field=0, typestr="<f4"):
        if hasattr(slab, "host_buffer"):  # CPU test double
            return self.torch.from_numpy(slab.host_buffer(name, field))
        dtype = self.torch.float64 if typestr == "<f8" else self.torch.float32
        return self.torch.as_tensor(slab.view(name, field, typestr), device=f"cuda:{slab.device}").view(dtype)

    def stream(self, slab):
        import contextlib

        if not getattr(slab, "stream_ptr", 0):
            return contextlib.nullcontext()
        return self.torch.cuda.stream(self.torch.cuda.ExternalStream(slab.stream_ptr, device=slab.device))

    def sendrecv(self, sends, recvs):
        ops = [self.dist.P2POp(self.dist.isend, t, peer, self.group) for t, peer in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group) for t, peer in recvs]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()

    def all_to_all(self, recv, send):
        self.dist.all_to_all_single(recv, send, group=self.group)

    def all_reduce(self, t):
        self.dist.all_reduce(t, group=self.group)


class LoopbackSlabs:
    """P slab contexts on ONE device, exchanging by device copies: the
    single-GPU check of the decomposed algorithm (NCCL cannot put two ranks on
    one GPU).  Not a performance path."""

    def __init__(self, dims, lengths, order, mode, alpha, nslabs, **kw):
        import torch

        self.torch = torch
        self.slabs = [SlabContext(dims, lengths, order, mode, alpha, nslabs, r, **kw) for r in range(nslabs)]
        self.P = nslabs
        self._lengths = np.asarray(lengths, dtype=np.float64)
        self._order = int(order)

    def _t(self, slab, name, field=0, typestr="<f4"):
        dtype = self.torch.float64 if typestr == "<f8" else self.torch.float32
        return self.torch.as_tensor(slab.view(name, field, typestr), device=f"cuda:{slab.device}").view(dtype)

    def _sync(self):
        for s in self.slabs:
            s.synchronize()
        self.torch.cuda.synchronize()

    def load_atoms(self, positions, charges):
        """Partition atoms by owning slab (bit-exact particle_map on the device)."""
        import paper_1702_04250_b200 as pb

        pos32 = np.ascontiguousarray(positions, dtype=np.float32)
        ctx = pb.PppmContext(self.slabs[0].dims, self._lengths, order=self._order, precision="mixed",
                             alpha=1.0, mode="ad")
        nodes = np.empty((3, pos32.shape[0]), dtype=np.int32)
        ctx.ctx("pppm_particle_map", nat.ptr(pos32), pos32.shape[0], nat.F32, nat.HOST, nat.ptr(nodes))
        ctx.close()
        owner = owner_of_nodes(nodes[2], self.slabs[0].dims[2], self.P)
        self.index = []
        for r, s in enumerate(self.slabs):
            sel = np.nonzero(owner == r)[0]
            self.index.append(sel)
            s.load_atoms(pos32[sel], np.asarray(charges)[sel])

    def step(self):
        P, S = self.P, self.slabs
        for s in S:
            s.make_rho()
        self._sync()
        for r, s in enumerate(S):
            self._t(S[(r - 1) % P], "RECV_HI").copy_(self._t(s, "RHO_GHOST_LO"))
            self._t(S[(r + 1) % P], "RECV_LO").copy_(self._t(s, "RHO_GHOST_HI"))
        self._sync()
        for s in S:
            s.add_ghosts()
            s.fft_fwd()
        self._sync()
        self._a2a("A2A_SEND", "A2A_RECV")
        for s in S:
            s.green()
        self._sync()
        total = sum(float(self._t(s, "ENERGY", 0, "<f8")[0]) for s in S)
        for s in S:
            self._t(s, "ENERGY", 0, "<f8")[0] = total
        self._a2a("A2A_SEND_F", "A2A_RECV_F")
        for s in S:
            s.fft_bwd()
        self._sync()
        for r, s in enumerate(S):
            for f in range(s.nfields):
                self._t(S[(r + 1) % P], "FIELD_GHOST_LO", f).copy_(self._t(s, "FIELD_TOP", f))
                self._t(S[(r - 1) % P], "FIELD_GHOST_HI", f).copy_(self._t(s, "FIELD_BOTTOM", f))
        self._sync()
        for s in S:
            s.fieldforce()
        self._sync()

    def _a2a(self, send_name, recv_name):
        P = self.P
        sends = [self._t(s, send_name) for s in self.slabs]
        recvs = [self._t(s, recv_name) for s in self.slabs]
        chunk = sends[0].numel() // P
        for r in range(P):
            for c in range(P):
                recvs[c][r * chunk:(r + 1) * chunk].copy_(sends[r][c * chunk:(c + 1) * chunk])
        self._sync()

    def forces(self, n_atoms):
        out = np.empty((n_atoms, 3))
        for sel, s in zip(self.index, self.slabs):
            out[sel] = s.forces()
        return out

    def energy(self):
        return self.slabs[0].energy()

    def close(self):
        for s in self.slabs:
            s.close()
