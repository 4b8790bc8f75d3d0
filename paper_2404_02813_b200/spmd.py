"""z-slab SPMD drivers over the librsfg slab primitives.

The volume is cut into contiguous z-slabs; every slab keeps h = max(R1, R2, 2)
halo planes of phi on each interior face and exchanges them once per step,
between ``step_interior`` (the xy passes of the owned planes, which need no
halo) and ``step_finish`` (xy passes of the halo planes, z pass, stencil,
update).  Every voxel runs the same arithmetic on the same inputs as the
monolithic volume, so any decomposition is bitwise identical to one GPU.

* ``plan_slabs``   -- the partition (shared by every backend and the CPU tests).
* ``SlabSet``      -- one process driving P slabs on one or more local GPUs;
                      halos pushed over peer links (rsfg_slab_link, default)
                      or exchanged between the step halves (rsfg_slab_exchange).
* ``DistSlab``     -- one slab per rank; halos pushed over CUDA-IPC peer links
                      (transport="ipc"), NCCL send/recv ("device") or
                      host-staged gloo ("host").
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import BlowupError, RsfParams, check, gaussian_kernel, options


def blowup_message(first_bad: int, nx: int, ny: int, iteration: int) -> str:
    """rsf::blowup_error text (rsf.cpp:346-352) for a global voxel index."""
    x, y, z = first_bad % nx, (first_bad // nx) % ny, first_bad // (nx * ny)
    return f"evolution produced a non-finite value at voxel ({x},{y},{z}), iteration {iteration}"


def halo_width(p: RsfParams) -> int:
    r1 = (len(gaussian_kernel(p.sigma1)) - 1) // 2
    r2 = (len(gaussian_kernel(p.sigma2)) - 1) // 2
    return max(r1, r2, 2)


def plan_slabs(nz: int, parts: int, halo: int) -> list[tuple[int, int]]:
    """Balanced contiguous z ranges; every slab must be >= halo planes thick."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(nz, parts)
    out, z = [], 0
    for r in range(parts):
        n = base + (1 if r < extra else 0)
        out.append((z, z + n))
        z += n
    if parts > 1 and min(b - a for a, b in out) < halo:
        raise ValueError(f"nz={nz} over {parts} slabs leaves a slab thinner than the halo ({halo})")
    return out


class Slab:
    """Thin owner of one rsfg_slab handle."""

    def __init__(self, nx, ny, nz, z0, z1, p: RsfParams, *, fields=2, device=0):
        self.lib = L.load()
        self.h = C.c_void_p()
        self.nx, self.ny, self.nz, self.z0, self.z1 = nx, ny, nz, z0, z1
        cp = p.to_c()
        opt = options(fields, device)
        check(self.lib.rsfg_slab_create(C.byref(self.h), nx, ny, nz, z0, z1, C.byref(cp), C.byref(opt)))
        zb, ze, halo = C.c_int32(), C.c_int32(), C.c_int32()
        check(self.lib.rsfg_slab_geometry(self.h, C.byref(zb), C.byref(ze), C.byref(halo)))
        self.zb, self.ze, self.halo = zb.value, ze.value, halo.value

    def upload(self, phi_vol, img_vol):
        """Takes the FULL volumes (numpy host arrays, or torch CUDA tensors on
        the slab's device) and uploads the held planes [zb, ze)."""
        if hasattr(phi_vol, "data_ptr"):  # torch CUDA tensors: device-to-device
            import torch
            ph = phi_vol[self.zb:self.ze].contiguous()
            im = img_vol[self.zb:self.ze].contiguous()
            # the slab copies on its own non-blocking stream: the producers of
            # these tensors (torch's stream) must be done first
            torch.cuda.synchronize(ph.device)
            check(self.lib.rsfg_slab_upload_device(self.h, ph.data_ptr(), im.data_ptr()))
            return
        ph = np.ascontiguousarray(phi_vol[self.zb:self.ze], np.float32)
        im = np.ascontiguousarray(img_vol[self.zb:self.ze], np.float32)
        check(self.lib.rsfg_slab_upload(self.h, ph.ctypes.data, im.ctypes.data))

    def local_range(self):
        lo, hi = C.c_float(), C.c_float()
        check(self.lib.rsfg_slab_local_range(self.h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def init(self, lo, hi):
        check(self.lib.rsfg_slab_init(self.h, lo, hi))

    def halo_views(self, side):
        s, r, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(self.lib.rsfg_slab_halo(self.h, side, C.byref(s), C.byref(r), C.byref(n)))
        return s.value, r.value, n.value

    def set_stream(self, stream: int):
        check(self.lib.rsfg_slab_set_stream(self.h, C.c_void_p(stream)))

    def step_interior(self):
        check(self.lib.rsfg_slab_step_interior(self.h))

    def step_finish(self):
        check(self.lib.rsfg_slab_step_finish(self.h))

    def peer_desc(self, ipc: bool) -> bytes:
        """This slab's link descriptor (rsfg_slab_peer_desc): raw device
        pointers (ipc=False, same process) or CUDA IPC handles (ipc=True)."""
        buf = C.create_string_buffer(L.RSFG_PEER_DESC_BYTES)
        check(self.lib.rsfg_slab_peer_desc(self.h, buf, 1 if ipc else 0))
        return buf.raw

    def link(self, side: int, desc: bytes):
        buf = C.create_string_buffer(desc, L.RSFG_PEER_DESC_BYTES)
        check(self.lib.rsfg_slab_link(self.h, side, buf))

    def step_linked(self):
        check(self.lib.rsfg_slab_step_linked(self.h))

    def counters(self):
        sc, bad = C.c_int64(), C.c_int64()
        check(self.lib.rsfg_slab_counters(self.h, C.byref(sc), C.byref(bad)))
        return sc.value, bad.value

    def download(self) -> np.ndarray:
        out = np.empty((self.z1 - self.z0, self.ny, self.nx), np.float32)
        check(self.lib.rsfg_slab_download(self.h, out.ctypes.data))
        return out

    def launches(self) -> int:
        return int(self.lib.rsfg_slab_launches(self.h))

    def close(self):
        if self.h:
            self.lib.rsfg_slab_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SlabSet:
    """P slabs in one process (one or several local GPUs).

    linked=True (default): peer halo links (rsfg_slab_link) -- each slab
    pushes its boundary planes into its neighbours' halos after its step and
    bumps their flags; no host sync, the copies overlap the next step's
    interior work.  linked=False: halos move with rsfg_slab_exchange between
    the interior and finish halves of every step."""

    def __init__(self, phi0, I, p: RsfParams, parts: int, *, fields=2, devices=None, check_every=25,
                 linked=True):
        nz, ny, nx = phi0.shape
        self.nx, self.ny = nx, ny
        self.check_every = max(1, check_every)
        self.iteration = 0
        self.halo = halo_width(p)
        self.ranges = plan_slabs(nz, parts, self.halo)
        devices = devices or [0] * parts
        self.slabs = [Slab(nx, ny, nz, a, b, p, fields=fields, device=devices[i % len(devices)])
                      for i, (a, b) in enumerate(self.ranges)]
        for s in self.slabs:
            s.upload(phi0, I)
        los, his = zip(*(s.local_range() for s in self.slabs))
        lo, hi = min(los), max(his)  # global [min I, max I] (volume.cpp:25-33)
        for s in self.slabs:
            s.init(lo, hi)
        self.linked = linked
        if linked:
            for a, b in zip(self.slabs, self.slabs[1:]):
                a.link(1, b.peer_desc(False))
                b.link(0, a.peer_desc(False))

    def step(self):
        lib = L.load()
        if self.linked:
            for s in self.slabs:
                s.step_linked()
            self.iteration += 1
            if self.iteration % self.check_every == 0:
                self.check_blowup()
            return
        for s in self.slabs:
            s.step_interior()
        for a, b in zip(self.slabs, self.slabs[1:]):
            check(lib.rsfg_slab_exchange(a.h, b.h))
        for s in self.slabs:
            s.step_finish()
        self.iteration += 1
        if self.iteration % self.check_every == 0:
            self.check_blowup()

    def check_blowup(self):
        """Raises BlowupError (rsf.cpp:346-352) if the LAST step produced a
        non-finite phi anywhere (smallest global voxel index).  A non-finite
        value spreads to every later step, so checking every check_every steps
        finds it; the reported iteration is the one checked."""
        bads = [b for b in (s.counters()[1] for s in self.slabs) if b >= 0]
        if bads:
            raise BlowupError(blowup_message(min(bads), self.nx, self.ny, self.iteration))

    def sign_changes(self) -> int:
        return sum(s.counters()[0] for s in self.slabs)

    def phi(self) -> np.ndarray:
        return np.concatenate([s.download() for s in self.slabs])

    def close(self):
        for s in self.slabs:
            s.close()


def start_halo_exchange(dist, rank, world, lo_views, hi_views):
    """Post the per-step halo sends/receives of one rank.

    lo_views / hi_views = (send, recv) tensors for the face toward z=0 / z=nz-1
    (None on a global face).  Shared by the NCCL driver and the gloo CPU tests
    so both exercise the same pairing.  Returns the requests to wait on."""
    ops = []
    if rank > 0 and lo_views[0] is not None:
        ops += [dist.P2POp(dist.isend, lo_views[0], rank - 1), dist.P2POp(dist.irecv, lo_views[1], rank - 1)]
    if rank < world - 1 and hi_views[0] is not None:
        ops += [dist.P2POp(dist.isend, hi_views[0], rank + 1), dist.P2POp(dist.irecv, hi_views[1], rank + 1)]
    return dist.batch_isend_irecv(ops) if ops else []


def held_range(z0, z1, nz, halo):
    """Planes a slab holds: [max(z0-h, 0), min(z1+h, nz)) (rsfg_slab_create)."""
    return max(z0 - halo, 0), min(z1 + halo, nz)


class _DevView:
    """__cuda_array_interface__ view of raw device memory (zero copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class DistSlab:
    """One slab per rank (torchrun, one process per GPU).

    transport="ipc" (default) is the B200-native data path: peer halo links over CUDA IPC
    (rsfg_slab_link) -- each rank copies its boundary planes straight into its
    neighbours' halo rows over NVLink and bumps their flag words; the process
    group only carries the one-time descriptor exchange and the scalar
    reductions.  It also runs with several ranks on one GPU (IPC between
    processes on the same device), which is how it is tested here.
    transport="device" posts NCCL send/recv on views of the slab's own
    device buffers, overlapped with the interior work.  transport="host" stages
    the halo planes through host memory for CPU-only process groups (gloo): it
    lets several ranks share one GPU, which is how this path is tested on
    single-GPU machines (tests/test_gpu_distslab.py)."""

    def __init__(self, phi0, I, p: RsfParams, *, fields=2, rank=None, world=None, device=None, transport="ipc",
                 check_every=25):
        import torch
        self.check_every = max(1, check_every)
        self.iteration = 0
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        nz, ny, nx = phi0.shape
        self.nx, self.ny = nx, ny
        self.halo = halo_width(p)
        self.ranges = plan_slabs(nz, self.world, self.halo)
        z0, z1 = self.ranges[self.rank]
        dev = torch.cuda.current_device() if device is None else device
        self.slab = Slab(nx, ny, nz, z0, z1, p, fields=fields, device=dev)
        self.slab.upload(phi0, I)
        self.stream = torch.cuda.current_stream()
        self.slab.set_stream(self.stream.cuda_stream)
        self.transport = transport
        self.red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        lo, hi = self.slab.local_range()
        t = torch.tensor([-lo, hi], dtype=torch.float32, device=self.red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        self.slab.init(-float(t[0]), float(t[1]))
        if transport == "ipc":
            descs = [None] * self.world
            dist.all_gather_object(descs, self.slab.peer_desc(True))
            if self.rank > 0:
                self.slab.link(0, descs[self.rank - 1])
            if self.rank < self.world - 1:
                self.slab.link(1, descs[self.rank + 1])
            torch.cuda.synchronize(dev)
            dist.barrier()

    def _views(self, side):
        send, recv, n = self.slab.halo_views(side)
        if n == 0:
            return None, None
        t = self.torch
        return t.as_tensor(_DevView(send, n), device="cuda"), t.as_tensor(_DevView(recv, n), device="cuda")

    def step(self):
        if self.transport == "ipc":
            self.slab.step_linked()
        elif self.transport == "host":
            self._step_host()
        else:
            reqs = start_halo_exchange(self.dist, self.rank, self.world, self._views(0), self._views(1))
            self.slab.step_interior()  # overlaps the exchange (no halo needed)
            for q in reqs:
                q.wait()
            self.slab.step_finish()
        self.iteration += 1
        if self.iteration % self.check_every == 0:
            self.check_blowup()

    def check_blowup(self):
        """Global first non-finite voxel of the last step (MIN over ranks of each
        slab's first bad index, rsf.cpp:346-352); raises BlowupError on every rank."""
        t = self.torch
        _, bad = self.slab.counters()
        big = t.iinfo(t.int64).max
        v = t.tensor([bad if bad >= 0 else big], dtype=t.int64, device=self.red_dev)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN)
        g = int(v.item())
        if g != big:
            raise BlowupError(blowup_message(g, self.nx, self.ny, self.iteration))

    def _step_host(self):
        self.stream.synchronize()  # the previous step's phi is complete
        views = [self._views(0), self._views(1)]
        staged = [(v[0].cpu(), self.torch.empty(v[1].shape, dtype=v[1].dtype)) if v[0] is not None else (None, None)
                  for v in views]
        reqs = start_halo_exchange(self.dist, self.rank, self.world, staged[0], staged[1])
        self.slab.step_interior()
        for q in reqs:
            q.wait()
        for v, st in zip(views, staged):
            if v[1] is not None:
                v[1].copy_(st[1])
        self.slab.step_finish()

    def phi_owned(self) -> np.ndarray:
        return self.slab.download()
