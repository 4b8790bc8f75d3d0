"""Python mirror of the reference RSF API over the CUDA C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/rsf/rsf.hpp:13-101):

    RsfParams, evolve(phi0, I, p, stop=None, stop_every=25),
    init_evolution(phi0, I, p) -> EvolutionState, evolve_step(state),
    energy(state), extract_mask(phi)

with exceptions ParamError / ShapeError / BlowupError standing in for
rsf::param_error / shape_error / blowup_error.  Volumes are numpy float32
arrays shaped (nz, ny, nx) -- the reference's x-fastest layout
(volume.hpp:35-40).  Everything runs in librsfg.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields as dc_fields

import numpy as np

from . import _lib as L


class RsfError(RuntimeError):
    pass


class ParamError(RsfError, ValueError):
    """rsf::param_error (core.hpp:11-14)."""


class ShapeError(RsfError, ValueError):
    """rsf::shape_error (core.hpp:16-20)."""


class BlowupError(RsfError):
    """rsf::blowup_error (core.hpp:28-32)."""


class CudaError(RsfError):
    pass


class VolumeIOError(OSError):
    """rsf::io_error (volume_io.cpp:24-137)."""


_ERRORS = {L.RSFG_ERR_PARAM: ParamError, L.RSFG_ERR_SHAPE: ShapeError, L.RSFG_ERR_BLOWUP: BlowupError,
           L.RSFG_ERR_IO: VolumeIOError}


def check(rc: int) -> None:
    if rc != L.RSFG_OK:
        raise _ERRORS.get(rc, CudaError)(f"[rsfg {rc}] {L.last_error()}")


@dataclass
class RsfParams:
    """rsf::RsfParams (rsf.hpp:13-26), same defaults."""

    sigma1: float = 5.0
    sigma2: float = 0.0
    alpha: float = 58.5225
    beta: float = 0.1
    epsilon: float = 1.0
    dt: float = 0.06
    max_iters: int = 100
    convergence_fraction: float = 0.0
    denom_floor: float = 1e-8
    grad_floor: float = 1e-8

    def to_c(self) -> L.rsfg_params:
        return L.rsfg_params(**{f.name: getattr(self, f.name) for f in dc_fields(self)})

    def validate(self) -> None:
        p = self.to_c()
        check(L.load().rsfg_params_validate(C.byref(p)))


def options(fields: int = 2, device: int = 0, check_every: int = 25) -> L.rsfg_options:
    o = L.rsfg_options()
    L.load().rsfg_options_default(C.byref(o))
    o.fields, o.device, o.check_every = fields, device, check_every
    return o


def _vol(a, name="volume") -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ShapeError(f"{name}: expected (nz, ny, nx) array, got shape {a.shape}")
    return a


def _check_same(a, b, what):
    if a.shape != b.shape:
        sa = "x".join(map(str, a.shape[::-1]))
        sb = "x".join(map(str, b.shape[::-1]))
        raise ShapeError(f"{what}: dims mismatch {sa} vs {sb}")  # volume.cpp:35-39


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def gaussian_kernel(sigma: float) -> np.ndarray:
    """gaussian_kernel (ops.cpp:9-29)."""
    w = (C.c_double * 1024)()
    r = C.c_int32()
    check(L.load().rsfg_gaussian_kernel(sigma, w, 1024, C.byref(r)))
    return np.array(w[: 2 * r.value + 1])


class KernelProfile:
    """rsf::KernelProfile (rsf.hpp:64-69): the reference's 14 stage rows
    (rsf.cpp:228-233) with seconds per row and the profiled iteration count.
    The kernels fuse stages, so each kernel's CUDA-event time lands on one row
    (``carrier``) and the rows fused into it stay 0 (include/rsfg.h,
    RSFG_STAGE_COUNT)."""

    kCount = L.RSFG_STAGE_COUNT

    def __init__(self):
        self.seconds = [0.0] * self.kCount
        self.iterations = 0

    @staticmethod
    def names() -> list[str]:
        lib = L.load()
        return [lib.rsfg_stage_name(i).decode() for i in range(L.RSFG_STAGE_COUNT)]

    @staticmethod
    def carrier() -> list[int]:
        lib = L.load()
        return [int(lib.rsfg_stage_carrier(i)) for i in range(L.RSFG_STAGE_COUNT)]

    def add(self, secs, iterations: int) -> None:
        for i in range(self.kCount):
            self.seconds[i] += float(secs[i])
        self.iterations += iterations


def evolve(phi0, I, p: RsfParams, stop=None, stop_every: int = 25, profile: KernelProfile | None = None, *,
           fields: int = 2, device: int = 0, report: L.rsfg_report | None = None) -> np.ndarray:
    """rsf::evolve (rsf.cpp:359-384): returns the evolved phi (same shape as phi0).
    ``profile`` (a KernelProfile) receives the per-row kernel seconds."""
    squeeze = np.ndim(phi0) == 2
    phi = _vol(phi0, "phi0").copy()
    img = _vol(I, "I")
    _check_same(phi, img, "evolve")
    nz, ny, nx = phi.shape
    cp = p.to_c()
    opt = options(fields, device)
    opt.profile_stages = 1 if profile is not None else 0
    rep = report if report is not None else L.rsfg_report()
    cb = L.STOP_FN(0)
    if stop is not None:
        def _cb(ptr, cx, cy, cz, it, _u):
            arr = np.ctypeslib.as_array(ptr, shape=(cz, cy, cx)).copy()
            return 1 if stop(arr, it) else 0
        cb = L.STOP_FN(_cb)
    check(L.load().rsfg_evolve(_ptr(img), _ptr(phi), nx, ny, nz, C.byref(cp), C.byref(opt), cb, None,
                               stop_every, C.byref(rep)))
    if profile is not None:
        profile.add(rep.stage_seconds, rep.iterations)
    return phi[0] if squeeze else phi


def evolve_multi(phi0, I, p: RsfParams, devices, stop=None, stop_every: int = 25, *, fields: int = 2,
                 report: L.rsfg_report | None = None):
    """rsf::evolve over several GPUs of this process (rsfg_evolve_multi):
    z-slabs on ``devices`` (a device may repeat) with peer halo links;
    bitwise equal to ``evolve`` on one device.  ``stop(phi, iteration)`` as in
    ``evolve`` (phi gathered from the slabs)."""
    phi = _vol(phi0, "phi0").copy()
    img = _vol(I, "I")
    _check_same(phi, img, "evolve")
    nz, ny, nx = phi.shape
    cp = p.to_c()
    opt = options(fields, int(devices[0]))
    devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
    rep = report if report is not None else L.rsfg_report()
    cb = L.STOP_FN(0)
    if stop is not None:
        def _cb(ptr, cx, cy, cz, it, _u):
            return 1 if stop(np.ctypeslib.as_array(ptr, shape=(cz, cy, cx)).copy(), it) else 0
        cb = L.STOP_FN(_cb)
    check(L.load().rsfg_evolve_multi(_ptr(img), _ptr(phi), nx, ny, nz, C.byref(cp), C.byref(opt), devs,
                                     len(devices), cb, None, stop_every, C.byref(rep)))
    return phi


def extract_mask(phi, device: int = 0) -> np.ndarray:
    """rsf::extract_mask (rsf.cpp:386-396): 1 where phi < 0."""
    a = np.ascontiguousarray(phi, dtype=np.float32)
    out = np.empty_like(a)
    check(L.load().rsfg_extract_mask(_ptr(a), _ptr(out), a.size, device))
    return out


class EvolutionState:
    """rsf::EvolutionState (rsf.hpp:54-61) held on the GPU."""

    def __init__(self, phi0, I, p: RsfParams, *, fields: int = 2, device: int = 0, check_every: int = 25):
        phi = _vol(phi0, "phi0")
        img = _vol(I, "I")
        _check_same(phi, img, "init_evolution")
        self.shape = phi.shape
        self.p = p
        self._h = C.c_void_p()
        cp = p.to_c()
        opt = options(fields, device, check_every)
        nz, ny, nx = phi.shape
        check(L.load().rsfg_state_create(C.byref(self._h), _ptr(phi), _ptr(img), nx, ny, nz, C.byref(cp),
                                         C.byref(opt)))

    @property
    def handle(self) -> int:
        return self._h.value

    @property
    def iteration(self) -> int:
        it = C.c_int32()
        check(L.load().rsfg_state_iteration(self._h, C.byref(it)))
        return it.value

    @property
    def phi(self) -> np.ndarray:
        out = np.empty(self.shape, np.float32)
        check(L.load().rsfg_state_read_phi(self._h, _ptr(out)))
        return out

    @phi.setter
    def phi(self, value) -> None:
        a = _vol(value, "phi")
        _check_same(a, np.empty(self.shape, np.float32), "phi")
        check(L.load().rsfg_state_write_phi(self._h, _ptr(a)))

    def step(self, profile: KernelProfile | None = None) -> float:
        f = C.c_double()
        if profile is None:
            check(L.load().rsfg_state_step(self._h, C.byref(f)))
        else:
            secs = (C.c_double * L.RSFG_STAGE_COUNT)()
            check(L.load().rsfg_state_step_profiled(self._h, C.byref(f), secs))
            profile.add(secs, 1)
        return f.value

    def set_params(self, p: RsfParams) -> None:
        """Step scalars for the next steps (evolve_step takes p on every call);
        sigma1/sigma2 stay the state's own."""
        cp = p.to_c()
        check(L.load().rsfg_state_set_params(self._h, C.byref(cp)))

    def run(self, n: int) -> L.rsfg_report:
        rep = L.rsfg_report()
        check(L.load().rsfg_state_run(self._h, n, C.byref(rep)))
        return rep

    def profile(self, steps: int) -> dict:
        """Mean CUDA-event ms per kernel group over `steps` steps (KernelProfile analogue)."""
        ms = (C.c_double * 2)()
        lib = L.load()
        check(lib.rsfg_state_profile(self._h, steps, ms))
        return {lib.rsfg_profile_name(i).decode().split(":")[0]: ms[i] for i in range(2)}

    def energy(self) -> np.ndarray:
        out = np.empty(self.shape, np.float32)
        check(L.load().rsfg_state_energy(self._h, _ptr(out)))
        return out

    def mask(self) -> np.ndarray:
        out = np.empty(self.shape, np.float32)
        check(L.load().rsfg_state_mask(self._h, _ptr(out)))
        return out

    def device_phi(self) -> int:
        d = C.c_void_p()
        check(L.load().rsfg_state_device_phi(self._h, C.byref(d)))
        return d.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(L.load().rsfg_state_stream(self._h, C.byref(s)))
        return s.value or 0

    def sync(self) -> None:
        check(L.load().rsfg_state_sync(self._h))

    def launches(self) -> int:
        return int(L.load().rsfg_state_launches(self._h))

    def close(self) -> None:
        if self._h:
            L.load().rsfg_state_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_evolution(phi0, I, p: RsfParams, **kw) -> EvolutionState:
    """rsf::init_evolution (rsf.cpp:293-313)."""
    p.validate()
    return EvolutionState(phi0, I, p, **kw)


class EvolveWorkspace:
    """rsf::EvolveWorkspace (rsf.hpp:72-77): accepted for signature parity;
    the device buffers live in the EvolutionState."""


def evolve_step(state: EvolutionState, I=None, p: RsfParams | None = None, ws: EvolveWorkspace | None = None,
                profile: KernelProfile | None = None) -> float:
    """rsf::evolve_step (rsf.hpp:87-88, rsf.cpp:324-357): returns the sign-change
    fraction.  ``I`` must be the image the state was created with (its device
    copy is used); ``p`` updates the step scalars (sigma stays the state's)."""
    if I is not None:
        _check_same(_vol(I, "I"), np.empty(state.shape, np.float32), "evolve_step")
    if p is not None:
        state.set_params(p)
    return state.step(profile)


def energy(state: EvolutionState, I=None, p: RsfParams | None = None) -> np.ndarray:
    """rsf::energy (rsf.hpp:82, rsf.cpp:315-322)."""
    if I is not None:
        _check_same(_vol(I, "I"), np.empty(state.shape, np.float32), "energy")
    if p is not None:
        p.validate()
        state.set_params(p)
    return state.energy()


def region_intensities(I, phi, sigma1: float, epsilon: float, denom_floor: float = 1e-8, device: int = 0):
    """rsf::region_intensities (rsf.hpp:39-41, rsf.cpp:235-266) on the GPU:
    (r_plus, r_minus), the clamped local means on each side of the contour."""
    img, ph = _vol(I, "I"), _vol(phi, "phi")
    _check_same(img, ph, "region_intensities")
    nz, ny, nx = img.shape
    rp, rm = np.empty_like(img), np.empty_like(img)
    check(L.load().rsfg_region_intensities(_ptr(img), _ptr(ph), nx, ny, nz, sigma1, epsilon, denom_floor, _ptr(rp),
                                           _ptr(rm), device))
    return rp, rm


def directional_forces(I, r_plus, r_minus, KI, KI2, device: int = 0):
    """rsf::directional_forces (rsf.hpp:47-50, rsf.cpp:268-291) on the GPU:
    (F_plus, F_minus) = (KI2 - 2 r KI) + r^2 in f64."""
    img = _vol(I, "I")
    arrs = [_vol(a, n) for a, n in ((r_plus, "r_plus"), (r_minus, "r_minus"), (KI, "KI"), (KI2, "KI2"))]
    for a in arrs:
        _check_same(img, a, "directional_forces")
    Fp, Fm = np.empty_like(img), np.empty_like(img)
    check(L.load().rsfg_directional_forces(*(_ptr(a) for a in arrs), img.size, _ptr(Fp), _ptr(Fm), device))
    return Fp, Fm


def phantom(nx, ny, nz, n_branches=12, radius_min=2.0, radius_max=4.0, tortuosity=0.25, foreground=200.0,
            background=50.0, rng_seed=1, tree_connected=True, axial_blur_sigma=0.0, noise_sigma=20.0,
            contrast_axis=0, contrast_lo=1.0, contrast_hi=1.0, noise_seed=7):
    """Tube-network phantom + perturb (reference phantom.cpp:55-214); returns (image, gt_mask)."""
    s = L.rsfg_phantom_spec()
    L.load().rsfg_phantom_default(C.byref(s))
    for k, v in dict(nx=nx, ny=ny, nz=nz, n_branches=n_branches, radius_min=radius_min, radius_max=radius_max,
                     tortuosity=tortuosity, foreground=foreground, background=background, rng_seed=rng_seed,
                     tree_connected=int(tree_connected), axial_blur_sigma=axial_blur_sigma,
                     noise_sigma=noise_sigma, contrast_axis=contrast_axis, contrast_lo=contrast_lo,
                     contrast_hi=contrast_hi, noise_seed=noise_seed).items():
        setattr(s, k, v)
    img = np.empty((nz, ny, nx), np.float32)
    gt = np.empty((nz, ny, nx), np.float32)
    rc = L.load().rsfg_phantom(C.byref(s), _ptr(img), _ptr(gt))
    if rc != 0:
        raise ParamError(f"phantom spec rejected (rc={rc})")
    return img, gt


def _phantom_spec(nx, ny, nz, **kw):
    s = L.rsfg_phantom_spec()
    L.load().rsfg_phantom_default(C.byref(s))
    for k, v in kw.items():
        setattr(s, k, v)
    s.nx, s.ny, s.nz = nx, ny, nz
    return s


def phantom_device(nx, ny, nz, n_branches=12, radius_min=2.0, radius_max=4.0, tortuosity=0.25, foreground=200.0,
                   background=50.0, rng_seed=1, tree_connected=True, axial_blur_sigma=0.0, noise_sigma=20.0,
                   contrast_axis=0, contrast_lo=1.0, contrast_hi=1.0, noise_seed=7, device=0, with_gt=True):
    """phantom() with the per-voxel work on the GPU.

    Returns (image, gt) as torch CUDA tensors of shape (nz, ny, nx) (gt None if
    with_gt is False).  Same spec and random streams as phantom(); outputs match
    it except where device and host libm round differently (vanishingly rare)."""
    import torch
    s = _phantom_spec(nx, ny, nz, n_branches=n_branches, radius_min=radius_min, radius_max=radius_max,
                      tortuosity=tortuosity, foreground=foreground, background=background, rng_seed=rng_seed,
                      tree_connected=int(tree_connected), axial_blur_sigma=axial_blur_sigma,
                      noise_sigma=noise_sigma, contrast_axis=contrast_axis, contrast_lo=contrast_lo,
                      contrast_hi=contrast_hi, noise_seed=noise_seed)
    dev = torch.device("cuda", device)
    img = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
    gt = torch.empty_like(img) if with_gt else None
    torch.cuda.synchronize(dev)
    n = C.c_int64()
    check(L.load().rsfg_phantom_device(C.byref(s), img.data_ptr(), gt.data_ptr() if gt is not None else None,
                                        device, C.byref(n)))
    return img, gt


def init_phi_device(image, sigma_b=3.0, response_threshold=0.1, nms_radius=0.0, dark=False, seed_radius=2.0,
                    max_seeds=1 << 20):
    """rsf::init_phi (seeding.cpp:221-235) on the GPU.

    image: torch CUDA float32 tensor (nz, ny, nx).  Returns (phi0 tensor,
    seeds int32 array (n, 3) of x, y, z, responses float32 array (n,)); the
    Jacobi iteration count of the distance solve is left in init_phi_device.iterations."""
    import torch
    nz, ny, nx = image.shape
    img = image.contiguous()
    phi = torch.empty_like(img)
    b = L.rsfg_blob_params(sigma_b, response_threshold, nms_radius, int(dark))
    xyz = np.zeros((max_seeds, 3), np.int32)
    resp = np.zeros(max_seeds, np.float32)
    n, it = C.c_int32(), C.c_int32()
    torch.cuda.synchronize(img.device)
    check(L.load().rsfg_init_phi_device(img.data_ptr(), nx, ny, nz, C.byref(b), seed_radius, phi.data_ptr(),
                                        img.device.index or 0, C.byref(n), xyz.ctypes.data_as(C.POINTER(C.c_int32)),
                                        resp.ctypes.data, max_seeds, C.byref(it)))
    k = min(n.value, max_seeds)
    init_phi_device.iterations = it.value
    return phi, xyz[:k].copy(), resp[:k].copy()


MERGE_MODES = {"linear": 0, "minimum": 1, "maximum": 2, "average": 3}  # rsf::MergeMode (tiling.hpp:26)


def plan_tiles(shape, tile_size, sigma1, sigma2=0.0):
    """rsf::plan_tiles (tiling.cpp:14-59).  shape/tile_size are (nx, ny, nz).
    Returns (tiles, curtain); each tile a dict of ix, iy, iz and (x, y, z)
    core_origin / core_extent / pad_origin / pad_extent tuples."""
    n, c = C.c_int32(), C.c_int32()
    check(L.load().rsfg_plan_tiles(*shape, *tile_size, sigma1, sigma2, None, 0, C.byref(n), C.byref(c)))
    buf = (L.rsfg_tile * n.value)()
    check(L.load().rsfg_plan_tiles(*shape, *tile_size, sigma1, sigma2, buf, n.value, C.byref(n), C.byref(c)))
    tiles = [{"ix": t.ix, "iy": t.iy, "iz": t.iz, "core_origin": tuple(t.core_origin),
              "core_extent": tuple(t.core_extent), "pad_origin": tuple(t.pad_origin),
              "pad_extent": tuple(t.pad_extent)} for t in buf]
    return tiles, c.value


def merge_phi_device(tile_phis, shape, tile_size, curtain, mode="linear", device=0):
    """rsf::merge_phi (tiling.cpp:99-193) on the GPU.  tile_phis: torch CUDA
    tensors of each tile's padded extent (nz, ny, nx), in plan_tiles order."""
    import torch
    nx, ny, nz = shape
    ts = [t.contiguous() for t in tile_phis]
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device=ts[0].device)
    ptrs = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    torch.cuda.synchronize(out.device)
    check(L.load().rsfg_merge_phi_device(ptrs, len(ts), nx, ny, nz, *tile_size, curtain, MERGE_MODES[mode],
                                         out.data_ptr(), device))
    return out


def run_pipeline(vol, p: "RsfParams", tile_size, *, sigma_b=3.0, response_threshold=0.1, nms_radius=0.0,
                 dark=False, global_seeding=False, merge="linear", seed_radius=2.0, fields=2, device=0,
                 spill_dir=None):
    """rsf::run_pipeline (tiling.cpp:201-275) on one GPU: returns (phi, mask,
    warnings) as host arrays / list of strings.  spill_dir: every tile's phi
    is written there (tile_file_name) plus layout.manifest, like the
    reference's PipelineOptions::spill_dir."""
    vol = np.ascontiguousarray(vol, np.float32)
    nz, ny, nx = vol.shape
    phi = np.empty_like(vol)
    mask = np.empty_like(vol)
    b = L.rsfg_blob_params(sigma_b, response_threshold, nms_radius, int(dark))
    o = L.rsfg_pipeline_options()
    L.load().rsfg_pipeline_options_default(C.byref(o))
    o.global_seeding, o.merge, o.seed_radius, o.device, o.fields = (int(global_seeding), MERGE_MODES[merge],
                                                                    seed_radius, device, fields)
    o.spill_dir = str(spill_dir).encode() if spill_dir else None
    cp = p.to_c()
    warn = C.create_string_buffer(1 << 16)
    nw = C.c_int32()
    check(L.load().rsfg_run_pipeline(_ptr(vol), nx, ny, nz, C.byref(cp), C.byref(b), *tile_size, C.byref(o),
                                     _ptr(phi), _ptr(mask), warn, len(warn), C.byref(nw)))
    lines = [w for w in warn.value.decode().split("\n") if w]
    return phi, mask, lines


def _tiles_c(tiles):
    buf = (L.rsfg_tile * len(tiles))()
    for b, t in zip(buf, tiles):
        b.ix, b.iy, b.iz = t["ix"], t["iy"], t["iz"]
        b.core_origin[:], b.core_extent[:] = t["core_origin"], t["core_extent"]
        b.pad_origin[:], b.pad_extent[:] = t["pad_origin"], t["pad_extent"]
    return buf


def tile_file_name(tile) -> str:
    """rsf::tile_file_name (tiling.cpp:195-199)."""
    buf = C.create_string_buffer(64)
    check(L.load().rsfg_tile_file_name(_tiles_c([tile]), buf, len(buf)))
    return buf.value.decode()


def save_manifest(path, shape, tile_size, curtain, tiles):
    """rsf::save_manifest (tiling.cpp:277-295)."""
    check(L.load().rsfg_save_manifest(str(path).encode(), *shape, *tile_size, curtain, _tiles_c(tiles), len(tiles)))


def load_manifest(path):
    """rsf::load_manifest (tiling.cpp:297-321): (shape, tile_size, curtain,
    tiles) with tiles as plan_tiles returns them."""
    d, ts, c, n = (C.c_int32 * 3)(), (C.c_int32 * 3)(), C.c_int32(), C.c_int32()
    hp = str(path).encode()
    check(L.load().rsfg_load_manifest(hp, d, ts, C.byref(c), None, 0, C.byref(n)))
    buf = (L.rsfg_tile * n.value)()
    check(L.load().rsfg_load_manifest(hp, d, ts, C.byref(c), buf, n.value, C.byref(n)))
    tiles = [{"ix": t.ix, "iy": t.iy, "iz": t.iz, "core_origin": tuple(t.core_origin),
              "core_extent": tuple(t.core_extent), "pad_origin": tuple(t.pad_origin),
              "pad_extent": tuple(t.pad_extent)} for t in buf]
    return tuple(d), tuple(ts), c.value, tiles


def merge_from_dir_device(directory, shape, tile_size, curtain, tiles, mode="linear", device=0):
    """rsf::merge_from_dir (tiling.cpp:323-332): the spilled tiles are read
    straight into device buffers and merged on the GPU; returns a torch CUDA
    tensor (nz, ny, nx)."""
    import torch
    nx, ny, nz = shape
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device=f"cuda:{device}")
    torch.cuda.synchronize(out.device)
    check(L.load().rsfg_merge_from_dir(str(directory).encode(), nx, ny, nz, *tile_size, curtain, _tiles_c(tiles),
                                       len(tiles), MERGE_MODES[mode], out.data_ptr(), device))
    return out


def read_volume_device(header, device=0):
    """rsf::read_volume (volume_io.cpp:24-113) straight into a torch CUDA
    tensor (nz, ny, nx); returns (volume, spacing (sx, sy, sz), value_range,
    h2d_bytes)."""
    import torch
    nx, ny, nz, eb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    sp = (C.c_double * 3)()
    hb = str(header).encode()
    check(L.load().rsfg_volume_info(hb, C.byref(nx), C.byref(ny), C.byref(nz), sp, C.byref(eb)))
    out = torch.empty((nz.value, ny.value, nx.value), dtype=torch.float32, device=torch.device("cuda", device))
    rng = (C.c_float * 2)()
    moved = C.c_int64()
    check(L.load().rsfg_read_volume_device(hb, out.data_ptr(), out.numel(), device, rng, C.byref(moved)))
    return out, tuple(sp), (rng[0], rng[1]), moved.value


def write_volume_device(header, vol, spacing=(1.0, 1.0, 1.0), device=0):
    """rsf::write_volume (volume_io.cpp:115-137) of a torch CUDA tensor."""
    nz, ny, nx = vol.shape
    sp = (C.c_double * 3)(*spacing)
    check(L.load().rsfg_write_volume_device(str(header).encode(), vol.contiguous().data_ptr(), nx, ny, nz, sp, None,
                                            device))


def overlap_device(a, b, device=0):
    """(dice, jaccard) (validation.cpp:41-52) of two torch CUDA tensors."""
    d, j = C.c_double(), C.c_double()
    check(L.load().rsfg_overlap_device(a.contiguous().data_ptr(), b.contiguous().data_ptr(), a.numel(), device,
                                       C.byref(d), C.byref(j)))
    return d.value, j.value


def threshold_phi0(image, level: float = 125.0, inside: float = -2.0, outside: float = 2.0) -> np.ndarray:
    """Documented threshold initialisation for throughput runs (SURVEY.md 8(d) cfg 4)."""
    return np.where(np.asarray(image) > level, np.float32(inside), np.float32(outside)).astype(np.float32)


def dice(a, b) -> float:
    """rsf::dice (validation.cpp:41-45) on masks (> 0.5 is foreground)."""
    a = np.asarray(a) > 0.5
    b = np.asarray(b) > 0.5
    na, nb = int(a.sum()), int(b.sum())
    if na + nb == 0:
        return 1.0
    return 2.0 * int(np.logical_and(a, b).sum()) / (na + nb)
