"""ctypes loaders for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -- our plain-C restatement, oracle/build/librsforacle.so
  (oracle/rsf_oracle.c, each function cites the reference file:line).
* ``RefLib``  -- the unmodified reference compiled from its own sources by
  oracle/Makefile into oracle/_ref/librsfref_v{3,4}.so, driven through the
  reference's public C++ API via oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "build" / "librsforacle.so"
REF_DIR = ROOT / "oracle" / "_ref"

F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
I64P = C.POINTER(C.c_int64)


class Params(C.Structure):
    """Field-for-field rsf::RsfParams (reference include/rsf/rsf.hpp:13-26)."""

    _fields_ = [
        ("sigma1", C.c_double),
        ("sigma2", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("epsilon", C.c_double),
        ("dt", C.c_double),
        ("max_iters", C.c_int32),
        ("convergence_fraction", C.c_double),
        ("denom_floor", C.c_double),
        ("grad_floor", C.c_double),
    ]


def params(**kw) -> Params:
    """RsfParams defaults (rsf.hpp:13-22) overridden by keyword."""
    d = dict(sigma1=5.0, sigma2=0.0, alpha=58.5225, beta=0.1, epsilon=1.0, dt=0.06, max_iters=100,
             convergence_fraction=0.0, denom_floor=1e-8, grad_floor=1e-8)
    d.update(kw)
    return Params(**d)


class Geom(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("zb", C.c_int), ("ze", C.c_int)]


def _shape(a):
    nz, ny, nx = a.shape
    return nx, ny, nz


class Oracle:
    """The plain-C restatement of the reference hot path."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = self.lib = C.CDLL(str(path))
        L.oracle_init.argtypes = [C.c_int, C.c_int, C.c_int, F32P, C.c_double, F32P, F32P,
                                  C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.oracle_step.argtypes = [C.c_int, C.c_int, C.c_int, F32P, F32P, F32P, F32P, C.c_float, C.c_float,
                                  C.POINTER(Params), F32P, I64P]
        L.oracle_step.restype = C.c_int64
        L.oracle_step_slab.argtypes = [C.POINTER(Geom), F32P, F32P, F32P, F32P, C.c_float, C.c_float,
                                       C.POINTER(Params), F32P, C.c_int, C.c_int, I64P]
        L.oracle_step_slab.restype = C.c_int64
        L.oracle_energy.argtypes = [C.c_int, C.c_int, C.c_int, F32P, F32P, F32P, F32P, C.c_float, C.c_float,
                                    C.POINTER(Params), F32P]
        L.oracle_convolve.argtypes = [C.c_int, C.c_int, C.c_int, F32P, C.c_double, F32P]
        L.oracle_gaussian_kernel.argtypes = [C.c_double, np.ctypeslib.ndpointer(np.float64), C.c_int]
        L.oracle_region_intensities.argtypes = [C.c_int, C.c_int, C.c_int, F32P, F32P, C.c_double, C.c_double,
                                                C.c_double, F32P, F32P]
        L.oracle_directional_forces.argtypes = [C.c_size_t, F32P, F32P, F32P, F32P, F32P, F32P]

    def gaussian_kernel(self, sigma):
        w = np.zeros(1024, np.float64)
        r = self.lib.oracle_gaussian_kernel(sigma, w, 1024)
        if r < 0:
            raise ValueError("bad sigma")
        return w[: 2 * r + 1].copy()

    def init(self, I, p: Params):
        nx, ny, nz = _shape(I)
        KI = np.empty_like(I)
        KI2 = np.empty_like(I)
        lo, hi = C.c_float(), C.c_float()
        self.lib.oracle_init(nx, ny, nz, I, p.sigma2, KI, KI2, C.byref(lo), C.byref(hi))
        return KI, KI2, lo.value, hi.value

    def step(self, phi, I, p: Params, static=None):
        """One evolve_step; returns (phi_next, sign_changes, first_bad_index or -1)."""
        nx, ny, nz = _shape(phi)
        KI, KI2, lo, hi = static if static is not None else self.init(I, p)
        out = np.empty_like(phi)
        bad = C.c_int64()
        sc = self.lib.oracle_step(nx, ny, nz, phi, I, KI, KI2, lo, hi, C.byref(p), out, C.byref(bad))
        return out, int(sc), int(bad.value)

    def step_slab(self, geom: Geom, phi, I, KI, KI2, lo, hi, p: Params, z0, z1):
        out = np.zeros_like(phi)
        bad = C.c_int64()
        sc = self.lib.oracle_step_slab(C.byref(geom), phi, I, KI, KI2, lo, hi, C.byref(p), out, z0, z1,
                                       C.byref(bad))
        return out, int(sc), int(bad.value)

    def energy(self, phi, I, p: Params, static=None):
        nx, ny, nz = _shape(phi)
        KI, KI2, lo, hi = static if static is not None else self.init(I, p)
        E = np.empty_like(phi)
        self.lib.oracle_energy(nx, ny, nz, phi, I, KI, KI2, lo, hi, C.byref(p), E)
        return E

    def convolve(self, v, sigma):
        nx, ny, nz = _shape(v)
        out = np.empty_like(v)
        self.lib.oracle_convolve(nx, ny, nz, v, sigma, out)
        return out

    def region_intensities(self, I, phi, sigma1, epsilon, denom_floor=1e-8):
        """(r_plus, r_minus) -- rsf::region_intensities (rsf.cpp:235-266)."""
        nx, ny, nz = _shape(I)
        rp, rm = np.empty_like(I), np.empty_like(I)
        self.lib.oracle_region_intensities(nx, ny, nz, I, phi, sigma1, epsilon, denom_floor, rp, rm)
        return rp, rm

    def directional_forces(self, r_plus, r_minus, KI, KI2):
        """(F_plus, F_minus) -- rsf::directional_forces (rsf.cpp:268-291)."""
        Fp, Fm = np.empty_like(KI), np.empty_like(KI)
        self.lib.oracle_directional_forces(KI.size, r_plus, r_minus, KI, KI2, Fp, Fm)
        return Fp, Fm

    def evolve(self, phi0, I, p: Params, iters=None):
        st = self.init(I, p)
        phi = phi0.copy()
        for _ in range(p.max_iters if iters is None else iters):
            phi, _, bad = self.step(phi, I, p, st)
            if bad >= 0:
                raise FloatingPointError(f"blowup at {bad}")
        return phi


def host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx512f" in f.read()
    except OSError:
        return False


def ref_so_path() -> Path | None:
    pref = ["v4", "v3"] if host_has_avx512() else ["v3"]
    for v in pref:
        p = REF_DIR / f"librsfref_{v}.so"
        if p.exists():
            return p
    return None


class RefLib:
    """The unmodified reference (compiled from /root/reference sources)."""

    def __init__(self, path: Path | None = None):
        path = path or ref_so_path()
        if path is None or not Path(path).exists():
            raise FileNotFoundError("oracle/_ref/librsfref_*.so missing: run `make -C oracle ref` here")
        self.path = Path(path)
        L = self.lib = C.CDLL(str(path))
        L.rsfref_last_error.restype = C.c_char_p
        L.rsfref_evolve.argtypes = [F32P, F32P, C.c_int, C.c_int, C.c_int, C.POINTER(Params)]
        L.rsfref_state_create.argtypes = [C.POINTER(C.c_void_p), F32P, F32P, C.c_int, C.c_int, C.c_int,
                                          C.POINTER(Params)]
        L.rsfref_state_step.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.rsfref_state_phi.argtypes = [C.c_void_p, F32P]
        L.rsfref_state_set_phi.argtypes = [C.c_void_p, F32P]
        L.rsfref_state_energy.argtypes = [C.c_void_p, F32P]
        L.rsfref_state_static.argtypes = [C.c_void_p, F32P, F32P, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.rsfref_state_destroy.argtypes = [C.c_void_p]
        L.rsfref_convolve.argtypes = [F32P, C.c_int, C.c_int, C.c_int, C.c_double, F32P]
        L.rsfref_extract_mask.argtypes = [F32P, C.c_int, C.c_int, C.c_int, F32P]
        L.rsfref_phantom.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_float, C.c_float, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                     C.c_int, C.c_double, C.c_double, C.c_uint64, F32P, F32P]
        L.rsfref_init_phi.argtypes = [F32P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_int, C.c_double, F32P, C.POINTER(C.c_int)]
        L.rsfref_detect_seeds.argtypes = [F32P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                          C.c_int, C.POINTER(C.c_int), F32P, C.c_int, C.POINTER(C.c_int)]
        L.rsfref_merge_phi.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, F32P]
        L.rsfref_run_pipeline.argtypes = [F32P, C.c_int, C.c_int, C.c_int, C.POINTER(Params), C.c_double,
                                          C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          F32P, F32P, C.POINTER(C.c_int)]
        L.rsfref_read_volume.argtypes = [C.c_char_p, F32P, C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), F32P]
        L.rsfref_dice.argtypes = [F32P, F32P, C.c_int, C.c_int, C.c_int]
        L.rsfref_dice.restype = C.c_double
        L.rsfref_set_workers.argtypes = [C.c_int]
        L.rsfref_region_intensities.argtypes = [F32P, F32P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                                C.c_double, F32P, F32P]
        L.rsfref_directional_forces.argtypes = [F32P, F32P, F32P, F32P, F32P, C.c_int, C.c_int, C.c_int, F32P,
                                                F32P]
        L.rsfref_workers.restype = C.c_int

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.rsfref_last_error().decode()
            raise {1: ValueError, 2: ValueError, 3: FloatingPointError, 8: OSError}.get(rc, RuntimeError)(msg)

    def set_workers(self, n):
        self.lib.rsfref_set_workers(n)

    def workers(self):
        return self.lib.rsfref_workers()

    def evolve(self, phi0, I, p: Params):
        nx, ny, nz = _shape(I)
        phi = np.ascontiguousarray(phi0, np.float32).copy()
        self._check(self.lib.rsfref_evolve(np.ascontiguousarray(I, np.float32), phi, nx, ny, nz, C.byref(p)))
        return phi

    def convolve(self, v, sigma):
        nx, ny, nz = _shape(v)
        out = np.empty_like(v)
        self._check(self.lib.rsfref_convolve(v, nx, ny, nz, sigma, out))
        return out

    def region_intensities(self, I, phi, sigma1, epsilon, denom_floor=1e-8):
        nx, ny, nz = _shape(I)
        rp, rm = np.empty_like(I), np.empty_like(I)
        self._check(self.lib.rsfref_region_intensities(I, phi, nx, ny, nz, sigma1, epsilon, denom_floor, rp, rm))
        return rp, rm

    def directional_forces(self, I, r_plus, r_minus, KI, KI2):
        nx, ny, nz = _shape(I)
        Fp, Fm = np.empty_like(I), np.empty_like(I)
        self._check(self.lib.rsfref_directional_forces(I, r_plus, r_minus, KI, KI2, nx, ny, nz, Fp, Fm))
        return Fp, Fm

    def phantom(self, nx, ny, nz, n_branches=12, rmin=2.0, rmax=4.0, tortuosity=0.25, fg=200.0, bg=50.0,
                seed=1, tree_connected=True, axial_blur=0.0, noise_sigma=20.0, contrast_axis=0, lo=1.0,
                hi=1.0, noise_seed=7):
        img = np.empty((nz, ny, nx), np.float32)
        gt = np.empty((nz, ny, nx), np.float32)
        self._check(self.lib.rsfref_phantom(nx, ny, nz, n_branches, rmin, rmax, tortuosity, fg, bg, seed,
                                            int(tree_connected), axial_blur, noise_sigma, contrast_axis, lo,
                                            hi, noise_seed, img, gt))
        return img, gt

    def init_phi(self, vol, sigma_b=3.0, threshold=0.1, nms=0.0, dark=False, seed_radius=2.0):
        nx, ny, nz = _shape(vol)
        phi = np.empty_like(vol)
        n = C.c_int()
        self._check(self.lib.rsfref_init_phi(vol, nx, ny, nz, sigma_b, threshold, nms, int(dark), seed_radius,
                                             phi, C.byref(n)))
        return phi, n.value

    def detect_seeds(self, vol, sigma_b=3.0, threshold=0.1, nms=0.0, dark=False, cap=1 << 20):
        """(xyz int32 (n, 3), responses float32 (n,)) in the reference's order."""
        nx, ny, nz = _shape(vol)
        xyz = np.zeros((cap, 3), np.int32)
        resp = np.zeros(cap, np.float32)
        n = C.c_int()
        self._check(self.lib.rsfref_detect_seeds(vol, nx, ny, nz, sigma_b, threshold, nms, int(dark),
                                                 xyz.ctypes.data_as(C.POINTER(C.c_int)), resp, cap, C.byref(n)))
        k = min(n.value, cap)
        return xyz[:k].copy(), resp[:k].copy()

    def merge_phi(self, tiles, shape, tile_size, sigma1, sigma2=0.0, mode=0):
        """merge_phi over plan_tiles(shape (nx, ny, nz), tile_size, sigma1, sigma2)."""
        nx, ny, nz = shape
        keep = [np.ascontiguousarray(t, np.float32) for t in tiles]
        ptrs = (C.c_void_p * len(keep))(*[t.ctypes.data for t in keep])
        out = np.empty((nz, ny, nx), np.float32)
        self._check(self.lib.rsfref_merge_phi(ptrs, len(keep), nx, ny, nz, *tile_size, sigma1, sigma2, mode, out))
        return out

    def run_pipeline(self, vol, p, tile_size, sigma_b=3.0, threshold=0.1, global_seeding=False, mode=0,
                     seed_radius=2.0):
        nx, ny, nz = _shape(vol)
        phi = np.empty_like(vol)
        mask = np.empty_like(vol)
        nw = C.c_int()
        self._check(self.lib.rsfref_run_pipeline(vol, nx, ny, nz, C.byref(p), sigma_b, threshold, *tile_size,
                                                 int(global_seeding), mode, seed_radius, phi, mask, C.byref(nw)))
        return phi, mask, nw.value

    def save_manifest(self, path, shape, tile_size, sigma1, sigma2=0.0):
        self._check(self.lib.rsfref_save_manifest(str(path).encode(), *shape, *tile_size, C.c_double(sigma1),
                                                  C.c_double(sigma2)))

    def merge_from_dir(self, directory, manifest, shape, mode=0):
        nx, ny, nz = shape
        out = np.empty((nz, ny, nx), np.float32)
        self._check(self.lib.rsfref_merge_from_dir(str(directory).encode(), str(manifest).encode(), mode,
                                                   out.ctypes.data_as(C.POINTER(C.c_float)), C.c_long(out.size)))
        return out

    def read_volume(self, header, cap=1 << 26):
        out = np.empty(cap, np.float32)
        nx, ny, nz = C.c_int(), C.c_int(), C.c_int()
        rng = np.empty(2, np.float32)
        self._check(self.lib.rsfref_read_volume(str(header).encode(), out, cap, C.byref(nx), C.byref(ny),
                                                C.byref(nz), rng))
        return out[:nx.value * ny.value * nz.value].reshape(nz.value, ny.value, nx.value).copy(), tuple(rng)

    def dice(self, a, b):
        nx, ny, nz = _shape(a)
        return self.lib.rsfref_dice(np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32),
                                    nx, ny, nz)

    def state(self, phi0, I, p: Params):
        return RefState(self, phi0, I, p)


class RefState:
    """rsf::init_evolution + evolve_step through the reference library."""

    def __init__(self, ref: RefLib, phi0, I, p: Params):
        self.ref, self.p = ref, p
        self.shape = I.shape
        self.h = C.c_void_p()
        nx, ny, nz = _shape(I)
        ref._check(ref.lib.rsfref_state_create(C.byref(self.h), np.ascontiguousarray(phi0, np.float32),
                                               np.ascontiguousarray(I, np.float32), nx, ny, nz, C.byref(p)))

    def step(self):
        f = C.c_double()
        self.ref._check(self.ref.lib.rsfref_state_step(self.h, C.byref(f)))
        return f.value

    def phi(self):
        out = np.empty(self.shape, np.float32)
        self.ref.lib.rsfref_state_phi(self.h, out)
        return out

    def set_phi(self, phi):
        self.ref.lib.rsfref_state_set_phi(self.h, np.ascontiguousarray(phi, np.float32))

    def energy(self):
        out = np.empty(self.shape, np.float32)
        self.ref._check(self.ref.lib.rsfref_state_energy(self.h, out))
        return out

    def static(self):
        KI = np.empty(self.shape, np.float32)
        KI2 = np.empty(self.shape, np.float32)
        lo, hi = C.c_float(), C.c_float()
        self.ref.lib.rsfref_state_static(self.h, KI, KI2, C.byref(lo), C.byref(hi))
        return KI, KI2, lo.value, hi.value

    def __del__(self):
        try:
            self.ref.lib.rsfref_state_destroy(self.h)
        except Exception:
            pass
