"""The drop-in boundary on CPU: librsfg.so loads, exports every entry point
include/rsfg.h declares, and its host-side logic (parameter validation,
kernel weights, the phantom generator) matches the reference."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    txt = (ROOT / "include" / "rsfg.h").read_text()
    return sorted(set(re.findall(r"\b(rsfg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2404_02813_b200._lib import LIB_PATH, SIGNATURES
    lib = C.CDLL(str(LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(SIGNATURES) | {"rsfg_stop_fn"}


def test_library_is_sm100a():
    import subprocess
    from paper_2404_02813_b200._lib import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("field,value,msg", [
    ("sigma1", -1.0, "sigma1 must be >= 0"), ("sigma2", -0.5, "sigma2 must be >= 0"),
    ("epsilon", 0.0, "epsilon must be > 0"), ("dt", 0.0, "dt must be > 0"),
    ("max_iters", 0, "max_iters must be >= 1"), ("convergence_fraction", 1.0, "must be in \\[0,1\\)"),
    ("denom_floor", 0.0, "denom_floor must be > 0"), ("grad_floor", -1.0, "grad_floor must be > 0")])
def test_param_validation_messages(field, value, msg):
    """RsfParams::validate (rsf.cpp:10-20): same checks, same messages."""
    import paper_2404_02813_b200 as rsf
    p = rsf.RsfParams(**{field: value})
    with pytest.raises(rsf.ParamError, match=msg):
        p.validate()


def test_defaults_match_reference():
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200 import _lib as L
    c = L.rsfg_params()
    L.load().rsfg_params_default(C.byref(c))
    p = rsf.RsfParams()
    for f in ("sigma1", "sigma2", "alpha", "beta", "epsilon", "dt", "max_iters", "convergence_fraction",
              "denom_floor", "grad_floor"):
        assert getattr(c, f) == getattr(p, f)


def test_gaussian_weights_match_reference(oracle):
    import paper_2404_02813_b200 as rsf
    for s in (0.0, 0.7, 3.0, 5.0, 6.0):
        assert np.array_equal(rsf.gaussian_kernel(s), oracle.gaussian_kernel(s))


def test_phantom_bit_exact_vs_reference(ref):
    import paper_2404_02813_b200 as rsf
    for kw, rkw in [({}, {}), (dict(axial_blur_sigma=2.0, contrast_axis=3, contrast_lo=0.6, contrast_hi=1.0,
                                    noise_sigma=25.0),
                               dict(axial_blur=2.0, contrast_axis=3, lo=0.6, hi=1.0, noise_sigma=25.0))]:
        a, ga = rsf.phantom(40, 36, 30, n_branches=4, **kw)
        b, gb = ref.phantom(40, 36, 30, n_branches=4, **rkw)
        assert np.array_equal(ga, gb)
        assert np.array_equal(a, b)


def test_threshold_init():
    import paper_2404_02813_b200 as rsf
    img = np.array([[[0.0, 200.0, 125.0]]], np.float32)
    assert rsf.threshold_phi0(img).tolist() == [[[2.0, -2.0, 2.0]]]


def test_slab_plan():
    from paper_2404_02813_b200.spmd import held_range, plan_slabs
    assert plan_slabs(512, 8, 9) == [(64 * i, 64 * (i + 1)) for i in range(8)]
    assert plan_slabs(10, 3, 2) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        plan_slabs(20, 4, 9)
    assert held_range(0, 64, 512, 9) == (0, 73)
    assert held_range(64, 128, 512, 9) == (55, 137)


@pytest.fixture(scope="module")
def c_caller(tmp_path_factory):
    """tests/c/abi_check.c compiled as C99 against include/rsfg.h + librsfg.so."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_2404_02813_b200._lib import LIB_PATH
    root = Path(__file__).resolve().parents[1]
    out = tmp_path_factory.mktemp("c") / "abi_check"
    lib = LIB_PATH.parent
    subprocess.run(["gcc", "-std=c99", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{root / 'include'}",
                    str(root / "tests" / "c" / "abi_check.c"), f"-L{lib}", "-lrsfg", f"-Wl,-rpath,{lib}", "-o",
                    str(out)], check=True, capture_output=True, text=True)
    return out


def test_plain_c_caller_cpu(c_caller, oracle):
    """A C99 host binds the boundary with no C++ or Python in between."""
    import json
    import subprocess
    r = json.loads(subprocess.run([str(c_caller), "cpu"], check=True, capture_output=True, text=True).stdout)
    assert r["default_ok"] == 1 and r["rc_dt"] == 1 and r["msg"] == "RsfParams: dt must be > 0"
    assert r["radius"] == 9 and r["w9"] == oracle.gaussian_kernel(3.0)[9]
    assert r["stage2"] == "K*H-I" and r["stage11"] == "R-combine" and r["version"].startswith("rsfg")
    assert r["n_tiles"] > 0 and r["curtain"] == 6


@pytest.mark.gpu
def test_plain_c_caller_gpu(c_caller, tmp_path):
    import json
    import subprocess
    import paper_2404_02813_b200 as rsf
    from _inputs import case
    nx, ny, nz = 64, 40, 36
    img, phi, _ = case(nx, ny, nz, n_branches=3)
    (tmp_path / "img.raw").write_bytes(np.ascontiguousarray(img, np.float32).tobytes())
    (tmp_path / "phi.raw").write_bytes(np.ascontiguousarray(phi, np.float32).tobytes())
    r = json.loads(subprocess.run([str(c_caller), "gpu", str(nx), str(ny), str(nz), str(tmp_path / "img.raw"),
                                   str(tmp_path / "phi.raw"), str(tmp_path)], check=True, capture_output=True,
                                  text=True).stdout)
    assert r["iterations"] == 12 and r["launches"] > 0
    want = rsf.evolve(phi, img, rsf.RsfParams(sigma1=3.0, max_iters=12))
    got = np.fromfile(tmp_path / "c_evolve.raw", np.float32).reshape(nz, ny, nx)
    got_m = np.fromfile(tmp_path / "c_evolve_multi.raw", np.float32).reshape(nz, ny, nx)
    assert np.array_equal(got, want) and np.array_equal(got_m, want)
