"""include/rsfgpu.hpp, the reference-shaped C++ surface (rsf::evolve,
init_phi, plan_tiles, run_pipeline with the namespace switched), compiled the
way a reference caller would compile it: g++ against the header and
librsfg.so.  tests/cpp/wrapper_check.cpp drives it; its results must equal
the ctypes API's bit for bit (both are one C-ABI call), and its seeds the
reference's."""
import json
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def wrapper_bin(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    from paper_2404_02813_b200._lib import LIB_PATH
    out = tmp_path_factory.mktemp("cpp") / "wrapper_check"
    lib = LIB_PATH.parent
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "wrapper_check.cpp"), f"-L{lib}", "-lrsfg",
                    f"-Wl,-rpath,{lib}", "-o", str(out)], check=True, capture_output=True, text=True)
    return out


def test_cpp_wrapper_host_logic(wrapper_bin, tmp_path):
    import paper_2404_02813_b200 as rsf
    r = json.loads(subprocess.run([str(wrapper_bin), "cpu", str(tmp_path)], check=True, capture_output=True,
                                  text=True).stdout)
    assert r["param_error"] == 1 and r["tile_error"] == 1
    assert r["manifest_roundtrip"] == 1 and r["io_error"] == 1 and r["last_name"] == "tile_z01_y01_x02.vmh"
    tiles, curtain = rsf.plan_tiles((100, 80, 60), (48, 40, 30), 2.0, 1.0)
    assert r["curtain"] == curtain
    want = [[t["ix"], t["iy"], t["iz"], *t["core_origin"], *t["core_extent"], *t["pad_origin"], *t["pad_extent"]]
            for t in tiles]
    assert r["tiles"] == want


@pytest.mark.gpu
def test_cpp_wrapper_gpu_matches_api(wrapper_bin, tmp_path, ref):
    import torch
    import paper_2404_02813_b200 as rsf
    from _inputs import case
    nx, ny, nz = 64, 48, 40
    img = np.ascontiguousarray(case(nx, ny, nz, n_branches=6, init="threshold")[0], dtype=np.float32)
    (tmp_path / "img.raw").write_bytes(img.tobytes())
    r = json.loads(subprocess.run([str(wrapper_bin), "gpu", str(nx), str(ny), str(nz), str(tmp_path / "img.raw"),
                                   str(tmp_path)], check=True, capture_output=True, text=True).stdout)

    def load(name):
        return np.fromfile(tmp_path / name, np.float32).reshape(nz, ny, nx)

    phi0_t, seeds, resp = rsf.init_phi_device(torch.from_numpy(img.copy()).cuda())
    phi0 = phi0_t.cpu().numpy()
    assert np.array_equal(load("init_phi.raw"), phi0)
    xyz_r, resp_r = ref.detect_seeds(img)
    assert r["n_seeds"] == len(xyz_r) == len(seeds)
    assert r["seed0"][:3] == xyz_r[0].tolist() and np.float32(r["seed0"][3]) == resp_r[0]

    p = rsf.RsfParams(sigma1=2.0, max_iters=20)
    phi = rsf.evolve(phi0, img, p)
    assert np.array_equal(load("evolve_phi.raw"), phi)
    assert np.array_equal(load("evolve_multi_phi.raw"), phi)  # rsfgpu::evolve_multi, two linked slabs
    assert np.array_equal(load("mask.raw"), rsf.extract_mask(phi))

    phi_p, mask_p, warn = rsf.run_pipeline(img, p, (nx // 2, ny // 2, nz // 2))
    assert r["n_tiles"] == 8 and r["n_warnings"] == len(warn)
    assert np.array_equal(load("pipe_phi.raw"), phi_p)
    assert np.array_equal(load("pipe_mask.raw"), mask_p)
    assert np.array_equal(load("merged_from_dir.raw"), phi_p)  # spill_dir + load_manifest + merge_from_dir
    assert (tmp_path / "layout.manifest").exists() and len(list(tmp_path.glob("tile_z*.vmh"))) == 8


PROFCHECK = ROOT / "oracle" / "_ref" / "profiling_check"
STAGES = ["H-I", "H+I", "K*H-I", "K*H+I", "K*H-", "K*H+", "delta", "grad", "grad-mag", "laplacian",
          "grad/|grad|", "R-combine", "E+", "E-"]  # rsf.cpp:228-233


def _profcheck():
    if Path("/root/reference/proj/src/profiling.cpp").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "profcheck"], check=True, capture_output=True)
    if not PROFCHECK.exists():
        pytest.skip("oracle/_ref/profiling_check not built (reference sources absent)")
    return PROFCHECK


def _rows(text):
    rows = {}
    for line in text.splitlines()[2:]:
        parts = line.split()
        if parts and parts[0] != "total":
            rows[" ".join(parts[:-2])] = (float(parts[-2]), float(parts[-1].rstrip("%")))
    return rows


def test_reference_profiling_cpp_compiles_against_wrapper():
    """The reference's own src/profiling.cpp (profile_evolution /
    profile_table, profiling.cpp:8-63) compiles UNMODIFIED against
    include/rsfgpu.hpp (namespace swap -Drsf=rsfgpu) and links to librsfg.so;
    its table lists the reference's 14 stage names in order."""
    out = subprocess.run([str(_profcheck()), "table"], check=True, capture_output=True, text=True).stdout
    assert list(_rows(out)) == STAGES


@pytest.mark.gpu
def test_reference_profile_evolution_on_gpu():
    """profile_evolution (reference code) timing our kernels: the rows that
    carry kernel time are non-zero, the stages fused into them read 0."""
    import paper_2404_02813_b200 as rsf
    out = subprocess.run([str(_profcheck()), "run", "64"], check=True, capture_output=True, text=True).stdout
    rows = _rows(out)
    assert list(rows) == STAGES
    carrier = rsf.KernelProfile.carrier()
    for i, name in enumerate(STAGES):
        if carrier[i] != i:
            assert rows[name][0] == 0.0, (name, rows[name])
    assert rows["K*H-I"][0] > 0 and rows["R-combine"][0] > 0
    assert abs(sum(v[1] for v in rows.values()) - 100.0) < 0.1
