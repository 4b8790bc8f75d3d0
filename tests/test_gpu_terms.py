"""Term-level APIs and the reference-shaped stepping surface on the GPU:

* region_intensities / directional_forces (rsf.hpp:39-50, rsf.cpp:235-291)
  against the oracle, the reference and the reference-generated golden
  vectors (tests/golden/terms_golden.npz);
* evolve_step(state, I, p, ws, profile): KernelProfile rows (rsf.cpp:228-233)
  filled from per-kernel CUDA events, and per-step parameters (p is passed on
  every call in the reference) -- against the oracle stepping with the same p.
"""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TERMS = Path(__file__).resolve().parent / "golden" / "terms_golden.npz"
GOLD = Path(__file__).resolve().parent / "golden" / "rsf_golden.npz"


def _rel(a, b, scale=1.0):
    return float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(scale, np.abs(b))))


def test_region_intensities_golden():
    import paper_2404_02813_b200 as rsf
    g, t = dict(np.load(GOLD)), dict(np.load(TERMS))
    for tag, s1 in {"s3": 3.0, "s15": 1.5}.items():
        rp, rm = rsf.region_intensities(g["img"], g["phi0"], s1, 1.0)
        # fp32 Heaviside + fp32 separable passes vs the reference's f64 ones:
        # relative 1e-4 of the intensity (r lies in [min I, max I])
        assert _rel(rp, t[f"rplus_{tag}"]) <= 1e-4, tag
        assert _rel(rm, t[f"rminus_{tag}"]) <= 1e-4, tag


@pytest.mark.parametrize("shape,s1,eps", [((40, 36, 28), 3.0, 1.0), ((33, 17, 9), 2.0, 0.5), ((24, 20, 16), 0.0, 1.0),
                                          ((64, 48, 40), 6.0, 1.0)])
def test_region_intensities_vs_oracle(oracle, shape, s1, eps):
    import paper_2404_02813_b200 as rsf
    from _inputs import random_case
    img, phi = random_case(*shape, seed=5)
    rp, rm = rsf.region_intensities(img, phi, s1, eps)
    wp, wm = oracle.region_intensities(img, phi, s1, eps)
    assert _rel(rp, wp) <= 1e-4 and _rel(rm, wm) <= 1e-4
    assert rp.min() >= img.min() and rp.max() <= img.max()  # clamp (rsf.cpp:259)


def test_region_intensities_errors():
    import paper_2404_02813_b200 as rsf
    img = np.ones((4, 5, 6), np.float32)
    with pytest.raises(rsf.ParamError, match="epsilon must be > 0"):
        rsf.region_intensities(img, img, 1.0, 0.0)
    with pytest.raises(rsf.ParamError, match="denom_floor must be > 0"):
        rsf.region_intensities(img, img, 1.0, 1.0, 0.0)
    with pytest.raises(rsf.ShapeError):
        rsf.region_intensities(img, np.ones((4, 5, 7), np.float32), 1.0, 1.0)


def test_directional_forces_bitwise(ref):
    """f64 pointwise with the reference's rounding points: bit-exact with the
    golden vectors and with the reference on random inputs."""
    import paper_2404_02813_b200 as rsf
    g, t = dict(np.load(GOLD)), dict(np.load(TERMS))
    Fp, Fm = rsf.directional_forces(g["img"], t["rplus_s3"], t["rminus_s3"], t["KI_s2_15"], t["KI2_s2_15"])
    assert np.array_equal(Fp, t["Fplus"]) and np.array_equal(Fm, t["Fminus"])
    rng = np.random.default_rng(3)
    a = [rng.uniform(0, 255, (20, 30, 40)).astype(np.float32) for _ in range(4)]
    a[3] = a[3] * a[3]
    got = rsf.directional_forces(a[0], a[0], a[1], a[2], a[3])
    want = ref.directional_forces(a[0], a[0], a[1], a[2], a[3])
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_kernel_profile_rows_and_parity(oracle):
    """evolve_step(..., &profile) gives the same phi as a plain step and books
    each kernel's CUDA-event time on its carrier row only."""
    import paper_2404_02813_b200 as rsf
    from _inputs import case
    from _oracle import params
    img, phi0, _ = case(64, 48, 40, n_branches=4)
    p = rsf.RsfParams(sigma1=3.0)
    a = rsf.init_evolution(phi0, img, p)
    b = rsf.init_evolution(phi0, img, p)
    prof, ws = rsf.KernelProfile(), rsf.EvolveWorkspace()
    for _ in range(3):
        fa = rsf.evolve_step(a, img, p, ws, prof)
        fb = b.step()
        assert fa == fb
    assert np.array_equal(a.phi, b.phi)
    assert prof.iterations == 3
    names, carrier = rsf.KernelProfile.names(), rsf.KernelProfile.carrier()
    assert names[2] == "K*H-I" and names[11] == "R-combine" and len(names) == 14
    for i, s in enumerate(prof.seconds):
        if carrier[i] != i:
            assert s == 0.0, names[i]
    assert prof.seconds[2] > 0 and prof.seconds[11] > 0
    # rsfg_evolve with profile_stages: same rows, same result as without
    prof2 = rsf.KernelProfile()
    e1 = rsf.evolve(phi0, img, rsf.RsfParams(sigma1=3.0, max_iters=4), profile=prof2)
    e2 = rsf.evolve(phi0, img, rsf.RsfParams(sigma1=3.0, max_iters=4))
    assert np.array_equal(e1, e2) and prof2.iterations == 4 and prof2.seconds[11] > 0
    ref = oracle.step(phi0.copy(), img, params(sigma1=3.0))[0]
    c = rsf.init_evolution(phi0, img, p)
    c.step(rsf.KernelProfile())
    assert float(np.abs(c.phi.astype(np.float64) - ref).max()) <= 1e-4


def test_evolve_step_takes_p_each_call(oracle):
    """The reference's evolve_step reads epsilon/alpha/beta/dt/floors from
    the p of THAT call (rsf.cpp:324-357); sigma stays the state's (st.k1)."""
    import paper_2404_02813_b200 as rsf
    from _inputs import case
    from _oracle import params
    img, phi0, _ = case(48, 40, 36, n_branches=3)
    st = rsf.init_evolution(phi0, img, rsf.RsfParams(sigma1=2.0))
    steps = [dict(dt=0.06), dict(dt=0.03, alpha=40.0), dict(epsilon=1.5, beta=0.2)]
    ostat = oracle.init(img, params(sigma1=2.0))
    want = phi0.copy()
    for kw in steps:
        rsf.evolve_step(st, img, rsf.RsfParams(sigma1=2.0, **kw), rsf.EvolveWorkspace())
        want, _, _ = oracle.step(want, img, params(sigma1=2.0, **kw), ostat)
    got = st.phi
    assert float(np.abs(got.astype(np.float64) - want).max()) <= 1e-3
    with pytest.raises(rsf.ShapeError):
        rsf.evolve_step(st, np.zeros((2, 2, 2), np.float32), rsf.RsfParams(sigma1=2.0), rsf.EvolveWorkspace())
