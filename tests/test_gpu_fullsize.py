"""Checks at the benchmark's full size (512^3, cfg 2, sigma1 = 3; SURVEY.md
8(d)) -- the same kernels and tile/ring/prefetch schedules the bench runs:

* one step against the compiled reference's evolve_step (P1, max relative
  |dphi| <= 1e-4), from a smooth phi0 (a threshold phi0 has exactly-zero
  gradients where rounding-level differences turn into O(1) curvature changes,
  even between two builds of the reference);
* size-independent properties: run-to-run determinism, 4-slab decomposition ==
  monolithic and the stored-Heaviside mode == kernel 1's own Heaviside, bitwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 512


@pytest.fixture(scope="module")
def inputs():
    import paper_2404_02813_b200 as rsf
    img, _ = rsf.phantom_device(N, N, N, n_branches=192, noise_sigma=20.0, with_gt=False)
    img = img.cpu().numpy()
    # smooth phi0: distance to a lattice of balls (radius 20, spacing 128)
    c = (np.arange(N, dtype=np.float32) % 128) - 64.0
    zz, yy, xx = np.meshgrid(c, c, c, indexing="ij", copy=False)
    phi = np.sqrt(xx * xx + yy * yy + zz * zz, dtype=np.float32) - 20.0
    return img, np.ascontiguousarray(phi, np.float32)


@pytest.mark.parametrize("sigma1", [3.0, 6.0])  # cfg 2 (R = 9) and cfg 3 (R = 18)
def test_fullsize_one_step_vs_reference(ref, inputs, sigma1):
    import paper_2404_02813_b200 as rsf
    from _oracle import params
    img, phi = inputs
    ref.set_workers(0)
    rs = ref.state(phi, img, params(sigma1=sigma1))
    frac_r = rs.step()
    want = rs.phi()
    st = rsf.init_evolution(phi, img, rsf.RsfParams(sigma1=sigma1))
    frac_g = st.step()
    got = st.phi
    d = np.abs(got.astype(np.float64) - want)
    assert float(d.max()) <= 1e-4, float(d.max())  # SURVEY 8(c) P1, absolute
    err = d / np.maximum(1.0, np.abs(want))
    assert float(err.max()) <= 1e-4, float(err.max())
    assert abs(frac_g - frac_r) * img.size <= max(2, 1e-5 * img.size)


@pytest.mark.slow
def test_fullsize_threshold_P3(ref, inputs):
    """The bench's own workload (cfg 2: 512^3, sigma1 = 3, threshold phi0)
    over a bounded run: 10 iterations on the GPU and in the compiled
    reference (all host cores), mask statistics of SURVEY.md 8(c) P3.

    A threshold phi0 (+-2) has exactly-zero gradients, so the reference is
    ill-conditioned on it: perturbing phi0 by ONE ulp in half the voxels moves
    the reference's own phi by a median 0.1-0.2 after 1-10 iterations (256^3:
    1.7 % of voxels stay within 1e-3 + 1e-4|phi|, 124 mask voxels flip).  The
    phi-closeness gate of P3 (>= 99.5 % close) therefore cannot apply here;
    the GPU is held to the reference's own conditioning instead: its mask
    mismatch within max(1e-5 N, 2x) and its phi closeness at least that of
    the 1-ulp-perturbed reference run."""
    import paper_2404_02813_b200 as rsf
    from _oracle import params
    img, _ = inputs
    phi0 = rsf.threshold_phi0(img)
    iters = 10
    ref.set_workers(0)
    p = params(sigma1=3.0, max_iters=iters)
    want = ref.evolve(phi0, img, p)
    sel = np.random.default_rng(0).random(phi0.shape) < 0.5
    phi0_ulp = np.where(sel, np.nextafter(phi0, np.float32(0)), phi0).astype(np.float32)
    want_ulp = ref.evolve(phi0_ulp, img, p)
    got = rsf.evolve(phi0, img, rsf.RsfParams(sigma1=3.0, max_iters=iters))
    m_ref = want < 0
    mismatch = int(np.count_nonzero(m_ref != (got < 0)))
    mismatch_ulp = int(np.count_nonzero(m_ref != (want_ulp < 0)))
    assert mismatch <= max(1e-5 * img.size, 2 * mismatch_ulp), (mismatch, mismatch_ulp)
    assert rsf.dice(got < 0, m_ref) >= 0.9999

    def close(a):
        return float((np.abs(a.astype(np.float64) - want) <= 1e-3 + 1e-4 * np.abs(want)).mean())

    c_gpu, c_ulp = close(got), close(want_ulp)
    print(f"threshold P3 512^3 x {iters}: mask mismatch gpu {mismatch} / 1-ulp ref {mismatch_ulp}; "
          f"phi close frac gpu {c_gpu:.4f} / 1-ulp ref {c_ulp:.4f}")
    assert c_gpu >= c_ulp, (c_gpu, c_ulp)


def test_fullsize_properties(inputs, monkeypatch):
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import SlabSet
    img, phi = inputs
    p = rsf.RsfParams(sigma1=3.0, max_iters=3)
    a = rsf.evolve(phi, img, p)
    assert np.array_equal(a, rsf.evolve(phi, img, p))  # deterministic
    ss = SlabSet(phi, img, p, 4)
    for _ in range(3):
        ss.step()
    assert np.array_equal(ss.phi(), a)  # slabs == monolithic
    ss.close()
    monkeypatch.setenv("RSFG_HH", "0")
    assert np.array_equal(rsf.evolve(phi, img, p), a)  # stored Heaviside == recomputed
