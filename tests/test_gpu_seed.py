"""phi0 initialisation on the GPU against the compiled
reference's init_phi / detect_seeds (seeding.cpp:83-235).

Seeds: same (x, y, z) set in the same order; responses equal up to FMA
contraction differences in the f64 Hessian (<= 1e-6 relative).  Distance:
the reference stops its Gauss-Seidel sweeps once the largest change is below
1e-3; the device iterates the same Godunov update to its fixed point, so the
fields agree to the reference's own convergence tolerance."""
import numpy as np
import pytest

from _inputs import case

pytestmark = pytest.mark.gpu

DIST_TOL = 2e-3


@pytest.mark.parametrize("shape,nb", [((48, 40, 36), 4), ((96, 80, 64), 10), ((64, 64, 20), 6)])
@pytest.mark.parametrize("dark", [False, True])
def test_seeds_and_phi0_match_reference(ref, shape, nb, dark):
    import torch
    import paper_2404_02813_b200 as rsf
    img, _, _ = case(*shape, n_branches=nb, init="threshold")
    if dark:
        img = np.ascontiguousarray(255.0 - img, dtype=np.float32)
    xyz_r, resp_r = ref.detect_seeds(np.ascontiguousarray(img), dark=dark)
    phi_r, n_r = ref.init_phi(np.ascontiguousarray(img), dark=dark)
    phi_g, xyz_g, resp_g = rsf.init_phi_device(torch.from_numpy(np.array(img)).cuda(), dark=dark)
    assert n_r == len(xyz_r) == len(xyz_g)
    assert np.array_equal(xyz_g, xyz_r)
    np.testing.assert_allclose(resp_g, resp_r, rtol=1e-6, atol=0)
    d = np.abs(phi_g.cpu().numpy().astype(np.float64) - phi_r)
    assert float(d.max()) <= DIST_TOL, float(d.max())


def test_init_phi_errors():
    import torch
    import paper_2404_02813_b200 as rsf
    flat = torch.full((8, 16, 16), 50.0, device="cuda")
    with pytest.raises(rsf.ParamError, match="no seeds detected"):
        rsf.init_phi_device(flat)
    with pytest.raises(rsf.ParamError, match="sigma_b must be > 0"):
        rsf.init_phi_device(flat, sigma_b=0.0)
    with pytest.raises(rsf.ShapeError, match="at least 5x5"):
        rsf.init_phi_device(torch.zeros((4, 4, 4), device="cuda"))
