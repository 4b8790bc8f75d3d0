"""P4: z-slab decomposition is bitwise identical to the monolithic volume."""
import numpy as np
import pytest

from _inputs import case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("fields", [2, 4])
def test_slabs_bitwise(parts, fields):
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import SlabSet
    img, phi, _ = case(40, 36, 32)
    p = rsf.RsfParams(sigma1=3.0)
    st = rsf.init_evolution(phi, img, p, fields=fields)
    ss = SlabSet(np.array(phi), np.array(img), p, parts, fields=fields, linked=False)  # exchange mode
    for _ in range(6):
        st.step()
        ss.step()
    mono = st.phi
    assert ss.sign_changes() >= 0
    assert np.array_equal(ss.phi(), mono)


@pytest.mark.parametrize("parts", [2, 3])
def test_slabs_bitwise_interior_tiles(parts):
    """Shape with interior tiles and several CTAs per slab (zst4 fast path)."""
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import SlabSet
    img, phi, _ = case(96, 28, 80)
    p = rsf.RsfParams(sigma1=3.0)
    st = rsf.init_evolution(phi, img, p)
    ss = SlabSet(np.array(phi), np.array(img), p, parts)
    for _ in range(4):
        st.step()
        ss.step()
    assert np.array_equal(ss.phi(), st.phi)


def test_slab_generic_radius_bitwise():
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import SlabSet
    img, phi, _ = case(40, 36, 60)
    p = rsf.RsfParams(sigma1=9.0)  # R = 27: generic runtime-tap path (specialised kernels stop at R = 24)
    st = rsf.init_evolution(phi, img, p)
    ss = SlabSet(np.array(phi), np.array(img), p, 2)
    for _ in range(3):
        st.step()
        ss.step()
    assert np.array_equal(ss.phi(), st.phi)


@pytest.mark.parametrize("parts,fields,sigma1", [(2, 2, 3.0), (3, 4, 3.0), (4, 2, 2.0), (2, 2, 7.0), (2, 2, 9.0)])
def test_linked_slabs_bitwise(parts, fields, sigma1):
    """Peer halo links (rsfg_slab_link / step_linked): pushes of the boundary
    planes + flag waits, no host synchronisation, several slabs on one GPU."""
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import SlabSet
    img, phi, _ = case(96, 28, 80)
    p = rsf.RsfParams(sigma1=sigma1)
    st = rsf.init_evolution(phi, img, p, fields=fields)
    ss = SlabSet(np.array(phi), np.array(img), p, parts, fields=fields, linked=True)
    for _ in range(7):
        st.step()
        ss.step()
    assert np.array_equal(ss.phi(), st.phi)
    ss.close()


@pytest.mark.parametrize("n", [2, 3])
def test_evolve_multi_bitwise(n):
    """rsfg_evolve_multi (the C-ABI multi-GPU entry; one device repeated here)."""
    import paper_2404_02813_b200 as rsf
    img, phi, _ = case(64, 48, 40, n_branches=4)
    p = rsf.RsfParams(sigma1=3.0, max_iters=30)
    rep = rsf._lib.rsfg_report()
    got = rsf.evolve_multi(phi, img, p, [0] * n, report=rep)
    assert np.array_equal(got, rsf.evolve(phi, img, p))
    assert rep.iterations == 30 and rep.gpu_launches > 0
    # StopCheck (rsf.cpp:379-381): called with the gathered volume every 10 steps, stop at 20
    seen = []

    def stop(phi_now, it):
        seen.append((it, phi_now.shape))
        return it >= 20

    got_s = rsf.evolve_multi(phi, img, p, [0] * n, stop, 10)
    assert seen == [(10, phi.shape), (20, phi.shape)]
    assert np.array_equal(got_s, rsf.evolve(phi, img, rsf.RsfParams(sigma1=3.0, max_iters=20)))


def test_evolve_multi_blowup_and_thin():
    import paper_2404_02813_b200 as rsf
    img, phi, _ = case(40, 36, 32)
    bad = np.array(phi)
    bad[20, 5, 7] = np.nan  # spreads to z = 18 through the normals within the first step
    p = rsf.RsfParams(sigma1=2.0, max_iters=5)
    with pytest.raises(rsf.BlowupError) as one:
        rsf.evolve(bad, img, p)
    assert "iteration 1" in str(one.value)
    want = str(one.value).split("] ", 1)[1]
    with pytest.raises(rsf.BlowupError) as multi:  # same first voxel as one device (global min index)
        rsf.evolve_multi(bad, img, p, [0, 0])
    assert str(multi.value).split("] ", 1)[1] == want
    with pytest.raises(rsf.ShapeError):
        rsf.evolve_multi(phi, img, rsf.RsfParams(sigma1=3.0, max_iters=5), [0] * 8)


def test_thin_slab_rejected():
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import plan_slabs
    with pytest.raises(ValueError):
        plan_slabs(16, 4, 9)
