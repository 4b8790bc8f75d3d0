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
    ss = SlabSet(np.array(phi), np.array(img), p, parts, fields=fields)
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
    img, phi, _ = case(40, 36, 48)
    p = rsf.RsfParams(sigma1=7.0)  # R = 21: generic path
    st = rsf.init_evolution(phi, img, p)
    ss = SlabSet(np.array(phi), np.array(img), p, 2)
    for _ in range(3):
        st.step()
        ss.step()
    assert np.array_equal(ss.phi(), st.phi)


def test_thin_slab_rejected():
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import plan_slabs
    with pytest.raises(ValueError):
        plan_slabs(16, 4, 9)
