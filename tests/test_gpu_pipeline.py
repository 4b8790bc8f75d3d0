"""Curtain tiling (reference tiling.cpp:14-275).

merge_phi on the device is bit-exact with the reference's for identical tile
fields (every mode).  run_pipeline composes the device seeding, distance and
evolution per tile; against the reference's run_pipeline it is held to the
full-run mask statistics of P3."""
import numpy as np
import pytest

from _inputs import case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["linear", "minimum", "maximum", "average"])
@pytest.mark.parametrize("shape,tile,sigma", [((70, 52, 41), (32, 24, 20), 2.0), ((64, 64, 64), (32, 32, 32), 3.0),
                                              ((40, 30, 20), (40, 30, 20), 1.0)])
def test_merge_phi_bitwise(ref, mode, shape, tile, sigma):
    import torch
    import paper_2404_02813_b200 as rsf
    tiles, curtain = rsf.plan_tiles(shape, tile, sigma)
    rng = np.random.default_rng(sum(shape))
    fields = [rng.normal(0, 5, t["pad_extent"][::-1]).astype(np.float32) for t in tiles]
    got = rsf.merge_phi_device([torch.from_numpy(f).cuda() for f in fields], shape, tile, curtain, mode).cpu().numpy()
    want = ref.merge_phi(fields, shape, tile, sigma, 0.0, rsf.api.MERGE_MODES[mode])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("global_seeding", [False, True])
def test_run_pipeline_vs_reference(ref, global_seeding):
    from _oracle import params
    import paper_2404_02813_b200 as rsf
    img, _, gt = case(96, 80, 64, n_branches=8, init="threshold")
    img = np.ascontiguousarray(img)
    p = rsf.RsfParams(sigma1=2.0, max_iters=20)
    phi_g, mask_g, warn_g = rsf.run_pipeline(img, p, (48, 40, 32), global_seeding=global_seeding)
    phi_r, mask_r, nw_r = ref.run_pipeline(img, params(sigma1=2.0, max_iters=20), (48, 40, 32),
                                           global_seeding=global_seeding)
    assert len(warn_g) == nw_r
    assert np.array_equal(mask_g, (phi_g < 0).astype(np.float32))
    mism = int(np.count_nonzero(mask_g != mask_r))
    assert mism <= max(4, 1e-4 * img.size), mism
    assert rsf.dice(mask_g, mask_r) >= 0.999
    assert abs(rsf.dice(mask_g, gt) - rsf.dice(mask_r, gt)) < 1e-3


def test_plan_tiles_errors():
    import paper_2404_02813_b200 as rsf
    with pytest.raises(rsf.ParamError, match="too small for curtain 9"):
        rsf.plan_tiles((64, 64, 64), (16, 16, 16), 3.0)
    with pytest.raises(rsf.ShapeError, match="bad volume dims"):
        rsf.plan_tiles((0, 64, 64), (32, 32, 32), 1.0)


def test_run_pipeline_spill_and_merge_from_dir(ref, tmp_path):
    """PipelineOptions::spill_dir (tiling.cpp:256-263) and merge_from_dir
    (tiling.cpp:323-332): every tile lands under its tile_file_name plus the
    reference's manifest; the reference's own load_manifest + merge_from_dir
    over our spill directory, and ours on the device, both reproduce the
    returned phi bit for bit."""
    import paper_2404_02813_b200 as rsf
    img, _, _ = case(80, 64, 48, n_branches=6, init="threshold")
    img = np.ascontiguousarray(img)
    shape, tile = (80, 64, 48), (40, 32, 24)
    p = rsf.RsfParams(sigma1=2.0, max_iters=10)
    for mode in ("linear", "average"):
        d = tmp_path / mode
        d.mkdir()
        phi, mask, _ = rsf.run_pipeline(img, p, tile, merge=mode, spill_dir=d)
        tiles, curtain = rsf.plan_tiles(shape, tile, 2.0)
        assert sorted(f.name for f in d.glob("*.vmh")) == sorted(rsf.tile_file_name(t) for t in tiles)
        ref.save_manifest(tmp_path / "ref.manifest", shape, tile, 2.0)
        assert (d / "layout.manifest").read_bytes() == (tmp_path / "ref.manifest").read_bytes()
        got = rsf.merge_from_dir_device(d, shape, tile, curtain, tiles, mode).cpu().numpy()
        assert np.array_equal(got, phi)
        want = ref.merge_from_dir(d, d / "layout.manifest", shape, rsf.api.MERGE_MODES[mode])
        assert np.array_equal(want, phi)
    with pytest.raises(rsf.VolumeIOError, match="cannot write"):
        rsf.run_pipeline(img, p, tile, spill_dir=tmp_path / "no" / "such" / "dir")
