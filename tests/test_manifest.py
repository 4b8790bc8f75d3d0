"""Tile spill layout (reference tiling.cpp:195-321): tile_file_name and the
manifest text written by save_manifest are byte-identical to the
reference's; load_manifest reads the reference's files back with its error
messages.  Host-only logic of librsfg.so (no GPU)."""
import pytest


@pytest.mark.parametrize("shape,tile,s1,s2", [((100, 80, 60), (48, 40, 30), 2.0, 1.0),
                                              ((64, 64, 64), (32, 32, 32), 3.0, 0.0),
                                              ((40, 30, 20), (40, 30, 20), 1.0, 0.0)])
def test_manifest_bytes_match_reference(ref, tmp_path, shape, tile, s1, s2):
    import paper_2404_02813_b200 as rsf
    tiles, curtain = rsf.plan_tiles(shape, tile, s1, s2)
    rsf.save_manifest(tmp_path / "ours.manifest", shape, tile, curtain, tiles)
    ref.save_manifest(tmp_path / "ref.manifest", shape, tile, s1, s2)
    assert (tmp_path / "ours.manifest").read_bytes() == (tmp_path / "ref.manifest").read_bytes()
    d, ts, c, back = rsf.load_manifest(tmp_path / "ref.manifest")
    assert (d, ts, c, back) == (tuple(shape), tuple(tile), curtain, tiles)


def test_tile_file_name():
    import paper_2404_02813_b200 as rsf
    tiles, _ = rsf.plan_tiles((100, 80, 60), (48, 40, 30), 2.0)
    names = [rsf.tile_file_name(t) for t in tiles]
    assert names[0] == "tile_z00_y00_x00.vmh" and names[-1] == "tile_z01_y01_x02.vmh"
    assert len(set(names)) == len(names)


@pytest.mark.parametrize("text,msg", [
    ("dims: 8 8 8\ncolour: red\n", "unknown manifest key 'colour:'"),
    ("dims: 8 8\ntile: 0 0 0 0 0 0 8 8 8 0 0 0 8 8 8\n", "garbled manifest line"),
    ("dims: 8 8 8\ntile_size: 8 8 8\ncurtain: 3\n", "manifest has no tiles"),
])
def test_load_manifest_errors(tmp_path, text, msg):
    import paper_2404_02813_b200 as rsf
    p = tmp_path / "bad.manifest"
    p.write_text(text)
    with pytest.raises(rsf.VolumeIOError, match=msg):
        rsf.load_manifest(p)
    with pytest.raises(rsf.VolumeIOError, match="cannot open manifest"):
        rsf.load_manifest(tmp_path / "missing.manifest")
