"""Volume I/O to the device and overlap metrics against the
compiled reference's read_volume / dice (volume_io.cpp:24-137,
validation.cpp:41-52)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write(tmp_path, name, arr, dtype, extra=""):
    raw = tmp_path / f"{name}.raw"
    arr.astype({"u8": np.uint8, "u16": "<u2", "f32": "<f4"}[dtype]).tofile(raw)
    nz, ny, nx = arr.shape
    hdr = tmp_path / f"{name}.vmh"
    hdr.write_text(f"# test volume\ndims: {nx} {ny} {nz}\nspacing: 1 1 2\ndtype: {dtype}\ndata: {raw.name}\n{extra}")
    return hdr


@pytest.mark.parametrize("dtype", ["u8", "u16", "f32"])
@pytest.mark.parametrize("shape", [(7, 9, 11), (64, 130, 257)])
def test_read_volume_bitwise(ref, tmp_path, dtype, shape):
    import paper_2404_02813_b200 as rsf
    rng = np.random.default_rng(len(shape) + shape[0])
    hi = {"u8": 255, "u16": 65535, "f32": 1000}[dtype]
    arr = rng.integers(0, hi + 1, shape) if dtype != "f32" else rng.normal(0, 100, shape)
    hdr = _write(tmp_path, "v", arr, dtype)
    got, spacing, rng_g, moved = rsf.read_volume_device(hdr)
    want, rng_r = ref.read_volume(hdr)
    assert np.array_equal(got.cpu().numpy(), want)
    assert rng_g == rng_r
    assert spacing == (1.0, 1.0, 2.0)
    assert moved == arr.size * {"u8": 1, "u16": 2, "f32": 4}[dtype]  # stored width over PCIe


def test_read_volume_header_range_and_errors(tmp_path):
    import paper_2404_02813_b200 as rsf
    arr = np.arange(60).reshape(3, 4, 5)
    hdr = _write(tmp_path, "r", arr, "u8", "range: -1 300\n")
    _, _, rng, _ = rsf.read_volume_device(hdr)
    assert rng == (-1.0, 300.0)
    bad = tmp_path / "bad.vmh"
    bad.write_text("dims: 5 4 3\ndtype: u8\ndata: r.raw\ncolour: red\n")
    with pytest.raises(rsf.VolumeIOError, match="unknown header key 'colour'"):
        rsf.read_volume_device(bad)
    short = _write(tmp_path, "s", arr, "u8")
    short.write_text(short.read_text().replace("dims: 5 4 3", "dims: 5 4 4"))
    with pytest.raises(rsf.VolumeIOError, match="payload size mismatch"):
        rsf.read_volume_device(short)
    with pytest.raises(rsf.VolumeIOError, match="cannot open volume header"):
        rsf.read_volume_device(tmp_path / "missing.vmh")


def test_write_then_read_roundtrip(ref, tmp_path):
    import torch
    import paper_2404_02813_b200 as rsf
    v = torch.randn(5, 6, 7, device="cuda") * 10
    hdr = tmp_path / "w.vmh"
    rsf.write_volume_device(hdr, v, spacing=(0.5, 0.5, 1.0))
    want, _ = ref.read_volume(hdr)
    assert np.array_equal(want, v.cpu().numpy())
    got, spacing, _, _ = rsf.read_volume_device(hdr)
    assert torch.equal(got, v) and spacing == (0.5, 0.5, 1.0)


@pytest.mark.parametrize("n", [1000, 513 * 517])
def test_overlap_metrics(ref, n):
    import torch
    import paper_2404_02813_b200 as rsf
    rng = np.random.default_rng(n)
    a = (rng.random((1, 1, n)) < 0.3).astype(np.float32)
    b = (rng.random((1, 1, n)) < 0.4).astype(np.float32)
    d, j = rsf.overlap_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert d == ref.dice(a, b)
    both = float(np.sum((a > 0.5) & (b > 0.5)))
    assert j == both / float(np.sum((a > 0.5) | (b > 0.5)))
    e = torch.zeros(10, device="cuda")
    assert rsf.overlap_device(e, e) == (1.0, 1.0)
