"""Small RSF cases for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck): every kernel variant the library ships -- xy2 (+ stored-Heaviside
xy2_hh), zst4 (fast and face/edge tiles, partial groups), the LDG fallbacks
(nx % 4 != 0), fields=4, a 32x4 large-radius zst4 tile (sigma 6), the generic
radius path (sigma 7), linked slabs (peer pushes + flag waits), the term APIs.
numpy + ctypes only (no torch), so the sanitizer sees just librsfg.so.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200.spmd import SlabSet  # noqa: E402


def case(nx, ny, nz, seed=0):
    rng = np.random.default_rng(seed)
    img = rng.uniform(0, 255, (nz, ny, nx)).astype(np.float32)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    r = np.sqrt((xx - nx / 2) ** 2 + (yy - ny / 2) ** 2 + (zz - nz / 2) ** 2)
    return img, (r - min(nx, ny, nz) / 4).astype(np.float32)


def main():
    if "--quick" in sys.argv:  # the pytest gate: stored-Heaviside xy2/zst4 (+ a face tile) and linked slabs
        img, phi = case(72, 40, 36)
        assert np.isfinite(rsf.evolve(phi, img, rsf.RsfParams(sigma1=3.0, max_iters=2))).all()
        img, phi = case(96, 28, 48)
        ss = SlabSet(phi, img, rsf.RsfParams(sigma1=2.0), 2, linked=True)
        ss.step()
        ss.step()
        ss.close()
        print("ok quick", flush=True)
        return
    runs = [((72, 40, 36), 3.0, 2), ((72, 40, 36), 3.0, 4), ((70, 34, 30), 3.0, 2),  # LDG fallback (nx % 4)
            ((96, 72, 40), 6.0, 2), ((64, 48, 40), 7.0, 2), ((64, 48, 60), 9.0, 2),  # R 21 specialised, R 27 generic
            ((68, 44, 42), 1.0, 2)]
    for shape, s1, fields in runs:
        img, phi = case(*shape)
        out = rsf.evolve(phi, img, rsf.RsfParams(sigma1=s1, max_iters=3), fields=fields)
        assert np.isfinite(out).all()
        print("ok", shape, s1, fields, flush=True)
    img, phi = case(96, 28, 80)
    p = rsf.RsfParams(sigma1=3.0)
    ss = SlabSet(phi, img, p, 3, linked=True)
    for _ in range(3):
        ss.step()
    ss.phi()
    ss.close()
    print("ok linked slabs", flush=True)
    st = rsf.init_evolution(phi, img, p)
    st.step(rsf.KernelProfile())
    st.energy()
    st.close()
    rp, rm = rsf.region_intensities(img, phi, 2.0, 1.0)
    rsf.directional_forces(img, rp, rm, img, img * img)
    print("ok terms", flush=True)


if __name__ == "__main__":
    main()
