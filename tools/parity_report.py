"""Parity margins of the CUDA path vs the oracle (prints numbers; tests assert).

    python tools/parity_report.py [N] > profiles/rNN_parity.txt

P1 (one step) / P2 (ten steps) for every kernel specialisation class --
sigma1 in {1, 3, 4, 4.5, 5, 5.5, 6} (R 3..18: xy2 32- and 64-row tiles, zst4
32x8 and 32x4 tiles, stored-Heaviside mode at R <= 9), sigma2 > 0, the
generic runtime-tap path (sigma1 = 7, R = 21), the LDG fallbacks (nx % 4 !=
0), fields 2 and 4 -- then cfg 1 (N^3 x 100 iterations) mask statistics.
Absolute and relative max |dphi| (P1 absolute 1e-4)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2404_02813_b200 as rsf  # noqa: E402
from _inputs import case  # noqa: E402
from _oracle import Oracle, params  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(1.0, np.abs(b))))


def absd(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)))


def main():
    o = Oracle()
    shapes = {"96x72x40": (96, 72, 40), "70x34x30 (nx%4!=0: LDG fallback)": (70, 34, 30)}
    for sname, shp in shapes.items():
        img, phi, gt = case(*shp, n_branches=4)
        sig = [(1.0, 0.0), (3.0, 0.0), (2.0, 1.5), (4.0, 0.0), (4.5, 0.0), (5.0, 0.0), (5.5, 0.0), (6.0, 0.0),
               (7.0, 0.0)] if sname.startswith("96") else [(3.0, 0.0), (6.0, 0.0)]
        for s1, s2 in sig:
            op = params(sigma1=s1, sigma2=s2)
            st_o = o.init(np.array(img), op)
            r1, _, _ = o.step(np.array(phi), np.array(img), op, st_o)
            r10 = np.array(phi)
            for _ in range(10):
                r10, _, _ = o.step(r10, np.array(img), op, st_o)
            for fields in (2, 4):
                st = rsf.init_evolution(phi, img, rsf.RsfParams(sigma1=s1, sigma2=s2), fields=fields)
                st.step()
                a1, e1 = absd(st.phi, r1), rel(st.phi, r1)
                st.run(9)
                a10, e10 = absd(st.phi, r10), rel(st.phi, r10)
                print(f"{sname} sigma1={s1} sigma2={s2} fields={fields}: P1 abs {a1:.2e} rel {e1:.2e} (tol 1e-4)  "
                      f"P2 abs {a10:.2e} rel {e10:.2e} (tol 1e-3)", flush=True)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    img, phi, gt = case(n, n, n, n_branches=max(1, int(12 * (n / 128) ** 2)))
    t0 = time.time()
    ref = o.evolve(np.array(phi), np.array(img), params(sigma1=3.0, max_iters=100))
    t_o = time.time() - t0
    for fields in (2, 4):
        got = rsf.evolve(phi, img, rsf.RsfParams(sigma1=3.0, max_iters=100), fields=fields)
        mm = int(np.count_nonzero((got < 0) != (ref < 0)))
        close = float(np.mean(np.abs(got.astype(np.float64) - ref) <= 1e-3 + 1e-4 * np.abs(ref)))
        print(f"cfg1 {n}^3 100 it fields={fields}: mask mismatch {mm} ({mm / phi.size:.2e}), "
              f"dice(gpu,ref)={rsf.dice(got < 0, ref < 0):.6f}, close-frac {close:.5f}, "
              f"dice vs gt: gpu {rsf.dice(got < 0, gt):.4f} ref {rsf.dice(ref < 0, gt):.4f}, "
              f"max|d| {np.abs(got - ref).max():.3e}  (oracle {t_o:.1f}s)")


if __name__ == "__main__":
    main()
