"""Locate the largest CUDA-vs-oracle deviations for one configuration."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2404_02813_b200 as rsf  # noqa: E402
from _inputs import case  # noqa: E402
from _oracle import Oracle, params  # noqa: E402

s1 = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
fields = int(sys.argv[2]) if len(sys.argv) > 2 else 4
img, phi, _ = case(40, 36, 32)
o = Oracle()
op = params(sigma1=s1)
E_ref = o.energy(np.array(phi), np.array(img), op)
st = rsf.init_evolution(phi, img, rsf.RsfParams(sigma1=s1), fields=fields)
E = st.energy()
d = np.abs(E.astype(np.float64) - E_ref)
idx = np.argsort(d.ravel())[::-1][:12]
print(f"sigma1={s1} fields={fields}: max|dE|={d.max():.3e} mean {d.mean():.3e}")
for i in idx:
    z, y, x = np.unravel_index(i, E.shape)
    print(f"  ({x},{y},{z}) E={E[z, y, x]:.6f} ref={E_ref[z, y, x]:.6f} phi={phi[z, y, x]:.4f} I={img[z, y, x]:.2f}")
bad = np.argwhere(d > 1e-3 * np.maximum(1, np.abs(E_ref)))
print("n bad:", len(bad), "z histogram:", np.bincount(bad[:, 0], minlength=32) if len(bad) else [])
