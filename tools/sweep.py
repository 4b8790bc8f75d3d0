"""Per-kernel CUDA-event timings over a few configurations (development aid)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    t0 = time.time()
    img, _ = rsf.phantom(n, n, n, n_branches=max(1, int(12 * (n / 128) ** 2)), noise_sigma=20.0)
    phi0 = rsf.threshold_phi0(img)
    print(f"phantom {n}^3 in {time.time() - t0:.1f}s", flush=True)
    for sigma in (3.0, 4.0, 5.0, 6.0):
        for fields in (2, 4):
            st = rsf.init_evolution(phi0, img, rsf.RsfParams(sigma1=sigma), fields=fields)
            st.run(3)
            prof = st.profile(10)
            tot = sum(prof.values())
            print(f"n={n} sigma={sigma} fields={fields}: " + " ".join(f"{k}={v:.3f}ms" for k, v in prof.items())
                  + f" step={tot:.3f}ms -> {img.size / tot * 1e3:.3e} voxel-iter/s", flush=True)
            st.close()


if __name__ == "__main__":
    main()
