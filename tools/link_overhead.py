"""Overhead of the peer-link slab path on ONE GPU: rsfg_evolve (one volume)
vs rsfg_evolve_multi with the volume split into 2 / 4 linked z-slabs on the
same device (512^3, sigma1 = 3, 100 iterations; loop phase only).  On one GPU
the slabs share the SMs, so the difference is the decomposition's own cost:
kernel 1 on the R halo planes per face, the pushes, the flag waits and the
extra launches."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200 import _lib as L  # noqa: E402


def main():
    n = 512
    img, _ = rsf.phantom(n, n, n, n_branches=192, noise_sigma=20.0)
    phi0 = rsf.threshold_phi0(img)
    p = rsf.RsfParams(sigma1=3.0, max_iters=100)
    out = {}
    for name, devs in (("1 volume", None), ("2 slabs", [0, 0]), ("4 slabs", [0, 0, 0, 0])):
        best = None
        for _ in range(2):
            rep = L.rsfg_report()
            if devs is None:
                rsf.evolve(phi0, img, p, report=rep)
            else:
                rsf.evolve_multi(phi0, img, p, devs, report=rep)
            best = rep.ms_loop if best is None else min(best, rep.ms_loop)
        out[name] = round(best / 100, 4)
        print(json.dumps({"config": name, "ms_per_step": out[name]}), flush=True)
    print(json.dumps({"overhead_2_slabs": round(out["2 slabs"] / out["1 volume"] - 1, 4),
                      "overhead_4_slabs": round(out["4 slabs"] / out["1 volume"] - 1, 4)}))


if __name__ == "__main__":
    main()
