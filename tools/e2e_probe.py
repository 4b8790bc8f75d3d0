"""Where the e2e time of rsfg_evolve goes (512^3, cfg 2, 200 iterations):
pageable numpy buffers vs pinned (torch pin_memory) buffers, alternating,
wall clock per call and the report's CUDA-event phases (h2d, init, loop,
d2h); `outside` = wall - phases (workspace allocation/free, setup)."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200 import _lib as L  # noqa: E402
from paper_2404_02813_b200.api import check, options  # noqa: E402


def main():
    import torch
    n = 512
    img, _ = rsf.phantom(n, n, n, n_branches=192, noise_sigma=20.0)
    phi0 = rsf.threshold_phi0(img)
    lib = rsf.load()
    cp, opt = rsf.RsfParams(sigma1=3.0, max_iters=200).to_c(), options(2, 0, 25)
    bufs = {"pageable": (np.array(img), np.empty_like(phi0))}
    ti, tp = torch.from_numpy(img).pin_memory(), torch.empty_like(torch.from_numpy(phi0)).pin_memory()
    bufs["pinned"] = (ti.numpy(), tp.numpy())
    for rnd in range(3):
        for kind in (["pageable", "pinned"] if rnd % 2 == 0 else ["pinned", "pageable"]):
            im, ph = bufs[kind]
            np.copyto(ph, phi0)
            rep = L.rsfg_report()
            t0 = time.perf_counter()
            check(lib.rsfg_evolve(im.ctypes.data, ph.ctypes.data, n, n, n, C.byref(cp), C.byref(opt), L.STOP_FN(0),
                                  None, 0, C.byref(rep)))
            wall = 1e3 * (time.perf_counter() - t0)
            ph_ms = rep.ms_h2d + rep.ms_init + rep.ms_loop + rep.ms_d2h
            print(json.dumps({"round": rnd, "kind": kind, "wall_ms": round(wall, 1), "h2d": round(rep.ms_h2d, 1),
                              "init": round(rep.ms_init, 1), "loop": round(rep.ms_loop, 1),
                              "d2h": round(rep.ms_d2h, 1), "setup": round(rep.ms_setup, 1),
                              "outside_ms": round(wall - ph_ms, 1),
                              "voxel_iter_per_s": n ** 3 * 200 / (wall * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
