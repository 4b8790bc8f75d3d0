"""Throughput vs Gaussian radius at 512^3 (cfg-2 volume, threshold phi0):
which kernel path each sigma takes (variant flags: 1 xy2, 2 zst4, 4 stored
Heaviside; 0 = the generic runtime-tap path) and voxel-iter/s from CUDA
events around K steps.  One JSON line per sigma.

    python tools/radius_sweep.py [--steps K] [sigma ...]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200.api import check, options  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sigmas", nargs="*", type=float, default=[3.0, 4.0, 4.5, 5.0, 5.5, 6.0, 7.0])
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch
    n = 512
    img, _ = rsf.phantom_device(n, n, n, n_branches=192, noise_sigma=20.0, with_gt=False)
    phi = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    lib = rsf.load()
    for s in a.sigmas:
        h = C.c_void_p()
        cp, opt = rsf.RsfParams(sigma1=s).to_c(), options(2, 0, 64)
        check(lib.rsfg_state_create_device(C.byref(h), phi.data_ptr(), img.data_ptr(), n, n, n, C.byref(cp),
                                           C.byref(opt)))
        rep = rsf._lib.rsfg_report()
        check(lib.rsfg_state_run(h, 3, C.byref(rep)))
        sp = C.c_void_p()
        check(lib.rsfg_state_stream(h, C.byref(sp)))
        stream = torch.cuda.ExternalStream(sp.value)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        check(lib.rsfg_state_run(h, a.steps, C.byref(rep)))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        fl = C.c_int32()
        check(lib.rsfg_state_variant(h, C.byref(fl), None, None))
        prof = (C.c_double * 2)()
        check(lib.rsfg_state_profile(h, 5, prof))
        r = (len(rsf.gaussian_kernel(s)) - 1) // 2
        print(json.dumps({"sigma1": s, "radius": r, "variant_flags": fl.value, "ms_per_step": round(ms, 3),
                          "kernel_ms": {"xy": round(prof[0], 3), "zst": round(prof[1], 3)},
                          "voxel_iter_per_s": n ** 3 / (ms * 1e-3)}), flush=True)
        lib.rsfg_state_destroy(h)


if __name__ == "__main__":
    main()
