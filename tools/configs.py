"""Throughput at every SURVEY.md 8(d) configuration that fits one B200
(cfg 2-5; cfg 1 is the CPU-parity case), device-resident inputs from the
device phantom (bit-exact with the reference generator), phi0 = threshold
initialisation, CUDA events around K steps.  One JSON line per config.

    python tools/configs.py [cfg2 cfg3 ...] [--steps K] [--warmup W]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200 import _lib as L  # noqa: E402
from paper_2404_02813_b200.api import check, options  # noqa: E402

CFGS = {
    "cfg2": dict(shape=(512, 512, 512), sigma1=3.0, spec=dict(n_branches=192, noise_sigma=20.0)),
    "cfg3": dict(shape=(512, 512, 512), sigma1=6.0, spec=dict(n_branches=192, noise_sigma=20.0)),
    "cfg4": dict(shape=(1024, 1024, 1024), sigma1=3.0,
                 spec=dict(n_branches=768, axial_blur_sigma=2.0, noise_sigma=25.0, contrast_axis=3,
                           contrast_lo=0.6, contrast_hi=1.0)),
    "cfg5": dict(shape=(2048, 2048, 1024), sigma1=4.0, spec=dict(n_branches=3072, radius_max=5.0, noise_sigma=15.0)),
}


def run(name, steps, warmup):
    import torch
    c = CFGS[name]
    nx, ny, nz = c["shape"]
    img, _ = rsf.phantom_device(nx, ny, nz, with_gt=False, **c["spec"])
    phi = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    lib = rsf.load()
    p = rsf.RsfParams(sigma1=c["sigma1"], sigma2=0.0)
    cp, opt = p.to_c(), options(2, 0, 64)
    h = C.c_void_p()
    check(lib.rsfg_state_create_device(C.byref(h), phi.data_ptr(), img.data_ptr(), nx, ny, nz, C.byref(cp),
                                       C.byref(opt)))
    del img, phi
    torch.cuda.empty_cache()
    sp = C.c_void_p()
    check(lib.rsfg_state_stream(h, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value)
    rep = L.rsfg_report()
    check(lib.rsfg_state_run(h, warmup, C.byref(rep)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    check(lib.rsfg_state_run(h, steps, C.byref(rep)))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    prof = (C.c_double * 2)()
    check(lib.rsfg_state_profile(h, 5, prof))
    lib.rsfg_state_destroy(h)
    torch.cuda.empty_cache()
    n = nx * ny * nz
    return {"config": name, "shape": [nx, ny, nz], "sigma1": c["sigma1"], "radius": len(rsf.gaussian_kernel(c["sigma1"])) // 2,
            "voxel_iter_per_s": n / (ms * 1e-3), "ms_per_step": ms, "kernel_ms": {"xy": prof[0], "zst": prof[1]},
            "hbm_GBps_at_40B_per_voxel": 40 * n / (ms * 1e-3) / 1e9, "steps": steps, "warmup": warmup,
            "data": "device phantom (bit-exact with the reference generator), threshold phi0"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=list(CFGS))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    for name in a.configs:
        print(json.dumps(run(name, a.steps, a.warmup)), flush=True)


if __name__ == "__main__":
    main()
