"""Strong-scaling model for cfg 4 / cfg 5 measured on ONE B200 (the
north_star's >= 85 % at 8 GPUs on 2048 x 2048 x 1024).

Only one-GPU boxes are available, so the P-GPU run is decomposed into what
each rank does and each part is timed on the device:

  t1        one step of the whole volume (rsfg_state_run, CUDA events);
  tP[r]     one step of rank r's z-slab of the P-way split, alone: the owned
            planes plus kernel 1 on its R halo planes per interior face -- the
            real per-rank work (rsfg_slab_step_interior + step_finish, halos
            static);
  push      the per-step halo traffic of an interior rank: 2 faces x R planes,
            at the measured 770 GB/s NVLink peer bandwidth
            (B200_PROFILING.md), overlapped with the next step's interior
            kernel-1 work on the copy engine.

  efficiency(P) = t1 / (P * max_r tP[r])          (push fully overlapped)
  bound(P)      = t1 / (P * (max_r tP[r] + push)) (push not overlapped at all)

    python tools/scaling_model.py [cfg4|cfg5] [--steps K]
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
from paper_2404_02813_b200.spmd import halo_width, plan_slabs  # noqa: E402

CFGS = {
    "cfg4": dict(shape=(1024, 1024, 1024), sigma1=3.0,
                 spec=dict(n_branches=768, axial_blur_sigma=2.0, noise_sigma=25.0, contrast_axis=3,
                           contrast_lo=0.6, contrast_hi=1.0)),
    "cfg5": dict(shape=(2048, 2048, 1024), sigma1=4.0, spec=dict(n_branches=3072, radius_max=5.0, noise_sigma=15.0)),
}
PEER_GBS = 770.0


def timed(torch, stream, fn, steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="cfg5", choices=list(CFGS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--parts", type=int, nargs="*", default=[2, 4, 8])
    a = ap.parse_args()
    import torch
    c = CFGS[a.cfg]
    nx, ny, nz = c["shape"]
    lib = rsf.load()
    p = rsf.RsfParams(sigma1=c["sigma1"], sigma2=0.0)
    cp, opt = p.to_c(), options(2, 0, 64)
    img, _ = rsf.phantom_device(nx, ny, nz, with_gt=False, **c["spec"])
    phi = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    torch.cuda.synchronize()

    # t1: the whole volume
    h = C.c_void_p()
    check(lib.rsfg_state_create_device(C.byref(h), phi.data_ptr(), img.data_ptr(), nx, ny, nz, C.byref(cp),
                                       C.byref(opt)))
    sp = C.c_void_p()
    check(lib.rsfg_state_stream(h, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value)
    rep = L.rsfg_report()
    check(lib.rsfg_state_run(h, 3, C.byref(rep)))
    t1 = timed(torch, stream, lambda: check(lib.rsfg_state_run(h, 1, C.byref(rep))), a.steps)
    lib.rsfg_state_destroy(h)
    torch.cuda.empty_cache()

    R = halo_width(p)
    out = {"config": a.cfg, "shape": [nx, ny, nz], "sigma1": c["sigma1"], "halo_planes": R, "t1_ms": round(t1, 3),
           "voxel_iter_per_s_1gpu": nx * ny * nz / (t1 * 1e-3), "parts": {}}
    plane_bytes = nx * ny * 4
    for P in a.parts:
        ranges = plan_slabs(nz, P, R)
        ranks = sorted({0, P // 2, P - 1})  # the two face ranks and an interior one
        times = {}
        for r in ranks:
            z0, z1 = ranges[r]
            s = C.c_void_p()
            check(lib.rsfg_slab_create(C.byref(s), nx, ny, nz, z0, z1, C.byref(cp), C.byref(opt)))
            zb, ze, hh = C.c_int32(), C.c_int32(), C.c_int32()
            check(lib.rsfg_slab_geometry(s, C.byref(zb), C.byref(ze), C.byref(hh)))
            ph = phi[zb.value:ze.value].contiguous()
            im = img[zb.value:ze.value].contiguous()
            torch.cuda.synchronize()
            check(lib.rsfg_slab_upload_device(s, ph.data_ptr(), im.data_ptr()))
            del ph, im
            lo, hi = C.c_float(), C.c_float()
            check(lib.rsfg_slab_local_range(s, C.byref(lo), C.byref(hi)))
            check(lib.rsfg_slab_init(s, lo, hi))
            sstream = torch.cuda.Stream()
            check(lib.rsfg_slab_set_stream(s, C.c_void_p(sstream.cuda_stream)))

            def one():
                check(lib.rsfg_slab_step_interior(s))
                check(lib.rsfg_slab_step_finish(s))

            for _ in range(3):
                one()
            times[r] = timed(torch, sstream, one, a.steps)
            lib.rsfg_slab_destroy(s)
            torch.cuda.empty_cache()
        tmax = max(times.values())
        push_ms = 2 * R * plane_bytes / (PEER_GBS * 1e9) * 1e3
        out["parts"][P] = {"slab_planes": ranges[0][1] - ranges[0][0],
                           "rank_ms": {str(k): round(v, 3) for k, v in times.items()},
                           "push_ms_per_step": round(push_ms, 3),
                           "efficiency_overlapped": round(t1 / (P * tmax), 4),
                           "efficiency_no_overlap": round(t1 / (P * (tmax + push_ms)), 4),
                           "voxel_iter_per_s_model": nx * ny * nz / (tmax * 1e-3)}
        print(json.dumps({"P": P, **out["parts"][P]}), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
