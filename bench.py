#!/usr/bin/env python3
"""Benchmark: RSF level-set evolution, voxel-iterations/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one RSF iteration (rsf::evolve_step, rsf.cpp:324-357) over the
whole volume.  Workload (BASELINE.json configs[1], SURVEY.md 8(d) cfg 2):
512^3 synthetic tube network (reference phantom spec, n_branches 192, noise
sigma 20), sigma1 = 3 (R = 9), sigma2 = 0, 3d-paper parameters, phi0 =
threshold initialisation.  N > 1 scales WEAKLY: each GPU owns a 512^3 z-slab
of a 512x512x(512 N) volume, with per-step NCCL halo exchange
(paper_2404_02813_b200/spmd.py).

`value`   : device-resident inputs, CUDA events around exactly K steps on the
            launching stream, max over ranks.  Inputs (1.5 GiB working set)
            are larger than L2, so no flush is needed.
`e2e`     : the same metric through the public C-ABI with HOST buffers
            (rsfg_evolve: H2D of I and phi0, init, the config's 200
            iterations, D2H of phi), wall clock per call.
`roofline`: dominant kernel, algorithmic bytes per launch / CUDA-event time.
`cpu_baseline`: the reference compiled from its own sources (oracle/_ref,
            all host cores) on a bounded z-slab sample of the same volume.
`--impl reference`: the reference CPU implementation alone (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "voxel-iterations/s at 512^3 fp32 (RSF level-set step)"
UNIT = "voxel-iter/s"
NX = NY = NZ = 512
SIGMA1 = 3.0
ITERS_CFG = 200  # configs[1]: 200 iterations
PHANTOM = dict(n_branches=192, radius_min=2.0, radius_max=4.0, tortuosity=0.25, foreground=200.0,
               background=50.0, rng_seed=1, tree_connected=True, noise_sigma=20.0, noise_seed=7)
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
# Implementation bytes per voxel each kernel must move at minimum.
KERNEL_BYTES = {2: {"xy": 16, "zst": 24}, 4: {"xy": 24, "zst": 32}}
ALGO_BYTES_STEP = 12  # read phi, read I, write phi' (fp32, sigma2 = 0)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def workload_config(n_gpus, fields):
    return {"workload": "cfg2: 512^3 synthetic tube network (SURVEY.md 8(d)), sigma1=3 (R=9), sigma2=0, "
                        "3d-paper params (alpha=58.5225, beta=0.1, eps=1, dt=0.06), phi0 = threshold init",
            "nx": NX, "ny": NY, "nz": NZ, "sigma1": SIGMA1, "sigma2": 0.0, "fields": fields,
            "iterations_per_job": ITERS_CFG,
            "decomposition": f"z-slabs x{n_gpus}" if n_gpus > 1 else "single volume",
            "l2": "inputs larger than L2 (1.5 GiB working set vs 126 MB L2); no flush"}


def make_inputs():
    import paper_2404_02813_b200 as rsf
    img, _gt = rsf.phantom(NX, NY, NZ, **PHANTOM)
    phi0 = rsf.threshold_phi0(img)
    return img, phi0


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ncu_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        k = d.get("kernels", {}).get(kernel_key)
        if k and k.get("config") == f"{NX}x{NY}x{NZ}":
            return k.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


# --------------------------------------------------------------- CPU (reference)
def reference_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib  # test-infrastructure loader of oracle/_ref (reference build)
    return RefLib()


def reference_sample(img, phi0, planes):
    """A z-slab sample [0, planes) of the same volume (reference is per-voxel rate
    limited once data exceed L3)."""
    return np.ascontiguousarray(img[:planes]), np.ascontiguousarray(phi0[:planes])


def run_reference(img, phi0, steps, warmup, planes):
    ref = reference_lib()
    from _oracle import params as ref_params
    ref.set_workers(0)  # all host cores (volume.cpp:18-22)
    si, sp = reference_sample(img, phi0, planes)
    st = ref.state(sp, si, ref_params(sigma1=SIGMA1, sigma2=0.0))
    for _ in range(warmup):
        st.step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        st.step()
        times.append(time.perf_counter() - t0)
    vox = si.size
    rate = vox * steps / sum(times)
    return rate, ref.workers(), vox, times


# ---------------------------------------------------------------------- GPU
def bench_single(args):
    import torch
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200 import _lib as L
    from paper_2404_02813_b200.api import check, options
    import ctypes as C

    torch.cuda.set_device(0)
    img, phi0 = make_inputs()
    nvox = img.size
    p = rsf.RsfParams(sigma1=SIGMA1, sigma2=0.0, max_iters=ITERS_CFG)
    lib = rsf.load()

    # ---- value: device-resident inputs
    d_img = torch.from_numpy(img).cuda()
    d_phi = torch.from_numpy(phi0).cuda()
    h = C.c_void_p()
    cp = p.to_c()
    opt = options(args.fields, 0, 64)
    check(lib.rsfg_state_create_device(C.byref(h), d_phi.data_ptr(), d_img.data_ptr(), NX, NY, NZ, C.byref(cp),
                                       C.byref(opt)))
    st_ptr = C.c_void_p()
    check(lib.rsfg_state_stream(h, C.byref(st_ptr)))
    stream = torch.cuda.ExternalStream(st_ptr.value)
    rep = L.rsfg_report()
    check(lib.rsfg_state_run(h, args.warmup, C.byref(rep)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.rsfg_state_launches(h)
    remaining, chunks = args.steps, []
    with ClockSampler() as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        while remaining > 0:
            n = min(remaining, 64)
            check(lib.rsfg_state_run(h, n, C.byref(rep)))
            remaining -= n
        e1.record(stream)
        torch.cuda.synchronize()
    launches = int(lib.rsfg_state_launches(h) - l0)
    ms = e0.elapsed_time(e1)
    ms_step = ms / args.steps
    value = nvox * args.steps / (ms / 1e3)

    # ---- per-kernel CUDA-event profile (same stream the kernels launch on)
    prof = (C.c_double * 2)()
    check(lib.rsfg_state_profile(h, 10, prof))
    kern = {"xy": prof[0], "zst": prof[1]}
    vflags, xyb, zstb = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.rsfg_state_variant(h, C.byref(vflags), C.byref(xyb), C.byref(zstb)))
    lib.rsfg_state_destroy(h)
    del d_img, d_phi
    torch.cuda.empty_cache()

    pk, pk_kind = peaks()
    peak = pk["hbm_gbs"]
    dom = max(kern, key=kern.get)
    kb = dict(KERNEL_BYTES[args.fields])
    kb.update(xy=xyb.value, zst=zstb.value)
    achieved = kb[dom] * nvox / (kern[dom] * 1e-3) / 1e9
    traffic = ncu_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_voxel": kb[dom], "peak_source": f"{pk_kind} hbm_gbs",
                "kernel_variant_flags": vflags.value,
                "bytes_note": "per-kernel minimum HBM bytes per voxel (rsfg_state_variant): kernel 2 also "
                              "writes the (H-, H- I) pairs in the stored-Heaviside mode (flag 4)",
                "kernel_ms": {k: round(v, 4) for k, v in kern.items()},
                "kernel_share": {k: round(v / sum(kern.values()), 3) for k, v in kern.items()}}
    step_gbs = ALGO_BYTES_STEP * value / 1e9
    step_roofline = {"bytes_per_voxel_iter": ALGO_BYTES_STEP, "achieved": round(step_gbs, 1),
                     "frac": round(step_gbs / peak, 4), "unit": "GB/s",
                     "note": "fused-minimum 12 B/voxel-iter (SURVEY.md 8(d)) over the whole step"}

    # ---- e2e: public C-ABI with pinned host buffers, H2D + D2H inside the timed region
    h_img = torch.from_numpy(img).pin_memory()
    h_phi = torch.empty_like(h_img).pin_memory()
    e2e_times, rep2 = [], L.rsfg_report()
    opt2 = options(args.fields, 0, 25)
    for i in range(1 + args.e2e_steps):
        h_phi.copy_(torch.from_numpy(phi0))
        t0 = time.perf_counter()
        check(lib.rsfg_evolve(h_img.data_ptr(), h_phi.data_ptr(), NX, NY, NZ, C.byref(cp), C.byref(opt2),
                              L.STOP_FN(0), None, 0, C.byref(rep2)))
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_times.append(dt)
    e2e_value = nvox * ITERS_CFG / statistics.median(e2e_times) if e2e_times else None
    e2e = {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * nvox * 4, "d2h_bytes_per_step": nvox * 4,
           "iterations_per_step": ITERS_CFG, "api": "rsfg_evolve (host buffers)",
           "phase_ms": {"h2d": round(rep2.ms_h2d, 2), "init": round(rep2.ms_init, 2),
                        "loop": round(rep2.ms_loop, 2), "d2h": round(rep2.ms_d2h, 2)}}

    # ---- CPU baseline: the reference itself on a bounded sample of the same volume
    cpu = None
    if not args.no_cpu:
        try:
            rate, cores, vox, times = run_reference(img, phi0, steps=3, warmup=1, planes=args.cpu_planes)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"reference init_evolution + 1 warm-up + 3 timed evolve_step on planes "
                             f"[0,{args.cpu_planes}) of the same 512^3 volume ({vox} voxels)"}
        except Exception as e:  # reference build missing on this host
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference phantom spec, seeded)",
           "config": workload_config(1, args.fields), "roofline": roofline, "step_roofline": step_roofline,
           "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(out))


def bench_multi(args):
    """N > 1: weak scaling.  The volume is 512 x 512 x (512 N) (the cfg-2 tube
    network with 192 N branches, same density), one 512^3 z-slab per rank
    (SURVEY.md 8(e)): per-step NCCL halo exchange of R planes each way,
    overlapped with the owned planes' xy work.  Every rank generates the same
    volume on its own GPU (device phantom, bit-exact with the reference
    generator) and uploads only its held planes.  value = all voxels x K steps
    / max over ranks of the CUDA-event time.  --backend gloo --share-gpu runs
    the same path with ranks sharing cuda:0 and host-staged halos (1-GPU test
    boxes)."""
    import torch
    import torch.distributed as dist
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import DistSlab, Slab

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    transport = "device" if args.backend == "nccl" else "host"
    nz_total = NZ * world
    spec = dict(PHANTOM)
    spec["n_branches"] = PHANTOM["n_branches"] * world
    img, _ = rsf.phantom_device(NX, NY, nz_total, with_gt=False, device=local,
                                **{k: v for k, v in spec.items() if k not in ("rng_seed", "noise_seed")},
                                rng_seed=spec["rng_seed"], noise_seed=spec["noise_seed"])
    phi0 = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    nvox = NX * NY * nz_total
    p = rsf.RsfParams(sigma1=SIGMA1, sigma2=0.0, max_iters=ITERS_CFG)
    ds = DistSlab(phi0, img, p, fields=args.fields, transport=transport)
    # host copies of this rank's held planes for the e2e leg (outside any timing)
    zb, ze = ds.slab.zb, ds.slab.ze
    h_img = torch.empty((nz_total, NY, NX), dtype=torch.float32).numpy()  # untouched planes stay unbacked
    h_phi = torch.empty((nz_total, NY, NX), dtype=torch.float32).numpy()
    h_img[zb:ze] = img[zb:ze].cpu().numpy()
    h_phi[zb:ze] = phi0[zb:ze].cpu().numpy()
    del img, phi0
    torch.cuda.empty_cache()
    for _ in range(args.warmup):
        ds.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ds.slab.launches()
    red_dev = "cuda" if args.backend == "nccl" else "cpu"
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(args.steps):
            ds.step()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    launches = torch.tensor([ds.slab.launches() - l0], device=red_dev, dtype=torch.int64)
    dist.all_reduce(launches)
    ms = float(ms.item())
    value = nvox * args.steps / (ms / 1e3)
    ds.slab.close()

    # e2e: this rank's host planes -> device (H2D), init, ITERS_CFG steps, D2H of
    # the owned planes; wall clock, max over ranks.
    e2e_t = []
    for i in range(1 + args.e2e_steps):
        dist.barrier()
        t0 = time.perf_counter()
        d2 = DistSlab(h_phi, h_img, p, fields=args.fields, transport=transport)
        for _ in range(ITERS_CFG):
            d2.step()
        _ = d2.phi_owned()
        d2.slab.close()
        t = torch.tensor([time.perf_counter() - t0], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i > 0:
            e2e_t.append(float(t.item()))
    if rank == 0:
        cfg = workload_config(world, args.fields)
        cfg.update({"workload": f"weak scaling: 512x512x{nz_total} tube network (cfg2 density, "
                                f"{spec['n_branches']} branches), one 512^3 z-slab per GPU, sigma1=3 (R=9), "
                                "3d-paper params, phi0 = threshold init",
                    "nz": nz_total, "decomposition": f"z-slabs x{world}, halo R=9 planes each way per step "
                                                     f"({args.backend}, overlapped with the owned planes' xy work)",
                    "l2": "inputs larger than L2; no flush"})
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (reference phantom spec, seeded; device generator)", "config": cfg,
               "e2e": {"value": nvox * ITERS_CFG / statistics.median(e2e_t) if e2e_t else None, "unit": UNIT,
                       "h2d_bytes_per_step": 2 * nvox * 4, "d2h_bytes_per_step": nvox * 4,
                       "iterations_per_step": ITERS_CFG, "api": "spmd.DistSlab (host buffers)"},
               "gpu_launches": int(launches.item()), "clocks": clk.summary(), "roofline": None,
               "cpu_baseline": None}
        print(json.dumps(out))
    dist.destroy_process_group()


def bench_reference(args):
    """--impl reference: the reference CPU implementation (oracle/_ref), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ref = reference_lib()
    # Input: the reference's own phantom + perturb (bit-identical to make_inputs()).
    img, _gt = ref.phantom(NX, NY, NZ, n_branches=PHANTOM["n_branches"], seed=PHANTOM["rng_seed"],
                           noise_sigma=PHANTOM["noise_sigma"], noise_seed=PHANTOM["noise_seed"])
    phi0 = np.where(img > 125, np.float32(-2.0), np.float32(2.0)).astype(np.float32)
    budget_s = 120.0
    planes = int(np.clip(3.0e7 * budget_s / max(1, args.steps + args.warmup) / (NX * NY), 16, 128))
    rate, cores, vox, times = run_reference(img, phi0, steps=args.steps, warmup=args.warmup, planes=planes)
    sample = f"{args.steps} timed evolve_step (after {args.warmup} warm-up) on planes [0,{planes}) of the 512^3 volume"
    out = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (reference)",
           "data": "synthetic (reference phantom spec, seeded)", "config": workload_config(1, 4),
           "impl": "reference",
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fields", type=int, default=2, choices=[2, 4])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-planes", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"], help="N > 1 halo transport")
    ap.add_argument("--share-gpu", action="store_true", help="N > 1 ranks all on cuda:0 (testing; gloo)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return bench_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return bench_multi(args)
    return bench_single(args)


if __name__ == "__main__":
    main()
