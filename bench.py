#!/usr/bin/env python3
"""Benchmark: RSF level-set evolution, voxel-iterations/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode weak|strong-cfg4|strong-cfg5] [--transport ipc|nccl|host]

A "step" is one RSF iteration (rsf::evolve_step, rsf.cpp:324-357) over the
whole volume.

N = 1 (default): BASELINE.json configs[1] = SURVEY.md 8(d) cfg 2 -- 512^3
synthetic tube network (reference phantom spec, n_branches 192, noise sigma
20), sigma1 = 3 (R = 9), sigma2 = 0, 3d-paper parameters, phi0 = threshold
initialisation.

N > 1: `--gpus N` launches N ranks itself (torch.distributed.run, one process
per GPU, 127.0.0.1) unless it is already running under torchrun; it refuses
to run with fewer than N visible GPUs (unless --share-gpu).  Modes:
  weak         each rank owns a 512^3 z-slab of 512 x 512 x (512 N) at the
               cfg-2 density (BASELINE metric "512^3 ... (1/2/4/8 B200)");
  strong-cfg4  cfg 4: 1024^3 light-sheet-like volume split over N ranks;
  strong-cfg5  cfg 5: 2048 x 2048 x 1024 micro-CT-like volume, sigma1 = 4.
The halo data path is the peer-link exchange (`--transport ipc`: boundary
planes pushed into the neighbours' halo rows over NVLink via CUDA IPC, flag
words instead of messages); `nccl` (send/recv) and `host` (gloo, host-staged)
are the alternatives.

`value`   : device-resident inputs, CUDA events around exactly K steps on the
            launching stream, max over ranks.  Inputs (>= 1.5 GiB working
            set) are larger than L2, so no flush is needed.
`e2e`     : the same metric through the public C-ABI with HOST buffers
            (rsfg_evolve: H2D of I and phi0, init, the config's iterations,
            D2H of phi) per call, wall clock.  The headline is PAGEABLE host
            memory (a std::vector, as the reference's caller passes it,
            tiling.cpp:251); pinned buffers are reported beside it.
`roofline`: the dominant kernel; achieved = SURVEY.md 8(d)'s 12 B per
            voxel-iteration x the voxels one launch processes / its average
            CUDA-event launch time (its share of the step is in kernel_share).
`cpu_baseline`: the reference compiled from its own sources (oracle/_ref,
            all host cores) on the same 512^3 volume.
`parity`  : 1-step |dphi| vs the reference at 512^3, and cfg 1 (128^3 x 100
            iterations) mask statistics vs the reference.
`--impl reference`: the reference CPU implementation alone (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
# SURVEY.md 8(d) cfg 4 / cfg 5 (strong scaling); iterations 100 each.
STRONG = {
    "strong-cfg4": dict(shape=(1024, 1024, 1024), sigma1=3.0, iters=100,
                        spec=dict(n_branches=768, axial_blur_sigma=2.0, noise_sigma=25.0, contrast_axis=3,
                                  contrast_lo=0.6, contrast_hi=1.0),
                        workload="cfg4: 1024^3 light-sheet-like tube network (768 branches, axial blur 2, "
                                 "z contrast 0.6-1.0, noise 25), sigma1=3 (R=9)"),
    "strong-cfg5": dict(shape=(2048, 2048, 1024), sigma1=4.0, iters=100,
                        spec=dict(n_branches=3072, radius_max=5.0, noise_sigma=15.0),
                        workload="cfg5: 2048x2048x1024 micro-CT-like tube network (3072 branches, r 2-5, "
                                 "noise 15), sigma1=4 (R=12)"),
}
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
ALGO_BYTES = 12  # read phi, read I, write phi' (fp32, sigma2 = 0) per voxel-iteration
# FP32 FMA-pipe lane-operations per voxel-iteration of the two kernels (FFMA/FMUL/FADD count 1,
# the packed f32x2 forms 2), from ncu's per-opcode instruction counts at 512^3, sigma1 = 3
# (profiles/r02_final_opcodes.txt), and the measured FMA-pipe peak of this B200 pool
# (profiles/r01_fma_peak.txt: 36.87 T lane-ops/s, FFMA2 19-tap convolution microbenchmark).
FP32_OPS = {"xy": 90.2, "zst": 93.0}
FP32_PEAK_T = 36.87


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        if "hbm_gbs" in d:
            return {"hbm_gbs": float(d["hbm_gbs"])}, "measured (hbm_gbs, MEASURED_PEAKS.json)"
        return PEAKS_FALLBACK, "fallback (MEASURED_PEAKS.json has no HBM key)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(n_gpus, fields, mode="weak"):
    return {"workload": "cfg2: 512^3 synthetic tube network (SURVEY.md 8(d)), sigma1=3 (R=9), sigma2=0, "
                        "3d-paper params (alpha=58.5225, beta=0.1, eps=1, dt=0.06), phi0 = threshold init",
            "nx": NX, "ny": NY, "nz": NZ, "sigma1": SIGMA1, "sigma2": 0.0, "fields": fields,
            "iterations_per_job": ITERS_CFG, "mode": mode,
            "decomposition": f"z-slabs x{n_gpus}" if n_gpus > 1 else "single volume",
            "l2": "inputs larger than L2 (1.5 GiB working set vs 126 MB L2); no flush"}


def make_inputs():
    import paper_2404_02813_b200 as rsf
    img, gt = rsf.phantom(NX, NY, NZ, **PHANTOM)
    phi0 = rsf.threshold_phi0(img)
    return img, phi0, gt


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index=0, period=0.005):
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


def ncu_traffic(kernel_key, config):
    """dram bytes per launch of that kernel from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        k = d.get("kernels", {}).get(kernel_key)
        if k and k.get("config") == config:
            return k.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


# --------------------------------------------------------------- CPU (reference)
def reference_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib  # test-infrastructure loader of oracle/_ref (reference build)
    return RefLib()


def run_reference(img, phi0, steps, warmup, planes=None):
    """Reference init_evolution + `warmup` untimed + `steps` timed evolve_step
    (all host cores) on planes [0, planes) (default: the whole volume).
    Returns (rate, cores, voxels, times, phi after the first step)."""
    ref = reference_lib()
    from _oracle import params as ref_params
    ref.set_workers(0)  # all host cores (volume.cpp:18-22)
    if planes is not None and planes < img.shape[0]:
        img, phi0 = np.ascontiguousarray(img[:planes]), np.ascontiguousarray(phi0[:planes])
    st = ref.state(phi0, img, ref_params(sigma1=SIGMA1, sigma2=0.0))
    phi1 = None
    for i in range(warmup):
        st.step()
        if i == 0:
            phi1 = st.phi()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        st.step()
        times.append(time.perf_counter() - t0)
    return img.size * steps / sum(times), ref.workers(), img.size, times, phi1


def parity_cfg1(lib_ref):
    """cfg 1: 128^3, 12 branches, noise 20, phi0 = the
    reference's init_phi; 100 iterations on the GPU and in the reference.
    BASELINE.md 3 statistics: mask sign-mismatch, Dice(GPU, CPU), Dice vs gt."""
    import paper_2404_02813_b200 as rsf
    from _oracle import params as ref_params
    img, gt = lib_ref.phantom(128, 128, 128, n_branches=12, seed=1, noise_sigma=20.0, noise_seed=7)
    phi0, _ = lib_ref.init_phi(img)
    want = lib_ref.evolve(phi0, img, ref_params(sigma1=3.0, max_iters=100))
    got = rsf.evolve(phi0, img, rsf.RsfParams(sigma1=3.0, max_iters=100))
    mg, mr, mt = got < 0, want < 0, gt > 0.5
    mism = int(np.count_nonzero(mg != mr))
    return {"config": "cfg1: 128^3, 12 branches, noise 20, phi0 = reference init_phi, sigma1=3, 100 iterations",
            "mask_mismatch": mism, "mask_mismatch_frac": mism / img.size,
            "dice_gpu_vs_ref": rsf.dice(mg, mr), "dice_gt_gpu": rsf.dice(mg, mt), "dice_gt_ref": rsf.dice(mr, mt),
            "gates": "P3: mismatch <= 1e-5 N, Dice(gpu, ref) >= 0.9999 (SURVEY.md 8(c))"}


# ---------------------------------------------------------------------- GPU
def bench_single(args):
    import ctypes as C
    import torch
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200 import _lib as L
    from paper_2404_02813_b200.api import check, options

    torch.cuda.set_device(0)
    img, phi0, gt = make_inputs()
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
    remaining = args.steps
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

    # ---- per-kernel CUDA-event profile on the kernels' own stream
    prof = (C.c_double * 2)()
    check(lib.rsfg_state_profile(h, 10, prof))
    kern = {"xy": prof[0], "zst": prof[1]}
    vflags, xyb, zstb = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.rsfg_state_variant(h, C.byref(vflags), C.byref(xyb), C.byref(zstb)))
    lib.rsfg_state_destroy(h)
    del d_img, d_phi
    torch.cuda.empty_cache()

    pk, pk_src = peaks()
    peak = pk["hbm_gbs"]
    dom = max(kern, key=kern.get)
    achieved = ALGO_BYTES * nvox / (kern[dom] * 1e-3) / 1e9
    own = {"xy": xyb.value, "zst": zstb.value}
    roofline = {"bound": "hbm", "kernel": {"xy": "kernel 1 (xy2_hh)", "zst": "kernel 2 (zst4)"}[dom],
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": ncu_traffic(dom, f"{NX}x{NY}x{NZ}"),
                "algorithmic_bytes_per_voxel": ALGO_BYTES, "launch_ms": round(kern[dom], 4),
                "peak_source": pk_src, "kernel_variant_flags": vflags.value,
                "basis": "SURVEY.md 8(d): 12 B per voxel-iteration x 512^3 voxels per launch / the launch's "
                         "CUDA-event time",
                "kernel_own_min_bytes_per_voxel": own,
                "kernel_own_frac": {k: round(own[k] * nvox / (kern[k] * 1e-3) / 1e9 / peak, 4) for k in kern},
                "kernel_ms": {k: round(v, 4) for k, v in kern.items()},
                "kernel_share": {k: round(v / sum(kern.values()), 3) for k, v in kern.items()},
                "step_frac": round(ALGO_BYTES * value / 1e9 / peak, 4)}
    # The path is FP32-throughput-bound: the same kernels against the FMA pipe.
    fp32_roofline = {"bound": "fp32 (FMA pipe; tensor cores unused)",
                     "ops_per_voxel_iter": round(sum(FP32_OPS.values()), 1),
                     "achieved": round(sum(FP32_OPS.values()) * value / 1e12, 2),
                     "peak": FP32_PEAK_T, "unit": "T FMA-pipe lane-ops/s",
                     "frac": round(sum(FP32_OPS.values()) * value / 1e12 / FP32_PEAK_T, 4),
                     "kernel_frac": {k: round(FP32_OPS[k] * nvox / (kern[k] * 1e-3) / 1e12 / FP32_PEAK_T, 4)
                                     for k in kern},
                     "basis": "ncu per-opcode counts (profiles/r02_final_opcodes.txt) x voxel-iter/s; peak = "
                              "measured FFMA2 throughput (profiles/r01_fma_peak.txt)"}

    # ---- 14-row stage profile (rsf::KernelProfile) over a few steps
    stage = rsf.KernelProfile()
    st = rsf.init_evolution(phi0, img, p, fields=args.fields)
    for _ in range(3):
        st.step(stage)
    stage_rows = {n: round(1e3 * s / max(1, stage.iterations), 4)
                  for n, s in zip(rsf.KernelProfile.names(), stage.seconds)}
    st.close()

    # ---- e2e: public C-ABI with HOST buffers, H2D + D2H inside the timed region
    def e2e_run(phi_buf, img_buf):
        times, rep2 = [], L.rsfg_report()
        opt2 = options(args.fields, 0, 25)
        for i in range(1 + args.e2e_steps):
            np.copyto(phi_buf, phi0)
            t0 = time.perf_counter()
            check(lib.rsfg_evolve(img_buf.ctypes.data, phi_buf.ctypes.data, NX, NY, NZ, C.byref(cp), C.byref(opt2),
                                  L.STOP_FN(0), None, 0, C.byref(rep2)))
            dt = time.perf_counter() - t0
            if i > 0:
                times.append(dt)
        return nvox * ITERS_CFG / statistics.median(times), rep2

    def phases(r):
        return {"h2d": round(r.ms_h2d, 2), "init": round(r.ms_init, 2), "loop": round(r.ms_loop, 2),
                "d2h": round(r.ms_d2h, 2)}

    e2e = None
    phi_gpu_final = None
    if args.e2e_steps > 0:
        page_img, page_phi = np.array(img), np.empty_like(phi0)  # ordinary (pageable) host memory
        e2e_page, rep_page = e2e_run(page_phi, page_img)
        phi_gpu_final = page_phi.copy()
        t_img = torch.from_numpy(img).pin_memory()
        t_phi = torch.empty_like(t_img).pin_memory()
        e2e_pin, rep_pin = e2e_run(t_phi.numpy(), t_img.numpy())
        del t_img, t_phi
        e2e = {"value": e2e_page, "unit": UNIT, "h2d_bytes_per_step": 2 * nvox * 4, "d2h_bytes_per_step": nvox * 4,
               "iterations_per_step": ITERS_CFG, "host_memory": "pageable (numpy / std::vector, as tiling.cpp:251)",
               "api": "rsfg_evolve (host buffers; device workspace allocated and freed inside every call)",
               "phase_ms": phases(rep_page),
               "pinned": {"value": e2e_pin, "phase_ms": phases(rep_pin)}}

    # ---- CPU baseline + parity: the reference itself on the same 512^3 volume
    cpu, parity = None, None
    if not args.no_cpu:
        try:
            rate, cores, vox, times, ref_phi1 = run_reference(img, phi0, steps=2, warmup=1)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
                   "sample": f"reference init_evolution + 1 warm-up + 2 timed evolve_step on the full 512^3 "
                             f"volume ({vox} voxels), all {cores} host threads"}
            st1 = rsf.init_evolution(phi0, img, p, fields=args.fields)
            st1.step()
            g1 = st1.phi
            st1.close()
            d = np.abs(g1.astype(np.float64) - ref_phi1)
            parity = {"cfg2_step1": {"max_abs_dphi": float(d.max()),
                                     "max_rel_dphi": float((d / np.maximum(1.0, np.abs(ref_phi1))).max()),
                                     "gate": "P1 max|dphi| <= 1e-4 (SURVEY.md 8(c))"},
                      "cfg2_200it_gpu_dice_vs_gt": (rsf.dice(phi_gpu_final < 0, gt > 0.5)
                                                    if phi_gpu_final is not None else None)}
            if not args.no_parity:
                parity["cfg1_100it"] = parity_cfg1(reference_lib())
        except Exception as e:  # reference build missing on this host
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference phantom spec, seeded)",
           "config": workload_config(1, args.fields), "roofline": roofline, "fp32_roofline": fp32_roofline,
           "cpu_baseline": cpu, "e2e": e2e,
           "parity": parity, "stage_ms_per_iter": stage_rows, "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(out), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def bench_multi(args, world, rank, local):
    """Multi-rank modes (module docstring).  value = all voxels x K steps /
    max over ranks of the CUDA-event time of the K steps."""
    import torch
    import torch.distributed as dist
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import DistSlab

    torch.cuda.set_device(local)
    if world == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    elif args.transport in ("nccl", "ipc") and not args.share_gpu:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    transport = {"nccl": "device", "ipc": "ipc", "host": "host"}[args.transport]
    if args.mode == "weak":
        nx, ny, nz_total = NX, NY, NZ * world
        spec = dict(PHANTOM)
        spec["n_branches"] = PHANTOM["n_branches"] * world
        sigma1, iters = SIGMA1, ITERS_CFG
        workload = (f"weak scaling: 512x512x{nz_total} tube network (cfg2 density, {spec['n_branches']} branches), "
                    "one 512^3 z-slab per GPU, sigma1=3 (R=9), 3d-paper params, phi0 = threshold init")
        scaling = "weak"
    else:
        c = STRONG[args.mode]
        nx, ny, nz_total = c["shape"]
        spec = dict(PHANTOM)
        spec.update(c["spec"])
        sigma1, iters = c["sigma1"], c["iters"]
        workload = c["workload"] + f", split into {world} z-slab(s), 3d-paper params, phi0 = threshold init"
        scaling = "strong"
    img, _ = rsf.phantom_device(nx, ny, nz_total, with_gt=False, device=local,
                                **{k: v for k, v in spec.items() if k not in ("rng_seed", "noise_seed")},
                                rng_seed=spec["rng_seed"], noise_seed=spec["noise_seed"])
    phi0 = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    nvox = nx * ny * nz_total
    p = rsf.RsfParams(sigma1=sigma1, sigma2=0.0, max_iters=iters)
    ds = DistSlab(phi0, img, p, fields=args.fields, transport=transport)
    zb, ze = ds.slab.zb, ds.slab.ze
    keep_host = args.e2e_steps > 0
    if keep_host:  # host copies of this rank's held planes for the e2e leg (outside any timing)
        h_img = np.zeros((nz_total, ny, nx), np.float32)  # untouched planes stay unbacked
        h_phi = np.zeros((nz_total, ny, nx), np.float32)
        h_img[zb:ze] = img[zb:ze].cpu().numpy()
        h_phi[zb:ze] = phi0[zb:ze].cpu().numpy()
    del img, phi0
    torch.cuda.empty_cache()
    red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    for _ in range(args.warmup):
        ds.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ds.slab.launches()
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

    # e2e: this rank's host planes -> device, init, the config's iterations,
    # D2H of the owned planes; wall clock, max over ranks.
    e2e_t = []
    for i in range(1 + args.e2e_steps if keep_host else 0):
        dist.barrier()
        t0 = time.perf_counter()
        d2 = DistSlab(h_phi, h_img, p, fields=args.fields, transport=transport)
        for _ in range(iters):
            d2.step()
        _ = d2.phi_owned()
        d2.slab.close()
        t = torch.tensor([time.perf_counter() - t0], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i > 0:
            e2e_t.append(float(t.item()))
    if rank == 0:
        cfg = {"workload": workload, "nx": nx, "ny": ny, "nz": nz_total, "sigma1": sigma1, "sigma2": 0.0,
               "fields": args.fields, "iterations_per_job": iters, "mode": args.mode,
               "decomposition": f"z-slabs x{world}, halo R planes each way per step ({args.transport})",
               "transport": args.transport, "l2": "inputs larger than L2; no flush"}
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": scaling, "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (reference phantom spec, seeded; device generator)", "config": cfg,
               "e2e": {"value": nvox * iters / statistics.median(e2e_t) if e2e_t else None, "unit": UNIT,
                       "h2d_bytes_per_step": 2 * nvox * 4, "d2h_bytes_per_step": nvox * 4,
                       "iterations_per_step": iters, "api": "spmd.DistSlab (host buffers)"},
               "gpu_launches": int(launches.item()), "clocks": clk.summary(), "roofline": None,
               "cpu_baseline": None}
        print(json.dumps(out), flush=True)
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
    # The full 512^3 volume (about 2.5 s per step on 16 host cores) unless
    # that would exceed ~5 minutes; then a z-slab sample, stated in `sample`.
    planes = NZ
    est_s = 2.6 * (args.steps + args.warmup)
    if est_s > 300:
        planes = int(np.clip(NZ * 300 / est_s, 16, NZ))
    rate, cores, vox, times, _ = run_reference(img, phi0, steps=args.steps, warmup=args.warmup, planes=planes)
    what = "the full 512^3 volume" if planes == NZ else f"planes [0,{planes}) of the 512^3 volume"
    sample = (f"{args.steps} timed evolve_step (after init_evolution and {args.warmup} warm-up) on {what} "
              f"({vox} voxels), {cores} host threads, {cpu_model()}")
    out = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (reference)",
           "data": "synthetic (reference phantom spec, seeded)", "config": workload_config(1, 4),
           "impl": "reference",
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                            "cpu_model": cpu_model()},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="weak", choices=["weak", *STRONG])
    ap.add_argument("--fields", type=int, default=2, choices=[2, 4])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl", "host"], help="N > 1 halo transport")
    ap.add_argument("--backend", default=None, choices=["nccl", "gloo"], help="(legacy) gloo == --transport host")
    ap.add_argument("--share-gpu", action="store_true", help="N > 1 ranks all on cuda:0 (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.backend == "gloo":
        args.transport = "host" if args.transport == "nccl" else args.transport
        args.share_gpu = True if args.transport == "host" else args.share_gpu
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    gpus = args.gpus if args.gpus is not None else world_env
    if world_env > 1 and gpus != world_env:
        sys.exit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world_env}")
    if gpus > 1 and world_env == 1:
        # one process per GPU: launch the N ranks ourselves
        if not args.share_gpu and args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < gpus:
                sys.exit(f"bench.py: --gpus {gpus} needs {gpus} visible GPUs, found {have}")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        return bench_reference(args)
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", rank))
    if gpus > 1 or args.mode != "weak":
        return bench_multi(args, gpus, rank, local)
    return bench_single(args)


if __name__ == "__main__":
    main()
