"""Multi-rank z-slab decomposition on CPU (gloo, world_size 2 and 3).

Each rank holds planes [zb, ze) of the volume, exchanges its halo planes with
its z-neighbours through spmd.start_halo_exchange (the same pairing the NCCL
driver uses) and steps its owned planes with the oracle's slab step.  The
gathered result must equal the monolithic oracle bitwise (P4 on CPU)."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, phi0, img, steps, sigma1, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist
    from _oracle import Geom, Oracle, params
    from paper_2404_02813_b200.spmd import held_range, plan_slabs, start_halo_exchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, ny, nx = phi0.shape
        op = params(sigma1=sigma1)
        halo = max((len(Oracle().gaussian_kernel(sigma1)) - 1) // 2, 2)
        z0, z1 = plan_slabs(nz, world, halo)[rank]
        zb, ze = held_range(z0, z1, nz, halo)
        o = Oracle()
        KI, KI2, lo, hi = o.init(img, op)  # static fields: global, computed once
        held = torch.from_numpy(np.ascontiguousarray(phi0[zb:ze]).copy())
        I_h = np.ascontiguousarray(img[zb:ze])
        KI_h, KI2_h = np.ascontiguousarray(KI[zb:ze]), np.ascontiguousarray(KI2[zb:ze])
        g = Geom(nx, ny, nz, zb, ze)
        for _ in range(steps):
            k_lo, k_hi = z0 - zb, ze - z1
            lo_v = (held[z0 - zb:z0 - zb + k_lo], held[0:k_lo]) if k_lo else (None, None)
            hi_v = (held[z1 - zb - k_hi:z1 - zb], held[z1 - zb:ze - zb]) if k_hi else (None, None)
            # contiguous receive buffers, copied back after the wait
            lo_r = torch.empty_like(lo_v[1]) if k_lo else None
            hi_r = torch.empty_like(hi_v[1]) if k_hi else None
            reqs = start_halo_exchange(dist, rank, world, (lo_v[0].contiguous() if k_lo else None, lo_r),
                                       (hi_v[0].contiguous() if k_hi else None, hi_r))
            for r in reqs:
                r.wait()
            if k_lo:
                held[0:k_lo] = lo_r
            if k_hi:
                held[z1 - zb:ze - zb] = hi_r
            out, _, _ = o.step_slab(g, held.numpy(), I_h, KI_h, KI2_h, lo, hi, op, z0, z1)
            held[z0 - zb:z1 - zb] = torch.from_numpy(out[z0 - zb:z1 - zb])
        q.put((rank, z0, z1, held[z0 - zb:z1 - zb].numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sigma1", [(2, 3.0), (3, 2.0)])
def test_slabs_gloo_bitwise(world, sigma1):
    from _inputs import random_case
    from _oracle import Oracle, params
    img, phi0 = random_case(20, 18, 30, seed=11)
    steps = 3
    ref = phi0.copy()
    o = Oracle()
    st = o.init(img, params(sigma1=sigma1))
    for _ in range(steps):
        ref, _, _ = o.step(ref, img, params(sigma1=sigma1), st)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, phi0, img, steps, sigma1, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([a for _, _, _, a in sorted(parts)])
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
