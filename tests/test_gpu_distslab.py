"""spmd.DistSlab end to end on the GPU: two ranks share cuda:0 over a gloo
process group (halo planes staged through host memory, transport="host"),
run the slab C-ABI kernels and must reproduce the monolithic volume bitwise
(P4).  The NCCL transport differs only in where the halo bytes travel."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

from _inputs import case

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, phi0, img, steps, sigma1, q, transport="host"):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    import paper_2404_02813_b200 as rsf
    from paper_2404_02813_b200.spmd import DistSlab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = DistSlab(phi0, img, rsf.RsfParams(sigma1=sigma1), transport=transport)
        for _ in range(steps):
            ds.step()
        torch.cuda.synchronize()
        q.put((rank, ds.slab.z0, ds.phi_owned(), ds.slab.launches()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,transport", [(2, (96, 28, 80), "host"), (3, (40, 36, 48), "host"),
                                                   (2, (96, 28, 80), "ipc"), (3, (64, 40, 48), "ipc")])
def test_distslab_bitwise_vs_monolithic(world, shape, transport):
    """transport="ipc": the peer-link data path across processes (CUDA IPC
    handles of each rank's phi buffers and flag words; on one GPU the
    "peers" are other processes on the same device)."""
    import paper_2404_02813_b200 as rsf
    img, phi, _ = case(*shape)
    img, phi = np.array(img), np.array(phi)
    steps, sigma1 = 6, 3.0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) * 8 + world + (4 if transport == "ipc" else 0)
    procs = [ctx.Process(target=_worker, args=(r, world, port, phi, img, steps, sigma1, q, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    got = np.concatenate([t[2] for t in parts])
    assert all(t[3] > 0 for t in parts)  # every rank launched kernels
    st = rsf.init_evolution(phi, img, rsf.RsfParams(sigma1=sigma1))
    for _ in range(steps):
        st.step()
    assert np.array_equal(got, st.phi)
