"""Do kernel-1 and kernel-2 CTAs co-resident on an SM beat running them back to
back?  Two independent states on their own streams vs one state alone (same
total voxels), aggregate voxel-iter/s.  Development aid."""
import ctypes as C
import json
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
from paper_2404_02813_b200 import _lib as L  # noqa: E402
from paper_2404_02813_b200.api import check, options  # noqa: E402
import torch  # noqa: E402


def make_state(nz):
    img, _ = rsf.phantom_device(512, 512, nz, n_branches=192 * nz // 512, noise_sigma=20.0, with_gt=False)
    phi = torch.where(img > 125.0, -2.0, 2.0).to(torch.float32)
    lib = rsf.load()
    cp, opt = rsf.RsfParams(sigma1=3.0).to_c(), options(2, 0, 64)
    h = C.c_void_p()
    check(lib.rsfg_state_create_device(C.byref(h), phi.data_ptr(), img.data_ptr(), 512, 512, nz, C.byref(cp),
                                       C.byref(opt)))
    return h


def run(hs, steps):
    lib = rsf.load()
    torch.cuda.synchronize()
    ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev[0].record()
    ts = [threading.Thread(target=lambda h=h: check(lib.rsfg_state_run(h, steps, C.byref(L.rsfg_report()))))
          for h in hs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for h in hs:
        check(lib.rsfg_state_sync(h))
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1])


one = make_state(512)
two = [make_state(256), make_state(256)]
run([one], 5), run(two, 5)
ms1 = run([one], 50)
ms2 = run(two, 50)
n = 512 ** 3 * 50
print(json.dumps({"one_state_512": n / (ms1 * 1e-3), "two_states_256_concurrent": n / (ms2 * 1e-3)}))
