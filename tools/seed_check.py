"""GPU init_phi vs the compiled reference at the bench
volume (512^3, cfg 2 phantom): seed-set equality, max |dphi0|, timings."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2404_02813_b200 as rsf  # noqa: E402
import torch  # noqa: E402
from _oracle import RefLib  # noqa: E402  (test infrastructure: the checker)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
img_d, _ = rsf.phantom_device(n, n, n, n_branches=max(1, int(12 * (n / 128) ** 2)), noise_sigma=20.0, with_gt=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
phi_g, xyz_g, resp_g = rsf.init_phi_device(img_d)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
img = img_d.cpu().numpy()
ref = RefLib()
ref.set_workers(0)
t0 = time.perf_counter()
phi_r, n_r = ref.init_phi(img)
t_ref = time.perf_counter() - t0
xyz_r, _ = ref.detect_seeds(img)
d = np.abs(phi_g.cpu().numpy().astype(np.float64) - phi_r)
print(json.dumps({"n": n, "seeds_gpu": len(xyz_g), "seeds_ref": int(n_r), "seed_sets_equal": bool(np.array_equal(xyz_g, xyz_r)),
                  "max_abs_dphi0": float(d.max()), "p99999_abs_dphi0": float(np.quantile(d, 0.99999)),
                  "gpu_s": round(t_gpu, 3), "jacobi_iterations": rsf.init_phi_device.iterations, "reference_s": round(t_ref, 2), "reference_cores": ref.workers()}))
