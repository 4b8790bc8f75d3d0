"""Device phantom vs host phantom on the bench volume, and device generation
times at the large configs (SURVEY.md 8(d) cfg 4/5).  Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_02813_b200 as rsf  # noqa: E402
import torch  # noqa: E402

out = {}
t0 = time.perf_counter()
img_h, gt_h = rsf.phantom(512, 512, 512, n_branches=192, noise_sigma=20.0)
out["host_512_s"] = round(time.perf_counter() - t0, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
img_d, gt_d = rsf.phantom_device(512, 512, 512, n_branches=192, noise_sigma=20.0)
torch.cuda.synchronize()
out["device_512_s"] = round(time.perf_counter() - t0, 3)
d = img_d.cpu().numpy()
out["mismatch_512"] = int(np.count_nonzero(d != img_h))
out["max_abs_diff_512"] = float(np.abs(d.astype(np.float64) - img_h).max())
out["gt_mismatch_512"] = int(np.count_nonzero(gt_d.cpu().numpy() != gt_h))
del img_d, gt_d
for name, (nx, ny, nz, kw) in {
        "cfg4_1024": (1024, 1024, 1024, dict(n_branches=768, axial_blur_sigma=2.0, noise_sigma=25.0, contrast_axis=3,
                                             contrast_lo=0.6, contrast_hi=1.0)),
        "cfg5_2048x2048x1024": (2048, 2048, 1024, dict(n_branches=3072, radius_max=5.0, noise_sigma=15.0))}.items():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    img, _ = rsf.phantom_device(nx, ny, nz, with_gt=False, **kw)
    torch.cuda.synchronize()
    out[f"device_{name}_s"] = round(time.perf_counter() - t0, 2)
    out[f"{name}_mean"] = float(img.mean())
    del img
    torch.cuda.empty_cache()
print(json.dumps(out))
