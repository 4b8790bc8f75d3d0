"""Generates tests/golden/rsf_golden.npz from the REFERENCE itself.

The reference (/root/reference/proj, built from its own sources by
oracle/Makefile into oracle/_ref/) is driven through its public C++ API
(init_evolution / evolve_step / energy / convolve_separable /
gaussian_kernel / generate_network / perturb / init_phi) via
oracle/ref_shim.cpp.  Run here (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

It also writes terms_golden.npz: rsf::region_intensities and
rsf::directional_forces (rsf.cpp:235-291) on the same inputs
(`python tests/golden/make_golden.py terms` writes only that file).
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from _oracle import RefLib, params  # noqa: E402


def main():
    ref = RefLib()
    ref.set_workers(1)
    out = {}
    nx, ny, nz = 24, 20, 16
    img, gt = ref.phantom(nx, ny, nz, n_branches=2, seed=3, noise_sigma=20.0, noise_seed=7)
    phi0, nseeds = ref.init_phi(img)
    out.update(img=img, gt=gt, phi0=phi0, nseeds=np.int32(nseeds))
    for tag, (s1, s2) in {"s3": (3.0, 0.0), "s2_15": (2.0, 1.5), "s0": (0.0, 0.0)}.items():
        p = params(sigma1=s1, sigma2=s2)
        st = ref.state(phi0, img, p)
        out[f"E_{tag}"] = st.energy()
        st.step()
        out[f"phi1_{tag}"] = st.phi()
        for _ in range(4):
            st.step()
        out[f"phi5_{tag}"] = st.phi()
    out["conv_img_s2"] = ref.convolve(img, 2.0)
    import ctypes as C
    buf = (C.c_double * 64)()
    r = C.c_int()
    ref.lib.rsfref_gaussian_kernel.argtypes = [C.c_double, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int)]
    ref.lib.rsfref_gaussian_kernel(3.0, buf, 64, C.byref(r))
    out["gauss_s3"] = np.array(buf[: 2 * r.value + 1])
    out["mask_phi5_s3"] = (out["phi5_s3"] < 0).astype(np.float32)
    out["evolve10_s3"] = ref.evolve(phi0, img, params(sigma1=3.0, max_iters=10))
    np.savez_compressed(HERE / "rsf_golden.npz", **out)
    print("wrote", HERE / "rsf_golden.npz", {k: v.shape for k, v in out.items()})


def terms():
    ref = RefLib()
    ref.set_workers(1)
    g = dict(np.load(HERE / "rsf_golden.npz"))
    img, phi0 = g["img"], g["phi0"]
    out = {}
    for tag, s1 in {"s3": 3.0, "s15": 1.5}.items():
        rp, rm = ref.region_intensities(img, phi0, s1, 1.0, 1e-8)
        out[f"rplus_{tag}"], out[f"rminus_{tag}"] = rp, rm
    st = ref.state(phi0, img, params(sigma1=3.0, sigma2=1.5))
    KI, KI2, _, _ = st.static()
    Fp, Fm = ref.directional_forces(img, out["rplus_s3"], out["rminus_s3"], KI, KI2)
    out.update(KI_s2_15=KI, KI2_s2_15=KI2, Fplus=Fp, Fminus=Fm)
    np.savez_compressed(HERE / "terms_golden.npz", **out)
    print("wrote", HERE / "terms_golden.npz", sorted(out))


if __name__ == "__main__":
    if sys.argv[1:] != ["terms"]:
        main()
    terms()
