"""Seeded synthetic inputs shared by the tests (SURVEY.md 8(d) generator)."""
from __future__ import annotations

import functools

import numpy as np


@functools.lru_cache(maxsize=16)
def case(nx, ny, nz, n_branches=3, seed=1, noise=20.0, init="seeds"):
    """(image, phi0, gt) from the reference phantom + perturb, phi0 from the
    reference init_phi (seeded distance, seeding.cpp:221-235) when the
    compiled reference is available, else the threshold initialisation."""
    from _oracle import RefLib
    try:
        ref = RefLib()
    except FileNotFoundError:
        ref = None
    if ref is not None:
        img, gt = ref.phantom(nx, ny, nz, n_branches=n_branches, seed=seed, noise_sigma=noise, noise_seed=7)
    else:
        from paper_2404_02813_b200 import phantom
        img, gt = phantom(nx, ny, nz, n_branches=n_branches, rng_seed=seed, noise_sigma=noise, noise_seed=7)
    if init == "seeds" and ref is not None:
        try:
            phi, _ = ref.init_phi(img)
        except ValueError:
            phi = np.where(img > 125, -2.0, 2.0).astype(np.float32)
    else:
        phi = np.where(img > 125, -2.0, 2.0).astype(np.float32)
    img.setflags(write=False)
    phi.setflags(write=False)
    gt.setflags(write=False)
    return img, phi, gt


def random_case(nx, ny, nz, seed=0):
    rng = np.random.default_rng(seed)
    img = rng.uniform(0, 255, (nz, ny, nx)).astype(np.float32)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    r = np.sqrt((xx - nx / 2) ** 2 + (yy - ny / 2) ** 2 + (zz - nz / 2) ** 2)
    phi = (r - min(nx, ny, nz) / 4).astype(np.float32) + rng.uniform(-0.3, 0.3, r.shape).astype(np.float32)
    return img, phi
