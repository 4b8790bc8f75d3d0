"""B200-native RSF level-set evolution (arXiv 2404.02813 hot path).

The product is librsfg.so (CUDA sm_100a kernels behind the C-ABI in
include/rsfg.h).  This package is the Python mirror of the reference API
for tests and benchmarks; see api.py.
"""
from .api import (  # noqa: F401
    BlowupError,
    EvolutionState,
    EvolveWorkspace,
    KernelProfile,
    ParamError,
    RsfParams,
    ShapeError,
    VolumeIOError,
    dice,
    energy,
    evolve,
    evolve_multi,
    evolve_step,
    extract_mask,
    gaussian_kernel,
    init_evolution,
    init_phi_device,
    merge_phi_device,
    overlap_device,
    read_volume_device,
    write_volume_device,
    plan_tiles,
    run_pipeline,
    tile_file_name,
    save_manifest,
    load_manifest,
    merge_from_dir_device,
    phantom,
    phantom_device,
    threshold_phi0,
    region_intensities,
    directional_forces,
)
from ._lib import LIB_PATH, load  # noqa: F401
