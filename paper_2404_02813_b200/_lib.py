"""ctypes binding of librsfg.so (the C-ABI declared in include/rsfg.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2404_02813_b200/csrc``).  There is no fallback: importing the
product API without the library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RSFG_LIB", PKG / "lib" / "librsfg.so"))

RSFG_OK = 0
RSFG_ERR_PARAM = 1
RSFG_ERR_SHAPE = 2
RSFG_ERR_BLOWUP = 3
RSFG_ERR_CUDA = 4
RSFG_ERR_COMM = 5
RSFG_ERR_OOM = 6
RSFG_ERR_STATE = 7
RSFG_ERR_IO = 8


class rsfg_params(C.Structure):
    _fields_ = [
        ("sigma1", C.c_double),
        ("sigma2", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("epsilon", C.c_double),
        ("dt", C.c_double),
        ("max_iters", C.c_int32),
        ("convergence_fraction", C.c_double),
        ("denom_floor", C.c_double),
        ("grad_floor", C.c_double),
    ]


class rsfg_options(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("fields", C.c_int32),
        ("check_every", C.c_int32),
        ("use_graphs", C.c_int32),
        ("reuse_workspace", C.c_int32),
        ("profile_stages", C.c_int32),
        ("reserved", C.c_int32 * 2),
    ]


RSFG_STAGE_COUNT = 14
RSFG_PEER_DESC_BYTES = 512


class rsfg_report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("blowup_iteration", C.c_int32),
        ("blowup_x", C.c_int32),
        ("blowup_y", C.c_int32),
        ("blowup_z", C.c_int32),
        ("last_sign_change_fraction", C.c_double),
        ("ms_h2d", C.c_double),
        ("ms_init", C.c_double),
        ("ms_loop", C.c_double),
        ("ms_d2h", C.c_double),
        ("gpu_launches", C.c_int64),
        ("stage_seconds", C.c_double * RSFG_STAGE_COUNT),
        ("ms_setup", C.c_double),
    ]


class rsfg_blob_params(C.Structure):
    _fields_ = [("sigma_b", C.c_double), ("response_threshold", C.c_double), ("nms_radius", C.c_double),
                ("dark", C.c_int32)]


class rsfg_tile(C.Structure):
    _fields_ = [("ix", C.c_int32), ("iy", C.c_int32), ("iz", C.c_int32), ("core_origin", C.c_int32 * 3),
                ("core_extent", C.c_int32 * 3), ("pad_origin", C.c_int32 * 3), ("pad_extent", C.c_int32 * 3)]


class rsfg_pipeline_options(C.Structure):
    _fields_ = [("global_seeding", C.c_int32), ("merge", C.c_int32), ("seed_radius", C.c_double),
                ("device", C.c_int32), ("fields", C.c_int32), ("spill_dir", C.c_char_p)]


class rsfg_phantom_spec(C.Structure):
    _fields_ = [
        ("nx", C.c_int32),
        ("ny", C.c_int32),
        ("nz", C.c_int32),
        ("n_branches", C.c_int32),
        ("radius_min", C.c_double),
        ("radius_max", C.c_double),
        ("tortuosity", C.c_double),
        ("foreground", C.c_float),
        ("background", C.c_float),
        ("rng_seed", C.c_uint64),
        ("tree_connected", C.c_int32),
        ("axial_blur_sigma", C.c_double),
        ("noise_sigma", C.c_double),
        ("contrast_axis", C.c_int32),
        ("contrast_lo", C.c_double),
        ("contrast_hi", C.c_double),
        ("noise_seed", C.c_uint64),
    ]


STOP_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_float), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p)

VP = C.c_void_p
FP = C.c_void_p  # float* passed as raw address (numpy .ctypes.data or device pointer)
I32 = C.c_int32
P = C.POINTER

# name -> (restype, argtypes); every entry point of include/rsfg.h
SIGNATURES = {
    "rsfg_last_error": (C.c_char_p, []),
    "rsfg_version": (C.c_char_p, []),
    "rsfg_params_default": (None, [P(rsfg_params)]),
    "rsfg_options_default": (None, [P(rsfg_options)]),
    "rsfg_params_validate": (C.c_int, [P(rsfg_params)]),
    "rsfg_gaussian_kernel": (C.c_int, [C.c_double, P(C.c_double), I32, P(I32)]),
    "rsfg_evolve": (C.c_int, [FP, FP, I32, I32, I32, P(rsfg_params), P(rsfg_options), STOP_FN, VP, I32,
                              P(rsfg_report)]),
    "rsfg_extract_mask": (C.c_int, [FP, FP, C.c_int64, I32]),
    "rsfg_release_workspace": (None, []),
    "rsfg_state_create": (C.c_int, [P(VP), FP, FP, I32, I32, I32, P(rsfg_params), P(rsfg_options)]),
    "rsfg_state_create_device": (C.c_int, [P(VP), FP, FP, I32, I32, I32, P(rsfg_params), P(rsfg_options)]),
    "rsfg_state_step": (C.c_int, [VP, P(C.c_double)]),
    "rsfg_state_run": (C.c_int, [VP, I32, P(rsfg_report)]),
    "rsfg_state_energy": (C.c_int, [VP, FP]),
    "rsfg_state_profile": (C.c_int, [VP, I32, P(C.c_double)]),
    "rsfg_profile_name": (C.c_char_p, [I32]),
    "rsfg_slab_peer_desc": (C.c_int, [VP, VP, I32]),
    "rsfg_slab_link": (C.c_int, [VP, I32, VP]),
    "rsfg_slab_step_linked": (C.c_int, [VP]),
    "rsfg_evolve_multi": (C.c_int, [FP, FP, I32, I32, I32, P(rsfg_params), P(rsfg_options), P(I32), I32, STOP_FN,
                                    VP, I32, P(rsfg_report)]),
    "rsfg_stage_name": (C.c_char_p, [I32]),
    "rsfg_stage_carrier": (C.c_int32, [I32]),
    "rsfg_state_step_profiled": (C.c_int, [VP, P(C.c_double), P(C.c_double)]),
    "rsfg_state_set_params": (C.c_int, [VP, P(rsfg_params)]),
    "rsfg_region_intensities": (C.c_int, [FP, FP, I32, I32, I32, C.c_double, C.c_double, C.c_double, FP, FP, I32]),
    "rsfg_region_intensities_device": (C.c_int, [VP, VP, I32, I32, I32, C.c_double, C.c_double, C.c_double, VP,
                                                 VP, I32]),
    "rsfg_directional_forces": (C.c_int, [FP, FP, FP, FP, C.c_int64, FP, FP, I32]),
    "rsfg_directional_forces_device": (C.c_int, [VP, VP, VP, VP, C.c_int64, VP, VP, I32]),
    "rsfg_state_read_phi": (C.c_int, [VP, FP]),
    "rsfg_state_write_phi": (C.c_int, [VP, FP]),
    "rsfg_state_mask": (C.c_int, [VP, FP]),
    "rsfg_state_iteration": (C.c_int, [VP, P(I32)]),
    "rsfg_state_device_phi": (C.c_int, [VP, P(VP)]),
    "rsfg_state_stream": (C.c_int, [VP, P(VP)]),
    "rsfg_state_sync": (C.c_int, [VP]),
    "rsfg_state_launches": (C.c_int64, [VP]),
    "rsfg_state_variant": (C.c_int, [VP, P(I32), P(I32), P(I32)]),
    "rsfg_state_destroy": (None, [VP]),
    "rsfg_slab_create": (C.c_int, [P(VP), I32, I32, I32, I32, I32, P(rsfg_params), P(rsfg_options)]),
    "rsfg_slab_geometry": (C.c_int, [VP, P(I32), P(I32), P(I32)]),
    "rsfg_slab_upload": (C.c_int, [VP, FP, FP]),
    "rsfg_slab_upload_device": (C.c_int, [VP, FP, FP]),
    "rsfg_slab_local_range": (C.c_int, [VP, P(C.c_float), P(C.c_float)]),
    "rsfg_slab_init": (C.c_int, [VP, C.c_float, C.c_float]),
    "rsfg_slab_halo": (C.c_int, [VP, I32, P(VP), P(VP), P(C.c_int64)]),
    "rsfg_slab_set_stream": (C.c_int, [VP, VP]),
    "rsfg_slab_exchange": (C.c_int, [VP, VP]),
    "rsfg_slab_step_interior": (C.c_int, [VP]),
    "rsfg_slab_step_finish": (C.c_int, [VP]),
    "rsfg_slab_counters": (C.c_int, [VP, P(C.c_int64), P(C.c_int64)]),
    "rsfg_slab_download": (C.c_int, [VP, FP]),
    "rsfg_slab_device_phi": (C.c_int, [VP, P(VP)]),
    "rsfg_slab_launches": (C.c_int64, [VP]),
    "rsfg_slab_destroy": (None, [VP]),
    "rsfg_phantom_default": (None, [P(rsfg_phantom_spec)]),
    "rsfg_phantom": (C.c_int, [P(rsfg_phantom_spec), FP, FP]),
    "rsfg_phantom_device": (C.c_int, [P(rsfg_phantom_spec), VP, VP, I32, P(C.c_int64)]),
    "rsfg_blob_params_default": (None, [P(rsfg_blob_params)]),
    "rsfg_pipeline_options_default": (None, [P(rsfg_pipeline_options)]),
    "rsfg_volume_info": (C.c_int, [C.c_char_p, P(I32), P(I32), P(I32), P(C.c_double), P(I32)]),
    "rsfg_read_volume_device": (C.c_int, [C.c_char_p, VP, C.c_int64, I32, P(C.c_float), P(C.c_int64)]),
    "rsfg_write_volume_device": (C.c_int, [C.c_char_p, VP, I32, I32, I32, P(C.c_double), P(C.c_float), I32]),
    "rsfg_overlap_device": (C.c_int, [VP, VP, C.c_int64, I32, P(C.c_double), P(C.c_double)]),
    "rsfg_plan_tiles": (C.c_int, [I32, I32, I32, I32, I32, I32, C.c_double, C.c_double, P(rsfg_tile), I32, P(I32),
                                  P(I32)]),
    "rsfg_merge_phi_device": (C.c_int, [P(VP), I32, I32, I32, I32, I32, I32, I32, I32, I32, VP, I32]),
    "rsfg_run_pipeline": (C.c_int, [FP, I32, I32, I32, P(rsfg_params), P(rsfg_blob_params), I32, I32, I32,
                                    P(rsfg_pipeline_options), FP, FP, C.c_char_p, I32, P(I32)]),
    "rsfg_init_phi_device": (C.c_int, [VP, I32, I32, I32, P(rsfg_blob_params), C.c_double, VP, I32, P(I32),
                                       P(I32), FP, I32, P(I32)]),
    "rsfg_tile_file_name": (C.c_int, [P(rsfg_tile), C.c_char_p, I32]),
    "rsfg_save_manifest": (C.c_int, [C.c_char_p, I32, I32, I32, I32, I32, I32, I32, P(rsfg_tile), I32]),
    "rsfg_load_manifest": (C.c_int, [C.c_char_p, P(I32), P(I32), P(I32), P(rsfg_tile), I32, P(I32)]),
    "rsfg_merge_from_dir": (C.c_int, [C.c_char_p, I32, I32, I32, I32, I32, I32, I32, P(rsfg_tile), I32, I32, VP,
                                      I32]),
    "rsfg_merge_from_dir_host": (C.c_int, [C.c_char_p, I32, I32, I32, I32, I32, I32, I32, P(rsfg_tile), I32, I32,
                                           FP, I32]),
    "rsfg_init_phi": (C.c_int, [FP, I32, I32, I32, P(rsfg_blob_params), C.c_double, FP, I32, P(I32),
                                P(I32), FP, I32, P(I32)]),
}

_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load librsfg.so (once).  Raises if it is missing: no fallback path."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} not built: run __graft_entry__.build() (nvcc sm_100a); "
                          "the RSF path has no CPU fallback")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load().rsfg_last_error().decode()
