"""ctypes binding of librefusion_b200.so (include/refusion_b200.h).

The product path: every call goes to the CUDA kernels through the C ABI. There
is no CPU fallback — importing this module on a machine without the built
library, or calling it without a GPU, raises."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# RF_LIB_PATH selects an alternative build of the same library (tuning runs).
LIB_PATH = os.environ.get("RF_LIB_PATH") or os.path.join(_HERE, "librefusion_b200.so")


class rf_intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("depth_scale", C.c_double)]


class rf_volume_config(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("truncation", C.c_double), ("block_side", C.c_int32),
                ("max_weight", C.c_int32), ("carve_weight", C.c_int32), ("reserved0", C.c_int32),
                ("min_depth", C.c_double), ("max_depth", C.c_double), ("carve_clip", C.c_double),
                ("max_blocks", C.c_uint64), ("hash_capacity", C.c_uint64)]


class rf_registration_config(C.Structure):
    _fields_ = [("color_weight", C.c_double), ("pyramid_levels", C.c_int32), ("max_iterations", C.c_int32),
                ("lm_lambda_init", C.c_double), ("lm_lambda_up", C.c_double), ("lm_lambda_down", C.c_double),
                ("convergence_eps", C.c_double), ("min_valid_residuals", C.c_int32), ("threads", C.c_int32),
                ("huber_depth", C.c_double), ("huber_color", C.c_double)]


class rf_mask_config(C.Structure):
    _fields_ = [("gamma", C.c_double), ("truncation", C.c_double), ("theta", C.c_double),
                ("erode_radius", C.c_int32), ("dilate_radius", C.c_int32), ("connectivity", C.c_int32),
                ("reserved0", C.c_int32), ("free_space", C.c_double)]


class rf_pipeline_config(C.Structure):
    _fields_ = [("volume", rf_volume_config), ("registration", rf_registration_config), ("mask", rf_mask_config),
                ("refine_enabled", C.c_int32), ("refine_window", C.c_int32), ("far_value", C.c_double),
                ("bisection_iterations", C.c_int32), ("dynamics_enabled", C.c_int32), ("threads", C.c_int32),
                ("reserved0", C.c_int32)]


class rf_frame(C.Structure):
    _fields_ = [("depth", C.c_void_p), ("rgb", C.c_void_p), ("intrinsics", rf_intrinsics), ("timestamp", C.c_double),
                ("memory", C.c_int32), ("reserved0", C.c_int32)]


class rf_frame_stats(C.Structure):
    _fields_ = [("frame_index", C.c_uint64), ("timestamp", C.c_double), ("tracking_lost", C.c_int32),
                ("converged", C.c_int32), ("registrations", C.c_int32), ("iterations", C.c_int32),
                ("valid_residuals", C.c_uint64), ("masked_pixels", C.c_uint64), ("final_error", C.c_double),
                ("runtime_ms", C.c_double)]


class rf_registration_result(C.Structure):
    _fields_ = [("pose", C.c_double * 12), ("converged", C.c_int32), ("iterations", C.c_int32),
                ("valid_residuals", C.c_uint64), ("final_error", C.c_double)]


class rf_linearize_result(C.Structure):
    _fields_ = [("H", C.c_double * 36), ("b", C.c_double * 6), ("depth_error", C.c_double),
                ("color_error", C.c_double), ("error", C.c_double), ("valid_count", C.c_uint64),
                ("degenerate", C.c_int32), ("reserved0", C.c_int32)]


class rf_frame_counters(C.Structure):
    _fields_ = [("dda_visits", C.c_uint64), ("new_blocks", C.c_uint64), ("visible_bricks", C.c_uint64),
                ("num_blocks", C.c_uint64), ("floodfill_rounds", C.c_int32), ("overflow", C.c_int32),
                ("passes", C.c_int32), ("reserved0", C.c_int32), ("pixel_passes", C.c_double)]


RF_OK, RF_INVALID_ARGUMENT, RF_TRACKING_LOST, RF_RESOURCE_LIMIT, RF_CUDA_ERROR, RF_IO_ERROR, RF_UNSUPPORTED, RF_FAILED = range(8)
RF_MEMORY_HOST, RF_MEMORY_DEVICE = 0, 1

# Every exported symbol of include/refusion_b200.h (checked by the CPU tests).
EXPORTS = [
    "rf_last_error", "rf_version", "rf_volume_create", "rf_volume_destroy", "rf_volume_num_blocks",
    "rf_volume_hash_capacity", "rf_volume_get_config", "rf_volume_allocate_blocks", "rf_volume_allocate_for_frame", "rf_volume_integrate",
    "rf_volume_carve", "rf_volume_sample", "rf_volume_get_voxels", "rf_volume_set_voxels", "rf_volume_export_blocks",
    "rf_volume_hash_occupancy", "rf_volume_reset", "rf_volume_save", "rf_volume_load", "rf_linearize",
    "rf_evaluate_depth_error", "rf_evaluate_color_error", "rf_register", "rf_mask_stages", "rf_raycast",
    "rf_pipeline_create", "rf_pipeline_destroy", "rf_pipeline_process_frame", "rf_pipeline_finalize",
    "rf_pipeline_volume", "rf_pipeline_tracking_losses", "rf_pipeline_trajectory", "rf_pipeline_last_mask",
    "rf_pipeline_last_residuals", "rf_pipeline_last_counters", "rf_host_alloc", "rf_host_free", "rf_device_alloc",
    "rf_device_free", "rf_copy_to_device", "rf_pipeline_set_profiling", "rf_pipeline_stage_times",
    "rf_pipeline_stream", "rf_synth_render", "rf_pipeline_profile_counters", "rf_diag_grid_barrier",
    "rf_diag_lm_step", "rf_volume_extract_mesh", "rf_mesh_counts", "rf_mesh_copy", "rf_mesh_device_buffers",
    "rf_mesh_write_ply", "rf_mesh_destroy", "rf_render_virtual_depth", "rf_pipeline_window_size",
    "rf_pipeline_set_debug_images", "rf_pipeline_last_refinement", "rf_pipeline_finalize_one", "rf_diag_pass_bench", "rf_pipeline_process_frames",
    "rf_ate_rmse", "rf_rpe_over_time", "rf_nearest_distances", "rf_distance_cdf", "rf_build_pyramid",
    "rf_volume_find_block", "rf_volume_write_block", "rf_diag_volume_check",
]

_lib = None


def load(path: str = LIB_PATH):
    """Loads the CUDA library; raises if it is missing (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_1905_02082_b200.build` "
                           "(the CUDA path has no CPU fallback)")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.rf_last_error.restype = C.c_char_p
    L.rf_version.restype = C.c_char_p
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("rf_last_error", "rf_version", "rf_host_alloc", "rf_device_alloc", "rf_volume_destroy",
                        "rf_pipeline_destroy", "rf_host_free", "rf_device_free", "rf_mesh_destroy"):
            fn.restype = C.c_int
    L.rf_host_alloc.restype = vp
    L.rf_host_alloc.argtypes = [C.c_size_t]
    L.rf_device_alloc.restype = vp
    L.rf_device_alloc.argtypes = [C.c_size_t, C.c_int]
    L.rf_host_free.argtypes = [vp]
    L.rf_device_free.argtypes = [vp]
    L.rf_volume_destroy.argtypes = [vp]
    L.rf_pipeline_destroy.argtypes = [vp]
    L.rf_mesh_destroy.argtypes = [vp]
    L.rf_copy_to_device.argtypes = [vp, vp, C.c_size_t]
    _lib = L
    return L


class RfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rf status {code}: {msg}")
        self.code = code


class TrackingLostError(RfError):
    """errors.hpp:14"""


class ResourceLimitError(RfError):
    """errors.hpp:19"""


class UnsupportedError(RfError):
    pass


def check(code: int):
    if code == RF_OK:
        return
    msg = load().rf_last_error().decode(errors="replace")
    if code == RF_TRACKING_LOST:
        raise TrackingLostError(code, msg)
    if code == RF_RESOURCE_LIMIT:
        raise ResourceLimitError(code, msg)
    if code == RF_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == RF_UNSUPPORTED:
        raise UnsupportedError(code, msg)
    raise RfError(code, msg)
