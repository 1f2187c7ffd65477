"""B200-native ReFusion hot path (Palazzolo et al., IROS 2019, arXiv 1905.02082).

Drop-in for the per-frame path of the CPU reference `tsdfslam`
(/root/reference/proj): voxel-hash allocation, TSDF + colour integration with
free-space carving, direct SDF + colour tracking, the dynamics mask, raycast.
The compute lives in hand-written sm_100a kernels behind the C ABI in
include/refusion_b200.h; this package is the Python mirror of the reference's
interfaces over that ABI."""
from ._lib import ResourceLimitError, RfError, TrackingLostError, UnsupportedError  # noqa: F401
from .api import (IDENTITY, VOXEL_DTYPE, Frame, Pipeline, TsdfVolume, build_mask, dilate, erode,  # noqa: F401
                  floodfill_depth, intrinsics, mask_config, mask_stages, pipeline_config, registration_config,
                  threshold_residuals, volume_config)

__all__ = ["Frame", "Pipeline", "TsdfVolume", "build_mask", "dilate", "erode", "floodfill_depth", "intrinsics",
           "mask_config", "mask_stages", "pipeline_config", "registration_config", "threshold_residuals",
           "volume_config", "TrackingLostError", "ResourceLimitError", "RfError", "UnsupportedError", "IDENTITY",
           "VOXEL_DTYPE"]
