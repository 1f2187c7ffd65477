#pragma once

#include "rf_common.cuh"

namespace rfb {

constexpr uint32_t kFlagCarve = 1u << 31;
constexpr uint32_t kFlagIntegrate = 1u << 30;
constexpr uint32_t kIndexMask = (1u << 30) - 1u;

struct AllocArgs {
    VolumeView V;
    const float* depth;
    const uint8_t* mask;
    Intr K;
    const double* pose;  // device, 12 doubles (camera-to-world)
    const int* lost;     // device flag; skip when set (may be null)
};

struct CullArgs {
    VolumeView V;
    Intr K;
    const double* pose;
    const int* lost;
    uint32_t* list;
    int do_carve, do_integrate;
    int carve_only_before;  // carve only bricks allocated before this frame
};

struct FuseArgs {
    VolumeView V;
    const float* depth;
    const uint8_t* rgb;
    const uint8_t* mask;
    Intr K;
    const double* pose;
    const int* lost;
    const uint32_t* list;
};

struct RaycastArgs {
    VolumeView V;
    Pose view;
    Intr K;
    int bisections;
    float* out;
};

__device__ void link_new(const VolumeView& V);
__global__ void k_link(VolumeView V);
__global__ void k_link_commit(VolumeView V);
__global__ void k_alloc(AllocArgs a);
__global__ void k_raycast(RaycastArgs a);
__global__ void k_alloc_coords(VolumeView V, const int* coords, int n, int* created);
__global__ void k_cull(CullArgs a);
__global__ void k_fuse(FuseArgs a);
__global__ void k_sample(VolumeView V, const double* pts, int n, int mode, double* value, double* grad,
                         uint8_t* valid);
__global__ void k_voxel_rw(VolumeView V, const int* vc, int n, Voxel* io, uint8_t* found, int write);
__global__ void k_occupancy(VolumeView V, uint8_t* bitmap);

}  // namespace rfb
