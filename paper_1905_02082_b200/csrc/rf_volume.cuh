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
    int assign;             // assign + cull the preceding k_alloc's pending bricks (assign_new)
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

// The refinement window fused in one pass per chunk of <= kMaxWin entries
// (RenderVirtualDepth, depth_refinement.cpp:25-30: AllocateForFrame then
// Integrate, entry after entry). A brick receives an entry's update only from
// the first entry that allocated it onwards (win_first), so allocating the
// whole chunk first changes nothing; every voxel applies its entries in order.
constexpr int kMaxWin = 16;
struct WindowArgs {
    VolumeView V;
    int n;                          // entries in the chunk
    const float* depth[kMaxWin];
    const uint8_t* rgb[kMaxWin];    // may be null
    const uint8_t* mask[kMaxWin];   // may be null
    const double* pose[kMaxWin];    // device, camera-to-world
    Intr K[kMaxWin];
    uint32_t* list;                 // visible bricks as {brick, entry bitmask} pairs
    // Optional per-entry brick lists (what AllocateForFrame of the entry
    // allocates, recorded when the frame entered the window): entries with a
    // list are inserted from it instead of re-walking their pixels.
    const int4* blist[kMaxWin];
    const uint32_t* bcount[kMaxWin];  // list length; kListOverflow: no list (walk)
};
constexpr uint32_t kListOverflow = 0xFFFFFFFFu;

struct RaycastArgs {
    VolumeView V;
    Pose view;
    Intr K;
    int bisections;
    float* out;          // virtual depth (may be null when `refined` is set)
    // RefineDepth (depth_refinement.cpp:82-93) fused: with `raw` set, pixels
    // whose raw depth is valid keep it and are not marched unless `out` wants
    // the full virtual image; the rest take the virtual depth or far_value.
    const float* raw;
    float* refined;
    float far_value;
};

// Marching cubes (rf_mesh.cu): per-cell state lives in one scratch buffer.
struct MeshArgs {
    VolumeView V;
    uint32_t n;  // bricks
    int min_weight;
    const uint32_t* order;  // rank -> pool index, bricks sorted by (x, y, z)
    const uint32_t* rank;   // pool index -> rank
    uint16_t* info;         // per cell: 0x100 complete | cube index
    uint16_t* owned;        // per cell: mask of the edges whose vertex it emits
    uint16_t* vloc;         // per cell: in-brick vertex offset
    uint16_t* floc;         // per cell: in-brick face offset
    uint32_t* vcount;       // per rank (n + 1)
    uint32_t* fcount;
    uint32_t* vbase;        // exclusive scans of vcount / fcount
    uint32_t* fbase;
    float* xyz;
    uint8_t* rgb;
    int32_t* faces;
};
size_t mesh_scratch_bytes(uint32_t n);
cudaError_t mesh_prepare(const VolumeView& V, uint32_t n, int min_weight, cudaStream_t stream, void* scratch,
                         size_t scratch_bytes, uint32_t* totals, MeshArgs* out);
cudaError_t mesh_emit(const MeshArgs& a, cudaStream_t stream);

__device__ void link_new(const VolumeView& V);
__global__ void k_link(VolumeView V);
__global__ void k_link_commit(VolumeView V);
__global__ void k_alloc(AllocArgs a);
__global__ void k_raycast(RaycastArgs a);
__global__ void k_alloc_coords(VolumeView V, const int* coords, int n, int* created);
__global__ void k_assign(VolumeView V, int* created);
__global__ void k_cull(CullArgs a);
__global__ void k_fuse(FuseArgs a);
__global__ void k_sample(VolumeView V, const double* pts, int n, int mode, double* value, double* grad,
                         uint8_t* valid);
__global__ void k_voxel_rw(VolumeView V, const int* vc, int n, Voxel* io, uint8_t* found, int write);
__global__ void k_occupancy(VolumeView V, uint8_t* bitmap);
__global__ void k_volume_check(VolumeView V, unsigned long long* err);
__global__ void k_vol_clear(VolumeView V, bool voxels);  // voxels=false: hash only
__global__ void k_win_first_reset(VolumeView V);
__global__ void k_alloc_window(WindowArgs a);
__global__ void k_insert_window(WindowArgs a);
__global__ void k_brick_list(VolumeView S, int4* dst, uint32_t cap, uint32_t* count);
__global__ void k_cull_window(WindowArgs a);
__global__ void k_fuse_window(WindowArgs a);

}  // namespace rfb
