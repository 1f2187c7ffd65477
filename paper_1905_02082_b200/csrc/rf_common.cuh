// Shared device types and primitives for the B200 ReFusion hot path.
//
// Arithmetic contract (parity with the CPU oracle / reference): everything is
// compiled with -fmad=false, so double expressions round exactly as written;
// each formula keeps the operation order of the reference expression it
// restates (file:line cited at the call site, paths under proj/).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rfb {

// ---------------------------------------------------------------- constants
constexpr int kSide = 8;                      // voxels per brick edge (VolumeConfig::block_side)
constexpr int kBrickVoxels = kSide * kSide * kSide;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint32_t kInvalid = 0xFFFFFFFFu;     // slot value before the winner publishes it / not found
constexpr uint32_t kOverflowed = 0xFFFFFFFEu;  // key claimed but no brick left (max_blocks reached)
constexpr int kCoordBias = 1 << 20;           // 21-bit signed range per axis, as mesh.cpp:31-37
constexpr int kAccN = 30;                     // 21 H + 6 b + E_d + E_c + count

// ---------------------------------------------------------------- types
struct Voxel {  // tsdf_volume.hpp:32-37, 8 bytes
    float sdf;
    uint8_t weight, r, g, b;
};
static_assert(sizeof(Voxel) == 8, "voxel layout");

struct alignas(16) HashSlot {  // open-addressed slot, key packed from the block coordinate
    unsigned long long key;
    uint32_t value;
    uint32_t pad;
};

struct Pose {  // camera-to-world; R row-major
    double R[9];
    double t[3];
};

struct Intr {
    double fx, fy, cx, cy;
    int w, h;
};

// Device view of one sparse volume (hash + brick pool).
struct VolumeView {
    HashSlot* slots;
    uint32_t hash_mask;
    uint32_t max_blocks;
    int4* coords;        // brick coordinate per pool index (w unused)
    Voxel* voxels;       // pool, kBrickVoxels per brick, x fastest then y then z
    uint32_t* counters;  // see VolumeCounters
    double voxel_size, truncation;
    int max_weight, carve_weight;
    double min_depth, max_depth, carve_clip;
};

// counters[] slots
enum VolumeCounters : int {
    kNumBlocks = 0,     // bricks allocated (may exceed max_blocks transiently on overflow)
    kOverflow = 1,      // set when an allocation hit max_blocks or the table filled
    kBlocksBefore = 2,  // snapshot of kNumBlocks before this frame's allocation
    kVisible = 3,       // compacted visible-brick count for carve/integrate
    kDdaVisits = 4,     // cells visited by the allocation walk (bytes model)
    kNewBlocks = 5,
    kNumCounters = 8
};

// ---------------------------------------------------------------- math
__host__ __device__ __forceinline__ void pose_apply(const Pose& P, double x, double y, double z, double o[3]) {
    // Pose::operator* (geometry.hpp:85-87): R*x + t, rows summed left to right.
    o[0] = ((P.R[0] * x + P.R[1] * y) + P.R[2] * z) + P.t[0];
    o[1] = ((P.R[3] * x + P.R[4] * y) + P.R[5] * z) + P.t[1];
    o[2] = ((P.R[6] * x + P.R[7] * y) + P.R[8] * z) + P.t[2];
}

__host__ __device__ __forceinline__ Pose pose_inverse(const Pose& P) {  // geometry.hpp:93-96
    Pose r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.R[3 * i + j] = P.R[3 * j + i];
    for (int i = 0; i < 3; ++i)
        r.t[i] = -(((r.R[3 * i] * P.t[0] + r.R[3 * i + 1] * P.t[1]) + r.R[3 * i + 2] * P.t[2]));
    return r;
}

__host__ __device__ __forceinline__ Pose pose_mul(const Pose& A, const Pose& B) {  // geometry.hpp:89-91
    Pose r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.R[3 * i + j] = (A.R[3 * i] * B.R[j] + A.R[3 * i + 1] * B.R[3 + j]) + A.R[3 * i + 2] * B.R[6 + j];
    for (int i = 0; i < 3; ++i)
        r.t[i] = ((A.R[3 * i] * B.t[0] + A.R[3 * i + 1] * B.t[1]) + A.R[3 * i + 2] * B.t[2]) + A.t[i];
    return r;
}

__device__ __forceinline__ bool depth_valid(float d) { return d > 0.0f && isfinite(d); }  // image.hpp:68

__device__ __forceinline__ double luma(uint8_t r, uint8_t g, uint8_t b) {  // image.hpp:80-83
    return 0.2126 * double(r) + 0.7152 * double(g) + 0.0722 * double(b);
}

// ---------------------------------------------------------------- hashing
// HashCoord (spatial_hash.hpp:13-18). Only the low bits survive the
// power-of-two mask, so the 64-bit products reduce to 32-bit ones.
__host__ __device__ __forceinline__ uint32_t hash_coord(int x, int y, int z) {
    return (uint32_t(x) * 73856093u) ^ (uint32_t(y) * 19349669u) ^ (uint32_t(z) * 83492791u);
}

__host__ __device__ __forceinline__ bool coord_in_range(int x, int y, int z) {
    return x >= -kCoordBias && x < kCoordBias && y >= -kCoordBias && y < kCoordBias && z >= -kCoordBias &&
           z < kCoordBias;
}

__host__ __device__ __forceinline__ unsigned long long pack_key(int x, int y, int z) {
    const unsigned long long ux = uint32_t(x + kCoordBias) & 0x1FFFFFu;
    const unsigned long long uy = uint32_t(y + kCoordBias) & 0x1FFFFFu;
    const unsigned long long uz = uint32_t(z + kCoordBias) & 0x1FFFFFu;
    return (uz << 42) | (uy << 21) | ux;
}

// Read-only lookup; valid in kernels that do not insert.
__device__ __forceinline__ uint32_t hash_find(const VolumeView& V, int x, int y, int z) {
    if (!coord_in_range(x, y, z)) return kInvalid;
    const unsigned long long key = pack_key(x, y, z);
    uint32_t idx = hash_coord(x, y, z) & V.hash_mask;
    for (uint32_t probe = 0; probe <= V.hash_mask; ++probe) {
        const uint4 s = __ldg(reinterpret_cast<const uint4*>(V.slots + idx));
        const unsigned long long k = (unsigned long long)s.x | ((unsigned long long)s.y << 32);
        if (k == key) return s.z >= kOverflowed ? kInvalid : s.z;
        if (k == kEmptyKey) return kInvalid;
        idx = (idx + 1) & V.hash_mask;
    }
    return kInvalid;
}

// Lock-free linear-probing insert (no deletion). Returns 1 when this thread
// created the brick, 0 when it already existed, -1 on overflow.
__device__ __forceinline__ int hash_insert(const VolumeView& V, int x, int y, int z) {
    if (!coord_in_range(x, y, z)) {
        atomicOr(&V.counters[kOverflow], 2u);
        return -1;
    }
    const unsigned long long key = pack_key(x, y, z);
    uint32_t idx = hash_coord(x, y, z) & V.hash_mask;
    for (uint32_t probe = 0; probe <= V.hash_mask; ++probe) {
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&V.slots[idx].key);
        if (k == key) {
            if (*reinterpret_cast<volatile uint32_t*>(&V.slots[idx].value) == kOverflowed) {
                atomicOr(&V.counters[kOverflow], 1u);  // AllocateBlock throws again (tsdf_volume.cpp:66-69)
                return -1;
            }
            return 0;
        }
        if (k == kEmptyKey) {
            const unsigned long long old = atomicCAS(&V.slots[idx].key, kEmptyKey, key);
            if (old == kEmptyKey) {
                const uint32_t b = atomicAdd(&V.counters[kNumBlocks], 1u);
                if (b >= V.max_blocks) {
                    atomicOr(&V.counters[kOverflow], 1u);
                    V.slots[idx].value = kOverflowed;
                    return -1;
                }
                V.coords[b] = make_int4(x, y, z, 0);
                V.slots[idx].value = b;
                return 1;
            }
            if (old == key) {
                if (*reinterpret_cast<volatile uint32_t*>(&V.slots[idx].value) == kOverflowed) {
                    atomicOr(&V.counters[kOverflow], 1u);
                    return -1;
                }
                return 0;
            }
        }
        idx = (idx + 1) & V.hash_mask;
    }
    atomicOr(&V.counters[kOverflow], 4u);
    return -1;
}

__device__ __forceinline__ const Voxel* brick_ptr(const VolumeView& V, uint32_t b) {
    return V.voxels + size_t(b) * kBrickVoxels;
}

// ---------------------------------------------------------------- sampling
// CellOf + GatherCorners + SampleWithGradientImpl (tsdf_volume.cpp:243-346),
// evaluated for the SDF and the intensity from one gather of the 8 corners.
struct CellSample {
    double sdf, gs[3];   // value and gradient of the SDF interpolant
    double inten, gi[3]; // value and gradient of the intensity interpolant
};

__device__ __forceinline__ bool gather_corners(const VolumeView& V, int bx, int by, int bz, uint2 c[8]) {
    const int lx = bx & 7, ly = by & 7, lz = bz & 7;
    const int Bx = bx >> 3, By = by >> 3, Bz = bz >> 3;  // arithmetic shift == FloorDiv by 8
    if (lx < 7 && ly < 7 && lz < 7) {
        const uint32_t b = hash_find(V, Bx, By, Bz);
        if (b == kInvalid) return false;
        const uint2* base = reinterpret_cast<const uint2*>(brick_ptr(V, b));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int off = ((lz + (k >> 2)) * 8 + (ly + ((k >> 1) & 1))) * 8 + (lx + (k & 1));
            c[k] = __ldg(base + off);
        }
    } else {
        uint32_t bricks[8];
        const int sx = lx == 7, sy = ly == 7, sz = lz == 7;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
            if ((dx && !sx) || (dy && !sy) || (dz && !sz)) {
                bricks[k] = kInvalid;
                continue;
            }
            bricks[k] = hash_find(V, Bx + dx, By + dy, Bz + dz);
            if (bricks[k] == kInvalid) return false;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int cx = lx + (k & 1), cy = ly + ((k >> 1) & 1), cz = lz + (k >> 2);
            const int bk = (cx >> 3) | ((cy >> 3) << 1) | ((cz >> 3) << 2);
            const uint2* base = reinterpret_cast<const uint2*>(brick_ptr(V, bricks[bk]));
            c[k] = __ldg(base + (((cz & 7) * 8 + (cy & 7)) * 8 + (cx & 7)));
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if ((c[k].y & 0xFFu) == 0u) return false;  // weight byte
    return true;
}

__device__ __forceinline__ float voxel_sdf(uint2 v) { return __uint_as_float(v.x); }
__device__ __forceinline__ double voxel_luma(uint2 v) {
    return luma(uint8_t(v.y >> 8), uint8_t(v.y >> 16), uint8_t(v.y >> 24));
}

__device__ __forceinline__ void cell_of(double px, double py, double pz, double s, int base[3], double f[3]) {
    const double g[3] = {px / s - 0.5, py / s - 0.5, pz / s - 0.5};  // tsdf_volume.cpp:279-283
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double fl = floor(g[i]);
        base[i] = int(fl);
        f[i] = g[i] - fl;
    }
}

template <bool kGrad, bool kIntensity>
__device__ __forceinline__ bool sample_point(const VolumeView& V, const double p[3], CellSample& out) {
    int base[3];
    double f[3];
    cell_of(p[0], p[1], p[2], V.voxel_size, base, f);
    uint2 c[8];
    if (!gather_corners(V, base[0], base[1], base[2], c)) return false;
    const double wx[2] = {1.0 - f[0], f[0]};
    const double wy[2] = {1.0 - f[1], f[1]};
    const double wz[2] = {1.0 - f[2], f[2]};
    double vs[8], vi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        vs[k] = double(voxel_sdf(c[k]));
        if (kIntensity) vi[k] = voxel_luma(c[k]);
    }
    double s = 0.0, in = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double w = wx[k & 1] * wy[(k >> 1) & 1] * wz[k >> 2];
        s += w * vs[k];
        if (kIntensity) in += w * vi[k];
    }
    out.sdf = s;
    out.inten = in;
    if (kGrad) {
        const double inv_s = 1.0 / V.voxel_size;
        double gs[3] = {0, 0, 0}, gi[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                gs[0] += wy[j] * wz[k] * (vs[1 + 2 * j + 4 * k] - vs[2 * j + 4 * k]);
                gs[1] += wx[j] * wz[k] * (vs[j + 2 + 4 * k] - vs[j + 4 * k]);
                gs[2] += wx[j] * wy[k] * (vs[j + 2 * k + 4] - vs[j + 2 * k]);
                if (kIntensity) {
                    gi[0] += wy[j] * wz[k] * (vi[1 + 2 * j + 4 * k] - vi[2 * j + 4 * k]);
                    gi[1] += wx[j] * wz[k] * (vi[j + 2 + 4 * k] - vi[j + 4 * k]);
                    gi[2] += wx[j] * wy[k] * (vi[j + 2 * k + 4] - vi[j + 2 * k]);
                }
            }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            out.gs[i] = gs[i] * inv_s;
            out.gi[i] = gi[i] * inv_s;
        }
    }
    return true;
}

// ---------------------------------------------------------------- grid sync
// Barrier + all-reduce across a cooperative grid: every CTA writes its
// partial vector, the last CTA to arrive folds all partials in CTA order
// (fixed order => run-to-run deterministic) and publishes the result, then
// releases the others. One L2 round trip per waiting CTA.
struct GridSync {
    unsigned int arrive;
    unsigned int gen;
    unsigned int pad[30];
};

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace rfb
