// Shared device types and primitives for the B200 ReFusion hot path.
//
// Arithmetic contract (parity with the CPU oracle / reference): everything is
// compiled with -fmad=false, so double expressions round exactly as written;
// each formula keeps the operation order of the reference expression it
// restates (file:line cited at the call site, paths under proj/).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Bounds / invariant checks of the checked build (tools/checked_build.sh:
// build --variant checked -DRF_CHECKED, run the GPU suite with RF_LIB_PATH).
// The GPU pool has no compute-sanitizer, so the hot kernels assert their own
// index ranges; a violation prints and traps (the test run fails loudly).
#ifdef RF_CHECKED
#define RF_ASSERT(c)                                                                       \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("RF_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   int(blockIdx.x), int(threadIdx.x));                                     \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define RF_ASSERT(c) ((void)0)
#endif

namespace rfb {

// Programmatic dependent launch (per-frame kernels): each kernel lets its
// stream successor launch as soon as all of its own CTAs are resident, and
// waits for its predecessor's completion (and memory flush) before touching
// any data. Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- constants
constexpr int kSide = 8;                      // voxels per brick edge (VolumeConfig::block_side)
constexpr int kBrickVoxels = kSide * kSide * kSide;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint32_t kInvalid = 0xFFFFFFFFu;     // slot value before the winner publishes it / not found
constexpr uint32_t kOverflowed = 0xFFFFFFFEu;  // key claimed but no brick left (max_blocks reached)
constexpr int kCoordBias = 1 << 20;           // 21-bit signed range per axis, as mesh.cpp:31-37
constexpr int kAccN = 30;                     // 21 H + 6 b + E_d + E_c + count
constexpr int kLinkStride = 8;                // u32 per brick link record (32 B)

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
    double ifx, ify;  // 1/fx, 1/fy (tracking passes back-project with reciprocals)
};

// Device view of one sparse volume (hash + brick pool).
struct VolumeView {
    HashSlot* slots;
    uint32_t hash_mask;
    uint32_t max_blocks;
    int4* coords;        // brick coordinate per pool index; w = its hash slot
    Voxel* voxels;       // pool, kBrickVoxels per brick, x fastest then y then z
    uint32_t* links;     // kLinkStride per HASH SLOT: [0] the slot's brick, [q] the brick at +(q&1, q>>1&1, q>>2)
    uint32_t* counters;  // see VolumeCounters
    uint32_t* win_first; // refinement temp volume only: per hash slot, first window entry that allocated it
    // Allocation order (model volumes; null for the refinement scratch/temp
    // volumes, whose brick order is unobservable): per hash slot the smallest
    // allocation ordinal that visited a pending key, and the slots claimed
    // since the last assignment (see hash_insert_ordered / assign_new).
    unsigned long long* ord;
    uint32_t* newlist;
    double voxel_size, truncation;
    double inv_voxel_size;  // 1.0 / voxel_size (the reference's inv_s, tsdf_volume.cpp:336)
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
    kNewBlocks = 5,     // keys claimed by the current allocation (pending until assign_new)
    kLinked = 6,        // bricks [0, kLinked) have link records
    kLinkDone = 7,      // link pass completion counter (last CTA advances kLinked)
    kHalt = 8,          // sticky: an allocation overflowed; later frames of a batch do nothing
    kNumCounters = 9
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
    constexpr uint32_t b = uint32_t(kCoordBias);
    return ((uint32_t(x) + b) | (uint32_t(y) + b) | (uint32_t(z) + b)) < 2u * b;
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

// Slot of a brick key (kInvalid when absent or overflowed).
__device__ __forceinline__ uint32_t hash_find_slot(const VolumeView& V, int x, int y, int z) {
    if (!coord_in_range(x, y, z)) return kInvalid;
    const unsigned long long key = pack_key(x, y, z);
    uint32_t idx = hash_coord(x, y, z) & V.hash_mask;
    for (uint32_t probe = 0; probe <= V.hash_mask; ++probe) {
        const uint4 s = __ldg(reinterpret_cast<const uint4*>(V.slots + idx));
        const unsigned long long k = (unsigned long long)s.x | ((unsigned long long)s.y << 32);
        if (k == key) return s.z >= kOverflowed ? kInvalid : idx;
        if (k == kEmptyKey) return kInvalid;
        idx = (idx + 1) & V.hash_mask;
    }
    return kInvalid;
}

// Continues a linear probe after slot `idx` missed; returns the key's slot
// (kInvalid when absent).
__device__ __forceinline__ uint32_t hash_find_slot_from(const VolumeView& V, unsigned long long key, uint32_t idx) {
    for (uint32_t probe = 0; probe < V.hash_mask; ++probe) {
        idx = (idx + 1) & V.hash_mask;
        const uint4 s = __ldg(reinterpret_cast<const uint4*>(V.slots + idx));
        const unsigned long long k = (unsigned long long)s.x | ((unsigned long long)s.y << 32);
        if (k == key) return idx;
        if (k == kEmptyKey) return kInvalid;
    }
    return kInvalid;
}

// Lock-free linear-probing insert (no deletion). Returns 1 when this thread
// created the brick, 0 when it already existed, -1 on overflow.
__device__ __forceinline__ int hash_insert(const VolumeView& V, int x, int y, int z, uint32_t* slot_out = nullptr) {
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
            if (slot_out) *slot_out = idx;
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
                V.coords[b] = make_int4(x, y, z, int(idx));  // w = hash slot (volume reset)
                V.slots[idx].value = b;
                if (slot_out) *slot_out = idx;
                return 1;
            }
            if (old == key) {
                if (*reinterpret_cast<volatile uint32_t*>(&V.slots[idx].value) == kOverflowed) {
                    atomicOr(&V.counters[kOverflow], 1u);
                    return -1;
                }
                if (slot_out) *slot_out = idx;
                return 0;
            }
        }
        idx = (idx + 1) & V.hash_mask;
    }
    atomicOr(&V.counters[kOverflow], 4u);
    return -1;
}

// AllocateBlock's insertion in allocation order (tsdf_volume.cpp:64-77,
// 93-113). The first visitor of a key claims its slot with atomicCAS and lists
// the slot; every visit of a still-pending key (value kInvalid: not yet a
// brick) folds its ordinal into ord[slot] with atomicMin. assign_new later
// hands out pool indices by ordinal, so the pool order -- blocks(), Save --
// is the reference's serial order whatever the thread schedule. A pending key
// is invisible to every lookup (hash_find treats kInvalid as absent).
__device__ __forceinline__ void hash_insert_ordered(const VolumeView& V, int x, int y, int z,
                                                    unsigned long long ordinal) {
    if (!coord_in_range(x, y, z)) {
        atomicOr(&V.counters[kOverflow], 2u);
        atomicOr(&V.counters[kHalt], 1u);
        return;
    }
    const unsigned long long key = pack_key(x, y, z);
    uint32_t idx = hash_coord(x, y, z) & V.hash_mask;
    for (uint32_t probe = 0; probe <= V.hash_mask; ++probe) {
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&V.slots[idx].key);
        if (k == kEmptyKey) {
            k = atomicCAS(&V.slots[idx].key, kEmptyKey, key);
            if (k == kEmptyKey) {
                const uint32_t at = atomicAdd(&V.counters[kNewBlocks], 1u);
                RF_ASSERT(at <= V.hash_mask);
                V.newlist[at] = idx;  // <= one entry per slot
                atomicMin(&V.ord[idx], ordinal);
                return;
            }
        }
        if (k == key) {
            if (*reinterpret_cast<volatile uint32_t*>(&V.slots[idx].value) == kInvalid) atomicMin(&V.ord[idx], ordinal);
            return;
        }
        idx = (idx + 1) & V.hash_mask;
    }
    atomicOr(&V.counters[kOverflow], 4u);
    atomicOr(&V.counters[kHalt], 1u);
}

__host__ __device__ __forceinline__ int4 unpack_key(unsigned long long k, uint32_t slot) {
    return make_int4(int(uint32_t(k & 0x1FFFFFu)) - kCoordBias, int(uint32_t((k >> 21) & 0x1FFFFFu)) - kCoordBias,
                     int(uint32_t((k >> 42) & 0x1FFFFFu)) - kCoordBias, int(slot));
}

// Pool indices for the keys claimed since the last assignment: key i gets
// before + rank(i), rank = the number of claimed keys whose first visit came
// earlier (ordinals are unique per key: a pixel walks distinct cells). Keys
// ranked past max_blocks get no brick -- the reference throws at the first of
// them (tsdf_volume.cpp:66-69) -- and stay pending until the host rebuilds
// the table (rf_capi.cu recover_overflow). `on_new(b, coord)` runs for each
// assigned brick; created[ordinal] (explicit AllocateBlock batches, whose
// ordinal is the coordinate's index) receives 1, or -1 past the budget.
// Grid-stride over the claimed keys; each CTA streams all ordinals through
// shared memory in tiles. Reads counters[kBlocksBefore] (== the brick count
// when the allocation started) and counters[kNewBlocks]; CTA 0 publishes
// counters[kNumBlocks] and the overflow flags.
template <class OnNew>
__device__ __forceinline__ void assign_new(const VolumeView& V, OnNew on_new, int* created = nullptr) {
    constexpr int kTile = 256;
    __shared__ unsigned long long s_ord[kTile];
    const uint32_t n = V.counters[kNewBlocks];
    const uint32_t before = V.counters[kBlocksBefore];
    const uint32_t budget = V.max_blocks > before ? V.max_blocks - before : 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        V.counters[kNumBlocks] = before + min(n, budget);
        if (n > budget) {
            atomicOr(&V.counters[kOverflow], 1u);
            atomicOr(&V.counters[kHalt], 1u);
        }
    }
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += stride) {  // CTA-uniform trip count
        const uint32_t i = i0 + threadIdx.x;
        uint32_t slot = 0;
        unsigned long long mine = 0;
        if (i < n) {
            slot = __ldcg(V.newlist + i);
            RF_ASSERT(slot <= V.hash_mask);
            mine = __ldcg(V.ord + slot);
            RF_ASSERT(mine != ~0ull);  // every claimed key has a first visit
        }
        uint32_t rank = 0;
        for (uint32_t t0 = 0; t0 < n; t0 += kTile) {
            __syncthreads();
            const uint32_t m = min(uint32_t(kTile), n - t0);
            for (uint32_t k = threadIdx.x; k < m; k += blockDim.x) s_ord[k] = __ldcg(V.ord + __ldcg(V.newlist + t0 + k));
            __syncthreads();
            for (uint32_t j = 0; j < m; ++j) rank += s_ord[j] < mine;
        }
        if (i < n) {
            RF_ASSERT(rank < n);
            if (rank < budget) {
                const uint32_t b = before + rank;
                RF_ASSERT(b < V.max_blocks);
                const int4 c = unpack_key(__ldcg(&V.slots[slot].key), slot);
                V.coords[b] = c;
                V.slots[slot].value = b;  // (ord[slot] stays: other CTAs may still be ranking against it;
                                          // an assigned slot never becomes pending again)
                if (created) created[mine] = 1;
                on_new(b, c);
            } else if (created) {
                created[mine] = -1;
            }
        }
    }
}

__device__ __forceinline__ const Voxel* brick_ptr(const VolumeView& V, uint32_t b) {
    RF_ASSERT(b < V.max_blocks);
    return V.voxels + size_t(b) * kBrickVoxels;
}

// ---------------------------------------------------------------- sampling
// CellOf + GatherCorners + SampleWithGradientImpl (tsdf_volume.cpp:243-346),
// evaluated for the SDF and the intensity from one gather of the 8 corners.
struct CellSample {
    double sdf, gs[3];   // value and gradient of the SDF interpolant
    double inten, gi[3]; // value and gradient of the intensity interpolant
};

// The 8 corners of the interpolation cell at voxel (bx,by,bz) live in the
// brick of the base voxel and, when the cell straddles brick faces (local
// coordinate 7 on an axis, one cell in three), in its +x/+y/+z neighbours.
// The neighbours come from a link record stored next to the hash slot
// (links[slot * 8 + q] = pool index of the brick at +(q&1, q>>1&1, q>>2)),
// so its load is issued together with the slot's, before the key compare:
// one dependent L2 round trip (slot + record) instead of two, and every
// lane runs the same code.
// n[Q | subset of K's bits], choosing each bit of K by its straddle flag.
template <int K, int Q = 0>
__device__ __forceinline__ uint32_t corner_brick(const uint32_t (&n)[8], bool sx, bool sy, bool sz) {
    if constexpr (K == 0) {
        return n[Q];
    } else {
        constexpr int top = (K & 4) ? 4 : ((K & 2) ? 2 : 1);
        const bool s = top == 4 ? sz : (top == 2 ? sy : sx);
        return s ? corner_brick<K & ~top, Q | top>(n, sx, sy, sz) : corner_brick<K & ~top, Q>(n, sx, sy, sz);
    }
}
__device__ __forceinline__ bool gather_corners(const VolumeView& V, int bx, int by, int bz, uint2 (&c)[8]) {
    const int lx = bx & 7, ly = by & 7, lz = bz & 7;
    const int cx = bx >> 3, cy = by >> 3, cz = bz >> 3;  // arithmetic shift == FloorDiv by 8
    if (!coord_in_range(cx, cy, cz)) return false;
    const unsigned long long key = pack_key(cx, cy, cz);
    uint32_t idx = hash_coord(cx, cy, cz) & V.hash_mask;
    const int smask = int(lx == 7) | (int(ly == 7) << 1) | (int(lz == 7) << 2);
    const uint4 s = __ldg(reinterpret_cast<const uint4*>(V.slots + idx));
    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = r0;
    if (smask) {
        r0 = __ldg(reinterpret_cast<const uint4*>(V.links + size_t(idx) * kLinkStride));
        r1 = __ldg(reinterpret_cast<const uint4*>(V.links + size_t(idx) * kLinkStride) + 1);
    }
    const unsigned long long k = (unsigned long long)s.x | ((unsigned long long)s.y << 32);
    uint32_t b0 = s.z;
    if (k != key) {  // empty slot, or a collision: continue the probe (rare)
        if (k == kEmptyKey) return false;
        idx = hash_find_slot_from(V, key, idx);
        if (idx == kInvalid) return false;
        b0 = __ldg(&V.slots[idx].value);
        if (smask) {
            r0 = __ldg(reinterpret_cast<const uint4*>(V.links + size_t(idx) * kLinkStride));
            r1 = __ldg(reinterpret_cast<const uint4*>(V.links + size_t(idx) * kLinkStride) + 1);
        }
    }
    // The brick of corner (dx, dy, dz) is n[q], q = (dx & sx) | (dy & sy) << 1 |
    // (dz & sz) << 2 with s* the straddle flags: a select tree on the three
    // flags over the corner's own axes (19 selects for the 8 corners, no
    // compare per candidate). Unloaded record words are never selected.
    const uint32_t n[8] = {b0, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const bool sx = lx == 7, sy = ly == 7, sz = lz == 7;
    bool bad = false;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int dx = kk & 1, dy = (kk >> 1) & 1, dz = kk >> 2;  // compile-time corner offset
        uint32_t b;
        switch (kk) {
            case 0: b = corner_brick<0>(n, sx, sy, sz); break;
            case 1: b = corner_brick<1>(n, sx, sy, sz); break;
            case 2: b = corner_brick<2>(n, sx, sy, sz); break;
            case 3: b = corner_brick<3>(n, sx, sy, sz); break;
            case 4: b = corner_brick<4>(n, sx, sy, sz); break;
            case 5: b = corner_brick<5>(n, sx, sy, sz); break;
            case 6: b = corner_brick<6>(n, sx, sy, sz); break;
            default: b = corner_brick<7>(n, sx, sy, sz); break;
        }
        // Straight-line from here: an absent or overflowed brick (index >=
        // kOverflowed) is remembered in `bad` and its corner loaded from brick 0
        // instead (a mapped address), so the 8 loads issue back to back without
        // a branch between them; the cell is rejected once, after the loads.
        bad |= b >= kOverflowed;
        b = b >= kOverflowed ? 0u : b;
        const int ox = (lx + dx) & 7, oy = (ly + dy) & 7, oz = (lz + dz) & 7;
        c[kk] = __ldg(reinterpret_cast<const uint2*>(brick_ptr(V, b)) + ((oz * 8 + oy) * 8 + ox));
    }
    bool ok = !bad;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) ok = ok && (c[kk].y & 0xFFu) != 0u;  // weight byte
    return ok;
}

// Link records (tsdf_volume.hpp:149-185 allocates; this only indexes): the
// record at brick b's hash slot (coords[b].w) lists the pool indices of its
// "+" neighbours, and b is entered into its "-" neighbours' records. Every
// write is a pure function of the key set, so concurrent writers of the same
// word agree.
// One word of link_brick: dir 0 fills own[q] (q = 0: the brick itself),
// dir 1 points the "-q" neighbour's record at b.
__device__ __forceinline__ void link_brick_item(const VolumeView& V, uint32_t b, int q, int dir) {
    RF_ASSERT(b < V.max_blocks);
    const int4 c = V.coords[b];
    RF_ASSERT(uint32_t(c.w) <= V.hash_mask);
    if (dir == 0) {
        V.links[size_t(uint32_t(c.w)) * kLinkStride + q] =
            q == 0 ? b : hash_find(V, c.x + (q & 1), c.y + ((q >> 1) & 1), c.z + (q >> 2));
    } else if (q != 0) {
        const uint32_t sa = hash_find_slot(V, c.x - (q & 1), c.y - ((q >> 1) & 1), c.z - (q >> 2));
        if (sa != kInvalid) V.links[size_t(sa) * kLinkStride + q] = b;
    }
}

__device__ __forceinline__ float voxel_sdf(uint2 v) { return __uint_as_float(v.x); }
__device__ __forceinline__ double voxel_luma(uint2 v) {
    return luma(uint8_t(v.y >> 8), uint8_t(v.y >> 16), uint8_t(v.y >> 24));
}
// Same value from a table of the three weighted channels (lut[c*256 + x] =
// w_c * x, each product rounded as in luma()), summed in luma()'s order:
// bit-identical, 3 shared loads instead of 3 int->f64 conversions + 3 DMUL.
__device__ __forceinline__ double voxel_luma_lut(uint2 v, const double* lut) {
    return (lut[(v.y >> 8) & 0xFFu] + lut[256 + ((v.y >> 16) & 0xFFu)]) + lut[512 + (v.y >> 24)];
}

// a / b correctly rounded from rb = RN(1 / b): q = RN(a rb) is within an ulp,
// the FMA residual is exact, and one correction step rounds correctly
// (Markstein); no IEEE division sequence on the walk's setup chain. A zero
// quotient comes out +0 where a / b gives -0; the walk only floors and
// subtracts these values, where the two zeros agree.
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double q = a * rb;
    return __fma_rn(__fma_rn(-q, b, a), rb, q);
}

// CellOf (tsdf_volume.cpp:279-283). kExact divides like the reference (the
// quotient correctly rounded through the reciprocal, div_rn); the
// tracking passes multiply by the precomputed reciprocal (last-bit
// differences only; parity there is held on the normal equations and poses).
template <bool kExact>
__device__ __forceinline__ void cell_of(double px, double py, double pz, const VolumeView& V, int base[3], double f[3]) {
    double g[3];
    if (kExact) {
        g[0] = div_rn(px, V.voxel_size, V.inv_voxel_size) - 0.5;
        g[1] = div_rn(py, V.voxel_size, V.inv_voxel_size) - 0.5;
        g[2] = div_rn(pz, V.voxel_size, V.inv_voxel_size) - 0.5;
    } else {
        g[0] = px * V.inv_voxel_size - 0.5;
        g[1] = py * V.inv_voxel_size - 0.5;
        g[2] = pz * V.inv_voxel_size - 0.5;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double fl = floor(g[i]);
        base[i] = int(fl);
        f[i] = g[i] - fl;
    }
}

// Trilinear value and analytic gradient (tsdf_volume.cpp:319-346) of the
// SDF and intensity interpolants from the 8 gathered corners.
template <bool kGrad, bool kIntensity>
__device__ __forceinline__ void interp_cell(const VolumeView& V, const uint2 (&c)[8], const double f[3],
                                            CellSample& out, const double* lut) {
    const double wx[2] = {1.0 - f[0], f[0]};
    const double wy[2] = {1.0 - f[1], f[1]};
    const double wz[2] = {1.0 - f[2], f[2]};
    double vs[8], vi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        vs[k] = double(voxel_sdf(c[k]));
        if (kIntensity) vi[k] = lut ? voxel_luma_lut(c[k], lut) : voxel_luma(c[k]);
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
        const double inv_s = V.inv_voxel_size;  // 1.0 / voxel_size, computed once on the host
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
}

// Exact integer Rec.709 luma times 1e4 (2126 r + 7152 g + 722 b < 2^22) as a
// double, without a conversion instruction: OR into the mantissa of 2^52.
// The weights split into bytes (2126 = 8 * 256 + 78, 7152 = 27 * 256 + 240,
// 722 = 2 * 256 + 210) make the sum two byte dot products: L = 256 dp4a(v, hi)
// + dp4a(v, lo) over the bytes {weight, r, g, b} (weight's multiplier 0).
__device__ __forceinline__ double voxel_luma_e4(uint2 v) {
    constexpr unsigned kHi = (2u << 24) | (27u << 16) | (8u << 8), kLo = (210u << 24) | (240u << 16) | (78u << 8);
    const unsigned int L = (__dp4a(v.y, kHi, 0u) << 8) + __dp4a(v.y, kLo, 0u);
    return __longlong_as_double(0x4330000000000000ll | (long long)L) - 4503599627370496.0;
}

// The same interpolant and gradients for the tracking Jacobian passes, as
// nested lerps with fused multiply-adds (shorter dependency chains, about
// half the fp64 instructions) and the intensity from exact integer lumas
// scaled once. Differs from interp_cell in the last bits only; the Jacobian
// passes are held to the normal-equation (1e-9) and pose (1e-4) bars, the
// value passes that must be bit-exact keep interp_cell.
template <bool kIntensity>
__device__ __forceinline__ void interp_cell_fast(const VolumeView& V, const uint2 (&c)[8], const double f[3],
                                                 CellSample& out) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = double(voxel_sdf(c[k]));
    // x-differences at the four (y, z) edges, then lerps in y and z
    const double dx00 = v[1] - v[0], dx10 = v[3] - v[2], dx01 = v[5] - v[4], dx11 = v[7] - v[6];
    const double x00 = __fma_rn(f[0], dx00, v[0]), x10 = __fma_rn(f[0], dx10, v[2]);
    const double x01 = __fma_rn(f[0], dx01, v[4]), x11 = __fma_rn(f[0], dx11, v[6]);
    const double y0 = __fma_rn(f[1], x10 - x00, x00), y1 = __fma_rn(f[1], x11 - x01, x01);
    out.sdf = __fma_rn(f[2], y1 - y0, y0);
    const double inv_s = V.inv_voxel_size;
    {
        const double gxz0 = __fma_rn(f[1], dx10 - dx00, dx00), gxz1 = __fma_rn(f[1], dx11 - dx01, dx01);
        out.gs[0] = __fma_rn(f[2], gxz1 - gxz0, gxz0) * inv_s;
        out.gs[1] = __fma_rn(f[2], (x11 - x01) - (x10 - x00), x10 - x00) * inv_s;
        out.gs[2] = (y1 - y0) * inv_s;
    }
    if (kIntensity) {
        double q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = voxel_luma_e4(c[k]);
        const double ex00 = q[1] - q[0], ex10 = q[3] - q[2], ex01 = q[5] - q[4], ex11 = q[7] - q[6];
        const double a00 = __fma_rn(f[0], ex00, q[0]), a10 = __fma_rn(f[0], ex10, q[2]);
        const double a01 = __fma_rn(f[0], ex01, q[4]), a11 = __fma_rn(f[0], ex11, q[6]);
        const double b0 = __fma_rn(f[1], a10 - a00, a00), b1 = __fma_rn(f[1], a11 - a01, a01);
        constexpr double kE4 = 1e-4;
        out.inten = __fma_rn(f[2], b1 - b0, b0) * kE4;
        const double gz0 = __fma_rn(f[1], ex10 - ex00, ex00), gz1 = __fma_rn(f[1], ex11 - ex01, ex01);
        const double s = inv_s * kE4;
        out.gi[0] = __fma_rn(f[2], gz1 - gz0, gz0) * s;
        out.gi[1] = __fma_rn(f[2], (a11 - a01) - (a10 - a00), a10 - a00) * s;
        out.gi[2] = (b1 - b0) * s;
    }
}

template <bool kGrad, bool kIntensity, bool kExact = true>
__device__ __forceinline__ bool sample_point(const VolumeView& V, const double p[3], CellSample& out,
                                             const double* lut = nullptr) {
    int base[3];
    double f[3];
    cell_of<kExact>(p[0], p[1], p[2], V, base, f);
    uint2 c[8];
    if (!gather_corners(V, base[0], base[1], base[2], c)) return false;
    if (!kExact && kGrad) interp_cell_fast<kIntensity>(V, c, f, out);
    else interp_cell<kGrad, kIntensity>(V, c, f, out, lut);
    return true;
}

// ---------------------------------------------------------------- grid sync
// Barrier + all-reduce across a cooperative grid: every CTA writes its
// partial vector, the last CTA to arrive folds all partials in CTA order
// (fixed order => run-to-run deterministic) and publishes the result, then
// releases the others. One L2 round trip per waiting CTA.
constexpr int kArriveLanes = 8;  // (<= 32) arrival counters on separate 128-B lines (parallel L2 atomics)
struct GridSync {
    unsigned long long lane[2][kArriveLanes][16];  // [launch parity][lane][0] = arrivals, rest padding
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
