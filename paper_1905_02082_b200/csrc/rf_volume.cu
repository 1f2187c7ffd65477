// Sparse-volume kernels: ray-segment brick allocation into the open-addressed
// hash, frustum culling into a compacted visible-brick list, and one fused
// carve+integrate sweep per visible 8^3 brick (one thread per voxel, the brick
// read and written once, coalesced 8-byte voxels).
#include "rf_volume.cuh"

namespace rfb {

// ---------------------------------------------------------------- allocation
// AllocateForFrame + WalkGridSegment (tsdf_volume.cpp:93-113,
// tsdf_volume.hpp:149-185), one thread per pixel, all cells inserted with
// atomicCAS. The set of inserted keys, and so the occupied-slot set of the
// linear-probing table, is independent of thread order.
// The ray segment of pixel p (AllocateForFrame, tsdf_volume.cpp:93-113):
// [max(d - tau, 1e-4), d + tau] along the pixel's ray, walked through the
// block grid (WalkGridSegment, tsdf_volume.hpp:149-185); `visit(cell)` for
// every block cell in order. Returns the cells visited (0: pixel unusable).
template <class Visit>
__device__ __forceinline__ unsigned walk_pixel(const VolumeView& V, const float* depth, const uint8_t* mask,
                                               const Intr& K, const double* pose, int p, Visit visit) {
    const int u = p % K.w, v = p / K.w;
    const float d = __ldg(depth + p);
    const bool masked = mask && __ldg(mask + p);
    if (!(depth_valid(d) && !(d < V.min_depth) && !(d > V.max_depth) && !masked)) return 0;
    Pose P;
    for (int i = 0; i < 12; ++i) (i < 9 ? P.R[i] : P.t[i - 9]) = __ldg(pose + i);
    const double tau = V.truncation;
    const double ext = double(kSide) * V.voxel_size;  // block_extent(), tsdf_volume.hpp:123
    const double rext = V.inv_voxel_size * (1.0 / double(kSide));  // RN(1/ext): RN(1/s) scaled by 2^-3
    const double dir0 = div_rn(double(u) - K.cx, K.fx, K.ifx), dir1 = div_rn(double(v) - K.cy, K.fy, K.ify);
    const double z0 = fmax(double(d) - tau, 1e-4);
    const double z1 = double(d) + tau;
    double w0[3], w1[3];
    pose_apply(P, z0 * dir0, z0 * dir1, z0 * 1.0, w0);
    pose_apply(P, z1 * dir0, z1 * dir1, z1 * 1.0, w1);
    const double p0[3] = {div_rn(w0[0], ext, rext), div_rn(w0[1], ext, rext), div_rn(w0[2], ext, rext)};
    const double p1[3] = {div_rn(w1[0], ext, rext), div_rn(w1[1], ext, rext), div_rn(w1[2], ext, rext)};
    int cell[3], end[3], step[3];
    double tmax[3], tdel[3];
    for (int i = 0; i < 3; ++i) {
        const double dd = p1[i] - p0[i];
        cell[i] = int(floor(p0[i]));
        end[i] = int(floor(p1[i]));
        step[i] = 0;
        tmax[i] = tdel[i] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        if (dd > 0) {
            step[i] = 1;
            tmax[i] = (floor(p0[i]) + 1.0 - p0[i]) / dd;
            tdel[i] = 1.0 / dd;
        } else if (dd < 0) {
            step[i] = -1;
            tmax[i] = (p0[i] - floor(p0[i])) / -dd;
            tdel[i] = 1.0 / -dd;
        }
    }
    const int max_steps = abs(end[0] - cell[0]) + abs(end[1] - cell[1]) + abs(end[2] - cell[2]) + 3;
    unsigned visits = 1;
    visit(cell);
    // The step loop on scalars (a runtime axis index would put tmax / cell in
    // local memory): the same comparisons and updates as WalkGridSegment.
    double t0 = tmax[0], t1 = tmax[1], t2 = tmax[2];
    for (int n = 0; n < max_steps && (cell[0] != end[0] || cell[1] != end[1] || cell[2] != end[2]); ++n) {
        const bool a1 = t1 < t0;
        const double tm01 = a1 ? t1 : t0;
        const bool a2 = t2 < tm01;
        const double tmin = a2 ? t2 : tm01;
        if (tmin > 1.0) break;
        if (a2) {
            t2 += tdel[2];
            cell[2] += step[2];
        } else if (a1) {
            t1 += tdel[1];
            cell[1] += step[1];
        } else {
            t0 += tdel[0];
            cell[0] += step[0];
        }
        visit(cell);
        ++visits;
    }
    return visits;
}

__global__ void k_alloc(AllocArgs a) {
    pdl_enter();
    if (a.lost && *a.lost) return;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned visits = 0;
    if (p < a.K.w * a.K.h) {
        // The walk runs one cell ahead of the inserts: the first hash slot of
        // the next cell is loaded while the current one is checked, and a cell
        // whose brick already sits in its first slot (almost all of them once
        // the scene is mapped) needs no atomic. Same key set as inserting every
        // visited cell (inserting a present key is a no-op). Model volumes
        // insert in allocation order: the ordinal of a visit is (pixel, step),
        // AllocateForFrame's raster order (tsdf_volume.cpp:96-111).
        const bool ordered = a.V.ord != nullptr;
        auto first_slot = [&](const int (&c)[3]) -> uint4 {
            if (!coord_in_range(c[0], c[1], c[2])) return make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u);
            return __ldg(reinterpret_cast<const uint4*>(a.V.slots + (hash_coord(c[0], c[1], c[2]) & a.V.hash_mask)));
        };
        auto settle = [&](const int (&c)[3], uint4 sl, unsigned step) {
            const unsigned long long k = (unsigned long long)sl.x | ((unsigned long long)sl.y << 32);
            if (coord_in_range(c[0], c[1], c[2]) && k == pack_key(c[0], c[1], c[2]) && sl.z < kOverflowed) return;
            if (ordered) hash_insert_ordered(a.V, c[0], c[1], c[2], ((unsigned long long)p << 32) | step);
            else hash_insert(a.V, c[0], c[1], c[2]);
        };
        int cur[3] = {0, 0, 0};
        uint4 cur_sl = make_uint4(0, 0, 0, 0);
        unsigned step = 0;
        visits = walk_pixel(a.V, a.depth, a.mask, a.K, a.pose, p, [&](const int (&c)[3]) {
            const uint4 next_sl = first_slot(c);
            if (step) settle(cur, cur_sl, step - 1);
            cur[0] = c[0];
            cur[1] = c[1];
            cur[2] = c[2];
            cur_sl = next_sl;
            ++step;
        });
        if (step) settle(cur, cur_sl, step - 1);
    }
    // warp-aggregated visit counter (for the algorithmic-bytes model)
    for (int o = 16; o > 0; o >>= 1) visits += __shfl_down_sync(0xffffffffu, visits, o);
    if ((threadIdx.x & 31) == 0 && visits) atomicAdd(&a.V.counters[kDdaVisits], visits);
}

// Explicit AllocateBlock (tsdf_volume.cpp:64-77) for a batch of coordinates,
// in index order on model volumes (ordinal = index; created[] is filled by
// k_assign), else unordered with created[i] = 1 / 0 / -1.
__global__ void k_alloc_coords(VolumeView V, const int* coords, int n, int* created) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (V.ord) {
        hash_insert_ordered(V, coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], (unsigned long long)i);
        return;
    }
    const int r = hash_insert(V, coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]);
    if (created) created[i] = r;
}

// Pool indices for an allocation's claimed keys (assign_new), standalone.
__global__ void k_assign(VolumeView V, int* created) {
    assign_new(V, [](uint32_t, int4) {}, created);
}

// ---------------------------------------------------------------- culling
// BlockOutsideFrustum (tsdf_volume.cpp:119-151) for every allocated brick,
// evaluated once for the carve bound (carve_clip) and the integrate bound
// (max_depth + truncation). Visible bricks are appended with their flags.
// The part of BlockOutsideFrustum that does not depend on the depth bound:
// min corner depth, and whether the brick is outside for any bound (corners
// behind the camera, or the projected corner box off the image). Then
// outside(max_z) = min_z > max_z || rest: the 16 divisions run once for both
// of k_cull's bounds.
struct FrustumTest {
    double min_z;
    bool rest;
    __device__ bool outside(double max_z) const { return min_z > max_z || rest; }
};
__device__ __forceinline__ FrustumTest frustum_test(const double cc[8][3], const Intr& K) {
    bool any_behind = false, any_front = false;
    double min_z = __longlong_as_double(0x7ff0000000000000ll);
    for (int c = 0; c < 8; ++c) {
        if (cc[c][2] <= 1e-9) any_behind = true;
        if (cc[c][2] > 1e-9) any_front = true;
        min_z = fmin(min_z, cc[c][2]);
    }
    if (any_behind) return {min_z, !any_front};
    double min_u = __longlong_as_double(0x7ff0000000000000ll), max_u = -min_u, min_v = min_u, max_v = -min_u;
    for (int c = 0; c < 8; ++c) {
        const double pu = K.fx * cc[c][0] / cc[c][2] + K.cx;
        const double pv = K.fy * cc[c][1] / cc[c][2] + K.cy;
        min_u = fmin(min_u, pu);
        max_u = fmax(max_u, pu);
        min_v = fmin(min_v, pv);
        max_v = fmax(max_v, pv);
    }
    return {min_z, max_u < -0.5 || min_u > K.w - 0.5 || max_v < -0.5 || min_v > K.h - 0.5};
}

__device__ __forceinline__ void cull_brick(const CullArgs& a, const Pose& W, double ext, int4 c, bool carve,
                                           bool integrate, uint32_t& flags) {
    double cc[8][3];
    for (int k = 0; k < 8; ++k) {
        const double x = (double(c.x) + double(k & 1)) * ext;
        const double y = (double(c.y) + double((k >> 1) & 1)) * ext;
        const double z = (double(c.z) + double(k >> 2)) * ext;
        pose_apply(W, x, y, z, cc[k]);
    }
    const FrustumTest ft = frustum_test(cc, a.K);
    if (carve && !ft.outside(a.V.carve_clip)) flags |= kFlagCarve;
    if (integrate && !ft.outside(a.V.max_depth + a.V.truncation)) flags |= kFlagIntegrate;
}

// The same test with the brick's 8 corners on 8 consecutive lanes (corner k
// on lane k of the group): each lane projects its corner, the group combines
// the flags and extremes with shuffles (min / max / or are exact and order
// free), so a brick costs one corner's chain instead of eight. Every lane of
// the group returns the brick's flags.
__device__ __forceinline__ uint32_t cull_brick_lanes(const CullArgs& a, const Pose& W, double ext, int4 c, int k,
                                                     bool carve, bool integrate) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double cc[3];
    pose_apply(W, (double(c.x) + double(k & 1)) * ext, (double(c.y) + double((k >> 1) & 1)) * ext,
               (double(c.z) + double(k >> 2)) * ext, cc);
    bool behind = cc[2] <= 1e-9, front = cc[2] > 1e-9;
    double min_z = fmin(inf, cc[2]), min_u = inf, max_u = -inf, min_v = inf, max_v = -inf;
    if (front) {
        min_u = max_u = a.K.fx * cc[0] / cc[2] + a.K.cx;  // (as frustum_test)
        min_v = max_v = a.K.fy * cc[1] / cc[2] + a.K.cy;
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        behind = __shfl_xor_sync(0xffffffffu, behind, o) || behind;
        front = __shfl_xor_sync(0xffffffffu, front, o) || front;
        min_z = fmin(min_z, __shfl_xor_sync(0xffffffffu, min_z, o));
        min_u = fmin(min_u, __shfl_xor_sync(0xffffffffu, min_u, o));
        max_u = fmax(max_u, __shfl_xor_sync(0xffffffffu, max_u, o));
        min_v = fmin(min_v, __shfl_xor_sync(0xffffffffu, min_v, o));
        max_v = fmax(max_v, __shfl_xor_sync(0xffffffffu, max_v, o));
    }
    const FrustumTest ft{min_z, behind ? !front
                                       : (max_u < -0.5 || min_u > a.K.w - 0.5 || max_v < -0.5 || min_v > a.K.h - 0.5)};
    uint32_t flags = 0;
    if (carve && !ft.outside(a.V.carve_clip)) flags |= kFlagCarve;
    if (integrate && !ft.outside(a.V.max_depth + a.V.truncation)) flags |= kFlagIntegrate;
    return flags;
}

// Appends the brick of every lane with flags to the visible list (one atomic per warp).
__device__ __forceinline__ void append_visible(const CullArgs& a, uint32_t b, uint32_t flags) {
    const unsigned vote = __ballot_sync(0xffffffffu, flags != 0);
    if (vote) {  // lanes take consecutive slots
        const int lane = threadIdx.x & 31;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&a.V.counters[kVisible], uint32_t(__popc(vote)));
        base = __shfl_sync(0xffffffffu, base, 0);
        RF_ASSERT(!flags || base + __popc(vote & ((1u << lane) - 1u)) < a.V.max_blocks);
        if (flags) a.list[base + __popc(vote & ((1u << lane) - 1u))] = b | flags;
    }
}

__global__ void k_cull(CullArgs a) {
    pdl_enter();
    if (a.lost && *a.lost) return;
    // With `assign`, this frame's allocation (k_alloc) left its new keys
    // pending: they receive their pool indices here (assign_new) and are culled
    // by the thread that assigns them, while the other threads cull the bricks
    // that existed before the frame. An overflowing allocation integrates
    // nothing (AllocateForFrame throws before Integrate, tsdf_volume.cpp:66-69;
    // the carve already happened, pipeline.cpp:26-28).
    const uint32_t old_n = a.assign ? a.V.counters[kBlocksBefore] : min(a.V.counters[kNumBlocks], a.V.max_blocks);
    const uint32_t before = a.carve_only_before ? min(a.V.counters[kBlocksBefore], old_n) : old_n;
    bool overflow = a.V.counters[kOverflow] != 0;
    if (a.assign) {
        const uint32_t n = a.V.counters[kNewBlocks];
        overflow = overflow || n > (a.V.max_blocks > old_n ? a.V.max_blocks - old_n : 0u);
    }
    const bool integrate = a.do_integrate && !overflow;
    Pose P;
    for (int i = 0; i < 12; ++i) (i < 9 ? P.R[i] : P.t[i - 9]) = __ldg(a.pose + i);
    const Pose W = pose_inverse(P);
    const double ext = double(kSide) * a.V.voxel_size;
    if (a.assign)
        assign_new(a.V, [&](uint32_t b, int4 c) {
            uint32_t flags = 0;
            cull_brick(a, W, ext, c, false, integrate, flags);  // new bricks: integrate only
            if (flags) {
                const uint32_t at = atomicAdd(&a.V.counters[kVisible], 1u);
                RF_ASSERT(at < a.V.max_blocks);
                a.list[at] = b | flags;
            }
        });
    const uint32_t stride = gridDim.x * blockDim.x;
    // 8 lanes per brick (one per corner), warp-uniform trip count so the whole
    // warp can aggregate its appends (the group's corner-0 lane appends)
    const uint64_t items = uint64_t(old_n) * 8u;
    for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); i0 < items; i0 += stride) {
        const uint64_t i = i0 + (threadIdx.x & 31u);
        const uint32_t b = uint32_t(i >> 3);
        const bool live = i < items;
        const uint32_t fl = cull_brick_lanes(a, W, ext, a.V.coords[live ? b : 0u], int(i & 7u),
                                             a.do_carve && b < before, integrate);
        append_visible(a, b, (live && (i & 7u) == 0) ? fl : 0u);
    }
}

// Link records for bricks allocated since the last link pass: grid-stride
// over [kLinked, num_blocks). The range is committed afterwards (commit_links
// in the next kernel on the stream, or link_new_commit's completion count).
// One thread per (brick, neighbour q, direction): the 14 hash probes of a
// brick's record run in parallel instead of as one thread's serial chain.
__device__ void link_new(const VolumeView& V) {
    const uint32_t hi = min(V.counters[kNumBlocks], V.max_blocks);
    const uint32_t lo = min(V.counters[kLinked], hi);
    const uint32_t items = (hi - lo) * 16u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x)
        link_brick_item(V, lo + i / 16u, int(i & 7u), int((i >> 3) & 1u));
}

__device__ __forceinline__ void commit_links(const VolumeView& V) {
    if (blockIdx.x == 0 && threadIdx.x == 0) V.counters[kLinked] = min(V.counters[kNumBlocks], V.max_blocks);
}

// link_new, then the last CTA to finish advances kLinked (kernels that cannot
// leave the commit to a successor).
__device__ void link_new_commit(const VolumeView& V) {
    __shared__ bool s_last;
    const uint32_t hi = min(V.counters[kNumBlocks], V.max_blocks);
    if (V.counters[kLinked] >= hi) return;  // nothing new (CTA-uniform)
    link_new(V);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this CTA's link records before its arrival
        s_last = atomicAdd(&V.counters[kLinkDone], 1u) == gridDim.x - 1;
        if (s_last) {
            V.counters[kLinked] = hi;
            V.counters[kLinkDone] = 0;
        }
    }
}

__global__ void k_link(VolumeView V) { link_new(V); }
__global__ void k_link_commit(VolumeView V) { commit_links(V); }

// ---------------------------------------------------------------- fusion
// CarveFreeSpace (tsdf_volume.cpp:204-241) then Integrate (:155-202) applied
// voxel by voxel inside one brick; the sdf is rounded to f32 between the two
// updates exactly as the sequential reference stores it.
// Exact arithmetic shortcuts for the fused update (results bit-identical to
// the reference's divisions, which stay as the fallback):
//  * Project: x = fx * X / Z + cx only feeds lround, so a reciprocal-based x
//    (within a few ulp) is exact unless x lies within 1e-9 of a half-integer;
//  * sdf = f32((sdf * w + u) / (w + k)): the quotient from a correctly rounded
//    reciprocal (table) is within 3 ulp of the f64 quotient; when every f64
//    in q * (1 +- 2^-50) rounds to the same f32, that f32 is the result;
//  * colour: lround(n / d) of integers n >= 0, d <= 256 is (2n + d) / (2d)
//    (no f64 quotient of such a fraction is within rounding of a half).
__device__ __forceinline__ double fuse_rcp(double x) {  // ~1 ulp, branch-free
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    return __fma_rn(r, __fma_rn(-x, r, 1.0), r);
}
// The pixel coordinate, or -1 for any value outside [0, INT_MAX] (the caller
// only tests 0 <= p < width). Away from half-integers every round-to-nearest
// agrees with lround, so the fast path converts with one F2I.
__device__ __forceinline__ int project_lround(double num, double z, double rz, double c) {
    const double xa = num * rz + c;
    const double fr = xa - floor(xa);
    if (fabs(xa) < 1e6 && fabs(fr - 0.5) > 1e-9) return __double2int_rn(xa);
    const long l = lround(num / z + c);  // Project, geometry.hpp:46-48
    return (l < 0 || l > 0x7fffffffL) ? -1 : int(l);
}
__device__ __forceinline__ float div_f32(double a, double b, double rb) {
    const double q = a * rb;
    const float lo = __double2float_rn(q * (1.0 - 0x1p-50)), hi = __double2float_rn(q * (1.0 + 0x1p-50));
    return lo == hi ? lo : float(a / b);
}
// lround((c * w + in) / (w + 1)) (tsdf_volume.cpp:190-196) = (2n + d) / (2d) with
// n = c * w + in, d = w + 1, as the high word of a multiply by M = ceil(2^32 /
// (2d)): exact for every numerator < 2^17 (n <= 255 * 255 + 255) and 2d <= 512
// (checked exhaustively: tools/micro/colour_magic.c), one IMAD.HI and no integer
// division on the per-voxel path.
__device__ __forceinline__ uint32_t colour_avg(uint32_t c, uint32_t w, uint32_t in, const uint32_t* cdiv) {
    const uint32_t d = w + 1u;
    return __umulhi(2u * (c * w + in) + d, cdiv[d]);
}
__device__ __forceinline__ uint32_t colour_magic(uint32_t d) {  // ceil(2^32 / (2d)), d >= 1
    return uint32_t(((1ull << 32) + 2ull * d - 1ull) / (2ull * d));
}

__global__ void __launch_bounds__(kBrickVoxels) k_fuse(FuseArgs a) {
    pdl_enter();
    if (a.lost && *a.lost) return;
    link_new_commit(a.V);  // index the bricks k_cull assigned, for the next frame's tracking
    __shared__ Pose W;
    __shared__ double s_rcp[512];  // RN(1 / i): i = w + 1 (integrate) or w + carve_weight (carve), <= 510
    __shared__ uint32_t s_cdiv[257];  // colour_avg multipliers by d = w + 1
    if (threadIdx.x == 0) {
        Pose P;
        for (int i = 0; i < 12; ++i) (i < 9 ? P.R[i] : P.t[i - 9]) = a.pose[i];
        W = pose_inverse(P);
    }
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s_rcp[i] = i ? 1.0 / double(i) : 0.0;
    for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdiv[i] = i ? colour_magic(uint32_t(i)) : 0u;
    __syncthreads();
    const uint32_t nvis = a.V.counters[kVisible];
    const int x = threadIdx.x & 7, y = (threadIdx.x >> 3) & 7, z = threadIdx.x >> 6;
    const double s = a.V.voxel_size, tau = a.V.truncation;
    const int cw = a.V.carve_weight, mw = a.V.max_weight;
    // Software-pipelined over this CTA's bricks: the list entry two bricks
    // ahead and the coordinates + this thread's voxel one brick ahead are in
    // flight while the current brick projects and reads the frame, so each
    // step waits on one dependent round trip (the depth gather), not four.
    const uint32_t G = gridDim.x;
    uint32_t i = blockIdx.x;
    uint32_t e_nx = i < nvis ? __ldcg(a.list + i) : 0u;
    uint32_t e_nx2 = i + G < nvis ? __ldcg(a.list + i + G) : 0u;
    int4 c_nx = make_int4(0, 0, 0, 0);
    uint2 v_nx = make_uint2(0, 0);
    uint2* p_nx = nullptr;  // this thread's voxel of the next brick
    if (i < nvis) {
        c_nx = a.V.coords[e_nx & kIndexMask];
        p_nx = reinterpret_cast<uint2*>(a.V.voxels + size_t(e_nx & kIndexMask) * kBrickVoxels + threadIdx.x);
        v_nx = *p_nx;
    }
    const bool has_mask = a.mask != nullptr, has_rgb = a.rgb != nullptr;
    RF_ASSERT(nvis <= a.V.max_blocks);
    for (; i < nvis; i += G) {
        const uint32_t e = e_nx;
        RF_ASSERT((e & kIndexMask) < min(a.V.counters[kNumBlocks], a.V.max_blocks));
        const int4 c = c_nx;
        uint2 raw = v_nx;
        uint2* const vp = p_nx;
        e_nx = e_nx2;
        if (i + 2 * G < nvis) e_nx2 = __ldcg(a.list + i + 2 * G);
        if (i + G < nvis) {
            c_nx = a.V.coords[e_nx & kIndexMask];
            p_nx = reinterpret_cast<uint2*>(a.V.voxels + size_t(e_nx & kIndexMask) * kBrickVoxels + threadIdx.x);
            v_nx = *p_nx;
        }
        const double cx = (double(c.x * kSide + x) + 0.5) * s;  // VoxelCenter, tsdf_volume.hpp:117-119
        const double cy = (double(c.y * kSide + y) + 0.5) * s;
        const double cz = (double(c.z * kSide + z) + 0.5) * s;
        double pc[3];
        pose_apply(W, cx, cy, cz, pc);
        if (!(pc[2] <= 1e-9)) {
            const double rz = fuse_rcp(pc[2]);
            const int pu = project_lround(a.K.fx * pc[0], pc[2], rz, a.K.cx);
            const int pv = project_lround(a.K.fy * pc[1], pc[2], rz, a.K.cy);
            if (pu >= 0 && pu < a.K.w && pv >= 0 && pv < a.K.h) {
                const int pix = pv * a.K.w + pu;
                const float d = __ldg(a.depth + pix);  // depth, mask and colour in one round trip
                const bool pix_masked = has_mask && __ldg(a.mask + pix);
                uint32_t cr = 0, cg = 0, cb = 0;
                if (has_rgb) {
                    const uint8_t* col = a.rgb + 3 * size_t(pix);
                    cr = __ldg(col);
                    cg = __ldg(col + 1);
                    cb = __ldg(col + 2);
                }
                float sdf = __uint_as_float(raw.x);
                uint32_t wgt = raw.y & 0xFFu, r = (raw.y >> 8) & 0xFFu, g = (raw.y >> 16) & 0xFFu,
                         bl = raw.y >> 24;
                bool dirty = false;
                if ((e & kFlagCarve) && pc[2] < a.V.carve_clip && depth_valid(d) && !(pc[2] >= double(d) - tau)) {
                    const double w = double(wgt);
                    sdf = div_f32(double(sdf) * w + tau * cw, w + cw, s_rcp[wgt + uint32_t(cw)]);
                    wgt = min(wgt + uint32_t(cw), uint32_t(mw));
                    dirty = true;
                }
                if ((e & kFlagIntegrate) && !pix_masked && depth_valid(d) &&
                    !(d < a.V.min_depth) && !(d > a.V.max_depth)) {
                    const double dist = double(d) - pc[2];
                    if (!(dist <= -tau)) {
                        const double clamped = fmin(dist, tau);
                        const double w = double(wgt);
                        sdf = div_f32(double(sdf) * w + clamped, w + 1.0, s_rcp[wgt + 1u]);
                        if (fabs(dist) <= tau && has_rgb) {
                            r = colour_avg(r, wgt, cr, s_cdiv);
                            g = colour_avg(g, wgt, cg, s_cdiv);
                            bl = colour_avg(bl, wgt, cb, s_cdiv);
                        }
                        wgt = min(wgt + 1u, uint32_t(mw));
                        dirty = true;
                    }
                }
                if (dirty) {
                    raw.x = __float_as_uint(sdf);
                    raw.y = (wgt & 0xFFu) | ((r & 0xFFu) << 8) | ((g & 0xFFu) << 16) | ((bl & 0xFFu) << 24);
                    *vp = raw;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- sampling
// Batch of SampleSdf / SampleIntensity / *WithGradient / SampleSdfGradient.
__global__ void k_sample(VolumeView V, const double* pts, int n, int mode, double* value, double* grad,
                         uint8_t* valid) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    CellSample cs;
    bool ok;
    double val = 0.0, g[3] = {0, 0, 0};
    if (mode == 4) {  // central differences, tsdf_volume.cpp:358-373
        ok = true;
        const double s = V.voxel_size;
        for (int axis = 0; axis < 3 && ok; ++axis) {
            double hi[3] = {p[0], p[1], p[2]}, lo[3] = {p[0], p[1], p[2]};
            hi[axis] = p[axis] + s;
            lo[axis] = p[axis] - s;
            CellSample a, b;
            ok = sample_point<false, false>(V, hi, a) && sample_point<false, false>(V, lo, b);
            if (ok) g[axis] = (a.sdf - b.sdf) / (2.0 * s);
        }
        if (ok) {
            sample_point<false, false>(V, p, cs);
            val = cs.sdf;
        }
    } else if (mode >= 2) {
        ok = sample_point<true, true>(V, p, cs);
        if (ok) {
            val = mode == 2 ? cs.sdf : cs.inten;
            for (int k = 0; k < 3; ++k) g[k] = mode == 2 ? cs.gs[k] : cs.gi[k];
        }
    } else {
        ok = sample_point<false, true>(V, p, cs);
        if (ok) val = mode == 0 ? cs.sdf : cs.inten;
    }
    value[i] = ok ? val : 0.0;
    if (grad)
        for (int k = 0; k < 3; ++k) grad[3 * i + k] = ok ? g[k] : 0.0;
    valid[i] = ok;
}

// ---------------------------------------------------------------- host mirror support
// Voxel access through VoxelHandle semantics (tsdf_volume.cpp:79-87).
__global__ void k_voxel_rw(VolumeView V, const int* vc, int n, Voxel* io, uint8_t* found, int write) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = vc[3 * i], y = vc[3 * i + 1], z = vc[3 * i + 2];
    const uint32_t b = hash_find(V, x >> 3, y >> 3, z >> 3);
    if (found) found[i] = b != kInvalid;
    if (b == kInvalid) return;
    Voxel* v = V.voxels + size_t(b) * kBrickVoxels + (((z & 7) * 8 + (y & 7)) * 8 + (x & 7));
    if (write) *v = io[i];
    else io[i] = *v;
}

// Structural invariants of a volume (the race detector for the lock-free
// inserts, the ranked assignment and the concurrent link writers; the GPU
// pool has no compute-sanitizer). err[] counts:
//  [0] occupied slots holding a value that is neither a brick < num_blocks nor pending
//  [1] bricks whose recorded slot does not hold their key and index
//  [2] keys stored twice (a probe from the key's home slot finds another slot first)
//  [3] link records that disagree with a fresh hash probe of the neighbour
//  [4] pending keys (claimed, no brick) outside an allocation in progress
__global__ void k_volume_check(VolumeView V, unsigned long long* err) {
    const uint32_t nb = min(V.counters[kNumBlocks], V.max_blocks);
    const uint32_t linked = min(V.counters[kLinked], nb);
    const uint32_t stride = gridDim.x * blockDim.x;
    unsigned long long e[5] = {0, 0, 0, 0, 0};
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= V.hash_mask; i += stride) {
        const HashSlot sl = V.slots[i];
        if (sl.key == kEmptyKey) continue;
        if (sl.value == kInvalid) {
            ++e[4];
            continue;
        }
        if (sl.value >= nb) ++e[0];
        const int4 c = unpack_key(sl.key, i);
        if (hash_find_slot(V, c.x, c.y, c.z) != i) ++e[2];
    }
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
        const int4 c = V.coords[b];
        const uint32_t slot = uint32_t(c.w);
        if (slot > V.hash_mask || V.slots[slot].key != pack_key(c.x, c.y, c.z) || V.slots[slot].value != b) {
            ++e[1];
            continue;
        }
        if (b >= linked) continue;
        const uint32_t* rec = V.links + size_t(slot) * kLinkStride;
        if (rec[0] != b) ++e[3];
        for (int q = 1; q < 8; ++q)
            if (rec[q] != hash_find(V, c.x + (q & 1), c.y + ((q >> 1) & 1), c.z + (q >> 2))) ++e[3];
    }
    for (int k = 0; k < 5; ++k)
        if (e[k]) atomicAdd(err + k, e[k]);
}

// Occupied-slot bitmap (for bit-exact hash-occupancy parity).
__global__ void k_occupancy(VolumeView V, uint8_t* bitmap) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= V.hash_mask; i += gridDim.x * blockDim.x)
        bitmap[i] = V.slots[i].key != kEmptyKey;
}

// Empties a volume in place for reuse (the refinement window's throw-away
// TsdfVolume, depth_refinement.cpp:25): every occupied hash slot belongs to
// one of the bricks [0, n) (no deletion, coords.w = slot), so clearing those
// slots, their voxels and link records restores the freshly created state
// without touching the rest of the table. Grid-stride over n read on device.
__global__ void k_vol_clear(VolumeView V, bool voxels) {
    const uint32_t n = min(V.counters[kNumBlocks], V.max_blocks);
    for (uint32_t b = blockIdx.x; b < n; b += gridDim.x) {
        uint4* vox = reinterpret_cast<uint4*>(V.voxels + size_t(b) * kBrickVoxels);
        if (voxels)
            for (int i = threadIdx.x; i < kBrickVoxels * int(sizeof(Voxel)) / 16; i += blockDim.x)
                vox[i] = make_uint4(0, 0, 0, 0);
        const uint32_t slot = uint32_t(V.coords[b].w);
        if (threadIdx.x < kLinkStride) V.links[size_t(slot) * kLinkStride + threadIdx.x] = kInvalid;
        if (threadIdx.x == 0) {
            if (V.win_first) V.win_first[slot] = 0xFFFFFFFFu;
            V.slots[slot].key = kEmptyKey;
            V.slots[slot].value = kInvalid;
        }
    }
}

// ---------------------------------------------------------------- refinement window
// Bricks already present before a chunk take updates from all of its entries.
__global__ void k_win_first_reset(VolumeView V) {
    const uint32_t n = min(V.counters[kNumBlocks], V.max_blocks);
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x)
        V.win_first[uint32_t(V.coords[b].w)] = 0u;
}

// AllocateForFrame of every entry of the chunk (one thread per entry pixel);
// each visited brick records the smallest entry that reached it.
__global__ void k_alloc_window(WindowArgs a) {
    const int P = a.K[0].w * a.K[0].h;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)P * a.n) return;
    const int j = int(i / P), p = int(i % P);
    if (a.bcount[j] && *a.bcount[j] != kListOverflow) return;  // inserted from its brick list
    walk_pixel(a.V, a.depth[j], a.mask[j], a.K[j], a.pose[j], p, [&](const int (&c)[3]) {
        uint32_t slot = kInvalid;
        if (hash_insert(a.V, c[0], c[1], c[2], &slot) >= 0 && slot != kInvalid) atomicMin(a.V.win_first + slot, uint32_t(j));
    });
}

// Inserts the entries' recorded brick lists (entry j's list = the bricks its
// AllocateForFrame allocates), each brick recording its smallest entry.
__global__ void k_insert_window(WindowArgs a) {
    for (int j = 0; j < a.n; ++j) {
        if (!a.bcount[j]) continue;
        const uint32_t cnt = *a.bcount[j];
        if (cnt == kListOverflow) continue;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
            const int4 c = a.blist[j][i];
            uint32_t slot = kInvalid;
            if (hash_insert(a.V, c.x, c.y, c.z, &slot) >= 0 && slot != kInvalid) atomicMin(a.V.win_first + slot, uint32_t(j));
        }
    }
}

// The bricks of a (scratch) volume as a list: AllocateForFrame's result for
// one window entry. count = kListOverflow when they do not fit (or the
// scratch volume overflowed): that entry is walked again at fusion time.
__global__ void k_brick_list(VolumeView S, int4* dst, uint32_t cap, uint32_t* count) {
    const uint32_t nb = S.counters[kNumBlocks];
    const bool ok = nb <= cap && nb <= S.max_blocks && S.counters[kOverflow] == 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = ok ? nb : kListOverflow;
    if (!ok) return;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) dst[i] = S.coords[i];
}

// Per brick: the entries (from its first one on) whose frustum it meets;
// links the new bricks for the ray-march.
__global__ void k_cull_window(WindowArgs a) {
    const uint32_t nb = min(a.V.counters[kNumBlocks], a.V.max_blocks);
    const double ext = double(kSide) * a.V.voxel_size;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t b0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); b0 < nb; b0 += stride) {
        const uint32_t b = b0 + (threadIdx.x & 31u);
        uint32_t bits = 0;
        if (b < nb) {
            const int4 c = a.V.coords[b];
            const uint32_t first = a.V.win_first[uint32_t(c.w)];
            for (int j = int(first); j < a.n; ++j) {
                Pose P;
                for (int i = 0; i < 12; ++i) (i < 9 ? P.R[i] : P.t[i - 9]) = __ldg(a.pose[j] + i);
                const Pose W = pose_inverse(P);
                double cc[8][3];
                for (int k = 0; k < 8; ++k) {
                    const double x = (double(c.x) + double(k & 1)) * ext;
                    const double y = (double(c.y) + double((k >> 1) & 1)) * ext;
                    const double z = (double(c.z) + double(k >> 2)) * ext;
                    pose_apply(W, x, y, z, cc[k]);
                }
                if (!frustum_test(cc, a.K[j]).outside(a.V.max_depth + a.V.truncation)) bits |= 1u << j;
            }
        }
        const unsigned vote = __ballot_sync(0xffffffffu, bits != 0);
        if (vote) {  // one atomic per warp, lanes take consecutive slots
            const int lane = threadIdx.x & 31;
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&a.V.counters[kVisible], uint32_t(__popc(vote)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (bits) {
                const uint32_t at = base + __popc(vote & ((1u << lane) - 1u));
                a.list[2 * at] = b;
                a.list[2 * at + 1] = bits;
            }
        }
    }
    link_new(a.V);
}

// Integrate (tsdf_volume.cpp:155-202) of the chunk's entries, in order, into
// each listed brick: the voxel is read once, updated by every entry whose bit
// is set, and written once.
__global__ void __launch_bounds__(kBrickVoxels, 2) k_fuse_window(WindowArgs a) {
    commit_links(a.V);
    __shared__ Pose Ws[kMaxWin];
    __shared__ double s_rcp[512];  // RN(1 / i) for the running averages (see div_f32)
    __shared__ uint32_t s_cdiv[257];  // colour_avg multipliers by d = w + 1
    if (threadIdx.x < a.n) {
        Pose P;
        for (int i = 0; i < 12; ++i) (i < 9 ? P.R[i] : P.t[i - 9]) = a.pose[threadIdx.x][i];
        Ws[threadIdx.x] = pose_inverse(P);
    }
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s_rcp[i] = i ? 1.0 / double(i) : 0.0;
    for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdiv[i] = i ? colour_magic(uint32_t(i)) : 0u;
    __syncthreads();
    const uint32_t nvis = a.V.counters[kVisible];
    const int x = threadIdx.x & 7, y = (threadIdx.x >> 3) & 7, z = threadIdx.x >> 6;
    const double s = a.V.voxel_size, tau = a.V.truncation;
    const int mw = a.V.max_weight;
    for (uint32_t i = blockIdx.x; i < nvis; i += gridDim.x) {
        const uint32_t b = __ldcg(a.list + 2 * i), bits = __ldcg(a.list + 2 * i + 1);
        const int4 c = a.V.coords[b];
        Voxel* vp = a.V.voxels + size_t(b) * kBrickVoxels + threadIdx.x;
        uint2 raw = *reinterpret_cast<uint2*>(vp);
        float sdf = __uint_as_float(raw.x);
        uint32_t wgt = raw.y & 0xFFu, r = (raw.y >> 8) & 0xFFu, g = (raw.y >> 16) & 0xFFu, bl = raw.y >> 24;
        bool dirty = false;
        const double cx = (double(c.x * kSide + x) + 0.5) * s;  // VoxelCenter, tsdf_volume.hpp:117-119
        const double cy = (double(c.y * kSide + y) + 0.5) * s;
        const double cz = (double(c.z * kSide + z) + 0.5) * s;
        // Entries in groups of kGroup: the frame reads of a group (projection
        // only depends on the entry's pose) are all issued before the first
        // update, then the updates run in window order.
        constexpr int kGroup = 4;
        for (uint32_t m = bits; m;) {
            int jj[kGroup];
            float dd[kGroup];
            double zz[kGroup];
            uint32_t col[kGroup];
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                jj[k] = -1;
                dd[k] = 0.f;
                zz[k] = 0.0;
                col[k] = 0u;
                if (!m) continue;
                const int j = __ffs(m) - 1;
                m &= m - 1u;
                const Intr& K = a.K[j];
                double pc[3];
                pose_apply(Ws[j], cx, cy, cz, pc);
                if (pc[2] <= 1e-9) continue;
                const double rz = fuse_rcp(pc[2]);
                const int pu = project_lround(K.fx * pc[0], pc[2], rz, K.cx);
                const int pv = project_lround(K.fy * pc[1], pc[2], rz, K.cy);
                if (!(pu >= 0 && pu < K.w && pv >= 0 && pv < K.h)) continue;
                const int pix = pv * K.w + pu;
                if (a.mask[j] && __ldg(a.mask[j] + pix)) continue;
                jj[k] = j;
                zz[k] = pc[2];
                dd[k] = __ldg(a.depth[j] + pix);
                if (a.rgb[j]) {
                    const uint8_t* cp = a.rgb[j] + 3 * size_t(pix);
                    col[k] = uint32_t(__ldg(cp)) | (uint32_t(__ldg(cp + 1)) << 8) | (uint32_t(__ldg(cp + 2)) << 16) |
                             0x1000000u;  // bit 24: the entry has colour
                }
            }
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                if (jj[k] < 0) continue;
                const float d = dd[k];
                if (!(depth_valid(d) && !(d < a.V.min_depth) && !(d > a.V.max_depth))) continue;
                const double dist = double(d) - zz[k];
                if (dist <= -tau) continue;
                const double clamped = fmin(dist, tau);
                const double w = double(wgt);
                sdf = div_f32(double(sdf) * w + clamped, w + 1.0, s_rcp[wgt + 1u]);
                if (fabs(dist) <= tau && (col[k] >> 24)) {
                    r = colour_avg(r, wgt, col[k] & 0xFFu, s_cdiv);
                    g = colour_avg(g, wgt, (col[k] >> 8) & 0xFFu, s_cdiv);
                    bl = colour_avg(bl, wgt, (col[k] >> 16) & 0xFFu, s_cdiv);
                }
                wgt = min(wgt + 1u, uint32_t(mw));
                dirty = true;
            }
        }
        if (dirty) {
            raw.x = __float_as_uint(sdf);
            raw.y = (wgt & 0xFFu) | ((r & 0xFFu) << 8) | ((g & 0xFFu) << 16) | ((bl & 0xFFu) << 24);
            *reinterpret_cast<uint2*>(vp) = raw;
        }
    }
}

}  // namespace rfb
