// Marching cubes over the zero level set: ExtractMesh / ExtractBlock
// (proj/src/mesh.cpp:50-181), with the reference's exact output order.
//
// The reference walks blocks sorted by (x, y, z), cells in (z, y, x) order and
// edges 0..11, emitting a vertex the first time its edge key (low voxel, axis)
// appears, first per block and then globally. Because an edge is active in
// every complete cell that contains it (activity depends only on its two
// endpoint signs), "first appearance" is a pure function of the cell set:
// the vertex of edge (v, axis) belongs to the complete cell among its (up to
// four) incident cells that is smallest in (block rank, cell index). That
// makes the order computable in parallel:
//
//   k_mesh_keys / sort / k_mesh_rank   block order (x, y, z) -> rank
//   k_mesh_cells                       per cell: complete flag + cube index
//   k_mesh_count                       per cell: owned-edge mask, face count,
//                                      in-brick prefix sums, per-brick totals
//   exclusive scans                    per-brick vertex / face bases
//   k_mesh_emit                        vertices of owned edges, faces (indices
//                                      through the owning cell)
//
// Every brick is processed by one 512-thread CTA (one thread per cell) from a
// 9^3-voxel shared-memory region (its own brick plus the "+" faces).
#include <algorithm>

#include <cub/cub.cuh>

#include "rf_volume.cuh"

namespace rfb {

#include "rf_mc_table.inc"

namespace {

constexpr int kR = kSide + 1;  // region edge (9)
constexpr int kRegion = kR * kR * kR;

__device__ __forceinline__ int corner_dx(int k) { return ((k + 1) >> 1) & 1; }  // 0,1,1,0,0,1,1,0
__device__ __forceinline__ int corner_dy(int k) { return (k >> 1) & 1; }        // 0,0,1,1,0,0,1,1
__device__ __forceinline__ int corner_dz(int k) { return k >> 2; }

__device__ const unsigned char kEdgeA[12] = {0, 1, 2, 3, 4, 5, 6, 7, 0, 1, 2, 3};  // mesh.cpp:24-25
__device__ const unsigned char kEdgeB[12] = {1, 2, 3, 0, 5, 6, 7, 4, 4, 5, 6, 7};
__device__ const unsigned char kEdgeAxis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};  // mesh.cpp:28
__device__ const unsigned char kEdgeLow[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};   // mesh.cpp:29
// Edge index of the edge (low corner = d, axis) of a cell, d given by its two
// perpendicular components (lower axis first).
__device__ const unsigned char kEdgeOf[3][4] = {{0, 2, 4, 6}, {3, 1, 7, 5}, {8, 9, 11, 10}};

__device__ __forceinline__ uint16_t edge_mask(int cube) {  // active edges: endpoint signs differ
    uint16_t m = 0;
#pragma unroll
    for (int e = 0; e < 12; ++e)
        if (((cube >> kEdgeA[e]) ^ (cube >> kEdgeB[e])) & 1) m |= uint16_t(1u << e);
    return m;
}

struct Region {
    uint2 vox[kRegion];
    uint8_t present[kRegion];
    uint32_t nb_pool[27];  // pool index of the brick at offset (dx,dy,dz) in {-1,0,1}^3
    uint32_t nb_rank[27];
    int4 coord;
    uint32_t rank;
};

__device__ __forceinline__ int nb_index(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }
__device__ __forceinline__ int rix(int x, int y, int z) { return (z * kR + y) * kR + x; }

// Loads the brick of rank r and its 27-neighbourhood indices into shared memory.
__device__ void load_region(const VolumeView& V, const uint32_t* order, const uint32_t* rank, uint32_t r,
                            Region& R) {
    const uint32_t pool = order[r];
    if (threadIdx.x == 0) {
        R.coord = V.coords[pool];
        R.rank = r;
    }
    __syncthreads();
    if (threadIdx.x < 27) {
        const int t = threadIdx.x;
        const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
        const uint32_t p = (t == 13) ? pool : hash_find(V, R.coord.x + dx, R.coord.y + dy, R.coord.z + dz);
        R.nb_pool[t] = p;
        R.nb_rank[t] = p == kInvalid ? 0xFFFFFFFFu : rank[p];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kRegion; i += blockDim.x) {
        const int x = i % kR, y = (i / kR) % kR, z = i / (kR * kR);
        const uint32_t p = R.nb_pool[nb_index(x >> 3, y >> 3, z >> 3)];
        if (p == kInvalid) {
            R.present[i] = 0;
            R.vox[i] = make_uint2(0, 0);
        } else {
            R.present[i] = 1;
            R.vox[i] = *reinterpret_cast<const uint2*>(V.voxels + size_t(p) * kBrickVoxels +
                                                       ((z & 7) * kSide + (y & 7)) * kSide + (x & 7));
        }
    }
    __syncthreads();
}

__device__ __forceinline__ float vox_sdf(uint2 v) { return __uint_as_float(v.x); }
__device__ __forceinline__ int vox_w(uint2 v) { return int(v.y & 0xFFu); }
__device__ __forceinline__ int vox_c(uint2 v, int ch) { return int((v.y >> (8 * (ch + 1))) & 0xFFu); }

struct MeshVertex {
    float p[3];
    uint8_t c[3];
};

// Vertex of edge e of the cell at local (x, y, z): mesh.cpp:94-124.
__device__ MeshVertex edge_vertex(const Region& R, double voxel_size, int x, int y, int z, int e) {
    int a = kEdgeA[e], b = kEdgeB[e];
    const int axis = kEdgeAxis[e];
    const int oa[3] = {corner_dx(a), corner_dy(a), corner_dz(a)};
    if (oa[axis] == 1) {  // canonical lower-to-upper direction
        const int t = a;
        a = b;
        b = t;
    }
    const uint2 va = R.vox[rix(x + corner_dx(a), y + corner_dy(a), z + corner_dz(a))];
    const uint2 vb = R.vox[rix(x + corner_dx(b), y + corner_dy(b), z + corner_dz(b))];
    const double sa = double(vox_sdf(va)), sb = double(vox_sdf(vb));
    const double denom = sb - sa;
    double t;
    if (fabs(denom) < 1e-12) {
        t = 0.5;
    } else {
        t = -sa / denom;
        t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);  // std::clamp
    }
    const int g[3] = {R.coord.x * kSide + x + corner_dx(a), R.coord.y * kSide + y + corner_dy(a),
                      R.coord.z * kSide + z + corner_dz(a)};
    MeshVertex m;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double p = (double(g[i]) + 0.5) * voxel_size;  // VoxelCenter (tsdf_volume.hpp:122-124)
        if (i == axis) p += t * voxel_size;
        m.p[i] = __double2float_rn(p);
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {  // LerpChannel + lround (mesh.cpp:45-47, 117-123)
        const double ca = double(vox_c(va, ch)), cb = double(vox_c(vb, ch));
        const float f = __double2float_rn(ca + (cb - ca) * t);
        m.c[ch] = uint8_t(lroundf(f));
    }
    return m;
}

// Triangle area test of mesh.cpp:133-136 (f32 edges and cross product, f64 norm).
__device__ __forceinline__ bool tri_ok(const MeshVertex& v0, const MeshVertex& v1, const MeshVertex& v2) {
    const float e1[3] = {v1.p[0] - v0.p[0], v1.p[1] - v0.p[1], v1.p[2] - v0.p[2]};
    const float e2[3] = {v2.p[0] - v0.p[0], v2.p[1] - v0.p[1], v2.p[2] - v0.p[2]};
    const float cx = e1[1] * e2[2] - e1[2] * e2[1];
    const float cy = e1[2] * e2[0] - e1[0] * e2[2];
    const float cz = e1[0] * e2[1] - e1[1] * e2[0];
    const double n = sqrt((double(cx) * double(cx) + double(cy) * double(cy)) + double(cz) * double(cz));
    return !(0.5 * n <= 1e-12);
}

struct CellRef {
    uint32_t pool, rank;
    int idx;
};

// Incident cells of edge (low voxel at local v, axis) in (rank, cell) order;
// returns the smallest complete one (the owner). v is relative to the brick.
__device__ CellRef edge_owner(const Region& R, const uint16_t* info, int vx, int vy, int vz, int axis, int* edge_out) {
    const int p = axis == 0 ? 1 : 0, q = axis == 2 ? 1 : 2;  // perpendicular axes, lower first
    CellRef best{kInvalid, 0xFFFFFFFFu, 0};
    int best_e = -1;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        int c[3] = {vx, vy, vz};
        c[p] -= d & 1;
        c[q] -= d >> 1;
        const int bx = c[0] < 0 ? -1 : (c[0] > 7 ? 1 : 0);
        const int by = c[1] < 0 ? -1 : (c[1] > 7 ? 1 : 0);
        const int bz = c[2] < 0 ? -1 : (c[2] > 7 ? 1 : 0);
        const int nb = nb_index(bx, by, bz);
        const uint32_t pool = R.nb_pool[nb];
        if (pool == kInvalid) continue;
        const int idx = (((c[2] & 7) * kSide) + (c[1] & 7)) * kSide + (c[0] & 7);
        if (!(info[size_t(pool) * kBrickVoxels + idx] & 0x100)) continue;
        const uint32_t rk = R.nb_rank[nb];
        if (rk < best.rank || (rk == best.rank && idx < best.idx)) {
            best = CellRef{pool, rk, idx};
            best_e = kEdgeOf[axis][d];
        }
    }
    *edge_out = best_e;
    return best;
}

}  // namespace

__global__ void k_mesh_keys(VolumeView V, uint32_t n, unsigned long long* keys, uint32_t* idx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = V.coords[i];
    const unsigned long long b = kCoordBias;
    keys[i] = ((unsigned long long)(c.x + b) << 42) | ((unsigned long long)(c.y + b) << 21) |
              (unsigned long long)(c.z + b);  // (x, y, z) lexicographic (mesh.cpp:152-156)
    idx[i] = i;
}

__global__ void k_mesh_rank(const uint32_t* order, uint32_t n, uint32_t* rank) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rank[order[i]] = i;
}

__global__ void __launch_bounds__(kBrickVoxels) k_mesh_cells(MeshArgs a) {
    __shared__ Region R;
    load_region(a.V, a.order, a.rank, blockIdx.x, R);
    const int x = threadIdx.x & 7, y = (threadIdx.x >> 3) & 7, z = threadIdx.x >> 6;
    bool complete = true;
    int cube = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = rix(x + corner_dx(k), y + corner_dy(k), z + corner_dz(k));
        complete = complete && R.present[i] && vox_w(R.vox[i]) >= a.min_weight;
        if (double(vox_sdf(R.vox[i])) < 0.0) cube |= 1 << k;
    }
    a.info[size_t(a.order[blockIdx.x]) * kBrickVoxels + threadIdx.x] = complete ? uint16_t(0x100 | cube) : 0;
}

__global__ void __launch_bounds__(kBrickVoxels) k_mesh_count(MeshArgs a) {
    __shared__ Region R;
    __shared__ typename cub::BlockScan<uint32_t, kBrickVoxels>::TempStorage scan;
    load_region(a.V, a.order, a.rank, blockIdx.x, R);
    const int x = threadIdx.x & 7, y = (threadIdx.x >> 3) & 7, z = threadIdx.x >> 6;
    const size_t cell = size_t(a.order[blockIdx.x]) * kBrickVoxels + threadIdx.x;
    const uint16_t inf = a.info[cell];
    uint32_t owned = 0, nf = 0;
    if (inf & 0x100) {
        const int cube = inf & 0xFF;
        const uint16_t em = edge_mask(cube);
        for (int e = 0; e < 12; ++e) {
            if (!((em >> e) & 1)) continue;
            const int lc = kEdgeLow[e];
            int eo;
            const CellRef o = edge_owner(R, a.info, x + corner_dx(lc), y + corner_dy(lc), z + corner_dz(lc),
                                         kEdgeAxis[e], &eo);
            if (o.rank == R.rank && o.idx == int(threadIdx.x)) owned |= 1u << e;
        }
        const double s = a.V.voxel_size;
        for (const signed char* t = kMcTri[cube]; *t != -1; t += 3) {
            const MeshVertex v0 = edge_vertex(R, s, x, y, z, t[0]);
            const MeshVertex v1 = edge_vertex(R, s, x, y, z, t[2]);
            const MeshVertex v2 = edge_vertex(R, s, x, y, z, t[1]);
            nf += tri_ok(v0, v1, v2);
        }
    }
    const uint32_t packed = uint32_t(__popc(owned)) | (nf << 16);
    uint32_t excl, total;
    cub::BlockScan<uint32_t, kBrickVoxels>(scan).ExclusiveSum(packed, excl, total);
    a.owned[cell] = uint16_t(owned);
    a.vloc[cell] = uint16_t(excl & 0xFFFF);
    a.floc[cell] = uint16_t(excl >> 16);
    if (threadIdx.x == 0) {
        a.vcount[blockIdx.x] = total & 0xFFFF;
        a.fcount[blockIdx.x] = total >> 16;
    }
}

__global__ void __launch_bounds__(kBrickVoxels) k_mesh_emit(MeshArgs a) {
    __shared__ Region R;
    load_region(a.V, a.order, a.rank, blockIdx.x, R);
    const int x = threadIdx.x & 7, y = (threadIdx.x >> 3) & 7, z = threadIdx.x >> 6;
    const size_t cell = size_t(a.order[blockIdx.x]) * kBrickVoxels + threadIdx.x;
    const uint16_t inf = a.info[cell];
    if (!(inf & 0x100)) return;
    const int cube = inf & 0xFF;
    const double s = a.V.voxel_size;
    const uint32_t owned = a.owned[cell];
    uint32_t vi = a.vbase[blockIdx.x] + a.vloc[cell];
    for (int e = 0; e < 12; ++e) {
        if (!((owned >> e) & 1)) continue;
        const MeshVertex m = edge_vertex(R, s, x, y, z, e);
        for (int i = 0; i < 3; ++i) {
            a.xyz[3 * size_t(vi) + i] = m.p[i];
            a.rgb[3 * size_t(vi) + i] = m.c[i];
        }
        ++vi;
    }
    uint32_t fi = a.fbase[blockIdx.x] + a.floc[cell];
    for (const signed char* t = kMcTri[cube]; *t != -1; t += 3) {
        const int es[3] = {t[0], t[2], t[1]};  // flipped winding (mesh.cpp:128-131)
        const MeshVertex v0 = edge_vertex(R, s, x, y, z, es[0]);
        const MeshVertex v1 = edge_vertex(R, s, x, y, z, es[1]);
        const MeshVertex v2 = edge_vertex(R, s, x, y, z, es[2]);
        if (!tri_ok(v0, v1, v2)) continue;
        for (int j = 0; j < 3; ++j) {
            const int e = es[j], lc = kEdgeLow[e];
            int eo;
            const CellRef o = edge_owner(R, a.info, x + corner_dx(lc), y + corner_dy(lc), z + corner_dz(lc),
                                         kEdgeAxis[e], &eo);
            const size_t oc = size_t(o.pool) * kBrickVoxels + o.idx;
            const uint32_t below = uint32_t(a.owned[oc]) & ((1u << eo) - 1u);
            a.faces[3 * size_t(fi) + j] = int32_t(a.vbase[o.rank] + a.vloc[oc] + __popc(below));
        }
        ++fi;
    }
}

size_t mesh_scratch_bytes(uint32_t n) {
    size_t sort_tmp = 0, scan_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, int(n), 0, 63);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (uint32_t*)nullptr, (uint32_t*)nullptr, int(n + 1));
    const size_t cells = size_t(n) * kBrickVoxels;
    return 4 * size_t(n) * 8 + 4 * (size_t(n) + 1) * 4 + 4 * cells * 2 + std::max(sort_tmp, scan_tmp) + 1024;
}

namespace {
template <class T>
T* carve(uint8_t*& p, size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += (count * sizeof(T) + 255) & ~size_t(255);
    return r;
}
}  // namespace

// Sorts, counts and scans; copies the (vertex, face) totals into `totals`
// (host) on `stream`. The caller syncs, sets a.xyz/rgb/faces and calls mesh_emit.
cudaError_t mesh_prepare(const VolumeView& V, uint32_t n, int min_weight, cudaStream_t stream, void* scratch,
                         size_t scratch_bytes, uint32_t* totals, MeshArgs* out) {
    uint8_t* p = static_cast<uint8_t*>(scratch);
    auto* keys_in = carve<unsigned long long>(p, n);
    auto* keys_out = carve<unsigned long long>(p, n);
    auto* idx_in = carve<uint32_t>(p, n);
    auto* order = carve<uint32_t>(p, n);
    auto* rank = carve<uint32_t>(p, n);
    auto* vcount = carve<uint32_t>(p, n + 1);
    auto* fcount = carve<uint32_t>(p, n + 1);
    auto* vbase = carve<uint32_t>(p, n + 1);
    auto* fbase = carve<uint32_t>(p, n + 1);
    const size_t cells = size_t(n) * kBrickVoxels;
    auto* info = carve<uint16_t>(p, cells);
    auto* owned = carve<uint16_t>(p, cells);
    auto* vloc = carve<uint16_t>(p, cells);
    auto* floc = carve<uint16_t>(p, cells);
    void* tmp = p;
    size_t tmp_bytes = scratch_bytes - size_t(p - static_cast<uint8_t*>(scratch));

    const unsigned g = (n + 255) / 256;
    k_mesh_keys<<<g, 256, 0, stream>>>(V, n, keys_in, idx_in);
    cudaError_t err = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, idx_in, order, int(n), 0, 63,
                                                      stream);
    if (err != cudaSuccess) return err;
    k_mesh_rank<<<g, 256, 0, stream>>>(order, n, rank);
    MeshArgs& a = *out;
    a = MeshArgs{};
    a.V = V;
    a.n = n;
    a.min_weight = min_weight;
    a.order = order;
    a.rank = rank;
    a.info = info;
    a.owned = owned;
    a.vloc = vloc;
    a.floc = floc;
    a.vcount = vcount;
    a.fcount = fcount;
    a.vbase = vbase;
    a.fbase = fbase;
    cudaMemsetAsync(vcount + n, 0, 4, stream);
    cudaMemsetAsync(fcount + n, 0, 4, stream);
    k_mesh_cells<<<n, kBrickVoxels, 0, stream>>>(a);
    k_mesh_count<<<n, kBrickVoxels, 0, stream>>>(a);
    if ((err = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, vcount, vbase, int(n + 1), stream)) != cudaSuccess)
        return err;
    if ((err = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, fcount, fbase, int(n + 1), stream)) != cudaSuccess)
        return err;
    cudaMemcpyAsync(totals, vbase + n, 4, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(totals + 1, fbase + n, 4, cudaMemcpyDeviceToHost, stream);
    return cudaGetLastError();
}

cudaError_t mesh_emit(const MeshArgs& a, cudaStream_t stream) {
    k_mesh_emit<<<a.n, kBrickVoxels, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace rfb
