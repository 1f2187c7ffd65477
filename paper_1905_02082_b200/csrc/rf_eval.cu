// Evaluation (evaluation.hpp:12-50): NearestDistances and DistanceCdf on the
// GPU, AteRmse / RpeOverTime on the host (a few thousand poses: O(n) host
// work, not worth a launch).
//
// NearestDistances (evaluation.cpp:96-217) keeps the reference's grid and
// search rule so the answer is the same set-minimum bit for bit:
//   cell  = max(|hi - lo| / 256, 1e-6) over the reference cloud's bounding box,
//   CellOf(p) = floor(p / cell) per axis (f32 promoted to f64),
//   shells of Chebyshev radius r from r_first to r_limit, clipped to the
//   reference cells' box, stopping once best <= (r - 1) * cell.
// B200 layout instead of the reference's hash of cells: the cell box is at
// most ~258^3 cells, so the grid is a dense counting sort — per-cell counts
// (atomicAdd, which also gives each point its rank inside the cell), an
// exclusive scan into cell starts, a scatter of the points as float4. One
// thread per query walks its shells over the dense starts array; distances
// are compared squared (sqrt is monotone and correctly rounded, so
// sqrt(min d^2) == min sqrt(d^2)) and the per-shell stop test uses the sqrt.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <vector>

#include <math_constants.h>

#include "rf_host.cuh"

namespace rfb {
namespace {

struct NnGrid {
    double cell;
    int lo[3], hi[3];  // min_cell_ / max_cell_ (evaluation.cpp:100-107)
    int dim[3];
};

__device__ __forceinline__ int cell_of(float p, double cell) {  // CellOf, evaluation.cpp:152-156
    return static_cast<int>(floor(static_cast<double>(p) / cell));
}

// float -> order-preserving uint32 key (for atomicMin/atomicMax bounding boxes)
__device__ __forceinline__ uint32_t f2key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
inline float key2f(uint32_t k) {
    const uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

// Bounding box of the reference cloud (evaluation.cpp:206-210): keys[0..2] min, [3..5] max.
__global__ void k_bbox(const float* __restrict__ p, uint64_t n, uint32_t* keys) {
    uint32_t mn[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, mx[3] = {0, 0, 0};
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        for (int a = 0; a < 3; ++a) {
            const uint32_t k = f2key(p[3 * i + a]);
            mn[a] = min(mn[a], k);
            mx[a] = max(mx[a], k);
        }
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xFFFFFFFFu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xFFFFFFFFu, mx[a], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) {
            atomicMin(keys + a, mn[a]);
            atomicMax(keys + 3 + a, mx[a]);
        }
}

__device__ __forceinline__ uint32_t cell_index(const NnGrid& g, int x, int y, int z) {
    return (uint32_t(z - g.lo[2]) * uint32_t(g.dim[1]) + uint32_t(y - g.lo[1])) * uint32_t(g.dim[0]) + uint32_t(x - g.lo[0]);
}

// Counting sort, pass 1: each point's cell and its rank inside the cell.
__global__ void k_cell_count(const float* __restrict__ p, uint64_t n, NnGrid g, uint32_t* counts, uint32_t* cid,
                             uint32_t* rank) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = cell_index(g, cell_of(p[3 * i], g.cell), cell_of(p[3 * i + 1], g.cell), cell_of(p[3 * i + 2], g.cell));
        cid[i] = c;
        rank[i] = atomicAdd(counts + c, 1u);
    }
}

// Exclusive scan of n uint32 in place, 4096 per block, block totals to `totals`.
constexpr int kScanThreads = 1024, kScanPer = 4;
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = s_warp[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
            if (lane >= o) t += y;
        }
        s_warp[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    *total = s_warp[31];
    return x - v + (w ? s_warp[w - 1] : 0u);
}
__global__ void __launch_bounds__(kScanThreads) k_scan_local(uint32_t* a, uint64_t n, uint32_t* totals) {
    __shared__ uint32_t s_warp[32];
    const uint64_t base = uint64_t(blockIdx.x) * kScanThreads * kScanPer + uint64_t(threadIdx.x) * kScanPer;
    uint32_t v[kScanPer], sum = 0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        v[j] = base + j < n ? a[base + j] : 0u;
        sum += v[j];
    }
    uint32_t total;
    uint32_t run = block_exclusive(sum, s_warp, &total);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        if (base + j < n) a[base + j] = run;
        run += v[j];
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = total;
}
__global__ void __launch_bounds__(kScanThreads) k_scan_totals(uint32_t* totals, uint32_t nb) {
    __shared__ uint32_t s_warp[32];
    uint32_t carry = 0;
    for (uint32_t c = 0; c < nb; c += kScanThreads) {
        const uint32_t i = c + threadIdx.x;
        const uint32_t v = i < nb ? totals[i] : 0u;
        uint32_t total;
        const uint32_t e = block_exclusive(v, s_warp, &total);
        if (i < nb) totals[i] = carry + e;
        carry += total;
        __syncthreads();
    }
}
__global__ void k_scan_add(uint32_t* a, uint64_t n, const uint32_t* totals) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i < n) a[i] += totals[i / (kScanThreads * kScanPer)];
}

// Counting sort, pass 2: points grouped by cell (order inside a cell is
// irrelevant: the search takes a minimum).
__global__ void k_scatter(const float* __restrict__ p, uint64_t n, const uint32_t* __restrict__ cid,
                          const uint32_t* __restrict__ rank, const uint32_t* __restrict__ starts, float4* sorted) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        sorted[starts[cid[i]] + rank[i]] = make_float4(p[3 * i], p[3 * i + 1], p[3 * i + 2], 0.f);
}

// NearestDistance (evaluation.cpp:126-149): the reference's shell walk, one
// thread per query, while it stays within kShellBudget cells. A query whose
// walk would exceed it (far outside the reference box, or in a large hole:
// the walk is then O(shells x box face)) is handed to k_nn_brute, which
// returns the same exact minimum over all reference points.
constexpr int kShellBudget = 4096;
__global__ void __launch_bounds__(128) k_nn_query(const float* __restrict__ q, uint64_t nq, const float4* __restrict__ pts,
                                                  const uint32_t* __restrict__ starts, NnGrid g, double* __restrict__ out,
                                                  uint32_t* heavy, uint32_t* n_heavy) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    const float qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
    const int qc[3] = {cell_of(qx, g.cell), cell_of(qy, g.cell), cell_of(qz, g.cell)};
    int r_limit = 0, r_first = 0, lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r_limit = max(r_limit, max(abs(qc[a] - g.lo[a]), abs(g.hi[a] - qc[a])));
        r_first = max(r_first, max(g.lo[a] - qc[a], qc[a] - g.hi[a]));
        lo[a] = g.lo[a] - qc[a];
        hi[a] = g.hi[a] - qc[a];
    }
    double best_sq = CUDART_INF, best = CUDART_INF;
    auto visit = [&](int x, int y, int z) {
        const uint32_t c = cell_index(g, x, y, z);
        const uint32_t e = starts[c + 1];
        for (uint32_t k = starts[c]; k < e; ++k) {
            const float4 p = pts[k];
            const double dx = double(p.x - qx), dy = double(p.y - qy), dz = double(p.z - qz);
            best_sq = fmin(best_sq, (dx * dx + dy * dy) + dz * dz);
        }
    };
    int spent = 0;
    for (int r = r_first; r <= r_limit; ++r) {
        if (best <= double(r - 1) * g.cell) break;
        if (r == 0) {
            visit(qc[0], qc[1], qc[2]);
            spent = 1;
        } else {
            // VisitShell (evaluation.cpp:161-191): two x faces, two y faces
            // without the x rims, two z faces without either rim, clipped.
            const int xy0 = max(-r, lo[1]), xy1 = min(r, hi[1]), xz0 = max(-r, lo[2]), xz1 = min(r, hi[2]);
            const int yx0 = max(-r + 1, lo[0]), yx1 = min(r - 1, hi[0]);
            const int zy0 = max(-r + 1, lo[1]), zy1 = min(r - 1, hi[1]);
            const int nxf = max(0, xy1 - xy0 + 1) * max(0, xz1 - xz0 + 1);
            const int nyf = max(0, yx1 - yx0 + 1) * max(0, xz1 - xz0 + 1);
            const int nzf = max(0, yx1 - yx0 + 1) * max(0, zy1 - zy0 + 1);
            int n = 0;
            for (int side = -r; side <= r; side += 2 * r) {
                n += (side >= lo[0] && side <= hi[0]) ? nxf : 0;
                n += (side >= lo[1] && side <= hi[1]) ? nyf : 0;
                n += (side >= lo[2] && side <= hi[2]) ? nzf : 0;
            }
            if (spent + n > kShellBudget) {
                out[i] = CUDART_INF;  // atomicMin target for k_nn_brute
                heavy[atomicAdd(n_heavy, 1u)] = uint32_t(i);
                return;
            }
            spent += n;
            for (int side = -r; side <= r; side += 2 * r) {
                if (side >= lo[0] && side <= hi[0])
                    for (int u = xy0; u <= xy1; ++u)
                        for (int v = xz0; v <= xz1; ++v) visit(qc[0] + side, qc[1] + u, qc[2] + v);
                if (side >= lo[1] && side <= hi[1])
                    for (int u = yx0; u <= yx1; ++u)
                        for (int v = xz0; v <= xz1; ++v) visit(qc[0] + u, qc[1] + side, qc[2] + v);
                if (side >= lo[2] && side <= hi[2])
                    for (int u = yx0; u <= yx1; ++u)
                        for (int v = zy0; v <= zy1; ++v) visit(qc[0] + u, qc[1] + v, qc[2] + side);
            }
        }
        best = sqrt(best_sq);
    }
    out[i] = best;
}

// Exact minimum over every reference point for the queries the shell walk
// gave up on: CTA (tile of kBruteQ heavy queries) x (chunk of points), each
// thread keeps a running min per query, then a block min and an atomicMin on
// the f64 bits (non-negative doubles order like their bit patterns).
constexpr int kBruteQ = 16, kBruteThreads = 256, kBrutePts = 64 * kBruteThreads;
__global__ void __launch_bounds__(kBruteThreads) k_nn_brute(const float* __restrict__ q, const uint32_t* __restrict__ heavy,
                                                            const uint32_t* __restrict__ n_heavy, const float4* __restrict__ pts,
                                                            uint64_t np, double* out) {
    __shared__ float s_q[kBruteQ][3];
    __shared__ double s_min[kBruteThreads / 32][kBruteQ];
    const uint32_t nh = *n_heavy, q0 = blockIdx.y * kBruteQ;
    if (q0 >= nh) return;
    const int nqt = min(kBruteQ, int(nh - q0));
    if (threadIdx.x < kBruteQ * 3) {
        const int j = threadIdx.x / 3, a = threadIdx.x % 3;
        s_q[j][a] = j < nqt ? q[3 * size_t(heavy[q0 + j]) + a] : 0.f;
    }
    __syncthreads();
    double m[kBruteQ];
#pragma unroll
    for (int j = 0; j < kBruteQ; ++j) m[j] = CUDART_INF;
    const uint64_t e1 = uint64_t(blockIdx.x + 1) * kBrutePts, end = np < e1 ? np : e1;
    for (uint64_t k = uint64_t(blockIdx.x) * kBrutePts + threadIdx.x; k < end; k += kBruteThreads) {
        const float4 p = pts[k];
#pragma unroll
        for (int j = 0; j < kBruteQ; ++j) {
            const double dx = double(p.x - s_q[j][0]), dy = double(p.y - s_q[j][1]), dz = double(p.z - s_q[j][2]);
            m[j] = fmin(m[j], (dx * dx + dy * dy) + dz * dz);
        }
    }
#pragma unroll
    for (int j = 0; j < kBruteQ; ++j) {
        for (int o = 16; o; o >>= 1) m[j] = fmin(m[j], __shfl_xor_sync(0xFFFFFFFFu, m[j], o));
        if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5][j] = m[j];
    }
    __syncthreads();
    if (threadIdx.x < nqt) {
        double v = s_min[0][threadIdx.x];
        for (int w = 1; w < kBruteThreads / 32; ++w) v = fmin(v, s_min[w][threadIdx.x]);
        atomicMin(reinterpret_cast<unsigned long long*>(out) + heavy[q0 + threadIdx.x],
                  (unsigned long long)__double_as_longlong(sqrt(v)));
    }
}

// DistanceCdf (evaluation.cpp:219-236) as a histogram: each distance lands in
// the first edge >= it (upper_bound(sorted, e_i) counts d <= e_i), NaN past the end.
__global__ void k_cdf_hist(const double* __restrict__ d, uint64_t n, const double* __restrict__ edges, int ne,
                           unsigned long long* hist) {
    extern __shared__ unsigned long long s_hist[];
    for (int i = threadIdx.x; i <= ne; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double x = d[i];
        int b = ne;
        if (x == x) {
            int l = 0, h = ne;  // first edge >= x
            while (l < h) {
                const int m = (l + h) >> 1;
                if (edges[m] < x) l = m + 1;
                else h = m;
            }
            b = l;
        }
        atomicAdd(s_hist + b, 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= ne; i += blockDim.x)
        if (s_hist[i]) atomicAdd(hist + i, s_hist[i]);
}

// Per-device scratch for the evaluation calls (grown, never shrunk).
struct EvalWs {
    cudaStream_t stream = nullptr;
    DevBuf q, ref, out, keys, counts, cid, rank, totals, sorted, d, edges, hist, heavy;
    std::mutex mu;
};
EvalWs& eval_ws(int device) {
    static std::mutex m;
    static std::map<int, EvalWs*> all;
    std::lock_guard<std::mutex> lk(m);
    EvalWs*& w = all[device];
    if (!w) {
        w = new EvalWs;  // process lifetime, like the per-device workspaces
        CK(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    }
    return *w;
}

int grid_for(uint64_t n, int threads) {
    return int(std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16));
}

// ------------------------------------------------------------------ host: trajectories
struct Traj {
    const double* t;
    const double* pose;  // 12 per entry
    uint64_t n;
};
struct P3 {
    double x, y, z;
};
P3 translation(const Traj& a, uint64_t i) { return {a.pose[12 * i + 9], a.pose[12 * i + 10], a.pose[12 * i + 11]}; }

// MatchTimestamps (dataset_io.cpp:41-71)
std::vector<std::pair<uint64_t, uint64_t>> match_timestamps(const Traj& a, const Traj& b, double max_dt) {
    struct Cand {
        double dt;
        uint64_t i, j;
    };
    std::vector<Cand> cands;
    uint64_t lo = 0;
    for (uint64_t i = 0; i < a.n; ++i) {
        while (lo < b.n && b.t[lo] < a.t[i] - max_dt) ++lo;
        for (uint64_t j = lo; j < b.n && b.t[j] <= a.t[i] + max_dt; ++j) cands.push_back({std::abs(a.t[i] - b.t[j]), i, j});
    }
    std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
        if (x.dt != y.dt) return x.dt < y.dt;
        if (x.i != y.i) return x.i < y.i;
        return x.j < y.j;
    });
    std::vector<char> ua(a.n, 0), ub(b.n, 0);
    std::vector<std::pair<uint64_t, uint64_t>> pairs;
    for (const Cand& c : cands) {
        if (ua[c.i] || ub[c.j]) continue;
        ua[c.i] = ub[c.j] = 1;
        pairs.emplace_back(c.i, c.j);
    }
    std::sort(pairs.begin(), pairs.end(), [&](const auto& x, const auto& y) { return a.t[x.first] < a.t[y.first]; });
    return pairs;
}

// Largest-eigenvalue eigenvector of a symmetric 4x4 (cyclic Jacobi).
void sym4_top_eigvec(double A[4][4], double v[4]) {
    double V[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0, diag = 0;
        for (int p = 0; p < 4; ++p) {
            diag += A[p][p] * A[p][p];
            for (int q = p + 1; q < 4; ++q) off += A[p][q] * A[p][q];
        }
        if (off <= 1e-300 || off <= 1e-34 * diag) break;
        for (int p = 0; p < 3; ++p)
            for (int q = p + 1; q < 4; ++q) {
                if (A[p][q] == 0.0) continue;
                const double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 4; ++k) {  // A <- A J
                    const double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 4; ++k) {  // A <- J^T A
                    const double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 4; ++k) {
                    const double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = c * vkp - s * vkq;
                    V[k][q] = s * vkp + c * vkq;
                }
            }
    }
    int m = 0;
    for (int k = 1; k < 4; ++k)
        if (A[k][k] > A[m][m]) m = k;
    for (int k = 0; k < 4; ++k) v[k] = V[k][m];
}

}  // namespace
}  // namespace rfb

using namespace rfb;

extern "C" {

// AteRmse (evaluation.cpp:26-62). The closed-form rigid alignment is Horn's
// unit-quaternion solution (the same optimum as the reference's SVD of the
// cross-covariance with the reflection guard); the oracle restates the SVD.
rf_status rf_ate_rmse(const double* est_t, const double* est_poses, uint64_t n_est, const double* gt_t,
                      const double* gt_poses, uint64_t n_gt, double max_dt, double* rmse, double alignment[12],
                      uint64_t* pairs_out) {
    return guard([&] {
        require((est_t && est_poses) || n_est == 0, RF_INVALID_ARGUMENT, "null estimated trajectory");
        require((gt_t && gt_poses) || n_gt == 0, RF_INVALID_ARGUMENT, "null ground-truth trajectory");
        const Traj est{est_t, est_poses, n_est}, gt{gt_t, gt_poses, n_gt};
        const auto pairs = match_timestamps(est, gt, max_dt);
        require(pairs.size() >= 3, RF_FAILED, "need at least 3 associated poses, got " + std::to_string(pairs.size()));
        P3 ce{0, 0, 0}, cg{0, 0, 0};
        for (const auto& [i, j] : pairs) {
            const P3 e = translation(est, i), g = translation(gt, j);
            ce = {ce.x + e.x, ce.y + e.y, ce.z + e.z};
            cg = {cg.x + g.x, cg.y + g.y, cg.z + g.z};
        }
        const double np = double(pairs.size());
        ce = {ce.x / np, ce.y / np, ce.z / np};
        cg = {cg.x / np, cg.y / np, cg.z / np};
        double S[3][3] = {};  // S_ab = sum (est - ce)_a (gt - cg)_b
        for (const auto& [i, j] : pairs) {
            const P3 e = translation(est, i), g = translation(gt, j);
            const double ev[3] = {e.x - ce.x, e.y - ce.y, e.z - ce.z}, gv[3] = {g.x - cg.x, g.y - cg.y, g.z - cg.z};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) S[a][b] += ev[a] * gv[b];
        }
        const double sxx = S[0][0], sxy = S[0][1], sxz = S[0][2], syx = S[1][0], syy = S[1][1], syz = S[1][2],
                     szx = S[2][0], szy = S[2][1], szz = S[2][2];
        double N[4][4] = {{sxx + syy + szz, syz - szy, szx - sxz, sxy - syx},
                          {syz - szy, sxx - syy - szz, sxy + syx, szx + sxz},
                          {szx - sxz, sxy + syx, -sxx + syy - szz, syz + szy},
                          {sxy - syx, szx + sxz, syz + szy, -sxx - syy + szz}};
        double q[4];
        sym4_top_eigvec(N, q);
        const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        const double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
        const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
                             2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                             2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
        const double t[3] = {cg.x - (R[0] * ce.x + R[1] * ce.y + R[2] * ce.z),
                             cg.y - (R[3] * ce.x + R[4] * ce.y + R[5] * ce.z),
                             cg.z - (R[6] * ce.x + R[7] * ce.y + R[8] * ce.z)};
        double sum_sq = 0.0;
        for (const auto& [i, j] : pairs) {
            const P3 e = translation(est, i), g = translation(gt, j);
            const double ax = R[0] * e.x + R[1] * e.y + R[2] * e.z + t[0] - g.x;
            const double ay = R[3] * e.x + R[4] * e.y + R[5] * e.z + t[1] - g.y;
            const double az = R[6] * e.x + R[7] * e.y + R[8] * e.z + t[2] - g.z;
            sum_sq += ax * ax + ay * ay + az * az;
        }
        if (rmse) *rmse = std::sqrt(sum_sq / np);
        if (alignment) {
            std::memcpy(alignment, R, sizeof R);
            std::memcpy(alignment + 9, t, sizeof t);
        }
        if (pairs_out) *pairs_out = pairs.size();
    });
}

// RpeOverTime (evaluation.cpp:64-92): up to `capacity` samples, *count = all of them.
rf_status rf_rpe_over_time(const double* est_t, const double* est_poses, uint64_t n_est, const double* gt_t,
                           const double* gt_poses, uint64_t n_gt, double delta, double max_dt, double* timestamps,
                           double* errors, uint64_t capacity, uint64_t* count) {
    return guard([&] {
        require(delta > 0, RF_INVALID_ARGUMENT, "delta must be positive");
        require((est_t && est_poses) || n_est == 0, RF_INVALID_ARGUMENT, "null estimated trajectory");
        require((gt_t && gt_poses) || n_gt == 0, RF_INVALID_ARGUMENT, "null ground-truth trajectory");
        const Traj est{est_t, est_poses, n_est}, gt{gt_t, gt_poses, n_gt};
        const auto pairs = match_timestamps(est, gt, max_dt);
        // out = a.Inverse() * b with Pose's algebra (geometry.hpp:69-108):
        // a^-1 = {Ra^T, -(Ra^T ta)}, then {Ra^T Rb, Ra^T tb + (-(Ra^T ta))}
        auto inv_mul = [](const double* a, const double* b, double* out) {
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    out[3 * r + c] = (a[r] * b[c] + a[3 + r] * b[3 + c]) + a[6 + r] * b[6 + c];
            for (int r = 0; r < 3; ++r) {
                const double ta = (a[r] * a[9] + a[3 + r] * a[10]) + a[6 + r] * a[11];
                const double tb = (a[r] * b[9] + a[3 + r] * b[10]) + a[6 + r] * b[11];
                out[9 + r] = tb + (-ta);
            }
        };
        uint64_t n = 0;
        for (size_t k = 0; k < pairs.size(); ++k) {
            const double target = est.t[pairs[k].first] + delta;
            size_t best = pairs.size();
            double best_err = max_dt;
            for (size_t m = k + 1; m < pairs.size(); ++m) {
                const double err = std::abs(est.t[pairs[m].first] - target);
                if (err <= best_err) {
                    best_err = err;
                    best = m;
                }
                if (est.t[pairs[m].first] > target + max_dt) break;
            }
            if (best == pairs.size()) continue;
            double rel_est[12], rel_gt[12], err[12];
            inv_mul(est.pose + 12 * pairs[k].first, est.pose + 12 * pairs[best].first, rel_est);
            inv_mul(gt.pose + 12 * pairs[k].second, gt.pose + 12 * pairs[best].second, rel_gt);
            inv_mul(rel_gt, rel_est, err);
            if (n < capacity) {
                if (timestamps) timestamps[n] = est.t[pairs[k].first];
                if (errors) errors[n] = std::sqrt((err[9] * err[9] + err[10] * err[10]) + err[11] * err[11]);
            }
            ++n;
        }
        if (count) *count = n;
    });
}

// NearestDistances (evaluation.cpp:203-217). memory = RF_MEMORY_HOST or
// RF_MEMORY_DEVICE for all three arrays; xyz f32 triples; out f64.
rf_status rf_nearest_distances(const float* queries, uint64_t nq, const float* reference, uint64_t nr, int32_t memory,
                               int device, double* out) {
    return guard([&] {
        require(nr > 0 && reference, RF_INVALID_ARGUMENT, "reference cloud is empty");
        if (nq == 0) return;
        require(queries && out, RF_INVALID_ARGUMENT, "null argument");
        require(memory == RF_MEMORY_HOST || memory == RF_MEMORY_DEVICE, RF_INVALID_ARGUMENT, "bad memory kind");
        CK(cudaSetDevice(device));
        EvalWs& w = eval_ws(device);
        std::lock_guard<std::mutex> lk(w.mu);
        cudaStream_t s = w.stream;
        const float* dq = queries;
        const float* dr = reference;
        double* dout = out;
        if (memory == RF_MEMORY_HOST) {
            w.q.ensure(nq * 12);
            w.ref.ensure(nr * 12);
            w.out.ensure(nq * 8);
            CK(cudaMemcpyAsync(w.q.p, queries, nq * 12, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(w.ref.p, reference, nr * 12, cudaMemcpyHostToDevice, s));
            dq = w.q.as<float>();
            dr = w.ref.as<float>();
            dout = w.out.as<double>();
        }
        // bounding box -> cell size and cell box (monotone CellOf: min/max cells are those of lo/hi)
        w.keys.ensure(6 * 4);
        const uint32_t init[6] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0, 0, 0};
        uint32_t keys[6];
        CK(cudaMemcpyAsync(w.keys.p, init, sizeof init, cudaMemcpyHostToDevice, s));
        k_bbox<<<grid_for(nr, 256), 256, 0, s>>>(dr, nr, w.keys.as<uint32_t>());
        CK(cudaMemcpyAsync(keys, w.keys.p, sizeof keys, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = key2f(keys[a]);
            hi[a] = key2f(keys[3 + a]);
        }
        const double ex = double(hi[0] - lo[0]), ey = double(hi[1] - lo[1]), ez = double(hi[2] - lo[2]);
        const double diag = std::sqrt((ex * ex + ey * ey) + ez * ez);
        NnGrid g{};
        g.cell = std::max(diag / 256.0, 1e-6);
        uint64_t ncell = 1;
        for (int a = 0; a < 3; ++a) {
            g.lo[a] = static_cast<int>(std::floor(double(lo[a]) / g.cell));
            g.hi[a] = static_cast<int>(std::floor(double(hi[a]) / g.cell));
            g.dim[a] = g.hi[a] - g.lo[a] + 1;
            require(g.dim[a] > 0 && g.dim[a] <= 4096, RF_INVALID_ARGUMENT, "reference cloud is not finite");
            ncell *= uint64_t(g.dim[a]);
        }
        require(ncell < (1ull << 31), RF_RESOURCE_LIMIT, "grid too large");
        // counting sort of the reference points by cell
        const uint64_t ns = ncell + 1;
        const uint32_t nb = uint32_t((ns + kScanThreads * kScanPer - 1) / (kScanThreads * kScanPer));
        w.counts.ensure(ns * 4);
        w.totals.ensure(size_t(nb) * 4);
        w.cid.ensure(nr * 4);
        w.rank.ensure(nr * 4);
        w.sorted.ensure(nr * 16);
        CK(cudaMemsetAsync(w.counts.p, 0, ns * 4, s));
        k_cell_count<<<grid_for(nr, 256), 256, 0, s>>>(dr, nr, g, w.counts.as<uint32_t>(), w.cid.as<uint32_t>(),
                                                       w.rank.as<uint32_t>());
        k_scan_local<<<nb, kScanThreads, 0, s>>>(w.counts.as<uint32_t>(), ns, w.totals.as<uint32_t>());
        k_scan_totals<<<1, kScanThreads, 0, s>>>(w.totals.as<uint32_t>(), nb);
        k_scan_add<<<unsigned((ns + 255) / 256), 256, 0, s>>>(w.counts.as<uint32_t>(), ns, w.totals.as<uint32_t>());
        k_scatter<<<grid_for(nr, 256), 256, 0, s>>>(dr, nr, w.cid.as<uint32_t>(), w.rank.as<uint32_t>(),
                                                    w.counts.as<uint32_t>(), w.sorted.as<float4>());
        w.heavy.ensure(nq * 4 + 4);
        uint32_t* n_heavy = w.heavy.as<uint32_t>() + nq;
        CK(cudaMemsetAsync(n_heavy, 0, 4, s));
        k_nn_query<<<unsigned((nq + 127) / 128), 128, 0, s>>>(dq, nq, w.sorted.as<float4>(), w.counts.as<uint32_t>(), g,
                                                              dout, w.heavy.as<uint32_t>(), n_heavy);
        uint32_t nh = 0;
        CK(cudaMemcpyAsync(&nh, n_heavy, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (nh) {
            const dim3 grid(unsigned((nr + kBrutePts - 1) / kBrutePts), (nh + kBruteQ - 1) / kBruteQ);
            k_nn_brute<<<grid, kBruteThreads, 0, s>>>(dq, w.heavy.as<uint32_t>(), n_heavy, w.sorted.as<float4>(), nr, dout);
        }
        CK(cudaGetLastError());
        if (memory == RF_MEMORY_HOST) CK(cudaMemcpyAsync(out, dout, nq * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

// DistanceCdf (evaluation.cpp:219-236). distances: host or device per
// `memory`; edges and cdf: host.
rf_status rf_distance_cdf(const double* distances, uint64_t n, int32_t memory, int device, const double* edges,
                          uint64_t ne, double* cdf) {
    return guard([&] {
        require(n > 0 && distances, RF_INVALID_ARGUMENT, "no distances");
        require(ne == 0 || (edges && cdf), RF_INVALID_ARGUMENT, "null argument");
        for (uint64_t i = 1; i < ne; ++i)
            require(edges[i] > edges[i - 1], RF_INVALID_ARGUMENT, "bin edges must be ascending");
        if (ne == 0) return;
        require(ne < 4096, RF_INVALID_ARGUMENT, "at most 4095 bin edges");
        require(memory == RF_MEMORY_HOST || memory == RF_MEMORY_DEVICE, RF_INVALID_ARGUMENT, "bad memory kind");
        CK(cudaSetDevice(device));
        EvalWs& w = eval_ws(device);
        std::lock_guard<std::mutex> lk(w.mu);
        cudaStream_t s = w.stream;
        const double* dd = distances;
        if (memory == RF_MEMORY_HOST) {
            w.d.ensure(n * 8);
            CK(cudaMemcpyAsync(w.d.p, distances, n * 8, cudaMemcpyHostToDevice, s));
            dd = w.d.as<double>();
        }
        w.edges.ensure(ne * 8);
        w.hist.ensure((ne + 1) * 8);
        CK(cudaMemcpyAsync(w.edges.p, edges, ne * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(w.hist.p, 0, (ne + 1) * 8, s));
        k_cdf_hist<<<grid_for(n, 256), 256, (ne + 1) * 8, s>>>(dd, n, w.edges.as<double>(), int(ne),
                                                              w.hist.as<unsigned long long>());
        CK(cudaGetLastError());
        std::vector<unsigned long long> h(ne + 1);
        CK(cudaMemcpyAsync(h.data(), w.hist.p, (ne + 1) * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        unsigned long long run = 0;
        for (uint64_t i = 0; i < ne; ++i) {
            run += h[i];
            cdf[i] = 100.0 * static_cast<double>(run) / static_cast<double>(n);
        }
    });
}

}  // extern "C"
