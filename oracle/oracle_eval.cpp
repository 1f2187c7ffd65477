// ORACLE — test infrastructure only (see oracle.hpp). CPU restatement of the
// reference's evaluation (proj/src/evaluation.cpp, proj/src/dataset_io.cpp
// MatchTimestamps) behind a flat C ABI for pytest. The product computes the
// rigid alignment with Horn's quaternion method; this file follows the
// reference's SVD route (evaluation.cpp:41-50), so agreement checks both.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <map>
#include <tuple>
#include <algorithm>
#include <vector>

#include "oracle.hpp"

using namespace oracle;

namespace {

struct Traj {
    const double* t;
    const double* pose;
    uint64_t n;
    V3d trans(uint64_t i) const { return {pose[12 * i + 9], pose[12 * i + 10], pose[12 * i + 11]}; }
    Pose at(uint64_t i) const { return Pose::FromArray(pose + 12 * i); }
};

// MatchTimestamps, dataset_io.cpp:41-71
std::vector<std::pair<uint64_t, uint64_t>> Match(const Traj& a, const Traj& b, double max_dt) {
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
        return std::tie(x.dt, x.i, x.j) < std::tie(y.dt, y.i, y.j);
    });
    std::vector<bool> ua(a.n, false), ub(b.n, false);
    std::vector<std::pair<uint64_t, uint64_t>> pairs;
    for (const Cand& c : cands) {
        if (ua[c.i] || ub[c.j]) continue;
        ua[c.i] = true;
        ub[c.j] = true;
        pairs.emplace_back(c.i, c.j);
    }
    std::sort(pairs.begin(), pairs.end(), [&](const auto& x, const auto& y) { return a.t[x.first] < a.t[y.first]; });
    return pairs;
}

// 3x3 SVD W = U diag(s) V^T by one-sided Jacobi, singular values descending
// (Eigen::JacobiSVD's ordering, which the reflection guard relies on).
void Svd3(const M3d& W, M3d& U, double s[3], M3d& V) {
    double a[3][3], v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) a[r][c] = W(r, c);
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double al = 0, be = 0, ga = 0;
                for (int r = 0; r < 3; ++r) {
                    al += a[r][p] * a[r][p];
                    be += a[r][q] * a[r][q];
                    ga += a[r][p] * a[r][q];
                }
                if (std::abs(ga) <= 1e-300 || std::abs(ga) <= 1e-17 * std::sqrt(al * be)) continue;
                rotated = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (int r = 0; r < 3; ++r) {
                    const double x = a[r][p], y = a[r][q];
                    a[r][p] = c * x - sn * y;
                    a[r][q] = sn * x + c * y;
                    const double vx = v[r][p], vy = v[r][q];
                    v[r][p] = c * vx - sn * vy;
                    v[r][q] = sn * vx + c * vy;
                }
            }
        if (!rotated) break;
    }
    double sv[3];
    for (int c = 0; c < 3; ++c) sv[c] = std::sqrt(a[0][c] * a[0][c] + a[1][c] * a[1][c] + a[2][c] * a[2][c]);
    int order[3] = {0, 1, 2};
    std::sort(order, order + 3, [&](int x, int y) { return sv[x] > sv[y]; });
    // U = A V / s for the significant singular values; the rest completes an
    // orthonormal basis (a zero-norm column of A carries no direction, and a
    // rounding-size one only noise), like the orthogonal U of Eigen's JacobiSVD.
    V3d u[3], col[3];
    const double tiny = 1e-13 * sv[order[0]];
    bool sig[3];
    for (int k = 0; k < 3; ++k) {
        const int c = order[k];
        s[k] = sv[c];
        for (int r = 0; r < 3; ++r) V(r, k) = v[r][c];
        col[k] = {a[0][c], a[1][c], a[2][c]};
        sig[k] = sv[c] > tiny && sv[c] > 0;
        u[k] = sig[k] ? col[k] / sv[c] : V3d{0, 0, 0};
    }
    auto unit = [](V3d x) { return x / Norm(x); };
    if (!sig[0]) u[0] = {1, 0, 0};
    if (!sig[1]) {
        const V3d e = std::abs(u[0].x) < 0.9 ? V3d{1, 0, 0} : V3d{0, 1, 0};
        u[1] = unit(Cross(u[0], e));
    }
    const V3d c2 = unit(Cross(u[0], u[1]));
    u[2] = (sig[2] && Dot(col[2], c2) < 0) ? -c2 : c2;
    for (int k = 0; k < 3; ++k)
        for (int r = 0; r < 3; ++r) U(r, k) = u[k][r];
}

double Det3(const M3d& m) {
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
           m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}

M3d Mul(const M3d& a, const M3d& b) {
    M3d r = M3d::Zero();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
    return r;
}

// GridNn, evaluation.cpp:96-199 (cells in a hash map, like CoordHashMap).
struct GridNn {
    double cell;
    const std::vector<float>& pts;
    V3i mn, mx;
    std::map<std::tuple<int, int, int>, std::pair<uint32_t, uint32_t>> cells;  // cell -> [start, end) in ids
    std::vector<uint32_t> ids;
    static std::tuple<int, int, int> Key(const V3i& c) { return {c.x, c.y, c.z}; }
    V3i CellOf(const float* p) const {
        return {int(std::floor(double(p[0]) / cell)), int(std::floor(double(p[1]) / cell)),
                int(std::floor(double(p[2]) / cell))};
    }
    GridNn(const std::vector<float>& points, double c) : cell(c), pts(points) {
        const size_t n = points.size() / 3;
        mn = {std::numeric_limits<int>::max(), std::numeric_limits<int>::max(), std::numeric_limits<int>::max()};
        mx = {std::numeric_limits<int>::min(), std::numeric_limits<int>::min(), std::numeric_limits<int>::min()};
        std::vector<V3i> coords(n);
        std::map<std::tuple<int, int, int>, std::vector<uint32_t>> buckets;
        for (size_t i = 0; i < n; ++i) {
            coords[i] = CellOf(&points[3 * i]);
            for (int a = 0; a < 3; ++a) {
                mn[a] = std::min(mn[a], coords[i][a]);
                mx[a] = std::max(mx[a], coords[i][a]);
            }
            buckets[{coords[i].x, coords[i].y, coords[i].z}].push_back(uint32_t(i));
        }
        for (auto& [k, v] : buckets) {
            const uint32_t s = uint32_t(ids.size());
            ids.insert(ids.end(), v.begin(), v.end());
            cells[k] = {s, uint32_t(ids.size())};
        }
    }
    double Nearest(const float* q) const {
        const V3i qc = CellOf(q);
        int r_limit = 0, r_first = 0;
        for (int a = 0; a < 3; ++a) {
            r_limit = std::max({r_limit, std::abs(qc[a] - mn[a]), std::abs(mx[a] - qc[a])});
            r_first = std::max({r_first, mn[a] - qc[a], qc[a] - mx[a]});
        }
        double best = std::numeric_limits<double>::infinity();
        auto fn = [&](const V3i& c) {
            const auto it = cells.find(Key(c));
            if (it == cells.end()) return;
            for (uint32_t k = it->second.first; k < it->second.second; ++k) {
                const float* p = &pts[3 * size_t(ids[k])];
                const V3d d{double(p[0] - q[0]), double(p[1] - q[1]), double(p[2] - q[2])};
                best = std::min(best, Norm(d));
            }
        };
        const V3i lo = mn - qc, hi = mx - qc;
        for (int r = r_first; r <= r_limit; ++r) {
            if (best <= (r - 1) * cell) break;
            if (r == 0) {
                fn(qc);
                continue;
            }
            auto face = [&](int axis, int side, int ua, int u0, int u1, int va, int v0, int v1) {
                if (side < lo[axis] || side > hi[axis]) return;
                u0 = std::max(u0, lo[ua]);
                u1 = std::min(u1, hi[ua]);
                v0 = std::max(v0, lo[va]);
                v1 = std::min(v1, hi[va]);
                V3i p;
                p[axis] = side;
                for (int u = u0; u <= u1; ++u) {
                    p[ua] = u;
                    for (int v = v0; v <= v1; ++v) {
                        p[va] = v;
                        fn(qc + p);
                    }
                }
            };
            for (int side = -r; side <= r; side += 2 * r) {
                face(0, side, 1, -r, r, 2, -r, r);
                face(1, side, 0, -r + 1, r - 1, 2, -r, r);
                face(2, side, 0, -r + 1, r - 1, 1, -r + 1, r - 1);
            }
        }
        return best;
    }
};

}  // namespace

extern "C" {

const char* o_last_error(void);
int o_eval_guard_set(const char* msg);

// AteRmse, evaluation.cpp:26-62. Returns 0, 1 (invalid) or 5 (runtime_error).
int o_ate_rmse(const double* et, const double* ep, uint64_t ne, const double* gt, const double* gp, uint64_t ng,
               double max_dt, double* rmse, double alignment[12], uint64_t* npairs) {
    const Traj est{et, ep, ne}, g{gt, gp, ng};
    const auto pairs = Match(est, g, max_dt);
    if (pairs.size() < 3) {
        o_eval_guard_set(("need at least 3 associated poses, got " + std::to_string(pairs.size())).c_str());
        return 5;
    }
    V3d ce{}, cg{};
    for (const auto& [i, j] : pairs) {
        ce = ce + est.trans(i);
        cg = cg + g.trans(j);
    }
    ce = ce / double(pairs.size());
    cg = cg / double(pairs.size());
    M3d w = M3d::Zero();
    for (const auto& [i, j] : pairs) {
        const V3d a = g.trans(j) - cg, b = est.trans(i) - ce;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) w(r, c) += a[r] * b[c];
    }
    M3d U, V;
    double s[3];
    Svd3(w, U, s, V);
    const M3d Vt = Transpose(V);
    M3d S = M3d::Identity();
    if (Det3(Mul(U, Vt)) < 0) S(2, 2) = -1.0;
    const M3d R = Mul(Mul(U, S), Vt);
    const V3d t = cg - R * ce;
    Pose al{R, t};
    double sum_sq = 0.0;
    for (const auto& [i, j] : pairs) {
        const V3d d = al * est.trans(i) - g.trans(j);
        sum_sq += Dot(d, d);
    }
    *rmse = std::sqrt(sum_sq / double(pairs.size()));
    al.ToArray(alignment);
    *npairs = pairs.size();
    return 0;
}

// RpeOverTime, evaluation.cpp:64-92. Returns the sample count (or -1: delta <= 0).
int64_t o_rpe_over_time(const double* et, const double* ep, uint64_t ne, const double* gt, const double* gp,
                        uint64_t ng, double delta, double max_dt, double* ts, double* err, uint64_t cap) {
    if (!(delta > 0)) return -1;
    const Traj est{et, ep, ne}, g{gt, gp, ng};
    const auto pairs = Match(est, g, max_dt);
    uint64_t n = 0;
    for (size_t k = 0; k < pairs.size(); ++k) {
        const double target = est.t[pairs[k].first] + delta;
        size_t best = pairs.size();
        double best_err = max_dt;
        for (size_t m = k + 1; m < pairs.size(); ++m) {
            const double e = std::abs(est.t[pairs[m].first] - target);
            if (e <= best_err) {
                best_err = e;
                best = m;
            }
            if (est.t[pairs[m].first] > target + max_dt) break;
        }
        if (best == pairs.size()) continue;
        const Pose rel_est = est.at(pairs[k].first).Inverse() * est.at(pairs[best].first);
        const Pose rel_gt = g.at(pairs[k].second).Inverse() * g.at(pairs[best].second);
        const Pose e = rel_gt.Inverse() * rel_est;
        if (n < cap) {
            ts[n] = est.t[pairs[k].first];
            err[n] = Norm(e.t);
        }
        ++n;
    }
    return int64_t(n);
}

// NearestDistances, evaluation.cpp:203-217. Returns 0 or 1 (empty reference).
int o_nearest_distances(const float* q, uint64_t nq, const float* r, uint64_t nr, double* out) {
    if (nr == 0) {
        o_eval_guard_set("reference cloud is empty");
        return 1;
    }
    std::vector<float> ref(r, r + 3 * nr);
    float lo[3] = {r[0], r[1], r[2]}, hi[3] = {r[0], r[1], r[2]};
    for (uint64_t i = 0; i < nr; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], r[3 * i + a]);
            hi[a] = std::max(hi[a], r[3 * i + a]);
        }
    const V3d d{double(hi[0] - lo[0]), double(hi[1] - lo[1]), double(hi[2] - lo[2])};
    const GridNn grid(ref, std::max(Norm(d) / 256.0, 1e-6));
    for (uint64_t i = 0; i < nq; ++i) out[i] = grid.Nearest(q + 3 * i);
    return 0;
}

// DistanceCdf, evaluation.cpp:219-236. Returns 0 or 1 (invalid argument).
int o_distance_cdf(const double* d, uint64_t n, const double* edges, uint64_t ne, double* cdf) {
    if (n == 0) {
        o_eval_guard_set("no distances");
        return 1;
    }
    for (uint64_t i = 1; i < ne; ++i)
        if (!(edges[i] > edges[i - 1])) {
            o_eval_guard_set("bin edges must be ascending");
            return 1;
        }
    std::vector<double> sorted(d, d + n);
    std::sort(sorted.begin(), sorted.end());
    for (uint64_t i = 0; i < ne; ++i) {
        const auto it = std::upper_bound(sorted.begin(), sorted.end(), edges[i]);
        cdf[i] = 100.0 * double(it - sorted.begin()) / double(sorted.size());
    }
    return 0;
}

}  // extern "C"
