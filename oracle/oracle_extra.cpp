// ORACLE — test infrastructure only (see oracle.hpp). Restatement of the
// reference's synthetic renderer (input generation for parity fixtures) and
// marching-cubes extraction. Paths relative to /root/reference/proj.
#include <algorithm>
#include <map>
#include <random>
#include <sstream>
#include <unordered_map>

#include "oracle.hpp"

namespace oracle {

#include "mc_table.inc"

// ---------------------------------------------------------------------------
// Quaternions (the Eigen::Quaterniond operations synth.cpp relies on)
// ---------------------------------------------------------------------------
static Quat Normalized(const Quat& q) {
    const double n = std::sqrt(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
}

Pose PoseFromQuat(const Quat& qin, const V3d& t) {  // geometry.hpp:78-79 (q.normalized().toRotationMatrix())
    const Quat q = Normalized(qin);
    const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
    const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
    const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
    const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
    Pose p;
    p.R(0, 0) = 1.0 - (tyy + tzz);
    p.R(0, 1) = txy - twz;
    p.R(0, 2) = txz + twy;
    p.R(1, 0) = txy + twz;
    p.R(1, 1) = 1.0 - (txx + tzz);
    p.R(1, 2) = tyz - twx;
    p.R(2, 0) = txz - twy;
    p.R(2, 1) = tyz + twx;
    p.R(2, 2) = 1.0 - (txx + tyy);
    p.t = t;
    return p;
}

Quat QuatFromMatrix(const M3d& m) {  // Eigen quaternion_assign_impl (Shepperd)
    Quat q;
    double t = (m(0, 0) + m(1, 1)) + m(2, 2);
    if (t > 0.0) {
        t = std::sqrt(t + 1.0);
        q.w = 0.5 * t;
        t = 0.5 / t;
        q.x = (m(2, 1) - m(1, 2)) * t;
        q.y = (m(0, 2) - m(2, 0)) * t;
        q.z = (m(1, 0) - m(0, 1)) * t;
    } else {
        int i = 0;
        if (m(1, 1) > m(0, 0)) i = 1;
        if (m(2, 2) > m(i, i)) i = 2;
        const int j = (i + 1) % 3, k = (j + 1) % 3;
        t = std::sqrt(((m(i, i) - m(j, j)) - m(k, k)) + 1.0);
        double c[3];
        c[i] = 0.5 * t;
        t = 0.5 / t;
        q.w = (m(k, j) - m(j, k)) * t;
        c[j] = (m(j, i) + m(i, j)) * t;
        c[k] = (m(k, i) + m(i, k)) * t;
        q.x = c[0];
        q.y = c[1];
        q.z = c[2];
    }
    return q;
}

static Quat Slerp(const Quat& a, double t, const Quat& b) {  // Eigen QuaternionBase::slerp
    const double one = 1.0 - std::numeric_limits<double>::epsilon();
    const double d = ((a.x * b.x + a.y * b.y) + a.z * b.z) + a.w * b.w;
    const double absd = std::abs(d);
    double s0, s1;
    if (absd >= one) {
        s0 = 1.0 - t;
        s1 = t;
    } else {
        const double theta = std::acos(absd);
        const double st = std::sin(theta);
        s0 = std::sin((1.0 - t) * theta) / st;
        s1 = std::sin(t * theta) / st;
    }
    if (d < 0) s1 = -s1;
    return {s0 * a.w + s1 * b.w, s0 * a.x + s1 * b.x, s0 * a.y + s1 * b.y, s0 * a.z + s1 * b.z};
}

// synth.cpp:26-45
static Pose InterpolatePose(const Pose& a, const Pose& b, double alpha) {
    const Quat q = Slerp(QuatFromMatrix(a.R), alpha, QuatFromMatrix(b.R));
    const V3d t = (1.0 - alpha) * a.t + alpha * b.t;
    return PoseFromQuat(q, t);
}

Pose Primitive::PoseAt(double time) const {
    if (keyframes.empty()) return Pose{};
    if (time <= keyframes.front().first) return keyframes.front().second;
    if (time >= keyframes.back().first) return keyframes.back().second;
    size_t hi = 1;
    while (keyframes[hi].first < time) ++hi;
    const auto& [t0, p0] = keyframes[hi - 1];
    const auto& [t1, p1] = keyframes[hi];
    return InterpolatePose(p0, p1, (time - t0) / (t1 - t0));
}

// synth.cpp:79-122
static double Intersect(const Primitive& p, const V3d& o, const V3d& d) {
    constexpr double kMiss = std::numeric_limits<double>::infinity();
    constexpr double kRayEps = 1e-6;
    switch (p.shape) {
        case 0: {
            const double denom = Dot(p.b, d);
            if (std::abs(denom) < 1e-12) return kMiss;
            const double t = Dot(p.b, p.a - o) / denom;
            return t > kRayEps ? t : kMiss;
        }
        case 1: {
            const V3d oc = o - p.a;
            const double a = Dot(d, d);
            const double half_b = Dot(oc, d);
            const double c = Dot(oc, oc) - p.b.x * p.b.x;
            const double disc = half_b * half_b - a * c;
            if (disc < 0) return kMiss;
            const double root = std::sqrt(disc);
            const double t0 = (-half_b - root) / a;
            if (t0 > kRayEps) return t0;
            const double t1 = (-half_b + root) / a;
            return t1 > kRayEps ? t1 : kMiss;
        }
        default: {
            double tn = -std::numeric_limits<double>::infinity(), tf = std::numeric_limits<double>::infinity();
            for (int i = 0; i < 3; ++i) {
                const double lo = p.a[i] - p.b[i], hi = p.a[i] + p.b[i];
                if (std::abs(d[i]) < 1e-15) {
                    if (o[i] < lo || o[i] > hi) return kMiss;
                    continue;
                }
                double t0 = (lo - o[i]) / d[i], t1 = (hi - o[i]) / d[i];
                if (t0 > t1) std::swap(t0, t1);
                tn = std::max(tn, t0);
                tf = std::min(tf, t1);
            }
            if (tn > tf || tf < kRayEps) return kMiss;
            return tn > kRayEps ? tn : tf;
        }
    }
}

static Rgb8 AlbedoAt(const Primitive& p, const V3d& hit) {  // synth.cpp:124-132
    if (!p.checker) return p.primary;
    long parity = 0;
    for (int i = 0; i < 3; ++i) parity += long(std::floor((hit[i] + 0.0123 * p.cell) / p.cell));
    return (parity & 1) ? p.secondary : p.primary;
}

Rendered RenderFrame(const Scene& s, size_t index) {  // synth.cpp:136-203
    if (index >= s.camera.size()) throw std::out_of_range("no such camera keyframe");
    const double time = s.camera[index].first;
    const Pose& cam = s.camera[index].second;
    const Intrinsics& k = s.intr;
    Rendered out;
    out.frame.timestamp = time;
    out.frame.intr = k;
    out.frame.depth = DepthImage(k.width, k.height, 0.f);
    out.frame.color = ColorImage(k.width, k.height, Rgb8{});
    out.true_depth = DepthImage(k.width, k.height, 0.f);
    out.labels = Mask(k.width, k.height, 0);
    struct View {
        M3d rot;
        V3d trans;
        const Primitive* prim;
    };
    std::vector<View> views;
    for (const Primitive& p : s.prims) {
        const Pose w2o = p.PoseAt(time).Inverse();
        views.push_back({w2o.R, w2o.t, &p});
    }
    const V3d origin = cam.t;
    for (int v = 0; v < k.height; ++v)
        for (int u = 0; u < k.width; ++u) {
            const V3d dir = cam.R * V3d{(u - k.cx) / k.fx, (v - k.cy) / k.fy, 1.0};
            double best = std::numeric_limits<double>::infinity();
            const View* bv = nullptr;
            for (const View& vw : views) {
                const V3d o = vw.rot * origin + vw.trans;
                const V3d d = vw.rot * dir;
                const double t = Intersect(*vw.prim, o, d);
                if (t < best) {
                    best = t;
                    bv = &vw;
                }
            }
            if (!bv) continue;
            out.true_depth(u, v) = float(best);
            out.labels(u, v) = bv->prim->dynamic ? 1 : 0;
            const V3d hit = bv->rot * (origin + best * dir) + bv->trans;
            out.frame.color(u, v) = AlbedoAt(*bv->prim, hit);
        }
    std::mt19937 rng(s.seed ^ static_cast<uint32_t>(index * 2654435761u));
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_real_distribution<double> uniform(0.0, 1.0);
    for (int v = 0; v < k.height; ++v)
        for (int u = 0; u < k.width; ++u) {
            const float z = out.true_depth(u, v);
            if (!DepthValid(z)) continue;
            if (s.dropout > 0.0 && uniform(rng) < s.dropout) continue;
            double noisy = z;
            if (s.noise_sigma_scale > 0.0) noisy += gauss(rng) * s.noise_sigma_scale * z * z;
            out.frame.depth(u, v) = noisy > 0.0 ? float(noisy) : 0.f;
        }
    return out;
}

// synth.cpp:207-351 (scene script parser)
static Pose ParsePose(std::istringstream& ls, const std::string& where) {
    double tx, ty, tz, qx, qy, qz, qw;
    if (!(ls >> tx >> ty >> tz >> qx >> qy >> qz >> qw))
        throw std::invalid_argument(where + ": expected tx ty tz qx qy qz qw");
    const Quat q{qw, qx, qy, qz};
    const double n = std::sqrt(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
    if (std::abs(n - 1.0) > 1e-3) throw std::invalid_argument(where + ": quaternion norm is not 1");
    return PoseFromQuat(Normalized(q), {tx, ty, tz});
}

static void ParseAlbedo(std::istringstream& ls, Primitive& p, const std::string& where) {
    std::string word, kind;
    if (!(ls >> word >> kind) || word != "albedo") throw std::invalid_argument(where + ": expected albedo");
    auto rgb = [&](Rgb8& o) {
        int r, g, b;
        if (!(ls >> r >> g >> b) || r < 0 || r > 255 || g < 0 || g > 255 || b < 0 || b > 255)
            throw std::invalid_argument(where + ": albedo channels must be 0..255");
        o = Rgb8{uint8_t(r), uint8_t(g), uint8_t(b)};
    };
    if (kind == "uniform") {
        rgb(p.primary);
    } else if (kind == "checker") {
        p.checker = true;
        if (!(ls >> p.cell) || !(p.cell > 0)) throw std::invalid_argument(where + ": checker cell");
        rgb(p.primary);
        rgb(p.secondary);
    } else {
        throw std::invalid_argument(where + ": unknown albedo kind");
    }
}

Scene Scene::Parse(const std::string& text) {
    Scene s;
    std::istringstream in(text);
    std::string line;
    size_t no = 0;
    while (std::getline(in, line)) {
        ++no;
        const std::string where = "scene line " + std::to_string(no);
        const size_t first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos || line[first] == '#') continue;
        std::istringstream ls(line);
        std::string dir;
        ls >> dir;
        if (dir == "intrinsics") {
            Intrinsics k;
            if (!(ls >> k.fx >> k.fy >> k.cx >> k.cy >> k.width >> k.height >> k.depth_scale) || !k.Valid())
                throw std::invalid_argument(where + ": invalid intrinsics");
            s.intr = k;
        } else if (dir == "noise") {
            if (!(ls >> s.noise_sigma_scale >> s.dropout) || s.noise_sigma_scale < 0 || s.dropout < 0 ||
                s.dropout >= 1)
                throw std::invalid_argument(where + ": invalid noise parameters");
        } else if (dir == "seed") {
            if (!(ls >> s.seed)) throw std::invalid_argument(where + ": invalid seed");
        } else if (dir == "primitive") {
            Primitive p;
            std::string motion, shape;
            if (!(ls >> p.name >> motion >> shape)) throw std::invalid_argument(where + ": primitive");
            if (motion != "static" && motion != "dynamic") throw std::invalid_argument(where + ": motion");
            p.dynamic = motion == "dynamic";
            if (shape == "plane") {
                p.shape = 0;
                if (!(ls >> p.a.x >> p.a.y >> p.a.z >> p.b.x >> p.b.y >> p.b.z)) throw std::invalid_argument(where);
                const double n = Norm(p.b);
                if (n < 1e-9) throw std::invalid_argument(where + ": plane normal");
                p.b = p.b / n;
            } else if (shape == "sphere") {
                p.shape = 1;
                if (!(ls >> p.a.x >> p.a.y >> p.a.z >> p.b.x) || !(p.b.x > 0)) throw std::invalid_argument(where);
                p.b.y = p.b.z = 0.0;
            } else if (shape == "box") {
                p.shape = 2;
                if (!(ls >> p.a.x >> p.a.y >> p.a.z >> p.b.x >> p.b.y >> p.b.z) ||
                    !(std::min(p.b.x, std::min(p.b.y, p.b.z)) > 0))
                    throw std::invalid_argument(where);
            } else {
                throw std::invalid_argument(where + ": unknown shape");
            }
            ParseAlbedo(ls, p, where);
            for (const Primitive& e : s.prims)
                if (e.name == p.name) throw std::invalid_argument(where + ": duplicate primitive");
            s.prims.push_back(std::move(p));
        } else if (dir == "keyframe") {
            std::string name;
            double t;
            if (!(ls >> name >> t)) throw std::invalid_argument(where + ": keyframe");
            const Pose pose = ParsePose(ls, where);
            Primitive* target = nullptr;
            for (Primitive& p : s.prims)
                if (p.name == name) target = &p;
            if (!target) throw std::invalid_argument(where + ": unknown primitive");
            if (!target->keyframes.empty() && t <= target->keyframes.back().first)
                throw std::invalid_argument(where + ": keyframe times must increase");
            target->keyframes.emplace_back(t, pose);
        } else if (dir == "camera") {
            double t;
            if (!(ls >> t)) throw std::invalid_argument(where + ": camera");
            if (!s.camera.empty() && t <= s.camera.back().first)
                throw std::invalid_argument(where + ": camera times must increase");
            s.camera.emplace_back(t, ParsePose(ls, where));
        } else {
            throw std::invalid_argument(where + ": unknown directive");
        }
    }
    return s;
}

// ---------------------------------------------------------------------------
// Marching cubes, mesh.cpp:22-181
// ---------------------------------------------------------------------------
namespace {
constexpr int kCornerOffset[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                     {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
constexpr int kEdgeEnds[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                  {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
constexpr int kEdgeAxis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};
constexpr int kEdgeLowCorner[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};

struct McTables {
    int tri[256][16];
    int edges[256];
    McTables() {
        int c = 0, n = 0;
        for (const char* p = kMcTriHex; *p && c < 256; ++p) {
            if (*p == ' ') {
                tri[c][n] = -1;
                ++c;
                n = 0;
            } else {
                tri[c][n++] = (*p >= 'a') ? (*p - 'a' + 10) : (*p - '0');
            }
        }
        for (int cube = 0; cube < 256; ++cube) {  // active edges: endpoint signs differ
            int e = 0;
            for (int k = 0; k < 12; ++k)
                if (((cube >> kEdgeEnds[k][0]) & 1) != ((cube >> kEdgeEnds[k][1]) & 1)) e |= 1 << k;
            edges[cube] = e;
        }
    }
};
const McTables& Tables() {
    static const McTables t;
    return t;
}

uint64_t EdgeKey(const V3i& v, int axis) {  // mesh.cpp:31-37
    constexpr uint64_t kBias = 1u << 20;
    const uint64_t x = (uint64_t(int64_t(v.x) + int64_t(kBias))) & 0x1FFFFF;
    const uint64_t y = (uint64_t(int64_t(v.y) + int64_t(kBias))) & 0x1FFFFF;
    const uint64_t z = (uint64_t(int64_t(v.z) + int64_t(kBias))) & 0x1FFFFF;
    return (((z << 21 | y) << 21) | x) << 2 | uint64_t(axis);
}

struct BlockMesh {
    std::vector<uint64_t> keys;
    std::vector<float> verts;
    std::vector<uint8_t> cols;
    std::vector<int32_t> faces;
};

float LerpChannel(uint8_t a, uint8_t b, double t) { return float(a + (double(b) - a) * t); }

BlockMesh ExtractBlock(const Volume& vol, const VoxelBlock& block, int min_weight) {  // mesh.cpp:50-145
    const McTables& T = Tables();
    const int side = vol.config().block_side;
    BlockMesh out;
    std::unordered_map<uint64_t, int> local;
    const Voxel* corners[8];
    double sdf[8];
    const V3i bb = block.coord * side;
    for (int z = 0; z < side; ++z)
        for (int y = 0; y < side; ++y)
            for (int x = 0; x < side; ++x) {
                const V3i base = bb + V3i{x, y, z};
                bool complete = true;
                for (int k = 0; k < 8 && complete; ++k) {
                    const V3i vc = base + V3i{kCornerOffset[k][0], kCornerOffset[k][1], kCornerOffset[k][2]};
                    const Voxel* v;
                    if (vc.x < bb.x + side && vc.y < bb.y + side && vc.z < bb.z + side) {
                        const V3i l = vc - bb;
                        v = &block.voxels[(size_t(l.z) * side + l.y) * side + l.x];
                    } else {
                        v = vol.VoxelHandle(vc);
                    }
                    if (!v || v->weight < min_weight) {
                        complete = false;
                        break;
                    }
                    corners[k] = v;
                    sdf[k] = double(v->sdf);
                }
                if (!complete) continue;
                int cube = 0;
                for (int k = 0; k < 8; ++k)
                    if (sdf[k] < 0.0) cube |= 1 << k;
                if (T.edges[cube] == 0) continue;
                int ev[12];
                for (int e = 0; e < 12; ++e) {
                    if (!(T.edges[cube] & (1 << e))) continue;
                    const int lc = kEdgeLowCorner[e];
                    const V3i low = base + V3i{kCornerOffset[lc][0], kCornerOffset[lc][1], kCornerOffset[lc][2]};
                    const uint64_t key = EdgeKey(low, kEdgeAxis[e]);
                    const auto found = local.find(key);
                    if (found != local.end()) {
                        ev[e] = found->second;
                        continue;
                    }
                    int a = kEdgeEnds[e][0], b = kEdgeEnds[e][1];
                    if (kCornerOffset[a][kEdgeAxis[e]] > kCornerOffset[b][kEdgeAxis[e]]) std::swap(a, b);
                    const double denom = sdf[b] - sdf[a];
                    const double t = std::abs(denom) < 1e-12 ? 0.5 : std::clamp(-sdf[a] / denom, 0.0, 1.0);
                    V3d p = vol.VoxelCenter(base + V3i{kCornerOffset[a][0], kCornerOffset[a][1], kCornerOffset[a][2]});
                    p[kEdgeAxis[e]] += t * vol.config().voxel_size;
                    const int idx = int(out.keys.size());
                    out.keys.push_back(key);
                    out.verts.push_back(float(p.x));
                    out.verts.push_back(float(p.y));
                    out.verts.push_back(float(p.z));
                    out.cols.push_back(uint8_t(std::lround(LerpChannel(corners[a]->r, corners[b]->r, t))));
                    out.cols.push_back(uint8_t(std::lround(LerpChannel(corners[a]->g, corners[b]->g, t))));
                    out.cols.push_back(uint8_t(std::lround(LerpChannel(corners[a]->b, corners[b]->b, t))));
                    local.emplace(key, idx);
                    ev[e] = idx;
                }
                for (const int* tri = T.tri[cube]; *tri != -1; tri += 3) {
                    const int i0 = ev[tri[0]], i1 = ev[tri[2]], i2 = ev[tri[1]];
                    if (i0 == i1 || i1 == i2 || i0 == i2) continue;
                    const float* v0 = &out.verts[3 * i0];
                    const float* v1 = &out.verts[3 * i1];
                    const float* v2 = &out.verts[3 * i2];
                    const float e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
                    const float e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
                    const float cx = e1[1] * e2[2] - e1[2] * e2[1];
                    const float cy = e1[2] * e2[0] - e1[0] * e2[2];
                    const float cz = e1[0] * e2[1] - e1[1] * e2[0];
                    const double n = std::sqrt((double(cx) * double(cx) + double(cy) * double(cy)) +
                                               double(cz) * double(cz));
                    if (0.5 * n <= 1e-12) continue;
                    out.faces.push_back(i0);
                    out.faces.push_back(i1);
                    out.faces.push_back(i2);
                }
            }
    return out;
}
}  // namespace

Mesh ExtractMesh(const Volume& vol, int min_weight, int threads) {  // mesh.cpp:149-181
    const auto& blocks = vol.blocks();
    std::vector<size_t> order(blocks.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const V3i& ca = blocks[a].coord;
        const V3i& cb = blocks[b].coord;
        if (ca.x != cb.x) return ca.x < cb.x;
        if (ca.y != cb.y) return ca.y < cb.y;
        return ca.z < cb.z;
    });
    std::vector<BlockMesh> parts(blocks.size());
    ParallelFor(order.size(), threads, [&](size_t i) { parts[i] = ExtractBlock(vol, blocks[order[i]], min_weight); });
    Mesh mesh;
    std::unordered_map<uint64_t, int> global;
    for (const BlockMesh& part : parts) {
        std::vector<int> remap(part.keys.size());
        for (size_t i = 0; i < part.keys.size(); ++i) {
            const auto [it, inserted] = global.emplace(part.keys[i], int(mesh.vertices.size() / 3));
            if (inserted) {
                mesh.vertices.insert(mesh.vertices.end(), &part.verts[3 * i], &part.verts[3 * i] + 3);
                mesh.colors.insert(mesh.colors.end(), &part.cols[3 * i], &part.cols[3 * i] + 3);
            }
            remap[i] = it->second;
        }
        for (int32_t f : part.faces) mesh.faces.push_back(remap[f]);
    }
    return mesh;
}

}  // namespace oracle
