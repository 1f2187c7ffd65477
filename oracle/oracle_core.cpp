// ORACLE — test infrastructure only (see oracle.hpp). CPU restatement of the
// reference's geometry, volume, registration, dynamics mask, ray-march and
// pipeline. Each function cites the reference file:line it follows; paths are
// relative to /root/reference/proj.
#include <algorithm>
#include <chrono>
#include <deque>
#include <thread>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------------------
// geometry.cpp:14-57
// ---------------------------------------------------------------------------
Pose ExpMap(const double xi[6]) {
    const V3d v{xi[0], xi[1], xi[2]};
    const V3d w{xi[3], xi[4], xi[5]};
    const double theta = Norm(w);
    const M3d hat = Skew(w);
    const M3d hat2 = hat * hat;
    double a, b, c;
    if (theta < 1e-6) {  // kSmallAngle, geometry.hpp:123
        const double t2 = theta * theta;
        a = 1.0 - t2 / 6.0;
        b = 0.5 - t2 / 24.0;
        c = 1.0 / 6.0 - t2 / 120.0;
    } else {
        const double t2 = theta * theta;
        a = std::sin(theta) / theta;
        b = (1.0 - std::cos(theta)) / t2;
        c = (theta - std::sin(theta)) / (t2 * theta);
    }
    M3d rot, vm;
    for (int i = 0; i < 9; ++i) {
        const double id = (i % 4 == 0) ? 1.0 : 0.0;
        rot.m[i] = (id + a * hat.m[i]) + b * hat2.m[i];
        vm.m[i] = (id + b * hat.m[i]) + c * hat2.m[i];
    }
    return {rot, vm * v};
}

void LogMap(const Pose& p, double xi[6]) {
    // Eigen::AngleAxisd(R) restated: angle from the quaternion.
    const Quat q = QuatFromMatrix(p.R);
    const double n = std::sqrt((q.x * q.x + q.y * q.y) + q.z * q.z);
    V3d w{0, 0, 0};
    if (n > 0) {
        const double angle = 2.0 * std::atan2(n, std::abs(q.w));
        const double sgn = q.w < 0 ? -1.0 : 1.0;
        w = {sgn * q.x / n * angle, sgn * q.y / n * angle, sgn * q.z / n * angle};
    }
    const double theta = Norm(w);
    const M3d hat = Skew(w);
    const M3d hat2 = hat * hat;
    M3d vinv;
    if (theta < 1e-6) {
        for (int i = 0; i < 9; ++i)
            vinv.m[i] = ((i % 4 == 0 ? 1.0 : 0.0) - 0.5 * hat.m[i]) + hat2.m[i] / 12.0;
    } else {
        const double half = 0.5 * theta;
        const double cot = std::cos(half) / std::sin(half);
        const double coeff = (1.0 - half * cot) / (theta * theta);
        for (int i = 0; i < 9; ++i)
            vinv.m[i] = ((i % 4 == 0 ? 1.0 : 0.0) - 0.5 * hat.m[i]) + coeff * hat2.m[i];
    }
    const V3d v = vinv * p.t;
    xi[0] = v.x; xi[1] = v.y; xi[2] = v.z;
    xi[3] = w.x; xi[4] = w.y; xi[5] = w.z;
}

// ---------------------------------------------------------------------------
// tsdf_volume.cpp
// ---------------------------------------------------------------------------
void VolumeConfig::Validate() const {  // tsdf_volume.cpp:40-52
    if (!(voxel_size > 0)) throw std::invalid_argument("voxel_size must be positive");
    if (!(truncation >= voxel_size))
        throw std::invalid_argument("truncation must be at least one voxel_size");
    if (block_side < 2) throw std::invalid_argument("block_side must be at least 2");
    if (max_weight < 1 || max_weight > 255)
        throw std::invalid_argument("max_weight must be in [1, 255]");
    if (carve_weight < 1 || carve_weight > max_weight)
        throw std::invalid_argument("carve_weight must be in [1, max_weight]");
    if (!(min_depth > 0) || !(max_depth > min_depth))
        throw std::invalid_argument("need 0 < min_depth < max_depth");
    if (!(carve_clip > 0)) throw std::invalid_argument("carve_clip must be positive");
    if (max_blocks == 0) throw std::invalid_argument("max_blocks must be positive");
}

const VoxelBlock* Volume::FindBlock(const V3i& bc) const {  // tsdf_volume.cpp:59-62
    const uint32_t* idx = index_.Find(bc);
    return idx ? &blocks_[*idx] : nullptr;
}

bool Volume::AllocateBlock(const V3i& bc) {  // tsdf_volume.cpp:64-77
    if (index_.Find(bc) != nullptr) return false;
    if (blocks_.size() >= cfg_.max_blocks)
        throw ResourceLimitError("voxel block budget exhausted (" +
                                 std::to_string(cfg_.max_blocks) + " blocks)");
    const int side = cfg_.block_side;
    VoxelBlock block;
    block.coord = bc;
    block.voxels.resize(size_t(side) * side * side);
    blocks_.push_back(std::move(block));
    index_.Insert(bc, uint32_t(blocks_.size() - 1));
    ++last_new_blocks;
    return true;
}

const Voxel* Volume::VoxelHandle(const V3i& v) const {  // tsdf_volume.cpp:79-87
    const int side = cfg_.block_side;
    const V3i bc{FloorDiv(v.x, side), FloorDiv(v.y, side), FloorDiv(v.z, side)};
    const VoxelBlock* block = FindBlock(bc);
    if (!block) return nullptr;
    const V3i l = v - bc * side;
    return &block->voxels[(size_t(l.z) * side + l.y) * side + l.x];
}


void Volume::AllocateForFrame(const DepthImage& depth, const Intrinsics& k, const Pose& c2w,
                              const Mask* mask) {  // tsdf_volume.cpp:93-113
    const double tau = cfg_.truncation;
    const double ext = block_extent();
    last_dda_visits = 0;
    last_new_blocks = 0;
    for (int v = 0; v < depth.h; ++v) {
        for (int u = 0; u < depth.w; ++u) {
            const float d = depth(u, v);
            if (!DepthValid(d) || d < cfg_.min_depth || d > cfg_.max_depth) continue;
            if (mask && (*mask)(u, v)) continue;
            const V3d dir{(u - k.cx) / k.fx, (v - k.cy) / k.fy, 1.0};
            const double z0 = std::max(double(d) - tau, 1e-4);
            const double z1 = double(d) + tau;
            const V3d w0 = c2w * (z0 * dir);
            const V3d w1 = c2w * (z1 * dir);
            WalkGridSegment(w0, w1, ext, [&](const V3i& b) {
                ++last_dda_visits;
                AllocateBlock(b);
            });
        }
    }
}

namespace {
// tsdf_volume.cpp:119-151
bool BlockOutsideFrustum(const V3i& bc, double ext, const Pose& w2c, const Intrinsics& k,
                         double max_z) {
    V3d cc[8];
    bool any_behind = false;
    double min_z = std::numeric_limits<double>::infinity();
    for (int c = 0; c < 8; ++c) {
        const V3d corner{(double(bc.x) + double(c & 1)) * ext, (double(bc.y) + double((c >> 1) & 1)) * ext,
                         (double(bc.z) + double(c >> 2)) * ext};
        cc[c] = w2c * corner;
        if (cc[c].z <= 1e-9) any_behind = true;
        min_z = std::min(min_z, cc[c].z);
    }
    if (min_z > max_z) return true;
    if (any_behind) {
        for (int c = 0; c < 8; ++c)
            if (cc[c].z > 1e-9) return false;
        return true;
    }
    double min_u = std::numeric_limits<double>::infinity(), max_u = -min_u;
    double min_v = min_u, max_v = -min_u;
    for (int c = 0; c < 8; ++c) {
        double pu, pv;
        Project(cc[c], k, pu, pv);
        min_u = std::min(min_u, pu);
        max_u = std::max(max_u, pu);
        min_v = std::min(min_v, pv);
        max_v = std::max(max_v, pv);
    }
    return max_u < -0.5 || min_u > k.width - 0.5 || max_v < -0.5 || min_v > k.height - 0.5;
}
}  // namespace

void Volume::Integrate(const Frame& f, const Pose& c2w, const Mask* mask,
                       int threads) {  // tsdf_volume.cpp:155-202
    const Pose w2c = c2w.Inverse();
    const double tau = cfg_.truncation;
    const int side = cfg_.block_side;
    const Intrinsics& k = f.intr;
    ParallelFor(blocks_.size(), threads, [&](size_t bi) {
        VoxelBlock& block = blocks_[bi];
        if (BlockOutsideFrustum(block.coord, block_extent(), w2c, k, cfg_.max_depth + tau)) return;
        const V3i base = block.coord * side;
        size_t idx = 0;
        for (int z = 0; z < side; ++z)
            for (int y = 0; y < side; ++y)
                for (int x = 0; x < side; ++x, ++idx) {
                    const V3d center = VoxelCenter(base + V3i{x, y, z});
                    const V3d pc = w2c * center;
                    if (pc.z <= 1e-9) continue;
                    double pu_d, pv_d;
                    Project(pc, k, pu_d, pv_d);
                    const int pu = int(std::lround(pu_d));
                    const int pv = int(std::lround(pv_d));
                    if (!f.depth.InBounds(pu, pv)) continue;
                    if (mask && (*mask)(pu, pv)) continue;
                    const float d = f.depth(pu, pv);
                    if (!DepthValid(d) || d < cfg_.min_depth || d > cfg_.max_depth) continue;
                    const double dist = double(d) - pc.z;
                    if (dist <= -tau) continue;
                    Voxel& vox = block.voxels[idx];
                    const double clamped = std::min(dist, tau);
                    const double w = vox.weight;
                    vox.sdf = float((double(vox.sdf) * w + clamped) / (w + 1.0));
                    if (std::abs(dist) <= tau && !f.color.Empty()) {
                        const Rgb8 c = f.color(pu, pv);
                        vox.r = uint8_t(std::lround((vox.r * w + c.r) / (w + 1.0)));
                        vox.g = uint8_t(std::lround((vox.g * w + c.g) / (w + 1.0)));
                        vox.b = uint8_t(std::lround((vox.b * w + c.b) / (w + 1.0)));
                    }
                    vox.weight = uint8_t(std::min<int>(vox.weight + 1, cfg_.max_weight));
                }
    });
}

void Volume::Carve(const DepthImage& depth, const Intrinsics& k, const Pose& c2w,
                   int threads) {  // tsdf_volume.cpp:204-241
    const Pose w2c = c2w.Inverse();
    const double tau = cfg_.truncation;
    const int side = cfg_.block_side;
    const int cw = cfg_.carve_weight;
    ParallelFor(blocks_.size(), threads, [&](size_t bi) {
        VoxelBlock& block = blocks_[bi];
        if (BlockOutsideFrustum(block.coord, block_extent(), w2c, k, cfg_.carve_clip)) return;
        const V3i base = block.coord * side;
        size_t idx = 0;
        for (int z = 0; z < side; ++z)
            for (int y = 0; y < side; ++y)
                for (int x = 0; x < side; ++x, ++idx) {
                    const V3d center = VoxelCenter(base + V3i{x, y, z});
                    const V3d pc = w2c * center;
                    if (pc.z <= 1e-9 || pc.z >= cfg_.carve_clip) continue;
                    double pu_d, pv_d;
                    Project(pc, k, pu_d, pv_d);
                    const int pu = int(std::lround(pu_d));
                    const int pv = int(std::lround(pv_d));
                    if (!depth.InBounds(pu, pv)) continue;
                    const float d = depth(pu, pv);
                    if (!DepthValid(d)) continue;
                    if (pc.z >= double(d) - tau) continue;
                    Voxel& vox = block.voxels[idx];
                    const double w = vox.weight;
                    vox.sdf = float((double(vox.sdf) * w + tau * cw) / (w + cw));
                    vox.weight = uint8_t(std::min<int>(vox.weight + cw, cfg_.max_weight));
                }
    });
}

bool Volume::GatherCorners(const V3i& base, const Voxel* corners[8]) const {  // tsdf_volume.cpp:243-268
    const int side = cfg_.block_side;
    const V3i b0{FloorDiv(base.x, side), FloorDiv(base.y, side), FloorDiv(base.z, side)};
    const V3i b1{FloorDiv(base.x + 1, side), FloorDiv(base.y + 1, side), FloorDiv(base.z + 1, side)};
    if (b0 == b1) {
        const VoxelBlock* block = FindBlock(b0);
        if (!block) return false;
        const V3i l = base - b0 * side;
        for (int c = 0; c < 8; ++c) {
            const int lx = l.x + (c & 1), ly = l.y + ((c >> 1) & 1), lz = l.z + (c >> 2);
            const Voxel& v = block->voxels[(size_t(lz) * side + ly) * side + lx];
            if (v.weight == 0) return false;
            corners[c] = &v;
        }
        return true;
    }
    for (int c = 0; c < 8; ++c) {
        const Voxel* v = VoxelHandle(base + V3i{c & 1, (c >> 1) & 1, c >> 2});
        if (!v || v->weight == 0) return false;
        corners[c] = v;
    }
    return true;
}

namespace {
struct Cell {  // tsdf_volume.cpp:272-283
    V3i base;
    double fx, fy, fz;
};
inline Cell CellOf(const V3d& p, double s) {
    const V3d g{p.x / s - 0.5, p.y / s - 0.5, p.z / s - 0.5};
    const V3d fl{std::floor(g.x), std::floor(g.y), std::floor(g.z)};
    return {{int(fl.x), int(fl.y), int(fl.z)}, g.x - fl.x, g.y - fl.y, g.z - fl.z};
}
inline double IntensityOf(const Voxel& v) { return Intensity(Rgb8{v.r, v.g, v.b}); }
}  // namespace

Sample Volume::SampleSdf(const V3d& p) const {  // tsdf_volume.cpp:291-303
    const Cell cell = CellOf(p, cfg_.voxel_size);
    const Voxel* c[8];
    if (!GatherCorners(cell.base, c)) return {};
    const double wx[2] = {1.0 - cell.fx, cell.fx};
    const double wy[2] = {1.0 - cell.fy, cell.fy};
    const double wz[2] = {1.0 - cell.fz, cell.fz};
    double value = 0.0;
    for (int k = 0; k < 8; ++k) value += wx[k & 1] * wy[(k >> 1) & 1] * wz[k >> 2] * double(c[k]->sdf);
    Sample s;
    s.value = value;
    s.valid = true;
    return s;
}

Sample Volume::SampleIntensity(const V3d& p) const {  // tsdf_volume.cpp:305-317
    const Cell cell = CellOf(p, cfg_.voxel_size);
    const Voxel* c[8];
    if (!GatherCorners(cell.base, c)) return {};
    const double wx[2] = {1.0 - cell.fx, cell.fx};
    const double wy[2] = {1.0 - cell.fy, cell.fy};
    const double wz[2] = {1.0 - cell.fz, cell.fz};
    double value = 0.0;
    for (int k = 0; k < 8; ++k) value += wx[k & 1] * wy[(k >> 1) & 1] * wz[k >> 2] * IntensityOf(*c[k]);
    Sample s;
    s.value = value;
    s.valid = true;
    return s;
}

template <typename F>
Sample Volume::SampleWithGradientImpl(const V3d& p, F&& value_of) const {  // tsdf_volume.cpp:319-346
    const Cell cell = CellOf(p, cfg_.voxel_size);
    const Voxel* c[8];
    if (!GatherCorners(cell.base, c)) return {};
    double val[8];
    for (int k = 0; k < 8; ++k) val[k] = value_of(*c[k]);
    const double wx[2] = {1.0 - cell.fx, cell.fx};
    const double wy[2] = {1.0 - cell.fy, cell.fy};
    const double wz[2] = {1.0 - cell.fz, cell.fz};
    Sample out;
    out.valid = true;
    for (int k = 0; k < 8; ++k) out.value += wx[k & 1] * wy[(k >> 1) & 1] * wz[k >> 2] * val[k];
    const double inv_s = 1.0 / cfg_.voxel_size;
    for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k) {
            out.gradient.x += wy[j] * wz[k] * (val[1 + 2 * j + 4 * k] - val[2 * j + 4 * k]);
            out.gradient.y += wx[j] * wz[k] * (val[j + 2 + 4 * k] - val[j + 4 * k]);
            out.gradient.z += wx[j] * wy[k] * (val[j + 2 * k + 4] - val[j + 2 * k]);
        }
    out.gradient = out.gradient * inv_s;
    return out;
}

Sample Volume::SampleSdfWithGradient(const V3d& p) const {
    return SampleWithGradientImpl(p, [](const Voxel& v) { return double(v.sdf); });
}
Sample Volume::SampleIntensityWithGradient(const V3d& p) const {
    return SampleWithGradientImpl(p, IntensityOf);
}
Sample Volume::SampleSdfGradient(const V3d& p) const {  // tsdf_volume.cpp:358-373
    Sample out;
    const double s = cfg_.voxel_size;
    for (int axis = 0; axis < 3; ++axis) {
        V3d off{0, 0, 0};
        off[axis] = s;
        const Sample hi = SampleSdf(p + off);
        const Sample lo = SampleSdf(p - off);
        if (!hi.valid || !lo.valid) return {};
        out.gradient[axis] = (hi.value - lo.value) / (2.0 * s);
    }
    out.value = SampleSdf(p).value;
    out.valid = true;
    return out;
}

// ---------------------------------------------------------------------------
// registration.cpp
// ---------------------------------------------------------------------------
namespace {
constexpr double kIntensityScale = 1.0 / 255.0;   // registration.cpp:22
constexpr double kRelativeDecreaseTol = 1e-6;     // registration.cpp:26

Accum CombineAccum(Accum a, const Accum& b) {  // registration.cpp:36-43
    for (int i = 0; i < 36; ++i) a.H[i] += b.H[i];
    for (int i = 0; i < 6; ++i) a.b[i] += b.b[i];
    a.depth_error += b.depth_error;
    a.color_error += b.color_error;
    a.valid += b.valid;
    return a;
}
}  // namespace

Accum Accumulate(const Volume& vol, const PyramidLevel& level, const Pose& pose, double cw,
                 bool with_jacobian, bool use_mask, int threads,
                 ResidualImage* out, const Robust& rb) {  // registration.cpp:49-117
    const bool use_color = cw > 0.0 && !level.intensity.Empty();
    const bool has_mask = use_mask && !level.mask.Empty();
    const double min_depth = vol.config().min_depth, max_depth = vol.config().max_depth;
    if (out) {
        out->squared = Image<float>(level.depth.w, level.depth.h, 0.f);
        out->valid = Mask(level.depth.w, level.depth.h, 0);
    }
    const size_t rows = size_t(level.depth.h);
    std::vector<Accum> partial(rows);
    ParallelFor(rows, threads, [&](size_t row) {
        Accum acc;
        const int v = int(row);
        for (int u = 0; u < level.depth.w; ++u) {
            const float d = level.depth(u, v);
            if (!DepthValid(d) || d < min_depth || d > max_depth) continue;
            const bool masked = has_mask && level.mask(u, v) != 0;
            if (masked && !out) continue;
            const V3d x = Backproject(u, v, d, level.intr);
            const V3d y = pose * x;
            if (with_jacobian && !masked) {
                const Sample sdf = vol.SampleSdfWithGradient(y);
                if (!sdf.valid) continue;
                const double r_d = sdf.value;
                const V3d yg = Cross(y, sdf.gradient);
                const double J[6] = {sdf.gradient.x, sdf.gradient.y, sdf.gradient.z, yg.x, yg.y, yg.z};
                // Huber extension: weight hd / |r| and cost 2 hd |r| - hd^2 beyond the threshold
                const double hd = rb.huber_depth, ad = std::fabs(r_d);
                const bool out_d = hd > 0.0 && ad > hd;
                const double wd = out_d ? hd / ad : 1.0;
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j) acc.H[6 * i + j] += out_d ? wd * (J[i] * J[j]) : J[i] * J[j];
                for (int i = 0; i < 6; ++i) acc.b[i] += out_d ? wd * (J[i] * r_d) : J[i] * r_d;
                acc.depth_error += out_d ? 2.0 * hd * ad - hd * hd : r_d * r_d;
                if (use_color) {
                    const Sample in = vol.SampleIntensityWithGradient(y);
                    const double r_c = (in.value - double(level.intensity(u, v))) * kIntensityScale;
                    const V3d yi = Cross(y, in.gradient);
                    double Jc[6] = {in.gradient.x, in.gradient.y, in.gradient.z, yi.x, yi.y, yi.z};
                    for (double& e : Jc) e *= kIntensityScale;
                    const double hc = rb.huber_color, ac = std::fabs(r_c);
                    const bool out_c = hc > 0.0 && ac > hc;
                    const double cwc = out_c ? cw * (hc / ac) : cw;
                    for (int i = 0; i < 6; ++i)
                        for (int j = 0; j < 6; ++j) acc.H[6 * i + j] += cwc * (Jc[i] * Jc[j]);
                    for (int i = 0; i < 6; ++i) acc.b[i] += cwc * (Jc[i] * r_c);
                    acc.color_error += out_c ? 2.0 * hc * ac - hc * hc : r_c * r_c;
                }
                ++acc.valid;
                if (out) {
                    out->squared(u, v) = float(r_d * r_d);
                    out->valid(u, v) = 1;
                }
            } else {
                const Sample sdf = vol.SampleSdf(y);
                if (!sdf.valid) continue;
                const double r_d = sdf.value;
                if (out) {
                    out->squared(u, v) = float(r_d * r_d);
                    out->valid(u, v) = (rb.residual_sign && r_d > 0.0) ? 3 : 1;
                }
                if (masked) continue;
                acc.depth_error += r_d * r_d;
                if (use_color) {
                    const Sample in = vol.SampleIntensity(y);
                    const double r_c = (in.value - double(level.intensity(u, v))) * kIntensityScale;
                    acc.color_error += r_c * r_c;
                }
                ++acc.valid;
            }
        }
        partial[row] = acc;
    });
    Accum acc;  // OrderedReduce fold, parallel.hpp:39-47
    for (size_t r = 0; r < rows; ++r) acc = CombineAccum(acc, partial[r]);
    return acc;
}

PyramidLevel LevelZero(const Frame& f, const Mask* mask) {  // registration.cpp:119-126
    PyramidLevel level;
    level.intr = f.intr;
    level.depth = f.depth;
    if (!f.color.Empty()) {  // image.hpp:85-91
        level.intensity = Image<float>(f.color.w, f.color.h);
        for (size_t i = 0; i < f.color.d.size(); ++i) level.intensity.d[i] = float(Intensity(f.color.d[i]));
    }
    if (mask) level.mask = *mask;
    return level;
}

std::vector<PyramidLevel> BuildPyramid(const Frame& f, const Mask* mask,
                                       int levels) {  // registration.cpp:144-182
    if (levels < 1) throw std::invalid_argument("pyramid needs at least one level");
    std::vector<PyramidLevel> pyr;
    pyr.reserve(levels);
    pyr.push_back(LevelZero(f, mask));
    for (int li = 1; li < levels; ++li) {
        const PyramidLevel& prev = pyr.back();
        PyramidLevel next;
        next.intr = f.intr.Scaled(li);
        const int w = next.intr.width, h = next.intr.height;
        if (w < 1 || h < 1) throw std::invalid_argument("image too small for pyramid level");
        next.depth = DepthImage(w, h, 0.f);
        if (!prev.intensity.Empty()) next.intensity = Image<float>(w, h, 0.f);
        if (!prev.mask.Empty()) next.mask = Mask(w, h, 0);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float closest = 0.f, isum = 0.f;
                uint8_t masked = 0;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) {
                        const int sx = 2 * x + dx, sy = 2 * y + dy;
                        const float d = prev.depth(sx, sy);
                        if (DepthValid(d) && (!DepthValid(closest) || d < closest)) closest = d;
                        if (!prev.intensity.Empty()) isum += prev.intensity(sx, sy);
                        if (!prev.mask.Empty() && prev.mask(sx, sy)) masked = 1;
                    }
                next.depth(x, y) = closest;
                if (!next.intensity.Empty()) next.intensity(x, y) = isum * 0.25f;
                if (!next.mask.Empty()) next.mask(x, y) = masked;
            }
        pyr.push_back(std::move(next));
    }
    return pyr;
}

// Eigen::LDLT (Eigen/src/Cholesky/LDLT.h, lower, unblocked with diagonal
// pivoting; solve through the pseudo-inverse of D) restated for a 6x6.
bool Ldlt6Solve(const double A[36], const double rhs[6], double x[6]) {
    const int n = 6;
    double m[36];
    for (int i = 0; i < 36; ++i) m[i] = A[i];
    // The factorisation only reads the lower triangle.
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) m[6 * i + j] = m[6 * j + i];
    int tr[6];
    double temp[6];
    bool found_zero_pivot = false, ret = true;
    for (int k = 0; k < n; ++k) {
        int big = k;
        double bigv = std::abs(m[6 * k + k]);
        for (int i = k + 1; i < n; ++i)
            if (std::abs(m[6 * i + i]) > bigv) {
                bigv = std::abs(m[6 * i + i]);
                big = i;
            }
        tr[k] = big;
        if (k != big) {
            for (int j = 0; j < k; ++j) std::swap(m[6 * k + j], m[6 * big + j]);
            for (int i = big + 1; i < n; ++i) std::swap(m[6 * i + k], m[6 * i + big]);
            std::swap(m[6 * k + k], m[6 * big + big]);
            for (int i = k + 1; i < big; ++i) {
                const double t = m[6 * i + k];
                m[6 * i + k] = m[6 * big + i];
                m[6 * big + i] = t;
            }
        }
        if (k > 0) {
            for (int j = 0; j < k; ++j) temp[j] = m[6 * j + j] * m[6 * k + j];
            double dot = 0.0;
            for (int j = 0; j < k; ++j) dot += m[6 * k + j] * temp[j];
            m[6 * k + k] -= dot;
            for (int i = k + 1; i < n; ++i) {
                double s = 0.0;
                for (int j = 0; j < k; ++j) s += m[6 * i + j] * temp[j];
                m[6 * i + k] -= s;
            }
        }
        const double akk = m[6 * k + k];
        const bool pivot_valid = std::abs(akk) > 0.0;
        if (k == 0 && !pivot_valid) {  // whole diagonal zero
            for (int j = 0; j < n; ++j) {
                tr[j] = j;
                for (int i = j + 1; i < n; ++i) m[6 * i + j] = 0.0;
            }
            break;
        }
        if (k < n - 1) {
            if (pivot_valid) {
                for (int i = k + 1; i < n; ++i) m[6 * i + k] /= akk;
            } else {
                for (int i = k + 1; i < n; ++i) ret = ret && (m[6 * i + k] == 0.0);
            }
        }
        if (found_zero_pivot && pivot_valid) ret = false;
        else if (!pivot_valid) found_zero_pivot = true;
    }
    if (!ret) return false;
    for (int i = 0; i < n; ++i) x[i] = rhs[i];
    for (int k = 0; k < n; ++k) std::swap(x[k], x[tr[k]]);
    for (int j = 0; j < n; ++j)  // unit lower forward solve, column oriented
        for (int i = j + 1; i < n; ++i) x[i] -= m[6 * i + j] * x[j];
    const double tol = std::numeric_limits<double>::min();
    for (int i = 0; i < n; ++i) {
        if (std::abs(m[6 * i + i]) > tol) x[i] /= m[6 * i + i];
        else x[i] = 0.0;
    }
    for (int j = n - 1; j >= 0; --j)  // unit upper (L^T) back solve
        for (int i = 0; i < j; ++i) x[i] -= m[6 * j + i] * x[j];
    for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[tr[k]]);
    return true;
}

// Jacobi eigenvalues of the symmetric 6x6 (stands in for
// Eigen::SelfAdjointEigenSolver, registration.cpp:136-138; only the
// informational `degenerate` flag depends on it).
bool Degenerate(const Accum& acc) {
    double a[36];
    for (int i = 0; i < 36; ++i) a[i] = acc.H[i];
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < 6; ++i)
            for (int j = i + 1; j < 6; ++j) off += a[6 * i + j] * a[6 * i + j];
        if (off < 1e-300) break;
        for (int p = 0; p < 6; ++p)
            for (int q = p + 1; q < 6; ++q) {
                const double apq = a[6 * p + q];
                if (std::abs(apq) < 1e-300) continue;
                const double theta = (a[6 * q + q] - a[6 * p + p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 6; ++k) {
                    const double akp = a[6 * k + p], akq = a[6 * k + q];
                    a[6 * k + p] = c * akp - s * akq;
                    a[6 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 6; ++k) {
                    const double apk = a[6 * p + k], aqk = a[6 * q + k];
                    a[6 * p + k] = c * apk - s * aqk;
                    a[6 * q + k] = s * apk + c * aqk;
                }
            }
    }
    double mn = a[0], mx = std::abs(a[0]);
    for (int i = 0; i < 6; ++i) {
        mn = std::min(mn, a[7 * i]);
        mx = std::max(mx, std::abs(a[7 * i]));
    }
    return acc.valid == 0 || mn <= 1e-12 * std::max(mx, 1.0);
}

RegistrationResult Register(const Volume& vol, const Frame& f, const Pose& init, const Mask* mask,
                            const RegistrationConfig& cfg) {  // registration.cpp:211-286
    if (cfg.pyramid_levels < 1) throw std::invalid_argument("pyramid_levels must be >= 1");
    if (cfg.max_iterations < 1) throw std::invalid_argument("max_iterations must be >= 1");
    const std::vector<PyramidLevel> pyr = BuildPyramid(f, mask, cfg.pyramid_levels);
    Pose pose = init;
    bool converged = false;
    int total = 0;
    Accum current;
    for (int li = cfg.pyramid_levels - 1; li >= 0; --li) {
        const PyramidLevel& level = pyr[li];
        const size_t min_valid =
            std::max<size_t>(size_t(std::max(cfg.min_valid_residuals, 1)) >> (2 * li), 16);
        const Robust rb{cfg.huber_depth, cfg.huber_color, false};
        current = Accumulate(vol, level, pose, cfg.color_weight, true, true, cfg.threads, nullptr, rb);
        if (current.valid < min_valid)
            throw TrackingLostError("only " + std::to_string(current.valid) +
                                    " valid residuals at pyramid level " + std::to_string(li));
        double lambda = cfg.lm_lambda_init;
        converged = false;
        for (int it = 0; it < cfg.max_iterations; ++it) {
            ++total;
            double dmax = current.H[0];
            for (int i = 1; i < 6; ++i) dmax = std::max(dmax, current.H[7 * i]);
            const double floor = 1e-3 * dmax + 1e-12;
            double damped[36];
            for (int i = 0; i < 36; ++i) damped[i] = current.H[i];
            for (int i = 0; i < 6; ++i) damped[7 * i] += lambda * std::max(current.H[7 * i], floor);
            double negb[6], delta[6];
            for (int i = 0; i < 6; ++i) negb[i] = -current.b[i];
            const bool ok = Ldlt6Solve(damped, negb, delta);
            bool finite = ok;
            for (int i = 0; i < 6 && finite; ++i) finite = std::isfinite(delta[i]);
            if (!finite) {
                lambda = std::min(lambda * cfg.lm_lambda_up, 1e12);
                continue;
            }
            const Pose cand = ExpMap(delta) * pose;
            const Accum trial = Accumulate(vol, level, cand, cfg.color_weight, true, true, cfg.threads, nullptr, rb);
            const double cur_err = current.depth_error + cfg.color_weight * current.color_error;
            const double trial_err = trial.depth_error + cfg.color_weight * trial.color_error;
            if (trial.valid >= min_valid && trial_err < cur_err) {
                const double decrease = cur_err - trial_err;
                pose = cand;
                current = trial;
                lambda = std::max(lambda / cfg.lm_lambda_down, 1e-12);
                double dn = 0.0;
                for (int i = 0; i < 6; ++i) dn += delta[i] * delta[i];
                if (std::sqrt(dn) < cfg.convergence_eps || decrease < kRelativeDecreaseTol * cur_err) {
                    converged = true;
                    break;
                }
            } else {
                lambda = std::min(lambda * cfg.lm_lambda_up, 1e12);
                if (lambda >= 1e12) {
                    converged = true;
                    break;
                }
            }
        }
    }
    RegistrationResult res;
    res.pose = pose;
    res.converged = converged;
    res.iterations = total;
    res.valid_residuals = current.valid;
    res.final_error = current.depth_error + cfg.color_weight * current.color_error;
    PyramidLevel full = pyr[0];
    full.mask = Mask();
    Robust sign;
    sign.residual_sign = cfg.residual_sign;
    Accumulate(vol, full, pose, 0.0, false, false, cfg.threads, &res.residuals, sign);
    return res;
}

// ---------------------------------------------------------------------------
// dynamics_mask.cpp:9-104
// ---------------------------------------------------------------------------
Mask ThresholdResiduals(const ResidualImage& r, const MaskConfig& c) {
    const double thr = c.gamma * c.truncation * c.truncation;
    Mask m(r.squared.w, r.squared.h, 0);
    for (int y = 0; y < m.h; ++y)
        for (int x = 0; x < m.w; ++x)
            if ((r.valid(x, y) && double(r.squared(x, y)) > thr) ||
                (c.free_space > 0.0 && (r.valid(x, y) & 2) && double(r.squared(x, y)) > c.free_space * c.free_space))
                m(x, y) = 1;  // the second clause: the free-space extension (off by default)
    return m;
}

static Mask Morphology(const Mask& m, int radius, bool erode) {  // dynamics_mask.cpp:22-47
    if (radius <= 0) return m;
    Mask out(m.w, m.h, 0);
    for (int y = 0; y < m.h; ++y)
        for (int x = 0; x < m.w; ++x) {
            bool value = erode;
            for (int dy = -radius; dy <= radius && value == erode; ++dy)
                for (int dx = -radius; dx <= radius; ++dx) {
                    const bool on = m.InBounds(x + dx, y + dy) && m(x + dx, y + dy) != 0;
                    if (erode && !on) {
                        value = false;
                        break;
                    }
                    if (!erode && on) {
                        value = true;
                        break;
                    }
                }
            out(x, y) = value ? 1 : 0;
        }
    return out;
}
Mask Erode(const Mask& m, int radius) { return Morphology(m, radius, true); }
Mask Dilate(const Mask& m, int radius) { return Morphology(m, radius, false); }

Mask FloodfillDepth(const Mask& seeds, const DepthImage& depth, double theta,
                    int connectivity) {  // dynamics_mask.cpp:59-96
    if (connectivity != 4 && connectivity != 8) throw std::invalid_argument("connectivity must be 4 or 8");
    if (seeds.w != depth.w || seeds.h != depth.h) throw std::invalid_argument("seed/depth size mismatch");
    static constexpr int kDx[8] = {1, -1, 0, 0, 1, 1, -1, -1};
    static constexpr int kDy[8] = {0, 0, 1, -1, 1, -1, 1, -1};
    Mask out(seeds.w, seeds.h, 0);
    std::deque<std::pair<int, int>> q;
    for (int y = 0; y < seeds.h; ++y)
        for (int x = 0; x < seeds.w; ++x)
            if (seeds(x, y)) {
                out(x, y) = 1;
                q.emplace_back(x, y);
            }
    while (!q.empty()) {
        const auto [x, y] = q.front();
        q.pop_front();
        const float dp = depth(x, y);
        if (!DepthValid(dp)) continue;
        const double bound = theta * double(dp);
        for (int k = 0; k < connectivity; ++k) {
            const int nx = x + kDx[k], ny = y + kDy[k];
            if (!out.InBounds(nx, ny) || out(nx, ny)) continue;
            const float dn = depth(nx, ny);
            if (!DepthValid(dn)) continue;
            if (std::abs(double(dp) - dn) < bound) {
                out(nx, ny) = 1;
                q.emplace_back(nx, ny);
            }
        }
    }
    return out;
}

Mask BuildMask(const ResidualImage& r, const DepthImage& depth, const MaskConfig& c) {
    const Mask raw = ThresholdResiduals(r, c);
    const Mask eroded = Erode(raw, c.erode_radius);
    const Mask grown = FloodfillDepth(eroded, depth, c.theta, c.connectivity);
    return Dilate(grown, c.dilate_radius);
}

// ---------------------------------------------------------------------------
// depth_refinement.cpp:22-93
// ---------------------------------------------------------------------------
DepthImage RaycastDepth(const Volume& vol, const Pose& view, const Intrinsics& k,
                        int bisections, int threads) {  // depth_refinement.cpp:32-79
    const VolumeConfig& vc = vol.config();
    const double step = vc.truncation / 2.0;
    const double z_begin = vc.min_depth, z_end = vc.max_depth;
    DepthImage out(k.width, k.height, 0.f);
    ParallelFor(size_t(k.height), threads, [&](size_t row) {
        const int v = int(row);
        for (int u = 0; u < k.width; ++u) {
            const V3d dir{(u - k.cx) / k.fx, (v - k.cy) / k.fy, 1.0};
            double prev_z = 0.0, prev_sdf = 0.0;
            bool prev_valid = false;
            for (double z = z_begin; z <= z_end; z += step) {
                const Sample s = vol.SampleSdf(view * (z * dir));
                if (!s.valid) {
                    prev_valid = false;
                    continue;
                }
                if (prev_valid && prev_sdf > 0.0 && s.value <= 0.0) {
                    double lo = prev_z, hi = z, lo_sdf = prev_sdf;
                    for (int it = 0; it < bisections; ++it) {
                        const double mid = 0.5 * (lo + hi);
                        const Sample m = vol.SampleSdf(view * (mid * dir));
                        if (!m.valid) break;
                        if (m.value > 0.0) {
                            lo = mid;
                            lo_sdf = m.value;
                        } else {
                            hi = mid;
                        }
                    }
                    const Sample hs = vol.SampleSdf(view * (hi * dir));
                    double crossing = 0.5 * (lo + hi);
                    if (hs.valid && lo_sdf - hs.value > 1e-12)
                        crossing = lo + (hi - lo) * lo_sdf / (lo_sdf - hs.value);
                    out(u, v) = float(crossing);
                    break;
                }
                prev_z = z;
                prev_sdf = s.value;
                prev_valid = true;
            }
        }
    });
    return out;
}

DepthImage RenderVirtualDepth(const std::vector<WindowEntry>& window, const Pose& view,
                              const Intrinsics& k, const VolumeConfig& vc, const RefinementConfig& rc,
                              int threads) {  // depth_refinement.cpp:22-31
    Volume temp(vc);
    for (const WindowEntry& e : window) {
        const Mask* m = e.mask.Empty() ? nullptr : &e.mask;
        temp.AllocateForFrame(e.frame.depth, e.frame.intr, e.pose, m);
        temp.Integrate(e.frame, e.pose, m, threads);
    }
    return RaycastDepth(temp, view, k, rc.bisection_iterations, threads);
}

DepthImage RefineDepth(const DepthImage& raw, const DepthImage& virt, double far_value) {  // :82-93
    if (raw.w != virt.w || raw.h != virt.h) throw std::invalid_argument("depth size mismatch");
    DepthImage out = raw;
    for (size_t i = 0; i < out.d.size(); ++i) {
        if (DepthValid(out.d[i])) continue;
        out.d[i] = DepthValid(virt.d[i]) ? virt.d[i] : float(far_value);
    }
    return out;
}

// ---------------------------------------------------------------------------
// config.cpp:12-48, pipeline.cpp:25-145
// ---------------------------------------------------------------------------
void PipelineConfig::Sync() {
    mask.truncation = volume.truncation;
    volume.Validate();
    if (!(mask.gamma > 0)) throw std::invalid_argument("gamma must be positive");
    if (!(mask.theta > 0)) throw std::invalid_argument("theta must be positive");
    if (mask.erode_radius < 0 || mask.dilate_radius < 0)
        throw std::invalid_argument("morphology radii must be non-negative");
    if (mask.connectivity != 4 && mask.connectivity != 8)
        throw std::invalid_argument("connectivity must be 4 or 8");
    if (!(registration.color_weight >= 0)) throw std::invalid_argument("color_weight must be non-negative");
    if (registration.pyramid_levels < 1) throw std::invalid_argument("pyramid_levels must be >= 1");
    if (registration.max_iterations < 1) throw std::invalid_argument("max_iterations must be >= 1");
    if (!(registration.lm_lambda_init > 0) || !(registration.lm_lambda_up > 1) ||
        !(registration.lm_lambda_down > 1))
        throw std::invalid_argument("invalid LM damping schedule");
    if (!(registration.convergence_eps > 0)) throw std::invalid_argument("convergence_eps must be positive");
    if (registration.min_valid_residuals < 1) throw std::invalid_argument("min_valid_residuals must be >= 1");
    if (refinement.window < 1) throw std::invalid_argument("refine_window must be >= 1");
    if (!(refinement.far_value > volume.max_depth)) throw std::invalid_argument("far_value must exceed max_depth");
    if (threads < 1) throw std::invalid_argument("threads must be >= 1");
}

Pipeline::Pipeline(PipelineConfig c) : cfg_((c.Sync(), c)), volume_(cfg_.volume) {}

void Pipeline::CarveAndIntegrate(const Frame& f, const Pose& p, const Mask* m) {  // pipeline.cpp:25-29
    volume_.Carve(f.depth, f.intr, p, cfg_.threads);
    volume_.AllocateForFrame(f.depth, f.intr, p, m);
    volume_.Integrate(f, p, m, cfg_.threads);
}

void Pipeline::IntegrateFront() {  // pipeline.cpp:31-55
    const WindowEntry& front = window_.front();
    const DepthImage virt = RenderVirtualDepth(window_, front.pose, front.frame.intr, cfg_.volume,
                                               cfg_.refinement, cfg_.threads);
    const DepthImage refined = RefineDepth(front.frame.depth, virt, cfg_.refinement.far_value);
    WindowEntry e = std::move(window_.front());
    window_.erase(window_.begin());
    pending_.erase(pending_.begin());
    Frame rf = std::move(e.frame);
    rf.depth = refined;
    CarveAndIntegrate(rf, e.pose, e.mask.Empty() ? nullptr : &e.mask);
}

FrameStats Pipeline::ProcessFrame(const Frame& f) {  // pipeline.cpp:57-131
    if (!f.intr.Valid() || f.depth.w != f.intr.width || f.depth.h != f.intr.height ||
        f.color.w != f.depth.w || f.color.h != f.depth.h)
        throw std::invalid_argument("frame images do not match the intrinsics");
    const auto start = std::chrono::steady_clock::now();
    FrameStats st;
    st.frame_index = frame_count_;
    st.timestamp = f.timestamp;
    last_has_mask = false;
    if (first_) {
        const Pose pose;
        volume_.AllocateForFrame(f.depth, f.intr, pose, nullptr);
        volume_.Integrate(f, pose, nullptr, cfg_.threads);
        trajectory_.push_back({f.timestamp, pose});
        current_ = pose;
        first_ = false;
        st.converged = 1;
    } else {
        if (cfg_.refinement.enabled && int(window_.size()) >= cfg_.refinement.window) IntegrateFront();
        Mask mask;
        try {
            RegistrationConfig rc = cfg_.registration;
            rc.residual_sign = cfg_.mask.free_space > 0.0;  // the free-space extension reads the sign
            RegistrationResult reg = Register(volume_, f, current_, nullptr, rc);
            st.registrations = 1;
            st.iterations = reg.iterations;
            if (cfg_.dynamics_enabled) {
                mask = BuildMask(reg.residuals, f.depth, cfg_.mask);
                size_t n = 0;
                for (uint8_t v : mask.d) n += v != 0;
                st.masked_pixels = n;
                if (n > 0) {
                    RegistrationResult r2 = Register(volume_, f, reg.pose, &mask, rc);
                    st.registrations = 2;
                    st.iterations += r2.iterations;
                    reg = std::move(r2);
                }
            }
            st.converged = reg.converged;
            st.valid_residuals = reg.valid_residuals;
            st.final_error = reg.final_error;
            trajectory_.push_back({f.timestamp, reg.pose});
            current_ = reg.pose;
            last_mask = mask;
            last_has_mask = !mask.Empty();
            last_residuals = reg.residuals;
            if (cfg_.refinement.enabled) {
                window_.push_back({f, reg.pose, std::move(mask)});
                pending_.push_back(frame_count_);
            } else {
                CarveAndIntegrate(f, reg.pose, mask.Empty() ? nullptr : &mask);
            }
        } catch (const TrackingLostError&) {
            st.tracking_lost = 1;
            ++losses_;
            trajectory_.push_back({f.timestamp, current_});
        }
    }
    st.runtime_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
    ++frame_count_;
    stats_.push_back(st);
    return st;
}

void Pipeline::Finalize() {  // pipeline.cpp:133-135
    while (!window_.empty()) IntegrateFront();
}

}  // namespace oracle
