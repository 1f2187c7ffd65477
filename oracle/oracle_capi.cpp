// ORACLE — test infrastructure only (see oracle.hpp). Flat C ABI over the
// restatement so pytest (ctypes) can drive it. Pose arrays are 12 doubles:
// row-major rotation then translation, camera-to-world.
#include <fstream>
#include <memory>
#include <cstring>
#include <memory>

#include "oracle.hpp"

using namespace oracle;

extern "C" {

struct OIntr {
    double fx, fy, cx, cy;
    int32_t width, height;
    double depth_scale;
};
struct OVolCfg {
    double voxel_size, truncation;
    int32_t block_side, max_weight, carve_weight, pad0;
    double min_depth, max_depth, carve_clip;
    uint64_t max_blocks;
};
struct ORegCfg {
    double color_weight;
    int32_t pyramid_levels, max_iterations;
    double lm_lambda_init, lm_lambda_up, lm_lambda_down, convergence_eps;
    int32_t min_valid_residuals, threads;
    double huber_depth, huber_color;  // extension (0: the reference)
};
struct OMaskCfg {
    double gamma, truncation, theta;
    int32_t erode_radius, dilate_radius, connectivity, pad0;
    double free_space;  // extension (0: the reference)
};
struct OPipeCfg {
    OVolCfg volume;
    ORegCfg reg;
    OMaskCfg mask;
    int32_t refine_enabled, refine_window;
    double far_value;
    int32_t bisection_iterations, dynamics_enabled, threads, pad0;
};
struct OStats {
    uint64_t frame_index;
    double timestamp;
    int32_t tracking_lost, converged, registrations, iterations;
    uint64_t valid_residuals, masked_pixels;
    double final_error, runtime_ms;
};

enum { O_OK = 0, O_INVALID = 1, O_LOST = 2, O_RESOURCE = 3, O_OTHER = 5 };
}

namespace {
thread_local std::string g_err;

template <typename F>
int Guard(F&& f) {
    try {
        f();
        return O_OK;
    } catch (const TrackingLostError& e) {
        g_err = e.what();
        return O_LOST;
    } catch (const ResourceLimitError& e) {
        g_err = e.what();
        return O_RESOURCE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return O_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return O_OTHER;
    }
}

}  // namespace

extern "C" int o_eval_guard_set(const char* m) {  // error text for oracle_eval.cpp
    g_err = m;
    return 0;
}

namespace {

Intrinsics ToIntr(const OIntr* k) {
    Intrinsics r;
    r.fx = k->fx; r.fy = k->fy; r.cx = k->cx; r.cy = k->cy;
    r.width = k->width; r.height = k->height; r.depth_scale = k->depth_scale;
    return r;
}
VolumeConfig ToVol(const OVolCfg* c) {
    VolumeConfig v;
    v.voxel_size = c->voxel_size; v.truncation = c->truncation; v.block_side = c->block_side;
    v.max_weight = c->max_weight; v.carve_weight = c->carve_weight; v.min_depth = c->min_depth;
    v.max_depth = c->max_depth; v.carve_clip = c->carve_clip; v.max_blocks = c->max_blocks;
    return v;
}
RegistrationConfig ToReg(const ORegCfg* c) {
    RegistrationConfig r;
    r.color_weight = c->color_weight; r.pyramid_levels = c->pyramid_levels;
    r.max_iterations = c->max_iterations; r.lm_lambda_init = c->lm_lambda_init;
    r.lm_lambda_up = c->lm_lambda_up; r.lm_lambda_down = c->lm_lambda_down;
    r.convergence_eps = c->convergence_eps; r.min_valid_residuals = c->min_valid_residuals;
    r.threads = c->threads;
    r.huber_depth = c->huber_depth; r.huber_color = c->huber_color;
    return r;
}
MaskConfig ToMask(const OMaskCfg* c) {
    MaskConfig m;
    m.gamma = c->gamma; m.truncation = c->truncation; m.theta = c->theta;
    m.erode_radius = c->erode_radius; m.dilate_radius = c->dilate_radius; m.connectivity = c->connectivity;
    m.free_space = c->free_space;
    return m;
}
DepthImage ToDepth(const float* d, int w, int h) {
    DepthImage img(w, h);
    std::memcpy(img.d.data(), d, sizeof(float) * size_t(w) * h);
    return img;
}
ColorImage ToColor(const uint8_t* rgb, int w, int h) {
    ColorImage img;
    if (!rgb) return img;
    img = ColorImage(w, h);
    std::memcpy(img.d.data(), rgb, 3 * size_t(w) * h);
    return img;
}
Mask ToMaskImg(const uint8_t* m, int w, int h) {
    Mask img(w, h);
    std::memcpy(img.d.data(), m, size_t(w) * h);
    return img;
}
Frame ToFrame(const float* depth, const uint8_t* rgb, const OIntr* k) {
    Frame f;
    f.intr = ToIntr(k);
    f.depth = ToDepth(depth, k->width, k->height);
    f.color = ToColor(rgb, k->width, k->height);
    return f;
}
void CopyResiduals(const ResidualImage& r, float* sq, uint8_t* valid) {
    if (sq) std::memcpy(sq, r.squared.d.data(), sizeof(float) * r.squared.d.size());
    if (valid) std::memcpy(valid, r.valid.d.data(), r.valid.d.size());
}
}  // namespace

extern "C" {

const char* o_last_error() { return g_err.c_str(); }

// ----------------------------------------------------------------- geometry
void o_expmap(const double xi[6], double pose[12]) { ExpMap(xi).ToArray(pose); }
void o_logmap(const double pose[12], double xi[6]) { LogMap(Pose::FromArray(pose), xi); }
uint64_t o_hash_coord(int32_t x, int32_t y, int32_t z) { return HashCoord({x, y, z}); }

int o_walk_segment(const double a[3], const double b[3], double ext, int32_t* cells, int max_cells) {
    int n = 0;
    WalkGridSegment(V3d{a[0], a[1], a[2]}, V3d{b[0], b[1], b[2]}, ext, [&](const V3i& c) {
        if (n < max_cells) {
            cells[3 * n] = c.x;
            cells[3 * n + 1] = c.y;
            cells[3 * n + 2] = c.z;
        }
        ++n;
    });
    return n;
}

// ----------------------------------------------------------------- hash map
void* oh_create(uint64_t cap) { return new CoordHashMap(cap); }
void oh_destroy(void* h) { delete static_cast<CoordHashMap*>(h); }
uint64_t oh_size(void* h) { return static_cast<CoordHashMap*>(h)->size(); }
uint64_t oh_capacity(void* h) { return static_cast<CoordHashMap*>(h)->capacity(); }
void oh_insert_batch(void* h, uint64_t n, const int32_t* c, const uint32_t* values, uint32_t* out_values,
                     uint8_t* inserted) {
    auto* m = static_cast<CoordHashMap*>(h);
    for (uint64_t i = 0; i < n; ++i) {
        const auto r = m->Insert({c[3 * i], c[3 * i + 1], c[3 * i + 2]}, values[i]);
        out_values[i] = r.first;
        inserted[i] = r.second;
    }
}
void oh_find_batch(void* h, uint64_t n, const int32_t* c, uint32_t* values, uint8_t* found) {
    auto* m = static_cast<CoordHashMap*>(h);
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t* v = m->Find({c[3 * i], c[3 * i + 1], c[3 * i + 2]});
        found[i] = v != nullptr;
        values[i] = v ? *v : 0;
    }
}

// ----------------------------------------------------------------- volume
void* ov_create(const OVolCfg* cfg) {
    Volume* v = nullptr;
    if (Guard([&] { v = new Volume(ToVol(cfg)); }) != O_OK) return nullptr;
    return v;
}
void ov_destroy(void* v) { delete static_cast<Volume*>(v); }
uint64_t ov_num_blocks(void* v) { return static_cast<Volume*>(v)->num_blocks(); }
uint64_t ov_hash_capacity(void* v) { return static_cast<Volume*>(v)->index().capacity(); }
uint64_t ov_last_dda_visits(void* v) { return static_cast<Volume*>(v)->last_dda_visits; }

// 1 new, 0 existed, -3 resource limit
int ov_allocate_block(void* v, int32_t x, int32_t y, int32_t z) {
    int r = 0;
    const int s = Guard([&] { r = static_cast<Volume*>(v)->AllocateBlock({x, y, z}) ? 1 : 0; });
    return s == O_OK ? r : -s;
}

// Blocks in allocation order: coords (3 x i32) and side^3 raw voxels each.
void ov_export(void* vp, int32_t* coords, uint8_t* voxels) {
    const Volume* v = static_cast<Volume*>(vp);
    const size_t n3 = size_t(v->config().block_side) * v->config().block_side * v->config().block_side;
    size_t i = 0;
    for (const VoxelBlock& b : v->blocks()) {
        coords[3 * i] = b.coord.x;
        coords[3 * i + 1] = b.coord.y;
        coords[3 * i + 2] = b.coord.z;
        if (voxels) std::memcpy(voxels + i * n3 * 8, b.voxels.data(), n3 * 8);
        ++i;
    }
}

// Writes voxels through VoxelHandle (the test_util.hpp FillVolume path).
// Returns how many coordinates had no allocated block.
uint64_t ov_set_voxels(void* vp, uint64_t n, const int32_t* c, const uint8_t* vox) {
    Volume* v = static_cast<Volume*>(vp);
    uint64_t missing = 0;
    for (uint64_t i = 0; i < n; ++i) {
        Voxel* h = v->VoxelHandle({c[3 * i], c[3 * i + 1], c[3 * i + 2]});
        if (!h) {
            ++missing;
            continue;
        }
        std::memcpy(h, vox + 8 * i, 8);
    }
    return missing;
}
void ov_get_voxels(void* vp, uint64_t n, const int32_t* c, uint8_t* vox, uint8_t* found) {
    const Volume* v = static_cast<Volume*>(vp);
    for (uint64_t i = 0; i < n; ++i) {
        const Voxel* h = v->VoxelHandle({c[3 * i], c[3 * i + 1], c[3 * i + 2]});
        found[i] = h != nullptr;
        if (h) std::memcpy(vox + 8 * i, h, 8);
        else std::memset(vox + 8 * i, 0, 8);
    }
}

// Occupied-slot bitmap of a linear-probing table of capacity `cap` holding
// the volume's block coordinates (spatial_hash.hpp:35-41 probing rule).
int ov_hash_occupancy(void* vp, uint64_t cap, uint8_t* bitmap) {
    const Volume* v = static_cast<Volume*>(vp);
    if (cap == 0 || (cap & (cap - 1)) || v->num_blocks() > cap) return O_INVALID;
    std::memset(bitmap, 0, cap);
    for (const VoxelBlock& b : v->blocks()) {
        uint64_t idx = HashCoord(b.coord) & (cap - 1);
        while (bitmap[idx]) idx = (idx + 1) & (cap - 1);
        bitmap[idx] = 1;
    }
    return O_OK;
}

int ov_allocate_for_frame(void* v, const float* depth, const OIntr* k, const double pose[12],
                          const uint8_t* mask) {
    return Guard([&] {
        const DepthImage d = ToDepth(depth, k->width, k->height);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        static_cast<Volume*>(v)->AllocateForFrame(d, ToIntr(k), Pose::FromArray(pose), mask ? &m : nullptr);
    });
}
int ov_integrate(void* v, const float* depth, const uint8_t* rgb, const OIntr* k, const double pose[12],
                 const uint8_t* mask, int threads) {
    return Guard([&] {
        const Frame f = ToFrame(depth, rgb, k);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        static_cast<Volume*>(v)->Integrate(f, Pose::FromArray(pose), mask ? &m : nullptr, threads);
    });
}
int ov_carve(void* v, const float* depth, const OIntr* k, const double pose[12], int threads) {
    return Guard([&] {
        static_cast<Volume*>(v)->Carve(ToDepth(depth, k->width, k->height), ToIntr(k),
                                       Pose::FromArray(pose), threads);
    });
}

// mode: 0 SampleSdf, 1 SampleIntensity, 2 SdfWithGradient, 3 IntensityWithGradient,
// 4 SampleSdfGradient (central differences)
void ov_sample(void* vp, int mode, uint64_t n, const double* pts, double* value, double* grad, uint8_t* valid) {
    const Volume* v = static_cast<Volume*>(vp);
    for (uint64_t i = 0; i < n; ++i) {
        const V3d p{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        Sample s;
        switch (mode) {
            case 0: s = v->SampleSdf(p); break;
            case 1: s = v->SampleIntensity(p); break;
            case 2: s = v->SampleSdfWithGradient(p); break;
            case 3: s = v->SampleIntensityWithGradient(p); break;
            default: s = v->SampleSdfGradient(p); break;
        }
        value[i] = s.value;
        if (grad) {
            grad[3 * i] = s.gradient.x;
            grad[3 * i + 1] = s.gradient.y;
            grad[3 * i + 2] = s.gradient.z;
        }
        valid[i] = s.valid;
    }
}

// ----------------------------------------------------------------- registration
// Pyramid levels packed one after another (level l is (w>>l) x (h>>l)).
int o_build_pyramid(const float* depth, const uint8_t* rgb, const uint8_t* mask, const OIntr* k, int levels,
                    float* out_depth, float* out_intensity, uint8_t* out_mask, double* out_intr /*4 per level*/) {
    return Guard([&] {
        const Frame f = ToFrame(depth, rgb, k);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        const auto pyr = BuildPyramid(f, mask ? &m : nullptr, levels);
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            const PyramidLevel& L = pyr[l];
            const size_t n = L.depth.d.size();
            std::memcpy(out_depth + off, L.depth.d.data(), n * 4);
            if (out_intensity && !L.intensity.Empty()) std::memcpy(out_intensity + off, L.intensity.d.data(), n * 4);
            if (out_mask && !L.mask.Empty()) std::memcpy(out_mask + off, L.mask.d.data(), n);
            if (out_intr) {
                out_intr[4 * l] = L.intr.fx;
                out_intr[4 * l + 1] = L.intr.fy;
                out_intr[4 * l + 2] = L.intr.cx;
                out_intr[4 * l + 3] = L.intr.cy;
            }
            off += n;
        }
    });
}

// registration.cpp:184-190
int o_linearize(void* vp, const float* depth, const uint8_t* rgb, const OIntr* k, const double pose[12],
                const ORegCfg* cfg, const uint8_t* mask, double H[36], double b[6], double errs[3],
                uint64_t* valid, int32_t* degenerate) {
    return Guard([&] {
        const Frame f = ToFrame(depth, rgb, k);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        const PyramidLevel level = LevelZero(f, mask ? &m : nullptr);
        const Accum acc = Accumulate(*static_cast<Volume*>(vp), level, Pose::FromArray(pose), cfg->color_weight,
                                     true, true, cfg->threads, nullptr, Robust{cfg->huber_depth, cfg->huber_color, false});
        std::memcpy(H, acc.H, sizeof(acc.H));
        std::memcpy(b, acc.b, sizeof(acc.b));
        errs[0] = acc.depth_error;
        errs[1] = acc.color_error;
        errs[2] = acc.depth_error + cfg->color_weight * acc.color_error;
        *valid = acc.valid;
        *degenerate = Degenerate(acc);
    });
}

// registration.cpp:192-209
int o_evaluate_depth_error(void* vp, const float* depth, const OIntr* k, const double pose[12],
                           const uint8_t* mask, int threads, double* error, float* res_sq, uint8_t* res_valid) {
    return Guard([&] {
        PyramidLevel level;
        level.intr = ToIntr(k);
        level.depth = ToDepth(depth, k->width, k->height);
        if (mask) level.mask = ToMaskImg(mask, k->width, k->height);
        ResidualImage r;
        const Accum acc = Accumulate(*static_cast<Volume*>(vp), level, Pose::FromArray(pose), 0.0, false, true,
                                     threads, &r);
        *error = acc.depth_error;
        CopyResiduals(r, res_sq, res_valid);
    });
}
int o_evaluate_color_error(void* vp, const float* depth, const uint8_t* rgb, const OIntr* k, const double pose[12],
                           const uint8_t* mask, int threads, double* error) {
    return Guard([&] {
        const Frame f = ToFrame(depth, rgb, k);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        const PyramidLevel level = LevelZero(f, mask ? &m : nullptr);
        *error = Accumulate(*static_cast<Volume*>(vp), level, Pose::FromArray(pose), 1.0, false, true, threads,
                            nullptr)
                     .color_error;
    });
}

int o_register(void* vp, const float* depth, const uint8_t* rgb, const OIntr* k, const double init[12],
               const uint8_t* mask, const ORegCfg* cfg, double pose_out[12], int32_t* converged,
               int32_t* iterations, uint64_t* valid, double* final_error, float* res_sq, uint8_t* res_valid) {
    return Guard([&] {
        const Frame f = ToFrame(depth, rgb, k);
        Mask m;
        if (mask) m = ToMaskImg(mask, k->width, k->height);
        const RegistrationResult r =
            Register(*static_cast<Volume*>(vp), f, Pose::FromArray(init), mask ? &m : nullptr, ToReg(cfg));
        r.pose.ToArray(pose_out);
        *converged = r.converged;
        *iterations = r.iterations;
        *valid = r.valid_residuals;
        *final_error = r.final_error;
        CopyResiduals(r.residuals, res_sq, res_valid);
    });
}

int o_ldlt6(const double A[36], const double rhs[6], double x[6]) { return Ldlt6Solve(A, rhs, x) ? 1 : 0; }

// ----------------------------------------------------------------- mask
void o_threshold(const float* sq, const uint8_t* valid, int w, int h, double gamma, double trunc, uint8_t* out) {
    ResidualImage r;
    r.squared = ToDepth(sq, w, h);
    r.valid = ToMaskImg(valid, w, h);
    MaskConfig c;
    c.gamma = gamma;
    c.truncation = trunc;
    const Mask m = ThresholdResiduals(r, c);
    std::memcpy(out, m.d.data(), m.d.size());
}
void o_erode(const uint8_t* in, int w, int h, int radius, uint8_t* out) {
    const Mask m = Erode(ToMaskImg(in, w, h), radius);
    std::memcpy(out, m.d.data(), m.d.size());
}
void o_dilate(const uint8_t* in, int w, int h, int radius, uint8_t* out) {
    const Mask m = Dilate(ToMaskImg(in, w, h), radius);
    std::memcpy(out, m.d.data(), m.d.size());
}
int o_floodfill(const uint8_t* seeds, const float* depth, int w, int h, double theta, int conn, uint8_t* out) {
    return Guard([&] {
        const Mask m = FloodfillDepth(ToMaskImg(seeds, w, h), ToDepth(depth, w, h), theta, conn);
        std::memcpy(out, m.d.data(), m.d.size());
    });
}
int o_build_mask(const float* sq, const uint8_t* valid, const float* depth, int w, int h, const OMaskCfg* cfg,
                 uint8_t* out) {
    return Guard([&] {
        ResidualImage r;
        r.squared = ToDepth(sq, w, h);
        r.valid = ToMaskImg(valid, w, h);
        const Mask m = BuildMask(r, ToDepth(depth, w, h), ToMask(cfg));
        std::memcpy(out, m.d.data(), m.d.size());
    });
}

// ----------------------------------------------------------------- raycast / mesh
int o_raycast(void* vp, const double pose[12], const OIntr* k, int bisections, int threads, float* out) {
    return Guard([&] {
        const DepthImage d = RaycastDepth(*static_cast<Volume*>(vp), Pose::FromArray(pose), ToIntr(k), bisections,
                                          threads);
        std::memcpy(out, d.d.data(), d.d.size() * 4);
    });
}

// RenderVirtualDepth (depth_refinement.cpp:22-80) over a window of n entries;
// masks[i] may be null. RefineDepth (:82-93) into `refined` when non-null.
int o_render_virtual_depth(int n, const float* const* depths, const uint8_t* const* rgbs,
                           const uint8_t* const* masks, const double* poses, const OIntr* k, const OVolCfg* vc,
                           const double view[12], int bisections, double far_value, int threads, float* out,
                           float* refined) {
    return Guard([&] {
        std::vector<WindowEntry> window(n);
        for (int i = 0; i < n; ++i) {
            window[i].frame = ToFrame(depths[i], rgbs ? rgbs[i] : nullptr, k);
            window[i].pose = Pose::FromArray(poses + 12 * i);
            if (masks && masks[i]) window[i].mask = ToMaskImg(masks[i], k->width, k->height);
        }
        RefinementConfig rc;
        rc.bisection_iterations = bisections;
        rc.far_value = far_value;
        const DepthImage v = RenderVirtualDepth(window, Pose::FromArray(view), ToIntr(k), ToVol(vc), rc, threads);
        std::memcpy(out, v.d.data(), sizeof(float) * v.d.size());
        if (refined && n > 0) {
            const DepthImage r = RefineDepth(window[0].frame.depth, v, far_value);
            std::memcpy(refined, r.d.data(), sizeof(float) * r.d.size());
        }
    });
}

void ov_config(void* vp, OVolCfg* o) {
    const VolumeConfig& c = static_cast<Volume*>(vp)->config();
    o->voxel_size = c.voxel_size;
    o->truncation = c.truncation;
    o->block_side = c.block_side;
    o->max_weight = c.max_weight;
    o->carve_weight = c.carve_weight;
    o->min_depth = c.min_depth;
    o->max_depth = c.max_depth;
    o->carve_clip = c.carve_clip;
    o->max_blocks = c.max_blocks;
}
// TsdfVolume::Save (tsdf_volume.cpp:375-403): "TSDFVOL\0", u32 version 1, the
// config, u64 block count, then per block in allocation order i32[3] + voxels.
int ov_save(void* vp, const char* path) {
    return Guard([&] {
        const Volume* v = static_cast<Volume*>(vp);
        const VolumeConfig& c = v->config();
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot open for writing: ") + path);
        auto w = [&](const auto& x) { out.write(reinterpret_cast<const char*>(&x), sizeof(x)); };
        out.write("TSDFVOL\0", 8);
        w(uint32_t(1));
        w(c.voxel_size);
        w(c.truncation);
        w(int32_t(c.block_side));
        w(int32_t(c.max_weight));
        w(int32_t(c.carve_weight));
        w(c.min_depth);
        w(c.max_depth);
        w(c.carve_clip);
        w(uint64_t(c.max_blocks));
        w(uint64_t(v->blocks().size()));
        for (const VoxelBlock& b : v->blocks()) {
            const int32_t cc[3] = {b.coord.x, b.coord.y, b.coord.z};
            out.write(reinterpret_cast<const char*>(cc), sizeof(cc));
            out.write(reinterpret_cast<const char*>(b.voxels.data()), std::streamsize(b.voxels.size() * sizeof(Voxel)));
        }
        if (!out) throw std::runtime_error(std::string("write failed: ") + path);
    });
}
// TsdfVolume::Load (tsdf_volume.cpp:405-449): AllocateBlock in file order.
void* ov_load(const char* path) {
    Volume* vol = nullptr;
    const int s = Guard([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot open volume snapshot: ") + path);
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, "TSDFVOL\0", 8) != 0) throw std::runtime_error("not a volume snapshot");
        auto r = [&](auto& x) { in.read(reinterpret_cast<char*>(&x), sizeof(x)); };
        uint32_t version = 0;
        r(version);
        if (version != 1) throw std::runtime_error("unsupported volume snapshot version");
        VolumeConfig c;
        int32_t bs = 0, mw = 0, cw = 0;
        uint64_t mb = 0, nb = 0;
        r(c.voxel_size);
        r(c.truncation);
        r(bs);
        r(mw);
        r(cw);
        r(c.min_depth);
        r(c.max_depth);
        r(c.carve_clip);
        r(mb);
        r(nb);
        if (!in) throw std::runtime_error("truncated volume snapshot");
        c.block_side = bs;
        c.max_weight = mw;
        c.carve_weight = cw;
        c.max_blocks = mb;
        auto v = std::make_unique<Volume>(c);
        for (uint64_t i = 0; i < nb; ++i) {
            int32_t cc[3];
            in.read(reinterpret_cast<char*>(cc), sizeof(cc));
            v->AllocateBlock(V3i{cc[0], cc[1], cc[2]});
            VoxelBlock& b = v->blocks_mut().back();
            in.read(reinterpret_cast<char*>(b.voxels.data()), std::streamsize(b.voxels.size() * sizeof(Voxel)));
            if (!in) throw std::runtime_error("truncated volume snapshot");
        }
        vol = v.release();
    });
    return s == O_OK ? vol : nullptr;
}

// WritePly (mesh.cpp:192-225): ASCII header, binary little-endian body; the
// colour properties only when the mesh has colours.
int o_mesh_write_ply(void* mp, const char* path) {
    return Guard([&] {
        const Mesh* m = static_cast<Mesh*>(mp);
        const size_t nv = m->vertices.size() / 3, nf = m->faces.size() / 3;
        const bool colored = !m->colors.empty();
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot open for writing: ") + path);
        out << "ply\nformat binary_little_endian 1.0\n";
        out << "element vertex " << nv << "\n";
        out << "property float x\nproperty float y\nproperty float z\n";
        if (colored) out << "property uchar red\nproperty uchar green\nproperty uchar blue\n";
        out << "element face " << nf << "\n";
        out << "property list uchar int vertex_indices\n";
        out << "end_header\n";
        for (size_t i = 0; i < nv; ++i) {
            out.write(reinterpret_cast<const char*>(&m->vertices[3 * i]), 12);
            if (colored) out.write(reinterpret_cast<const char*>(&m->colors[3 * i]), 3);
        }
        for (size_t i = 0; i < nf; ++i) {
            const uint8_t three = 3;
            out.write(reinterpret_cast<const char*>(&three), 1);
            out.write(reinterpret_cast<const char*>(&m->faces[3 * i]), 12);
        }
        if (!out) throw std::runtime_error(std::string("write failed: ") + path);
    });
}

void* o_mesh_extract(void* vp, int min_weight, int threads) {
    return new Mesh(ExtractMesh(*static_cast<Volume*>(vp), min_weight, threads));
}
void o_mesh_counts(void* m, uint64_t* nv, uint64_t* nf) {
    *nv = static_cast<Mesh*>(m)->vertices.size() / 3;
    *nf = static_cast<Mesh*>(m)->faces.size() / 3;
}
void o_mesh_copy(void* mp, float* v, uint8_t* c, int32_t* f) {
    const Mesh* m = static_cast<Mesh*>(mp);
    std::memcpy(v, m->vertices.data(), m->vertices.size() * 4);
    std::memcpy(c, m->colors.data(), m->colors.size());
    std::memcpy(f, m->faces.data(), m->faces.size() * 4);
}
void o_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

// ----------------------------------------------------------------- synth
void* o_scene_parse(const char* text) {
    Scene* s = nullptr;
    if (Guard([&] { s = new Scene(Scene::Parse(text)); }) != O_OK) return nullptr;
    return s;
}
void o_scene_free(void* s) { delete static_cast<Scene*>(s); }
uint64_t o_scene_num_frames(void* s) { return static_cast<Scene*>(s)->camera.size(); }
void o_scene_intrinsics(void* s, OIntr* k) {
    const Intrinsics& i = static_cast<Scene*>(s)->intr;
    k->fx = i.fx; k->fy = i.fy; k->cx = i.cx; k->cy = i.cy;
    k->width = i.width; k->height = i.height; k->depth_scale = i.depth_scale;
}
void o_scene_camera(void* s, uint64_t i, double* t, double pose[12]) {
    const auto& c = static_cast<Scene*>(s)->camera[i];
    *t = c.first;
    c.second.ToArray(pose);
}
// World-to-object pose of primitive i at time t (RenderFrame's views, synth.cpp:155-158).
uint64_t o_scene_num_prims(void* s) { return static_cast<Scene*>(s)->prims.size(); }
void o_scene_w2o(void* s, uint64_t i, double t, double pose[12]) {
    static_cast<Scene*>(s)->prims[i].PoseAt(t).Inverse().ToArray(pose);
}
int o_render(void* sp, uint64_t i, float* depth, uint8_t* rgb, float* true_depth, uint8_t* labels) {
    return Guard([&] {
        const Rendered r = RenderFrame(*static_cast<Scene*>(sp), i);
        std::memcpy(depth, r.frame.depth.d.data(), r.frame.depth.d.size() * 4);
        if (rgb) std::memcpy(rgb, r.frame.color.d.data(), r.frame.color.d.size() * 3);
        if (true_depth) std::memcpy(true_depth, r.true_depth.d.data(), r.true_depth.d.size() * 4);
        if (labels) std::memcpy(labels, r.labels.d.data(), r.labels.d.size());
    });
}

// ----------------------------------------------------------------- pipeline
void* op_create(const OPipeCfg* c) {
    Pipeline* p = nullptr;
    const int s = Guard([&] {
        PipelineConfig pc;
        pc.volume = ToVol(&c->volume);
        pc.registration = ToReg(&c->reg);
        pc.mask = ToMask(&c->mask);
        pc.refinement.enabled = c->refine_enabled != 0;
        pc.refinement.window = c->refine_window;
        pc.refinement.far_value = c->far_value;
        pc.refinement.bisection_iterations = c->bisection_iterations;
        pc.dynamics_enabled = c->dynamics_enabled != 0;
        pc.threads = c->threads;
        p = new Pipeline(pc);
    });
    return s == O_OK ? p : nullptr;
}
void op_destroy(void* p) { delete static_cast<Pipeline*>(p); }
int op_process(void* pp, double timestamp, const float* depth, const uint8_t* rgb, const OIntr* k, OStats* out,
               double pose_out[12]) {
    return Guard([&] {
        Pipeline* p = static_cast<Pipeline*>(pp);
        Frame f = ToFrame(depth, rgb, k);
        f.timestamp = timestamp;
        const FrameStats s = p->ProcessFrame(f);
        out->frame_index = s.frame_index;
        out->timestamp = s.timestamp;
        out->tracking_lost = s.tracking_lost;
        out->converged = s.converged;
        out->registrations = s.registrations;
        out->iterations = s.iterations;
        out->valid_residuals = s.valid_residuals;
        out->masked_pixels = s.masked_pixels;
        out->final_error = s.final_error;
        out->runtime_ms = s.runtime_ms;
        p->trajectory().back().second.ToArray(pose_out);
    });
}
int op_finalize(void* p) {
    return Guard([&] { static_cast<Pipeline*>(p)->Finalize(); });
}
void* op_volume(void* p) { return &static_cast<Pipeline*>(p)->volume(); }
uint64_t op_losses(void* p) { return static_cast<Pipeline*>(p)->losses(); }
int op_last_mask(void* pp, uint8_t* out) {
    Pipeline* p = static_cast<Pipeline*>(pp);
    if (!p->last_has_mask) return 0;
    std::memcpy(out, p->last_mask.d.data(), p->last_mask.d.size());
    return 1;
}
void op_last_residuals(void* pp, float* sq, uint8_t* valid) {
    CopyResiduals(static_cast<Pipeline*>(pp)->last_residuals, sq, valid);
}

}  // extern "C"
