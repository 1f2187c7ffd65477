// ORACLE — test infrastructure only. A flat C ABI over the REFERENCE itself:
// the unmodified tsdfslam sources (/root/reference/proj/src) compiled against
// the Eigen / doctest / libpng stand-ins in oracle/ref_shim (oracle/Makefile
// target `ref`, output oracle/_ref/libtsdfslam_ref.so). Used to pin the oracle
// restatement to the reference code (tests/test_reference_build.py) and as
// bench.py's reference arm / cpu_baseline ("kind": "reference"). The structs
// match oracle_capi.cpp's (the same ctypes mirrors drive both).
#include <cstdint>
#include <cstring>
#include <string>

#include "tsdfslam/config.hpp"
#include "tsdfslam/errors.hpp"
#include "tsdfslam/mesh.hpp"
#include "tsdfslam/pipeline.hpp"
#include "tsdfslam/synth.hpp"
#include "tsdfslam/tsdf_volume.hpp"

using namespace tsdfslam;

extern "C" {
struct RIntr {
    double fx, fy, cx, cy;
    int32_t width, height;
    double depth_scale;
};
struct RVolCfg {
    double voxel_size, truncation;
    int32_t block_side, max_weight, carve_weight, pad0;
    double min_depth, max_depth, carve_clip;
    uint64_t max_blocks;
};
struct RRegCfg {
    double color_weight;
    int32_t pyramid_levels, max_iterations;
    double lm_lambda_init, lm_lambda_up, lm_lambda_down, convergence_eps;
    int32_t min_valid_residuals, threads;
    double huber_depth, huber_color;  // the oracle's extension knobs: layout only, the reference has none
};
struct RMaskCfg {
    double gamma, truncation, theta;
    int32_t erode_radius, dilate_radius, connectivity, pad0;
    double free_space;  // (layout only, as above)
};
struct RPipeCfg {
    RVolCfg volume;
    RRegCfg reg;
    RMaskCfg mask;
    int32_t refine_enabled, refine_window;
    double far_value;
    int32_t bisection_iterations, dynamics_enabled, threads, pad0;
};
struct RStats {
    uint64_t frame_index;
    double timestamp;
    int32_t tracking_lost, converged, registrations, iterations;
    uint64_t valid_residuals, masked_pixels;
    double final_error, runtime_ms;
};
enum { R_OK = 0, R_INVALID = 1, R_LOST = 2, R_RESOURCE = 3, R_OTHER = 5 };
}

namespace {
thread_local std::string g_err;
template <typename F>
int Guard(F&& f) {
    try {
        f();
        return R_OK;
    } catch (const ResourceLimitError& e) {
        g_err = e.what();
        return R_RESOURCE;
    } catch (const TrackingLostError& e) {
        g_err = e.what();
        return R_LOST;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return R_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return R_OTHER;
    }
}
PipelineConfig ToConfig(const RPipeCfg* c) {
    PipelineConfig pc;
    VolumeConfig& v = pc.volume;
    v.voxel_size = c->volume.voxel_size;
    v.truncation = c->volume.truncation;
    v.block_side = c->volume.block_side;
    v.max_weight = c->volume.max_weight;
    v.carve_weight = c->volume.carve_weight;
    v.min_depth = c->volume.min_depth;
    v.max_depth = c->volume.max_depth;
    v.carve_clip = c->volume.carve_clip;
    v.max_blocks = static_cast<std::size_t>(c->volume.max_blocks);
    RegistrationConfig& r = pc.registration;
    r.color_weight = c->reg.color_weight;
    r.pyramid_levels = c->reg.pyramid_levels;
    r.max_iterations = c->reg.max_iterations;
    r.lm_lambda_init = c->reg.lm_lambda_init;
    r.lm_lambda_up = c->reg.lm_lambda_up;
    r.lm_lambda_down = c->reg.lm_lambda_down;
    r.convergence_eps = c->reg.convergence_eps;
    r.min_valid_residuals = c->reg.min_valid_residuals;
    r.threads = c->reg.threads;
    MaskConfig& m = pc.mask;
    m.gamma = c->mask.gamma;
    m.theta = c->mask.theta;
    m.erode_radius = c->mask.erode_radius;
    m.dilate_radius = c->mask.dilate_radius;
    m.connectivity = c->mask.connectivity;
    pc.refinement.enabled = c->refine_enabled != 0;
    pc.refinement.window = c->refine_window;
    pc.refinement.far_value = c->far_value;
    pc.refinement.bisection_iterations = c->bisection_iterations;
    pc.dynamics_enabled = c->dynamics_enabled != 0;
    pc.threads = c->threads;
    pc.Sync();  // the mask threshold follows the volume truncation (config.cpp)
    return pc;
}
void ToArray(const Pose& p, double out[12]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) out[3 * i + j] = p.rotation()(i, j);
    for (int i = 0; i < 3; ++i) out[9 + i] = p.translation()(i);
}
}  // namespace

extern "C" {
const char* r_last_error() { return g_err.c_str(); }

// ---- SceneScript / RenderFrame (synth.cpp)
void* r_scene_parse(const char* text) {
    SceneScript* s = nullptr;
    if (Guard([&] { s = new SceneScript(SceneScript::Parse(text)); }) != R_OK) return nullptr;
    return s;
}
void r_scene_free(void* s) { delete static_cast<SceneScript*>(s); }
uint64_t r_scene_num_frames(void* s) { return static_cast<SceneScript*>(s)->camera.size(); }
void r_scene_intrinsics(void* s, RIntr* k) {
    const CameraIntrinsics& i = static_cast<SceneScript*>(s)->intrinsics;
    *k = RIntr{i.fx, i.fy, i.cx, i.cy, i.width, i.height, i.depth_scale};
}
int r_render(void* sp, uint64_t i, float* depth, uint8_t* rgb, float* true_depth, uint8_t* labels) {
    return Guard([&] {
        const RenderedFrame r = RenderFrame(*static_cast<SceneScript*>(sp), i);
        const std::size_t n = r.frame.depth.PixelCount();
        std::memcpy(depth, r.frame.depth.data(), n * 4);
        if (rgb) std::memcpy(rgb, r.frame.color.data(), n * 3);
        if (true_depth) std::memcpy(true_depth, r.true_depth.data(), n * 4);
        if (labels) std::memcpy(labels, r.dynamic_labels.data(), n);
    });
}

// ---- Pipeline (pipeline.hpp)
void* r_pipe_create(const RPipeCfg* c) {
    Pipeline* p = nullptr;
    if (Guard([&] { p = new Pipeline(ToConfig(c)); }) != R_OK) return nullptr;
    return p;
}
void r_pipe_destroy(void* p) { delete static_cast<Pipeline*>(p); }
int r_pipe_process(void* pp, double timestamp, const float* depth, const uint8_t* rgb, const RIntr* k, RStats* out,
                   double pose_out[12]) {
    return Guard([&] {
        Pipeline* p = static_cast<Pipeline*>(pp);
        Frame f;
        f.timestamp = timestamp;
        f.intrinsics.fx = k->fx;
        f.intrinsics.fy = k->fy;
        f.intrinsics.cx = k->cx;
        f.intrinsics.cy = k->cy;
        f.intrinsics.width = k->width;
        f.intrinsics.height = k->height;
        f.intrinsics.depth_scale = k->depth_scale;
        f.depth = DepthImage(k->width, k->height, 0.f);
        std::memcpy(f.depth.data(), depth, f.depth.PixelCount() * 4);
        f.color = ColorImage(k->width, k->height, Rgb8{0, 0, 0});
        if (rgb) std::memcpy(static_cast<void*>(f.color.data()), rgb, f.color.PixelCount() * 3);
        const FrameStats s = p->ProcessFrame(f);
        *out = RStats{s.frame_index, s.timestamp, s.tracking_lost ? 1 : 0, s.converged ? 1 : 0, s.registrations,
                      s.iterations, s.valid_residuals, s.masked_pixels, s.final_error, s.runtime_ms};
        ToArray(p->trajectory().back().pose, pose_out);
    });
}
int r_pipe_finalize(void* p) {
    return Guard([&] { static_cast<Pipeline*>(p)->Finalize(); });
}
uint64_t r_pipe_num_blocks(void* p) { return static_cast<Pipeline*>(p)->volume().num_blocks(); }
// blocks() in allocation order: coords (3 i32 each) and voxels (512 x 8 B each)
void r_pipe_export(void* pp, int32_t* coords, uint8_t* voxels) {
    const TsdfVolume& v = static_cast<Pipeline*>(pp)->volume();
    std::size_t i = 0;
    for (const VoxelBlock& b : v.blocks()) {
        coords[3 * i] = b.coord.x();
        coords[3 * i + 1] = b.coord.y();
        coords[3 * i + 2] = b.coord.z();
        if (voxels) std::memcpy(voxels + i * b.voxels.size() * 8, b.voxels.data(), b.voxels.size() * 8);
        ++i;
    }
}
int r_pipe_save(void* p, const char* path) {
    return Guard([&] { static_cast<Pipeline*>(p)->volume().Save(path); });
}
int r_pipe_write_ply(void* p, const char* path, int min_weight) {
    return Guard([&] { WritePly(path, ExtractMesh(static_cast<Pipeline*>(p)->volume(), min_weight, 1)); });
}
}
