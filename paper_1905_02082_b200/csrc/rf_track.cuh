// Direct SDF + colour tracking (registration.cpp) and the dynamics mask
// (dynamics_mask.cpp) as device phases of one persistent cooperative kernel.
#pragma once

#include "rf_grid.cuh"

namespace rfb {

constexpr int kMaxLevels = 6;
constexpr int kTrackThreads = kGridThreads;  // 12 warps at <= 168 registers (tools/pass_bench.py: 16.6 vs 19.9 us per L0 pass at 256)
constexpr int kTrackMinBlocks = 1;  // one CTA per SM: 148 grid partials
// Per-thread cache of the Jacobian passes' pixel inputs {depth, intensity}:
// one 8-byte entry per pixel step (a thread meets the same pixels in every
// pass of a level), in dynamic shared memory sized per launch from the frame
// (TrackArgs::pxc_steps): 6 steps at 640x480, 17 at 1280x720. The floodfill's
// tile flags reuse the same bytes after the registrations.
constexpr size_t kTrackMaxDynSmem = 96 * 1024;

struct RegParams {  // RegistrationConfig, registration.hpp:13-23
    double color_weight;
    int levels, max_iterations;
    double lambda_init, lambda_up, lambda_down, eps;
    int min_valid;
    double huber_d, huber_c;  // Huber extension (0: off, the reference's least squares)
};

struct MaskParams {  // MaskConfig, dynamics_mask.hpp:10-17
    double gamma, truncation, theta;
    int erode_radius, dilate_radius, connectivity;
    double free_space;  // free-space seed extension (0: off)
};

// Device images of one frame and its pyramid. Level 0 depth/rgb are the
// inputs; coarser levels are built in-kernel.
struct FrameView {
    const float* depth0;
    const uint8_t* rgb0;      // may be null (no colour)
    float* depth[kMaxLevels]; // [0] unused
    float* inten[kMaxLevels]; // [0] unused (computed from rgb0 on the fly)
    uint8_t* mask[kMaxLevels];// [0] = mask used by masked registration
    Intr K[kMaxLevels];
    float* res_sq;            // full-resolution residual image
    uint8_t* res_valid;
    uint8_t* mwork[3];        // mask build scratch
    int* ffstamp;             // floodfill per-tile round stamps (32x32 tiles)
    uint8_t* grow;            // floodfill growth-edge bits per pixel
};

struct TrackOut {
    double pose[12];
    int32_t lost, converged, registrations, iterations;
    unsigned long long valid, masked;
    double final_error;
    double acc[kAccN];  // last accumulation (linearize/evaluate entry points)
    int32_t rounds;     // floodfill rounds (diagnostic)
    int32_t passes;     // pixel passes run (Accumulate calls)
    double pixel_passes;  // sum over passes of the level's pixel count (bytes model)
};

constexpr int kTracePasses = 256;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

enum TrackMode : int {
    kModeFrame = 0,      // pyramid, register, mask, register under mask (pipeline.cpp:81-99)
    kModeRegister = 1,   // pyramid + one Register with optional mask
    kModeLinearize = 2,  // one Jacobian pass at level 0 (Linearize)
    kModeEvalDepth = 3,  // value pass at level 0 writing residuals (EvaluateDepthError)
    kModeEvalColor = 4,  // value pass at level 0, colour error (EvaluateColorError)
    kModeMask = 5,       // BuildMask stages on given residuals
    kModePassBench = 6,  // diagnostics: bench_iters Jacobian passes at bench_level (timeline in out)
    kModePyramid = 7,    // BuildPyramid only (level-0 intensity included), for rf_build_pyramid
};

struct TrackArgs {
    int mode;
    int use_mask;        // kModeRegister/Linearize/Eval: mask[0] is valid
    int dynamics;        // kModeFrame: build mask + second registration
    int mask_stages;     // kModeMask: bit0 threshold, bit1 erode, bit2 floodfill, bit3 dilate
    VolumeView V;
    FrameView F;
    RegParams reg;
    MaskParams mp;
    GridCtx grid;
    unsigned long long* trace;  // optional per-pass timeline (RF_TRACE_FILE), kTracePasses x 8
    double* pose_state;  // in: initial pose; out: tracked pose (kModeFrame/Register)
    TrackOut* out;
    uint32_t* vol_counters;  // kModeFrame: snapshot kNumBlocks -> kBlocksBefore
    int bench_iters, bench_level;  // kModePassBench
    int pxc_steps;       // pixel-cache entries per thread (dynamic shared memory)
    int dyn_bytes;       // dynamic shared memory of this launch
};

}  // namespace rfb
