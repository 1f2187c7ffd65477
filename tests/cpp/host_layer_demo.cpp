// Drives the C++ host layer (include/refusion_b200.hpp) the way a caller of
// the reference's tsdfslam::Pipeline would (proj/tools/main.cpp:90-141):
// frames in, trajectory + mesh out. Used by tests/test_cpp_host.py.
//
//   host_layer_demo <in.bin> <out.bin> [refine|nodebug]
// in.bin : i32 W, H, N; f64 fx, fy, cx, cy; then N x (f64 t, f32 depth[W*H], u8 rgb[W*H*3])
// out.bin: i32 N; N x (f64 t, f64 pose[12], i32 lost, i32 regs, i32 iters, u64 masked);
//          u64 nv, nf, nblocks; then error-behaviour flags (i32 x 3)
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>

#include "refusion_b200.hpp"

namespace ts = tsdfslam_b200;

int main(int argc, char** argv) {
    if (argc != 3 && argc != 4) {
        std::cerr << "usage: host_layer_demo in.bin out.bin [refine|nodebug]\n";
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    int32_t w, h, n;
    double k4[4];
    in.read(reinterpret_cast<char*>(&w), 4).read(reinterpret_cast<char*>(&h), 4).read(reinterpret_cast<char*>(&n), 4);
    in.read(reinterpret_cast<char*>(k4), 32);
    ts::CameraIntrinsics k;
    k.fx = k4[0];
    k.fy = k4[1];
    k.cx = k4[2];
    k.cy = k4[3];
    k.width = w;
    k.height = h;

    ts::PipelineConfig cfg;
    const std::string opt = argc == 4 ? argv[3] : "";
    cfg.refinement.enabled = opt == "refine";  // default-on in the reference; TrackingConfig turns it off (acceptance.cpp:136)
    cfg.refinement.window = 3;
    ts::Pipeline pipe(cfg);
    std::size_t debug_calls = 0, debug_masks = 0, debug_refined = 0;
    if (opt != "nodebug")  // without a sink RunSequence submits frames in batches (ProcessFrames)
        pipe.set_debug_sink([&](const ts::FrameDebug& d) {
            ++debug_calls;
            if (d.mask) debug_masks += ts::CountMasked(*d.mask) > 0;
            if (d.refined_depth && d.virtual_depth) ++debug_refined;
        });
    int frames_read = 0;
    ts::FrameSource src = [&]() -> std::optional<ts::Frame> {
        if (frames_read == n) return std::nullopt;
        ts::Frame f;
        f.intrinsics = k;
        f.depth = ts::DepthImage(w, h);
        f.color = ts::ColorImage(w, h);
        in.read(reinterpret_cast<char*>(&f.timestamp), 8);
        in.read(reinterpret_cast<char*>(f.depth.data()), std::streamsize(4) * w * h);
        in.read(reinterpret_cast<char*>(f.color.data()), std::streamsize(3) * w * h);
        ++frames_read;
        return f;
    };
    const ts::SequenceSummary sum = ts::RunSequence(pipe, src);

    std::ofstream out(argv[2], std::ios::binary);
    const int32_t nf = int32_t(sum.frames);
    out.write(reinterpret_cast<const char*>(&nf), 4);
    for (std::size_t i = 0; i < sum.frames; ++i) {
        const ts::TrajectoryEntry& e = pipe.trajectory()[i];
        const ts::FrameStats& s = pipe.stats()[i];
        out.write(reinterpret_cast<const char*>(&e.timestamp), 8);
        out.write(reinterpret_cast<const char*>(e.pose.data()), 96);
        const int32_t v[3] = {s.tracking_lost, s.registrations, s.iterations};
        out.write(reinterpret_cast<const char*>(v), 12);
        const uint64_t m = s.masked_pixels;
        out.write(reinterpret_cast<const char*>(&m), 8);
    }
    const ts::Mesh mesh = ts::ExtractMesh(pipe.volume());
    const uint64_t counts[3] = {mesh.vertices.size(), mesh.faces.size(), pipe.volume().num_blocks()};
    out.write(reinterpret_cast<const char*>(counts), 24);

    // Error behaviour mirrors the reference's exceptions (errors.hpp).
    int32_t flags[3] = {0, 0, 0};
    try {
        ts::VolumeConfig bad;
        bad.voxel_size = -1;
        ts::TsdfVolume v(bad);
    } catch (const std::invalid_argument&) {
        flags[0] = 1;
    }
    try {
        ts::VolumeConfig tiny;
        tiny.max_blocks = 2;
        ts::TsdfVolume v(tiny);
        ts::DepthImage d(w, h, 1.0f);
        v.AllocateForFrame(d, k, ts::Pose::Identity());
    } catch (const ts::ResourceLimitError&) {
        flags[1] = 1;
    }
    try {
        ts::TsdfVolume v(ts::VolumeConfig{});
        ts::Frame f;
        f.intrinsics = k;
        f.depth = ts::DepthImage(w, h, 0.0f);  // nothing valid
        ts::Register(v, f, ts::Pose::Identity(), nullptr, ts::RegistrationConfig{});
    } catch (const ts::TrackingLostError&) {
        flags[2] = 1;
    }
    out.write(reinterpret_cast<const char*>(flags), 12);
    const uint64_t dbg[3] = {debug_calls, debug_masks, debug_refined};
    out.write(reinterpret_cast<const char*>(dbg), 24);
    std::printf("frames %zu losses %zu debug %zu/%zu/%zu vertices %zu faces %zu\n", sum.frames, sum.tracking_losses,
                debug_calls, debug_masks, debug_refined, mesh.vertices.size(), mesh.faces.size());
    return 0;
}
