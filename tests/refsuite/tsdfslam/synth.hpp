// Reference-suite compat header (tests only): the reference's synth.hpp
// (SceneScript / RenderFrame, the test-scene generator its suites render
// their inputs with) over the oracle's restatement of RenderFrame (liboracle,
// bit-identical to the reference build), so the suites get the same input
// bytes; everything they then test runs on the B200 host layer.
#pragma once
#include <cstdint>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "refusion_b200.hpp"

extern "C" {
struct OIntrCompat {
    double fx, fy, cx, cy;
    int32_t width, height;
    double depth_scale;
};
void* o_scene_parse(const char* text);
void o_scene_free(void* s);
uint64_t o_scene_num_frames(void* s);
void o_scene_intrinsics(void* s, OIntrCompat* k);
void o_scene_camera(void* s, uint64_t i, double* t, double pose[12]);
int o_render(void* s, uint64_t i, float* depth, uint8_t* rgb, float* true_depth, uint8_t* labels);
const char* o_last_error();
}

namespace tsdfslam {
using namespace tsdfslam_b200;

struct SceneScript {
    CameraIntrinsics intrinsics;
    double noise_sigma_scale = 0.0;
    double dropout = 0.0;
    std::uint32_t seed = 0;
    std::vector<std::pair<double, Pose>> camera;  // camera-to-world
    std::string source;                           // the script, rendered by the oracle

    static SceneScript Parse(const std::string& text) {
        void* h = o_scene_parse(text.c_str());
        if (!h) throw std::invalid_argument(std::string("scene script: ") + o_last_error());
        SceneScript s;
        s.source = text;
        OIntrCompat k{};
        o_scene_intrinsics(h, &k);
        s.intrinsics.fx = k.fx;
        s.intrinsics.fy = k.fy;
        s.intrinsics.cx = k.cx;
        s.intrinsics.cy = k.cy;
        s.intrinsics.width = k.width;
        s.intrinsics.height = k.height;
        s.intrinsics.depth_scale = k.depth_scale;
        for (uint64_t i = 0; i < o_scene_num_frames(h); ++i) {
            double t = 0.0, p[12];
            o_scene_camera(h, i, &t, p);
            s.camera.emplace_back(t, Pose::FromArray(p));
        }
        o_scene_free(h);
        return s;
    }
    static SceneScript ParseFile(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw std::runtime_error("cannot open " + path);
        std::stringstream ss;
        ss << in.rdbuf();
        return Parse(ss.str());
    }
};

struct RenderedFrame {
    Frame frame;
    DepthImage true_depth;
    PixelMask dynamic_labels;
};

inline RenderedFrame RenderFrame(const SceneScript& scene, std::size_t frame_index) {
    void* h = o_scene_parse(scene.source.c_str());
    if (!h) throw std::invalid_argument(std::string("scene script: ") + o_last_error());
    if (frame_index >= o_scene_num_frames(h)) {
        o_scene_free(h);
        throw std::out_of_range("frame index beyond the camera path");
    }
    const CameraIntrinsics& k = scene.intrinsics;
    RenderedFrame r;
    r.frame.intrinsics = k;
    r.frame.timestamp = scene.camera[frame_index].first;
    r.frame.depth = DepthImage(k.width, k.height, 0.f);
    r.frame.color = ColorImage(k.width, k.height, Rgb8{});
    r.true_depth = DepthImage(k.width, k.height, 0.f);
    r.dynamic_labels = PixelMask(k.width, k.height, 0);
    const int rc = o_render(h, frame_index, r.frame.depth.data(), reinterpret_cast<uint8_t*>(r.frame.color.data()),
                            r.true_depth.data(), r.dynamic_labels.data());
    o_scene_free(h);
    if (rc != 0) throw std::runtime_error(std::string("RenderFrame: ") + o_last_error());
    return r;
}

}  // namespace tsdfslam
