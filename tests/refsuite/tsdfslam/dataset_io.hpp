// Reference-suite compat header (tests only): the declarations of the
// reference's dataset_io.hpp that its acceptance program names for its
// optional TUM-sequence criterion. Dataset I/O is out of scope:
// these throw, and the criterion skips before calling them unless
// TUM_DATA_DIR is set.
#pragma once
#include <stdexcept>
#include <string>
#include <vector>

#include "refusion_b200.hpp"

namespace tsdfslam {
using namespace tsdfslam_b200;

struct AssociatedFrame {
    double timestamp = 0.0;
    std::string rgb_path, depth_path, label_path;
};
struct SequenceManifest {
    std::string root;
    CameraIntrinsics intrinsics;
    std::vector<AssociatedFrame> frames;
};
inline SequenceManifest LoadSequenceDir(const std::string&, double = 0.02) {
    throw std::runtime_error("dataset I/O is out of scope for the B200 path");
}
inline Frame LoadFrame(const SequenceManifest&, std::size_t) {
    throw std::runtime_error("dataset I/O is out of scope for the B200 path");
}
inline Trajectory ReadTrajectory(const std::string&) {
    throw std::runtime_error("dataset I/O is out of scope for the B200 path");
}
}  // namespace tsdfslam
