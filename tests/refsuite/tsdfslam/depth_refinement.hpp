// Reference-suite compat header (tests only): the reference's depth_refinement.hpp
// resolved to the B200 host layer, so the reference's own test sources
// compile unchanged against the GPU implementation.
#pragma once
#include "refusion_b200.hpp"
namespace tsdfslam {
using namespace tsdfslam_b200;
}  // namespace tsdfslam
