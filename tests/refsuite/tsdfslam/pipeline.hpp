// Reference-suite compat header (tests only): the reference's pipeline.hpp
// resolved to the B200 host layer, so the reference's own test sources
// compile unchanged against the GPU implementation.
#pragma once
#include "refusion_b200.hpp"
#include "tsdfslam/dataset_io.hpp"  // as the reference pipeline.hpp does
namespace tsdfslam {
using namespace tsdfslam_b200;
}  // namespace tsdfslam
