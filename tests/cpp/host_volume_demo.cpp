// The reference's voxel-access idioms through the C++ host layer
// (include/refusion_b200.hpp), as proj/tests/test_tsdf.cpp and test_util.hpp
// use them: AllocateBlock, a mutable VoxelHandle written in place, FindBlock,
// SampleSdf reading the written values, BuildPyramid. Prints one line per
// check; exit code 0 when all hold. Used by tests/test_gpu_boundary.py.
#include <cmath>
#include <cstdio>

#include "refusion_b200.hpp"

namespace ts = tsdfslam_b200;

static int failures = 0;
static void check(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "ok" : "FAIL", what);
    failures += ok ? 0 : 1;
}

int main() {
    ts::VolumeConfig vc;
    vc.voxel_size = 0.02;
    vc.max_blocks = 64;
    ts::TsdfVolume vol(vc);
    check(vol.AllocateBlock({0, 0, 0}), "AllocateBlock creates");
    check(!vol.AllocateBlock({0, 0, 0}), "AllocateBlock of an existing block returns false");
    check(vol.FindBlock({0, 0, 0}) != nullptr && vol.FindBlock({5, 5, 5}) == nullptr, "FindBlock");
    check(vol.VoxelHandle(ts::Vec3i{100, 0, 0}) == nullptr, "VoxelHandle outside allocated blocks is null");

    // test_util.hpp:48-58 style: write every voxel of the block through mutable handles
    for (int z = 0; z < 8; ++z)
        for (int y = 0; y < 8; ++y)
            for (int x = 0; x < 8; ++x) {
                ts::Voxel* v = vol.VoxelHandle(ts::Vec3i{x, y, z});
                v->sdf = float(0.01 * x);
                v->weight = 10;
                v->r = v->g = v->b = 100;
            }
    const ts::VoxelBlock* b = vol.FindBlock({0, 0, 0});
    check(b && b->voxels[7].sdf == float(0.07) && b->voxels[7].weight == 10, "FindBlock sees handle writes");
    // the write-back happens before the GPU samples: trilinear between voxels 2 and 3 along x
    const ts::Vec3 p{(2.5 + 0.5) * 0.02, 3.5 * 0.02, 3.5 * 0.02};
    const ts::SdfSample s = vol.SampleSdf(p);
    check(s.valid && std::fabs(s.value - 0.025) < 1e-6, "SampleSdf reads the handle writes on the GPU");
    // a pointer taken before a GPU operation stays valid; a new handle sees the current state
    const ts::Voxel* held = vol.VoxelHandle(ts::Vec3i{1, 1, 1});
    check(held != nullptr && held->weight == 10, "held const handle");
    const auto blocks = vol.blocks();
    check(blocks.size() == 1 && blocks[0].voxels[0].weight == 10, "blocks() after write-back");
    const std::string path = "/tmp/host_volume_demo.bin";
    vol.Save(path);
    ts::TsdfVolume loaded = ts::TsdfVolume::Load(path);
    const ts::Voxel* lv = loaded.VoxelHandle(ts::Vec3i{3, 2, 1});
    check(lv && lv->sdf == float(0.03) && lv->weight == 10, "Save/Load keep handle writes");

    // BuildPyramid (test_registration.cpp:50-77)
    ts::Frame f;
    f.intrinsics.fx = f.intrinsics.fy = 10.0;
    f.intrinsics.cx = 3.5;
    f.intrinsics.cy = 1.5;
    f.intrinsics.width = 8;
    f.intrinsics.height = 4;
    f.depth = ts::DepthImage(8, 4);
    f.color = ts::ColorImage(8, 4);
    for (int v = 0; v < 4; ++v)
        for (int u = 0; u < 8; ++u) {
            f.depth(u, v) = float(1.0 + u + 8.0 * v);
            const auto g = std::uint8_t(10 * u + v);
            f.color(u, v) = ts::Rgb8{g, g, g};
        }
    f.depth(2, 1) = 0.f;
    ts::PixelMask mask(8, 4, 0);
    mask(5, 2) = 1;
    const auto pyr = ts::BuildPyramid(f, &mask, 3);
    check(pyr.size() == 3 && pyr[1].depth.width() == 4 && pyr[2].depth.height() == 1, "pyramid sizes");
    check(pyr[1].intrinsics.fx == 5.0, "pyramid intrinsics");
    check(pyr[1].depth(0, 0) == 1.0f && pyr[1].depth(1, 0) == 3.0f, "closest valid depth");
    check(std::fabs(pyr[1].intensity(0, 0) - (0.0 + 10.0 + 1.0 + 11.0) / 4.0) < 1e-4, "mean intensity");
    check(pyr[1].mask(2, 1) == 1 && pyr[1].mask(0, 0) == 0 && pyr[2].mask(1, 0) == 1, "mask spreads");
    bool threw = false;
    try {
        ts::BuildPyramid(f, nullptr, 0);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    check(threw, "BuildPyramid(levels = 0) throws std::invalid_argument");
    return failures ? 1 : 0;
}
