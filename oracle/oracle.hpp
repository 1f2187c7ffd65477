// ORACLE — test infrastructure only. CPU restatement of the reference hot path
// (/root/reference/proj, the `tsdfslam` C++20 library). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it. The product (paper_1905_02082_b200) never links or calls it.
//
// Why a restatement and not the reference itself: the reference needs Eigen3,
// libpng, doctest and CLI11, none of which exist in this image (no network),
// so per the task rules it is treated as unbuildable.
// Every function below cites the reference file:line it follows. Arithmetic
// contract (the thing the CUDA path must reproduce bit for bit where parity
// is bit-exact): IEEE double, no FMA contraction (-ffp-contract=off), small
// dense products summed left to right, exactly the operation order written in
// the reference expressions.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <algorithm>
#include <utility>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------------------
// Small fixed-size linear algebra (replaces the Eigen subset the reference uses)
// ---------------------------------------------------------------------------
struct V3d {
    double x = 0, y = 0, z = 0;
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
struct V3i {
    int x = 0, y = 0, z = 0;
    int& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    int operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    bool operator==(const V3i& o) const { return x == o.x && y == o.y && z == o.z; }
    bool operator!=(const V3i& o) const { return !(*this == o); }
};
inline V3d operator+(const V3d& a, const V3d& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3d operator-(const V3d& a, const V3d& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3d operator*(double s, const V3d& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3d operator*(const V3d& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3d operator/(const V3d& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline V3d operator-(const V3d& a) { return {-a.x, -a.y, -a.z}; }
inline V3i operator+(const V3i& a, const V3i& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3i operator-(const V3i& a, const V3i& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3i operator*(const V3i& a, int s) { return {a.x * s, a.y * s, a.z * s}; }
inline double Dot(const V3d& a, const V3d& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline V3d Cross(const V3d& a, const V3d& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double Norm(const V3d& a) { return std::sqrt(Dot(a, a)); }
inline V3d ToD(const V3i& v) { return {double(v.x), double(v.y), double(v.z)}; }

// Row-major 3x3.
struct M3d {
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    double& operator()(int r, int c) { return m[3 * r + c]; }
    double operator()(int r, int c) const { return m[3 * r + c]; }
    static M3d Identity() { return M3d{}; }
    static M3d Zero() {
        M3d z;
        for (double& v : z.m) v = 0;
        return z;
    }
};
inline V3d operator*(const M3d& a, const V3d& x) {
    return {(a(0, 0) * x.x + a(0, 1) * x.y) + a(0, 2) * x.z,
            (a(1, 0) * x.x + a(1, 1) * x.y) + a(1, 2) * x.z,
            (a(2, 0) * x.x + a(2, 1) * x.y) + a(2, 2) * x.z};
}
inline M3d operator*(const M3d& a, const M3d& b) {
    M3d r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r(i, j) = (a(i, 0) * b(0, j) + a(i, 1) * b(1, j)) + a(i, 2) * b(2, j);
    return r;
}
inline M3d Transpose(const M3d& a) {
    M3d r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r(i, j) = a(j, i);
    return r;
}

// proj/include/tsdfslam/geometry.hpp:11-38
struct Intrinsics {
    double fx = 525.0, fy = 525.0, cx = 319.5, cy = 239.5;
    int width = 640, height = 480;
    double depth_scale = 5000.0;
    bool Valid() const {
        return fx > 0.0 && fy > 0.0 && width > 0 && height > 0 && cx > 0.0 && cx < double(width) &&
               cy > 0.0 && cy < double(height) && depth_scale > 0.0;
    }
    Intrinsics Scaled(int level) const {  // geometry.hpp:27-37
        const double s = 1.0 / static_cast<double>(1 << level);
        Intrinsics k = *this;
        k.fx *= s;
        k.fy *= s;
        k.cx *= s;
        k.cy *= s;
        k.width = width >> level;
        k.height = height >> level;
        return k;
    }
};

// geometry.hpp:41-48
inline V3d Backproject(double u, double v, double depth, const Intrinsics& k) {
    return {(u - k.cx) / k.fx * depth, (v - k.cy) / k.fy * depth, depth};
}
inline void Project(const V3d& x, const Intrinsics& k, double& pu, double& pv) {
    pu = k.fx * x.x / x.z + k.cx;
    pv = k.fy * x.y / x.z + k.cy;
}

// Camera-to-world rigid transform, geometry.hpp:69-108.
struct Pose {
    M3d R = M3d::Identity();
    V3d t{};
    V3d operator*(const V3d& x) const { return R * x + t; }
    Pose operator*(const Pose& o) const { return {R * o.R, R * o.t + t}; }
    Pose Inverse() const {
        const M3d rt = Transpose(R);
        return {rt, -(rt * t)};
    }
    void ToArray(double out[12]) const {
        for (int i = 0; i < 9; ++i) out[i] = R.m[i];
        out[9] = t.x;
        out[10] = t.y;
        out[11] = t.z;
    }
    static Pose FromArray(const double in[12]) {
        Pose p;
        for (int i = 0; i < 9; ++i) p.R.m[i] = in[i];
        p.t = {in[9], in[10], in[11]};
        return p;
    }
};

inline M3d Skew(const V3d& w) {  // geometry.hpp:111-115
    M3d s;
    s.m[0] = 0.0; s.m[1] = -w.z; s.m[2] = w.y;
    s.m[3] = w.z; s.m[4] = 0.0; s.m[5] = -w.x;
    s.m[6] = -w.y; s.m[7] = w.x; s.m[8] = 0.0;
    return s;
}
Pose ExpMap(const double xi[6]);   // geometry.cpp:14-38 (xi = v, w)
void LogMap(const Pose& p, double xi[6]);  // geometry.cpp:40-57

// ---------------------------------------------------------------------------
// Images (image.hpp:13-103): row-major, owned vectors.
// ---------------------------------------------------------------------------
template <typename T>
struct Image {
    int w = 0, h = 0;
    std::vector<T> d;
    Image() = default;
    Image(int w_, int h_, T fill = T{}) : w(w_), h(h_), d(size_t(w_) * h_, fill) {}
    bool Empty() const { return d.empty(); }
    bool InBounds(int x, int y) const { return x >= 0 && x < w && y >= 0 && y < h; }
    T& operator()(int x, int y) { return d[size_t(y) * w + x]; }
    const T& operator()(int x, int y) const { return d[size_t(y) * w + x]; }
};
struct Rgb8 {
    uint8_t r = 0, g = 0, b = 0;
};
using DepthImage = Image<float>;
using ColorImage = Image<Rgb8>;
using Mask = Image<uint8_t>;
inline bool DepthValid(float d) { return d > 0.0f && std::isfinite(d); }  // image.hpp:68
inline double Intensity(const Rgb8& c) {                                    // image.hpp:80-83
    return 0.2126 * double(c.r) + 0.7152 * double(c.g) + 0.0722 * double(c.b);
}
struct Frame {
    double timestamp = 0.0;
    Intrinsics intr;
    DepthImage depth;
    ColorImage color;
};

// ---------------------------------------------------------------------------
// Spatial hash, spatial_hash.hpp:13-86
// ---------------------------------------------------------------------------
inline uint64_t HashCoord(const V3i& c) {
    const uint64_t hx = uint64_t(uint32_t(c.x)) * uint64_t{73856093u};
    const uint64_t hy = uint64_t(uint32_t(c.y)) * uint64_t{19349669u};
    const uint64_t hz = uint64_t(uint32_t(c.z)) * uint64_t{83492791u};
    return hx ^ hy ^ hz;
}

class CoordHashMap {
  public:
    explicit CoordHashMap(size_t initial_capacity = 1024) {
        size_t cap = 16;
        while (cap < initial_capacity) cap <<= 1;
        slots_.resize(cap);
    }
    size_t size() const { return size_; }
    size_t capacity() const { return slots_.size(); }
    size_t ProbeSlot(const V3i& c) const {
        size_t idx = HashCoord(c) & (slots_.size() - 1);
        while (slots_[idx].used && slots_[idx].coord != c) idx = (idx + 1) & (slots_.size() - 1);
        return idx;
    }
    const uint32_t* Find(const V3i& c) const {
        const size_t idx = ProbeSlot(c);
        return slots_[idx].used ? &slots_[idx].value : nullptr;
    }
    std::pair<uint32_t, bool> Insert(const V3i& c, uint32_t value) {
        if ((size_ + 1) * 4 > slots_.size() * 3) Grow();
        const size_t idx = ProbeSlot(c);
        if (slots_[idx].used) return {slots_[idx].value, false};
        slots_[idx] = Slot{c, value, true};
        ++size_;
        return {value, true};
    }
    bool SlotUsed(size_t i) const { return slots_[i].used; }
    const V3i& SlotCoord(size_t i) const { return slots_[i].coord; }

  private:
    struct Slot {
        V3i coord{};
        uint32_t value = 0;
        bool used = false;
    };
    void Grow() {
        std::vector<Slot> old = std::move(slots_);
        slots_.assign(old.size() * 2, Slot{});
        for (const Slot& s : old) {
            if (!s.used) continue;
            size_t idx = HashCoord(s.coord) & (slots_.size() - 1);
            while (slots_[idx].used) idx = (idx + 1) & (slots_.size() - 1);
            slots_[idx] = s;
        }
    }
    std::vector<Slot> slots_;
    size_t size_ = 0;
};

// ---------------------------------------------------------------------------
// TSDF volume, tsdf_volume.hpp:14-134 / tsdf_volume.cpp
// ---------------------------------------------------------------------------
struct VolumeConfig {
    double voxel_size = 0.01, truncation = 0.1;
    int block_side = 8, max_weight = 64, carve_weight = 1;
    double min_depth = 0.1, max_depth = 5.0, carve_clip = 4.0;
    uint64_t max_blocks = 1000000;
    void Validate() const;
};
struct Voxel {
    float sdf = 0.f;
    uint8_t weight = 0, r = 0, g = 0, b = 0;
};
static_assert(sizeof(Voxel) == 8, "voxel is 8 bytes");
struct VoxelBlock {
    V3i coord;
    std::vector<Voxel> voxels;
};
struct Sample {
    double value = 0.0;
    V3d gradient{};
    bool valid = false;
};

struct ResourceLimitError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TrackingLostError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline int FloorDiv(int a, int b) {  // tsdf_volume.hpp:136-140
    int q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

class Volume {
  public:
    explicit Volume(VolumeConfig c) : cfg_(c) { cfg_.Validate(); }
    const VolumeConfig& config() const { return cfg_; }
    const std::vector<VoxelBlock>& blocks() const { return blocks_; }
    std::vector<VoxelBlock>& blocks_mut() { return blocks_; }
    size_t num_blocks() const { return blocks_.size(); }
    double block_extent() const { return cfg_.block_side * cfg_.voxel_size; }
    const CoordHashMap& index() const { return index_; }

    bool AllocateBlock(const V3i& bc);
    const VoxelBlock* FindBlock(const V3i& bc) const;
    const Voxel* VoxelHandle(const V3i& v) const;
    Voxel* VoxelHandle(const V3i& v) {
        return const_cast<Voxel*>(static_cast<const Volume*>(this)->VoxelHandle(v));
    }
    V3d VoxelCenter(const V3i& v) const {
        return {(double(v.x) + 0.5) * cfg_.voxel_size, (double(v.y) + 0.5) * cfg_.voxel_size,
                (double(v.z) + 0.5) * cfg_.voxel_size};
    }
    void AllocateForFrame(const DepthImage& depth, const Intrinsics& k, const Pose& c2w,
                          const Mask* mask);
    void Integrate(const Frame& f, const Pose& c2w, const Mask* mask, int threads);
    void Carve(const DepthImage& depth, const Intrinsics& k, const Pose& c2w, int threads);
    Sample SampleSdf(const V3d& p) const;
    Sample SampleIntensity(const V3d& p) const;
    Sample SampleSdfWithGradient(const V3d& p) const;
    Sample SampleIntensityWithGradient(const V3d& p) const;
    Sample SampleSdfGradient(const V3d& p) const;
    bool GatherCorners(const V3i& base, const Voxel* corners[8]) const;

    // Counters for the bench's algorithmic-bytes model (not in the reference).
    uint64_t last_dda_visits = 0, last_new_blocks = 0;

  private:
    template <typename F>
    Sample SampleWithGradientImpl(const V3d& p, F&& value_of) const;
    VolumeConfig cfg_;
    CoordHashMap index_;
    std::vector<VoxelBlock> blocks_;
};

template <typename Fn>
void WalkGridSegment(const V3d& a, const V3d& b, double ext, Fn&& fn) {  // tsdf_volume.hpp:149-185
    const V3d p0 = a / ext;
    const V3d p1 = b / ext;
    const V3d d = p1 - p0;
    V3i cell{int(std::floor(p0.x)), int(std::floor(p0.y)), int(std::floor(p0.z))};
    const V3i end{int(std::floor(p1.x)), int(std::floor(p1.y)), int(std::floor(p1.z))};
    V3i step{0, 0, 0};
    const double inf = std::numeric_limits<double>::infinity();
    double t_max[3] = {inf, inf, inf}, t_delta[3] = {inf, inf, inf};
    for (int i = 0; i < 3; ++i) {
        if (d[i] > 0) {
            step[i] = 1;
            t_max[i] = (std::floor(p0[i]) + 1.0 - p0[i]) / d[i];
            t_delta[i] = 1.0 / d[i];
        } else if (d[i] < 0) {
            step[i] = -1;
            t_max[i] = (p0[i] - std::floor(p0[i])) / -d[i];
            t_delta[i] = 1.0 / -d[i];
        }
    }
    const int max_steps = std::abs(end.x - cell.x) + std::abs(end.y - cell.y) +
                          std::abs(end.z - cell.z) + 3;
    fn(cell);
    for (int n = 0; n < max_steps && cell != end; ++n) {
        int axis = 0;
        if (t_max[1] < t_max[axis]) axis = 1;
        if (t_max[2] < t_max[axis]) axis = 2;
        if (t_max[axis] > 1.0) break;
        t_max[axis] += t_delta[axis];
        cell[axis] += step[axis];
        fn(cell);
    }
}

// ---------------------------------------------------------------------------
// Registration, registration.hpp / registration.cpp
// ---------------------------------------------------------------------------
struct RegistrationConfig {
    double color_weight = 0.025;
    int pyramid_levels = 3, max_iterations = 20;
    double lm_lambda_init = 1e-4, lm_lambda_up = 10.0, lm_lambda_down = 2.0;
    double convergence_eps = 1e-5;
    int min_valid_residuals = 100;
    int threads = 1;
    // Extensions (not in the reference; 0 / false reproduce it): Huber
    // weighting of the depth / colour residuals, and the residual sign in
    // bit 1 of ResidualImage::valid (set by the pipeline when the mask's
    // free-space term is on).
    double huber_depth = 0.0, huber_color = 0.0;
    bool residual_sign = false;
};
struct Robust {  // the extensions Accumulate applies
    double huber_depth = 0.0, huber_color = 0.0;
    bool residual_sign = false;
};
struct ResidualImage {
    Image<float> squared;
    Mask valid;
};
struct PyramidLevel {
    Intrinsics intr;
    DepthImage depth;
    Image<float> intensity;
    Mask mask;
};
struct Accum {
    double H[36] = {0};
    double b[6] = {0};
    double depth_error = 0.0, color_error = 0.0;
    size_t valid = 0;
};
struct RegistrationResult {
    Pose pose;
    bool converged = false;
    int iterations = 0;
    size_t valid_residuals = 0;
    double final_error = 0.0;
    ResidualImage residuals;
};
std::vector<PyramidLevel> BuildPyramid(const Frame& f, const Mask* mask, int levels);
Accum Accumulate(const Volume& vol, const PyramidLevel& level, const Pose& pose, double cw,
                 bool with_jacobian, bool use_mask, int threads, ResidualImage* out,
                 const Robust& rb = Robust());
PyramidLevel LevelZero(const Frame& f, const Mask* mask);
RegistrationResult Register(const Volume& vol, const Frame& f, const Pose& init, const Mask* mask,
                            const RegistrationConfig& cfg);
// Eigen::LDLT<Matrix6> restated (pivoted, lower). Returns false on NumericalIssue.
bool Ldlt6Solve(const double A[36], const double rhs[6], double x[6]);
bool Degenerate(const Accum& acc);  // registration.cpp:128-139

// ---------------------------------------------------------------------------
// Dynamics mask, dynamics_mask.cpp
// ---------------------------------------------------------------------------
struct MaskConfig {
    double gamma = 0.5, truncation = 0.1, theta = 0.007;
    int erode_radius = 2, dilate_radius = 2, connectivity = 4;
    double free_space = 0.0;  // extension (0: off): positive residuals > free_space also seed the mask
};
Mask ThresholdResiduals(const ResidualImage& r, const MaskConfig& c);
Mask Erode(const Mask& m, int radius);
Mask Dilate(const Mask& m, int radius);
Mask FloodfillDepth(const Mask& seeds, const DepthImage& depth, double theta, int connectivity);
Mask BuildMask(const ResidualImage& r, const DepthImage& depth, const MaskConfig& c);

// ---------------------------------------------------------------------------
// Pipeline, pipeline.cpp:25-131 (refinement window supported)
// ---------------------------------------------------------------------------
struct RefinementConfig {
    bool enabled = true;
    int window = 10;
    double far_value = 8.0;
    int bisection_iterations = 8;
};
struct PipelineConfig {
    VolumeConfig volume;
    RegistrationConfig registration;
    MaskConfig mask;
    RefinementConfig refinement;
    bool dynamics_enabled = true;
    int threads = 1;
    void Sync();
};
struct FrameStats {
    uint64_t frame_index = 0;
    double timestamp = 0.0;
    int32_t tracking_lost = 0, converged = 0, registrations = 0, iterations = 0;
    uint64_t valid_residuals = 0, masked_pixels = 0;
    double final_error = 0.0, runtime_ms = 0.0;
};
struct WindowEntry {
    Frame frame;
    Pose pose;
    Mask mask;
};

// Ray-march of RenderVirtualDepth (depth_refinement.cpp:32-79) on a given volume.
DepthImage RaycastDepth(const Volume& vol, const Pose& view, const Intrinsics& k,
                        int bisection_iterations, int threads);
DepthImage RenderVirtualDepth(const std::vector<WindowEntry>& window, const Pose& view,
                              const Intrinsics& k, const VolumeConfig& vc,
                              const RefinementConfig& rc, int threads);
DepthImage RefineDepth(const DepthImage& raw, const DepthImage& virt, double far_value);

class Pipeline {
  public:
    explicit Pipeline(PipelineConfig c);
    FrameStats ProcessFrame(const Frame& f);
    void Finalize();
    Volume& volume() { return volume_; }
    const std::vector<std::pair<double, Pose>>& trajectory() const { return trajectory_; }
    const std::vector<FrameStats>& stats() const { return stats_; }
    size_t losses() const { return losses_; }
    // Artifacts of the most recent registered frame (debug sink analogue).
    Mask last_mask;
    ResidualImage last_residuals;
    bool last_has_mask = false;

  private:
    void IntegrateFront();
    void CarveAndIntegrate(const Frame& f, const Pose& p, const Mask* m);
    PipelineConfig cfg_;
    Volume volume_;
    std::vector<WindowEntry> window_;
    std::vector<size_t> pending_;
    std::vector<std::pair<double, Pose>> trajectory_;
    std::vector<FrameStats> stats_;
    Pose current_;
    bool first_ = true;
    size_t frame_count_ = 0, losses_ = 0;
};

// ---------------------------------------------------------------------------
// Marching cubes, mesh.cpp:50-181
// ---------------------------------------------------------------------------
struct Mesh {
    std::vector<float> vertices;  // xyz
    std::vector<uint8_t> colors;  // rgb
    std::vector<int32_t> faces;   // i0 i1 i2
};
Mesh ExtractMesh(const Volume& vol, int min_weight, int threads);

// ---------------------------------------------------------------------------
// Synthetic scenes, synth.hpp / synth.cpp (input generation for parity runs)
// ---------------------------------------------------------------------------
struct Quat {
    double w = 1, x = 0, y = 0, z = 0;
};
struct Primitive {
    std::string name;
    bool dynamic = false;
    int shape = 0;  // 0 plane, 1 sphere, 2 box
    V3d a{}, b{0, 0, 1};
    bool checker = false;
    double cell = 0.25;
    Rgb8 primary{200, 200, 200}, secondary{60, 60, 60};
    std::vector<std::pair<double, Pose>> keyframes;
    Pose PoseAt(double time) const;
};
struct Scene {
    Intrinsics intr;
    double noise_sigma_scale = 0.0, dropout = 0.0;
    uint32_t seed = 0;
    std::vector<Primitive> prims;
    std::vector<std::pair<double, Pose>> camera;
    static Scene Parse(const std::string& text);
};
struct Rendered {
    Frame frame;
    DepthImage true_depth;
    Mask labels;
};
Rendered RenderFrame(const Scene& s, size_t i);
Pose PoseFromQuat(const Quat& q, const V3d& t);
Quat QuatFromMatrix(const M3d& m);

// ---------------------------------------------------------------------------
// Parallel helpers, parallel.hpp:15-47
// ---------------------------------------------------------------------------
// parallel.hpp:15-34
template <typename Fn>
void ParallelFor(size_t count, int threads, const Fn& fn) {
    if (count == 0) return;
    if (threads <= 1 || count == 1) {
        for (size_t i = 0; i < count; ++i) fn(i);
        return;
    }
    const size_t workers = std::min<size_t>(size_t(threads), count);
    std::vector<std::thread> pool;
    pool.reserve(workers);
    const size_t chunk = (count + workers - 1) / workers;
    for (size_t w = 0; w < workers; ++w) {
        const size_t begin = w * chunk;
        const size_t end = std::min(count, begin + chunk);
        if (begin >= end) break;
        pool.emplace_back([&fn, begin, end] {
            for (size_t i = begin; i < end; ++i) fn(i);
        });
    }
    for (auto& t : pool) t.join();
}


}  // namespace oracle
