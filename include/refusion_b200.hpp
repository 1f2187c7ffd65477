// refusion_b200.hpp — C++ host layer over the C ABI (refusion_b200.h).
//
// Mirrors the tracker/map interfaces of the CPU reference `tsdfslam`
// (/root/reference/proj/include/tsdfslam: geometry.hpp, image.hpp,
// tsdf_volume.hpp, registration.hpp, dynamics_mask.hpp, mesh.hpp,
// pipeline.hpp, errors.hpp) with the same class / function names, argument
// meaning and exceptions, so a caller of the reference switches by changing
// the include and the namespace (`namespace tsdfslam = tsdfslam_b200;`).
// Eigen is not a dependency: vectors are std::array<double, 3>, rotations
// row-major std::array<double, 9>. With REFUSION_B200_EIGEN defined (and
// Eigen on the include path) the vector, rotation and pose types are the
// reference's Eigen types instead, so the reference's own sources (its test
// suites) compile unchanged against this layer (tests/refsuite).
//
// Everything computes on the GPU: the methods marshal host images into an
// rf_frame and call one C entry point. Header-only; link with
// -lrefusion_b200 (paper_1905_02082_b200/librefusion_b200.so).
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "refusion_b200.h"
#ifdef REFUSION_B200_EIGEN
#include <Eigen/Core>
#include <Eigen/Geometry>
#endif

namespace tsdfslam_b200 {

// ---------------------------------------------------------------- errors (errors.hpp:9-21)
struct InsufficientOverlapError : std::runtime_error {
    explicit InsufficientOverlapError(const std::string& what) : std::runtime_error(what) {}
};
struct TrackingLostError : std::runtime_error {
    explicit TrackingLostError(const std::string& what) : std::runtime_error(what) {}
};
struct ResourceLimitError : std::runtime_error {
    explicit ResourceLimitError(const std::string& what) : std::runtime_error(what) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};

// Rethrows an rf_status as the reference's exception type.
inline void Check(rf_status s) {
    if (s == RF_OK) return;
    const std::string msg = rf_last_error();
    switch (s) {
        case RF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case RF_TRACKING_LOST: throw TrackingLostError(msg);
        case RF_RESOURCE_LIMIT: throw ResourceLimitError(msg);
        case RF_IO_ERROR: throw std::runtime_error(msg);
        case RF_FAILED: throw std::runtime_error(msg);
        case RF_UNSUPPORTED: throw std::invalid_argument("unsupported on the CUDA path: " + msg);
        default: throw CudaError(msg);
    }
}

#ifdef REFUSION_B200_EIGEN
using Vec3 = Eigen::Vector3d;
using Vec3i = Eigen::Vector3i;
using Vec3f = Eigen::Vector3f;
using Mat3 = Eigen::Matrix3d;
#else
using Vec3 = std::array<double, 3>;
using Vec3i = std::array<int, 3>;
using Vec3f = std::array<float, 3>;
using Mat3 = std::array<double, 9>;  // row-major
#endif

// ---------------------------------------------------------------- geometry (geometry.hpp:11-108)
struct CameraIntrinsics {
    double fx = 525.0, fy = 525.0, cx = 319.5, cy = 239.5;
    int width = 640, height = 480;
    double depth_scale = 5000.0;

    bool Valid() const {
        return fx > 0.0 && fy > 0.0 && width > 0 && height > 0 && cx > 0.0 && cx < double(width) && cy > 0.0 &&
               cy < double(height) && depth_scale > 0.0;
    }
    CameraIntrinsics Scaled(int level) const {
        const double s = 1.0 / double(1 << level);
        CameraIntrinsics k = *this;
        k.fx *= s;
        k.fy *= s;
        k.cx *= s;
        k.cy *= s;
        k.width = width >> level;
        k.height = height >> level;
        return k;
    }
    rf_intrinsics c() const { return rf_intrinsics{fx, fy, cx, cy, width, height, depth_scale}; }
};

// Camera-to-world rigid transform; the C ABI's 12-double layout (R row-major, t).
class Pose {
  public:
    Pose() : m_{1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0} {}
    Pose(const Mat3& rotation, const Vec3& translation) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m_[3 * i + j] = M(rotation, i, j);
        for (int i = 0; i < 3; ++i) m_[9 + i] = translation[i];
    }
#ifdef REFUSION_B200_EIGEN
    Pose(const Eigen::Quaterniond& q, const Vec3& translation) : Pose(Mat3(q.normalized().toRotationMatrix()), translation) {}
#endif
    static Pose Identity() { return Pose(); }
    static Pose FromArray(const double p[12]) {
        Pose r;
        std::memcpy(r.m_.data(), p, 12 * sizeof(double));
        return r;
    }
    Mat3 rotation() const {
        Mat3 r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) M(r, i, j) = m_[3 * i + j];
        return r;
    }
    Vec3 translation() const { return Vec3{m_[9], m_[10], m_[11]}; }
    const double* data() const { return m_.data(); }
    double* data() { return m_.data(); }
#ifdef REFUSION_B200_EIGEN
    Eigen::Matrix4d Matrix() const {  // homogeneous 4x4 (geometry.hpp:96-101)
        Eigen::Matrix4d T = Eigen::Matrix4d::Identity();
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j) T(i, j) = m_[3 * i + j];
            T(i, 3) = m_[9 + i];
        }
        return T;
    }
#else
    std::array<double, 16> Matrix() const {  // homogeneous 4x4, row-major
        return {m_[0], m_[1], m_[2], m_[9], m_[3], m_[4], m_[5], m_[10], m_[6], m_[7], m_[8], m_[11], 0, 0, 0, 1};
    }
#endif

    Vec3 operator*(const Vec3& x) const {
        Vec3 r;
        for (int i = 0; i < 3; ++i) r[i] = m_[3 * i] * x[0] + m_[3 * i + 1] * x[1] + m_[3 * i + 2] * x[2] + m_[9 + i];
        return r;
    }
    Pose operator*(const Pose& o) const {
        Pose r;
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j)
                r.m_[3 * i + j] = m_[3 * i] * o.m_[j] + m_[3 * i + 1] * o.m_[3 + j] + m_[3 * i + 2] * o.m_[6 + j];
            r.m_[9 + i] = m_[3 * i] * o.m_[9] + m_[3 * i + 1] * o.m_[10] + m_[3 * i + 2] * o.m_[11] + m_[9 + i];
        }
        return r;
    }
    // Rotation orthonormal with determinant +1 and all entries finite, to `tol` (geometry.hpp:103).
    bool IsValid(double tol = 1e-9) const {
        for (double x : m_)
            if (!std::isfinite(x)) return false;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                const double d = m_[3 * i] * m_[3 * j] + m_[3 * i + 1] * m_[3 * j + 1] + m_[3 * i + 2] * m_[3 * j + 2];
                if (std::abs(d - (i == j ? 1.0 : 0.0)) > tol) return false;
            }
        const double det = m_[0] * (m_[4] * m_[8] - m_[5] * m_[7]) - m_[1] * (m_[3] * m_[8] - m_[5] * m_[6]) +
                           m_[2] * (m_[3] * m_[7] - m_[4] * m_[6]);
        return std::abs(det - 1.0) <= tol;
    }
    Pose Inverse() const {
        Pose r;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) r.m_[3 * i + j] = m_[3 * j + i];
        for (int i = 0; i < 3; ++i)
            r.m_[9 + i] = -(r.m_[3 * i] * m_[9] + r.m_[3 * i + 1] * m_[10] + r.m_[3 * i + 2] * m_[11]);
        return r;
    }

  private:
#ifdef REFUSION_B200_EIGEN
    static double M(const Mat3& r, int i, int j) { return r(i, j); }
    static double& M(Mat3& r, int i, int j) { return r(i, j); }
#else
    static double M(const Mat3& r, int i, int j) { return r[3 * i + j]; }
    static double& M(Mat3& r, int i, int j) { return r[3 * i + j]; }
#endif
    std::array<double, 12> m_;
};

inline constexpr double kSmallAngle = 1e-6;  // ExpMap / LogMap series branch (geometry.hpp:123)
// W with W x = w x x (geometry.hpp:110-114).
inline Mat3 SkewMatrix(const Vec3& w) {
    Mat3 s;
    const double e[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
#ifdef REFUSION_B200_EIGEN
            s(i, j) = e[3 * i + j];
#else
            s[3 * i + j] = e[3 * i + j];
#endif
        }
    return s;
}
// Twist / ExpMap / LogMap (geometry.hpp:53-121): se(3) increments on the
// host (the GPU's LM applies its own ExpMap in the tracking kernel).
#ifdef REFUSION_B200_EIGEN
using Vec6 = Eigen::Matrix<double, 6, 1>;
#else
using Vec6 = std::array<double, 6>;
#endif
struct Twist {
    Vec3 v = Vec3{0.0, 0.0, 0.0};  // translational part (m)
    Vec3 w = Vec3{0.0, 0.0, 0.0};  // rotational part (rad)
    Twist() = default;
    Twist(const Vec3& v_in, const Vec3& w_in) : v(v_in), w(w_in) {}
    explicit Twist(const Vec6& xi) : v(Vec3{xi[0], xi[1], xi[2]}), w(Vec3{xi[3], xi[4], xi[5]}) {}
    Vec6 Vector() const {
        Vec6 xi;
        for (int i = 0; i < 3; ++i) {
            xi[i] = v[i];
            xi[3 + i] = w[i];
        }
        return xi;
    }
    double Norm() const {
        double s = 0.0;
        for (int i = 0; i < 3; ++i) s += v[i] * v[i] + w[i] * w[i];
        return std::sqrt(s);
    }
};
// exp of the twist: R = I + a W + b W^2, t = (I + b W + c W^2) v with
// a = sin t / t, b = (1 - cos t) / t^2, c = (t - sin t) / t^3 (series below 1e-6).
inline Pose ExpMap(const Twist& xi) {
    const double w0 = xi.w[0], w1 = xi.w[1], w2 = xi.w[2];
    const double t2 = w0 * w0 + w1 * w1 + w2 * w2, th = std::sqrt(t2);
    double a, b, c;
    if (th < kSmallAngle) {
        a = 1.0 - t2 / 6.0;
        b = 0.5 - t2 / 24.0;
        c = 1.0 / 6.0 - t2 / 120.0;
    } else {
        a = std::sin(th) / th;
        b = (1.0 - std::cos(th)) / t2;
        c = (th - std::sin(th)) / (t2 * th);
    }
    const double W[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
    double W2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) W2[3 * i + j] = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
    double p[12];
    for (int i = 0; i < 9; ++i) {
        const double id = (i % 4 == 0) ? 1.0 : 0.0;
        p[i] = id + a * W[i] + b * W2[i];
    }
    for (int i = 0; i < 3; ++i) {
        double s = 0.0;
        for (int j = 0; j < 3; ++j) {
            const double id = i == j ? 1.0 : 0.0;
            s += (id + b * W[3 * i + j] + c * W2[3 * i + j]) * xi.v[j];
        }
        p[9 + i] = s;
    }
    return Pose::FromArray(p);
}
// log of the pose (rotation angle < pi): w from the skew part of R, v = V^-1 t.
inline Twist LogMap(const Pose& pose) {
    const double* m = pose.data();
    const double cos_t = std::max(-1.0, std::min(1.0, 0.5 * (m[0] + m[4] + m[8] - 1.0)));
    const double th = std::acos(cos_t), s = std::sin(th);
    const double k = th < kSmallAngle ? 0.5 + th * th / 12.0 : th / (2.0 * s);
    const Vec3 w{k * (m[7] - m[5]), k * (m[2] - m[6]), k * (m[3] - m[1])};
    const double t2 = th * th;
    // V^-1 = I - W / 2 + (1 - (t sin t) / (2 (1 - cos t))) / t^2 W^2
    const double d = th < kSmallAngle ? 1.0 / 12.0 : (1.0 - th * s / (2.0 * (1.0 - cos_t))) / t2;
    const double W[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    Vec3 v{0.0, 0.0, 0.0};
    for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j) {
            const double W2 = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
            const double id = i == j ? 1.0 : 0.0;
            acc += (id - 0.5 * W[3 * i + j] + d * W2) * m[9 + j];
        }
        v[i] = acc;
    }
    return Twist(v, w);
}

// Backproject / Project (geometry.hpp:41-48): host-side camera model helpers.
inline Vec3 Backproject(double u, double v, double depth, const CameraIntrinsics& k) {
    return Vec3{(u - k.cx) / k.fx * depth, (v - k.cy) / k.fy * depth, depth};
}
#ifdef REFUSION_B200_EIGEN
using Vec2 = Eigen::Vector2d;
#else
using Vec2 = std::array<double, 2>;
#endif
inline Vec2 Project(const Vec3& x, const CameraIntrinsics& k) {
    return Vec2{k.fx * x[0] / x[2] + k.cx, k.fy * x[1] / x[2] + k.cy};
}

// FloorDiv (tsdf_volume.hpp:136-140): integer division rounding toward -inf.
inline int FloorDiv(int a, int b) {
    const int q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// WalkGridSegment (tsdf_volume.hpp:147-185): fn(cell) for every cell of size
// cell_extent the segment [a, b] passes through, in traversal order -- the
// host twin of the walk k_alloc runs per pixel (same floors, crossing times
// and tie order), for callers that enumerate cells themselves.
template <typename Fn>
void WalkGridSegment(const Vec3& a, const Vec3& b, double cell_extent, Fn&& fn) {
    const double inf = HUGE_VAL;
    double p0[3], p1[3], tmax[3], tdel[3];
    int cell[3], end[3], step[3];
    for (int i = 0; i < 3; ++i) {
        p0[i] = a[i] / cell_extent;
        p1[i] = b[i] / cell_extent;
        const double d = p1[i] - p0[i];
        cell[i] = int(std::floor(p0[i]));
        end[i] = int(std::floor(p1[i]));
        step[i] = d > 0 ? 1 : (d < 0 ? -1 : 0);
        tmax[i] = d > 0 ? (std::floor(p0[i]) + 1.0 - p0[i]) / d : (d < 0 ? (p0[i] - std::floor(p0[i])) / -d : inf);
        tdel[i] = d > 0 ? 1.0 / d : (d < 0 ? 1.0 / -d : inf);
    }
    auto visit = [&] { fn(Vec3i{cell[0], cell[1], cell[2]}); };
    visit();
    const int max_steps = std::abs(end[0] - cell[0]) + std::abs(end[1] - cell[1]) + std::abs(end[2] - cell[2]) + 3;
    for (int n = 0; n < max_steps && (cell[0] != end[0] || cell[1] != end[1] || cell[2] != end[2]); ++n) {
        const int ax = tmax[2] < (tmax[1] < tmax[0] ? tmax[1] : tmax[0]) ? 2 : (tmax[1] < tmax[0] ? 1 : 0);
        if (tmax[ax] > 1.0) break;
        tmax[ax] += tdel[ax];
        cell[ax] += step[ax];
        visit();
    }
}

// HashCoord / CoordHashMap (spatial_hash.hpp:10-83): the volume's brick hash
// (the same multiply-XOR hash and linear probing the GPU table uses,
// csrc/rf_common.cuh) as a host container from integer 3D coordinates to
// 32-bit values, for callers that index coordinates themselves. Power-of-two
// capacity, doubled before an insert would pass load 3/4; no removal.
inline std::uint64_t HashCoord(const Vec3i& c) {
    return (std::uint64_t(std::uint32_t(c[0])) * 73856093ull) ^ (std::uint64_t(std::uint32_t(c[1])) * 19349669ull) ^
           (std::uint64_t(std::uint32_t(c[2])) * 83492791ull);
}
class CoordHashMap {
  public:
    explicit CoordHashMap(std::size_t initial_capacity = 1024) {
        std::size_t n = 16;
        while (n < initial_capacity) n *= 2;
        Reset(n);
    }
    std::size_t size() const { return count_; }
    std::size_t capacity() const { return used_.size(); }
    // The slot `coord` probes to: its own, or the empty slot that ends its probe.
    std::size_t ProbeSlot(const Vec3i& coord) const {
        const std::size_t mask = used_.size() - 1;
        std::size_t i = std::size_t(HashCoord(coord)) & mask;
        while (used_[i] && !Same(keys_[i], coord)) i = (i + 1) & mask;
        return i;
    }
    const std::uint32_t* Find(const Vec3i& coord) const {
        const std::size_t i = ProbeSlot(coord);
        return used_[i] ? &values_[i] : nullptr;
    }
    // {stored value, true} when inserted; {existing value, false} when present.
    std::pair<std::uint32_t, bool> Insert(const Vec3i& coord, std::uint32_t value) {
        if (4 * (count_ + 1) > 3 * used_.size()) Rehash(2 * used_.size());
        const std::size_t i = ProbeSlot(coord);
        if (used_[i]) return {values_[i], false};
        used_[i] = 1;
        keys_[i] = Key{coord[0], coord[1], coord[2]};
        values_[i] = value;
        ++count_;
        return {value, true};
    }
    template <typename Fn>
    void ForEach(Fn&& fn) const {  // slot order
        for (std::size_t i = 0; i < used_.size(); ++i)
            if (used_[i]) fn(Vec3i{keys_[i][0], keys_[i][1], keys_[i][2]}, values_[i]);
    }

  private:
    using Key = std::array<int, 3>;
    static bool Same(const Key& k, const Vec3i& c) { return k[0] == c[0] && k[1] == c[1] && k[2] == c[2]; }
    void Reset(std::size_t n) {
        used_.assign(n, 0);
        keys_.assign(n, Key{0, 0, 0});
        values_.assign(n, 0u);
        count_ = 0;
    }
    void Rehash(std::size_t n) {  // re-inserts in the old slot order
        std::vector<std::uint8_t> used = std::move(used_);
        std::vector<Key> keys = std::move(keys_);
        std::vector<std::uint32_t> values = std::move(values_);
        Reset(n);
        for (std::size_t i = 0; i < used.size(); ++i) {
            if (!used[i]) continue;
            const Vec3i c{keys[i][0], keys[i][1], keys[i][2]};
            const std::size_t j = ProbeSlot(c);
            used_[j] = 1;
            keys_[j] = keys[i];
            values_[j] = values[i];
            ++count_;
        }
    }
    std::vector<std::uint8_t> used_;
    std::vector<Key> keys_;
    std::vector<std::uint32_t> values_;
    std::size_t count_ = 0;
};

// ---------------------------------------------------------------- images (image.hpp:13-103)
template <typename T>
class Image {
  public:
    Image() = default;
    Image(int width, int height, T fill = T{})
        : width_(width), height_(height), data_(std::size_t(width) * height, fill) {}
    int width() const { return width_; }
    int height() const { return height_; }
    bool Empty() const { return data_.empty(); }
    std::size_t PixelCount() const { return data_.size(); }
    bool InBounds(int x, int y) const { return x >= 0 && x < width_ && y >= 0 && y < height_; }
    T& operator()(int x, int y) { return data_[std::size_t(y) * width_ + x]; }
    const T& operator()(int x, int y) const { return data_[std::size_t(y) * width_ + x]; }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    void Fill(T value) { data_.assign(data_.size(), value); }
    bool SameSize(int w, int h) const { return width_ == w && height_ == h; }
    template <typename U>
    bool SameSize(const Image<U>& o) const {
        return SameSize(o.width(), o.height());
    }
    friend bool operator==(const Image& a, const Image& b) {
        return a.width_ == b.width_ && a.height_ == b.height_ && a.data_ == b.data_;
    }

  private:
    int width_ = 0, height_ = 0;
    std::vector<T> data_;
};

struct Rgb8 {
    std::uint8_t r = 0, g = 0, b = 0;
    friend bool operator==(const Rgb8&, const Rgb8&) = default;
};
static_assert(sizeof(Rgb8) == 3);

using DepthImage = Image<float>;
using ColorImage = Image<Rgb8>;
using PixelMask = Image<std::uint8_t>;

inline bool DepthValid(float d) { return d > 0.0f && std::isfinite(d); }
inline std::size_t CountMasked(const PixelMask& m) {
    std::size_t n = 0;
    for (std::size_t i = 0; i < m.PixelCount(); ++i) n += m.data()[i] != 0;
    return n;
}

struct Frame {
    double timestamp = 0.0;
    CameraIntrinsics intrinsics;
    DepthImage depth;
    ColorImage color;
    bool SizesConsistent() const {
        return depth.SameSize(intrinsics.width, intrinsics.height) && color.SameSize(depth);
    }
};

namespace detail {
inline rf_frame ToC(const Frame& f) {
    rf_frame c{};
    c.depth = f.depth.data();
    c.rgb = f.color.Empty() ? nullptr : reinterpret_cast<const std::uint8_t*>(f.color.data());
    c.intrinsics = f.intrinsics.c();
    c.timestamp = f.timestamp;
    c.memory = RF_MEMORY_HOST;
    return c;
}
inline rf_frame ToC(const DepthImage& d, const CameraIntrinsics& k) {
    rf_frame c{};
    c.depth = d.data();
    c.intrinsics = k.c();
    c.memory = RF_MEMORY_HOST;
    return c;
}
inline void RequireSize(const DepthImage& d, const CameraIntrinsics& k) {
    if (!d.SameSize(k.width, k.height)) throw std::invalid_argument("depth image does not match the intrinsics");
}
inline const std::uint8_t* MaskPtr(const PixelMask* m, int w, int h) {
    if (!m || m->Empty()) return nullptr;
    if (!m->SameSize(w, h)) throw std::invalid_argument("mask size does not match the frame");
    return m->data();
}
}  // namespace detail

// ---------------------------------------------------------------- volume (tsdf_volume.hpp:14-134)
struct VolumeConfig {
    double voxel_size = 0.01, truncation = 0.1;
    int block_side = 8, max_weight = 64, carve_weight = 1;
    double min_depth = 0.1, max_depth = 5.0, carve_clip = 4.0;
    std::size_t max_blocks = 1000000;
    std::size_t hash_capacity = 0;  // GPU only: 0 = next power of two >= 4/3 max_blocks

    void Validate() const {
        if (!(voxel_size > 0) || !(truncation >= voxel_size) || block_side < 2 || max_weight < 1 ||
            max_weight > 255 || carve_weight < 1 || carve_weight > max_weight || !(min_depth > 0) ||
            !(max_depth > min_depth) || !(carve_clip > 0) || max_blocks == 0)
            throw std::invalid_argument("invalid VolumeConfig");
    }
    rf_volume_config c() const {
        rf_volume_config r{};
        r.voxel_size = voxel_size;
        r.truncation = truncation;
        r.block_side = block_side;
        r.max_weight = max_weight;
        r.carve_weight = carve_weight;
        r.min_depth = min_depth;
        r.max_depth = max_depth;
        r.carve_clip = carve_clip;
        r.max_blocks = max_blocks;
        r.hash_capacity = hash_capacity;
        return r;
    }
};

struct Voxel {
    float sdf = 0.f;
    std::uint8_t weight = 0;
    std::uint8_t r = 0, g = 0, b = 0;
};
static_assert(sizeof(Voxel) == 8);

struct VoxelBlock {
    Vec3i coord{};
    std::vector<Voxel> voxels;  // 512, x fastest
};

struct SdfSample {
    double value = 0.0;
    bool valid = false;
};
struct SdfGradientSample {
    double value = 0.0;
    Vec3 gradient{};
    bool valid = false;
};

struct Mesh {  // mesh.hpp:14-18
    std::vector<Vec3f> vertices;
    std::vector<Rgb8> colors;
    std::vector<Vec3i> faces;
};

// Voxel access follows the reference: FindBlock returns a block pointer and
// VoxelHandle a (const or mutable) voxel pointer (tsdf_volume.cpp:59-91).
// The voxels live on the GPU, so the host layer keeps a lazy mirror of the
// bricks a caller touches: a brick is fetched with one hash probe
// (rf_volume_find_block) on first access, writes through a mutable handle
// mark it dirty, and every GPU operation on the volume first writes dirty
// bricks back (rf_volume_write_block) and then invalidates the mirror. A
// pointer stays valid (the brick's storage is never freed while the volume
// lives); after a GPU operation its contents are refreshed by the next
// FindBlock / VoxelHandle of that brick.
class TsdfVolume {
  public:
    explicit TsdfVolume(VolumeConfig config, int device = 0) : config_(config), owned_(true) {
        config_.Validate();
        const rf_volume_config c = config_.c();
        Check(rf_volume_create(&c, device, &h_));
    }
    ~TsdfVolume() {
        if (owned_ && h_) rf_volume_destroy(h_);
    }
    TsdfVolume(const TsdfVolume&) = delete;
    TsdfVolume& operator=(const TsdfVolume&) = delete;
    TsdfVolume(TsdfVolume&& o) noexcept
        : config_(o.config_), h_(o.h_), owned_(o.owned_), mirror_(std::move(o.mirror_)), generation_(o.generation_) {
        o.h_ = nullptr;
    }

    const VolumeConfig& config() const { return config_; }
    rf_volume* handle() const { return h_; }

    std::size_t num_blocks() const {
        std::uint64_t n = 0;
        Check(rf_volume_num_blocks(h_, &n));
        return n;
    }

    void AllocateForFrame(const DepthImage& depth, const CameraIntrinsics& k, const Pose& camera_to_world,
                          const PixelMask* mask = nullptr) {
        detail::RequireSize(depth, k);
        Sync();
        const rf_frame f = detail::ToC(depth, k);
        Check(rf_volume_allocate_for_frame(h_, &f, camera_to_world.data(), detail::MaskPtr(mask, k.width, k.height)));
    }
    void Integrate(const Frame& frame, const Pose& camera_to_world, const PixelMask* mask = nullptr,
                   int /*threads*/ = 1) {
        if (!frame.SizesConsistent() && !(frame.color.Empty() && frame.depth.SameSize(frame.intrinsics.width,
                                                                                      frame.intrinsics.height)))
            throw std::invalid_argument("frame sizes are inconsistent");
        Sync();
        const rf_frame f = detail::ToC(frame);
        Check(rf_volume_integrate(h_, &f, camera_to_world.data(),
                                  detail::MaskPtr(mask, frame.intrinsics.width, frame.intrinsics.height)));
    }
    void CarveFreeSpace(const DepthImage& depth, const CameraIntrinsics& k, const Pose& camera_to_world,
                        int /*threads*/ = 1) {
        detail::RequireSize(depth, k);
        Sync();
        const rf_frame f = detail::ToC(depth, k);
        Check(rf_volume_carve(h_, &f, camera_to_world.data()));
    }

    // Batched sampling (one launch for all points); single-point forms below.
    std::vector<SdfGradientSample> Sample(int mode, const std::vector<Vec3>& points) const {
        Sync();
        const std::size_t n = points.size();
        std::vector<double> val(n), grad(3 * n);
        std::vector<std::uint8_t> ok(n);
        if (n) Check(rf_volume_sample(h_, mode, points[0].data(), n, val.data(), grad.data(), ok.data()));
        std::vector<SdfGradientSample> out(n);
        for (std::size_t i = 0; i < n; ++i) {
            out[i].value = val[i];
            out[i].gradient = {grad[3 * i], grad[3 * i + 1], grad[3 * i + 2]};
            out[i].valid = ok[i] != 0;
        }
        return out;
    }
    SdfSample SampleSdf(const Vec3& p) const { return Value(0, p); }
    SdfSample SampleIntensity(const Vec3& p) const { return Value(1, p); }
    SdfGradientSample SampleSdfWithGradient(const Vec3& p) const { return Sample(2, {p})[0]; }
    SdfGradientSample SampleIntensityWithGradient(const Vec3& p) const { return Sample(3, {p})[0]; }
    SdfGradientSample SampleSdfGradient(const Vec3& p) const { return Sample(4, {p})[0]; }

    // FindBlock (tsdf_volume.cpp:59-62): nullptr when the block is not allocated.
    const VoxelBlock* FindBlock(const Vec3i& block_coord) const {
        const Mirror* m = Fetch(block_coord);
        return m ? &m->block : nullptr;
    }
    // VoxelHandle (tsdf_volume.cpp:79-91): nullptr when the voxel's block is not allocated.
    const Voxel* VoxelHandle(const Vec3i& voxel) const {
        Mirror* m = Fetch(BlockOf(voxel));
        return m ? &m->block.voxels[LocalIndex(voxel)] : nullptr;
    }
    Voxel* VoxelHandle(const Vec3i& voxel) {
        Mirror* m = Fetch(BlockOf(voxel));
        if (!m) return nullptr;
        m->dirty = true;  // written back before the next GPU operation
        return &m->block.voxels[LocalIndex(voxel)];
    }
    bool SetVoxel(const Vec3i& voxel, const Voxel& value) {
        Voxel* v = VoxelHandle(voxel);
        if (!v) return false;
        *v = value;
        return true;
    }
    Vec3 VoxelCenter(const Vec3i& v) const {
        return {(v[0] + 0.5) * config_.voxel_size, (v[1] + 0.5) * config_.voxel_size,
                (v[2] + 0.5) * config_.voxel_size};
    }
    double block_extent() const { return config_.block_side * config_.voxel_size; }

    bool AllocateBlock(const Vec3i& block_coord) {
        Sync();
        std::int32_t created = 0;
        Check(rf_volume_allocate_blocks(h_, block_coord.data(), 1, &created));
        return created == 1;
    }
    // blocks() in allocation order (a device -> host copy).
    std::vector<VoxelBlock> blocks() const {
        Sync();
        std::uint64_t n = 0;
        Check(rf_volume_export_blocks(h_, nullptr, nullptr, 0, &n));
        std::vector<std::int32_t> c(3 * n);
        std::vector<Voxel> v(n * 512);
        if (n)
            Check(rf_volume_export_blocks(h_, c.data(), reinterpret_cast<std::uint8_t*>(v.data()), n, &n));
        std::vector<VoxelBlock> out(n);
        for (std::size_t i = 0; i < n; ++i) {
            out[i].coord = {c[3 * i], c[3 * i + 1], c[3 * i + 2]};
            out[i].voxels.assign(v.begin() + i * 512, v.begin() + (i + 1) * 512);
        }
        return out;
    }

    void Save(const std::string& path) const {
        Sync();
        Check(rf_volume_save(h_, path.c_str()));
    }
    static TsdfVolume Load(const std::string& path, int device = 0) {
        rf_volume* h = nullptr;
        Check(rf_volume_load(path.c_str(), device, &h));
        return TsdfVolume(h, true);
    }
    static TsdfVolume Borrow(rf_volume* h) { return TsdfVolume(h, false); }

    // Writes back bricks modified through mutable VoxelHandles and invalidates
    // the mirror; every GPU operation on the volume calls it first.
    void Sync() const {
        for (auto& [coord, m] : mirror_) {
            if (!m->dirty) continue;
            std::int32_t found = 0;
            Check(rf_volume_write_block(h_, coord.data(), reinterpret_cast<const std::uint8_t*>(m->block.voxels.data()),
                                        &found));
            m->dirty = false;
        }
        ++generation_;
    }

  private:
    struct Mirror {
        VoxelBlock block;
        bool dirty = false;
        bool present = false;
        std::uint64_t generation = 0;
    };
    TsdfVolume(rf_volume* h, bool owned) : h_(h), owned_(owned) {
        rf_volume_config c{};
        Check(rf_volume_get_config(h_, &c));  // a loaded or borrowed volume reports its own config
        config_.voxel_size = c.voxel_size;
        config_.truncation = c.truncation;
        config_.block_side = c.block_side;
        config_.max_weight = c.max_weight;
        config_.carve_weight = c.carve_weight;
        config_.min_depth = c.min_depth;
        config_.max_depth = c.max_depth;
        config_.carve_clip = c.carve_clip;
        config_.max_blocks = c.max_blocks;
        config_.hash_capacity = c.hash_capacity;
    }
    static int FloorDiv8(int a) { return a >= 0 ? a / 8 : -((-a + 7) / 8); }  // FloorDiv (tsdf_volume.hpp:136-140)
    static Vec3i BlockOf(const Vec3i& v) { return {FloorDiv8(v[0]), FloorDiv8(v[1]), FloorDiv8(v[2])}; }
    static std::size_t LocalIndex(const Vec3i& v) {
        const Vec3i b = BlockOf(v);
        return (std::size_t(v[2] - 8 * b[2]) * 8 + std::size_t(v[1] - 8 * b[1])) * 8 + std::size_t(v[0] - 8 * b[0]);
    }
    Mirror* Fetch(const Vec3i& bc) const {
        const std::array<int, 3> key{bc[0], bc[1], bc[2]};
        auto it = mirror_.find(key);
        if (it != mirror_.end() && it->second->generation == generation_)
            return it->second->present ? it->second.get() : nullptr;
        std::vector<Voxel> vox(512);
        std::int32_t found = 0;
        Check(rf_volume_find_block(h_, bc.data(), reinterpret_cast<std::uint8_t*>(vox.data()), &found));
        if (it == mirror_.end()) it = mirror_.emplace(key, std::make_unique<Mirror>()).first;
        Mirror& m = *it->second;
        m.generation = generation_;
        m.present = found != 0;  // absence is cached too, until the next GPU operation
        if (!found) return nullptr;
        m.block.coord = bc;
        if (m.block.voxels.size() != 512) m.block.voxels.resize(512);
        std::memcpy(m.block.voxels.data(), vox.data(), 512 * sizeof(Voxel));  // in place: handed-out pointers stay valid
        m.dirty = false;
        return &m;
    }
    SdfSample Value(int mode, const Vec3& p) const {
        const SdfGradientSample s = Sample(mode, {p})[0];
        return SdfSample{s.value, s.valid};
    }
    VolumeConfig config_;
    rf_volume* h_ = nullptr;
    bool owned_ = false;
    mutable std::map<std::array<int, 3>, std::unique_ptr<Mirror>> mirror_;
    mutable std::uint64_t generation_ = 1;
};

// ---------------------------------------------------------------- registration (registration.hpp:13-85)
struct RegistrationConfig {
    double color_weight = 0.025;
    int pyramid_levels = 3, max_iterations = 20;
    double lm_lambda_init = 1e-4, lm_lambda_up = 10.0, lm_lambda_down = 2.0, convergence_eps = 1e-5;
    int min_valid_residuals = 100, threads = 1;
    double huber_depth = 0.0, huber_color = 0.0;  // extension, off by default (see rf_registration_config)
    rf_registration_config c() const {
        return rf_registration_config{color_weight,   pyramid_levels, max_iterations, lm_lambda_init,
                                      lm_lambda_up,   lm_lambda_down, convergence_eps, min_valid_residuals,
                                      threads,        huber_depth,    huber_color};
    }
};

struct ResidualImage {
    Image<float> squared;
    PixelMask valid;
};

struct LinearizeResult {
#ifdef REFUSION_B200_EIGEN
    Eigen::Matrix<double, 6, 6> H = Eigen::Matrix<double, 6, 6>::Zero();
    Eigen::Matrix<double, 6, 1> b = Eigen::Matrix<double, 6, 1>::Zero();
#else
    std::array<double, 36> H{};  // row-major 6x6
    std::array<double, 6> b{};
#endif
    double depth_error = 0.0, color_error = 0.0, error = 0.0;
    std::size_t valid_count = 0;
    bool degenerate = false;
};

struct RegistrationResult {
    Pose pose = Pose::Identity();
    bool converged = false;
    int iterations = 0;
    std::size_t valid_residuals = 0;
    double final_error = 0.0;
    ResidualImage residuals;
};

using IntensityImage = Image<float>;

struct PyramidLevel {  // registration.hpp:32-37
    CameraIntrinsics intrinsics;
    DepthImage depth;
    IntensityImage intensity;  // empty when the frame has no color
    PixelMask mask;            // empty when no pixels are excluded
};

// BuildPyramid (registration.hpp:42): level 0 is the input, each level halves
// the previous one (closest valid depth, mean intensity, any-of mask).
inline std::vector<PyramidLevel> BuildPyramid(const Frame& frame, const PixelMask* mask, int levels, int device = 0) {
    if (levels < 1) throw std::invalid_argument("pyramid needs at least one level");
    const int w = frame.intrinsics.width, h = frame.intrinsics.height;
    std::size_t total = 0;
    for (int l = 0; l < levels; ++l) total += std::size_t(w >> l) * std::size_t(h >> l);
    const bool color = !frame.color.Empty();
    const std::uint8_t* m = detail::MaskPtr(mask, w, h);
    std::vector<float> depth(total), inten(color ? total : 0);
    std::vector<std::uint8_t> mout(m ? total : 0);
    std::vector<rf_intrinsics> k(levels);
    const rf_frame f = detail::ToC(frame);
    Check(rf_build_pyramid(&f, m, levels, device, depth.data(), color ? inten.data() : nullptr,
                           m ? mout.data() : nullptr, k.data()));
    std::vector<PyramidLevel> out(levels);
    std::size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        const int lw = w >> l, lh = h >> l;
        const std::size_t n = std::size_t(lw) * lh;
        PyramidLevel& L = out[l];
        L.intrinsics = frame.intrinsics.Scaled(l);
        L.depth = DepthImage(lw, lh);
        std::memcpy(L.depth.data(), depth.data() + off, n * sizeof(float));
        if (color) {
            L.intensity = IntensityImage(lw, lh);
            std::memcpy(L.intensity.data(), inten.data() + off, n * sizeof(float));
        }
        if (m) {
            L.mask = PixelMask(lw, lh);
            std::memcpy(L.mask.data(), mout.data() + off, n);
        }
        off += n;
    }
    return out;
}

inline LinearizeResult Linearize(const TsdfVolume& volume, const Frame& frame, const Pose& pose,
                                 const RegistrationConfig& config, const PixelMask* mask = nullptr) {
    volume.Sync();
    const rf_frame f = detail::ToC(frame);
    const rf_registration_config c = config.c();
    rf_linearize_result r{};
    Check(rf_linearize(volume.handle(), &f, pose.data(), &c,
                       detail::MaskPtr(mask, frame.intrinsics.width, frame.intrinsics.height), &r));
    LinearizeResult out;
    for (int i = 0; i < 6; ++i) {
        for (int j = 0; j < 6; ++j) {
#ifdef REFUSION_B200_EIGEN
            out.H(i, j) = r.H[6 * i + j];
#else
            out.H[6 * i + j] = r.H[6 * i + j];
#endif
        }
        out.b[i] = r.b[i];
    }
    out.depth_error = r.depth_error;
    out.color_error = r.color_error;
    out.error = r.error;
    out.valid_count = r.valid_count;
    out.degenerate = r.degenerate != 0;
    return out;
}

inline std::pair<double, ResidualImage> EvaluateDepthError(const TsdfVolume& volume, const Frame& frame,
                                                           const Pose& pose, const PixelMask* mask = nullptr,
                                                           int /*threads*/ = 1) {
    volume.Sync();
    const int w = frame.intrinsics.width, h = frame.intrinsics.height;
    const rf_frame f = detail::ToC(frame);
    ResidualImage res{Image<float>(w, h), PixelMask(w, h)};
    double e = 0.0;
    Check(rf_evaluate_depth_error(volume.handle(), &f, pose.data(), detail::MaskPtr(mask, w, h), &e,
                                  res.squared.data(), res.valid.data()));
    return {e, std::move(res)};
}

inline double EvaluateColorError(const TsdfVolume& volume, const Frame& frame, const Pose& pose,
                                 const PixelMask* mask = nullptr, int /*threads*/ = 1) {
    volume.Sync();
    const rf_frame f = detail::ToC(frame);
    double e = 0.0;
    Check(rf_evaluate_color_error(volume.handle(), &f, pose.data(),
                                  detail::MaskPtr(mask, frame.intrinsics.width, frame.intrinsics.height), &e));
    return e;
}

inline RegistrationResult Register(const TsdfVolume& volume, const Frame& frame, const Pose& initial_pose,
                                   const PixelMask* mask, const RegistrationConfig& config) {
    volume.Sync();
    const int w = frame.intrinsics.width, h = frame.intrinsics.height;
    const rf_frame f = detail::ToC(frame);
    const rf_registration_config c = config.c();
    rf_registration_result r{};
    RegistrationResult out;
    out.residuals = ResidualImage{Image<float>(w, h), PixelMask(w, h)};
    Check(rf_register(volume.handle(), &f, initial_pose.data(), detail::MaskPtr(mask, w, h), &c, &r,
                      out.residuals.squared.data(), out.residuals.valid.data()));
    out.pose = Pose::FromArray(r.pose);
    out.converged = r.converged != 0;
    out.iterations = r.iterations;
    out.valid_residuals = r.valid_residuals;
    out.final_error = r.final_error;
    return out;
}

// ---------------------------------------------------------------- dynamics mask (dynamics_mask.hpp:10-41)
struct MaskConfig {
    double gamma = 0.5, truncation = 0.1, theta = 0.007;
    int erode_radius = 2, dilate_radius = 2, connectivity = 4;
    double free_space = 0.0;  // extension, off by default (see rf_mask_config)
    rf_mask_config c() const {
        return rf_mask_config{gamma, truncation, theta, erode_radius, dilate_radius, connectivity, 0, free_space};
    }
};

namespace detail {
inline PixelMask MaskStages(const float* sq, const std::uint8_t* valid, const float* depth, int w, int h,
                            const MaskConfig& config, int stages, int device = 0) {
    PixelMask out(w, h);
    const rf_mask_config c = config.c();
    std::uint64_t n = 0;
    Check(rf_mask_stages(sq, valid, depth, w, h, &c, stages, device, out.data(), &n));
    return out;
}
}  // namespace detail

inline PixelMask ThresholdResiduals(const ResidualImage& r, const MaskConfig& config) {
    return detail::MaskStages(r.squared.data(), r.valid.data(), nullptr, r.squared.width(), r.squared.height(),
                              config, 1);
}
inline PixelMask Erode(const PixelMask& mask, int radius) {
    MaskConfig c;
    c.erode_radius = radius;
    return detail::MaskStages(nullptr, mask.data(), nullptr, mask.width(), mask.height(), c, 2);
}
inline PixelMask Dilate(const PixelMask& mask, int radius) {
    MaskConfig c;
    c.dilate_radius = radius;
    return detail::MaskStages(nullptr, mask.data(), nullptr, mask.width(), mask.height(), c, 8);
}
inline PixelMask FloodfillDepth(const PixelMask& seeds, const DepthImage& depth, double theta, int connectivity) {
    MaskConfig c;
    c.theta = theta;
    c.connectivity = connectivity;
    return detail::MaskStages(nullptr, seeds.data(), depth.data(), seeds.width(), seeds.height(), c, 4);
}
inline PixelMask BuildMask(const ResidualImage& r, const DepthImage& depth, const MaskConfig& config) {
    return detail::MaskStages(r.squared.data(), r.valid.data(), depth.data(), depth.width(), depth.height(), config,
                              15);
}
// ResidualHistogram (dynamics_mask.hpp:38-41): counts of the valid squared
// residuals in `bins` equal bins over [0, max_value], values beyond it in the
// last bin. A diagnostic over a host image, off the per-frame path: computed here.
inline std::vector<std::size_t> ResidualHistogram(const ResidualImage& r, int bins, double max_value) {
    if (bins < 1 || !(max_value > 0)) throw std::invalid_argument("bad histogram shape");
    std::vector<std::size_t> hist(static_cast<std::size_t>(bins), 0);
    const std::size_t n = std::size_t(r.squared.width()) * r.squared.height();
    for (std::size_t i = 0; i < n; ++i) {
        if (!r.valid.data()[i]) continue;
        const int b = static_cast<int>(double(r.squared.data()[i]) / max_value * bins);
        ++hist[static_cast<std::size_t>(b < bins - 1 ? b : bins - 1)];
    }
    return hist;
}

// ---------------------------------------------------------------- raycast / mesh
// Ray-march of RenderVirtualDepth (depth_refinement.cpp:32-79) over `volume`.
inline DepthImage Raycast(const TsdfVolume& volume, const Pose& view_pose, const CameraIntrinsics& k,
                          int bisection_iterations = 8) {
    volume.Sync();
    DepthImage out(k.width, k.height);
    const rf_intrinsics ck = k.c();
    Check(rf_raycast(volume.handle(), view_pose.data(), &ck, bisection_iterations, out.data()));
    return out;
}

inline Mesh ExtractMesh(const TsdfVolume& volume, int min_weight = 2, int /*threads*/ = 1) {
    volume.Sync();
    rf_mesh* m = nullptr;
    Check(rf_volume_extract_mesh(volume.handle(), min_weight, &m));
    Mesh out;
    std::uint64_t nv = 0, nf = 0;
    rf_status s = rf_mesh_counts(m, &nv, &nf);
    if (s == RF_OK) {
        out.vertices.resize(nv);
        out.colors.resize(nv);
        out.faces.resize(nf);
        s = rf_mesh_copy(m, out.vertices.empty() ? nullptr : out.vertices[0].data(),
                         out.colors.empty() ? nullptr : &out.colors[0].r,
                         out.faces.empty() ? nullptr : out.faces[0].data());
    }
    rf_mesh_destroy(m);
    Check(s);
    return out;
}

// WritePly / ReadPly / WritePointCloudPly (mesh.hpp:27-32): binary little-endian
// PLY, float x/y/z, uchar red/green/blue per vertex when the mesh has colours,
// uchar-counted int index lists. Host-side I/O of a host mesh (the device mesh
// writes the same bytes through rf_mesh_write_ply).
namespace detail {
inline void WritePlyFile(const std::string& path, const std::vector<Vec3f>& v, const std::vector<Rgb8>* colors,
                         const std::vector<Vec3i>* faces) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open for writing: " + path);
    std::string h = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(v.size()) +
                    "\nproperty float x\nproperty float y\nproperty float z\n";
    if (colors) h += "property uchar red\nproperty uchar green\nproperty uchar blue\n";
    if (faces) h += "element face " + std::to_string(faces->size()) + "\nproperty list uchar int vertex_indices\n";
    h += "end_header\n";
    bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size();
    for (std::size_t i = 0; ok && i < v.size(); ++i) {
        const float p[3] = {v[i][0], v[i][1], v[i][2]};
        ok = std::fwrite(p, 4, 3, f) == 3 && (!colors || std::fwrite(&(*colors)[i].r, 1, 3, f) == 3);
    }
    for (std::size_t i = 0; ok && faces && i < faces->size(); ++i) {
        const unsigned char n = 3;
        const std::int32_t idx[3] = {(*faces)[i][0], (*faces)[i][1], (*faces)[i][2]};
        ok = std::fwrite(&n, 1, 1, f) == 1 && std::fwrite(idx, 4, 3, f) == 3;
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write failed: " + path);
}
}  // namespace detail

inline void WritePly(const std::string& path, const Mesh& mesh) {
    const bool colored = !mesh.vertices.empty() && mesh.colors.size() == mesh.vertices.size();
    detail::WritePlyFile(path, mesh.vertices, colored ? &mesh.colors : nullptr, &mesh.faces);
}
inline void WritePointCloudPly(const std::string& path, const std::vector<Vec3f>& points) {
    detail::WritePlyFile(path, points, nullptr, nullptr);
}
inline Mesh ReadPly(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    auto fail = [&](const std::string& why) {
        std::fclose(f);
        return std::runtime_error("malformed PLY " + path + ": " + why);
    };
    char line[256];
    auto next = [&]() -> std::string {
        if (!std::fgets(line, sizeof(line), f)) return std::string("\x01");  // end of file marker
        std::string s(line);
        while (!s.empty() && (s.back() == '\n' || s.back() == '\r')) s.pop_back();
        return s;
    };
    if (next() != "ply") throw fail("missing magic");
    if (next() != "format binary_little_endian 1.0") throw fail("not binary little endian");
    std::size_t nv = 0, nf = 0;
    int vprops = 0;
    bool colored = false, faces = false, in_vertex = false;
    for (;;) {
        const std::string s = next();
        if (s == "\x01") throw fail("no end_header");
        if (s == "end_header") break;
        if (s.rfind("element vertex ", 0) == 0) {
            nv = std::stoull(s.substr(15));
            in_vertex = true;
        } else if (s.rfind("element face ", 0) == 0) {
            nf = std::stoull(s.substr(13));
            faces = true;
            in_vertex = false;
        } else if (s.rfind("property ", 0) == 0) {
            if (in_vertex) {
                if (s == "property uchar red") colored = true;
                ++vprops;
            } else if (faces && s != "property list uchar int vertex_indices") {
                throw fail("unsupported face property");
            }
        } else if (s.rfind("comment", 0) != 0) {
            throw fail("unexpected header line");
        }
    }
    if (vprops != (colored ? 6 : 3)) throw fail("unsupported vertex properties");
    Mesh m;
    m.vertices.resize(nv);
    if (colored) m.colors.resize(nv);
    for (std::size_t i = 0; i < nv; ++i) {
        float p[3];
        if (std::fread(p, 4, 3, f) != 3) throw fail("truncated vertices");
        m.vertices[i] = Vec3f{p[0], p[1], p[2]};
        if (colored && std::fread(&m.colors[i].r, 1, 3, f) != 3) throw fail("truncated colours");
    }
    m.faces.resize(nf);
    for (std::size_t i = 0; i < nf; ++i) {
        unsigned char n = 0;
        std::int32_t idx[3];
        if (std::fread(&n, 1, 1, f) != 1 || n != 3 || std::fread(idx, 4, 3, f) != 3) throw fail("bad face");
        m.faces[i] = Vec3i{idx[0], idx[1], idx[2]};
    }
    std::fclose(f);
    return m;
}

// ---------------------------------------------------------------- pipeline (pipeline.hpp:18-96, config.hpp:12-24)
struct RefinementConfig {  // depth_refinement.hpp:12-17
    bool enabled = true;
    int window = 10;
    double far_value = 8.0;
    int bisection_iterations = 8;
};

// WindowEntry / FrameWindow (depth_refinement.hpp:19-44): the host form of the
// refinement window. Pipeline keeps its own window on the device; this one is
// for callers that drive RenderVirtualDepth themselves.
struct WindowEntry {
    Frame frame;
    Pose pose = Pose::Identity();
    PixelMask mask;  // may be empty
};
class FrameWindow {
  public:
    explicit FrameWindow(std::size_t capacity) : capacity_(capacity) {}
    std::size_t capacity() const { return capacity_; }
    std::size_t size() const { return entries_.size(); }
    bool Empty() const { return entries_.empty(); }
    bool Full() const { return entries_.size() >= capacity_; }
    void Push(WindowEntry entry) {  // depth_refinement.cpp:10-13
        if (Full()) throw std::logic_error("frame window is full");
        entries_.push_back(std::move(entry));
    }
    WindowEntry PopFront() {  // depth_refinement.cpp:15-20
        if (entries_.empty()) throw std::logic_error("frame window is empty");
        WindowEntry e = std::move(entries_.front());
        entries_.pop_front();
        return e;
    }
    const std::deque<WindowEntry>& entries() const { return entries_; }

  private:
    std::size_t capacity_;
    std::deque<WindowEntry> entries_;
};

// RenderVirtualDepth (depth_refinement.cpp:22-80): the window fused into a
// throw-away volume on the GPU and ray-marched from view_pose
// (rf_render_virtual_depth: all entries uploaded and fused in one pass when
// they share a size; a mixed-size window goes through a TsdfVolume entry by
// entry). An empty window has no surface: all pixels invalid.
inline DepthImage RenderVirtualDepth(const FrameWindow& window, const Pose& view_pose, const CameraIntrinsics& k,
                                     const VolumeConfig& volume_config, const RefinementConfig& config,
                                     int /*threads*/ = 1) {
    volume_config.Validate();
    DepthImage out(k.width, k.height, 0.f);
    const auto& es = window.entries();
    if (es.empty()) return out;
    bool same = true;
    for (const WindowEntry& e : es) {
        if (!e.frame.depth.SameSize(e.frame.intrinsics.width, e.frame.intrinsics.height))
            throw std::invalid_argument("depth size does not match the intrinsics");
        same = same && e.frame.intrinsics.width == es.front().frame.intrinsics.width &&
               e.frame.intrinsics.height == es.front().frame.intrinsics.height;
    }
    if (!same) {
        TsdfVolume temp(volume_config);
        for (const WindowEntry& e : es) {
            const PixelMask* m = e.mask.Empty() ? nullptr : &e.mask;
            temp.AllocateForFrame(e.frame.depth, e.frame.intrinsics, e.pose, m);
            temp.Integrate(e.frame, e.pose, m);
        }
        return Raycast(temp, view_pose, k, config.bisection_iterations);
    }
    std::vector<rf_frame> frames;
    std::vector<double> poses;
    std::vector<const std::uint8_t*> masks;
    for (const WindowEntry& e : es) {
        frames.push_back(detail::ToC(e.frame));
        poses.insert(poses.end(), e.pose.data(), e.pose.data() + 12);
        masks.push_back(detail::MaskPtr(&e.mask, e.frame.intrinsics.width, e.frame.intrinsics.height));
    }
    const rf_intrinsics ck = k.c();
    const rf_volume_config vc = volume_config.c();
    Check(rf_render_virtual_depth(frames.data(), poses.data(), masks.data(), std::int32_t(frames.size()),
                                  view_pose.data(), &ck, &vc, config.bisection_iterations, config.far_value, 0,
                                  out.data(), nullptr));
    return out;
}

// RefineDepth (depth_refinement.cpp:82-93): raw where valid, else virtual
// where valid, else far_value. Host-side: one pass over one image.
inline DepthImage RefineDepth(const DepthImage& raw, const DepthImage& virtual_depth, double far_value) {
    if (!raw.SameSize(virtual_depth)) throw std::invalid_argument("depth size mismatch");
    DepthImage out = raw;
    for (int y = 0; y < out.height(); ++y)
        for (int x = 0; x < out.width(); ++x)
            if (!DepthValid(out(x, y)))
                out(x, y) = DepthValid(virtual_depth(x, y)) ? virtual_depth(x, y) : static_cast<float>(far_value);
    return out;
}

struct PipelineConfig {
    VolumeConfig volume;
    RegistrationConfig registration;
    MaskConfig mask;
    RefinementConfig refinement;
    bool dynamics_enabled = true;
    int threads = 1;
    double max_dt = 0.02;

    void Sync() {  // config.cpp: the mask threshold follows the volume truncation
        mask.truncation = volume.truncation;
        volume.Validate();
    }
    rf_pipeline_config c() const {
        rf_pipeline_config r{};
        r.volume = volume.c();
        r.registration = registration.c();
        r.mask = mask.c();
        r.refine_enabled = refinement.enabled ? 1 : 0;
        r.refine_window = refinement.window;
        r.far_value = refinement.far_value;
        r.bisection_iterations = refinement.bisection_iterations;
        r.dynamics_enabled = dynamics_enabled ? 1 : 0;
        r.threads = threads;
        return r;
    }
};

struct FrameStats {
    std::size_t frame_index = 0;
    double timestamp = 0.0;
    bool tracking_lost = false, converged = false;
    int registrations = 0, iterations = 0;
    std::size_t valid_residuals = 0, masked_pixels = 0;
    double final_error = 0.0, runtime_ms = 0.0;
};

struct FrameDebug {
    std::size_t frame_index = 0;
    double timestamp = 0.0;
    const PixelMask* mask = nullptr;
    const ResidualImage* residuals = nullptr;
    const DepthImage* virtual_depth = nullptr;
    const DepthImage* refined_depth = nullptr;
};

struct TrajectoryEntry {
    double timestamp = 0.0;
    Pose pose;
};
using Trajectory = std::vector<TrajectoryEntry>;

class Pipeline {
  public:
    explicit Pipeline(PipelineConfig config, int device = 0) : config_(std::move(config)) {
        config_.Sync();
        const rf_pipeline_config c = config_.c();
        Check(rf_pipeline_create(&c, device, &h_));
        rf_volume* v = nullptr;
        Check(rf_pipeline_volume(h_, &v));
        volume_.emplace(TsdfVolume::Borrow(v));
    }
    ~Pipeline() {
        volume_.reset();
        if (h_) rf_pipeline_destroy(h_);
    }
    Pipeline(const Pipeline&) = delete;
    Pipeline& operator=(const Pipeline&) = delete;
    Pipeline(Pipeline&& o) noexcept
        : config_(std::move(o.config_)), h_(o.h_), volume_(std::move(o.volume_)), trajectory_(std::move(o.trajectory_)),
          stats_(std::move(o.stats_)), debug_sink_(std::move(o.debug_sink_)),
          last_refinement_emitted_(o.last_refinement_emitted_), last_w_(o.last_w_), last_h_(o.last_h_) {
        o.h_ = nullptr;
        o.volume_.reset();
    }

    FrameStats ProcessFrame(const Frame& frame) {
        if (!frame.depth.SameSize(frame.intrinsics.width, frame.intrinsics.height) ||
            (!frame.color.Empty() && !frame.color.SameSize(frame.depth)))
            throw std::invalid_argument("frame sizes are inconsistent");
        volume_->Sync();
        const rf_frame f = detail::ToC(frame);
        rf_frame_stats s{};
        double pose[12];
        Check(rf_pipeline_process_frame(h_, &f, &s, pose));
        const FrameStats out = Record(frame.timestamp, s, pose);
        if (debug_sink_) EmitDebug(frame, out);
        return out;
    }
    // ProcessFrame over several frames with their GPU work enqueued back to
    // back (rf_pipeline_process_frames); per-frame debug records need
    // ProcessFrame, so with a debug sink this is a plain loop.
    std::vector<FrameStats> ProcessFrames(const std::vector<Frame>& frames) {
        std::vector<FrameStats> out;
        if (debug_sink_) {
            for (const Frame& f : frames) out.push_back(ProcessFrame(f));
            return out;
        }
        std::vector<rf_frame> cf;
        for (const Frame& f : frames) {
            if (!f.depth.SameSize(f.intrinsics.width, f.intrinsics.height) ||
                (!f.color.Empty() && !f.color.SameSize(f.depth)))
                throw std::invalid_argument("frame sizes are inconsistent");
            cf.push_back(detail::ToC(f));
        }
        std::vector<rf_frame_stats> st(frames.size());
        std::vector<double> poses(12 * frames.size());
        volume_->Sync();
        Check(rf_pipeline_process_frames(h_, cf.data(), cf.size(), st.data(), poses.data()));
        for (std::size_t i = 0; i < frames.size(); ++i)
            out.push_back(Record(frames[i].timestamp, st[i], poses.data() + 12 * i));
        return out;
    }
    void Finalize() {  // pipeline.cpp:133-135 (IntegrateFront until the window is empty)
        volume_->Sync();
        if (!debug_sink_) {
            Check(rf_pipeline_finalize(h_));
            return;
        }
        while (window_size() > 0) {  // one IntegrateFront per call so each gets its debug record
            Check(rf_pipeline_finalize_one(h_));
            EmitRefinement();
        }
    }

    const Trajectory& trajectory() const { return trajectory_; }
    const TsdfVolume& volume() const { return *volume_; }
    const std::vector<FrameStats>& stats() const { return stats_; }
    const PipelineConfig& config() const { return config_; }
    std::size_t tracking_losses() const {
        std::uint64_t n = 0;
        Check(rf_pipeline_tracking_losses(h_, &n));
        return n;
    }
    // With a sink installed the refinement window also renders the full
    // virtual depth image (FrameDebug::virtual_depth), not only its holes.
    void set_debug_sink(std::function<void(const FrameDebug&)> sink) {
        debug_sink_ = std::move(sink);
        Check(rf_pipeline_set_debug_images(h_, debug_sink_ ? 1 : 0));
    }
    std::size_t window_size() const {
        std::uint64_t n = 0;
        Check(rf_pipeline_window_size(h_, &n));
        return n;
    }
    rf_pipeline* handle() const { return h_; }

  private:
    FrameStats Record(double timestamp, const rf_frame_stats& s, const double pose[12]) {
        FrameStats out;
        out.frame_index = s.frame_index;
        out.timestamp = s.timestamp;
        out.tracking_lost = s.tracking_lost != 0;
        out.converged = s.converged != 0;
        out.registrations = s.registrations;
        out.iterations = s.iterations;
        out.valid_residuals = s.valid_residuals;
        out.masked_pixels = s.masked_pixels;
        out.final_error = s.final_error;
        out.runtime_ms = s.runtime_ms;
        trajectory_.push_back(TrajectoryEntry{timestamp, Pose::FromArray(pose)});
        stats_.push_back(out);
        return out;
    }
    void EmitRefinement() {  // IntegrateFront's debug record (pipeline.cpp:45-54)
        std::int32_t has = 0;
        std::uint64_t index = 0;
        Check(rf_pipeline_last_refinement(h_, nullptr, nullptr, &index, &has));
        if (!has || index == last_refinement_emitted_) return;
        last_refinement_emitted_ = index;
        const int w = stats_.empty() ? 0 : last_w_, h = last_h_;
        DepthImage virt(w, h), refined(w, h);
        Check(rf_pipeline_last_refinement(h_, virt.data(), refined.data(), &index, &has));
        FrameDebug d;
        d.frame_index = index;
        d.timestamp = index < stats_.size() ? stats_[index].timestamp : 0.0;
        d.virtual_depth = &virt;
        d.refined_depth = &refined;
        debug_sink_(d);
    }
    void EmitDebug(const Frame& frame, const FrameStats& st) {
        last_w_ = frame.intrinsics.width;
        last_h_ = frame.intrinsics.height;
        if (config_.refinement.enabled) EmitRefinement();  // IntegrateFront runs before registration
        if (st.frame_index == 0 || st.tracking_lost) return;  // no registration record (pipeline.cpp:66-76, 122-127)
        const int w = frame.intrinsics.width, h = frame.intrinsics.height;
        FrameDebug d;
        d.frame_index = st.frame_index;
        d.timestamp = st.timestamp;
        PixelMask mask(w, h);
        std::int32_t has_mask = 0;
        Check(rf_pipeline_last_mask(h_, mask.data(), &has_mask));
        ResidualImage res{Image<float>(w, h), PixelMask(w, h)};
        Check(rf_pipeline_last_residuals(h_, res.squared.data(), res.valid.data()));
        d.residuals = &res;
        if (has_mask) d.mask = &mask;
        debug_sink_(d);
    }

    PipelineConfig config_;
    rf_pipeline* h_ = nullptr;
    std::optional<TsdfVolume> volume_;
    Trajectory trajectory_;
    std::vector<FrameStats> stats_;
    std::function<void(const FrameDebug&)> debug_sink_;
    std::uint64_t last_refinement_emitted_ = ~std::uint64_t(0);
    int last_w_ = 0, last_h_ = 0;
};

using FrameSource = std::function<std::optional<Frame>()>;
struct SequenceSummary {
    std::size_t frames = 0;
    std::size_t tracking_losses = 0;
};

// RunSequence (pipeline.cpp:137-145).
// Frames are pulled in batches of up to 64 and processed with their GPU work
// enqueued back to back (results identical to one ProcessFrame at a time).
inline SequenceSummary RunSequence(Pipeline& pipeline, const FrameSource& source) {
    SequenceSummary s;
    std::vector<Frame> batch;
    bool more = true;
    while (more) {
        batch.clear();
        while (batch.size() < 64) {
            std::optional<Frame> f = source();
            if (!f) {
                more = false;
                break;
            }
            batch.push_back(std::move(*f));
        }
        if (!batch.empty()) pipeline.ProcessFrames(batch);
        s.frames += batch.size();
    }
    pipeline.Finalize();
    s.tracking_losses = pipeline.tracking_losses();
    return s;
}

// ---------------------------------------------------------------- evaluation (evaluation.hpp:12-50)
struct AteResult {
    double rmse = 0.0;
    Pose alignment;  // rigid transform mapping estimated into ground truth
    std::size_t pairs = 0;
};

namespace detail {
inline void Flatten(const Trajectory& tr, std::vector<double>& ts, std::vector<double>& poses) {
    ts.resize(tr.size());
    poses.resize(12 * tr.size());
    for (std::size_t i = 0; i < tr.size(); ++i) {
        ts[i] = tr[i].timestamp;
        std::memcpy(poses.data() + 12 * i, tr[i].pose.data(), 12 * sizeof(double));
    }
}
}  // namespace detail

// AteRmse (evaluation.cpp:26-62); throws std::runtime_error below 3 pairs.
inline AteResult AteRmse(const Trajectory& estimated, const Trajectory& ground_truth, double max_dt = 0.02) {
    std::vector<double> et, ep, gt, gp;
    detail::Flatten(estimated, et, ep);
    detail::Flatten(ground_truth, gt, gp);
    AteResult r;
    std::uint64_t pairs = 0;
    Check(rf_ate_rmse(et.data(), ep.data(), et.size(), gt.data(), gp.data(), gt.size(), max_dt, &r.rmse,
                      r.alignment.data(), &pairs));
    r.pairs = static_cast<std::size_t>(pairs);
    return r;
}

struct RpeSample {
    double timestamp = 0.0;
    double translation_error = 0.0;  // meters over the delta interval
};

// RpeOverTime (evaluation.cpp:64-92)
inline std::vector<RpeSample> RpeOverTime(const Trajectory& estimated, const Trajectory& ground_truth,
                                          double delta = 1.0, double max_dt = 0.02) {
    std::vector<double> et, ep, gt, gp;
    detail::Flatten(estimated, et, ep);
    detail::Flatten(ground_truth, gt, gp);
    std::vector<double> ts(et.size() + 1), err(et.size() + 1);
    std::uint64_t n = 0;
    Check(rf_rpe_over_time(et.data(), ep.data(), et.size(), gt.data(), gp.data(), gt.size(), delta, max_dt,
                           ts.data(), err.data(), ts.size(), &n));
    std::vector<RpeSample> out(static_cast<std::size_t>(n));
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = {ts[i], err[i]};
    return out;
}

// NearestDistances (evaluation.cpp:203-217) on the GPU; `threads` is accepted and ignored.
inline std::vector<double> NearestDistances(const std::vector<Vec3f>& queries, const std::vector<Vec3f>& reference,
                                            int threads = 1, int device = 0) {
    (void)threads;
    std::vector<double> out(queries.size());
    Check(rf_nearest_distances(queries.empty() ? nullptr : queries[0].data(), queries.size(),
                               reference.empty() ? nullptr : reference[0].data(), reference.size(), RF_MEMORY_HOST,
                               device, out.data()));
    return out;
}

// DistanceCdf (evaluation.cpp:219-236)
inline std::vector<double> DistanceCdf(const std::vector<double>& distances, const std::vector<double>& bin_edges,
                                       int device = 0) {
    std::vector<double> cdf(bin_edges.size());
    Check(rf_distance_cdf(distances.data(), distances.size(), RF_MEMORY_HOST, device, bin_edges.data(),
                          bin_edges.size(), cdf.data()));
    return cdf;
}

}  // namespace tsdfslam_b200
