// GPU synthetic RGB-D renderer: the analytic scenes of
// synth.cpp:79-203 (plane / sphere / box, inside-out box rooms, checker
// albedo, keyframed dynamic objects) rendered one thread per pixel, so the
// bench can feed >= 1000 frames/s per GPU without a host bottleneck.
//
// Depth noise sigma = k*z^2 uses a counter-based generator (splitmix64 of
// seed, frame, pixel) + Box-Muller instead of std::mt19937 /
// std::normal_distribution: same distribution, not the same bytes. Parity
// runs therefore use oracle-rendered frames; this renderer only makes
// workloads.
#include <cstring>

#include "../../include/refusion_b200.h"
#include "rf_common.cuh"

namespace rfb {

struct SynthPrim {
    int shape, dynamic, checker, pad;
    double a[3], b[3];
    double cell;
    double w2o[12];  // world-to-object at this frame's time (R row-major, t)
    uint8_t primary[4], secondary[4];
};

constexpr int kMaxSynthPrims = 32;

struct SynthArgs {
    SynthPrim prims[kMaxSynthPrims];
    int nprims;
    Pose cam;
    Intr K;
    double noise, dropout;
    unsigned long long seed, frame;
    float* depth;
    uint8_t* rgb;
    uint8_t* labels;
};

__device__ __forceinline__ double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

__device__ double intersect(const SynthPrim& p, const double o[3], const double d[3]) {  // synth.cpp:79-122
    const double kMiss = __longlong_as_double(0x7ff0000000000000ll);
    const double kRayEps = 1e-6;
    if (p.shape == 0) {
        const double denom = dot3(p.b, d);
        if (fabs(denom) < 1e-12) return kMiss;
        const double am[3] = {p.a[0] - o[0], p.a[1] - o[1], p.a[2] - o[2]};
        const double t = dot3(p.b, am) / denom;
        return t > kRayEps ? t : kMiss;
    }
    if (p.shape == 1) {
        const double oc[3] = {o[0] - p.a[0], o[1] - p.a[1], o[2] - p.a[2]};
        const double a = dot3(d, d), hb = dot3(oc, d), c = dot3(oc, oc) - p.b[0] * p.b[0];
        const double disc = hb * hb - a * c;
        if (disc < 0) return kMiss;
        const double root = sqrt(disc);
        const double t0 = (-hb - root) / a;
        if (t0 > kRayEps) return t0;
        const double t1 = (-hb + root) / a;
        return t1 > kRayEps ? t1 : kMiss;
    }
    double tn = -kMiss, tf = kMiss;
    for (int i = 0; i < 3; ++i) {
        const double lo = p.a[i] - p.b[i], hi = p.a[i] + p.b[i];
        if (fabs(d[i]) < 1e-15) {
            if (o[i] < lo || o[i] > hi) return kMiss;
            continue;
        }
        double t0 = (lo - o[i]) / d[i], t1 = (hi - o[i]) / d[i];
        if (t0 > t1) {
            const double s = t0;
            t0 = t1;
            t1 = s;
        }
        tn = fmax(tn, t0);
        tf = fmin(tf, t1);
    }
    if (tn > tf || tf < kRayEps) return kMiss;
    return tn > kRayEps ? tn : tf;
}

__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double uniform01(unsigned long long x) { return (double(x >> 11) + 0.5) * 0x1.0p-53; }

__global__ void k_synth(const SynthArgs* __restrict__ A) {
    const SynthArgs& a = *A;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.K.w * a.K.h) return;
    const int u = i % a.K.w, v = i / a.K.w;
    const double dc[3] = {(double(u) - a.K.cx) / a.K.fx, (double(v) - a.K.cy) / a.K.fy, 1.0};
    double dir[3];
    for (int r = 0; r < 3; ++r) dir[r] = (a.cam.R[3 * r] * dc[0] + a.cam.R[3 * r + 1] * dc[1]) + a.cam.R[3 * r + 2] * dc[2];
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bi = -1;
    for (int k = 0; k < a.nprims; ++k) {
        const SynthPrim& p = a.prims[k];
        double o[3], d[3];
        for (int r = 0; r < 3; ++r) {
            o[r] = ((p.w2o[3 * r] * a.cam.t[0] + p.w2o[3 * r + 1] * a.cam.t[1]) + p.w2o[3 * r + 2] * a.cam.t[2]) + p.w2o[9 + r];
            d[r] = (p.w2o[3 * r] * dir[0] + p.w2o[3 * r + 1] * dir[1]) + p.w2o[3 * r + 2] * dir[2];
        }
        const double t = intersect(p, o, d);
        if (t < best) {
            best = t;
            bi = k;
        }
    }
    float depth = 0.f;
    uint8_t col[3] = {0, 0, 0}, label = 0;
    if (bi >= 0) {
        const SynthPrim& p = a.prims[bi];
        depth = float(best);
        label = p.dynamic ? 1 : 0;
        const uint8_t* c = p.primary;
        if (p.checker) {  // synth.cpp:124-132
            long parity = 0;
            const double w[3] = {a.cam.t[0] + best * dir[0], a.cam.t[1] + best * dir[1], a.cam.t[2] + best * dir[2]};
            double hit[3];
            for (int r = 0; r < 3; ++r)
                hit[r] = ((p.w2o[3 * r] * w[0] + p.w2o[3 * r + 1] * w[1]) + p.w2o[3 * r + 2] * w[2]) + p.w2o[9 + r];
            for (int r = 0; r < 3; ++r) parity += long(floor((hit[r] + 0.0123 * p.cell) / p.cell));
            if (parity & 1) c = p.secondary;
        }
        col[0] = c[0];
        col[1] = c[1];
        col[2] = c[2];
    }
    a.labels[i] = label;
    a.rgb[3 * i] = col[0];
    a.rgb[3 * i + 1] = col[1];
    a.rgb[3 * i + 2] = col[2];
    float out = 0.f;
    if (depth_valid(depth)) {
        const unsigned long long base = splitmix(a.seed ^ splitmix(a.frame * 0x100000001B3ull + (unsigned long long)i));
        bool dropped = a.dropout > 0.0 && uniform01(splitmix(base + 1)) < a.dropout;
        if (!dropped) {
            double noisy = depth;
            if (a.noise > 0.0) {
                const double u1 = uniform01(splitmix(base + 2)), u2 = uniform01(splitmix(base + 3));
                const double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
                noisy += g * a.noise * double(depth) * double(depth);
            }
            out = noisy > 0.0 ? float(noisy) : 0.f;
        }
    }
    a.depth[i] = out;
}

}  // namespace rfb

using namespace rfb;

extern "C" rf_status rf_synth_render(const void* prims, int32_t nprims, const double cam_pose[12],
                                     const rf_intrinsics* k, double noise_sigma_scale, double dropout, uint64_t seed,
                                     uint64_t frame_index, float* depth, uint8_t* rgb, uint8_t* labels, int device) {
    if (!prims || !cam_pose || !k || !depth || !rgb || !labels || nprims < 0 || nprims > kMaxSynthPrims)
        return RF_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return RF_CUDA_ERROR;
    SynthArgs h{};
    const unsigned char* src = static_cast<const unsigned char*>(prims);
    for (int i = 0; i < nprims; ++i) {
        // host layout (rf_synth_primitive in synth.py): 4 i32, a[3], b[3], cell, w2o[12], primary[4], secondary[4]
        const unsigned char* p = src + size_t(i) * 176;
        SynthPrim& q = h.prims[i];
        std::memcpy(&q.shape, p, 16);
        std::memcpy(q.a, p + 16, 24);
        std::memcpy(q.b, p + 40, 24);
        std::memcpy(&q.cell, p + 64, 8);
        std::memcpy(q.w2o, p + 72, 96);
        std::memcpy(q.primary, p + 168, 4);
        std::memcpy(q.secondary, p + 172, 4);
    }
    h.nprims = nprims;
    for (int i = 0; i < 9; ++i) h.cam.R[i] = cam_pose[i];
    for (int i = 0; i < 3; ++i) h.cam.t[i] = cam_pose[9 + i];
    h.K.fx = k->fx;
    h.K.fy = k->fy;
    h.K.cx = k->cx;
    h.K.cy = k->cy;
    h.K.w = k->width;
    h.K.h = k->height;
    h.noise = noise_sigma_scale;
    h.dropout = dropout;
    h.seed = seed;
    h.frame = frame_index;
    h.depth = depth;
    h.rgb = rgb;
    h.labels = labels;
    SynthArgs* d = nullptr;
    if (cudaMalloc(&d, sizeof(SynthArgs)) != cudaSuccess) return RF_CUDA_ERROR;
    cudaMemcpy(d, &h, sizeof(SynthArgs), cudaMemcpyHostToDevice);
    const int n = k->width * k->height;
    k_synth<<<(n + 127) / 128, 128>>>(d);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaFree(d);
    return e == cudaSuccess ? RF_OK : RF_CUDA_ERROR;
}
