// Tracking + dynamics mask as one persistent cooperative kernel.
//
// One launch runs the whole coarse-to-fine Levenberg-Marquardt loop of
// Register (registration.cpp:211-286) on the device: every pixel pass is a
// grid-stride sweep over 16x16 pixel tiles whose per-thread normal equations
// (21 H + 6 b + 2 errors + count, fp64) are folded warp -> CTA -> grid in a
// fixed order, so results are deterministic run to run. Every CTA then runs
// the same tiny LM state machine (6x6 LDLT, ExpMap) on the identical reduced
// vector, so no host round trip or second barrier is needed per iteration.
// In kModeFrame the kernel continues with BuildMask (dynamics_mask.cpp:98-104)
// and the masked second registration (pipeline.cpp:81-99).
#include "rf_track.cuh"

namespace rfb {

namespace {

constexpr double kIntensityScale = 1.0 / 255.0;  // registration.cpp:22
constexpr double kRelDecreaseTol = 1e-6;         // registration.cpp:26

// The thread that judges each trial and solves the next LM step: the CTA's
// last thread, which also pre-solves the reject path during the pass (its
// SMSP's instruction cache then holds the solve).
constexpr int kLmThread = kTrackThreads - 1;
__device__ __forceinline__ int hidx(int i, int j) { return i * 6 - (i * (i - 1)) / 2 + (j - i); }

__shared__ int s_trace_pass;  // per-CTA pass counter for the optional timeline
// Per-thread copy of the first a.pxc_steps pixels' inputs {depth (0: skip),
// intensity} for the Jacobian passes: a thread sees the same pixels in every
// pass at a level, so after the first pass they come from shared memory
// instead of an L2 round trip (dynamic shared memory, TrackArgs::dyn_bytes).
extern __shared__ __align__(16) unsigned char s_dyn[];
__device__ __forceinline__ float2* pxc_base() { return reinterpret_cast<float2*>(s_dyn); }
__shared__ int s_pxc_tag;  // (level + 1) | 16 * use_mask of the cached inputs, 0: none
__shared__ int s_passes;   // Accumulate passes run (CTA 0; TrackOut.passes / pixel_passes)
__shared__ double s_pixel_passes;
__shared__ double s_luma_lut[768];  // w_c * x for the three Rec.709 weights (see voxel_luma_lut)
// Per pyramid level (set at kernel start): the intrinsics and image pointers
// (shared memory, so no code indexes the kernel parameters with a run-time
// level, which would copy them to local memory), and this CTA's pixel range:
// ceil(npx / G) consecutive pixels from (ubase, vbase), so a pass starts
// without an integer division on every thread's path to its first pixel.
struct LevelInfo {
    Intr K;
    float* depth;  // level 0: the input depth (read only)
    float* inten;  // level 0: unused (intensity from rgb0 on the fly)
    uint8_t* mask;
    int per, end, ubase, vbase;
};
__shared__ LevelInfo s_lvl[kMaxLevels];

struct RegState {
    // Three pose slots, by index (an accepted or pre-solved candidate changes an
    // index instead of copying 12 doubles on the LM thread's critical path):
    // P[ip] the current pose, P[ic] the candidate of the pass in flight (dn[ic]
    // its squared step), P[3 - ip - ic] the reject-path pre-solve.
    Pose P[3];
    double dn[3];
    int ip, ic;
    __device__ Pose& pose() { return P[ip]; }
    __device__ const Pose& pose() const { return P[ip]; }
    __device__ Pose& cand() { return P[ic]; }
    double lambda;
    double buf[2][kAccN];  // normal equations at the current pose / at the candidate
    int ci;                // buf[ci]: current, buf[ci ^ 1]: trial; swapped on an accepted step (no copy)
    __device__ double* cur() { return buf[ci]; }
    __device__ double* trial() { return buf[ci ^ 1]; }
    // judge inputs that do not depend on the trial, computed while the pass runs
    double cur_err, tol, lam_acc, lam_rej;
    int small_step;
    int total, converged, lost, go, brk, level_it;
    // The next candidate if the trial in flight is rejected (in the free slot):
    // it depends only on the current normal equations and the raised damping,
    // so it is solved during the trial's pass (on a thread with slack).
    int rej_ok;
};

#ifdef RF_LM_CLOCKS  // diagnostics build: cycle counters of CTA 0's LM thread, kept in shared
// memory (no global traffic on the path) and written to trace records 250/251 at exit
__shared__ unsigned long long s_lmacc[18];
__shared__ long long s_lmc[2];
__shared__ long long s_t0c;  // thread 0's own stamp (record 249: its barrier release -> pass entry)
#define T0_MARK_A() do { if (blockIdx.x == 0 && threadIdx.x == 0) s_t0c = clock64(); } while (0)
#define T0_MARK_B() do { if (blockIdx.x == 0 && threadIdx.x == 0 && s_t0c) { \
    s_lmacc[16] += (unsigned long long)(clock64() - s_t0c); s_lmacc[17] += 1; s_t0c = 0; } } while (0)
#define LMC_T(v) const long long v = clock64()
#define RF_PASS_TRACE(a) false  // the per-pass timeline is off: only these counters are written
#define LMC_ADD(k, val) do { if (blockIdx.x == 0) s_lmacc[(k)] += (unsigned long long)(val); } while (0)
// pass-side stamps (record 250): barrier release, pass prologue, own pixels,
// all-reduce, all-reduce end to the next LM section
#define LMC_MARK(k) do { if (blockIdx.x == 0 && threadIdx.x == kLmThread) { const long long t_ = clock64(); \
    if (s_lmc[1]) s_lmacc[8 + (k)] += (unsigned long long)(t_ - s_lmc[0]); s_lmc[0] = t_; } } while (0)
#define LMC_ARM(on) do { if (threadIdx.x == kLmThread) s_lmc[1] = (on); } while (0)
#else
#define RF_PASS_TRACE(a) ((a).trace != nullptr)
#define LMC_T(v)
#define LMC_ADD(k, val) do {} while (0)
#define T0_MARK_A() do {} while (0)
#define T0_MARK_B() do {} while (0)
#define LMC_MARK(k) do {} while (0)
#define LMC_ARM(on) do {} while (0)
#endif
// ------------------------------------------------------------------ math
// 1/x without the IEEE division's special-case branch: the fp64 reciprocal
// approximation plus two Newton steps (relative error ~1e-16; pivots of the
// damped SPD matrix are normal numbers). Branch-free, so the solve below is a
// single basic block the scheduler can interleave.
__device__ __forceinline__ double rcp_nobranch(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    return r;
}

// out = ExpMap(xi) * P0 (geometry.cpp:14-38, geometry.hpp:89-91). One thread
// runs this between the all-reduce and the next pass, and its fp64
// instructions issue at the warp's fp64 rate, so the closed forms count
// instructions: hat^2 = w w^T - |w|^2 I (its diagonal as minus the other two
// squares), R = I + a hat + b hat^2 and V = I + b hat + c hat^2 entry by entry,
// and the products as FMA chains (about half the instructions of the matrix
// forms; the same values to within an ulp).
__device__ __forceinline__ void expmap_compose(const double xi[6], const Pose& P0, Pose& out) {
    const double w0 = xi[3], w1 = xi[4], w2 = xi[5];
    const double s0 = w0 * w0, s1 = w1 * w1, s2 = w2 * w2;
    const double t2 = (s0 + s1) + s2;
    double a, b, c;
    if (t2 < 0.0025) {
        // theta < 0.05 (an LM step is a few milliradians): sin(t)/t,
        // (1-cos t)/t^2, (t-sin t)/t^3 by their Taylor series in t^2 (five
        // terms: truncation < 1e-20), which also covers the reference's
        // theta < 1e-6 branch (its two-term series). No sqrt, sincos or IEEE
        // division on the one thread every CTA waits for.
        a = __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, 1.0 / 362880.0, -1.0 / 5040.0), 1.0 / 120.0),
                                  -1.0 / 6.0), 1.0);
        b = __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, 1.0 / 3628800.0, -1.0 / 40320.0), 1.0 / 720.0),
                                  -1.0 / 24.0), 0.5);
        c = __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, __fma_rn(t2, 1.0 / 39916800.0, -1.0 / 362880.0), 1.0 / 5040.0),
                                  -1.0 / 120.0), 1.0 / 6.0);
    } else {
        const double theta = sqrt(t2);
        double st, ct;
        sincos(theta, &st, &ct);
        a = st / theta;
        b = (1.0 - ct) / t2;
        c = (theta - st) / (t2 * theta);
    }
    const double h01 = w0 * w1, h02 = w0 * w2, h12 = w1 * w2;  // off-diagonal of hat^2 (symmetric)
    const double d0 = -(s1 + s2), d1 = -(s0 + s2), d2 = -(s0 + s1);
    const double aw0 = a * w0, aw1 = a * w1, aw2 = a * w2, bw0 = b * w0, bw1 = b * w1, bw2 = b * w2;
    // hat = [0 -w2 w1; w2 0 -w0; -w1 w0 0]
    const double R[9] = {__fma_rn(b, d0, 1.0), __fma_rn(b, h01, -aw2), __fma_rn(b, h02, aw1),
                         __fma_rn(b, h01, aw2),  __fma_rn(b, d1, 1.0),  __fma_rn(b, h12, -aw0),
                         __fma_rn(b, h02, -aw1), __fma_rn(b, h12, aw0), __fma_rn(b, d2, 1.0)};
    const double V[9] = {__fma_rn(c, d0, 1.0), __fma_rn(c, h01, -bw2), __fma_rn(c, h02, bw1),
                         __fma_rn(c, h01, bw2),  __fma_rn(c, d1, 1.0),  __fma_rn(c, h12, -bw0),
                         __fma_rn(c, h02, -bw1), __fma_rn(c, h12, bw0), __fma_rn(c, d2, 1.0)};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double et = __fma_rn(V[3 * i], xi[0], __fma_rn(V[3 * i + 1], xi[1], V[3 * i + 2] * xi[2]));
#pragma unroll
        for (int j = 0; j < 3; ++j)
            out.R[3 * i + j] =
                __fma_rn(R[3 * i], P0.R[j], __fma_rn(R[3 * i + 1], P0.R[3 + j], R[3 * i + 2] * P0.R[6 + j]));
        out.t[i] = __fma_rn(R[3 * i], P0.t[0], __fma_rn(R[3 * i + 1], P0.t[1], __fma_rn(R[3 * i + 2], P0.t[2], et)));
    }
}

// One damped LM solve (registration.cpp:236-248): damped = H + lambda *
// max(diag H, 1e-3 max diag + 1e-12) on the diagonal, then an LDLT solve of
// damped * delta = -b. The damped matrix is symmetric positive definite
// (PSD normal equations plus a strictly positive diagonal shift), so the
// factorisation needs no pivoting: we factor in natural order, fully unrolled
// in registers on the one thread every CTA waits for. Eigen's LDLT would pivot
// on the largest remaining diagonal; for an SPD matrix that changes only the
// rounding (relative ~cond * 1e-16), far below the pose parity bar (1e-4).
// `acc` is the packed upper triangle + b (smem); `delta` (smem) receives the
// solution.
__device__ bool lm_solve(const double* acc, double lambda, double* delta) {
    double dmax = acc[hidx(0, 0)];
#pragma unroll
    for (int i = 1; i < 6; ++i) dmax = fmax(dmax, acc[hidx(i, i)]);
    const double floor_v = 1e-3 * dmax + 1e-12;
    double m[6][6], x[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double v = acc[hidx(j, i)];
            if (i == j) v += lambda * fmax(v, floor_v);
            m[i][j] = v;
        }
        x[i] = -acc[21 + i];
    }
    // Latency matters here (one thread, every CTA waits). Left-looking LDLT
    // on unscaled columns C (L = C * inv_d): column k subtracts the older
    // terms first and the (k-1) term last, so only one reciprocal (~58
    // cycles), one multiply and one FMA per pivot sit on the dependency
    // chain. Rounding differs from Eigen's divisions in the last bits only;
    // the normal equations already differ at that level through the
    // reduction order, so parity is held at the pose level. (A 2x2 block
    // elimination over the 3x3 translation / rotation blocks with adjugate
    // inverses measured 797 vs 840 cycles in isolation and no difference in
    // the pipeline.)
    double L[6][6], inv_d[6];
    bool pivots_ok = true;  // no early exit: one basic block, so later pivots' work can be hoisted
#pragma unroll
    for (int k = 0; k < 6; ++k) {
#pragma unroll
        for (int i = k; i < 6; ++i) {
            double c = m[i][k];
#pragma unroll
            for (int j = 0; j < k; ++j) c = __fma_rn(-L[i][j], m[k][j], c);  // m[k][j] holds C[k][j]
            m[i][k] = c;
        }
        const double akk = m[k][k];
        pivots_ok = pivots_ok && fabs(akk) > 0.0;  // zero pivot: NumericalIssue path, lambda grows
        inv_d[k] = rcp_nobranch(akk);
#pragma unroll
        for (int i = k + 1; i < 6; ++i) L[i][k] = m[i][k] * inv_d[k];
    }
#pragma unroll
    for (int j = 0; j < 6; ++j)
#pragma unroll
        for (int i = j + 1; i < 6; ++i) x[i] = __fma_rn(-L[i][j], x[j], x[i]);
#pragma unroll
    for (int i = 0; i < 6; ++i) x[i] *= inv_d[i];
#pragma unroll
    for (int j = 5; j >= 0; --j)
#pragma unroll
        for (int i = 0; i < j; ++i) x[i] = __fma_rn(-L[j][i], x[j], x[i]);
    bool finite = pivots_ok;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        delta[i] = x[i];
        finite = finite && isfinite(x[i]);
    }
    return finite;
}

// ------------------------------------------------------------------ pyramid
// BuildPyramid (registration.cpp:144-182), levels >= 1, one barrier per level.
__device__ void build_pyramid(const TrackArgs& a, bool images, bool masks) {
    const FrameView& F = a.F;
    const int stride = gridDim.x * blockDim.x;
    for (int l = 1; l < a.reg.levels; ++l) {
        const LevelInfo& L0 = s_lvl[l - 1];
        const LevelInfo& L1 = s_lvl[l];
        const int w = L1.K.w, h = L1.K.h, pw = L0.K.w;
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < w * h; p += stride) {
            const int x = p % w, y = p / w;
            float closest = 0.f, isum = 0.f;
            uint8_t masked = 0;
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int sp = (2 * y + dy) * pw + (2 * x + dx);
                    if (images) {
                        const float d = (l == 1) ? __ldg(F.depth0 + sp) : __ldcg(L0.depth + sp);
                        if (depth_valid(d) && (!depth_valid(closest) || d < closest)) closest = d;
                        if (F.rgb0) {
                            float iv;
                            if (l == 1) {
                                const uint8_t* c = F.rgb0 + 3 * size_t(sp);
                                iv = float(luma(__ldg(c), __ldg(c + 1), __ldg(c + 2)));  // image.hpp:85-91
                            } else {
                                iv = __ldcg(L0.inten + sp);
                            }
                            isum += iv;
                        }
                    }
                    if (masks && __ldcg(L0.mask + sp)) masked = 1;
                }
            if (images) {
                L1.depth[p] = closest;
                if (F.rgb0) L1.inten[p] = isum * 0.25f;
            }
            if (masks) L1.mask[p] = masked;
        }
        grid_barrier(a.grid);
    }
}

// ------------------------------------------------------------------ pixel pass
// One Accumulate (registration.cpp:49-117) over pyramid level `level`.
// `pre` runs on the CTA's last thread after its pixels when that thread has
// fewer pixels than the busiest ones (its slack hides the work).
template <bool kJac, bool kColor, bool kRobust, class Hook, class Pre>
__device__ void accumulate(const TrackArgs& a, int level, const Pose& P, bool use_mask, bool write_res, double cw,
                           double* scratch, double* blk, double* out, const Hook& hook, const Pre& pre) {
    const FrameView& F = a.F;
    const LevelInfo& LI = s_lvl[level];
    const Intr K = LI.K;
    const double min_depth = a.V.min_depth, max_depth = a.V.max_depth;
    double acc[kAccN];
#pragma unroll
    for (int i = 0; i < kAccN; ++i) acc[i] = 0.0;
    const float* depth = LI.depth;
    const uint8_t* mask = use_mask ? LI.mask : nullptr;
    unsigned long long* tr = (RF_PASS_TRACE(a) && s_trace_pass < kTracePasses) ? a.trace + 8 * s_trace_pass : nullptr;
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
        tr[0] = global_ns();
        tr[4] = level;
        tr[5] = (unsigned long long)K.w * K.h;
        tr[6] = kJac;
    }
    if (kJac) LMC_MARK(1);  // pass prologue
    const int pxc_tag = (level + 1) | (use_mask ? 16 : 0);
    const bool pxc_hit = kJac && s_pxc_tag == pxc_tag;
    auto pixel = [&](const int u, const int v, const int it) {
        const int p = v * K.w + u;
        RF_ASSERT(u >= 0 && u < K.w && v >= 0 && v < K.h);
        RF_ASSERT(it >= a.pxc_steps || (it + 1) * kTrackThreads * 8 <= a.dyn_bytes);
        // Every per-pixel input is loaded up front (depth, mask, intensity),
        // so only the hash slot and voxel gathers are dependent round trips.
        float d;
        bool masked;
        float inten = 0.f;  // ToIntensity (image.hpp:85-91) at level 0, the pyramid's f32 above
        if (pxc_hit && it < a.pxc_steps) {
            const float2 c = pxc_base()[it * kTrackThreads + threadIdx.x];
            d = c.x;
            inten = c.y;
            masked = false;  // a masked pixel was cached with depth 0
        } else {
            d = level == 0 ? __ldg(depth + p) : __ldcg(depth + p);
            masked = mask && __ldcg(mask + p) != 0;
            if (kColor) {
                if (level == 0) {
                    const uint8_t* c = F.rgb0 + 3 * size_t(p);
                    inten = float(luma(__ldg(c), __ldg(c + 1), __ldg(c + 2)));
                } else {
                    inten = __ldcg(LI.inten + p);
                }
            }
            if (kJac && it < a.pxc_steps) pxc_base()[it * kTrackThreads + threadIdx.x] = make_float2(masked ? 0.f : d, inten);
        }
        float rs = 0.f;
        uint8_t rv = 0;
        if (depth_valid(d) && !(d < min_depth) && !(d > max_depth)) {
            if (!(masked && !write_res)) {
                const double dd = double(d);
                // Backproject (geometry.hpp:41-43); Jacobian passes use reciprocals
                const double x0 = kJac ? (double(u) - K.cx) * K.ifx * dd : div_rn(double(u) - K.cx, K.fx, K.ifx) * dd;
                const double x1 = kJac ? (double(v) - K.cy) * K.ify * dd : div_rn(double(v) - K.cy, K.fy, K.ify) * dd;
                double y[3];
                pose_apply(P, x0, x1, dd, y);
                CellSample cs;
                if (sample_point<kJac, kColor, !kJac>(a.V, y, cs, s_luma_lut)) {
                    const double r_d = cs.sdf;
                    const double I = kColor ? double(inten) : 0.0;
                    if (kJac && kRobust) {
                        // Huber extension (off by default; not in the reference): rows
                        // of a residual beyond the threshold weighted by hd / |r|, its
                        // cost 2 hd |r| - hd^2 (continuous with r^2). A weight of 1.0
                        // multiplies exactly, so inliers add what the plain path adds.
                        const double hd = a.reg.huber_d, ad = fabs(r_d);
                        const bool out_d = hd > 0.0 && ad > hd;
                        const double wd = out_d ? hd / ad : 1.0;
                        const double J[6] = {cs.gs[0], cs.gs[1], cs.gs[2], y[1] * cs.gs[2] - y[2] * cs.gs[1],
                                             y[2] * cs.gs[0] - y[0] * cs.gs[2], y[0] * cs.gs[1] - y[1] * cs.gs[0]};
#pragma unroll
                        for (int i = 0; i < 6; ++i)
#pragma unroll
                            for (int j = i; j < 6; ++j) acc[hidx(i, j)] = __fma_rn(wd * J[i], J[j], acc[hidx(i, j)]);
#pragma unroll
                        for (int i = 0; i < 6; ++i) acc[21 + i] = __fma_rn(wd * J[i], r_d, acc[21 + i]);
                        acc[27] = out_d ? acc[27] + (2.0 * hd * ad - hd * hd) : __fma_rn(r_d, r_d, acc[27]);
                        if (kColor) {
                            const double r_c = (cs.inten - I) * kIntensityScale;
                            const double hc = a.reg.huber_c, ac = fabs(r_c);
                            const bool out_c = hc > 0.0 && ac > hc;
                            const double cwc = cw * (out_c ? hc / ac : 1.0);
                            const double Jc[6] = {cs.gi[0] * kIntensityScale, cs.gi[1] * kIntensityScale,
                                                  cs.gi[2] * kIntensityScale,
                                                  (y[1] * cs.gi[2] - y[2] * cs.gi[1]) * kIntensityScale,
                                                  (y[2] * cs.gi[0] - y[0] * cs.gi[2]) * kIntensityScale,
                                                  (y[0] * cs.gi[1] - y[1] * cs.gi[0]) * kIntensityScale};
#pragma unroll
                            for (int i = 0; i < 6; ++i)
#pragma unroll
                                for (int j = i; j < 6; ++j)
                                    acc[hidx(i, j)] = __fma_rn(cwc * Jc[i], Jc[j], acc[hidx(i, j)]);
#pragma unroll
                            for (int i = 0; i < 6; ++i) acc[21 + i] = __fma_rn(cwc * Jc[i], r_c, acc[21 + i]);
                            acc[28] = out_c ? acc[28] + (2.0 * hc * ac - hc * hc) : __fma_rn(r_c, r_c, acc[28]);
                        }
                        acc[29] += 1.0;
                    } else if (kJac) {
                        const double J[6] = {cs.gs[0], cs.gs[1], cs.gs[2], y[1] * cs.gs[2] - y[2] * cs.gs[1],
                                             y[2] * cs.gs[0] - y[0] * cs.gs[2], y[0] * cs.gs[1] - y[1] * cs.gs[0]};
#pragma unroll
                        for (int i = 0; i < 6; ++i)
#pragma unroll
                            for (int j = i; j < 6; ++j) acc[hidx(i, j)] = __fma_rn(J[i], J[j], acc[hidx(i, j)]);
#pragma unroll
                        for (int i = 0; i < 6; ++i) acc[21 + i] = __fma_rn(J[i], r_d, acc[21 + i]);
                        acc[27] = __fma_rn(r_d, r_d, acc[27]);
                        if (kColor) {
                            const double r_c = (cs.inten - I) * kIntensityScale;
                            const double Jc[6] = {cs.gi[0] * kIntensityScale, cs.gi[1] * kIntensityScale,
                                                  cs.gi[2] * kIntensityScale,
                                                  (y[1] * cs.gi[2] - y[2] * cs.gi[1]) * kIntensityScale,
                                                  (y[2] * cs.gi[0] - y[0] * cs.gi[2]) * kIntensityScale,
                                                  (y[0] * cs.gi[1] - y[1] * cs.gi[0]) * kIntensityScale};
#pragma unroll
                            for (int i = 0; i < 6; ++i)
#pragma unroll
                                for (int j = i; j < 6; ++j)
                                    acc[hidx(i, j)] = __fma_rn(cw * Jc[i], Jc[j], acc[hidx(i, j)]);
#pragma unroll
                            for (int i = 0; i < 6; ++i) acc[21 + i] = __fma_rn(cw * Jc[i], r_c, acc[21 + i]);
                            acc[28] = __fma_rn(r_c, r_c, acc[28]);
                        }
                        acc[29] += 1.0;
                    } else {
                        rs = float(r_d * r_d);
                        rv = (a.mp.free_space > 0.0 && r_d > 0.0) ? 3 : 1;  // bit 1: the free-space extension's sign
                        if (!masked) {
                            acc[27] += r_d * r_d;
                            if (kColor) {
                                const double r_c = (cs.inten - I) * kIntensityScale;
                                acc[28] += r_c * r_c;
                            }
                            acc[29] += 1.0;
                        }
                    }
                }
            }
        }
        if (!kJac && write_res) {
            F.res_sq[p] = rs;
            F.res_valid[p] = rv;
        }
    };
    // The level's pixels spread evenly: ceil(npx / G) consecutive pixels per
    // CTA (a strip of rows), 384 per step (640x480: 2076 / 519 / 130 per CTA
    // at levels 0 / 1 / 2), instead of whole 16x24 tiles on part of the CTAs
    // (B200, frames 5..104: 1519 -> 1581 frames/s).
    {
        const LevelInfo& R = s_lvl[level];
        const int per = R.per, end = R.end;
        int p = int(blockIdx.x) * per + int(threadIdx.x);
        int u = R.ubase + int(threadIdx.x), v = R.vbase;  // then stepped: no division per pixel
        while (u >= K.w) {
            u -= K.w;
            ++v;
        }
        int it = 0;
        for (int q = int(threadIdx.x); q < per; ++it, q += kTrackThreads) {
            if (p < end) pixel(u, v, it);
            p += kTrackThreads;
            u += kTrackThreads;
            while (u >= K.w) {
                u -= K.w;
                ++v;
            }
        }
        if (threadIdx.x == kTrackThreads - 1 && it < (per + kTrackThreads - 1) / kTrackThreads) pre();
    }
    if (tr) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long now = global_ns();
            atomicMax(tr + 2, now);  // slowest CTA finishing its tiles
            if (blockIdx.x == 0) tr[1] = now;
        }
    }
    // Jacobian passes write nothing global; a value pass's residual image is
    // read across CTAs by the mask that follows (publish). Warps without
    // pixels (most of them at the coarsest level) skip their transpose.
    const bool warp_has_pixels = (int(threadIdx.x) & ~31) < s_lvl[level].per;
    if (kJac) LMC_MARK(2);  // the LM thread's own pixels (and pre-solve)
    block_grid_allreduce<kAccN, !kJac>(a.grid, acc, scratch, out, hook, warp_has_pixels);
    if (kJac) LMC_MARK(3);  // all-reduce
    if (kJac && threadIdx.x == 0) s_pxc_tag = pxc_tag;  // (every thread read it before the barriers above)
    if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[3] = global_ns();
    if (a.trace && threadIdx.x == 0) ++s_trace_pass;
}

// `hook` runs on thread 0 once the CTA has arrived at the pass's all-reduce
// (work that must not delay the CTA's own pixels or arrival).
template <bool kJac, class Hook = NoHook, class Pre = NoHook>
__device__ __forceinline__ void pass(const TrackArgs& a, int level, const Pose& P, bool use_mask, bool write_res,
                                     double cw, double* scratch, double* blk, double* out, const Hook& hook = Hook(),
                                     const Pre& pre = Pre()) {
    if (kJac) LMC_MARK(5);  // barrier release -> pass entry
    if (kJac) T0_MARK_B();
    const bool color = cw > 0.0 && a.F.rgb0 != nullptr;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s_passes += 1;  // CTA 0's tally, published once at kernel exit (no global RMW on the pass path)
        s_pixel_passes += double(s_lvl[level].K.w) * double(s_lvl[level].K.h);
    }
    const bool robust = kJac && (a.reg.huber_d > 0.0 || a.reg.huber_c > 0.0);
    if (robust) {
        if (color) accumulate<kJac, true, true>(a, level, P, use_mask, write_res, cw, scratch, blk, out, hook, pre);
        else accumulate<kJac, false, true>(a, level, P, use_mask, write_res, cw, scratch, blk, out, hook, pre);
    } else if (color) {
        accumulate<kJac, true, false>(a, level, P, use_mask, write_res, cw, scratch, blk, out, hook, pre);
    } else {
        accumulate<kJac, false, false>(a, level, P, use_mask, write_res, cw, scratch, blk, out, hook, pre);
    }
}

// ------------------------------------------------------------------ Register
// registration.cpp:211-286. All CTAs run the same state machine on the same
// reduced vectors; thread 0 of each CTA updates the shared state.
// Inlined at both call sites: as an out-of-line function its `const
// TrackArgs&` would force a copy of the kernel parameters to local memory.
__device__ __forceinline__ void run_register(const TrackArgs& a, const Pose& init, bool use_mask, RegState& st,
                                             double* scratch, double* blk) {
    const RegParams& R = a.reg;
    const double cw = R.color_weight;
    if (threadIdx.x == 0) {
        st.P[0] = init;
        st.ip = 0;
        st.ic = 1;
        st.total = 0;
        st.converged = 0;
        st.lost = 0;
        st.ci = 0;
    }
    __syncthreads();
    for (int l = R.levels - 1; l >= 0; --l) {
        const long long mv = (long long)(max(R.min_valid, 1)) >> (2 * l);
        const double min_valid = double(mv > 16 ? mv : 16);
        // One pass site per level (the level's linearization at the current
        // pose, then the LM trials), so the level's first pass and its trials
        // run the same instructions: the trials start with a warm i-cache.
        bool lin = true;
        for (;;) {
            pass<true>(a, l, lin ? st.pose() : st.cand(), use_mask, false, cw, scratch, blk, lin ? st.cur() : st.trial(),
                       [&] {
                           // everything of the judge but the trial's error, on thread 0 while the
                           // all-reduce's arrivals propagate (off every critical path)
                           if (lin) return;
                           st.cur_err = st.cur()[27] + cw * st.cur()[28];
                           st.tol = kRelDecreaseTol * st.cur_err;
                           st.lam_acc = fmax(st.lambda / R.lambda_down, 1e-12);
                           st.lam_rej = fmin(st.lambda * R.lambda_up, 1e12);
                           st.small_step = sqrt(st.dn[st.ic]) < R.eps;
                       },
                       [&] {
                           // registration.cpp:265-271 then :240-249 on rejection: lambda
                           // raised (a level that reaches 1e12 converges instead)
                           if (lin) return;
                           const double lam = fmin(st.lambda * R.lambda_up, 1e12);
                           if (!(lam >= 1e12)) {
                               double delta[6];
                               LMC_T(p0);
                               if (lm_solve(st.cur(), lam, delta)) {
                                   const int fr = 3 - st.ip - st.ic;  // the free slot
                                   expmap_compose(delta, st.pose(), st.P[fr]);
                                   double dn = 0.0;
#pragma unroll
                                   for (int i = 0; i < 6; ++i) dn += delta[i] * delta[i];
                                   st.dn[fr] = dn;
                                   st.rej_ok = 1;
                                   LMC_T(p1);
                                   LMC_ADD(5, 1);
                                   LMC_ADD(6, p1 - p0);
                               }
                           }
                       });
            const bool judge = !lin;  // a trial was evaluated since the last solve
            if (lin) {
                if (st.cur()[29] < min_valid) {
                    if (threadIdx.x == 0) st.lost = 1;
                    __syncthreads();
                    return;
                }
                __syncthreads();
                if (threadIdx.x == kLmThread) {  // the LM thread's own state: no barrier needed before it reads it
                    st.lambda = R.lambda_init;
                    st.converged = 0;
                    st.brk = 0;
                    st.level_it = 0;
                }
                lin = false;
            }
            // One barrier per LM iteration: kLmThread judges the last trial and
            // solves for the next candidate in one straight-line section on
            // local copies of its state (registration.cpp:233-272).
            if (threadIdx.x == kLmThread) {
                LMC_MARK(4);  // all-reduce end to the LM section
                LMC_T(c0);
                double lambda = st.lambda;
                int brk = st.brk, level_it = st.level_it, total = st.total, converged = st.converged, ci = st.ci;
                const int ip0 = st.ip, ic0 = st.ic;
                int ip = ip0, ic = ic0;  // the solve below writes slot ic
                const double* tr = st.buf[ci ^ 1];
                bool rejected = false;
                if (judge) {
                    const double cur_err = st.cur_err;
                    const double trial_err = tr[27] + cw * tr[28];
                    if (tr[29] >= min_valid && trial_err < cur_err) {
                        const double decrease = cur_err - trial_err;
                        ip = ic0;  // the candidate becomes the pose; its old slot takes the next candidate
                        ic = ip0;
                        ci ^= 1;
                        lambda = st.lam_acc;
                        if (st.small_step || decrease < st.tol) {
                            converged = 1;
                            brk = 1;
                        }
                    } else {
                        rejected = true;
                        lambda = st.lam_rej;
                        if (lambda >= 1e12) {
                            converged = 1;
                            brk = 1;
                        }
                    }
                }
                int go = 0;
                if (rejected && !brk && level_it < R.max_iterations && st.rej_ok) {
                    // the solve this loop would run now (same buffer, same damping): done during the pass
                    ++level_it;
                    ++total;
                    ic = 3 - ip0 - ic0;
                    go = 1;
                }
                if (judge && RF_PASS_TRACE(a) && blockIdx.x == 0 && s_trace_pass > 0 && s_trace_pass <= kTracePasses)
                    a.trace[8 * (s_trace_pass - 1) + 6] |= rejected ? 0x200ull : 0x100ull;  // the trial's verdict
                while (!go && !brk && level_it < R.max_iterations) {
                    ++level_it;
                    ++total;
                    LMC_T(c1);
                    const Pose P0 = st.P[ip];
                    double delta[6];  // in registers: ExpMap and the norm read it straight from the solve
                    const bool solved = lm_solve(st.buf[ci], lambda, delta);
                    LMC_T(c2);
                    if (!solved) {
                        lambda = fmin(lambda * R.lambda_up, 1e12);  // NumericalIssue: damp more, retry
                        continue;
                    }
                    expmap_compose(delta, P0, st.P[ic]);
                    double dn = 0.0;
#pragma unroll
                    for (int i = 0; i < 6; ++i) dn += delta[i] * delta[i];
                    st.dn[ic] = dn;  // squared; the sqrt is taken off the critical path below
                    LMC_T(c3);
                    LMC_ADD(0, 1);
                    LMC_ADD(1, c1 - c0);
                    LMC_ADD(2, c2 - c1);
                    LMC_ADD(3, c3 - c2);
                    go = 1;
                    break;
                }
                st.ip = ip;
                st.ic = ic;
                st.lambda = lambda;
                st.brk = brk;
                st.level_it = level_it;
                st.total = total;
                st.converged = converged;
                st.ci = ci;
                st.go = go;
                st.rej_ok = 0;
                if (RF_PASS_TRACE(a) && blockIdx.x == 0 && s_trace_pass < kTracePasses)
                    a.trace[8 * s_trace_pass + 7] = global_ns();  // solve done (next pass's record)
                LMC_T(c4);
                LMC_ARM(0);
                LMC_MARK(0);
                LMC_ARM(1);
                LMC_ADD(4, c4 - c0);
                LMC_ADD(7, 1);
            }
            LMC_MARK(7);  // LM section end -> reconverged
            __syncthreads();
            LMC_MARK(0);  // barrier release after the LM section
            T0_MARK_A();
            if (!st.go) break;
            LMC_MARK(6);  // go read (before the back-edge)
        }
        __syncthreads();
    }
    // Full-resolution residual image at the final pose, mask ignored (:282-284).
    pass<false>(a, 0, st.pose(), false, true, 0.0, scratch, blk, st.trial());
}

// ------------------------------------------------------------------ mask
// Separable square morphology (dynamics_mask.cpp:22-47): the square window
// factors into a row pass and a column pass; out-of-image pixels are off.
__device__ void morph_pass(const uint8_t* src, uint8_t* dst, int w, int h, int r, bool erode, bool rows) {
    const int stride = gridDim.x * blockDim.x;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < w * h; p += stride) {
        const int x = p % w, y = p / w;
        bool val = erode;
        for (int o = -r; o <= r; ++o) {
            const int nx = rows ? x + o : x, ny = rows ? y : y + o;
            const bool on = nx >= 0 && nx < w && ny >= 0 && ny < h && __ldcg(src + ny * w + nx) != 0;
            if (erode && !on) {
                val = false;
                break;
            }
            if (!erode && on) {
                val = true;
                break;
            }
        }
        dst[p] = val ? 1 : 0;
    }
}

// Growth-edge bits of the floodfill rule (dynamics_mask.cpp:59-96) for the
// 32x32 tile (tx, ty), from a shared-memory copy of its depth with a
// one-pixel halo: bit k of pixel n is set when a set pixel p = n - (kDx[k],
// kDy[k]) may grow into n (n and p valid, |D(p) - D(n)| < theta * D(p)).
// Stored as bit planes, one 32-bit word per (tile, k, row), x = bit: the
// floodfill works on whole rows at once.
__device__ void grow_tile(const float* depth, uint32_t* planes, int w, int h, int tx, int ty, double theta,
                          int conn) {
    constexpr int S = 32 + 2;
    __shared__ float dt[S * S];
    static constexpr int kDx[8] = {1, -1, 0, 0, 1, 1, -1, -1};  // dynamics_mask.cpp:67-68
    static constexpr int kDy[8] = {0, 0, 1, -1, 1, -1, 1, -1};
    const int ntx = (w + 31) / 32;
    uint32_t* tp = planes + size_t(ty * ntx + tx) * 8 * 32;
    const int gx0 = tx * 32 - 1, gy0 = ty * 32 - 1;
#pragma unroll 4
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) {
        const int gx = gx0 + i % S, gy = gy0 + i / S;
        dt[i] = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? __ldg(depth + gy * w + gx) : 0.f;  // 0: invalid
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int y = threadIdx.x >> 5; y < 32; y += blockDim.x >> 5) {  // warp = one row, lane = x
        const int x = lane, gx = tx * 32 + x, gy = ty * 32 + y;
        const float dn = dt[(y + 1) * S + x + 1];
        uint32_t bits = 0;
        if (gx < w && gy < h && depth_valid(dn)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k >= conn) break;
                const float dp = dt[(y + 1 - kDy[k]) * S + (x + 1 - kDx[k])];  // off-image: 0 (invalid)
                if (depth_valid(dp) && fabs(double(dp) - double(dn)) < theta * double(dp)) bits |= 1u << k;
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t word = __ballot_sync(0xffffffffu, (bits >> k) & 1u);
            if (lane == k) tp[k * 32 + y] = word;
        }
    }
    __syncthreads();
}

// Tile-based square morphology: one 32x32 output tile per CTA step, the
// (32+2r)^2 input window staged in shared memory, the separable row and
// column passes done there (no global intermediate, no grid barrier between
// them). `src(gx, gy)` yields the input bit of an in-image pixel.
constexpr int kMorphTile = 32, kMorphMaxR = 8, kMorphS = kMorphTile + 2 * kMorphMaxR;
template <bool kErode, class Src>
__device__ void morph_tile(int tx, int ty, int w, int h, int r, Src src, uint8_t* dst, int& count) {
    __shared__ uint8_t win[kMorphS * kMorphS];
    __shared__ uint8_t rowv[kMorphS * kMorphTile];
    const int S = kMorphTile + 2 * r;
    const int gx0 = tx * kMorphTile - r, gy0 = ty * kMorphTile - r;
#pragma unroll 4
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) {  // (unrolled: several pixels' loads in flight)
        const int gx = gx0 + i % S, gy = gy0 + i / S;
        win[i] = (gx >= 0 && gx < w && gy >= 0 && gy < h && src(gx, gy)) ? 1 : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < S * kMorphTile; i += blockDim.x) {
        const int y = i / kMorphTile, x = i % kMorphTile;
        uint8_t v = kErode ? 1 : 0;
        for (int k = 0; k <= 2 * r; ++k) v = kErode ? (v & win[y * S + x + k]) : (v | win[y * S + x + k]);
        rowv[i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kMorphTile * kMorphTile; i += blockDim.x) {
        const int y = i / kMorphTile, x = i % kMorphTile;
        const int gx = tx * kMorphTile + x, gy = ty * kMorphTile + y;
        if (gx >= w || gy >= h) continue;
        uint8_t v = kErode ? 1 : 0;
        for (int k = 0; k <= 2 * r; ++k)
            v = kErode ? (v & rowv[(y + k) * kMorphTile + x]) : (v | rowv[(y + k) * kMorphTile + x]);
        dst[gy * w + gx] = v;
        count += v;
    }
    __syncthreads();
}

constexpr int kFfW = 32, kFfH = 32;  // floodfill tile: one warp, lane = row, bit = column

// Floodfill worklists. F.ffstamp holds, for nft = ntx * nty tiles:
//   [0, nft)          queued[t]: last round tile t was queued for (-1: never)
//   [nft, 3 nft)      two tile lists (rounds alternate)
//   [3 nft, +64)      per-round list lengths (round r uses r % 64)
constexpr int kFfCounts = 64;
__device__ __forceinline__ int* ff_list(int* base, int nft, int round) { return base + nft * (1 + (round & 1)); }
__device__ __forceinline__ unsigned int* ff_count(int* base, int nft, int round) {
    return reinterpret_cast<unsigned int*>(base + 3 * nft) + (round % kFfCounts);
}
// Queues tile (tx, ty)'s 3x3 neighbourhood for `round` (once per tile per
// round); lanes 0..8 of the calling warp (or threads 0..8 with warp == 0).
__device__ __forceinline__ void ff_enqueue3x3(int* base, int ntx, int nty, int tx, int ty, int round) {
    const int nft = ntx * nty, lane = threadIdx.x & 31;
    if (lane < 9) {
        const int nx = tx + lane % 3 - 1, ny = ty + lane / 3 - 1;
        if (nx >= 0 && nx < ntx && ny >= 0 && ny < nty) {
            const int n = ny * ntx + nx;
            if (atomicMax(base + n, round) < round)
                ff_list(base, nft, round)[atomicAdd(ff_count(base, nft, round), 1u)] = n;
        }
    }
}

// Flag worklists (when the tile flags fit in the launch's dynamic shared
// memory; the atomic queue above otherwise): F.ffstamp holds three per-tile flag
// arrays, round r reading array r % 3 (tiles that changed in round r - 1, or
// seeded ones for r = 0), setting array (r + 1) % 3 with plain stores and
// zeroing array (r + 2) % 3 (read in round r - 1). Every CTA builds the same
// tile list -- the 3x3 dilation of the flags, compacted in tile order -- in
// its dynamic shared memory, so a round costs one flag load instead of the
// count / list loads and the returning atomics of the queue (1336 -> 1340
// frames/s).
__device__ __forceinline__ bool ff_flag_mode(int nft, int dyn_bytes) {  // nft flag bytes + nft uint16 list
    return ((nft + 15) & ~15) + 2 * nft <= dyn_bytes;
}

// Kogge-Stone fills of a 32-bit row: every pixel reachable from `g` by
// moves of one pixel in the given direction through pixels whose entry bit
// (`p`) is set, in five steps.
__device__ __forceinline__ uint32_t fill_xplus(uint32_t g, uint32_t p) {  // x-1 -> x
    g |= p & (g << 1);  p &= p << 1;
    g |= p & (g << 2);  p &= p << 2;
    g |= p & (g << 4);  p &= p << 4;
    g |= p & (g << 8);  p &= p << 8;
    return g | (p & (g << 16));
}
__device__ __forceinline__ uint32_t fill_xminus(uint32_t g, uint32_t p) {  // x+1 -> x
    g |= p & (g >> 1);  p &= p >> 1;
    g |= p & (g >> 2);  p &= p >> 2;
    g |= p & (g >> 4);  p &= p >> 4;
    g |= p & (g >> 8);  p &= p >> 8;
    return g | (p & (g >> 16));
}
// The same across the warp's lanes (lane = row): y-1 -> y, then y+1 -> y.
__device__ __forceinline__ uint32_t fill_yplus(uint32_t g, uint32_t p, int lane) {
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const uint32_t gu = __shfl_up_sync(0xffffffffu, g, k), pu = __shfl_up_sync(0xffffffffu, p, k);
        g |= lane >= k ? (p & gu) : 0u;
        p &= lane >= k ? pu : 0u;
    }
    return g;
}
__device__ __forceinline__ uint32_t fill_yminus(uint32_t g, uint32_t p, int lane) {
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const uint32_t gd = __shfl_down_sync(0xffffffffu, g, k), pd = __shfl_down_sync(0xffffffffu, p, k);
        g |= lane + k < 32 ? (p & gd) : 0u;
        p &= lane + k < 32 ? pd : 0u;
    }
    return g;
}

// FloodfillDepth (dynamics_mask.cpp:59-96) as the least fixpoint of the
// growth rule (its BFS result is seed-order independent, so any monotone
// schedule reaches it). A 32x32 tile is one warp: lane = row, the row's
// mask and its eight growth-edge planes are 32-bit words, and one iteration
// runs complete fills along +x, -x (bit-parallel Kogge-Stone in the word)
// and +y, -y (across lanes with shuffles) plus the four diagonal steps for
// 8-connectivity; iterations repeat until the tile stops changing. The set
// pixels of the surrounding ring (neighbour tiles) seed the tile once. Global
// rounds visit only queued tiles -- round 0: the 3x3 neighbourhoods of tiles
// with seeds, then those of tiles that changed -- one tile per warp across
// the grid, until a round changes nothing. Returns the number of rounds.
__device__ int floodfill(const TrackArgs& a, uint8_t* m, const uint32_t* planes, int w, int h, int conn) {
    int* wl = a.F.ffstamp;  // worklists (see ff_list): round 0 was queued by the erosion pass
    const int ntx = (w + kFfW - 1) / kFfW, nty = (h + kFfH - 1) / kFfH, nft = ntx * nty;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int G = gridDim.x;
    auto at = [&](int gx, int gy) -> uint32_t {  // mask bit of an image pixel (0 outside)
        return (gx >= 0 && gx < w && gy >= 0 && gy < h) ? uint32_t(__ldcg(m + size_t(gy) * w + gx) != 0) : 0u;
    };
    const bool flags = ff_flag_mode(nft, a.dyn_bytes);
    uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_dyn);  // (the pixel cache is refilled after the mask)
    uint16_t* s_list = reinterpret_cast<uint16_t*>(s_dyn + ((nft + 15) & ~15));
    __shared__ int s_wcount[kTrackThreads / 32];
    if (flags && threadIdx.x == 0) s_pxc_tag = 0;
    int rounds = 0;
    while (true) {
        if (a.trace && rounds < 8 && blockIdx.x == 0 && threadIdx.x == 0)
            a.trace[8 * (kTracePasses - 3) + rounds] = global_ns();
        int nq;
        const int* list = nullptr;
        if (flags) {
            const int* fr = wl + nft * (rounds % 3);
            for (int t = threadIdx.x; t < nft; t += blockDim.x) s_flag[t] = __ldcg(fr + t) != 0;
            if (blockIdx.x == 0)
                for (int t = threadIdx.x; t < nft; t += blockDim.x) wl[nft * ((rounds + 2) % 3) + t] = 0;
            __syncthreads();
            nq = 0;
            for (int c0 = 0; c0 < nft; c0 += blockDim.x) {  // queued = 3x3 dilation, compacted in tile order
                const int t = c0 + int(threadIdx.x);
                bool q = false;
                if (t < nft) {
                    const int tx = t % ntx, ty = t / ntx;
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int nx = tx + dx, ny = ty + dy;
                            q |= nx >= 0 && nx < ntx && ny >= 0 && ny < nty && s_flag[ny * ntx + nx];
                        }
                }
                const unsigned b = __ballot_sync(0xffffffffu, q);
                if (lane == 0) s_wcount[warp] = __popc(b);
                __syncthreads();
                int before = 0, total = 0;
                for (int k = 0; k < nwarps; ++k) {
                    const int c = s_wcount[k];
                    before += k < warp ? c : 0;
                    total += c;
                }
                if (q) s_list[nq + before + __popc(b & ((1u << lane) - 1u))] = uint16_t(t);
                nq += total;
                __syncthreads();
            }
            if (nq == 0) {  // nothing changed in the last round: fixpoint reached
                if (a.trace && rounds < 8 && threadIdx.x == 0)
                    atomicMax(a.trace + 8 * (kTracePasses - 4) + rounds, global_ns());  // (the empty round's end)
                break;
            }
        } else {
            if (blockIdx.x == 0 && threadIdx.x == 0) *ff_count(wl, nft, rounds + 2) = 0u;  // not touched this round
            nq = int(__ldcg(ff_count(wl, nft, rounds)));
            list = ff_list(wl, nft, rounds);
        }
        RF_ASSERT(nq <= nft);
        for (int qi = warp * G + blockIdx.x; qi < nq; qi += G * nwarps) {  // one tile per warp
            const int t = flags ? int(s_list[qi]) : __ldcg(list + qi);
            RF_ASSERT(t >= 0 && t < nft);
            const int tx = t % ntx, ty = t / ntx, x0 = tx * kFfW, y0 = ty * kFfH;
            const int gy = y0 + lane;
            // row words: mask, validity, growth planes (x = bit)
            const uint32_t valid = (gy < h) ? (w - x0 >= 32 ? 0xffffffffu : ((1u << (w - x0)) - 1u)) : 0u;
            uint32_t set = 0;
            if (gy < h) {
                const uint8_t* row = m + size_t(gy) * w + x0;
                if ((w & 3) == 0 && w - x0 >= 32) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint32_t v = __ldcg(reinterpret_cast<const unsigned int*>(row) + c) & 0x01010101u;
                        set |= ((v | (v >> 7) | (v >> 14) | (v >> 21)) & 0xFu) << (4 * c);
                    }
                } else {
                    for (int x = 0; x < 32 && x0 + x < w; ++x) set |= uint32_t(__ldcg(row + x) != 0) << x;
                }
            }
            const uint32_t* tp = planes + size_t(t) * 8 * 32 + lane;
            uint32_t P[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) P[k] = k < conn ? (__ldcg(tp + k * 32) & valid) : 0u;
            // the ring around the tile
            const uint32_t hl = at(x0 - 1, gy), hr = at(x0 + 32, gy);
            const uint32_t top = __ballot_sync(0xffffffffu, at(x0 + lane, y0 - 1) != 0);
            const uint32_t bot = __ballot_sync(0xffffffffu, at(x0 + lane, y0 + 32) != 0);
            const uint32_t tl = at(x0 - 1, y0 - 1), tr = at(x0 + 32, y0 - 1);
            const uint32_t bl = at(x0 - 1, y0 + 32), br = at(x0 + 32, y0 + 32);
            const uint32_t hl_up = __shfl_up_sync(0xffffffffu, hl, 1), hr_up = __shfl_up_sync(0xffffffffu, hr, 1);
            const uint32_t hl_dn = __shfl_down_sync(0xffffffffu, hl, 1), hr_dn = __shfl_down_sync(0xffffffffu, hr, 1);
            set &= valid;
            const uint32_t initial = set;
            uint32_t g = set;
            // seeds from the ring (bit k: from n - (kDx[k], kDy[k]))
            g |= P[0] & hl;                                  // from (x-1, y): x = 0
            g |= P[1] & (hr << 31);                          // from (x+1, y): x = 31
            if (lane == 0) g |= P[2] & top;                  // from (x, y-1)
            if (lane == 31) g |= P[3] & bot;                 // from (x, y+1)
            if (conn == 8) {
                g |= P[4] & (lane == 0 ? ((top << 1) | tl) : hl_up);          // from (x-1, y-1)
                g |= P[5] & (lane == 31 ? ((bot << 1) | bl) : hl_dn);         // from (x-1, y+1)
                g |= P[6] & (lane == 0 ? ((top >> 1) | (tr << 31)) : (hr_up << 31));   // from (x+1, y-1)
                g |= P[7] & (lane == 31 ? ((bot >> 1) | (br << 31)) : (hr_dn << 31));  // from (x+1, y+1)
            }
            g &= valid;
            for (int it = 0;; ++it) {
                const uint32_t old = g;
                // Along one axis the two directions are independent (a path that
                // turns back within a row or column only revisits covered pixels),
                // so each pair runs as two parallel chains on the same input.
                g = fill_xplus(g, P[0]) | fill_xminus(g, P[1]);
                g = fill_yplus(g, P[2], lane) | fill_yminus(g, P[3], lane);
                if (conn == 8) {
                    const uint32_t gu0 = __shfl_up_sync(0xffffffffu, g, 1);
                    const uint32_t gd0 = __shfl_down_sync(0xffffffffu, g, 1);
                    const uint32_t gu = lane > 0 ? gu0 : 0u, gdn = lane < 31 ? gd0 : 0u;
                    g |= (P[4] & (gu << 1)) | (P[5] & (gdn << 1)) | (P[6] & (gu >> 1)) | (P[7] & (gdn >> 1));
                }
                if (!__any_sync(0xffffffffu, g != old)) break;
                if (it > 4096) __trap();  // cannot happen (monotone, <= 1024 pixels); fail loudly
            }
            uint32_t grew = g & ~initial;
            const bool changed = __any_sync(0xffffffffu, grew != 0);
            while (grew) {
                const int x = __ffs(grew) - 1;
                m[size_t(gy) * w + x0 + x] = 1;
                grew &= grew - 1u;
            }
            if (a.trace && lane == 0) atomicAdd(a.trace + 8 * (kTracePasses - 2), 1ull);  // tile visits
            if (changed) {
                if (flags) {
                    if (lane == 0) wl[nft * ((rounds + 1) % 3) + t] = 1;
                } else {
                    ff_enqueue3x3(wl, ntx, nty, tx, ty, rounds + 1);
                }
            }
        }
        if (a.trace && rounds < 8 && threadIdx.x == 0) atomicMax(a.trace + 8 * (kTracePasses - 4) + rounds, global_ns());
        grid_barrier(a.grid);
        ++rounds;
        if (!flags && __ldcg(ff_count(wl, nft, rounds)) == 0u) break;  // nothing queued: fixpoint reached
    }
    return rounds;
}

// BuildMask (dynamics_mask.cpp:98-104) on the full-resolution residual image.
// Stages: bit0 threshold, bit1 erode, bit2 floodfill, bit3 dilate (a stage
// that is off is the identity; without bit0 the input mask is mwork[0]).
// Pass A (one barrier): threshold + erode per 32x32 tile, growth bits, stamp
// reset. Floodfill rounds. Pass C: dilate per tile + CountMasked, closed by
// the all-reduce. The result lands in F.mask[0]; returns the masked count.
__device__ double build_mask(const TrackArgs& a, int stages, double* scratch, double* blk, double* red,
                             int* rounds) {
    const FrameView& F = a.F;
    const int w = F.K[0].w, h = F.K[0].h;
    const int stride = gridDim.x * blockDim.x;
    const MaskParams& M = a.mp;
    unsigned long long* mt = (a.trace && blockIdx.x == 0 && threadIdx.x == 0) ? a.trace + 8 * (kTracePasses - 1) : nullptr;
    if (mt) mt[0] = global_ns();
    const int re = (stages & 2) ? M.erode_radius : 0, rd = (stages & 8) ? M.dilate_radius : 0;
    const int ntx = (w + kMorphTile - 1) / kMorphTile, nty = (h + kMorphTile - 1) / kMorphTile;
    const uint8_t* input = F.mwork[0];
    uint8_t* seeds = F.mwork[1];
    const double thr = M.gamma * M.truncation * M.truncation;  // ThresholdResiduals (dynamics_mask.cpp:9-18)
    // free-space extension (off: 0): a valid residual whose signed sdf is
    // positive (bit 1 of valid, set by the residual pass only when enabled)
    // and whose square exceeds free_space^2 also seeds the mask
    const double fs2 = M.free_space > 0.0 ? M.free_space * M.free_space : INFINITY;
    const bool do_thr = stages & 1;
    if (re <= kMorphMaxR) {
        for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
            int nseed = 0;
            morph_tile<true>(t % ntx, t / ntx, w, h, re,
                             [&](int gx, int gy) -> bool {  // both loads issued together (no short-circuit)
                                 const int p = gy * w + gx;
                                 if (!do_thr) return __ldcg(input + p) != 0;
                                 const uint8_t valid = __ldcg(F.res_valid + p);
                                 const float sq = __ldcg(F.res_sq + p);
                                 return ((valid != 0) & (double(sq) > thr)) | ((valid & 2) != 0 && double(sq) > fs2);
                             },
                             seeds, nseed);
            if (stages & 4) {  // the floodfill's growth bits (same 32x32 tiling) and round-0 worklist
                grow_tile(F.depth0, reinterpret_cast<uint32_t*>(F.grow), w, h, t % ntx, t / ntx, M.theta,
                          M.connectivity);
                if (__syncthreads_or(nseed)) {
                    if (!ff_flag_mode(ntx * nty, a.dyn_bytes)) ff_enqueue3x3(F.ffstamp, ntx, nty, t % ntx, t / ntx, 0);
                    else if (threadIdx.x == 0) F.ffstamp[t] = 1;  // round 0's flags
                }
            }
        }
    } else {  // wide windows: threshold, then separable passes through global memory
        uint8_t* thr_img = F.mwork[2];
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < w * h; p += stride)
            thr_img[p] = do_thr ? (((__ldcg(F.res_valid + p) && double(__ldcg(F.res_sq + p)) > thr) ||
                                    ((__ldcg(F.res_valid + p) & 2) && double(__ldcg(F.res_sq + p)) > fs2)) ? 1 : 0)
                                : __ldcg(input + p);
        grid_barrier(a.grid);
        morph_pass(thr_img, F.grow, w, h, re, true, true);
        grid_barrier(a.grid);
        morph_pass(F.grow, seeds, w, h, re, true, false);
        grid_barrier(a.grid);  // F.grow is reused below
    }
    if ((stages & 4) && re > kMorphMaxR) {  // (the tiled path above did this with the erosion)
        for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
            grow_tile(F.depth0, reinterpret_cast<uint32_t*>(F.grow), w, h, t % ntx, t / ntx, M.theta, M.connectivity);
            int any = 0;
            const int x0 = (t % ntx) * kMorphTile, y0 = (t / ntx) * kMorphTile;
            for (int i = threadIdx.x; i < kMorphTile * kMorphTile; i += blockDim.x) {
                const int gx = x0 + i % kMorphTile, gy = y0 + i / kMorphTile;
                any |= (gx < w && gy < h && __ldcg(seeds + gy * w + gx)) ? 1 : 0;
            }
            if (__syncthreads_or(any)) {
                if (!ff_flag_mode(ntx * nty, a.dyn_bytes)) ff_enqueue3x3(F.ffstamp, ntx, nty, t % ntx, t / ntx, 0);
                else if (threadIdx.x == 0) F.ffstamp[t] = 1;
            }
        }
    }
    grid_barrier(a.grid);
    if (mt) mt[1] = mt[2] = mt[3] = global_ns();
    *rounds = 0;
    if (stages & 4) *rounds = floodfill(a, seeds, reinterpret_cast<const uint32_t*>(F.grow), w, h, M.connectivity);
    if (mt) mt[4] = global_ns();
    int cnt = 0;
    if (rd <= kMorphMaxR) {
        for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x)
            morph_tile<false>(t % ntx, t / ntx, w, h, rd, [&](int gx, int gy) { return __ldcg(seeds + gy * w + gx) != 0; },
                              F.mask[0], cnt);
    } else {
        morph_pass(seeds, F.mwork[2], w, h, rd, false, true);
        grid_barrier(a.grid);
        morph_pass(F.mwork[2], F.mask[0], w, h, rd, false, false);
        grid_barrier(a.grid);
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < w * h; p += stride) cnt += __ldcg(F.mask[0] + p) ? 1 : 0;
    }
    if (mt) mt[5] = global_ns();
    const double v[1] = {double(cnt)};
    block_grid_allreduce<1>(a.grid, v, scratch, red);
    if (mt) mt[6] = global_ns();
    return red[0];
}

__device__ void write_out(const TrackArgs& a, const RegState& st) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) a.out->pose[i] = st.pose().R[i];
        for (int i = 0; i < 3; ++i) a.out->pose[9 + i] = st.pose().t[i];
    }
}

}  // namespace

// The body of k_track (every mode); the kernel publishes CTA 0's pass tally after it.
__device__ __forceinline__ void track_main(const TrackArgs& a, RegState& st, double* scratch, double* blk,
                                           double* red, bool lead) {
    if ((a.mode == kModeFrame && a.dynamics) || a.mode == kModeMask) {  // floodfill worklists (ff_list)
        const int nft = ((a.F.K[0].w + kFfW - 1) / kFfW) * ((a.F.K[0].h + kFfH - 1) / kFfH);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * nft + kFfCounts; i += gridDim.x * blockDim.x)
            a.F.ffstamp[i] = (i < nft && !ff_flag_mode(nft, a.dyn_bytes)) ? -1 : 0;
    }

    if (a.mode == kModeLinearize || a.mode == kModeEvalDepth || a.mode == kModeEvalColor) {
        Pose P;
        for (int i = 0; i < 9; ++i) P.R[i] = a.pose_state[i];
        for (int i = 0; i < 3; ++i) P.t[i] = a.pose_state[9 + i];
        if (a.mode == kModeLinearize)
            pass<true>(a, 0, P, a.use_mask, false, a.reg.color_weight, scratch, blk, red);
        else if (a.mode == kModeEvalDepth)
            pass<false>(a, 0, P, a.use_mask, true, 0.0, scratch, blk, red);
        else
            pass<false>(a, 0, P, a.use_mask, false, 1.0, scratch, blk, red);
        if (lead)
            for (int i = 0; i < kAccN; ++i) a.out->acc[i] = red[i];
        return;
    }
    if (a.mode == kModeMask) {
        grid_barrier(a.grid);  // worklist reset above, before the erosion pass queues round 0
        int rounds = 0;
        const double cnt = build_mask(a, a.mask_stages, scratch, blk, red, &rounds);
        if (lead) {
            a.out->masked = (unsigned long long)cnt;
            a.out->rounds = rounds;
        }
        return;
    }

    if (a.mode == kModeFrame && a.vol_counters && __ldcg(a.vol_counters + kHalt)) {
        // An earlier frame of this batch overflowed the block budget: the host
        // throws ResourceLimitError at that frame, so this one must leave no
        // trace (no pose update, no allocation / integration: lost = 2 gates
        // the launches that follow).
        if (lead) a.out->lost = 2;
        return;
    }
    if (a.mode == kModePyramid) {  // BuildPyramid (registration.cpp:144-182) as a public entry point
        const FrameView& F = a.F;
        if (F.rgb0)  // LevelZero: ToIntensity (registration.cpp:119-126, image.hpp:85-91)
            for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < F.K[0].w * F.K[0].h; p += gridDim.x * blockDim.x) {
                const uint8_t* c = F.rgb0 + 3 * size_t(p);
                F.inten[0][p] = float(luma(__ldg(c), __ldg(c + 1), __ldg(c + 2)));
            }
        build_pyramid(a, true, a.use_mask);
        return;
    }
    Pose init;
    for (int i = 0; i < 9; ++i) init.R[i] = a.pose_state[i];
    for (int i = 0; i < 3; ++i) init.t[i] = a.pose_state[9 + i];
    if (a.mode == kModePassBench) {
        build_pyramid(a, true, false);
        const unsigned long long t0 = global_ns();
        for (int it = 0; it < a.bench_iters; ++it)
            pass<true>(a, a.bench_level, init, false, false, a.reg.color_weight, scratch, blk, red);
        if (lead) {
            a.out->final_error = double(global_ns() - t0) * 1e-3 / a.bench_iters;  // us per pass (barrier incl.)
            for (int i = 0; i < kAccN; ++i) a.out->acc[i] = red[i];
        }
        return;
    }
    const bool masked_reg = a.mode == kModeRegister && a.use_mask;
    build_pyramid(a, true, masked_reg);
    // kModeFrame: pipeline.cpp:79-122 (tracking part). Both registrations go
    // through one run_register site (one copy of the pass code for both).
    int registrations = 0, iterations = 0, rounds = 0;
    double masked = 0.0;
    bool reg_mask = masked_reg;
    for (int r = 0;; ++r) {
        run_register(a, r == 0 ? init : st.pose(), reg_mask, st, scratch, blk);  // registration 2 starts at 1's pose
        if (a.mode == kModeRegister || st.lost) break;
        registrations = r + 1;
        iterations += st.total;
        if (r == 1 || !a.dynamics) break;
        masked = build_mask(a, 15, scratch, blk, red, &rounds);
        if (!(masked > 0.0)) break;
        build_pyramid(a, false, true);
        __syncthreads();
        reg_mask = true;
    }

    if (a.mode == kModeRegister) {
        if (lead) {
            a.out->lost = st.lost;
            a.out->converged = st.converged;
            a.out->iterations = st.total;
            a.out->registrations = 1;
            a.out->valid = (unsigned long long)st.cur()[29];
            a.out->final_error = st.cur()[27] + a.reg.color_weight * st.cur()[28];
            for (int i = 0; i < kAccN; ++i) a.out->acc[i] = st.cur()[i];
        }
        write_out(a, st);
        return;
    }
    if (lead) {
        TrackOut* o = a.out;
        o->lost = st.lost;
        o->registrations = registrations;
        o->iterations = iterations;
        o->masked = (unsigned long long)masked;
        o->rounds = rounds;
        o->converged = st.lost ? 0 : st.converged;
        o->valid = st.lost ? 0ull : (unsigned long long)st.cur()[29];
        o->final_error = st.lost ? 0.0 : st.cur()[27] + a.reg.color_weight * st.cur()[28];
        if (!st.lost) {  // hold the previous pose on loss (pipeline.cpp:117-122)
            for (int i = 0; i < 9; ++i) a.pose_state[i] = st.pose().R[i];
            for (int i = 0; i < 3; ++i) a.pose_state[9 + i] = st.pose().t[i];
        }
        for (int i = 0; i < 12; ++i) o->pose[i] = a.pose_state[i];
        if (a.vol_counters) {  // frame bookkeeping for the allocate / cull / fuse launches that follow
            a.vol_counters[kBlocksBefore] = a.vol_counters[kNumBlocks];
            a.vol_counters[kVisible] = 0;
            a.vol_counters[kDdaVisits] = 0;
            a.vol_counters[kNewBlocks] = 0;
            a.vol_counters[kOverflow] = 0;
        }
    }
}

__global__ void __launch_bounds__(kTrackThreads, kTrackMinBlocks) k_track(TrackArgs a) {
    pdl_enter();
    __shared__ RegState st;
    __shared__ double scratch[(kTrackThreads / 32) * 32];
    __shared__ double blk[kAccN + 2];
    __shared__ double red[kAccN + 2];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (lead && a.out) {
        s_passes = 0;
        s_pixel_passes = 0.0;
    }
    if (threadIdx.x == 0) {
        s_trace_pass = 0;
        s_pxc_tag = 0;
    }
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l)  // static indices into the kernel parameters
        if (threadIdx.x == l) {
            LevelInfo& L = s_lvl[l];
            L.K = a.F.K[l];
            L.depth = l == 0 ? const_cast<float*>(a.F.depth0) : a.F.depth[l];
            L.inten = a.F.inten[l];
            L.mask = a.F.mask[l];
            const int npx = L.K.w * L.K.h, per = (npx + int(gridDim.x) - 1) / int(gridDim.x);
            const int start = min(npx, int(blockIdx.x) * per);
            L.per = per;
            L.end = min(npx, start + per);
            L.vbase = L.K.w > 0 ? start / L.K.w : 0;
            L.ubase = start - L.vbase * L.K.w;
        }
    for (int i = threadIdx.x; i < 768; i += blockDim.x) {
        const double w = i < 256 ? 0.2126 : (i < 512 ? 0.7152 : 0.0722);  // image.hpp:80-83
        s_luma_lut[i] = w * double(i & 255);
    }
    grid_init(a.grid);
#ifdef RF_LM_CLOCKS
    if (threadIdx.x < 18) s_lmacc[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) s_t0c = 0;
    LMC_ARM(0);
    __syncthreads();
#endif
    track_main(a, st, scratch, blk, red, lead);
#ifdef RF_LM_CLOCKS
    __syncthreads();
    if (a.trace && blockIdx.x == 0 && threadIdx.x < 18)
        a.trace[8 * (threadIdx.x < 8 ? 251 : (threadIdx.x < 16 ? 250 : 249)) + (threadIdx.x & 7)] = s_lmacc[threadIdx.x];
#endif
    if (lead && a.out) {
        a.out->passes = s_passes;
        a.out->pixel_passes = s_pixel_passes;
    }
}

}  // namespace rfb

// ---------------------------------------------------------------- diagnostics
namespace rfb {
// Back-to-back grid all-reduces (no pixel work): the fixed per-pass cost of
// the persistent tracking kernel's barrier. reduce = 0 is a bare barrier.
__global__ void __launch_bounds__(kTrackThreads, kTrackMinBlocks) k_grid_bench(GridCtx g, int iters, int reduce) {
    __shared__ double blk[32], red[32], scratch[(kTrackThreads / 32) * 32];
    grid_init(g);
    if (threadIdx.x < 32) blk[threadIdx.x] = double(blockIdx.x + threadIdx.x);
    __syncthreads();
    for (int i = 0; i < iters; ++i) {
        if (reduce == 1) {
            double v[kAccN];
            for (int k = 0; k < kAccN; ++k) v[k] = blk[k % 32];
            block_grid_allreduce<kAccN, false>(g, v, scratch, red);
        } else if (reduce == 2) {  // the CTA-local part only: transpose reduce + warp-0 sum
            double v[32];
            for (int k = 0; k < 32; ++k) v[k] = k < kAccN ? blk[k] : 0.0;
            scratch[(threadIdx.x >> 5) * 32 + (threadIdx.x & 31)] = warp_transpose_reduce(v);
            __syncthreads();
            if (threadIdx.x < kAccN) {
                double t = 0.0;
                for (int w = 0; w < int(blockDim.x >> 5); ++w) t += scratch[w * 32 + threadIdx.x];
                red[threadIdx.x] = t;
            }
            __syncthreads();
            if (threadIdx.x < 32) blk[threadIdx.x] = red[threadIdx.x] * 1e-30 + blk[threadIdx.x];
            __syncthreads();
        } else if (reduce == 3) {  // one value: the grid exchange without the 30-wide fold
            double v[1] = {blk[0]};
            block_grid_allreduce<1, false>(g, v, scratch, red);
        } else if (reduce == 4) {  // the exchange alone: thread 0 stores a line, every CTA polls all lines
            const unsigned int bar = s_ll_bar;
            const uint32_t flag = (g.seq << 12) | (bar & 0xFFFu);
            uint4* buf = g.ll + size_t(bar & 1u) * gridDim.x * 32;
            __syncthreads();
            if (threadIdx.x == 0) {
                st_line(buf + blockIdx.x * 32, blk[0], flag);
                s_ll_bar = bar + 1u;
            }
            double acc = 0.0;
            for (int i = threadIdx.x; i < int(gridDim.x); i += blockDim.x) {
                uint4 t = ld_line(buf + i * 32);
                while (!line_ready(t, flag)) t = ld_line(buf + i * 32);
                acc += line_value(t);
            }
            if (acc == 12345.0) blk[1] = acc;
            __syncthreads();
        } else {
            grid_barrier(g);
        }
    }
}

// Latency of one LM step on one thread (lm_solve + ExpMap + pose product),
// the serial section every CTA runs between two pixel passes. Cycles per
// step are written to out[0..2] (solve, expmap+compose, total).
__global__ void k_lm_bench(int iters, double* out) {
    __shared__ double acc[kAccN];
    __shared__ double delta[6];
    if (threadIdx.x == 0) {
        for (int i = 0; i < kAccN; ++i) acc[i] = 0.0;
        for (int i = 0; i < 6; ++i) {
            acc[hidx(i, i)] = 10.0 + i;
            if (i < 5) acc[hidx(i, i + 1)] = 0.5;
            acc[21 + i] = 0.01 * (i + 1);
        }
    }
    __syncwarp();
    Pose pose{};
    for (int i = 0; i < 3; ++i) pose.R[4 * i] = 1.0;
    long long t_solve = 0, t_rest = 0;
    double lambda = 1e-4;
    for (int it = 0; it < iters; ++it) {
        const long long t0 = clock64();
        const bool ok = lm_solve(acc, lambda, delta);
        const long long t1 = clock64();
        if (threadIdx.x != 0) continue;
        double d[6];
        for (int i = 0; i < 6; ++i) d[i] = delta[i];
        const Pose p0 = pose;
        expmap_compose(d, p0, pose);
        const long long t2 = clock64();
        t_solve += t1 - t0;
        t_rest += t2 - t1;
        lambda = ok ? lambda * 1.0000001 : lambda;
        acc[21] += pose.t[0] * 1e-12;  // keep the chain live
    }
    if (threadIdx.x != 0) return;
    out[0] = double(t_solve) / iters;
    out[1] = double(t_rest) / iters;
    out[2] = double(t_solve + t_rest) / iters;
}
}  // namespace rfb
