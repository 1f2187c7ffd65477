// Volume raycast: the ray-march of RenderVirtualDepth
// (depth_refinement.cpp:32-79), one thread per pixel, marching the sparse
// volume through the hash with the reference's accumulated z += tau/2 steps,
// 8 bisections and the final linear interpolation.
#include "rf_volume.cuh"

namespace rfb {

__device__ __forceinline__ bool sdf_at(const VolumeView& V, const Pose& P, double z, double d0, double d1,
                                       double& val) {
    double p[3];
    pose_apply(P, z * d0, z * d1, z * 1.0, p);
    CellSample cs;
    if (!sample_point<false, false>(V, p, cs)) return false;
    val = cs.sdf;
    return true;
}

__global__ void k_raycast(RaycastArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.K.w * a.K.h) return;
    const int u = i % a.K.w, v = i / a.K.w;
    if (a.raw) {
        const float r = a.raw[i];
        if (depth_valid(r)) {
            a.refined[i] = r;
            if (!a.out) return;
        }
    }
    const double step = a.V.truncation / 2.0;
    const double d0 = (double(u) - a.K.cx) / a.K.fx, d1 = (double(v) - a.K.cy) / a.K.fy;
    double prev_z = 0.0, prev_sdf = 0.0;
    bool prev_valid = false;
    float out = 0.f;
    for (double z = a.V.min_depth; z <= a.V.max_depth; z += step) {
        double s;
        if (!sdf_at(a.V, a.view, z, d0, d1, s)) {
            prev_valid = false;
            continue;
        }
        if (prev_valid && prev_sdf > 0.0 && s <= 0.0) {
            double lo = prev_z, hi = z, lo_sdf = prev_sdf;
            for (int it = 0; it < a.bisections; ++it) {
                const double mid = 0.5 * (lo + hi);
                double m;
                if (!sdf_at(a.V, a.view, mid, d0, d1, m)) break;
                if (m > 0.0) {
                    lo = mid;
                    lo_sdf = m;
                } else {
                    hi = mid;
                }
            }
            double hs;
            const bool hv = sdf_at(a.V, a.view, hi, d0, d1, hs);
            double crossing = 0.5 * (lo + hi);
            if (hv && lo_sdf - hs > 1e-12) crossing = lo + (hi - lo) * lo_sdf / (lo_sdf - hs);
            out = float(crossing);
            break;
        }
        prev_z = z;
        prev_sdf = s;
        prev_valid = true;
    }
    if (a.out) a.out[i] = out;
    if (a.raw && !depth_valid(a.raw[i])) a.refined[i] = depth_valid(out) ? out : a.far_value;
}

}  // namespace rfb
