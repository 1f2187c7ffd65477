// Grid all-reduce of 30 doubles across 148 CTAs (one 384-thread CTA per SM,
// cooperative launch), two exchange shapes over flagged 16-byte lines:
//   flat  — every CTA folds every CTA's row (k_track's shape: 148 x 148 x 480 B
//           = 10.5 MB of L2 reads per exchange);
//   rs-ag — reduce-scatter + all-gather: CTA j < 30 folds column j of the 148
//           rows (fixed tree order) and publishes one line; every CTA then
//           reads the 30 result lines (~150 KB of L2 reads, one more hop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rsag_bench rsag_bench.cu
#include <cstdio>
#include <cstdint>

constexpr int NV = 30;
__device__ __forceinline__ void st_line(uint4* p, double v, uint32_t flag) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(uint32_t(b)), "r"(flag),
                 "r"(uint32_t(b >> 32)), "r"(flag) : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ bool ready(uint4 v, uint32_t f) { return v.y == f && v.w == f; }
__device__ __forceinline__ double val(uint4 v) { return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x)); }

__device__ double fold_rows(const uint4* buf, int n, int j, int c, int nw, uint32_t flag) {
    constexpr int kRows = 13;
    uint4 r[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
        const int i = c + k * nw;
        r[k] = i < n ? ld_line(buf + i * 32 + j) : make_uint4(0u, flag, 0u, flag);
    }
    for (;;) {
        int missing = 0;
#pragma unroll
        for (int k = 0; k < kRows; ++k)
            if (!ready(r[k], flag)) {
                ++missing;
                r[k] = ld_line(buf + (c + k * nw) * 32 + j);
            }
        if (!missing) break;
    }
    double v[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) v[k] = val(r[k]);
#pragma unroll
    for (int h = 1; h < kRows; h *= 2)
#pragma unroll
        for (int i = 0; i + h < kRows; i += 2 * h) v[i] += v[i + h];
    return v[0];
}

__global__ void __launch_bounds__(384, 1) k_ex(uint4* rows, uint4* res, int iters, int mode, int spread, double* out) {
    __shared__ double s_fold[12][32];
    __shared__ double s_part[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int G = gridDim.x;
    double my = double(blockIdx.x) * 1e-3;
    for (int it = 0; it < iters; ++it) {
        const uint32_t flag = uint32_t(it + 1);
        uint4* buf = rows + size_t(it & 1) * G * 32;
        uint4* rbuf = res + size_t(it & 1) * 32;
        if (warp == 0 && lane < NV) st_line(buf + blockIdx.x * 32 + lane, my + lane, flag);
        double tot = 0.0;
        if (mode == 0) {
            const double s = lane < NV ? fold_rows(buf, G, lane, warp, nw, flag) : 0.0;
            s_fold[warp][lane] = s;
            __syncthreads();
            if (threadIdx.x < NV) {
                double v[12];
#pragma unroll
                for (int c = 0; c < 12; ++c) v[c] = s_fold[c][threadIdx.x];
#pragma unroll
                for (int h = 1; h < 12; h *= 2)
#pragma unroll
                    for (int i = 0; i + h < 12; i += 2 * h) v[i] += v[i + h];
                tot = v[0];
            }
        } else {
            // reducer CTAs: value j on CTA j * spread (spread 1: CTAs 0..29; spread 4: every 4th CTA)
            const int j = (blockIdx.x % spread == 0) ? int(blockIdx.x) / spread : NV;
            if (j < NV) {
                // threads 0..G-1 each poll one row's line of value j
                double x = 0.0;
                if (threadIdx.x < G) {
                    uint4 t = ld_line(buf + threadIdx.x * 32 + j);
                    while (!ready(t, flag)) t = ld_line(buf + threadIdx.x * 32 + j);
                    x = val(t);
                }
                if (warp < 5) {
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                    if (lane == 0) s_part[warp] = x;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    const double s = ((s_part[0] + s_part[1]) + (s_part[2] + s_part[3])) + s_part[4];
                    st_line(rbuf + j, s, flag);
                }
            }
            if (threadIdx.x < NV) {
                uint4 t = ld_line(rbuf + threadIdx.x);
                while (!ready(t, flag)) t = ld_line(rbuf + threadIdx.x);
                tot = val(t);
            }
        }
        if (threadIdx.x < NV) my = tot * 1e-9 + my;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = my;
}

int main() {
    uint4 *rows, *res;
    double* out;
    cudaMalloc(&rows, 2 * 148 * 32 * sizeof(uint4));
    cudaMalloc(&res, 2 * 32 * sizeof(uint4));
    cudaMalloc(&out, 148 * sizeof(double));
    cudaFuncSetAttribute(k_ex, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    const int iters = 2000;
    for (int v : {0, 1, 2, 0, 1, 2}) {
        const int mode = v > 0, spread = v == 2 ? 4 : 1;
        cudaMemset(rows, 0, 2 * 148 * 32 * sizeof(uint4));
        cudaMemset(res, 0, 2 * 32 * sizeof(uint4));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.blockDim = dim3(384);
        cfg.gridDim = dim3(148);
        cfg.dynamicSmemBytes = 150 * 1024;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaLaunchKernelEx(&cfg, k_ex, rows, res, 10, mode, spread, out);
        cudaMemset(rows, 0, 2 * 148 * 32 * sizeof(uint4));
        cudaMemset(res, 0, 2 * 32 * sizeof(uint4));
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_ex, rows, res, iters, mode, spread, out);
        cudaEventRecord(e1);
        cudaError_t e2 = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-14s %.3f us per 30-value all-reduce  (%s / %s)\n", v == 0 ? "flat" : (v == 1 ? "rs-ag" : "rs-ag spread4"),
               1e3 * ms / iters, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
}
