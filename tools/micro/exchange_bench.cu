// Grid all-reduce exchange microbenchmark (B200, 1 CTA x 384 threads per SM,
// cooperative launch): the flagged-line exchange of k_track (every CTA folds
// every CTA's 30-double row from L2) against a cluster pre-reduction where
// the CTAs of a cluster combine over DSMEM first and only cluster leaders
// exchange through L2 (followers get the result over DSMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange_bench exchange_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

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
// generic-address (DSMEM-capable) flagged lines, cluster scope
__device__ __forceinline__ void st_gen(uint4* p, uint4 v) {
    asm volatile("st.relaxed.cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_gen(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double val(uint4 v) { return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x)); }

// Fold rows [0, n) of element j in CTA-index order by chunk c (rows c, c + nw, ...), all
// of the chunk's rows in flight at once (as k_track does).
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
            if (r[k].y != flag || r[k].w != flag) {
                ++missing;
                r[k] = ld_line(buf + (c + k * nw) * 32 + j);
            }
        if (!missing) break;
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kRows; ++k) s += val(r[k]);
    return s;
}

// mode 0: flat (every CTA folds all G rows). mode 1: cluster pre-reduction over DSMEM.
__global__ void __launch_bounds__(384, 1) k_ex(uint4* lines, int iters, int mode, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double s_fold[12][32];
    __shared__ uint4 s_in[8][32];   // leader: lines from the cluster's other CTAs
    __shared__ uint4 s_res[32];     // follower: the result lines from the leader
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int G = gridDim.x;
    const int cs = mode ? int(cl.num_blocks()) : 1, rank = mode ? int(cl.block_rank()) : 0;
    const int nlead = G / cs, lead_id = blockIdx.x / cs;
    for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) (&s_in[0][0])[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 32; i += blockDim.x) s_res[i] = make_uint4(0, 0, 0, 0);
    if (mode) cl.sync();
    double my = double(blockIdx.x) * 1e-3;
    for (int it = 0; it < iters; ++it) {
        const uint32_t flag = uint32_t(it + 1);
        uint4* buf = lines + size_t(it & 1) * G * 32;
        if (mode == 0) {
            if (warp == 0 && lane < NV) st_line(buf + blockIdx.x * 32 + lane, my + lane, flag);
            const double s = lane < NV ? fold_rows(buf, G, lane, warp, nw, flag) : 0.0;
            s_fold[warp][lane] = s;
            __syncthreads();
            if (threadIdx.x < NV) {
                double t = 0.0;
                for (int c = 0; c < nw; ++c) t += s_fold[c][threadIdx.x];
                my = t * 1e-9 + my;
            }
            __syncthreads();
        } else {
            if (rank != 0) {  // follower: push the row into the leader's shared memory
                if (warp == 0 && lane < NV) {
                    uint4* dst = cl.map_shared_rank(&s_in[rank][0], 0);
                    const unsigned long long b = (unsigned long long)__double_as_longlong(my + lane);
                    st_gen(dst + lane, make_uint4(uint32_t(b), flag, uint32_t(b >> 32), flag));
                }
            } else if (warp == 0 && lane < NV) {  // leader: combine the cluster, then publish one row
                double s = my + lane;
                for (int r = 1; r < cs; ++r) {
                    uint4 t = ld_gen(&s_in[r][lane]);
                    while (t.y != flag || t.w != flag) t = ld_gen(&s_in[r][lane]);
                    s += val(t);
                }
                st_line(buf + lead_id * 32 + lane, s, flag);
            }
            double tot = 0.0;
            if (rank == 0) {
                const double s = lane < NV ? fold_rows(buf, nlead, lane, warp, nw, flag) : 0.0;
                s_fold[warp][lane] = s;
                __syncthreads();
                if (threadIdx.x < NV) {
                    for (int c = 0; c < nw; ++c) tot += s_fold[c][threadIdx.x];
                    for (int r = 1; r < cs; ++r) {  // forward the result to the followers
                        uint4* dst = cl.map_shared_rank(&s_res[0], r);
                        const unsigned long long b = (unsigned long long)__double_as_longlong(tot);
                        st_gen(dst + threadIdx.x, make_uint4(uint32_t(b), flag, uint32_t(b >> 32), flag));
                    }
                }
            } else if (threadIdx.x < NV) {
                uint4 t = ld_gen(&s_res[threadIdx.x]);
                while (t.y != flag || t.w != flag) t = ld_gen(&s_res[threadIdx.x]);
                tot = val(t);
            }
            if (threadIdx.x < NV) my = tot * 1e-9 + my;
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = my;
    if (mode) cl.sync();
}

int main() {
    uint4* lines;
    double* out;
    cudaMalloc(&lines, 2 * 148 * 32 * sizeof(uint4));
    cudaMalloc(&out, 148 * sizeof(double));
    cudaFuncSetAttribute(k_ex, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_ex, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    const int iters = 2000;
    for (int cs : {1, 2, 4}) {
        cudaMemset(lines, 0, 2 * 148 * 32 * sizeof(uint4));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[2];
        int na = 0;
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na++].val.cooperative = 1;
        if (cs > 1) {
            attr[na].id = cudaLaunchAttributeClusterDimension;
            attr[na].val.clusterDim.x = cs;
            attr[na].val.clusterDim.y = 1;
            attr[na++].val.clusterDim.z = 1;
        }
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = 150 * 1024;  // one CTA per SM, as k_track
        cfg.attrs = attr;
        cfg.numAttrs = na;
        int grid = 148;
        if (cs > 1) {
            int ncl = 0;
            cfg.gridDim = dim3(cs);
            cudaOccupancyMaxActiveClusters(&ncl, (void*)k_ex, &cfg);
            grid = ncl * cs;
        }
        cfg.gridDim = dim3(grid);
        const int mode = cs > 1;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaLaunchKernelEx(&cfg, k_ex, lines, 10, mode, out);  // warm
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_ex, lines, iters, mode, out);
        cudaEventRecord(e1);
        cudaError_t e2 = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cluster %d: grid %3d  %.3f us per 30-value exchange  (%s / %s)\n", cs, grid, 1e3 * ms / iters,
               cudaGetErrorString(e), cudaGetErrorString(e2));
    }
}
