// Grid-wide barrier with a deterministic all-reduce for cooperative
// (persistent) kernels: one CTA per SM slot, every CTA runs the same control
// flow, so device-resident loops (the LM iterations, the floodfill fixpoint)
// need no host round trip.
#pragma once

#include "rf_common.cuh"

namespace rfb {

constexpr int kRedStride = 32;  // doubles per CTA partial slot

struct GridCtx {
    GridSync* sync;      // zero-initialised once
    double* partials;    // gridDim.x * kRedStride
    double* result;      // kRedStride
};

// Sum over the CTA of NV doubles held per thread. Deterministic tree:
// warp shuffles, then warps folded in order. Result valid in `out` (smem)
// for all threads after return. `scratch` needs (blockDim/32) * NV doubles.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double* scratch, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double x = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) scratch[warp * NV + i] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += scratch[w * NV + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

// All CTAs call with their CTA-level vector `mine` (smem, NV entries). On
// return `out` (smem) holds the sum over CTAs folded in CTA index order.
// NV == 0 is a plain grid barrier.
template <int NV>
__device__ __noinline__ void grid_allreduce(const GridCtx& g, const double* mine, double* out) {
    __shared__ unsigned int s_last, s_gen;
    if (NV > 0 && threadIdx.x < NV) {
        g.partials[blockIdx.x * kRedStride + threadIdx.x] = mine[threadIdx.x];
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire(&g.sync->gen);
        __threadfence();
        const unsigned int prev = atomicAdd(&g.sync->arrive, 1u);
        s_gen = gen;
        s_last = (prev == gridDim.x - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (NV > 0) {
            __shared__ double red[32][NV > 0 ? NV : 1];
            const int nchunk = blockDim.x >> 5;
            const int j = threadIdx.x & 31, c = threadIdx.x >> 5;
            const int G = gridDim.x;
            const int per = (G + nchunk - 1) / nchunk;
            if (j < NV) {
                double s = 0.0;
                const int lo = c * per, hi = min(G, lo + per);
                for (int i = lo; i < hi; ++i) s += __ldcg(g.partials + i * kRedStride + j);
                red[c][j] = s;
            }
            __syncthreads();
            if (threadIdx.x < NV) {
                double s = 0.0;
                for (int cc = 0; cc < nchunk; ++cc) s += red[cc][threadIdx.x];
                out[threadIdx.x] = s;
                g.result[threadIdx.x] = s;
                __threadfence();
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            g.sync->arrive = 0u;
            __threadfence();
            st_release(&g.sync->gen, s_gen + 1u);
        }
    } else {
        if (threadIdx.x == 0) {
            // Bounded spin: a co-residency bug must fail loudly, never hang the GPU.
            unsigned long long spins = 0;
            while (ld_acquire(&g.sync->gen) == s_gen) {
                if (++spins > (1ull << 25)) __trap();  // ~10+ s of L2 round trips
            }
        }
        __syncthreads();
        if (NV > 0 && threadIdx.x < NV) out[threadIdx.x] = __ldcg(g.result + threadIdx.x);
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(const GridCtx& g) { grid_allreduce<0>(g, nullptr, nullptr); }

}  // namespace rfb
