// Grid-wide barrier with a deterministic all-reduce for cooperative
// (persistent) kernels: every CTA runs the same control flow, so
// device-resident loops (the LM iterations, the floodfill fixpoint) need no
// host round trip.
//
// Design (one L2 round trip on the critical path): each CTA writes its
// partial vector into a double-buffered slot, arrives on a monotonically
// increasing 64-bit counter with one release atomic, polls it relaxed until
// the barrier's target count, then every CTA folds all partials itself in CTA
// index order. No "last CTA reduces and re-publishes" chain, no reset inside
// a launch: consecutive launches alternate between two counters and each
// launch zeroes the one the next launch will use.
#pragma once

#include "rf_common.cuh"

namespace rfb {

constexpr int kRedStride = 32;  // doubles per CTA partial slot

struct GridCtx {
    GridSync* sync;      // counters live here (zero-initialised once)
    double* partials;    // 2 * gridDim.x * kRedStride (double-buffered)
    double* result;      // unused by the current barrier (kept for ABI stability)
    int parity;          // which counter this launch uses (host alternates)
};

__shared__ unsigned int s_grid_bar;  // barriers completed by this CTA in this launch

__device__ __forceinline__ unsigned long long* grid_counter(const GridCtx& g, int parity, int lane) {
    return &g.sync->lane[parity][lane][0];
}

// Call once at kernel start, before any barrier, from all threads.
__device__ __forceinline__ void grid_init(const GridCtx& g) {
    if (threadIdx.x == 0) s_grid_bar = 0;
    if (blockIdx.x == 0 && threadIdx.x < kArriveLanes)
        *grid_counter(g, g.parity ^ 1, threadIdx.x) = 0ull;  // next launch's counters
    __syncthreads();
}

// Butterfly transpose-reduction of 32 per-lane values: after 31 shuffles lane
// j holds the warp total of value j (fixed tree => deterministic).
__device__ __forceinline__ double warp_transpose_reduce(double (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = upper ? v[i] : v[i + o];
            const double keep = upper ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// CTA sum of NV (<= 32) doubles per thread. Result in `out` (smem) for all
// threads after return; `scratch` holds (blockDim/32) * 32 doubles.
template <int NV>
__device__ __forceinline__ void block_reduce(const double (&in)[NV], double* scratch, double* out) {
    static_assert(NV <= 32, "block_reduce handles up to 32 values");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i < NV ? in[i] : 0.0;
    scratch[warp * 32 + lane] = warp_transpose_reduce(v);
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += scratch[w * 32 + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifndef RF_POLL_ACQ
#define RF_POLL_ACQ 0
#endif

struct NoHook {
    __device__ void operator()() const {}
};

// Warp 0: arrive on the barrier's counter (after the CTA's partial stores,
// which warp 0 has observed through a CTA or warp barrier), run `hook` on
// lane 0 while the arrivals propagate, and poll until every CTA has arrived.
template <class Hook = NoHook>
__device__ __forceinline__ void grid_arrive_wait(const GridCtx& g, unsigned int bar, const Hook& hook = Hook()) {
    const int G = gridDim.x;
    // CTAs arrive on kArriveLanes counters (blockIdx % lanes) so the
    // arrival atomics spread over separate L2 lines; lanes 0..7 of warp 0
    // each poll one counter.
    const int lane = threadIdx.x;
    if (lane == 0) {  // release is cumulative: covers the CTA's partial stores ordered by the barrier
        red_release_add(grid_counter(g, g.parity, blockIdx.x % kArriveLanes), 1ull);
        hook();
    }
    const int l = lane % kArriveLanes;
    const unsigned long long per = (unsigned long long)(G / kArriveLanes + (l < G % kArriveLanes ? 1 : 0));
    const unsigned long long target = (unsigned long long)(bar + 1u) * per;
    const unsigned long long* cnt = grid_counter(g, g.parity, l);
    // Relaxed polling, then one acquire. Bounded: a co-residency bug must
    // fail loudly, never hang the GPU.
    unsigned long long spins = 0;
#if RF_POLL_ACQ
    // acquire polling: the load that sees the target is the acquire (no extra L2 trip)
    while (!__all_sync(0xffffffffu, ld_acquire_u64(cnt) >= target)) {
        if (++spins > (1ull << 26)) __trap();
    }
#else
    while (!__all_sync(0xffffffffu, ld_relaxed_u64(cnt) >= target)) {
        if (++spins > (1ull << 26)) __trap();
    }
    (void)ld_acquire_u64(cnt);
#endif
    if (lane == 0) s_grid_bar = bar + 1u;
}

// All threads, after grid_arrive_wait: `out` (smem) = the sum of every CTA's
// partial, folded in CTA index order.
template <int NV>
__device__ __forceinline__ void grid_fold(const double* buf, double* out) {
    const int G = gridDim.x;
    __shared__ double red[32][32];
    const int j = threadIdx.x & 31, c = threadIdx.x >> 5, nchunk = blockDim.x >> 5;
    double s = 0.0;
    if (j < NV) {
        // chunk c folds CTA rows c, c+nchunk, ... in order; all of the
        // chunk's loads are issued before the first add (one L2 latency).
        constexpr int kRows = 24;
        double v[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const int i = c + r * nchunk;
            v[r] = i < G ? __ldcg(buf + i * kRedStride + j) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) s += v[r];
        for (int i = c + kRows * nchunk; i < G; i += nchunk) s += __ldcg(buf + i * kRedStride + j);
    }
    red[c][j] = s;
    __syncthreads();
    if (threadIdx.x < NV) {
        double t = 0.0;
        for (int cc = 0; cc < nchunk; ++cc) t += red[cc][threadIdx.x];
        out[threadIdx.x] = t;
    }
}

// All CTAs call with their CTA vector `mine` (smem, NV entries). On return
// `out` (smem) holds the sum over CTAs folded in CTA index order (identical
// in every CTA, independent of arrival order). NV == 0 is a plain barrier.
// Inlined at every call site: as a __noinline__ call the ABI spilled live state
// to the stack around each barrier (912 B stack, 1413 vs 1532 frames/s).
#ifndef RF_GRID_NOINLINE
#define RF_GRID_NOINLINE 0
#endif
#if RF_GRID_NOINLINE
#define RF_GRID_INLINE __noinline__
#else
#define RF_GRID_INLINE __forceinline__
#endif
template <int NV>
__device__ RF_GRID_INLINE void grid_allreduce(const GridCtx& g, const double* mine, double* out) {
    const int G = gridDim.x;
    const unsigned int bar = s_grid_bar;  // read before thread 0 advances it
    double* buf = g.partials + size_t(bar & 1u) * G * kRedStride;
    if (NV > 0 && threadIdx.x < NV) __stcg(buf + blockIdx.x * kRedStride + threadIdx.x, mine[threadIdx.x]);
    __syncthreads();
    if (threadIdx.x < 32) grid_arrive_wait(g, bar);
    __syncthreads();
    if (NV > 0) grid_fold<NV>(buf, out);
    __syncthreads();
}

// Block sum + grid all-reduce of NV (<= 30) per-thread doubles in one: warp
// partials by the transpose reduce, then warp 0 sums them (fixed warp order)
// and stores the CTA vector straight into its grid slot before arriving, with
// no CTA-wide barrier between the block sum and the arrival. Same sums, same
// order as block_reduce + grid_allreduce.
template <int NV, class Hook = NoHook>
__device__ __forceinline__ void block_grid_allreduce(const GridCtx& g, const double (&in)[NV], double* scratch,
                                                     double* out, const Hook& hook = Hook()) {
    static_assert(NV <= 32, "one warp holds the CTA vector");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i < NV ? in[i] : 0.0;
    scratch[warp * 32 + lane] = warp_transpose_reduce(v);
    const unsigned int bar = s_grid_bar;  // read before warp 0 advances it (it does so after the barrier)
    double* buf = g.partials + size_t(bar & 1u) * gridDim.x * kRedStride;
    __syncthreads();
    if (warp == 0) {
        if (lane < NV) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += scratch[w * 32 + lane];
            __stcg(buf + blockIdx.x * kRedStride + lane, s);
        }
        __syncwarp();  // orders the lanes' partial stores before lane 0's release
        grid_arrive_wait(g, bar, hook);
    }
    __syncthreads();
    grid_fold<NV>(buf, out);
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(const GridCtx& g) { grid_allreduce<0>(g, nullptr, nullptr); }

}  // namespace rfb
