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
constexpr int kGridThreads = 384;  // CTA size of the cooperative kernels that use these primitives
constexpr int kGridWarps = kGridThreads / 32;

struct GridCtx {
    GridSync* sync;      // counters live here (zero-initialised once)
    double* partials;    // 2 * gridDim.x * kRedStride (double-buffered)
    double* result;      // unused by the current barrier (kept for ABI stability)
    int parity;          // which counter this launch uses (host alternates)
    uint4* ll;           // all-reduce lines: 2 * gridDim.x * 32 (double-buffered), see block_grid_allreduce
    uint32_t seq;        // launch sequence number (host, 1..2^20-1): flags are (seq << 12) | reduce index
};

__shared__ unsigned int s_grid_bar;  // barriers completed by this CTA in this launch
__shared__ unsigned int s_ll_bar;    // all-reduces completed by this CTA in this launch
__shared__ double s_fold[32][32];    // per-chunk sums of the all-reduce fold

__device__ __forceinline__ unsigned long long* grid_counter(const GridCtx& g, int parity, int lane) {
    return &g.sync->lane[parity][lane][0];
}

// Call once at kernel start, before any barrier, from all threads.
__device__ __forceinline__ void grid_init(const GridCtx& g) {
    if (threadIdx.x == 0) {
        s_grid_bar = 0;
        s_ll_bar = 0;
    }
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

// Fixed-shape pairwise sums (deterministic, log-depth dependency chains
// instead of one add per term): N values in registers, and the first n <= N
// values at stride `stride` (missing terms are 0.0).
template <int N>
__device__ __forceinline__ double tree_sum_regs(double (&v)[N]) {
#pragma unroll
    for (int h = 1; h < N; h *= 2)
#pragma unroll
        for (int i = 0; i + h < N; i += 2 * h) v[i] += v[i + h];
    return v[0];
}
template <int N>
__device__ __forceinline__ double tree_sum(const double* p, int stride, int n) {
    double v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = i < n ? p[i * stride] : 0.0;
    return tree_sum_regs(v);
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
    while (!__all_sync(0xffffffffu, ld_relaxed_u64(cnt) >= target)) {
        if (++spins > (1ull << 26)) __trap();
    }
    (void)ld_acquire_u64(cnt);
    if (lane == 0) s_grid_bar = bar + 1u;
}

// Grid-wide barrier with release/acquire semantics (global writes before it
// are visible to every CTA after it): warp 0 arrives on the launch's counter
// and polls it. Inlined at every call site (a __noinline__ call spilled live
// state around each barrier).
__device__ __forceinline__ void grid_barrier(const GridCtx& g) {
    const unsigned int bar = s_grid_bar;  // read before thread 0 advances it
    __syncthreads();
    if (threadIdx.x < 32) grid_arrive_wait(g, bar);
    __syncthreads();
}

// Flagged lines (the low-latency protocol of NCCL's LL transport): a double
// travels as one 16-byte store {lo32, flag, hi32, flag}; each 8-byte half is
// single-copy atomic, so a reader that sees the expected flag in both halves
// holds the complete value. No fence, no counter, no acquire round trip.
#define RF_LINE_SCOPE "relaxed.gpu"  // STRONG.GPU (volatile, STRONG.SYS, measured 0.7% slower)
__device__ __forceinline__ void st_line(uint4* p, double v, uint32_t flag) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    asm volatile("st." RF_LINE_SCOPE ".global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(uint32_t(b)), "r"(flag),
                 "r"(uint32_t(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_line(const uint4* p) {
    uint4 v;
    asm volatile("ld." RF_LINE_SCOPE ".global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ bool line_ready(const uint4& v, uint32_t flag) { return v.y == flag && v.w == flag; }
__device__ __forceinline__ double line_value(const uint4& v) {
    return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}

// Block sum + grid all-reduce of NV (<= 30) per-thread doubles. Warp
// partials by the transpose reduce, warp 0 sums them (fixed warp order) and
// stores the CTA's vector as flagged lines; then every CTA folds all CTAs'
// lines in CTA index order as they arrive (chunk c of 32 threads folds rows
// c, c + nchunk, ...; each thread polls only the rows it still misses).
// Deterministic: the sums do not depend on arrival order. The critical path is
// the partials' one-way trip to L2 plus one polling round trip.
// kPublish: the CTAs wrote global data before this call that others read after
// it (residual images, masks): the partial store then acts as a release
// (fence after the CTA barrier) and the observation of all partials as an
// acquire. `hook` runs on thread 0 right after its CTA's partial is stored.
// Double buffering by the reduce index is safe: a CTA writes reduce i + 2 only
// after every CTA's partial of i + 1, i.e. after every CTA finished folding i.
// `warp_active` false: the warp's values are all zero (no pixels); it skips
// the transpose and contributes zeros (the same sums bit for bit: x + 0.0 = x).
template <int NV, bool kPublish = true, class Hook = NoHook>
__device__ __forceinline__ void block_grid_allreduce(const GridCtx& g, const double (&in)[NV], double* scratch,
                                                     double* out, const Hook& hook = Hook(),
                                                     bool warp_active = true) {
    static_assert(NV <= 32, "one warp holds the CTA vector");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kGridWarps;
    const int G = gridDim.x;
    if (NV == 1) {  // one value: a plain butterfly (fixed tree, deterministic)
        double t = in[0];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        scratch[warp * 32 + lane] = lane == 0 ? t : 0.0;
    } else if (warp_active) {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = i < NV ? in[i] : 0.0;
        scratch[warp * 32 + lane] = warp_transpose_reduce(v);
    } else {
        scratch[warp * 32 + lane] = 0.0;
    }
    const unsigned int bar = s_ll_bar;  // read before lane 0 of warp 0 advances it (after the barrier below)
    const uint32_t flag = (g.seq << 12) | (bar & 0xFFFu);
    uint4* buf = g.ll + size_t(bar & 1u) * G * 32;
    __syncthreads();
    if (warp == 0) {
        double sum = 0.0;
        if (lane < NV) sum = tree_sum<kGridWarps>(scratch + lane, 32, nw);
        if (kPublish) __threadfence();  // release: the CTA's writes (ordered by the barrier above) first
        if (lane < NV) st_line(buf + blockIdx.x * 32 + lane, sum, flag);
        if (lane == 0) {
            hook();
            s_ll_bar = bar + 1u;
        }
    }
    const int j = lane, c = warp;
    double s = 0.0;
    if (j < NV) {
        constexpr int kRows = 13;  // rows per chunk in flight (148 CTAs / 12 warps)
        uint4 r[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            const int i = c + k * nw;
            r[k] = i < G ? ld_line(buf + i * 32 + j) : make_uint4(0u, flag, 0u, flag);
        }
        unsigned long long spins = 0;
        for (;;) {
            int missing = 0;
#pragma unroll
            for (int k = 0; k < kRows; ++k) {
                if (!line_ready(r[k], flag)) {
                    ++missing;
                    r[k] = ld_line(buf + (c + k * nw) * 32 + j);
                }
            }
            if (!missing) break;
            if (++spins > (1ull << 26)) __trap();  // a co-residency bug fails loudly, never hangs
        }
        double v[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k) v[k] = line_value(r[k]);  // rows past G hold +0.0
        s = tree_sum_regs(v);
        for (int i = c + kRows * nw; i < G; i += nw) {
            uint4 t = ld_line(buf + i * 32 + j);
            for (unsigned long long sp = 0; !line_ready(t, flag); t = ld_line(buf + i * 32 + j))
                if (++sp > (1ull << 26)) __trap();
            s += line_value(t);
        }
        if (kPublish) __threadfence();  // acquire: the other CTAs' writes before their partials
    }
    s_fold[c][j] = s;
    __syncthreads();
    if (threadIdx.x < NV) out[threadIdx.x] = tree_sum<kGridWarps>(&s_fold[0][threadIdx.x], 32, nw);
    __syncthreads();
}


}  // namespace rfb
