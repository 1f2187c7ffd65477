// Dependent-load latency of the load flavours the tracking kernel uses
// (LDG.CONSTANT via __ldg, plain LDG, LDG.STRONG.GPU via __ldcg) on a small,
// L1-resident array, one thread, after a warm-up pass: cycles per load. Then
// whether a sweep of relaxed.gpu loads (the all-reduce's polling: 152 KB of
// flagged lines) evicts L1-resident data, with and without L1::no_allocate.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint4 ld_relaxed(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint4 ld_relaxed_na(const uint4* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ long long chase(const uint64_t* p, uint64_t& i) {
    long long t0 = clock64();
    for (int s = 0; s < 256; ++s) i = __ldg(p + i);
    return clock64() - t0;
}
__global__ void k(const uint64_t* p, int n, const uint4* big, int nbig, long long* out) {
    uint64_t i = 0;
    unsigned acc = 0;
    if (threadIdx.x == 0) {
        for (int r = 0; r < 2; ++r)
            for (int s = 0; s < n; ++s) i = __ldg(p + i);
        long long t0 = clock64();
        for (int s = 0; s < 1024; ++s) i = __ldg(p + i);
        long long t1 = clock64();
        for (int s = 0; s < 1024; ++s) i = p[i];
        long long t2 = clock64();
        for (int s = 0; s < 1024; ++s) i = __ldcg(p + i);
        long long t3 = clock64();
        out[0] = (t1 - t0); out[1] = (t2 - t1); out[2] = (t3 - t2);
        for (int s = 0; s < n; ++s) i = __ldg(p + i);  // warm again
        out[3] = chase(p, i);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < nbig; s += blockDim.x) acc += ld_relaxed(big + s).x;  // sweep, allocating
    __syncthreads();
    if (threadIdx.x == 0) out[4] = chase(p, i);
    if (threadIdx.x == 0) for (int s = 0; s < n; ++s) i = __ldg(p + i);  // warm again
    __syncthreads();
    for (int s = threadIdx.x; s < nbig; s += blockDim.x) acc += ld_relaxed_na(big + s).x;  // sweep, no-allocate
    __syncthreads();
    if (threadIdx.x == 0) out[5] = chase(p, i);
    if (threadIdx.x == 0) out[6] = (long long)i + acc;
}
int main() {
    const int n = 1024;  // 8 KB ring, stride 33 elements
    uint64_t h[n];
    for (int s = 0; s < n; ++s) h[s] = (s + 33) % n;
    uint64_t* d; long long* o; uint4* big;
    const int nbig = 152 * 1024 / 16;
    cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMalloc(&big, nbig * 16); cudaMemset(big, 0, nbig * 16);
    cudaMallocManaged(&o, 8 * sizeof(long long));
    for (int r = 0; r < 2; ++r) { k<<<1, 384>>>(d, n, big, nbig, o); cudaDeviceSynchronize(); }
    printf("ldg.nc %.1f  ld %.1f  ld.cg %.1f cycles/load\n", o[0] / 1024.0, o[1] / 1024.0, o[2] / 1024.0);
    printf("L1-resident chase: before %.1f, after a 152 KB relaxed.gpu sweep %.1f, after a no_allocate sweep %.1f cycles/load\n",
           o[3] / 256.0, o[4] / 256.0, o[5] / 256.0);
}
