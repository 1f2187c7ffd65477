// Latency of `S2R Rx, SR_CgaCtaId` (the shared-window base the compiler
// rematerialises before shared accesses whose address it cannot keep in a
// register): time a dependent chain S2R -> LEA -> LDS per iteration.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cga_s2r cga_s2r.cu
#include <cstdio>
__global__ void __launch_bounds__(384, 1) k(unsigned long long* out, float* sink, int iters) {
    __shared__ float s[2][384];
    s[0][threadIdx.x] = threadIdx.x;
    s[1][threadIdx.x] = 2 * threadIdx.x;
    __syncthreads();
    unsigned long long a = 0, b = 0;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        unsigned r;
        const unsigned long long t0 = clock64();
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
        const unsigned long long t1 = clock64() + r;
        a += t1 - t0;
        unsigned base;
        const unsigned long long t2 = clock64();
        asm volatile("{ .reg .u64 g; cvta.shared.u64 g, %1; cvt.u32.u64 %0, g; }" : "=r"(base) : "l"((unsigned long long)(size_t)0));
        const unsigned long long t3 = clock64() + (base & 1);
        b += t3 - t2;
        acc += s[it & 1][(threadIdx.x + it) % 384] + float(base & 0);
    }
    sink[threadIdx.x] = acc;
    if (threadIdx.x == 383) { out[2 * blockIdx.x] = a / iters; out[2 * blockIdx.x + 1] = b / iters; }
}
int main() {
    unsigned long long* out; float* sink;
    cudaMallocManaged(&out, 148 * 16); cudaMalloc(&sink, 384 * 4);
    k<<<148, 384>>>(out, sink, 100);
    cudaDeviceSynchronize();
    double a = 0, b = 0;
    for (int i = 0; i < 148; ++i) { a += out[2 * i]; b += out[2 * i + 1]; }
    printf("cluster_ctarank read %.0f cycles, cvta.shared %.0f cycles\n", a / 148, b / 148);
    return 0;
}
