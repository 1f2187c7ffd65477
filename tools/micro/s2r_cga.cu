// Latency of the special-register read the compiler emits before a generic
// shared-memory access (S2R SR_CgaCtaId), and of a generic-pointer shared load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o s2r_cga s2r_cga.cu
#include <cstdio>
__device__ __noinline__ float* launder(float* p) { return p; }
__global__ void __launch_bounds__(384, 1) k(unsigned long long* out, float* sink, int iters) {
    __shared__ float s[384];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    unsigned long long a = 0, b = 0;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        unsigned r;
        const unsigned long long t0 = clock64();
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
        const unsigned long long t1 = clock64() + (r & 0);  // depend on r
        a += t1 - t0;
        float* g = launder(s);  // generic pointer into shared memory
        const unsigned long long t2 = clock64();
        acc += g[(threadIdx.x + it) % 384];
        const unsigned long long t3 = clock64() + (acc > 1e30f);
        b += t3 - t2;
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
    printf("cluster_ctarank read %.0f cycles, generic shared load %.0f cycles\n", a / 148, b / 148);
    return 0;
}
