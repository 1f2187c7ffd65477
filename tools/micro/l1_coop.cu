// L1 hit latency under the tracking kernel's launch configuration: cooperative
// launch, 384 threads, one CTA per SM, 96 KB dynamic shared memory attribute,
// carveout preference MaxL1, with and without griddepcontrol (PDL).
#include <cstdio>
#include <cstdint>
extern __shared__ unsigned char dyn[];
__global__ void __launch_bounds__(384, 1) k(const uint64_t* p, int n, long long* out, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    dyn[threadIdx.x] = 1;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t i = 0;
    for (int r = 0; r < 2; ++r)
        for (int s = 0; s < n; ++s) i = __ldg(p + i);
    long long t0 = clock64();
    for (int s = 0; s < 1024; ++s) i = __ldg(p + i);
    out[0] = clock64() - t0;
    out[1] = (long long)i + dyn[5];
}
int main() {
    const int n = 1024;
    uint64_t h[n];
    for (int s = 0; s < n; ++s) h[s] = (s + 33) % n;
    uint64_t* d; long long* o;
    cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMallocManaged(&o, 2 * sizeof(long long));
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxL1));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t dynb : {size_t(18432), size_t(96 * 1024)})
        for (int pdl : {0, 1}) {
            int nn = n;
            void* args[] = {&d, &nn, &o, &pdl};
            for (int r = 0; r < 2; ++r) {
                cudaLaunchCooperativeKernel((void*)k, dim3(sms), dim3(384), args, dynb, 0);
                cudaDeviceSynchronize();
            }
            printf("dyn %zu pdl %d: %.1f cycles/load (%s)\n", dynb, pdl, o[0] / 1024.0, cudaGetErrorString(cudaGetLastError()));
        }
}
