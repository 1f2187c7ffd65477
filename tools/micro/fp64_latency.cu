// Dependent-latency microbenchmark of the fp64 operations on the LM solve's
// critical path (one thread): DFMA, DADD, DMUL, MUFU.RCP64H-based fast_rcp,
// IEEE division, and an smem load. Prints cycles per dependent operation.
#include <cstdio>
__device__ __forceinline__ double fast_rcp(double x) {
    double r = double(__frcp_rn(float(x)));
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
    return r;
}
__global__ void k(double seed, double* out, long long* cyc) {
    __shared__ double sm[64];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 64; ++i) sm[i] = seed + i;
    const int N = 1024;
    double x = seed, y = seed * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __fma_rn(x, 1.0000001, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) y = __dadd_rn(y, 1e-9);
    long long t2 = clock64();
    double z = seed;
    for (int i = 0; i < N; ++i) z = __dmul_rn(z, 1.0000001);
    long long t3 = clock64();
    double w = seed + 1.0;
    for (int i = 0; i < N; ++i) w = fast_rcp(w) + 1.0;
    long long t4 = clock64();
    double v = seed + 1.0;
    for (int i = 0; i < N; ++i) v = 1.0 / v + 1.0;
    long long t5 = clock64();
    int idx = 0;
    double s = 0;
    for (int i = 0; i < N; ++i) { s = sm[idx]; idx = int(s) & 31; }
    long long t6 = clock64();
    out[0] = x + y + z + w + v + s;
    cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 8); cudaMallocManaged(&c, 6 * 8);
    k<<<1, 32>>>(1.5, o, c);
    k<<<1, 32>>>(1.5, o, c);
    cudaDeviceSynchronize();
    const char* n[6] = {"dfma", "dadd", "dmul", "fast_rcp+dadd", "ieee_div+dadd", "lds+cvt"};
    for (int i = 0; i < 6; ++i) printf("%-16s %6.1f cycles/op\n", n[i], c[i] / 1024.0);
}
