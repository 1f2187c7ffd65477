// Cost of a loop's back-edge as a function of the loop body's code size
// (instruction-cache capacity probe for k_track's LM loop).
// Each iteration: BODY straight-line FMAs on every thread, a CTA barrier, a
// short serial section on the last thread, a barrier; the last thread stamps
// clock64 just before the back-edge and at the loop top.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o backedge backedge.cu -DBODY=1024
#include <cstdio>
#ifndef BODY
#define BODY 1024  // instructions in the body (16 B each)
#endif
#define F1 asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(y), "f"(z));
#define F8 F1 F1 F1 F1 F1 F1 F1 F1
#define F64 F8 F8 F8 F8 F8 F8 F8 F8
#define F512 F64 F64 F64 F64 F64 F64 F64 F64

#ifndef STREAM_KB
#define STREAM_KB 0  // per CTA per iteration: global bytes streamed (L2 pressure)
#endif
__global__ void __launch_bounds__(384, 1) k(int iters, float* out, unsigned long long* cyc, const float4* buf) {
    float x = threadIdx.x * 1e-3f, y = 0.999f, z = 1e-4f;
    __shared__ float s;
    unsigned long long tot = 0, t_end = 0;
    for (int it = 0; it < iters; ++it) {
        if (threadIdx.x == 383) {
            const unsigned long long t = clock64();
            if (it > 0) tot += t - t_end;
        }
#pragma unroll
        for (int r = 0; r < BODY / 512; ++r) { F512 }
#if (BODY % 512) >= 64
#pragma unroll
        for (int r = 0; r < (BODY % 512) / 64; ++r) { F64 }
#endif
#if STREAM_KB > 0
        {
            const size_t chunk = STREAM_KB * 1024 / 16, nchunks = (size_t(256) << 20) / 16 / chunk;
            const float4* b = buf + ((size_t(blockIdx.x) * iters + it) % nchunks) * chunk;
            float4 acc4 = make_float4(0, 0, 0, 0);
            for (int i = threadIdx.x; i < STREAM_KB * 1024 / 16; i += 384) {
                const float4 v4 = __ldcg(b + i);
                acc4.x += v4.x;
            }
            x += acc4.x * 1e-30f;
        }
#endif
        __syncthreads();
        if (threadIdx.x == 383) {
            float v = x;
            for (int i = 0; i < 16; ++i) v = v * 1.0001f + 1e-7f;
            s = v;
        }
        __syncthreads();
        x += s * 1e-9f;
        if (threadIdx.x == 383) t_end = clock64();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 383) cyc[blockIdx.x] = tot / (iters - 1);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sms * 384 * 4);
    cudaMallocManaged(&cyc, sms * 8);
    float4* buf = nullptr;
    const size_t bytes = (size_t(256) << 20) + 16;  // streamed cyclically (2x the L2)
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    k<<<sms, 384>>>(4, out, cyc, buf);
    k<<<sms, 384>>>(200, out, cyc, buf);
    cudaDeviceSynchronize();
    double m = 0;
    for (int i = 0; i < sms; ++i) m += cyc[i];
    printf("BODY %d instr (%.1f KB), %d KB streamed per CTA per iteration: back-edge + loop top %.0f cycles (mean over %d CTAs)\n",
           BODY, BODY * 16 / 1024.0, STREAM_KB, m / sms, sms);
    return 0;
}
