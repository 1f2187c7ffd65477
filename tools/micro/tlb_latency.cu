// Dependent-load latency over a few L1-resident lines spread across P distinct
// 2 MB pages (the tracking kernel's gathers touch the hash table, the link
// records and the brick pool: ~100 pages at C2): does the translation cost
// show up on L1 hits?
#include <cstdio>
#include <cstdint>
__global__ void k(const uint64_t* base, const uint64_t* start, int hops, long long* out) {
    if (threadIdx.x != 0) return;
    const uint64_t* q = start;
    for (int r = 0; r < 3 * hops; ++r) q = base + __ldg(q);  // warm (L1 + TLB)
    long long t0 = clock64();
    for (int r = 0; r < hops; ++r) q = base + __ldg(q);
    out[0] = clock64() - t0;
    out[1] = (long long)(q - base);
}
int main() {
    const size_t page = 2u << 20, span = size_t(4) << 30;  // 4 GB region like the brick pool
    uint64_t* d;
    if (cudaMalloc(&d, span) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    long long* o;
    cudaMallocManaged(&o, 2 * sizeof(long long));
    for (int pages : {1, 8, 16, 32, 64, 128, 256, 1024}) {
        // a cycle visiting one 8-byte slot in each of `pages` pages spread over the span
        const size_t stride = span / pages / page * page;
        for (int i = 0; i < pages; ++i) {
            uint64_t next = (uint64_t)(((i + 1) % pages) * stride / 8 + ((i * 37) % 64) * 16);
            uint64_t here = (uint64_t)(i * stride / 8 + ((i * 37 + 37 * 0) % 64) * 16);
            here = (uint64_t)(i * stride / 8 + ((i * 37) % 64) * 16);
            cudaMemcpy(d + here, &next, 8, cudaMemcpyHostToDevice);
        }
        const int hops = 4096;
        for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(d, d, hops, o); cudaDeviceSynchronize(); }
        printf("%5d pages: %.1f cycles/load\n", pages, o[0] / double(hops));
    }
}
