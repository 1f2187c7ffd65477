// Does a cooperative launch accept a cluster dimension on this GPU, and how
// many clusters of each size can be co-resident (1 CTA of 384 threads per SM)?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* out) {
    cg::grid_group g = cg::this_grid();
    cg::cluster_group c = cg::this_cluster();
    __shared__ int x;
    if (threadIdx.x == 0) x = blockIdx.x;
    c.sync();
    int* peer = c.map_shared_rank(&x, (c.block_rank() + 1) % c.num_blocks());
    const int v = *peer;
    c.sync();
    g.sync();
    if (threadIdx.x == 0) atomicAdd(out, v >= 0 ? 1 : 0);
}
int main() {
    int* out;
    cudaMallocManaged(&out, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.blockDim = dim3(384);
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        int nclusters = 0;
        cfg.gridDim = dim3(cs);
        cudaError_t e0 = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k, &cfg);
        const int grid = nclusters * cs;
        cfg.gridDim = dim3(grid);
        *out = 0;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, out);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("cluster %2d: max active clusters %3d (%s) -> grid %3d: launch %s, sync %s, ctas ok %d\n", cs, nclusters,
               cudaGetErrorString(e0), grid, cudaGetErrorString(e), cudaGetErrorString(e2), *out);
        cudaGetLastError();
    }
}
