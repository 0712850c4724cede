// dev probe: how many clusters of 2 / 3 / 4 CTAs (one CTA per SM: ~210 KB dynamic smem)
// can be co-resident on this GPU (cudaOccupancyMaxActiveClusters), and a timed launch
// of a persistent cluster grid to confirm every SM runs a CTA.
#include <cuda_runtime.h>
#include <cstdio>

__global__ void probe(unsigned* sm_of_cta) {
    extern __shared__ unsigned char smem[];
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) sm_of_cta[blockIdx.x] = smid;
    smem[threadIdx.x] = 1;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 210 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs = 1; cs <= 4; ++cs) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs of %d SMs) %s\n", cs, n, n * cs, nsm, cudaGetErrorString(e));
    }
    return 0;
}
