// How many clusters of 2 / 4 / 8 CTAs (one CTA per SM: ~227 KB of shared
// memory each) are co-resident on this GPU (cudaOccupancyMaxActiveClusters).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
    extern __shared__ int s[];
    if (p) p[0] = s[0];
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int smem = 226 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("%s: %d SMs\n", prop.name, prop.multiProcessorCount);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64, 1, 1);
        cfg.blockDim = dim3(352, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: max active clusters %d (%d SMs busy) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
