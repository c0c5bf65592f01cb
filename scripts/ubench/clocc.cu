// Max co-resident thread-block clusters on this GPU for cluster sizes 1..16 at a given dynamic shared
// memory per CTA (1 CTA per SM): the wave width of the cluster-resident batched kernel.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main(int argc, char** argv) {
  int smem = argc > 1 ? atoi(argv[1]) : 200 * 1024, threads = argc > 2 ? atoi(argv[2]) : 512;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dummy, &cfg);
    printf("smem %d threads %d cluster %2d: max active clusters %d (%d CTAs) %s\n", smem, threads, cs, n, n * cs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
