#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1,1,1) k(){}
__global__ void kk(float*p){ extern __shared__ float s[]; if(p) p[0]=s[0]; }
int main(){
  for (int cs : {2, 4, 8}) for (int smem : {100*1024, 180*1024, 200*1024}) {
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148,1,1); cfg.blockDim = dim3(192,1,1); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kk, &cfg);
    printf("cluster %d smem %d KB: max active clusters %d (%d CTAs) %s\n", cs, smem/1024, n, n*cs, cudaGetErrorString(e));
  }
}
