// How many clusters of size C can be co-resident (cudaOccupancyMaxActiveClusters)
// for a 1-CTA/SM kernel with ~190 KB smem, and where do they land (smid per CTA).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(int* out) {
  extern __shared__ char sm[];
  unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  cg::cluster_group c = cg::this_cluster();
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  sm[threadIdx.x] = 1;
  c.sync();
}
int main() {
  int* d; cudaMalloc(&d, 4096 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 190 * 1024, 220 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int C : {1, 2, 4, 8, 9, 10, 12, 14, 16}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(C * 16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
      printf("{\"smem_kb\":%d,\"cluster\":%d,\"max_active_clusters\":%d,\"ctas\":%d,\"err\":\"%s\"}\n", smem / 1024, C, ncl,
             ncl * C, cudaGetErrorString(e));
    }
  }
  return 0;
}
