#include "gemm.cuh"
#include <cstdio>
using namespace lemo;
struct EpiNop { __device__ void operator()(int, bool, int, uint32_t, int) const {} };
int main() {
  for (int smem : {140000, 165000, 180000, 197888, 220000}) {
    cudaFuncSetAttribute(gemm_tn_pair_kernel<EpiNop>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)gemm_tn_pair_kernel<EpiNop>, &cfg);
    printf("smem %d: max active 2-CTA clusters %d (%s)\n", smem, n, cudaGetErrorString(e));
  }
  return 0;
}
