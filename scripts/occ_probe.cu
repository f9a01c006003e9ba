#include <cstdio>
#include <cuda_runtime.h>
template <int CS> __global__ void __cluster_dims__(CS,1,1) __launch_bounds__(192) kk(int* p){ extern __shared__ int s[]; if(p) p[threadIdx.x]=s[threadIdx.x]; }
template <int CS> void q(int smem, int threads){
  cudaFuncSetAttribute(kk<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(CS*64); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
  int n=0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)kk<CS>, &cfg);
  int nb=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kk<CS>, threads, smem);
  printf("CS=%d smem=%d threads=%d -> max active clusters %d (%s), blocks/SM %d\n", CS, smem, threads, n, cudaGetErrorString(e), nb);
}
int main(){ for(int sm: {99328, 101*1024, 110*1024, 60*1024}) { q<1>(sm,192); q<2>(sm,192); q<4>(sm,192); q<8>(sm,192);} 
 cudaDeviceProp p; cudaGetDeviceProperties(&p,0); printf("SMs %d smem/SM %zu smem/block optin %zu\n", p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin); }
