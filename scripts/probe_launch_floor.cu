// Probe: per-launch cost of kernel skeletons (graph of back-to-back launches):
// empty kernel; + 200 KB dynamic smem; + TMEM alloc/dealloc; + mbarrier init.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_launch_floor.cu -o build_probe/probe_launch_floor
#include <cstdio>
#include "common.cuh"
using namespace seed;

template <int MODE>
__global__ void __launch_bounds__(416, 1) skel(int* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[20];
  if (MODE >= 2 && threadIdx.x == 0) {
    for (int i = 0; i < 20; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (MODE >= 1 && (threadIdx.x >> 5) == 8) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && out) out[blockIdx.x] = sm[0] + (int)slot;
  tc_fence_before();
  __syncthreads();
  if (MODE >= 1 && (threadIdx.x >> 5) == 8) tmem_dealloc(slot, 256);
}

template <int MODE>
float time_it(int grid, size_t smem) {
  cudaFuncSetAttribute(skel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 50; ++i) skel<MODE><<<grid, 416, smem, s>>>(nullptr);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / 50;
}

int main() {
  for (int grid : {1, 148}) {
    printf("grid %3d: empty %.2f us | 200KB smem %.2f us | +TMEM %.2f us | +mbar %.2f us\n", grid,
           time_it<0>(grid, 0), time_it<0>(grid, 200 * 1024), time_it<1>(grid, 200 * 1024),
           time_it<2>(grid, 200 * 1024));
  }
  return 0;
}
