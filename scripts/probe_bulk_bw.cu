// Probe: HBM read bandwidth of 1D TMA bulk copies (cp.async.bulk global->shared)
// in the shape the window-conv kernels use: one producer thread per CTA, a ring
// of S slabs of B bytes, consumer = one thread that only waits and releases.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_bulk_bw.cu -o build_probe/probe_bulk_bw
#include <cstdio>
#include "common.cuh"
using namespace seed;

__device__ __forceinline__ void cpa16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__global__ void __launch_bounds__(160, 1) bulk_stream(const uint8_t* src, int64_t nslabs, int slab,
                                                     int stages, int threads_issue) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], threads_issue == 128 ? 128 : 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threads_issue == 128 && warp < 4) {   // cp.async 16 B by 4 warps (LDGSTS)
    int it = 0;
    for (int64_t t = blockIdx.x; t < nslabs; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      const uint32_t d = smem_u32(sm + (size_t)s * slab);
      for (int c = threadIdx.x; c < slab / 16; c += 128) cpa16(d + c * 16, src + t * slab + c * 16);
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  } else if (threads_issue != 128 && warp == 0) {
    int it = 0;
    for (int64_t t = blockIdx.x; t < nslabs; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      if (threads_issue == 1) {
        if (lane == 0) {
          mbar_expect_tx(&full[s], slab);
          bulk_g2s(smem_u32(sm + (size_t)s * slab), src + t * slab, slab, &full[s]);
        }
      } else {   // split the slab into 32 copies, one per lane
        if (lane == 0) mbar_expect_tx(&full[s], slab);
        __syncwarp();
        const int part = slab / 32;
        bulk_g2s(smem_u32(sm + (size_t)s * slab + lane * part), src + t * slab + lane * part, part, &full[s]);
      }
    }
  } else if (warp == 4 && lane == 0) {
    int it = 0;
    for (int64_t t = blockIdx.x; t < nslabs; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  const size_t total = 38ull << 20;
  uint8_t* src;
  cudaMalloc(&src, total + (1 << 20));
  cudaMemset(src, 1, total);
  uint8_t* flush;
  cudaMalloc(&flush, 256ull << 20);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int slab : {19456, 40960}) {
    for (int stages : {4, 8}) {
      if ((size_t)stages * slab > 200 * 1024) continue;
      for (int ti : {1, 32, 128}) {
        const int64_t n = total / slab;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(flush, rep, 256ull << 20);
          cudaEventRecord(a);
          bulk_stream<<<148, 160, stages * slab>>>(src, n, slab, stages, ti);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        printf("slab %6d B stages %d issuers %2d: %.2f us  %.0f GB/s\n", slab, stages, ti, best * 1000,
               (double)n * slab / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
