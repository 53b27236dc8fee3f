// Probe: tcgen05.shift.cta_group::1.down — which TMEM lanes / columns it moves, what
// lane 0 holds afterwards, whether it is ordered after preceding tcgen05.mma of the
// same thread, and its issue cost (for a column-tap-stacked 3x3 conv whose epilogue
// would combine D[g-1] / D[g] / D[g+1] at one lane after shifting two parts down).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_tmem_shift.cu -o /tmp/probe_tmem_shift && /tmp/probe_tmem_shift
#include <cstdio>
#include <vector>
#include "common.cuh"

using namespace seed;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_shift_down(uint32_t taddr) {
  asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(taddr) : "memory");
}

// mode 0: fill, shift cols [c0, c0+8) once (nshift times), dump 32 cols.
// mode 1: timing: nshift shifts back to back over col slices 0,8,16,24 round robin
__global__ void run(int mode, int c0, int nshift, float* out, long long* cyc) {
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 64);
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase;
  const int row = warp * 32 + lane;
  for (int c = 0; c < 32; c += 16) {
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint((float)(row * 100 + c + k));
    tmem_st16(t + ((uint32_t)(warp * 32) << 16) + c, v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    long long t0 = clock64();
    if (mode == 0) {
      for (int i = 0; i < nshift; ++i)
        if (lane == 0) tc_shift_down(t + c0);
    } else {
      for (int i = 0; i < nshift; ++i)
        if (lane == 0) tc_shift_down(t + (i & 3) * 8);
    }
    __syncwarp();
    if (lane == 0) tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) *cyc = t1 - t0;
  }
  __syncthreads();
  tc_fence_after();
  for (int c = 0; c < 32; c += 16) {
    float v[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int k = 0; k < 16; ++k) out[row * 32 + c + k] = v[k];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(t, 64);
}

int main() {
  float* d;
  long long* dc;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaMalloc(&dc, 8);
  std::vector<float> h(128 * 32);
  long long cyc;
  for (int c0 : {0, 8}) {
    run<<<1, 128>>>(0, c0, 1, d, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("shift.down once at col %d: value = row*100 + col before the shift\n", c0);
    for (int r : {0, 1, 2, 31, 32, 33, 63, 64, 95, 96, 126, 127}) {
      printf("  lane %3d:", r);
      for (int c = 0; c < 20; ++c) printf(" %6.0f", h[r * 32 + c]);
      printf("\n");
    }
  }
  for (int n : {1, 16, 64, 256, 1024}) {
    run<<<1, 128>>>(1, 0, n, d, dc);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("%5d shifts (8-column slices round robin): %lld cycles, %.1f per shift\n", n, cyc, (double)cyc / n);
  }
  return 0;
}
