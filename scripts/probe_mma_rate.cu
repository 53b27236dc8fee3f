// Probe: issue rate of tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) with both
// operands in shared memory, by operand layout (K-major SW32 / SW64 / SW128, MN-major
// SW32 / SW128) and N.  One CTA per SM, one thread issues R MMAs back to back into
// one accumulator (the window convs' pattern), commit + wait, clock64 around it.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_mma_rate.cu -o /tmp/probe_mma_rate && /tmp/probe_mma_rate
#include <cstdio>
#include "common.cuh"

using namespace seed;

__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(p));
  return p != 0;
}

// warp-uniform issue: all 32 lanes run the loop, one elected lane issues; nacc accumulators
template <int N>
__global__ void rate_w(int layout_a, int rb_a, int reps, int nacc, long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3F803F80u, 0, 0x3F803F80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint32_t A = smem_u32(sm), Bm = smem_u32(sm + 32768);
    const uint64_t ad = umma_desc(A, 16, 8 * rb_a, layout_a);
    const uint64_t bd = umma_desc(Bm, 16, 1024, 2);
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + (uint32_t)((k % nacc) * N)),
            "l"(ad + (uint64_t)(k * 2)), "l"(bd + (uint64_t)(k * 2)), "r"(idesc), "r"(1)
            : "memory");
    }
    if (elect_one()) tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 256); }
}

template <int N, int M = 128>
__global__ void rate(int layout_a, int rb_a, int a_mn, int reps, long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3F803F80u, 0, 0x3F803F80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(M, N, a_mn != 0, false);
    const uint32_t A = smem_u32(sm), Bm = smem_u32(sm + 32768);
    // A: K-major: SBO = 8 rows * rb; MN-major: LBO = atom stride (rb * 1 row, the
    // shifted-window pattern), SBO = 8 k-rows * rb
    const uint64_t ad = a_mn ? umma_desc(A, rb_a, 8 * rb_a, layout_a)
                             : umma_desc(A, 16, 8 * rb_a, layout_a);
    const uint64_t bd = umma_desc(Bm, 16, 1024, 2);   // B: K-major SW128
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) tc_mma_bf16(tbase, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, 1);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 256); }
}

template <int N, int M = 128>
void run(const char* name, int layout, int rb, int mn, long long* d) {
  const int reps = 512;
  cudaFuncSetAttribute(rate<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  rate<N, M><<<148, 128, 100 * 1024>>>(layout, rb, mn, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-14s M=%3d N=%3d: %7.1f cycles / MMA  (%s)\n", name, M, N, s / 148 / (reps * 8.0),
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

// NI issuing warps, each one elected lane issuing into its own accumulator
template <int N, int NI>
__global__ void rate_multi(int reps, long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3F803F80u, 0, 0x3F803F80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  __syncthreads();
  tc_fence_after();
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp < NI) {
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint32_t A = smem_u32(sm + warp * 8192), Bm = smem_u32(sm + 40960);
    const uint64_t ad = umma_desc(A, 16, 8 * 32, 6);
    const uint64_t bd = umma_desc(Bm, 16, 1024, 2);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc_mma_bf16_w(tbase + (uint32_t)(warp * 64), ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, 1);
    }
    tc_commit_w(&bar[warp]);
    mbar_wait(&bar[warp], 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 256); }
}

template <int N, int NI>
void run_multi(long long* d) {
  const int reps = 512;
  cudaFuncSetAttribute(rate_multi<N, NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  rate_multi<N, NI><<<148, 128, 100 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("issuers=%d N=%3d: %7.1f cycles per MMA (all issuers)  (%s)\n", NI, N,
         s / 148 / (reps * 8.0 * NI), e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

template <int N>
void run_w(const char* name, int layout, int rb, int nacc, long long* d) {
  const int reps = 512;
  cudaFuncSetAttribute(rate_w<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  rate_w<N><<<148, 128, 100 * 1024>>>(layout, rb, reps, nacc, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("warp %-9s N=%3d acc=%d: %7.1f cycles / MMA  (%s)\n", name, N, nacc, s / 148 / (reps * 8.0),
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  // layout codes: 2 = SW128, 4 = SW64, 6 = SW32
  run<16>("K SW32", 6, 32, 0, d);
  run<16>("K SW64", 4, 64, 0, d);
  run<16>("K SW128", 2, 128, 0, d);
  run<16>("MN SW32", 6, 32, 1, d);
  run<16>("MN SW64", 4, 64, 1, d);
  run<16>("MN SW128", 2, 128, 1, d);
  run<32>("K SW32", 6, 32, 0, d);
  run<32>("K SW64", 4, 64, 0, d);
  run<32>("K SW128", 2, 128, 0, d);
  run<32>("MN SW32", 6, 32, 1, d);
  run<32>("MN SW64", 4, 64, 1, d);
  run<32>("MN SW128", 2, 128, 1, d);
  run<64>("K SW128", 2, 128, 0, d);
  run<128>("K SW128", 2, 128, 0, d);
  run<256>("K SW128", 2, 128, 0, d);
  run_multi<16, 1>(d);
  run_multi<16, 2>(d);
  run_multi<16, 4>(d);
  run_multi<48, 2>(d);
  run<48>("MN SW32", 6, 32, 1, d);
  run<48, 64>("MN SW32", 6, 32, 1, d);
  run<96>("MN SW64", 4, 64, 1, d);
  run<96, 64>("MN SW64", 4, 64, 1, d);
  run<16, 64>("K SW32", 6, 32, 0, d);
  run_w<16>("K SW32", 6, 32, 1, d);
  run_w<16>("K SW32", 6, 32, 2, d);
  run_w<16>("K SW32", 6, 32, 4, d);
  run_w<16>("K SW128", 2, 128, 1, d);
  run_w<32>("K SW64", 4, 64, 1, d);
  run_w<32>("K SW64", 4, 64, 4, d);
  run_w<64>("K SW128", 2, 128, 1, d);
  run_w<128>("K SW128", 2, 128, 1, d);
  run_w<256>("K SW128", 2, 128, 1, d);
  return 0;
}
