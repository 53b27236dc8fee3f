// Probe of tcgen05.mma shared-memory operand layouts used by the space-to-depth
// shifted-window convolutions (conv_s2d.cu).  The host builds raw shared-memory
// images in which every element sits at an absolute-address-swizzled byte
// offset (as a linear copy of a pre-swizzled global buffer lands them), the
// kernel runs K/16 MMAs with the given descriptors, and the host compares D
// with the logical product.  Swizzle rule (address bits): SW128 b[4:6]^=b[7:9],
// SW64 b[4:5]^=b[7:8], SW32 b[4]^=b[7].
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_umma_layouts.cu -o build_probe/probe_umma_layouts
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>
#include <cmath>
#include "common.cuh"

using namespace seed;

constexpr int IMG = 64 * 1024;   // bytes per operand image

struct Desc {
  int start, lbo, sbo, layout, kstep;   // kstep = start advance per K=16
};

__global__ void run(const uint8_t* a_img, const uint8_t* b_img, Desc ad, Desc bd, int N, int K,
                    int a_mn, int b_mn, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* As = sm;
  uint8_t* Bs = sm + IMG;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < IMG / 16; i += blockDim.x) {
    ((uint4*)As)[i] = ((const uint4*)a_img)[i];
    ((uint4*)Bs)[i] = ((const uint4*)b_img)[i];
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc(&tbase, 64);
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N, a_mn, b_mn);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t a = umma_desc(smem_u32(As) + ad.start + ks * ad.kstep, ad.lbo, ad.sbo, ad.layout);
      const uint64_t b = umma_desc(smem_u32(Bs) + bd.start + ks * bd.kstep, bd.lbo, bd.sbo, bd.layout);
      tc_mma_bf16(d, a, b, idesc, ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int n0 = 0; n0 < N; n0 += 16) {
    float v[16];
    tmem_ld16(d + ((uint32_t)(tid & ~31) << 16) + n0, v);
    for (int n = 0; n < 16; ++n) out[tid * 64 + n0 + n] = v[n];
  }
  __syncthreads();
  if (tid < 32) tmem_dealloc(d, 64);
}

static uint32_t swz(uint32_t addr, int mode) {   // mode: 128, 64, 32, 0
  switch (mode) {
    case 128: return addr ^ (((addr >> 7) & 7) << 4);
    case 64: return addr ^ (((addr >> 7) & 3) << 4);
    case 32: return addr ^ (((addr >> 7) & 1) << 4);
    default: return addr;
  }
}

// element address functions: (index0, index1) -> byte offset (pre-swizzle)
using AddrFn = std::function<uint32_t(int, int)>;

static float rnd() { return (float)(rand() % 17 - 8) / 8.f; }

static bool test(const char* name, int N, int K, int a_mn, int b_mn, AddrFn a_addr, int a_swz,
                 AddrFn b_addr, int b_swz, Desc ad, Desc bd, uint8_t* dA, uint8_t* dB, float* dO,
                 bool a_ones = false) {
  // logical A[m][k] (m<128), B[n][k]
  std::vector<float> A(128 * K), B(N * K);
  std::vector<uint16_t> ai(IMG / 2, 0), bi(IMG / 2, 0);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < K; ++k) A[m * K + k] = a_ones ? 1.f : rnd();
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) B[n * K + k] = rnd();
  auto bf = [](float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); };
  std::vector<int> aset(IMG / 2, -1);
  bool conflict = false;
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < K; ++k) {
      const uint32_t off = swz(a_addr(m, k), a_swz) / 2;
      if (off >= IMG / 2) { printf("%s: A addr out of range\n", name); return false; }
      if (aset[off] >= 0 && ai[off] != bf(A[m * K + k])) conflict = true;
      ai[off] = bf(A[m * K + k]);
      aset[off] = 1;
    }
  if (conflict) {   // overlapping windows: logical A is what the image holds
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < K; ++k) {
        const uint16_t h = ai[swz(a_addr(m, k), a_swz) / 2];
        uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4);
        A[m * K + k] = f;
      }
  }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) bi[swz(b_addr(n, k), b_swz) / 2] = bf(B[n * K + k]);
  cudaMemcpy(dA, ai.data(), IMG, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, bi.data(), IMG, cudaMemcpyHostToDevice);
  run<<<1, 128, 2 * IMG + 1024>>>(dA, dB, ad, bd, N, K, a_mn, b_mn, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: cuda error %s\n", name, cudaGetErrorString(e)); exit(1); }
  std::vector<float> o(128 * 64);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
      maxerr = std::max(maxerr, std::fabs(ref - o[m * 64 + n]));
    }
  printf("%-58s max|err| = %-9g %s\n", name, maxerr, maxerr < 1e-3 ? "OK" : "MISMATCH");
  return maxerr < 1e-3;
}

int main() {
  uint8_t *dA, *dB; float* dO;
  cudaMalloc(&dA, IMG); cudaMalloc(&dB, IMG); cudaMalloc(&dO, 128 * 64 * 4);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * IMG + 1024);
  srand(7);
  // B operand used by the K-major-A tests: K-major SW128, N rows of 128 B (K = 64)
  auto bK128 = [](int n, int k) { return (uint32_t)(n * 128 + k * 2); };
  for (int s : {0, 3, 5}) {
    // 1. K-major SW64 A: rows of 64 B (K = 32), shifted start by s rows
    char nm[128];
    snprintf(nm, sizeof nm, "A K-major SW64, shift %d rows, N=64 B K-major SW64", s);
    auto a64 = [s](int m, int k) { return (uint32_t)((m + s) * 64 + k * 2); };
    auto b64 = [](int n, int k) { return (uint32_t)(n * 64 + k * 2); };
    test(nm, 64, 32, 0, 0, a64, 64, b64, 64, Desc{s * 64, 16, 512, 4, 32}, Desc{0, 16, 512, 4, 32},
         dA, dB, dO);
  }
  for (int s : {0, 3}) {
    // 2. MN-major SW128 A with rows = k, B MN-major SW64 (N = 32, 64-byte k rows)
    char nm[128];
    snprintf(nm, sizeof nm, "A MN SW128 (LBO 128), B MN-major SW64 N=32, shift %d", s);
    auto a = [s](int m, int k) { return (uint32_t)((k + s + (m >= 64)) * 128 + (m & 63) * 2); };
    auto b = [](int n, int k) { return (uint32_t)(k * 64 + n * 2); };
    test(nm, 32, 64, 1, 1, a, 128, b, 64, Desc{s * 128, 128, 1024, 2, 2048},
         Desc{0, 512, 512, 4, 1024}, dA, dB, dO);
    // 3. B MN-major SW32 (N = 16, 32-byte k rows)
    snprintf(nm, sizeof nm, "A MN SW128 (LBO 128), B MN-major SW32 N=16, shift %d", s);
    auto b32 = [](int n, int k) { return (uint32_t)(k * 32 + n * 2); };
    test(nm, 16, 64, 1, 1, a, 128, b32, 32, Desc{s * 128, 128, 1024, 2, 2048},
         Desc{0, 256, 256, 6, 512}, dA, dB, dO);
    // 3b. B MN-major SW32 with a row shift (dY window starting mid-atom)
    snprintf(nm, sizeof nm, "B MN-major SW32 N=16 shifted %d rows", s + 1);
    auto b32s = [s](int n, int k) { return (uint32_t)((k + s + 1) * 32 + n * 2); };
    test(nm, 16, 64, 1, 1, a, 128, b32s, 32, Desc{s * 128, 128, 1024, 2, 2048},
         Desc{(s + 1) * 32, 256, 256, 6, 512}, dA, dB, dO);
  }
  // 4. all-ones A (MN-major, LBO = SBO = 0: one 1 KB block of ones reused)
  {
    auto a = [](int m, int k) { return (uint32_t)((k & 7) * 128 + (m & 63) * 2); };
    auto b = [](int n, int k) { return (uint32_t)(k * 64 + n * 2); };
    test("A = ones (MN SW128, LBO=SBO=0), B MN-major SW64 N=32", 32, 64, 1, 1, a, 128, b, 64,
         Desc{0, 0, 0, 2, 0}, Desc{0, 512, 512, 4, 1024}, dA, dB, dO, true);
  }
  // 5. K-major SW128 A shifted, B K-major SW128 N=16 (conv forward form)
  {
    auto a = [](int m, int k) { return (uint32_t)((m + 13) * 128 + k * 2); };
    test("A K-major SW128 shift 13, B K-major SW128 N=16", 16, 64, 0, 0, a, 128, bK128, 128,
         Desc{13 * 128, 16, 1024, 2, 32}, Desc{0, 16, 1024, 2, 32}, dA, dB, dO);
  }
  return 0;
}
