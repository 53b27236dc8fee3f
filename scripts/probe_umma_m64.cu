// Probe: where does tcgen05.mma (cta_group::1, kind::f16) with M = 64 put the 64
// rows of D in tensor memory?  The weight-gradient form (win_engine.cuh
// win3_wgrad_kernel): A = input rows as an MN-major SW32 operand whose atoms are
// one-row shifts (LBO = 32 B), B = dY rows MN-major SW32 (N = 48: 3 atoms), K =
// reduction rows.  Dumps all 128 lanes x N columns and maps each logical row m
// to the lane holding it (and checks the values).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_umma_m64.cu -o /tmp/probe_umma_m64 && /tmp/probe_umma_m64
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "common.cuh"

using namespace seed;

constexpr int IMG = 64 * 1024;

__global__ void run(const uint8_t* a_img, const uint8_t* b_img, int M, int N, int K, int blbo, float* out) {
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
  // zero the accumulator region first (so unwritten lanes read 0)
  for (int n0 = 0; n0 < 64; n0 += 16) {
    uint32_t z[16] = {0};
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(d + ((uint32_t)(tid & ~31) << 16) + n0), "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]),
                    "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]),
                    "r"(z[13]), "r"(z[14]), "r"(z[15]) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_bf16(M, N, true, true);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t a = umma_desc(smem_u32(As) + ks * 16 * 32, 32, 8 * 32, 6);
      const uint64_t b = umma_desc(smem_u32(Bs) + ks * 16 * 32, blbo, 8 * 32, 6);
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

static uint32_t swz32(uint32_t addr) { return addr ^ (((addr >> 7) & 1) << 4); }
static float rnd() { return (float)(rand() % 17 - 8) / 8.f; }

int main() {
  uint8_t *dA, *dB; float* dO;
  cudaMalloc(&dA, IMG); cudaMalloc(&dB, IMG); cudaMalloc(&dO, 128 * 64 * 4);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * IMG + 1024);
  srand(3);
  const int K = 64, N = 48, bstride = 5;   // B atom j starts j*bstride rows later
  for (int M : {128, 64}) {
    // X rows (16 channels, 32 B) and dY rows (16 channels): row r at byte r*32, SW32 of the address
    const int rows = K + 16;
    std::vector<float> X(rows * 16), Y(rows * 16);
    for (auto& v : X) v = rnd();
    for (auto& v : Y) v = rnd();
    auto bf = [](float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); };
    std::vector<uint16_t> ai(IMG / 2, 0), bi(IMG / 2, 0);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < 16; ++c) {
        ai[swz32(r * 32 + c * 2) / 2] = bf(X[r * 16 + c]);
        bi[swz32(r * 32 + c * 2) / 2] = bf(Y[r * 16 + c]);
      }
    cudaMemcpy(dA, ai.data(), IMG, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bi.data(), IMG, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, 128 * 64 * 4);
    run<<<1, 128, 2 * IMG + 1024>>>(dA, dB, M, N, K, bstride * 32, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("M=%d: cuda error %s\n", M, cudaGetErrorString(e)); return 1; }
    std::vector<float> o(128 * 64);
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    // logical D[m = atom*16 + c][n = j*16 + co] = sum_k X[k + atom][c] * Y[k + j*bstride][co]
    printf("M=%d N=%d (A MN SW32 LBO=32, B MN SW32 LBO=%d rows):\n", M, N, bstride);
    int found = 0;
    for (int m = 0; m < M; ++m) {
      std::vector<double> ref(N);
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)X[(k + m / 16) * 16 + m % 16] * Y[(k + (n / 16) * bstride) * 16 + n % 16];
        ref[n] = s;
      }
      int lane = -1;
      for (int l = 0; l < 128 && lane < 0; ++l) {
        double err = 0;
        for (int n = 0; n < N; ++n) err = std::max(err, std::fabs(ref[n] - o[l * 64 + n]));
        if (err < 1e-3) lane = l;
      }
      if (lane >= 0) ++found;
      if (m % 8 == 0 || lane < 0) printf("  row %3d -> lane %d\n", m, lane);
    }
    printf("  rows found: %d / %d\n", found, M);
  }
  return 0;
}
