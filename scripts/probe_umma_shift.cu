// Probe: can a tcgen05.mma operand descriptor start at a row offset that is
// not a multiple of the 8-row 128B-swizzle atom (a "shifted window" over rows
// written with the absolute-address 128B swizzle, as TMA writes them)?
//   test K : K-major A (rows = M), start shifted by s rows, base_offset field 0 or s&7
//   test MN: MN-major A (rows = K, 64 M per 128-byte row), LBO = 128 (second MN atom =
//            window shifted by one more row), start shifted by s rows
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1910_06591_b200/csrc \
//      scripts/probe_umma_shift.cu -o /tmp/probe_umma_shift
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "common.cuh"

using namespace seed;

constexpr int ROWS = 320;   // data rows of 128 bytes (64 bf16)

__device__ __forceinline__ uint32_t swz(int row, int chunk) {   // absolute-address SW128
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}

__global__ void probe(const __nv_bfloat16* data, const __nv_bfloat16* bmat, int mode, int s,
                      int boff, float* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint8_t* As = sm;                       // ROWS x 128 B
  uint8_t* Bs = sm + ROWS * 128;          // 16 x 128 B (K-major, 64 k)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int c = tid; c < ROWS * 8; c += blockDim.x) {
    const int r = c >> 3, ch = c & 7;
    *(uint4*)(As + swz(r, ch)) = *(const uint4*)(data + r * 64 + ch * 8);
  }
  for (int c = tid; c < 16 * 8; c += blockDim.x) {
    const int r = c >> 3, ch = c & 7;
    *(uint4*)(Bs + swz(r, ch)) = *(const uint4*)(bmat + r * 64 + ch * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (tid < 32) tmem_alloc(&tbase, 32);
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, 16, mode == 1, false);
    for (int ks = 0; ks < 4; ++ks) {
      uint64_t ad, bd;
      if (mode == 0) {   // K-major: row pitch 128, atom stride 1024, k16 step = 32 B
        ad = umma_desc(smem_u32(As) + s * 128 + ks * 32, 16, 1024, 2);
      } else {           // MN-major: rows = k; LBO = MN-atom stride = 128 (one-row shift)
        ad = umma_desc(smem_u32(As) + (s + ks * 16) * 128, 128, 1024, 2);
      }
      ad |= (uint64_t)(boff & 7) << 49;
      bd = umma_desc(smem_u32(Bs) + ks * 32, 16, 1024, 2);
      tc_mma_bf16(d, ad, bd, idesc, ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(d + ((uint32_t)(tid & ~31) << 16), v);
  for (int n = 0; n < 16; ++n) out[tid * 16 + n] = v[n];
  __syncthreads();
  if (tid < 32) tmem_dealloc(d, 32);
}

int main() {
  std::vector<__nv_bfloat16> hd(ROWS * 64), hb(16 * 64);
  std::vector<float> fd(ROWS * 64), fb(16 * 64);
  srand(1);
  for (int i = 0; i < ROWS * 64; ++i) { fd[i] = (float)(rand() % 17 - 8) / 8.f; hd[i] = __float2bfloat16(fd[i]); }
  for (int i = 0; i < 16 * 64; ++i) { fb[i] = (float)(rand() % 17 - 8) / 8.f; hb[i] = __float2bfloat16(fb[i]); }
  __nv_bfloat16 *dd, *db; float* dout;
  cudaMalloc(&dd, hd.size() * 2); cudaMalloc(&db, hb.size() * 2); cudaMalloc(&dout, 128 * 16 * 4);
  cudaMemcpy(dd, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  const int smem = ROWS * 128 + 16 * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> o(128 * 16);
  for (int mode = 0; mode < 2; ++mode)
    for (int bmode = 0; bmode < 2; ++bmode)
      for (int s = 0; s < 12; ++s) {
        const int boff = bmode ? (s & 7) : 0;
        probe<<<1, 128, smem>>>(dd, db, mode, s, boff, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 16; ++n) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) {
              const double a = mode == 0 ? fd[(s + m) * 64 + k]
                                         : fd[(s + k + (m >= 64 ? 1 : 0)) * 64 + (m & 63)];
              ref += a * fb[n * 64 + k];
            }
            maxerr = std::max(maxerr, std::fabs(ref - o[m * 16 + n]));
          }
        printf("mode %s s=%2d base_offset=%d  max|err| = %g %s\n", mode ? "MN" : "K ", s, boff, maxerr,
               maxerr < 1e-3 ? "OK" : "MISMATCH");
      }
  return 0;
}
