// gemm_debug.cu — seed_debug_gemm: the tcgen05 engine on plain bf16 matrices
// (test / benchmark hook, include/seed.h).  Covers all four operand-major
// combinations and split-K with a deterministic fixed-order reduction.
#include "gemm_tc.cuh"

namespace seed {

template <bool AT, bool BT, bool ASYNC_MODE>
struct DebugGemm {
  static constexpr bool A_MN = AT, B_MN = BT;
  static constexpr bool ASYNC = ASYNC_MODE;
  const void* dummy = k_ones_chunk;
  int M, N, K, kb_per_split;
  const __nv_bfloat16* A;
  const __nv_bfloat16* B;
  float* D;        // [M][N]
  __device__ uint4 load_a(int i, int j) const {
    return AT ? ld16(A + (size_t)i * M + j) : ld16(A + (size_t)i * K + j);
  }
  __device__ uint4 load_b(int i, int j) const {
    return BT ? ld16(B + (size_t)i * N + j) : ld16(B + (size_t)i * K + j);
  }
  __device__ const void* ptr_a(int i, int j) const {
    return AT ? A + (size_t)i * M + j : A + (size_t)i * K + j;
  }
  __device__ const void* ptr_b(int i, int j) const {
    return BT ? B + (size_t)i * N + j : B + (size_t)i * K + j;
  }
  __device__ void store(int m, int n, float v) const { D[(size_t)m * N + n] = v; }
  static constexpr bool ROW_OUT = true;
  __device__ float* out_row(int m) const { return D + (size_t)m * N; }
  __device__ float post(int, int, float v) const { return v; }
};

template <int BN, bool AT, bool BT>
static seed_status run_dbg(int M, int N, int K, const void* A, const void* B, float* D,
                           int splits, void* ws, cudaStream_t st) {
  if (splits < 0) {  // register-staged producer
    DebugGemm<AT, BT, false> p;
    p.M = M; p.N = N; p.K = K;
    p.A = (const __nv_bfloat16*)A;
    p.B = (const __nv_bfloat16*)B;
    p.D = D;
    return launch_gemm<BN>(p, -splits, st, (float*)ws);
  }
  DebugGemm<AT, BT, true> p;
  p.M = M; p.N = N; p.K = K;
  p.A = (const __nv_bfloat16*)A;
  p.B = (const __nv_bfloat16*)B;
  p.D = D;
  return launch_gemm<BN>(p, splits, st, (float*)ws);
}

template <int BN>
static seed_status dbg_bn(int M, int N, int K, const void* A, int at, const void* B, int bt,
                          float* D, int splits, void* ws, cudaStream_t st) {
  if (!at && !bt) return run_dbg<BN, false, false>(M, N, K, A, B, D, splits, ws, st);
  if (!at && bt) return run_dbg<BN, false, true>(M, N, K, A, B, D, splits, ws, st);
  if (at && !bt) return run_dbg<BN, true, false>(M, N, K, A, B, D, splits, ws, st);
  return run_dbg<BN, true, true>(M, N, K, A, B, D, splits, ws, st);
}

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_debug_gemm(int M, int N, int K, const void* A, int a_t, const void* B,
                                       int b_t, float* D, int bn, int splits, void* ws,
                                       void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || M % 8 || N % 8 || K % 8) return SEED_E_SHAPE;
  if (!A || !B || !D || !aligned16(A) || !aligned16(B)) return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  switch (bn) {
    case 16: return dbg_bn<16>(M, N, K, A, a_t, B, b_t, D, splits, ws, st);
    case 32: return dbg_bn<32>(M, N, K, A, a_t, B, b_t, D, splits, ws, st);
    case 64: return dbg_bn<64>(M, N, K, A, a_t, B, b_t, D, splits, ws, st);
    case 128: return dbg_bn<128>(M, N, K, A, a_t, B, b_t, D, splits, ws, st);
    case 256: return dbg_bn<256>(M, N, K, A, a_t, B, b_t, D, splits, ws, st);
    default: return SEED_E_ARG;
  }
}

#ifdef SEED_LSTM_PROF
extern "C" int seed_debug_gemm_prof(long long* out) {
  return cudaMemcpyFromSymbol(out, seed::g_gemm_prof, sizeof(seed::g_gemm_prof)) == cudaSuccess ? 0 : 5;
}
#endif
