// vtrace.cu — K1: V-trace targets as a lane-group reverse affine scan (H6).
//
// Definition: S:140 / include/seed.h seed_vtrace (IMPALA recursion).
// The recursion acc_t = delta_t + gamma_t c_t acc_{t+1} (acc = vs - V) is an
// affine map x -> b_t + a_t x per step, so a trajectory is processed by a
// group of G lanes: lane l owns 4 consecutive steps (one float4 per input
// array), composes its 4 maps serially, the group runs a log2(G)-step suffix
// scan of maps with shuffles, and each lane then finishes its own 4 outputs.
// Trajectories longer than 4G are processed in chunks from the end with a
// carried accumulator.  HBM traffic is exactly 28 B per (b,t) + 4 B per b.
#include "common.cuh"
#include "vtrace_scan.cuh"

namespace seed {

template <int G, bool VEC>
__global__ void __launch_bounds__(256) vtrace_kernel(
    int T, int B, const float* __restrict__ blp, const float* __restrict__ tlp,
    const float* __restrict__ rew, const float* __restrict__ disc,
    const float* __restrict__ val, const float* __restrict__ boot, float rho_bar, float c_bar,
    float lam, float* __restrict__ vs_out, float* __restrict__ pg_out, int* flag) {
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int lane = threadIdx.x % G;
  const bool active = gid < B;
  const int b = active ? gid : B - 1;  // keep the whole warp in the shuffles
  const size_t row = (size_t)b * T;
  VtraceLaneState st;
  st.init(boot[b]);
  bool bad = !isfinite(st.carry_vs);
  const int CH = 4 * G;
  const int nch = (T + CH - 1) / CH;
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int t0 = ch * CH + 4 * lane;
    float d[4], r[4], g[4], v[4];
    if (VEC && t0 + 3 < T) {
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(blp + row + t0));
      const float4 x1 = __ldg(reinterpret_cast<const float4*>(tlp + row + t0));
      const float4 x2 = __ldg(reinterpret_cast<const float4*>(rew + row + t0));
      const float4 x3 = __ldg(reinterpret_cast<const float4*>(disc + row + t0));
      const float4 x4 = __ldg(reinterpret_cast<const float4*>(val + row + t0));
      d[0] = x1.x - x0.x; d[1] = x1.y - x0.y; d[2] = x1.z - x0.z; d[3] = x1.w - x0.w;
      r[0] = x2.x; r[1] = x2.y; r[2] = x2.z; r[3] = x2.w;
      g[0] = x3.x; g[1] = x3.y; g[2] = x3.z; g[3] = x3.w;
      v[0] = x4.x; v[1] = x4.y; v[2] = x4.z; v[3] = x4.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        if (t < T) {
          d[j] = __ldg(tlp + row + t) - __ldg(blp + row + t);
          r[j] = __ldg(rew + row + t);
          g[j] = __ldg(disc + row + t);
          v[j] = __ldg(val + row + t);
        } else {
          d[j] = 0.f; r[j] = 0.f; g[j] = 0.f; v[j] = 0.f;
        }
      }
    }
    float vs[4], pg[4];
    bad |= vtrace_chunk<G>(st, lane, t0, T, d, r, g, v, rho_bar, c_bar, lam, vs, pg);
    if (active) {
      if (VEC && t0 + 3 < T) {
        *reinterpret_cast<float4*>(vs_out + row + t0) = make_float4(vs[0], vs[1], vs[2], vs[3]);
        *reinterpret_cast<float4*>(pg_out + row + t0) = make_float4(pg[0], pg[1], pg[2], pg[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (t0 + j < T) {
            vs_out[row + t0 + j] = vs[j];
            pg_out[row + t0 + j] = pg[j];
          }
      }
    }
  }
  if (bad && active && flag) *flag = 1;
}

template <int G>
static void launch_vtrace_g(bool vec, int T, int B, const float* blp, const float* tlp,
                            const float* rew, const float* disc, const float* val,
                            const float* boot, float rho_bar, float c_bar, float lam, float* vs,
                            float* pg, int* flag, cudaStream_t st) {
  const long long threads = (long long)B * G;
  const int blocks = (int)((threads + 255) / 256);
  if (vec)
    vtrace_kernel<G, true><<<blocks, 256, 0, st>>>(T, B, blp, tlp, rew, disc, val, boot,
                                                   rho_bar, c_bar, lam, vs, pg, flag);
  else
    vtrace_kernel<G, false><<<blocks, 256, 0, st>>>(T, B, blp, tlp, rew, disc, val, boot,
                                                    rho_bar, c_bar, lam, vs, pg, flag);
}

int vtrace_group_size(int T) {
  int need = (T + 3) / 4, G = 1;
  while (G < need && G < 32) G <<= 1;
  return G;
}

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_vtrace(int T, int B, const float* blp, const float* tlp,
                                   const float* rew, const float* disc, const float* val,
                                   const float* boot, float rho_bar, float c_bar, float lam,
                                   float* vs, float* pg, int* flag, void* stream) {
  if (T < 1 || B < 1) return SEED_E_SHAPE;
  if (!blp || !tlp || !rew || !disc || !val || !boot || !vs || !pg) return SEED_E_ARG;
  if (!(c_bar > 0.f) || !(rho_bar >= c_bar) || !(lam >= 0.f && lam <= 1.f)) return SEED_E_ARG;
  const bool vec = (T % 4 == 0) && aligned16(blp) && aligned16(tlp) && aligned16(rew) &&
                   aligned16(disc) && aligned16(val) && aligned16(vs) && aligned16(pg);
  cudaStream_t st = (cudaStream_t)stream;
  switch (vtrace_group_size(T)) {
    case 1: launch_vtrace_g<1>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
    case 2: launch_vtrace_g<2>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
    case 4: launch_vtrace_g<4>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
    case 8: launch_vtrace_g<8>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
    case 16: launch_vtrace_g<16>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
    default: launch_vtrace_g<32>(vec, T, B, blp, tlp, rew, disc, val, boot, rho_bar, c_bar, lam, vs, pg, flag, st); break;
  }
  return last_launch();
}
