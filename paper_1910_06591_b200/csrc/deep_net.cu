// deep_net.cu — max-pool kernels and the channel-padding obs conversion of the
// IMPALA-deep torso (deep_net.cuh).
#include "deep_net.cuh"

namespace seed {

__global__ void maxpool_fwd_kernel(int64_t n, int H, int W, int H2, int W2, int C, int pt, int pl,
                                   const bf16* __restrict__ in, bf16* __restrict__ out,
                                   bf16* __restrict__ outr, uint8_t* __restrict__ arg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t q = i / C;
    const int ox = (int)(q % W2); q /= W2;
    const int oy = (int)(q % H2);
    const int64_t f = q / H2;
    float best = -INFINITY;
    int barg = 0;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      const int y = oy * 2 - pt + ky;
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const int x = ox * 2 - pl + kx;
        if (y < 0 || x < 0 || y >= H || x >= W) continue;
        const float v = bf2f(in[((f * H + y) * W + x) * C + c]);
        if (v > best) {   // strict: the first maximum in (ky, kx) order wins
          best = v;
          barg = ky * 3 + kx;
        }
      }
    }
    out[i] = to_bf(best);
    outr[i] = to_bf(fmaxf(best, 0.f));
    arg[i] = (uint8_t)barg;
  }
}

__global__ void maxpool_bwd_kernel(int64_t n, int H, int W, int H2, int W2, int C, int pt, int pl,
                                   const bf16* __restrict__ dout, const uint8_t* __restrict__ arg,
                                   bf16* __restrict__ din) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t q = i / C;
    const int x = (int)(q % W); q /= W;
    const int y = (int)(q % H);
    const int64_t f = q / H;
    float s = 0.f;
    // windows (oy, ox) with oy*2 - pt <= y <= oy*2 - pt + 2, in ascending order
    const int oy_hi = (y + pt) >> 1, ox_hi = (x + pl) >> 1;
    for (int oy = oy_hi - 1; oy <= oy_hi; ++oy) {
      if (oy < 0 || oy >= H2) continue;
      const int ky = y - (oy * 2 - pt);
      if (ky < 0 || ky > 2) continue;
      for (int ox = ox_hi - 1; ox <= ox_hi; ++ox) {
        if (ox < 0 || ox >= W2) continue;
        const int kx = x - (ox * 2 - pl);
        if (kx < 0 || kx > 2) continue;
        const int64_t o = ((f * H2 + oy) * W2 + ox) * C + c;
        if (arg[o] == ky * 3 + kx) s += bf2f(dout[o]);
      }
    }
    din[i] = to_bf(s);
  }
}

__global__ void obs_to_bf16_pad_kernel(int64_t npix, int C, int Cp, const uint8_t* __restrict__ obs,
                                       bf16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix * Cp;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t px = i / Cp;
    const int c = (int)(i % Cp);
    out[i] = to_bf(c < C ? (float)obs[px * C + c] : 0.f);
  }
}

}  // namespace seed
