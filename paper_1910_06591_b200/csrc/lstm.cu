// lstm.cu — K7/K8: persistent cluster LSTM core over T+1 serial steps.
//
// Definition (P:591 core inputs; S:47/S:57 reset; reading C15): for t = 0..T,
//   if done_t: (h, c) <- 0;  z = Xproj_t + W_h h;  i,f,o = sigmoid, g = tanh
//   c = f c + i g;  h = o tanh(c)
// The input projection Xproj = W_x x_t + b for all (T+1)B rows is one tcgen05
// GEMM beforehand; only the recurrent product is serial.  A cluster of 8 CTAs
// serves 32 batch rows: CTA r owns hidden units [32r, 32r+32), keeps its
// 128x256 slice of W_h (i,f,g,o rows of those units) resident in shared
// memory for all steps, computes its 32x128 gate block with mma.sync
// (latency-bound recurrence: the per-step product is 32x128x256), updates the
// cell for its units, and broadcasts its slice of h_t to the 8 CTAs through
// distributed shared memory; one cluster barrier per step.
// BPTT mirrors it: each CTA forms dz for its 128 gate columns, multiplies by
// its W_h slice (dz W_h, 32x256 partial), scatters the partial columns to the
// owning CTAs over DSMEM, and each owner sums the 8 partials in fixed order
// (deterministic, no atomics).
#include "lstm.cuh"
#include "gemm_tc.cuh"

namespace seed {

constexpr int HP = LSTM_U + 8;  // padded bf16 row for W slice / h buffers (conflict-free ldmatrix)
constexpr int DP = 128 + 8;     // padded bf16 row for dz
constexpr int GP = 128 + 4;     // padded fp32 row for the gate pre-activations
constexpr int RP = 36;          // padded fp32 row for the dh reduction slots

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// CTA r's W_h slice: local row lc = gate*32 + j  <-  global row gate*U + 32r + j.
// cp.async (16 B, L2 only), 16 chunks per thread (blockDim 256), left in flight:
// the caller overlaps its other setup loads and calls cp_async_wait_all().
__device__ __forceinline__ void load_wh_slice(__nv_bfloat16* Ws, const __nv_bfloat16* wh, int r) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int c = threadIdx.x + 256 * q, lc = c >> 5, kc = c & 31;
    const int gr = (lc >> 5) * LSTM_U + 32 * r + (lc & 31);
    cp_async16(smem_u32(Ws + lc * HP + kc * 8), wh + (size_t)gr * LSTM_U + kc * 8, true);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---- DSMEM transaction handshake (no cluster barrier inside the step loop):
// a producer writes its slice into every CTA's buffer with st.async, which
// credits the receiving CTA's mbarrier with the bytes; the receiver arms the
// barrier once per phase with the total bytes it expects and waits on it.
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f32x2(uint32_t raddr, float a, float b, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
      "f"(a), "f"(b), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void mbar_arm_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

constexpr int MAX_T1 = 257;

#ifdef SEED_LSTM_PROF
// diagnostic build only: per-step clock64 stamps of CTA 0, thread 0
// [kernel 0 fwd / 1 bwd][step][stamp 0..3]
__device__ long long g_lstm_prof[2][MAX_T1 + 1][4];
#define LSTM_STAMP(K, T, I) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_lstm_prof[K][T][I] = clock64();
extern "C" int seed_debug_lstm_prof(long long* out) {
  return cudaMemcpyFromSymbol(out, g_lstm_prof, sizeof(g_lstm_prof)) == cudaSuccess ? 0 : 5;
}
#else
#define LSTM_STAMP(K, T, I)
#endif
// BB = batch rows per cluster (template, multiple of 8).  The recurrent
// products put the 16-row MMA side on the gate / hidden columns and the batch
// rows on the 8-wide N side (NT = BB/8 n-tiles), so no MMA row is padding.
template <int BB>
struct LstmCfg {
  static constexpr int MR = BB;
  static constexpr int NT = MR / 8;
  static constexpr int FWD_SMEM =
      128 * HP * 2 + 2 * MR * HP * 2 + MR * GP * 4 + MR * 32 * 4 + 32 * MAX_T1 + 64;
  static constexpr int BWD_SMEM =
      128 * HP * 2 + MR * DP * 2 + 2 * 8 * MR * RP * 4 + MR * 32 * 4 + 32 * MAX_T1 + 64;
  static constexpr uint32_t H_TX_BYTES = BB * LSTM_U * 2;     // h rows from 8 CTAs, bf16
  static constexpr uint32_t R_TX_BYTES = 8 * MR * 32 * 4;     // 8 partial dh slices, fp32
};

template <int BBT>
__global__ void __cluster_dims__(LSTM_CLUSTER, 1, 1) __launch_bounds__(256, 1)
    lstm_fwd_kernel(const LstmFwdArgs a) {
  LSTM_STAMP(0, MAX_T1, 0)
  using Cfg = LstmCfg<BBT>;
  constexpr int U = LSTM_U, MR = Cfg::MR, NT = Cfg::NT;
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* Ws = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* hb = Ws + 128 * HP;
  float* gpre = reinterpret_cast<float*>(hb + 2 * MR * HP);
  float* cst = gpre + MR * GP;
  uint8_t* dn_s = reinterpret_cast<uint8_t*>(cst + MR * 32);   // [BBT][T1]
  uint64_t* hbar = reinterpret_cast<uint64_t*>(dn_s + ((32 * MAX_T1 + 15) & ~15));
  const int r = (int)cluster_rank();
  const int b0 = (blockIdx.x / LSTM_CLUSTER) * BBT;
  const int BB = min(BBT, a.B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T1 = a.T1;

  if (tid == 0) {
    mbar_init(&hbar[0], 1);
    mbar_init(&hbar[1], 1);
    fence_mbar_init();
  }
  // W_h's image was last written by the previous step's Adam (>= 2 kernels back, all of
  // which waited on their predecessors): start its load before the PDL wait so it
  // overlaps the preceding kernel's tail
  load_wh_slice(Ws, a.wh, r);   // in flight during the state loads below
  pdl_wait_trig();
  for (int i = tid; i < BBT * T1; i += 256) {
    const int b = i / T1, t = i % T1;
    dn_s[i] = (b < BB) ? a.done[(size_t)(b0 + b) * T1 + t] : 0;
  }
  // bf16 h_{-1} for all MR rows (zero past B and on a step-0 reset), float4 reads
  // issued unconditionally (all in flight), the reset applied afterwards
#pragma unroll
  for (int q = 0; q < MR * U / 4 / 256; ++q) {
    const int idx = tid + 256 * q, b = idx / (U / 4), k = (idx % (U / 4)) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b < BB) {
      const int bb = b0 + b;
      const int srow = a.state_rows ? a.state_rows[bb] : bb;
      const float4 h4 = *reinterpret_cast<const float4*>(a.h0 + (size_t)srow * U + k);
      if (!a.done[(size_t)bb * T1]) v = h4;
    }
    *reinterpret_cast<uint2*>(hb + b * HP + k) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
  for (int idx = tid; idx < MR * 32; idx += 256) {
    const int b = idx >> 5, j = idx & 31;
    float c = 0.f, h = 0.f;
    if (b < BB) {
      const int bb = b0 + b;
      const int srow = a.state_rows ? a.state_rows[bb] : bb;
      const float c0 = a.c0[(size_t)srow * U + 32 * r + j], h0 = a.h0[(size_t)srow * U + 32 * r + j];
      if (!a.done[(size_t)bb * T1]) { c = c0; h = h0; }
      if (a.Hprev) a.Hprev[((size_t)bb * T1) * U + 32 * r + j] = __float2bfloat16_rn(h);
    }
    cst[b * 32 + j] = c;
  }
  cp_async_wait_all();
  __syncthreads();
  cluster_sync_all();   // barriers initialised everywhere before any st.async
  LSTM_STAMP(0, MAX_T1, 1)

  // per-thread cell work: NQ (row, unit pair) items; BBT*16 items per CTA
  constexpr int NQ = (BBT * 16 + 255) / 256;
  int it_b[NQ], it_j[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int idx = tid + 256 * q;
    it_b[q] = idx < BBT * 16 ? idx >> 4 : BBT;   // BBT = no item
    it_j[q] = (idx & 15) * 2;
  }
  // remote (DSMEM) base addresses of the h buffers and barriers of the 8 CTAs
  uint32_t rh[LSTM_CLUSTER], rbar[2][LSTM_CLUSTER];
#pragma unroll
  for (int s2 = 0; s2 < LSTM_CLUSTER; ++s2) {
    rh[s2] = mapa_u32(smem_u32(hb), s2);
    rbar[0][s2] = mapa_u32(smem_u32(&hbar[0]), s2);
    rbar[1][s2] = mapa_u32(smem_u32(&hbar[1]), s2);
  }
  float2 xq[NQ][4];
  auto load_x = [&](int t) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (it_b[q] < BB) {
        const float* xp = a.xproj + ((size_t)(b0 + it_b[q]) * T1 + t) * (4 * U) + 32 * r + it_j[q];
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) xq[q][gq] = __ldg(reinterpret_cast<const float2*>(xp + gq * U));
      }
    }
  };
  load_x(0);
  const int gid = lane >> 2, tig = lane & 3;
  // this warp's 16 W_h rows as mma A fragments, register-resident for all steps
  uint32_t wfrag[16][4];
#pragma unroll
  for (int ks = 0; ks < 16; ++ks)
    ldsm_x4(smem_u32(Ws + (warp * 16 + (lane & 15)) * HP + ks * 16 + (lane >> 4) * 8), wfrag[ks]);
  for (int t = 0; t < T1; ++t) {
    const int cur = t & 1, nbuf = cur ^ 1;
    LSTM_STAMP(0, t, 0)
    if (tid == 0 && t + 1 < T1) mbar_arm_tx(&hbar[nbuf], Cfg::H_TX_BYTES);
    if (t > 0) mbar_wait(&hbar[cur], ((t - 1) >> 1) & 1);
    LSTM_STAMP(0, t, 1)
    const __nv_bfloat16* hcur = hb + cur * MR * HP;
    // z^T[gate col][b] = W_h slice (A, 16 gate rows per warp) x h^T (B, NT
    // n-tiles of 8 batch rows); four independent K chains (ks mod 4) shorten
    // the dependent HMMA sequence, summed in fixed order afterwards.
    float acc[4][NT][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.f;
    const int mi = lane >> 3;
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const uint32_t (&af)[4] = wfrag[ks];
      if constexpr (NT == 1) {
        uint32_t b2[2];
        ldsm_x2(smem_u32(hcur + (lane & 7) * HP + ks * 16 + (mi & 1) * 8), b2);
        mma16816(acc[ks & 3][0], af, b2[0], b2[1]);
      } else {
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          uint32_t bfr[4];
          ldsm_x4(smem_u32(hcur + (np * 16 + (mi >> 1) * 8 + (lane & 7)) * HP + ks * 16 + (mi & 1) * 8),
                  bfr);
          mma16816(acc[ks & 3][2 * np], af, bfr[0], bfr[1]);
          mma16816(acc[ks & 3][2 * np + 1], af, bfr[2], bfr[3]);
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float v = (acc[0][nt][q] + acc[1][nt][q]) + (acc[2][nt][q] + acc[3][nt][q]);
        const int col = warp * 16 + gid + (q >> 1) * 8, row = nt * 8 + tig * 2 + (q & 1);
        gpre[row * GP + col] = v;
      }
    __syncthreads();
    LSTM_STAMP(0, t, 2)
    float2 xc[NQ][4];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) xc[q][gq] = xq[q][gq];
    if (t + 1 < T1) load_x(t + 1);   // prefetch: in flight during this step's cell + exchange
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int b = it_b[q], j = it_j[q];
      if (b >= BBT) continue;
      if (b < BB) {
        const int bb = b0 + b;
        const size_t row = (size_t)bb * T1 + t;
        const int col = 32 * r + j;
        const float* gp = gpre + b * GP + j;
        float hv[2], cv[2], gi[2], gf[2], gg[2], go[2];
        const float xiv[2] = {xc[q][0].x, xc[q][0].y}, xfv[2] = {xc[q][1].x, xc[q][1].y},
                    xgv[2] = {xc[q][2].x, xc[q][2].y}, xov[2] = {xc[q][3].x, xc[q][3].y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          gi[e] = sigm(gp[e] + xiv[e]);
          gf[e] = sigm(gp[32 + e] + xfv[e]);
          gg[e] = tanh_fast(gp[64 + e] + xgv[e]);
          go[e] = sigm(gp[96 + e] + xov[e]);
          cv[e] = gf[e] * cst[b * 32 + j + e] + gi[e] * gg[e];
          hv[e] = go[e] * tanh_fast(cv[e]);
        }
        if (t + 1 < T1) {
          const bool dn = dn_s[b * T1 + t + 1] != 0;
          const float h0n = dn ? 0.f : hv[0], h1n = dn ? 0.f : hv[1];
          cst[b * 32 + j] = dn ? 0.f : cv[0];
          cst[b * 32 + j + 1] = dn ? 0.f : cv[1];
          const uint32_t pv = pack_bf16(h0n, h1n);
          const uint32_t off = (uint32_t)((nbuf * MR * HP + b * HP + col) * 2);
#pragma unroll
          for (int s2 = 0; s2 < LSTM_CLUSTER; ++s2)
            st_async_u32(rh[s2] + off, pv, nbuf ? rbar[1][s2] : rbar[0][s2]);
          if (a.Hprev) *reinterpret_cast<uint32_t*>(a.Hprev + (row + 1) * U + col) = pv;
        } else if (a.hT) {
          const int srow = a.state_rows ? a.state_rows[bb] : bb;
          *reinterpret_cast<float2*>(a.hT + (size_t)srow * U + col) = make_float2(hv[0], hv[1]);
          *reinterpret_cast<float2*>(a.cT + (size_t)srow * U + col) = make_float2(cv[0], cv[1]);
        }
        *reinterpret_cast<float2*>(a.H + row * U + col) = make_float2(hv[0], hv[1]);
        if (a.Hb)
          *reinterpret_cast<uint32_t*>(a.Hb + row * U + col) = pack_bf16(hv[0], hv[1]);
        if (a.C) *reinterpret_cast<float2*>(a.C + row * U + col) = make_float2(cv[0], cv[1]);
        if (a.gates) {
          float* gq2 = a.gates + row * (4 * U) + col;
          *reinterpret_cast<float2*>(gq2) = make_float2(gi[0], gi[1]);
          *reinterpret_cast<float2*>(gq2 + U) = make_float2(gf[0], gf[1]);
          *reinterpret_cast<float2*>(gq2 + 2 * U) = make_float2(gg[0], gg[1]);
          *reinterpret_cast<float2*>(gq2 + 3 * U) = make_float2(go[0], go[1]);
        }
      } else if (t + 1 < T1) {
        // rows beyond B still credit the receivers' transaction count (zeros)
        const uint32_t off = (uint32_t)((nbuf * MR * HP + b * HP + 32 * r + j) * 2);
#pragma unroll
        for (int s2 = 0; s2 < LSTM_CLUSTER; ++s2)
          st_async_u32(rh[s2] + off, 0u, nbuf ? rbar[1][s2] : rbar[0][s2]);
      }
    }
    __syncthreads();   // gpre / cst reuse
    LSTM_STAMP(0, t, 3)
  }
  LSTM_STAMP(0, MAX_T1, 2)
  cluster_sync_all();
}

template <int BBT>
__global__ void __cluster_dims__(LSTM_CLUSTER, 1, 1) __launch_bounds__(256, 1)
    lstm_bwd_kernel(const LstmBwdArgs a) {
  LSTM_STAMP(1, MAX_T1, 0)
  using Cfg = LstmCfg<BBT>;
  constexpr int U = LSTM_U, MR = Cfg::MR, NT = Cfg::NT;
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* Ws = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* dzs = Ws + 128 * HP;
  float* red = reinterpret_cast<float*>(dzs + MR * DP);   // [2][8][MR][RP]
  float* dcs = red + 2 * 8 * MR * RP;                      // [MR][32]
  uint8_t* dn_s = reinterpret_cast<uint8_t*>(dcs + MR * 32);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(dn_s + ((32 * MAX_T1 + 15) & ~15));
  const int r = (int)cluster_rank();
  const int b0 = (blockIdx.x / LSTM_CLUSTER) * BBT;
  const int BB = min(BBT, a.B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T1 = a.T1;

  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    fence_mbar_init();
  }
  load_wh_slice(Ws, a.wh, r);   // before the PDL wait, as in the forward
  pdl_wait_trig();
  for (int i = tid; i < BBT * T1; i += 256) {
    const int b = i / T1, t = i % T1;
    dn_s[i] = (b < BB) ? a.done[(size_t)(b0 + b) * T1 + t] : 0;
  }
  for (int i = tid; i < MR * DP; i += 256) dzs[i] = __float2bfloat16_rn(0.f);
  for (int i = tid; i < MR * 32; i += 256) dcs[i] = 0.f;
  cp_async_wait_all();
  __syncthreads();
  cluster_sync_all();
  LSTM_STAMP(1, MAX_T1, 1)

  // per-thread cell work: NQ (row, unit) items; prefetched per step
  constexpr int NQ = (BBT * 32 + 255) / 256;
  float pdh[NQ], pg[NQ][4], pc[NQ], pcp[NQ];
  auto load_in = [&](int t) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int idx = tid + 256 * q, b = idx >> 5, j = idx & 31;
      if (idx < BBT * 32 && b < BB) {
        const int bb = b0 + b;
        const size_t row = (size_t)bb * T1 + t;
        const int col = 32 * r + j;
        pdh[q] = __ldg(a.dH + row * U + col);
        const float* gq = a.gates + row * (4 * U) + col;
#pragma unroll
        for (int k = 0; k < 4; ++k) pg[q][k] = __ldg(gq + k * U);
        pc[q] = __ldg(a.C + row * U + col);
        pcp[q] = t > 0 ? __ldg(a.C + (row - 1) * U + col) : __ldg(a.c0 + (size_t)bb * U + col);
      }
    }
  };
  load_in(T1 - 1);
  const int gid = lane >> 2, tig = lane & 3;
  // W_h^T fragments (hidden units of CTA `warp` x this CTA's 128 gate columns),
  // register-resident for all steps
  uint32_t wtfrag[8][2][4];
  {
    const int mi = lane >> 3;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        ldsm_x4_t(smem_u32(Ws + (ks * 16 + (mi >> 1) * 8 + (lane & 7)) * HP + 32 * warp + mt * 16 +
                           (mi & 1) * 8),
                  wtfrag[ks][mt]);
  }
  for (int u = 0; u < T1; ++u) {
    const int t = T1 - 1 - u;
    // partials produced at step u land in buffer u&1; consumed at step u+1
    LSTM_STAMP(1, u, 0)
    if (tid == 0 && t > 0) mbar_arm_tx(&rbar[u & 1], Cfg::R_TX_BYTES);
    if (u > 0) mbar_wait(&rbar[(u - 1) & 1], ((u - 1) >> 1) & 1);
    LSTM_STAMP(1, u, 1)
    const float* rin = red + ((u - 1) & 1) * 8 * MR * RP;
    float cdh[NQ], cg[NQ][4], cc[NQ], ccp[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      cdh[q] = pdh[q]; cc[q] = pc[q]; ccp[q] = pcp[q];
#pragma unroll
      for (int k = 0; k < 4; ++k) cg[q][k] = pg[q][k];
    }
    if (t > 0) load_in(t - 1);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int idx = tid + 256 * q;
      const int b = idx >> 5, j = idx & 31;
      if (idx < BBT * 32 && b < BB) {
        const int bb = b0 + b;
        const size_t row = (size_t)bb * T1 + t;
        const int col = 32 * r + j;
        float dh = cdh[q];
        if (u > 0 && !dn_s[b * T1 + t + 1]) {
          float s = 0.f;
#pragma unroll
          for (int src = 0; src < LSTM_CLUSTER; ++src) s += rin[(src * MR + b) * RP + j];
          dh += s;
        }
        const float gi = cg[q][0], gf = cg[q][1], gg = cg[q][2], go = cg[q][3];
        const bool dn = dn_s[b * T1 + t] != 0;
        const float cp = dn ? 0.f : ccp[q];
        const float tc = tanh_fast(cc[q]);
        const float dc = dcs[b * 32 + j] + dh * go * (1.f - tc * tc);
        const float dzi = dc * gg * gi * (1.f - gi);
        const float dzf = dc * cp * gf * (1.f - gf);
        const float dzg = dc * gi * (1.f - gg * gg);
        const float dzo = dh * tc * go * (1.f - go);
        dcs[b * 32 + j] = dn ? 0.f : dc * gf;
        __nv_bfloat16* dg = a.dG + row * (4 * U) + col;
        const __nv_bfloat16 bi = __float2bfloat16_rn(dzi), bf = __float2bfloat16_rn(dzf),
                            bg = __float2bfloat16_rn(dzg), bo = __float2bfloat16_rn(dzo);
        dg[0] = bi;
        dg[U] = bf;
        dg[2 * U] = bg;
        dg[3 * U] = bo;
        dzs[b * DP + j] = bi;
        dzs[b * DP + 32 + j] = bf;
        dzs[b * DP + 64 + j] = bg;
        dzs[b * DP + 96 + j] = bo;
      }
    }
    __syncthreads();
    LSTM_STAMP(1, u, 2)
    if (t > 0) {
      // partial dh^T[j][b] over this CTA's 128 gate columns: A = W_h slice^T
      // (2 m-tiles of 16 hidden units owned by CTA `warp`), B = dz^T (NT
      // n-tiles of 8 batch rows); two K chains (ks parity), fixed-order sum.
      float acc[2][2][NT][4];
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[c2][i][j][q] = 0.f;
      const int mi = lane >> 3;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t (&af)[2][4] = wtfrag[ks];
        if constexpr (NT == 1) {
          uint32_t b2[2];
          ldsm_x2(smem_u32(dzs + (lane & 7) * DP + ks * 16 + (mi & 1) * 8), b2);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) mma16816(acc[ks & 1][mt][0], af[mt], b2[0], b2[1]);
        } else {
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {
            uint32_t bfr[4];
            ldsm_x4(smem_u32(dzs + (np * 16 + (mi >> 1) * 8 + (lane & 7)) * DP + ks * 16 + (mi & 1) * 8),
                    bfr);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              mma16816(acc[ks & 1][mt][2 * np], af[mt], bfr[0], bfr[1]);
              mma16816(acc[ks & 1][mt][2 * np + 1], af[mt], bfr[2], bfr[3]);
            }
          }
        }
      }
      // hidden units [32*warp, 32*warp+32) belong to CTA `warp`: its slot r of buffer u&1
      // CTA `warp` owns these hidden units (mapa per step: no dynamically indexed arrays)
      const uint32_t base = mapa_u32(smem_u32(red), warp) + (uint32_t)(((u & 1) * 8 + r) * MR * RP * 4);
      const uint32_t rb = mapa_u32(smem_u32(&rbar[u & 1]), warp);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = mt * 16 + gid + (q >> 1) * 8, row = nt * 8 + tig * 2 + (q & 1);
            st_async_u32(base + (row * RP + j) * 4,
                         __float_as_uint(acc[0][mt][nt][q] + acc[1][mt][nt][q]), rb);
          }
    }
    __syncthreads();   // dzs / dcs reuse
    LSTM_STAMP(1, u, 3)
  }
  LSTM_STAMP(1, MAX_T1, 2)
  cluster_sync_all();
}

template <int BBT>
static seed_status launch_fwd(const LstmFwdArgs& a, cudaStream_t st) {
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, lstm_fwd_kernel<BBT>, LstmCfg<BBT>::FWD_SMEM));
    return launch_k(lstm_fwd_kernel<BBT>, dim3(ceil_div(a.B, BBT) * LSTM_CLUSTER), dim3(256),
                  (size_t)LstmCfg<BBT>::FWD_SMEM, st, a);
}
template <int BBT>
static seed_status launch_bwd(const LstmBwdArgs& a, cudaStream_t st) {
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, lstm_bwd_kernel<BBT>, LstmCfg<BBT>::BWD_SMEM));
    return launch_k(lstm_bwd_kernel<BBT>, dim3(ceil_div(a.B, BBT) * LSTM_CLUSTER), dim3(256),
                  (size_t)LstmCfg<BBT>::BWD_SMEM, st, a);
}

// rows per cluster: spread small batches over more clusters (more SMs per step),
// fill 32-row clusters for large ones (148 SMs / 8 = 18 clusters resident)
// batch rows per 8-CTA cluster.  Forward: 16 from 33 rows on (measured at c4, B = 128:
// 8 rows 58.6 us, 16 rows 52.4, 32 rows 90.1); backward: 8 while the clusters fit the
// 148 SMs (c4: 8 rows 53.2 us, 16 rows 66.4) — its per-step exchange is heavier
static int lstm_rows_per_cluster(int B) {
  if (B <= 4 * 8) return 8;
  if (B <= 9 * 16) return 16;
  return 32;
}
static int lstm_bwd_rows_per_cluster(int B) {
  if (B <= 18 * 8) return 8;
  return lstm_rows_per_cluster(B);
}

seed_status lstm_forward(const LstmFwdArgs& a, cudaStream_t st) {
  if (a.T1 > MAX_T1) return SEED_E_SHAPE;
  switch (lstm_rows_per_cluster(a.B)) {
    case 8: return launch_fwd<8>(a, st);
    case 16: return launch_fwd<16>(a, st);
    default: return launch_fwd<32>(a, st);
  }
}

seed_status lstm_backward(const LstmBwdArgs& a, cudaStream_t st) {
  if (a.T1 > MAX_T1) return SEED_E_SHAPE;
  switch (lstm_bwd_rows_per_cluster(a.B)) {
    case 8: return launch_bwd<8>(a, st);
    case 16: return launch_bwd<16>(a, st);
    default: return launch_bwd<32>(a, st);
  }
}

}  // namespace seed
