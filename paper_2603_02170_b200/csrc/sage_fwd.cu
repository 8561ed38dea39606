// sage_fwd.cu -- K2: SageBwd forward, Alg. 1, one CTA per
// (head, 128-query block i).  tcgen05 kind::i8 MMAs with TMEM accumulators, TMA
// into 128B/64B-swizzled shared memory, warp-specialised roles:
//   warps 0-3  softmax + correction + epilogue (thread t owns query row t = TMEM lane t)
//   warp  4    TMA producer (Q^_i once, K^_j / V^_j ring)
//   warp  5    TMEM allocator + MMA issuer (one thread)
// Per kv tile j (Alg. 1 lines 7-10, with the corrections of reading A7):
//   S_ij   = MM(Q^_i, K^_j) s_Q s_K tau            int32 in TMEM S[j%2], scaled in fp32
//   m_ij   = max(m, rowmax S_ij);  alpha = e^{m - m_ij}
//   P~     = e^{S - m_ij} = e^{S - rowmax} e^{rowmax - m_ij}
//   s_P    = e^{rowmax - m_ij}/127,  P^ = RNE(P~/s_P) = RNE(127 e^{S - rowmax})  in [0,127]
//   l      = alpha l + e^{rowmax - m_ij} sum(e^{S - rowmax})
//   O      = alpha O + MM(P^, V^_j) s_P s_V        (int32 in TMEM PV[j%2], drained to fp32 regs)
// All exponentials are base 2 on log2(e)-prescaled logits (one MUFU.EX2 per score).
#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

constexpr int kStages = 3;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct FwdSmem {
  static constexpr int kTile = kBlk * D;        // bytes of an int8 [128][D] tile
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kP = kV + kStages * kTile;  // 2 x [128][128] int8
  static constexpr int kBias = kP + 2 * kBlk * kBlk;  // 2 x 128 floats (Q-smoothing)
  static constexpr int kBar = kBias + 2 * kBlk * 4;
  static constexpr int kNumBars = 1 + 4 * kStages + 12;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;  // slack for 1024-byte alignment
};

template <int D, bool CAUSAL, bool QSMOOTH>
__global__ void __launch_bounds__(kThreads, 1)
    sage_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const float* __restrict__ q_scale,
                    const float* __restrict__ k_scale, const float* __restrict__ v_scale,
                    const float* __restrict__ bias, __nv_bfloat16* __restrict__ o, float* __restrict__ lse, int N,
                    int BH, float tau) {
  using L = FwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by offsetting the __shared__ array itself, so every
  // derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kStages;
  uint64_t* v_full = k_empty + kStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;  // [2]
  uint64_t* s_empty = s_full + 2;        // [2]
  uint64_t* p_full = s_empty + 2;        // [2]
  uint64_t* p_empty = p_full + 2;        // [2]
  uint64_t* o_full = p_empty + 2;        // [2]
  uint64_t* o_empty = o_full + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  float* bias_s = reinterpret_cast<float*>(smem + L::kBias);

  const int T = N / kBlk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // Longest-first order for causal: high query blocks have the most kv tiles.
  const int tile = blockIdx.x;
  // head-major order (the CTAs of one head share K^/V^ through L2); causal: longest (high i) first
  const int bh = tile / T;
  const int i = CAUSAL ? (T - 1 - tile % T) : (tile % T);
  const int nj = CAUSAL ? i + 1 : T;
  const int row0 = bh * N + i * kBlk;  // first global row of this q block

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(s_empty + b, 128);
      mbar_init(p_full + b, 128);
      mbar_init(p_empty + b, 1);
      mbar_init(o_full + b, 1);
      mbar_init(o_empty + b, 128);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;          // S[b] at columns 128*b
  const uint32_t tPV = tmem + 256;   // PV[b] at columns 256 + D*b

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(q_full, L::kTile);
      tma_load_2d(smem + L::kQ, &tm_q, q_full, 0, row0);
      for (int j = 0; j < nj; ++j) {
        const int st = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const int krow = bh * N + j * kBlk;
        mbar_wait(k_empty + st, ph ^ 1);
        mbar_expect_tx(k_full + st, L::kTile);
        tma_load_2d(smem + L::kK + st * L::kTile, &tm_k, k_full + st, 0, krow);
        mbar_wait(v_empty + st, ph ^ 1);
        mbar_expect_tx(v_full + st, L::kTile);
        tma_load_2d(smem + L::kV + st * L::kTile, &tm_v, v_full + st, 0, krow);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_i8(128, 128, false, false);
      constexpr uint32_t kIdPV = idesc_i8(128, D, false, true);
      const uint32_t q_addr = smem_u32(smem + L::kQ);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int st = j % kStages, b = j & 1;
        mbar_wait(k_full + st, (j / kStages) & 1);
        mbar_wait(s_empty + b, ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(smem + L::kK + st * L::kTile);
#pragma unroll
        for (int kk = 0; kk < D / 32; ++kk)
          mma_i8(tS + 128 * b, desc_kmajor(q_addr, D, kk * 32), desc_kmajor(k_addr, D, kk * 32), kIdS, kk > 0);
        mma_commit(k_empty + st);
        mma_commit(s_full + b);
      };
      auto issue_pv = [&](int j) {
        const int st = j % kStages, b = j & 1;
        mbar_wait(p_full + b, (j >> 1) & 1);
        mbar_wait(v_full + st, (j / kStages) & 1);
        mbar_wait(o_empty + b, ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(smem + L::kP + b * kBlk * kBlk);
        const uint32_t v_addr = smem_u32(smem + L::kV + st * L::kTile);
#pragma unroll
        for (int kk = 0; kk < kBlk / 32; ++kk)
          mma_i8(tPV + D * b, desc_kmajor(p_addr, 128, kk * 32), desc_mnmajor(v_addr, D, kk * 32), kIdPV, kk > 0);
        mma_commit(v_empty + st);
        mma_commit(p_empty + b);
        mma_commit(o_full + b);
      };
      for (int j = 0; j < nj; ++j) {
        issue_s(j);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nj - 1);
    }
  } else {
    // ------------------------------------------------------------ softmax / correction (128 threads)
    const int r = threadIdx.x;  // query row within the block == TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const float sq = q_scale[(size_t)bh * T + i];
    const float tau2 = tau * kLog2e;
    float oacc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) oacc[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    float prev_alpha = 0.f, prev_spv = 0.f;

    auto correct = [&](int j, float alpha, float spv) {
      const int b = j & 1;
      mbar_wait(o_full + b, (j >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tPV + D * b + c0 + lane_off, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          oacc[c0 + e] = fmaf(alpha, oacc[c0 + e], __int2float_rn((int)v[e]) * spv);
      }
      tc_fence_before();
      mbar_arrive(o_empty + b);
    };

    for (int j = 0; j < nj; ++j) {
      const int b = j & 1;
      const float c2 = sq * k_scale[(size_t)bh * T + j] * tau2;  // int32 -> log2-domain logit
      const bool diag = CAUSAL && (j == i);
      if constexpr (QSMOOTH) {
        // bias row (tau*log2e * mu_Qi . K_sm[n]) for this kv tile, shared by all rows
        named_bar_sync(1, 128);
        bias_s[b * kBlk + r] = bias[((size_t)bh * T + i) * N + (size_t)j * kBlk + r] * tau2;
        named_bar_sync(1, 128);
      }
      mbar_wait(s_full + b, (j >> 1) & 1);
      tc_fence_after();
      // pass 1: row max (on int32 when there is no per-column bias)
      float rm;
      if constexpr (!QSMOOTH) {
        int mx = INT_MIN;
#pragma unroll 1
        for (int c0 = 0; c0 < kBlk; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tS + 128 * b + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!diag || c0 + e <= r) mx = max(mx, (int)v[e]);
        }
        rm = __int2float_rn(mx) * c2;  // max commutes with the positive scale
      } else {
        rm = -INFINITY;
#pragma unroll 1
        for (int c0 = 0; c0 < kBlk; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tS + 128 * b + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!diag || c0 + e <= r) rm = fmaxf(rm, fmaf(__int2float_rn((int)v[e]), c2, bias_s[b * kBlk + c0 + e]));
        }
      }
      const float m_new = fmaxf(m, rm);
      const float alpha = ex2(m - m_new);
      const float e_rm = ex2(rm - m_new);
      // pass 2: e = 2^{S - rowmax}, P^ = RNE(127 e) -> swizzled K-major smem row r
      mbar_wait(p_empty + b, ((j >> 1) & 1) ^ 1);
      uint8_t* prow = smem + L::kP + b * kBlk * kBlk;
      float rs = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < kBlk; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tS + 128 * b + c0 + lane_off, v);
        tmem_wait_ld();
        uint32_t pk[8];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          uint32_t w = 0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = e4 * 4 + t;
            float s2 = QSMOOTH ? fmaf(__int2float_rn((int)v[e]), c2, bias_s[b * kBlk + c0 + e]) - rm
                               : fmaf(__int2float_rn((int)v[e]), c2, -rm);
            float p = ex2(s2);
            if (diag && c0 + e > r) p = 0.f;
            rs += p;
            w |= rne_small(127.f * p) << (8 * t);
          }
          pk[e4] = w;
        }
        const int chunk = c0 / 16;
        *reinterpret_cast<uint4*>(prow + sw_offset(r, chunk, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(prow + sw_offset(r, chunk + 1, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
      tc_fence_before();
      mbar_arrive(s_empty + b);
      fence_proxy_async_smem();
      mbar_arrive(p_full + b);
      l = fmaf(alpha, l, e_rm * rs);
      const float spv = e_rm * (1.f / 127.f) * v_scale[(size_t)bh * T + j];
      m = m_new;
      if (j > 0) correct(j - 1, prev_alpha, prev_spv);
      prev_alpha = alpha;
      prev_spv = spv;
    }
    correct(nj - 1, prev_alpha, prev_spv);
    // epilogue: O = acc / l (Alg. 1 line 13), L = m + ln l (line 14, natural log)
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = o + ((size_t)row0 + r) * D;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 8) {
      __nv_bfloat162 h[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(oacc[c0 + 2 * e] * inv_l, oacc[c0 + 2 * e + 1] * inv_l);
      *reinterpret_cast<uint4*>(orow + c0) = *reinterpret_cast<uint4*>(h);
    }
    lse[(size_t)row0 + r] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool C, bool QS>
cudaError_t launch_t(const FwdArgs& a, cudaStream_t s) {
  auto kern = sage_fwd_kernel<D, C, QS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<D>::kAlloc);
  if (e != cudaSuccess) return e;
  const int T = a.N / kBlk;
  kern<<<a.BH * T, kThreads, FwdSmem<D>::kAlloc, s>>>(a.tm_q, a.tm_k, a.tm_v, a.q_scale, a.k_scale, a.v_scale,
                                                       a.bias, a.o, a.lse, a.N, a.BH, a.tau);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fwd(const FwdArgs& a, cudaStream_t s) {
  if (a.d == 128) {
    if (a.causal) return a.qsmooth ? launch_t<128, true, true>(a, s) : launch_t<128, true, false>(a, s);
    return a.qsmooth ? launch_t<128, false, true>(a, s) : launch_t<128, false, false>(a, s);
  }
  if (a.causal) return a.qsmooth ? launch_t<64, true, true>(a, s) : launch_t<64, true, false>(a, s);
  return a.qsmooth ? launch_t<64, false, true>(a, s) : launch_t<64, false, false>(a, s);
}

}  // namespace sage
