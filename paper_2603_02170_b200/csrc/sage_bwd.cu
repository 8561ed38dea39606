// sage_bwd.cu -- K4: SageBwd backward, Alg. 2.  One CTA per
// (head, 128-key block j), looping over query blocks i (kv-stationary, Alg. 2 loop
// order: j outer, i inner).  Everything is computed transposed so that
// TMEM lanes are key rows:
//   S^T   = MM(K^_j, Q^_i)          kind::i8   A K^_j K-major, B Q^_i K-major     (line 5)
//   P     = exp(S - L_i);  psi(P) over the 128x128 tile (reading A11)               (line 5-6)
//   dP^T  = V_j dO_i^T               kind::f16  bf16 operands, fp32 accumulation     (line 8)
//   dS    = P o (dP - D_i);  psi(dS) over the tile                                   (line 9)
//   dV_j += MM(P^^T, dO^_i) s_P s_dO    A P^^T smem K-major, B dO^_i MN-major        (line 7)
//   dK_j += MM(dS^^T, Q^_i) s_dS s_Q tau  (+ tau s_dS colsum(dS^) mu_Qi)  (line 11)
//   dQ_i += MM(dS^, K^_j) s_dS s_K tau    A dS^ (the dS^^T tile read MN-major), B K^_j MN-major (line 10)
// dV_j, dK_j accumulate in fp32 registers (the per-tile scales forbid int32
// accumulation across tiles); dQ_i is reduced across key blocks with fp32
// red.global.add into a [B,H,N,d] accumulator (finalised to bf16 by K5).
// Roles: warps 0-3 / 4-7 = two compute warpgroups (query columns 0-63 / 64-127 of
// each tile, and d columns [0,d/2) / [d/2,d) of every drain), warp 8 = TMA
// producer, warp 9 = TMEM allocator + MMA issuer.
#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

constexpr int kThreads = 320;
constexpr int kStages = 2;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct BwdSmem {
  static constexpr int kTile = kBlk * D;           // int8 [128][D]
  static constexpr int kK = 0;                     // K^_j
  static constexpr int kV = kK + kTile;            // V_j bf16: D/64 panels of [128][64]
  static constexpr int kStage = kV + 2 * kTile;    // per stage: Q^_i, dO_i (bf16 panels), dO^_i, L2, delta
  static constexpr int kSQ = 0, kSDO = kTile, kSDOQ = 3 * kTile, kSL = 4 * kTile, kSDelta = 4 * kTile + 512;
  static constexpr int kStageBytes = 4 * kTile + 1024;
  static constexpr int kPt = kStage + kStages * kStageBytes;  // P^^T [128 kv][128 q]
  static constexpr int kDSt = kPt + kBlk * kBlk;              // dS^^T [128 kv][128 q]
  static constexpr int kRed = kDSt + kBlk * kBlk;             // 2 x 8 floats
  static constexpr int kRowSum = kRed + 64;                   // [2][128] int
  static constexpr int kBar = kRowSum + 2 * kBlk * 4;
  static constexpr int kNumBars = 1 + 2 * kStages + 10;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;
  static constexpr uint32_t kStageTx = 4 * kTile + 1024;
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// max over the 256 compute threads (warps 0-7), named barrier 1
__device__ __forceinline__ float block_max256(float v, float* red, int warp) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  named_bar_sync(1, 256);
  float r = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) r = fmaxf(r, red[w]);
  return r;
}

template <int D, bool CAUSAL, bool QSMOOTH>
__global__ void __launch_bounds__(kThreads, 1)
    sage_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_doq, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ q_scale,
                    const float* __restrict__ k_scale, const float* __restrict__ do_scale,
                    const float* __restrict__ l2g, const float* __restrict__ deltag, const float* __restrict__ bias,
                    const float* __restrict__ mu_q, float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dk,
                    __nv_bfloat16* __restrict__ dv, int N, int BH, float tau) {
  using L = BwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;              // [kStages]
  uint64_t* q_empty = q_full + kStages;     // [kStages]
  uint64_t* s_full = q_empty + kStages;
  uint64_t* dp_full = s_full + 1;
  uint64_t* dv_full = s_full + 2;
  uint64_t* dk_full = s_full + 3;
  uint64_t* dq_full = s_full + 4;
  uint64_t* s_free = s_full + 5;            // 256 arrivals each
  uint64_t* dp_free = s_full + 6;
  uint64_t* ds_ready = s_full + 7;
  uint64_t* dk_free = s_full + 8;
  uint64_t* dq_free = s_full + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  float* red = reinterpret_cast<float*>(smem + L::kRed);
  int* rowsum_s = reinterpret_cast<int*>(smem + L::kRowSum);

  const int T = N / kBlk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x;
  const int j = tile / BH;  // causal: low j has the most query blocks -> scheduled first
  const int bh = tile % BH;
  const int i0 = CAUSAL ? j : 0;
  const int n_it = T - i0;
  const int krow = bh * N + j * kBlk;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(q_full + s, 1);
      mbar_init(q_empty + s, 1);
    }
    for (int b = 0; b < 5; ++b) mbar_init(s_full + b, 1);
    for (int b = 5; b < 10; ++b) mbar_init(s_full + b, 256);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;         // S^T   cols [0,128)   int32  (lanes = key rows)
  const uint32_t tDP = tmem + 128;  // dP^T  cols [128,256) fp32 -> dS fp32 -> dV tile int32 [0,D)
  const uint32_t tDK = tmem + 256;  // dK tile int32 [0,D)
  const uint32_t tDQ = tmem + 384;  // dQ tile int32 [0,D)  (lanes = query rows)

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_doq);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_do);
      mbar_expect_tx(kv_full, 3 * L::kTile);
      tma_load_2d(smem + L::kK, &tm_k, kv_full, 0, krow);
#pragma unroll
      for (int p = 0; p < D / 64; ++p) tma_load_2d(smem + L::kV + p * 16384, &tm_v, kv_full, p * 64, krow);
      for (int it = 0; it < n_it; ++it) {
        const int s = it % kStages, i = i0 + it;
        const int qrow = bh * N + i * kBlk;
        uint8_t* st = smem + L::kStage + s * L::kStageBytes;
        mbar_wait(q_empty + s, ((it / kStages) & 1) ^ 1);
        mbar_expect_tx(q_full + s, L::kStageTx);
        tma_load_2d(st + L::kSQ, &tm_q, q_full + s, 0, qrow);
#pragma unroll
        for (int p = 0; p < D / 64; ++p) tma_load_2d(st + L::kSDO + p * 16384, &tm_do, q_full + s, p * 64, qrow);
        tma_load_2d(st + L::kSDOQ, &tm_doq, q_full + s, 0, qrow);
        bulk_load(st + L::kSL, l2g + qrow, 512, q_full + s);
        bulk_load(st + L::kSDelta, deltag + qrow, 512, q_full + s);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_i8(128, 128, false, false);     // S^T
      constexpr uint32_t kIdDP = idesc_bf16(128, 128, false, false);  // dP^T
      constexpr uint32_t kIdDV = idesc_i8(128, D, false, true);       // dV, dK (B MN-major)
      constexpr uint32_t kIdDQ = idesc_i8(128, D, true, true);        // dQ (A, B MN-major)
      const uint32_t k_addr = smem_u32(smem + L::kK);
      const uint32_t v_addr = smem_u32(smem + L::kV);
      const uint32_t pt_addr = smem_u32(smem + L::kPt);
      const uint32_t dst_addr = smem_u32(smem + L::kDSt);
      auto stage_addr = [&](int it) { return smem_u32(smem + L::kStage + (it % kStages) * L::kStageBytes); };
      auto issue_s = [&](int it) {
        mbar_wait(q_full + it % kStages, (it / kStages) & 1);
        tc_fence_after();
        const uint32_t q_addr = stage_addr(it) + L::kSQ;
#pragma unroll
        for (int kk = 0; kk < D / 32; ++kk)
          mma_i8(tS, desc_kmajor(k_addr, D, kk * 32), desc_kmajor(q_addr, D, kk * 32), kIdS, kk > 0);
        mma_commit(s_full);
      };
      auto issue_dp = [&](int it) {
        const uint32_t do_addr = stage_addr(it) + L::kSDO;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t po = (kk / 4) * 16384, ko = (kk % 4) * 32;
          mma_bf16(tDP, desc_kmajor(v_addr + po, 128, ko), desc_kmajor(do_addr + po, 128, ko), kIdDP, kk > 0);
        }
        mma_commit(dp_full);
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      issue_dp(0);
      for (int it = 0; it < n_it; ++it) {
        const uint32_t ph = it & 1;
        if (it + 1 < n_it) {
          mbar_wait(s_free, ph);  // pass 2 of `it` has consumed S^T
          issue_s(it + 1);
        }
        mbar_wait(ds_ready, ph);
        mbar_wait(dk_free, ph ^ 1);
        mbar_wait(dq_free, ph ^ 1);
        tc_fence_after();
        const uint32_t q_addr = stage_addr(it) + L::kSQ;
        const uint32_t doq_addr = stage_addr(it) + L::kSDOQ;
#pragma unroll
        for (int kk = 0; kk < kBlk / 32; ++kk)
          mma_i8(tDP, desc_kmajor(pt_addr, 128, kk * 32), desc_mnmajor(doq_addr, D, kk * 32), kIdDV, kk > 0);
        mma_commit(dv_full);
#pragma unroll
        for (int kk = 0; kk < kBlk / 32; ++kk)
          mma_i8(tDK, desc_kmajor(dst_addr, 128, kk * 32), desc_mnmajor(q_addr, D, kk * 32), kIdDV, kk > 0);
        mma_commit(dk_full);
#pragma unroll
        for (int kk = 0; kk < kBlk / 32; ++kk)
          mma_i8(tDQ, desc_mnmajor(dst_addr, 128, kk * 32), desc_mnmajor(k_addr, D, kk * 32), kIdDQ, kk > 0);
        mma_commit(dq_full);
        mma_commit(q_empty + it % kStages);
        if (it + 1 < n_it) {
          mbar_wait(dp_free, ph);  // dV tile of `it` drained out of the dP columns
          tc_fence_after();
          issue_dp(it + 1);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ compute warpgroups (256 threads)
    const int wg = warp / 4;
    const int r = (warp % 4) * 32 + lane;  // TMEM lane: key row (S, dP, dV, dK) or query row (dQ)
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    const int qc0 = wg * 64;               // this warpgroup's query columns of the tile
    constexpr int kHalf = D / 2;           // this warpgroup's d columns of every drain
    const int dc0 = wg * kHalf;
    const float tau2 = tau * kLog2e;
    const float sk = k_scale[(size_t)bh * T + j];
    float dv_acc[kHalf], dk_acc[kHalf];
#pragma unroll
    for (int c = 0; c < kHalf; ++c) dv_acc[c] = dk_acc[c] = 0.f;

    for (int it = 0; it < n_it; ++it) {
      const int i = i0 + it, s = it % kStages;
      const uint32_t ph = it & 1;
      const uint8_t* st = smem + L::kStage + s * L::kStageBytes;
      const float* Ls = reinterpret_cast<const float*>(st + L::kSL);
      const float* Ds = reinterpret_cast<const float*>(st + L::kSDelta);
      const float sq = q_scale[(size_t)bh * T + i];
      const float sdo = do_scale[(size_t)bh * T + i];
      const float c2 = sq * sk * tau2;
      const float b2 = QSMOOTH ? bias[((size_t)bh * T + i) * N + (size_t)j * kBlk + r] * tau2 : 0.f;
      const bool diag = CAUSAL && (i == j);
      mbar_wait(q_full + s, (it / kStages) & 1);
      mbar_wait(s_full, ph);
      tc_fence_after();
      // pass 1: max over the tile of t = log2 P = S*c2 + b2 - L2[q]
      float tmax = -INFINITY;
#pragma unroll 1
      for (int cc = 0; cc < 64; cc += 32) {
        uint32_t v[32];
        tmem_ld32(tS + qc0 + cc + lane_off, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int q = qc0 + cc + e;
          const float t = fmaf(__int2float_rn((int)v[e]), c2, b2 - Ls[q]);
          if (!diag || r <= q) tmax = fmaxf(tmax, t);
        }
      }
      const float amax_p = ex2(block_max256(tmax, red, warp));
      const float inv_p = amax_p > 0.f ? __fdiv_rn(127.f, amax_p) : 0.f;
      const float s_p = amax_p * (1.f / 127.f);
      mbar_wait(dp_full, ph);
      tc_fence_after();
      // pass 2: P, psi(P) -> P^^T smem; dS = P (dP - delta) -> back into the dP columns
      uint8_t* pt = smem + L::kPt;
      float dsmax = 0.f;
#pragma unroll 1
      for (int cc = 0; cc < 64; cc += 16) {
        uint32_t sv[16], dpv[16];
        tmem_ld16(tS + qc0 + cc + lane_off, sv);
        tmem_ld16(tDP + qc0 + cc + lane_off, dpv);
        tmem_wait_ld();
        uint32_t pk[4];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          uint32_t w = 0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = e4 * 4 + t, q = qc0 + cc + e;
            float p = ex2(fmaf(__int2float_rn((int)sv[e]), c2, b2 - Ls[q]));
            if (diag && r > q) p = 0.f;
            w |= rne_small(fminf(p * inv_p, 127.f)) << (8 * t);
            const float ds = p * (__uint_as_float(dpv[e]) - Ds[q]);
            dsmax = fmaxf(dsmax, fabsf(ds));
            dpv[e] = __float_as_uint(ds);
          }
          pk[e4] = w;
        }
        tmem_st16(tDP + qc0 + cc + lane_off, dpv);
        *reinterpret_cast<uint4*>(pt + sw_offset(r, (qc0 + cc) / 16, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(s_free);
      const float amax_ds = block_max256(dsmax, red + 8, warp);
      const float inv_ds = amax_ds > 0.f ? __fdiv_rn(127.f, amax_ds) : 0.f;
      const float s_ds = amax_ds * (1.f / 127.f);
      // pass 3: psi(dS) -> dS^^T smem (K-major for dK, read MN-major for dQ)
      uint8_t* dst = smem + L::kDSt;
      int rsum = 0;
#pragma unroll 1
      for (int cc = 0; cc < 64; cc += 16) {
        uint32_t dsv[16];
        tmem_ld16(tDP + qc0 + cc + lane_off, dsv);
        tmem_wait_ld();
        uint32_t pk[4];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          uint32_t w = 0;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float x = fminf(fmaxf(__uint_as_float(dsv[e4 * 4 + t]) * inv_ds, -127.f), 127.f);
            const uint32_t qb = rne_small(x);
            if (QSMOOTH) rsum += (int)(int8_t)(qb & 0xFF);
            w |= (qb & 0xFFu) << (8 * t);
          }
          pk[e4] = w;
        }
        *reinterpret_cast<uint4*>(dst + sw_offset(r, (qc0 + cc) / 16, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      if (QSMOOTH) rowsum_s[wg * kBlk + r] = rsum;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_ready);
      if (QSMOOTH) named_bar_sync(2, 256);
      // drain dV tile: dV_j += tile * s_P * s_dO_i  (Alg. 2 line 7)
      mbar_wait(dv_full, ph);
      tc_fence_after();
      {
        const float f = s_p * sdo;
#pragma unroll
        for (int c0 = 0; c0 < kHalf; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tDP + dc0 + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) dv_acc[c0 + e] = fmaf(__int2float_rn((int)v[e]), f, dv_acc[c0 + e]);
        }
      }
      tc_fence_before();
      mbar_arrive(dp_free);
      // drain dK tile: dK_j += tile * s_dS * s_Q * tau (+ Q-smoothing bias branch)  (line 11)
      mbar_wait(dk_full, ph);
      tc_fence_after();
      {
        const float f = s_ds * sq * tau;
        const float fb = QSMOOTH ? tau * s_ds * (float)(rowsum_s[r] + rowsum_s[kBlk + r]) : 0.f;
        const float* muq = QSMOOTH ? mu_q + ((size_t)bh * T + i) * D + dc0 : nullptr;
#pragma unroll
        for (int c0 = 0; c0 < kHalf; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tDK + dc0 + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            float add = __int2float_rn((int)v[e]) * f;
            if (QSMOOTH) add = fmaf(fb, muq[c0 + e], add);
            dk_acc[c0 + e] += add;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(dk_free);
      // drain dQ tile: dQ_i += tile * s_dS * s_K * tau, fp32 reduction across key blocks (line 10)
      mbar_wait(dq_full, ph);
      tc_fence_after();
      {
        const float f = s_ds * sk * tau;
        float* grow = dq_acc + ((size_t)bh * N + (size_t)i * kBlk + r) * D + dc0;
#pragma unroll
        for (int c0 = 0; c0 < kHalf; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tDQ + dc0 + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            red_add_v4(grow + c0 + e, __int2float_rn((int)v[e]) * f, __int2float_rn((int)v[e + 1]) * f,
                       __int2float_rn((int)v[e + 2]) * f, __int2float_rn((int)v[e + 3]) * f);
        }
      }
      tc_fence_before();
      mbar_arrive(dq_free);
    }
    // epilogue: dK_j, dV_j rows -> bf16
    const size_t orow = ((size_t)krow + r) * D + dc0;
#pragma unroll
    for (int c0 = 0; c0 < kHalf; c0 += 8) {
      __nv_bfloat162 hk[4], hv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hk[e] = __floats2bfloat162_rn(dk_acc[c0 + 2 * e], dk_acc[c0 + 2 * e + 1]);
        hv[e] = __floats2bfloat162_rn(dv_acc[c0 + 2 * e], dv_acc[c0 + 2 * e + 1]);
      }
      *reinterpret_cast<uint4*>(dk + orow + c0) = *reinterpret_cast<uint4*>(hk);
      *reinterpret_cast<uint4*>(dv + orow + c0) = *reinterpret_cast<uint4*>(hv);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool C, bool QS>
cudaError_t launch_t(const BwdArgs& a, cudaStream_t s) {
  auto kern = sage_bwd_kernel<D, C, QS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem<D>::kAlloc);
  if (e != cudaSuccess) return e;
  const int T = a.N / kBlk;
  kern<<<a.BH * T, kThreads, BwdSmem<D>::kAlloc, s>>>(a.tm_q, a.tm_k, a.tm_doq, a.tm_v, a.tm_do, a.q_scale,
                                                       a.k_scale, a.do_scale, a.l2, a.delta, a.bias, a.mu_q,
                                                       a.dq_acc, a.dk, a.dv, a.N, a.BH, a.tau);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bwd(const BwdArgs& a, cudaStream_t s) {
  if (a.d == 128) {
    if (a.causal) return a.qsmooth ? launch_t<128, true, true>(a, s) : launch_t<128, true, false>(a, s);
    return a.qsmooth ? launch_t<128, false, true>(a, s) : launch_t<128, false, false>(a, s);
  }
  if (a.causal) return a.qsmooth ? launch_t<64, true, true>(a, s) : launch_t<64, true, false>(a, s);
  return a.qsmooth ? launch_t<64, false, true>(a, s) : launch_t<64, false, false>(a, s);
}

}  // namespace sage
