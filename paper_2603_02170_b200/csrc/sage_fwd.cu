// sage_fwd.cu -- K2: SageBwd forward, Alg. 1, one CTA per
// (head, 128-query block i), two CTAs resident per SM (TMEM 256 columns, <= 113 KB smem,
// setmaxnreg) so one CTA's softmax overlaps the other's MMAs and TMEM round trips.  Within a CTA
// S is double-buffered in TMEM (PV_j reuses S_j's buffer once S_j is consumed), and the O update
// for tile j-1 runs before tile j's exponential pass, so S_{j+1} is on the tensor cores while
// tile j is being exponentiated.
// tcgen05 kind::i8 MMAs with TMEM accumulators, TMA into 128B/64B-swizzled shared
// memory, warp-specialised roles:
//   warps 0-3  softmax + correction + epilogue (thread t owns query row t = TMEM lane t)
//   warp  4    TMA producer (Q^_i once, K^_j / V^_j ring), one elected lane
//   warp  5    TMEM allocator + MMA issuer, one elected lane
//   warps 6-7  idle (they complete warpgroup 1 for setmaxnreg)
// Per kv tile j (Alg. 1 lines 7-10, with the corrections of reading A7):
//   S_ij   = MM(Q^_i, K^_j) s_Q s_K tau            int32 in TMEM, scaled in fp32
//   m_ij   = max(m, rowmax S_ij);  alpha = e^{m - m_ij}
//   P~     = e^{S - m_ij} = e^{S - rowmax} e^{rowmax - m_ij}
//   s_P    = e^{rowmax - m_ij}/127,  P^ = RNE(P~/s_P) = RNE(127 e^{S - rowmax})  in [0,127]
//   l      = alpha l + e^{rowmax - m_ij} sum(e^{S - rowmax})
//   O      = alpha O + MM(P^, V^_j) s_P s_V        (int32 in TMEM, drained to fp32 registers)
// All exponentials are base 2 on log2(e)-prescaled logits (one MUFU.EX2 per score); the
// factor 127 is folded into the exponent, p' = 2^{s - rowmax + log2 127} = 127 e^{S - rowmax}.
#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

constexpr int kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLog2_127 = 6.988684686772166f;
constexpr float kLog2_255 = 7.994353436858858f;
constexpr float kLog2_448 = 8.807354922057604f;
// Groups of 4 (of the 8 per 32-column chunk) whose exponentials run on the FMA pipe (ex2_poly2), at
// d=128 (measured: 1 group = 12.5% of the exponentials, C4 K2 4.52 -> 4.40 ms; 2 neutral, 3 slower;
// none at d=64, where it does not help)
// softmax warpgroup registers (setmaxnreg); the other warpgroup gets 256 - this (2 CTAs per SM)
#ifndef SAGE_K2_REGS
#define SAGE_K2_REGS 216  // measured: 184 -> 216 takes C3 K2 0.966 -> 0.893 ms, C4 4.39 -> 4.35 ms
#endif
#ifndef SAGE_K2_PAIR
#define SAGE_K2_PAIR 1  // d=128: pass 1 and the O update load two 32-column TMEM chunks per wait
#endif                  // (measured: C3 K2 0.911 -> 0.877 ms, C4 4.44 -> 4.40; d=64 neutral, so off there)
#ifndef SAGE_K2_POLY
#define SAGE_K2_POLY 1
#endif
#ifndef SAGE_K2_HGROUP
#define SAGE_K2_HGROUP 4  // CTA order: groups of this many heads, within a group the longest query blocks first
                          // across its heads (1 = head-major), as in K4
#endif
#ifndef SAGE_K2_P2DB
#define SAGE_K2_P2DB 1  // pass 2 in 16-column pieces, the next piece's TMEM load in flight (0: 32-column chunks)
#endif

#ifndef SAGE_TRACE
#define SAGE_TRACE 0
#endif
// Profiling-only timeline (libsage_trace.so, SAGE_ABLATE bit 8), read back by sage_debug_trace
// after the K4 timeline: [4 CTAs][64 tiles][24 events] clock64 stamps.
constexpr int kTrCtas = 4, kTrTiles = 64, kTrEvents = 24;
__device__ unsigned long long g_trace_fwd[kTrCtas * kTrTiles * kTrEvents];
#define TRF(ev, jj)                                                                 \
  do {                                                                              \
    if (SAGE_TRACE && (ablate & 8) && blockIdx.x < kTrCtas && (jj) < kTrTiles)      \
      g_trace_fwd[(blockIdx.x * kTrTiles + (jj)) * kTrEvents + (ev)] = clock64();   \
  } while (0)

// Test-only dump (libsage_trace.so, SAGE_ABLATE bit 16, sage_debug_fwd_dump): K2's own S accumulator,
// per-token P^ and s_P and the PV accumulator of every processed tile, heads bh < g_fdump.heads.
__device__ FwdDump g_fdump;
#define FDUMPING (SAGE_TRACE && (ablate & 16) && bh < g_fdump.heads)

template <int D>
struct FwdSmem {
  static constexpr int kStages = D == 64 ? 3 : 2;
  static constexpr int kTile = kBlk * D;        // bytes of an int8 [128][D] tile
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + kStages * kTile;
  static constexpr int kP = kV + kStages * kTile;  // [128][128] int8 P^, K-major 128B-swizzled
  static constexpr int kBias = kP + kBlk * kBlk;   // 2 x 128 floats (Q-smoothing)
  static constexpr int kBar = kBias + 2 * kBlk * 4;
  static constexpr int kNumBars = 1 + 4 * kStages + 5;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;  // slack for 1024-byte alignment
};

// FP8 (SAGE_PV_FP8): P^ and V^ in E4M3 and P^V^ as a kind::f8f6f4 MMA (fp32 accumulator) -- a separate
// instantiation, the INT8 path of Alg. 1 untouched.  RAG: N is not a multiple of 128 (reading A33; the
// last kv tile's missing keys are masked -- a separate instantiation keeps the check out of the common
// kernels' inner loops, where it cost 8-20%)
template <int D, bool CAUSAL, bool QSMOOTH, bool FP8, bool RAG>
__global__ void __launch_bounds__(kThreads, 2)
    sage_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const float* __restrict__ q_scale,
                    const float* __restrict__ k_scale, const float* __restrict__ v_scale,
                    const float* __restrict__ bias, void* __restrict__ o_out, float* __restrict__ lse, int N,
                    int BH, float tau, int pu8, int fp16, int f32out, IoLayout io, int ablate_arg) {
  const int ablate = SAGE_TRACE ? ablate_arg : 0;
  using L = FwdSmem<D>;
  constexpr int kStages = L::kStages;
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
  uint64_t* s_full = v_empty + kStages;  // [2] MMA -> softmax: S_j in buffer j&1 (two in flight)
  uint64_t* p_full = s_full + 2;         // softmax -> MMA (4 warps): S_j read, P^_j written
  uint64_t* o_full = s_full + 3;         // MMA -> softmax: PV_j in TMEM (P^_j read)
  uint64_t* o_empty = s_full + 4;        // softmax -> MMA (4 warps): PV_j drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  float* bias_s = reinterpret_cast<float*>(smem + L::kBias);

  // N need not be a multiple of 128 (reading A33): T blocks, the library's tiles padded to Np rows per head
  const int T = num_blocks(N), Np = T * kBlk;
  const int warp = threadIdx.x / 32;
  const uint32_t one = blockDim.x / kThreads;  // a runtime 1 (i2f2 on the FMA pipe, SAGE_I2F_FMA)
  // heads in groups of SAGE_K2_HGROUP (the group's CTAs share its K^/V^ through L2); within a group, causal:
  // longest (high i) first across its heads, so the longest CTAs never start in the grid's last wave
  const int tile = blockIdx.x;
  constexpr int kHG = SAGE_K2_HGROUP;
  const int grp = tile / (kHG * T), g_heads = min(kHG, BH - grp * kHG), within = tile - grp * kHG * T;
  const int bh = grp * kHG + within % g_heads, idx = within / g_heads;
  const int i = CAUSAL ? (T - 1 - idx) : idx;
  const int nj = CAUSAL ? i + 1 : T;
  const int row0 = bh * Np + i * kBlk;  // first row of this q block in the padded int8 tiles
  const int kv_last = N - (T - 1) * kBlk;  // keys of the last kv block (128 unless N is ragged)
  // the tile dumps (test build) are laid out for N % 128 == 0 only
  const bool dump_ok = N == Np;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_full + 1, 1);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 4);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Two 128-column buffers; tile j uses buffer j&1: S_j, then (S_j consumed) PV_j in its first D
  // columns and, for d=64, P^_j (the A operand of PV_j, 32 columns) right after PV_j.
  // S_{j+1} is computed while tile j's softmax runs.
  auto tbuf = [&](int j) { return tmem + (uint32_t)(j & 1) * 128; };
  constexpr bool kPTmem = D == 64;

  if (warp >= 4) {
    reg_dealloc<256 - SAGE_K2_REGS>();
    if (warp == 4) {
      // ---------------------------------------------------------- TMA producer
      if (elect_one()) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_expect_tx(q_full, L::kTile);
        tma_load_2d(smem + L::kQ, &tm_q, q_full, 0, row0);
      }
      __syncwarp();
      for (int j = 0; j < nj; ++j) {
        const int st = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const int krow = bh * Np + j * kBlk;
        mbar_wait(k_empty + st, ph ^ 1);
        if (elect_one()) {
          mbar_expect_tx(k_full + st, L::kTile);
          tma_load_2d(smem + L::kK + st * L::kTile, &tm_k, k_full + st, 0, krow);
        }
        __syncwarp();
        mbar_wait(v_empty + st, ph ^ 1);
        if (elect_one()) {
          mbar_expect_tx(v_full + st, L::kTile);
          tma_load_2d(smem + L::kV + st * L::kTile, &tm_v, v_full + st, 0, krow);
        }
        __syncwarp();
      }
    } else if (warp == 5) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t kIdS = idesc_i8(128, 128, false, false);
      // P^ is s8 in 0..127, or u8 in 0..255 with SAGE_P_U8 (u8 x s8 MMA)
      const uint32_t kIdPV = FP8 ? idesc_e4m3(128, D, false, true)
                                 : pu8 ? idesc_i8(128, D, false, true, true) : idesc_i8(128, D, false, true);
      const uint32_t q_addr = smem_u32(smem + L::kQ);
      const uint32_t k0 = smem_u32(smem + L::kK), v0 = smem_u32(smem + L::kV);
      const uint32_t p_addr = smem_u32(smem + L::kP);
      auto issue_s = [&](int j) {  // S_j = Q^_i K^_j^T (line 7)
        const int st = j % kStages;
        mbar_wait(k_full + st, (j / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t k_addr = k0 + st * L::kTile;
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk)
            mma_i8(tbuf(j), desc_kmajor(q_addr, D, kk * 32), desc_kmajor(k_addr, D, kk * 32), kIdS, kk > 0);
          mma_commit(k_empty + st);
          mma_commit(s_full + (j & 1));
          TRF(0, j);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int j) {  // PV_j = P^_j V^_j (line 10)
        const int st = j % kStages;
        mbar_wait(v_full + st, (j / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t v_addr = v0 + st * L::kTile;
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk) {
            if constexpr (kPTmem) {
              if constexpr (FP8)
                mma_f8_ts(tbuf(j), tbuf(j) + D + kk * 8, desc_mnmajor(v_addr, D, kk * 32), kIdPV, kk > 0);
              else
                mma_i8_ts(tbuf(j), tbuf(j) + D + kk * 8, desc_mnmajor(v_addr, D, kk * 32), kIdPV, kk > 0);
            } else {
              if constexpr (FP8)
                mma_f8(tbuf(j), desc_kmajor(p_addr, 128, kk * 32), desc_mnmajor(v_addr, D, kk * 32), kIdPV, kk > 0);
              else
                mma_i8(tbuf(j), desc_kmajor(p_addr, 128, kk * 32), desc_mnmajor(v_addr, D, kk * 32), kIdPV, kk > 0);
            }
          }
          mma_commit(v_empty + st);
          mma_commit(o_full);
          TRF(1, j);
        }
        __syncwarp();
      };
      mbar_wait(q_full, 0);
      issue_s(0);
      if (nj > 1) issue_s(1);
      for (int j = 0; j < nj; ++j) {
        mbar_wait(p_full, j & 1);  // S_j consumed, P^_j written (and PV_{j-1} drained)
        TRF(6, j);
        issue_pv(j);               // into S_j's buffer
        if (j + 2 < nj) {
          mbar_wait(o_empty, j & 1);  // PV_j drained (done early in tile j+1)
          issue_s(j + 2);            // into the same buffer
        }
      }
    }
  } else {
    reg_alloc<SAGE_K2_REGS>();
    // ------------------------------------------------------------ softmax / correction (128 threads)
    const int r = threadIdx.x;  // query row within the block == TMEM lane
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    // this row's O in the I/O layout, formed before the tile loop (the strides are not live inside it)
    const long long o_off = io.row(bh, (long long)i * kBlk + r);
    const float sq = q_scale[(size_t)bh * T + i];
    const float tau2 = tau * kLog2e;
    // P^ levels: 127, or 255 for the unsigned variant (SAGE_P_U8)
    const float log2_pmax = FP8 ? kLog2_448 : pu8 ? kLog2_255 : kLog2_127;
    const float inv_pmax = FP8 ? 1.f / 448.f : pu8 ? 1.f / 255.f : 1.f / 127.f;
    float oacc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) oacc[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    float prev_alpha = 0.f, prev_spv = 0.f;
    uint8_t* prow = smem + L::kP;

    // O = alpha O + PV s_P s_V  (Alg. 1 line 10, reading A7); alpha == 1 skips the rescale
    auto correct = [&](int jj, float alpha, float spv) {
      const uint32_t tPV = tbuf(jj);
      const float2 f = make_float2(spv, spv);
      const bool rescale = __any_sync(0xffffffffu, alpha != 1.f);
      constexpr int kPair = (SAGE_K2_PAIR && D == 128) ? 2 : 1;  // 32-column chunks per TMEM wait
#pragma unroll
      for (int cp = 0; cp < D; cp += 32 * kPair) {
        uint32_t vv[kPair][32];
#pragma unroll
        for (int h = 0; h < kPair; ++h) tmem_ld32(tPV + cp + 32 * h + lane_off, vv[h]);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < kPair; ++h) {
        const int c0 = cp + 32 * h;
        uint32_t(&v)[32] = vv[h];
        if (FDUMPING && dump_ok && g_fdump.pv) {
          int32_t* dst = g_fdump.pv + (((size_t)bh * T + jj) * N + (size_t)i * kBlk + r) * D + c0;
#pragma unroll
          for (int e = 0; e < 32; e += 4) *reinterpret_cast<uint4*>(dst + e) = make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float2 acc = make_float2(oacc[c0 + e], oacc[c0 + e + 1]);
          if (rescale) acc = fmul2(acc, make_float2(alpha, alpha));
          const float2 pv = FP8 ? make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1]))  // fp32 D
                                : i2f2(v[e], v[e + 1], one);
          acc = ffma2(pv, f, acc);
          oacc[c0 + e] = acc.x;
          oacc[c0 + e + 1] = acc.y;
        }
        }
      }
      tc_fence_before();
      warp_arrive(o_empty);
    };

    for (int j = 0; j < nj; ++j) {
      const float c2 = sq * k_scale[(size_t)bh * T + j] * tau2;  // int32 -> log2-domain logit
      const float sv = v_scale[(size_t)bh * T + j];
      // columns c < lim take part: the causal mask (key n > query r, reading A14) and the keys a short
      // last block lacks (A33); lim >= 1 always
      const bool diag = CAUSAL && (j == i);
      const bool ragged = RAG && j == T - 1;
      const int lim = RAG ? min(diag ? r + 1 : kBlk, ragged ? kv_last : kBlk) : r + 1;
      const bool masked = diag || ragged;
      const float* bj = bias_s + (j & 1) * kBlk;
      if constexpr (QSMOOTH) {
        // bias row (tau*log2e * mu_Qi . K_sm[n]) for this kv tile, shared by all rows; two slots
        // so one barrier per tile suffices (slot j&1 was last read in tile j-2)
        bias_s[(j & 1) * kBlk + r] = bias[((size_t)bh * T + i) * Np + (size_t)j * kBlk + r] * tau2;
        named_bar_sync(1, 128);
      }
      mbar_wait(s_full + (j & 1), (j >> 1) & 1);
      tc_fence_after();
      if (r == 0) TRF(2, j);
      if (FDUMPING && dump_ok && g_fdump.s) {  // the int32 S accumulator of tile (i, j), unmasked (Alg. 1 line 7)
        int32_t* dst = g_fdump.s + ((size_t)bh * N + (size_t)i * kBlk + r) * N + (size_t)j * kBlk;
#pragma unroll 1
        for (int c0 = 0; c0 < kBlk; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbuf(j) + c0 + lane_off, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<uint4*>(dst + c0 + e) = make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
      }
      // pass 1: row max (on int32 when there is no per-column bias)
      float rm;
      if constexpr (!QSMOOTH) {
        int mx = INT_MIN;
        constexpr int kPair1 = (SAGE_K2_PAIR && D == 128) ? 2 : 1;
#pragma unroll
        for (int cp = 0; cp < kBlk; cp += 32 * kPair1) {
          uint32_t vv[kPair1][32];
#pragma unroll
          for (int h = 0; h < kPair1; ++h) tmem_ld32(tbuf(j) + cp + 32 * h + lane_off, vv[h]);
          tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < kPair1; ++h) {
            const int c0 = cp + 32 * h;
            uint32_t(&v)[32] = vv[h];
            if (masked) {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (c0 + e < lim) mx = max(mx, (int)v[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 32; e += 2) mx = max(mx, max((int)v[e], (int)v[e + 1]));
            }
          }
        }
        rm = __int2float_rn(mx) * c2;  // max commutes with the positive scale
        if (r == 0) TRF(3, j);
      } else {
        rm = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < kBlk; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbuf(j) + c0 + lane_off, v);
          tmem_wait_ld();
          if (masked) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c0 + e < lim) rm = fmaxf(rm, fmaf(__int2float_rn((int)v[e]), c2, bj[c0 + e]));
          } else {  // packed: two logits per FFMA2, a three-input max per pair
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              const float4 b4 = *reinterpret_cast<const float4*>(bj + c0 + e);
              const float2 a = ffma2(i2f2(v[e], v[e + 1], one),
                                     make_float2(c2, c2), make_float2(b4.x, b4.y));
              const float2 b = ffma2(i2f2(v[e + 2], v[e + 3], one),
                                     make_float2(c2, c2), make_float2(b4.z, b4.w));
              rm = fmax3(rm, fmax3(a.x, a.y, b.x), b.y);
            }
          }
        }
      }
      const float m_new = fmaxf(m, rm);
      const float alpha = ex2(m - m_new);
      const float e_rm = ex2(rm - m_new);
      const float sub = rm - log2_pmax;  // p' = 2^{s - rm + log2 127} = 127 e^{S - rowmax}
      // O update for tile j-1 first: PV_{j-1} is ready by now, and draining it frees its buffer
      // for S_{j+1}, which then runs on the tensor cores during this tile's pass 2
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        correct(j - 1, prev_alpha, prev_spv);
      }
      // pass 2: p' and P^ = RNE(p') -> the A operand of PV_j (d=64: TMEM after PV_j's columns;
      // d=128: swizzled K-major smem, free since PV_{j-1} completed)
      float2 rs2 = make_float2(0.f, 0.f);
      uint32_t pw[kPTmem ? 32 : 1];
      // one 16-column piece of pass 2: columns c0 .. c0+15 of S_j (v) -> 16 P^ bytes
      auto pass2_16 = [&](const uint32_t* v, int c0) {
        uint32_t pk[4];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int e = e4 * 4;
          float2 a = i2f2(v[e], v[e + 1], one);
          float2 b = i2f2(v[e + 2], v[e + 3], one);
          if constexpr (QSMOOTH) {
            const float4 b4 = *reinterpret_cast<const float4*>(bj + c0 + e);
            a = ffma2(a, make_float2(c2, c2), fadd2(make_float2(b4.x, b4.y), make_float2(-sub, -sub)));
            b = ffma2(b, make_float2(c2, c2), fadd2(make_float2(b4.z, b4.w), make_float2(-sub, -sub)));
          } else {
            a = ffma2(a, make_float2(c2, c2), make_float2(-sub, -sub));
            b = ffma2(b, make_float2(c2, c2), make_float2(-sub, -sub));
          }
          // FMA-pipe exponentials (MUFU offload) for SAGE_K2_POLY groups of 4 of every 32 columns
          if (((c0 % 32) / 4 + e4) < (D == 128 ? SAGE_K2_POLY : 0)) {
            a = ex2_poly2(a);
            b = ex2_poly2(b);
          } else {
            a = make_float2(ex2(a.x), ex2(a.y));
            b = make_float2(ex2(b.x), ex2(b.y));
          }
          if (masked) {  // causal mask (reading A14), missing keys (A33) -> P = 0
            if (c0 + e >= lim) a.x = 0.f;
            if (c0 + e + 1 >= lim) a.y = 0.f;
            if (c0 + e + 2 >= lim) b.x = 0.f;
            if (c0 + e + 3 >= lim) b.y = 0.f;
          }
          rs2 = fadd2(rs2, fadd2(a, b));
          if constexpr (FP8) {
            pk[e4] = e4m3x2(a.x, a.y) | (e4m3x2(b.x, b.y) << 16);
          } else {
            const float2 qa = fadd2(a, make_float2(kMagic, kMagic));
            const float2 qb = fadd2(b, make_float2(kMagic, kMagic));
            pk[e4] = pack4_magic(qa.x, qa.y, qb.x, qb.y);
          }
        }
        if (FDUMPING && dump_ok && g_fdump.p) {
          uint8_t* dst = g_fdump.p + ((size_t)bh * N + (size_t)i * kBlk + r) * N + (size_t)j * kBlk + c0;
          *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        if constexpr (kPTmem) {
#pragma unroll
          for (int w = 0; w < 4; ++w) pw[c0 / 4 + w] = pk[w];
        } else {
          *reinterpret_cast<uint4*>(prow + sw_offset(r, c0 / 16, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      };
      if constexpr (SAGE_K2_P2DB && !QSMOOTH) {
        // 16-column pieces streamed through two register buffers: piece c+1's TMEM load is in flight
        // while piece c is exponentiated (measured: C4 K2 4.39 -> 4.25 ms; with Q-smoothing the 32-column
        // loop below is faster: C3 0.876 vs 0.944 ms)
        tmem_stream<16, kBlk / 16>(tbuf(j) + lane_off, [&](uint32_t(&v)[16], int c) { pass2_16(v, c * 16); });
      } else {
#pragma unroll
      for (int c0 = 0; c0 < kBlk; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tbuf(j) + c0 + lane_off, v);
        tmem_wait_ld();
        uint32_t pk[8];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const int e = e4 * 4;
          float2 a = i2f2(v[e], v[e + 1], one);
          float2 b = i2f2(v[e + 2], v[e + 3], one);
          if constexpr (QSMOOTH) {
            const float4 b4 = *reinterpret_cast<const float4*>(bj + c0 + e);
            a = ffma2(a, make_float2(c2, c2), fadd2(make_float2(b4.x, b4.y), make_float2(-sub, -sub)));
            b = ffma2(b, make_float2(c2, c2), fadd2(make_float2(b4.z, b4.w), make_float2(-sub, -sub)));
          } else {
            a = ffma2(a, make_float2(c2, c2), make_float2(-sub, -sub));
            b = ffma2(b, make_float2(c2, c2), make_float2(-sub, -sub));
          }
          if (e4 < (D == 128 ? SAGE_K2_POLY : 0)) {  // FMA-pipe exponentials (MUFU offload)
            a = ex2_poly2(a);
            b = ex2_poly2(b);
          } else {
            a = make_float2(ex2(a.x), ex2(a.y));
            b = make_float2(ex2(b.x), ex2(b.y));
          }
          if (masked) {  // causal mask (reading A14), missing keys (A33) -> P = 0
            if (c0 + e >= lim) a.x = 0.f;
            if (c0 + e + 1 >= lim) a.y = 0.f;
            if (c0 + e + 2 >= lim) b.x = 0.f;
            if (c0 + e + 3 >= lim) b.y = 0.f;
          }
          rs2 = fadd2(rs2, fadd2(a, b));
          if constexpr (FP8) {
            pk[e4] = e4m3x2(a.x, a.y) | (e4m3x2(b.x, b.y) << 16);
          } else {
            const float2 qa = fadd2(a, make_float2(kMagic, kMagic));
            const float2 qb = fadd2(b, make_float2(kMagic, kMagic));
            pk[e4] = pack4_magic(qa.x, qa.y, qb.x, qb.y);
          }
        }
        if (FDUMPING && dump_ok && g_fdump.p) {
          uint8_t* dst = g_fdump.p + ((size_t)bh * N + (size_t)i * kBlk + r) * N + (size_t)j * kBlk + c0;
          *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(dst + 16) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        if constexpr (kPTmem) {
#pragma unroll
          for (int w = 0; w < 8; ++w) pw[c0 / 4 + w] = pk[w];
        } else {
          const int chunk = c0 / 16;
          *reinterpret_cast<uint4*>(prow + sw_offset(r, chunk, 128)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(prow + sw_offset(r, chunk + 1, 128)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      }
      if constexpr (kPTmem) {
        tmem_st32(tbuf(j) + D + lane_off, pw);  // S_j's columns [D, D+32) have all been read
        tmem_wait_st();
      } else {
        fence_proxy_async_smem();
      }
      tc_fence_before();
      warp_arrive(p_full);
      if (r == 0) TRF(4, j);
      // l = alpha l + e^{rowmax - m_ij} sum(e^{S - rowmax})  (line 8, reading A7)
      l = fmaf(alpha, l, e_rm * inv_pmax * (rs2.x + rs2.y));
      const float spv = e_rm * inv_pmax * sv;
      if (FDUMPING && dump_ok && g_fdump.sp) g_fdump.sp[((size_t)bh * N + (size_t)i * kBlk + r) * T + j] = e_rm * inv_pmax;
      m = m_new;
      prev_alpha = alpha;
      prev_spv = spv;
    }
    mbar_wait(o_full, (nj - 1) & 1);
    tc_fence_after();
    correct(nj - 1, prev_alpha, prev_spv);
    // epilogue: O = acc / l (Alg. 1 line 13), L = m + ln l (line 14, natural log); the padded rows of a
    // short last block (A33) are not written
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
    if (i * kBlk + r >= N) {
    } else if (f32out) {  // SAGE_FP32_OUT
      float4* orow = reinterpret_cast<float4*>(static_cast<float*>(o_out) + o_off);
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 4)
        orow[c0 / 4] = make_float4(oacc[c0] * inv_l, oacc[c0 + 1] * inv_l, oacc[c0 + 2] * inv_l, oacc[c0 + 3] * inv_l);
    } else {
      // O in the I/O type (bf16, or fp16 with SAGE_FP16): 8 values per 16-byte store
      uint4* orow = reinterpret_cast<uint4*>(static_cast<uint16_t*>(o_out) + o_off);
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 8) {
        uint32_t h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = pack2_io(oacc[c0 + 2 * e] * inv_l, oacc[c0 + 2 * e + 1] * inv_l, fp16);
        orow[c0 / 8] = make_uint4(h[0], h[1], h[2], h[3]);
      }
    }
    if (i * kBlk + r < N)
      lse[(size_t)bh * N + i * kBlk + r] = l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int D, bool C, bool QS, bool F8, bool RAG>
cudaError_t launch_t(const FwdArgs& a, cudaStream_t s) {
  auto kern = sage_fwd_kernel<D, C, QS, F8, RAG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<D>::kAlloc);
  if (e != cudaSuccess) return e;
  const int T = num_blocks(a.N);
  kern<<<a.BH * T, kThreads, FwdSmem<D>::kAlloc, s>>>(a.tm_q, a.tm_k, a.tm_v, a.q_scale, a.k_scale, a.v_scale,
                                                       a.bias, a.o, a.lse, a.N, a.BH, a.tau, a.pu8 ? 1 : 0,
                                                       a.fp16 ? 1 : 0, a.f32out ? 1 : 0, a.io, a.ablate);
  return cudaGetLastError();
}

}  // namespace

cudaError_t set_fwd_dump(const FwdDump& d) { return cudaMemcpyToSymbol(g_fdump, &d, sizeof(d)); }

cudaError_t read_fwd_trace(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace_fwd)) bytes = sizeof(g_trace_fwd);
  return cudaMemcpyFromSymbol(host, g_trace_fwd, bytes);
}

template <int D, bool F8, bool RAG>
cudaError_t launch_r(const FwdArgs& a, cudaStream_t s) {
  if (a.causal) return a.qsmooth ? launch_t<D, true, true, F8, RAG>(a, s) : launch_t<D, true, false, F8, RAG>(a, s);
  return a.qsmooth ? launch_t<D, false, true, F8, RAG>(a, s) : launch_t<D, false, false, F8, RAG>(a, s);
}

template <int D, bool F8>
cudaError_t launch_d(const FwdArgs& a, cudaStream_t s) {
  return a.N % kBlk ? launch_r<D, F8, true>(a, s) : launch_r<D, F8, false>(a, s);
}

cudaError_t launch_fwd(const FwdArgs& a, cudaStream_t s) {
  if (a.d == 128) return a.pvfp8 ? launch_d<128, true>(a, s) : launch_d<128, false>(a, s);
  return a.pvfp8 ? launch_d<64, true>(a, s) : launch_d<64, false>(a, s);
}

}  // namespace sage
