// sage_debug.cu -- one UMMA tile through the same descriptor / swizzle / TMEM code the
// fused kernels use (Tier-B parity, sage_debug_umma in include/sage.h).
#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

// mode 0: D[128][128] = A[128][K] B[128][K]^T, A/B K-major int8 via TMA (the S tile)
// mode 1: D[128][N]   = A[128][128] B,  A K-major written by threads (P^), B [128 K][N] MN-major TMA (PV, dV, dK)
// mode 2: D[128][N]   = A B, A MN-major given as A^T [128 K][128 M] written by threads (dS^^T),
//                      B [128 K][N] MN-major TMA (dQ)
// mode 3: fp32 D[128][128] = A[128][K] B[128][K]^T, bf16 K-major panels via TMA (dP^T)
// mode 4: as mode 1 with A read from TMEM (tcgen05.st by threads, "TS" MMA): the P^ / dS^^T in TMEM paths
// mode 5: as mode 3 with A read from TMEM (bf16, 2 per 32-bit column): the V_j-in-TMEM dP^T path
// modes 6 / 7: as 1 / 4 with an unsigned u8 A operand (the SAGE_P_U8 P^ paths)
template <int MODE_, int K, int N>
__global__ void __launch_bounds__(128, 1)
    debug_umma_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                      const int8_t* __restrict__ a_host_layout, void* __restrict__ out) {
  constexpr int MODE = MODE_ == 6 ? 1 : MODE_ == 7 ? 4 : MODE_;
  constexpr bool kU8 = MODE_ >= 6;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kABytes = (MODE == 3 || MODE == 5) ? 128 * K * 2 : (MODE == 0 ? 128 * K : 128 * 128);
  constexpr int kBBytes = (MODE == 3 || MODE == 5) ? 128 * K * 2 : (MODE == 0 ? 128 * K : 128 * N);
  uint8_t* sa = smem;
  uint8_t* sb = smem + kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kABytes + kBBytes);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(slot, 256);
  // thread-written operands (the P^ / dS^^T paths of the fused kernels)
  if (MODE == 1 || MODE == 2) {
    const int r = threadIdx.x;
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(sa + sw_offset(r, c, 128)) =
          *reinterpret_cast<const uint4*>(a_host_layout + r * 128 + c * 16);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (MODE == 4 || MODE == 5) {  // A row r -> TMEM lane r, columns [128, 128 + row_bytes/4)
    const int r = threadIdx.x;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    constexpr int kRowWords = MODE == 4 ? 32 : K / 2;
    for (int c0 = 0; c0 < kRowWords; c0 += 32) {
      uint32_t w[32];
      for (int e = 0; e < 32; ++e) w[e] = reinterpret_cast<const uint32_t*>(a_host_layout)[r * kRowWords + c0 + e];
      tmem_st32(tmem + 128 + c0 + lane_off, w);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (threadIdx.x == 0) {
    mbar_expect_tx(bars, (MODE == 0 || MODE == 3 ? kABytes : 0) + kBBytes);
    if (MODE == 5) {
      for (int p = 0; p < K / 64; ++p) tma_load_2d(sb + p * 16384, &tmb, bars, p * 64, 0);
    }
    if (MODE == 0) {
      tma_load_2d(sa, &tma, bars, 0, 0);
      tma_load_2d(sb, &tmb, bars, 0, 0);
    } else if (MODE == 3) {
      for (int p = 0; p < K / 64; ++p) {
        tma_load_2d(sa + p * 16384, &tma, bars, p * 64, 0);
        tma_load_2d(sb + p * 16384, &tmb, bars, p * 64, 0);
      }
    } else if (MODE != 5) {
      tma_load_2d(sb, &tmb, bars, 0, 0);
    }
    mbar_wait(bars, 0);
    tc_fence_after();
    const uint32_t a = smem_u32(sa), b = smem_u32(sb);
    if (MODE == 0) {
      for (int kk = 0; kk < K / 32; ++kk)
        mma_i8(tmem, desc_kmajor(a, K, kk * 32), desc_kmajor(b, K, kk * 32), idesc_i8(128, 128, false, false), kk > 0);
    } else if (MODE == 1) {
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tmem, desc_kmajor(a, 128, kk * 32), desc_mnmajor(b, N, kk * 32), idesc_i8(128, N, false, true, kU8),
               kk > 0);
    } else if (MODE == 2) {
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tmem, desc_mnmajor(a, 128, kk * 32), desc_mnmajor(b, N, kk * 32), idesc_i8(128, N, true, true), kk > 0);
    } else if (MODE == 3) {
      for (int kk = 0; kk < K / 16; ++kk) {
        const uint32_t po = (kk / 4) * 16384, ko = (kk % 4) * 32;
        mma_bf16(tmem, desc_kmajor(a + po, 128, ko), desc_kmajor(b + po, 128, ko), idesc_bf16(128, 128, false, false),
                 kk > 0);
      }
    } else if (MODE == 4) {
      for (int kk = 0; kk < 4; ++kk)
        mma_i8_ts(tmem, tmem + 128 + kk * 8, desc_mnmajor(b, N, kk * 32), idesc_i8(128, N, false, true, kU8), kk > 0);
    } else {
      for (int kk = 0; kk < K / 16; ++kk) {
        const uint32_t po = (kk / 4) * 16384, ko = (kk % 4) * 32;
        mma_bf16_ts(tmem, tmem + 128 + kk * 8, desc_kmajor(b + po, 128, ko), idesc_bf16(128, 128, false, false), kk > 0);
      }
    }
    mma_commit(bars + 1);
  }
  __syncwarp();
  mbar_wait(bars + 1, 0);
  tc_fence_after();
  constexpr int kCols = (MODE == 0 || MODE == 3 || MODE == 5) ? 128 : N;
  const int r = threadIdx.x;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  uint32_t* o = reinterpret_cast<uint32_t*>(out) + (size_t)r * kCols;
  for (int c0 = 0; c0 < kCols; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + c0 + lane_off, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) o[c0 + e] = v[e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int MODE, int K, int N>
cudaError_t run(const CUtensorMap* tma, const CUtensorMap* tmb, const void* a, void* d, cudaStream_t s) {
  const int smem = 1024 + 2 * 128 * 256 + 64;
  auto kern = debug_umma_kernel<MODE, K, N>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<1, 128, smem, s>>>(*tma, *tmb, reinterpret_cast<const int8_t*>(a), d);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_debug_umma(int mode, int K, int N, const CUtensorMap* tma, const CUtensorMap* tmb,
                              const void* a, void* d, cudaStream_t s) {
  switch (mode) {
    case 0: return K == 128 ? run<0, 128, 128>(tma, tmb, a, d, s) : run<0, 64, 128>(tma, tmb, a, d, s);
    case 1: return N == 128 ? run<1, 128, 128>(tma, tmb, a, d, s) : run<1, 128, 64>(tma, tmb, a, d, s);
    case 2: return N == 128 ? run<2, 128, 128>(tma, tmb, a, d, s) : run<2, 128, 64>(tma, tmb, a, d, s);
    case 3: return K == 128 ? run<3, 128, 128>(tma, tmb, a, d, s) : run<3, 64, 128>(tma, tmb, a, d, s);
    case 4: return N == 128 ? run<4, 128, 128>(tma, tmb, a, d, s) : run<4, 128, 64>(tma, tmb, a, d, s);
    case 5: return K == 128 ? run<5, 128, 128>(tma, tmb, a, d, s) : run<5, 64, 128>(tma, tmb, a, d, s);
    case 6: return N == 128 ? run<6, 128, 128>(tma, tmb, a, d, s) : run<6, 128, 64>(tma, tmb, a, d, s);
    default: return N == 128 ? run<7, 128, 128>(tma, tmb, a, d, s) : run<7, 128, 64>(tma, tmb, a, d, s);
  }
}

}  // namespace sage
