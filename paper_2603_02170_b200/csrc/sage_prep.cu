// sage_prep.cu -- the HBM-bound passes around the fused kernels:
//   K0  smoothing statistics mu_K, mu_Q   (fixed-order fp64 sums, reading A17)
//   K1  per-block INT8 psi of Q(-mu_Q), K-mu_K, V  (Alg. 1 line 3)
//   Q-smoothing bias mu_Qi . K_sm^T       (reading A13)
//   K3  backward prep: delta, psi(dO), L*log2(e), zero dQ accumulator  (Alg. 2 lines 2, 6)
//   K5  dQ fp32 -> bf16
//   QK-norm: per-row rstd, the normalised bf16 Q/K computed on the fly inside K0 / K1 /
//       the bias kernel, and the RMSNorm backward (dX, dgamma) fused with the dQ finalisation
// Built without --use_fast_math; every FP32 op that decides a bit-exact INT8 value
// is an explicit round-to-nearest intrinsic (__fsub_rn, __fmul_rn, __fdiv_rn) so
// nvcc cannot contract it (reading A4).
#include <cuda_fp16.h>

#include <type_traits>

#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

constexpr int kVec = 8;  // bf16 elements per 16-byte vector
constexpr int nrm_smem_rows = 128;  // QK-norm partial sums of squares: [128 rows][column groups] doubles

// I/O element type (bf16, or fp16 with SAGE_FP16): conversions of packed pairs and single values.
template <typename T>
struct Io;
template <>
struct Io<__nv_bfloat16> {
  using T2 = __nv_bfloat162;
  static __device__ __forceinline__ float2 to2(T2 h) { return __bfloat1622float2(h); }
  static __device__ __forceinline__ T2 from2(float a, float b) { return __floats2bfloat162_rn(a, b); }
  static __device__ __forceinline__ float to1(__nv_bfloat16 x) { return __bfloat162float(x); }
  static __device__ __forceinline__ float round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
};
template <>
struct Io<__half> {
  using T2 = __half2;
  static __device__ __forceinline__ float2 to2(T2 h) { return __half22float2(h); }
  static __device__ __forceinline__ T2 from2(float a, float b) { return __floats2half2_rn(a, b); }
  static __device__ __forceinline__ float to1(__half x) { return __half2float(x); }
  static __device__ __forceinline__ float round(float x) { return __half2float(__float2half_rn(x)); }
};

template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const typename Io<T>::T2* h = reinterpret_cast<const typename Io<T>::T2*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 t = Io<T>::to2(h[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]) {
  unpack8<T>(*reinterpret_cast<const uint4*>(p), f);
}
template <typename T>
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  typename Io<T>::T2* h = reinterpret_cast<typename Io<T>::T2*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = Io<T>::from2(f[2 * e], f[2 * e + 1]);
  return u;
}

// q = RNE(fl32(x * inv)) for four values, packed as int8x4.  fl32(y + 1.5*2^23) holds RNE(y) in
// its low bits (|y| < 2^22), so the rounding is an FADD instead of an XU-pipe F2I; |y| <= 127(1+2^-23)
// because inv = fl32(127/amax), hence |RNE(y)| <= 127 and no clamp is needed (readings A1, A2, A4).
__device__ __forceinline__ uint32_t quant4(const float* x, float inv) {
  constexpr float kMagic = 12582912.0f;
  uint32_t b[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) b[e] = __float_as_uint(__fadd_rn(__fmul_rn(x[e], inv), kMagic));
  return __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
}

// QK-norm output (readings A24/A25): y = io(fl32(fl32(x * rstd) * gamma)), io = the I/O type (bf16, or
// fp16 with SAGE_FP16): the value an unfused RMSNorm module would hand to the attention; every later
// step sees exactly these values.
template <typename T>
__device__ __forceinline__ float qk_norm(float x, float r, float g) {
  return Io<T>::round(__fmul_rn(__fmul_rn(x, r), g));
}

// QK-norm row statistics of a 128-row chunk (reading A24): rstd = fl32(1 / sqrt(sum_c x^2 / D + eps)).
// Each of the 256 threads holds NR rows x 8 columns (row r0 + k*RS, column group g of G); it writes
// its partial sums of squares (double: bf16 squares and their sums are exact unless a row's squares
// span > 30 binades, so the order is immaterial) to shared memory, then one thread per row adds the
// G partials and takes the IEEE double sqrt and division once, rounding to fp32 once.  Result in
// rs_s[128] (and rstd_out[128] if non-null).  All 256 threads must call it.
template <typename T, int G, int D, int NR, int RS>
__device__ __forceinline__ void chunk_rstd(const uint4 (&raw)[NR], int g, int r0, double* ssq, float* rs_s, float eps,
                                           float* rstd_out) {
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const typename Io<T>::T2* h = reinterpret_cast<const typename Io<T>::T2*>(&raw[k]);
    double ss = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 t = Io<T>::to2(h[e]);
      ss = fma((double)t.x, (double)t.x, ss);
      ss = fma((double)t.y, (double)t.y, ss);
    }
    ssq[(r0 + k * RS) * G + g] = ss;
  }
  __syncthreads();
  if (threadIdx.x < kBlk) {
    double ss = 0.0;
#pragma unroll
    for (int j = 0; j < G; ++j) ss += ssq[threadIdx.x * G + j];
    const float rs = __double2float_rn(1.0 / sqrt(ss / (double)D + (double)eps));
    rs_s[threadIdx.x] = rs;
    if (rstd_out) rstd_out[threadIdx.x] = rs;
  }
  __syncthreads();
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------- K0: column sums
// part[bh][t][c] = sum_{r=0..127} x[bh][128t + r][c] in double (reading A17).  One CTA per
// 128-row chunk: thread (g, q) sums rows q, q+R, ... of column group g (8 columns, 16-byte
// loads), then the R partials are combined in fixed order q = 0..R-1.  Sums of bf16 values in
// double are exact unless a column spans > 53-8-log2(N) binades, so the order cannot change the
// result for any realistic input; it is fixed anyway.
// RAG (every kernel below): N is not a multiple of 128 (reading A33).  The short-block checks compile
// away for RAG = false, so the common case keeps its unconditional load batches.
template <typename T, int D, bool QKN, bool RAG>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ x, double* __restrict__ part,
                                                     NormIn nrm, IoLayout io, int nT, int N) {
  constexpr int kGroups = D / kVec;        // 8 (d=64) or 16 (d=128)
  constexpr int kR = 256 / kGroups;        // 32 or 16 row phases
  __shared__ double red[kR][D];
  const long long chunk = blockIdx.x;      // bh * T + t
  const int g = threadIdx.x % kGroups, q = threadIdx.x / kGroups;
  const T* p = x + io.row(chunk / nT, (chunk % nT) * kBlk) + g * kVec;
  const int nv = RAG ? min(kBlk, N - (int)(chunk % nT) * kBlk) : kBlk;  // rows this chunk holds (A33)
  double acc[kVec];
  float gam[kVec];
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    acc[e] = 0.0;
    gam[e] = QKN ? nrm.gamma[g * kVec + e] : 1.f;
  }
  constexpr int kRows = kBlk / kR;  // rows per thread: all loads issued before any arithmetic
  uint4 raw[kRows];
#pragma unroll
  for (int k = 0; k < kRows; ++k)
    raw[k] = q + k * kR < nv ? *reinterpret_cast<const uint4*>(p + (q + k * kR) * io.sn) : make_uint4(0, 0, 0, 0);
  __shared__ double ssq[QKN ? nrm_smem_rows * kGroups : 1];
  __shared__ float rs_s[QKN ? kBlk : 1];
  if constexpr (QKN) chunk_rstd<T, kGroups, D, kRows, kR>(raw, g, q, ssq, rs_s, nrm.eps, nullptr);
#pragma unroll
  for (int k = 0; k < kRows; ++k) {
    float f[kVec];
    unpack8<T>(raw[k], f);
    if constexpr (QKN) {  // QK-norm (A24/A25)
      const float rs = rs_s[q + k * kR];
#pragma unroll
      for (int e = 0; e < kVec; ++e) f[e] = qk_norm<T>(f[e], rs, gam[e]);
    }
#pragma unroll
    for (int e = 0; e < kVec; ++e) acc[e] += (double)f[e];
  }
#pragma unroll
  for (int e = 0; e < kVec; ++e) red[q][g * kVec + e] = acc[e];
  __syncthreads();
  if (threadIdx.x < D) {
    double s = 0.0;
#pragma unroll 4
    for (int k = 0; k < kR; ++k) s += red[k][threadIdx.x];
    part[chunk * D + threadIdx.x] = s;
  }
}

// mu[bh][c] = fl32((sum over chunks, sequential in t) / N)
__global__ void colmean_kernel(const double* __restrict__ part, float* __restrict__ mu, int N, int d, int BH) {
  int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= BH * d) return;
  int bh = item / d, c = item % d, T = num_blocks(N);
  const double* p = part + (size_t)bh * T * d + c;
  double total = 0.0;
  // sequential in t (A17); the loads of 8 chunks are issued ahead of their adds
  int t = 0;
  for (; t + 8 <= T; t += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = p[(size_t)(t + u) * d];
#pragma unroll
    for (int u = 0; u < 8; ++u) total += x[u];
  }
  for (; t < T; ++t) total += p[(size_t)t * d];
  mu[item] = __double2float_rn(total / (double)N);
}

// mu_Q[bh][t][c] = fl32(part / rows of block t)  (the last block of a ragged N is short, A33)
__global__ void blockmean_kernel(const double* __restrict__ part, float* __restrict__ mu_q, size_t n, int d, int N) {
  size_t item = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n) return;
  const int t = (int)((item / d) % num_blocks(N));
  mu_q[item] = __double2float_rn(part[item] / (double)min(kBlk, N - t * kBlk));
}

// ---------------------------------------------------------------- K1: psi
// One CTA quantises one 128 x d block: x_sm = fl32(x - mu); amax; scale = fl32(amax/127);
// inv = fl32(127/amax) (0 for an all-zero block, A3); q = clamp(RNE(fl32(x_sm*inv)), +-127).
template <typename TI, int D, bool QKN, bool RAG>
__global__ void __launch_bounds__(256, 3) quantize_kernel(QuantJobs jobs, int T, IoLayout io, int N) {
  // blockIdx.y selects the tensor (Q, K, V): one launch for all three psi passes
  const QuantJob& job = jobs.j[blockIdx.y];
  const TI* __restrict__ x = static_cast<const TI*>(job.x);
  const float* __restrict__ mu = job.mu;
  const int mu_mode = job.mu_mode;
  int8_t* __restrict__ xq = job.xq;
  float* __restrict__ scale = job.scale;
  constexpr int kPerThread = kBlk * D / 256;      // 64 (D=128) or 32 (D=64)
  constexpr int kIters = kPerThread / kVec;       // 8 or 4
  constexpr int kGroups = D / kVec;               // 16 or 8 column groups per row
  constexpr int kRowsPerPass = 256 / kGroups;     // 16 or 32
  __shared__ float red[8];
  const long long blk = blockIdx.x;               // bh * T + t
  const int bh = (int)(blk / T), t = (int)(blk % T);
  const int g = threadIdx.x % kGroups, r0 = threadIdx.x / kGroups;
  const TI* xb = x + io.row(bh, (long long)t * kBlk);
  const int nv = RAG ? min(kBlk, N - t * kBlk) : kBlk;  // rows this block holds (A33); the rest quantise to 0
  float m[kVec];
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    int c = g * kVec + e;
    m[e] = mu_mode == 0 ? 0.f : (mu_mode == 1 ? mu[(size_t)bh * D + c] : mu[((size_t)bh * T + t) * D + c]);
  }
  // pass 1: every row's 16-byte vector is loaded before any arithmetic (kIters loads in flight);
  // the (QK-normed) bf16 values stay packed in registers for pass 2, which recomputes x - mu
  uint4 raw[kIters];
#pragma unroll
  for (int it = 0; it < kIters; ++it)
    raw[it] = r0 + it * kRowsPerPass < nv ? *reinterpret_cast<const uint4*>(xb + (r0 + it * kRowsPerPass) * io.sn + g * kVec)
                                          : make_uint4(0, 0, 0, 0);
  // QK-norm row statistics (A24), kept for the backward (QKN launches: every job with gamma)
  __shared__ double ssq[QKN ? nrm_smem_rows * kGroups : 1];
  __shared__ float rs_s[QKN ? kBlk : 1];
  if constexpr (QKN) {
    if (job.gamma)
      chunk_rstd<TI, kGroups, D, kIters, kRowsPerPass>(raw, g, r0, ssq, rs_s, job.eps, job.rstd + blk * kBlk);
  }
  float amax = 0.f;
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    float v[kVec];
    unpack8<TI>(raw[it], v);
    if (QKN && job.gamma) {  // QK-norm (A25) before the smoothing subtraction
      float gam[kVec];
#pragma unroll
      for (int e = 0; e < kVec; ++e) gam[e] = job.gamma[g * kVec + e];
      const float rs = rs_s[r0 + it * kRowsPerPass];
#pragma unroll
      for (int e = 0; e < kVec; ++e) v[e] = qk_norm<TI>(v[e], rs, gam[e]);
      raw[it] = pack8<TI>(v);  // exact: qk_norm values are I/O-type values
    }
    if (r0 + it * kRowsPerPass < nv) {
#pragma unroll
      for (int e = 0; e < kVec; ++e) amax = fmaxf(amax, fabsf(__fsub_rn(v[e], m[e])));
    }
  }
  amax = warp_max(amax);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) amax = fmaxf(amax, red[w]);
  // INT8: scale = fl32(amax/127), q = RNE(fl32(x * fl32(127/amax))); E4M3 (SAGE_PV_FP8, V only):
  // scale = fl32(amax/448), q = e4m3_rne(fl32(x * fl32(448/amax))), saturating
  const float qmax = job.fp8 ? 448.f : 127.f;
  const float sc = __fdiv_rn(amax, qmax);
  const float inv = amax > 0.f ? __fdiv_rn(qmax, amax) : 0.f;
  if (threadIdx.x == 0) scale[blk] = sc;
  int8_t* qb = xq + blk * kBlk * D;
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    int r = r0 + it * kRowsPerPass;
    float v[kVec];
    unpack8<TI>(raw[it], v);
#pragma unroll
    for (int e = 0; e < kVec; ++e) v[e] = __fsub_rn(v[e], m[e]);
    uint32_t w[2];
    if (r >= nv) {
      w[0] = w[1] = 0u;
    } else if (job.fp8) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* x = v + 4 * h;
        w[h] = e4m3x2(__fmul_rn(x[0], inv), __fmul_rn(x[1], inv)) |
               (e4m3x2(__fmul_rn(x[2], inv), __fmul_rn(x[3], inv)) << 16);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) w[h] = quant4(v + 4 * h, inv);
    }
    *reinterpret_cast<uint2*>(qb + (size_t)r * D + g * kVec) = make_uint2(w[0], w[1]);
  }
}

// ---------------------------------------------------------------- Q-smoothing bias
// bias[bh][i][n] = sum_c mu_Q[bh][i][c] * fl32(K[n][c] - mu_K[c]) in fp32, four partial sums over
// c mod 4 (reading A13; fp32, so compared to the fp64 oracle within 1e-5 relative).  K2 and K4 read
// the same stored bias, so the forward and the backward see identical logits.
// CTA = (bh, 128-key block, group of kBiasI query blocks); thread = key n holds its smoothed K row in
// registers, the group's mu_Q rows are broadcast from shared memory.
constexpr int kBiasI = 32;
template <typename TI, int D, bool RAG>
#ifndef SAGE_BIAS_MINB
#define SAGE_BIAS_MINB 3  // 3 CTAs per SM (168 registers, 24 B prologue spill at D=128): C3 610.7 -> 612.8 TOPS
#endif
__global__ void __launch_bounds__(128, SAGE_BIAS_MINB) qsmooth_bias_kernel(const TI* __restrict__ k,
                                                           const float* __restrict__ mu_k,
                                                           const float* __restrict__ mu_q, float* __restrict__ bias,
                                                           int N, NormIn nrm, IoLayout io) {
  __shared__ float4 mq[kBiasI][D / 4];
  const int T = num_blocks(N), Np = T * kBlk;
  const long long blk = blockIdx.x;    // bh * T + jn
  const int bh = (int)(blk / T), jn = (int)(blk % T);
  const int i0 = blockIdx.y * kBiasI, ni = min(kBiasI, T - i0);
  const int n = threadIdx.x;
  const bool valid = !RAG || jn * kBlk + n < N;  // a key the short last block lacks gets bias 0 (A33)
  for (int e = threadIdx.x; e < ni * (D / 4); e += blockDim.x)
    mq[e / (D / 4)][e % (D / 4)] = reinterpret_cast<const float4*>(mu_q + ((size_t)bh * T + i0) * D)[e];
  float ks[D];
  const TI* krow = k + io.row(bh, (long long)jn * kBlk + n);
  const float* mk = mu_k + (size_t)bh * D;
  const float rs = nrm.gamma ? nrm.rstd[blk * kBlk + n] : 1.f;  // written by K1's K job
  uint4 raw[D / kVec];  // the whole K row in flight before any use (the loads' latency dominates)
#pragma unroll
  for (int c8 = 0; c8 < D / kVec; ++c8)
    raw[c8] = valid ? *reinterpret_cast<const uint4*>(krow + c8 * kVec) : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int c = 0; c < D; c += kVec) {
    float f[kVec];
    unpack8<TI>(raw[c / kVec], f);
    if (nrm.gamma) {
#pragma unroll
      for (int e = 0; e < kVec; ++e) f[e] = qk_norm<TI>(f[e], rs, nrm.gamma[c + e]);
    }
    const float4 m0 = *reinterpret_cast<const float4*>(mk + c), m1 = *reinterpret_cast<const float4*>(mk + c + 4);
    const float mm[kVec] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int e = 0; e < kVec; ++e) ks[c + e] = valid ? __fsub_rn(f[e], mm[e]) : 0.f;
  }
  __syncthreads();
  float* out = bias + ((size_t)bh * T + i0) * Np + (size_t)jn * kBlk + n;
  // FFMA2 over column pairs (c, c+1): mu_Q's float4 and the K row are already register pairs, so no
  // repacking; two query blocks per pass and two accumulator pairs each (8 partial sums) for ILP
#pragma unroll 1
  for (int ii = 0; ii < ni; ii += 2) {
    const int i1 = ii + 1 < ni ? ii + 1 : ii;
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
#pragma unroll
    for (int c4 = 0; c4 < D / 4; ++c4) {
      const float4 m = mq[ii][c4], m1 = mq[i1][c4];
      const float2 k01 = make_float2(ks[4 * c4], ks[4 * c4 + 1]), k23 = make_float2(ks[4 * c4 + 2], ks[4 * c4 + 3]);
      a0 = ffma2(make_float2(m.x, m.y), k01, a0);
      a1 = ffma2(make_float2(m.z, m.w), k23, a1);
      b0 = ffma2(make_float2(m1.x, m1.y), k01, b0);
      b1 = ffma2(make_float2(m1.z, m1.w), k23, b1);
    }
    const float2 sa = fadd2(a0, a1), sb = fadd2(b0, b1);
    out[(size_t)ii * Np] = sa.x + sa.y;
    if (ii + 1 < ni) out[(size_t)(ii + 1) * Np] = sb.x + sb.y;
  }
}

// ---------------------------------------------------------------- K3: backward prep
// delta[r] = sum_c dO[r][c] * O[r][c] (Alg. 2 line 2) from the O the forward stored (A15): every product
// of two I/O-type values is exact in fp64 (and of an I/O value with an fp32 O, SAGE_FP32_OUT), and the
// fp64 sum of a row's d products is exact unless they span > 37 binades, so delta = fl32(exact sum):
// the same bits as the oracle's fp64 row sum rounded to fp32.
template <typename TO>
__device__ __forceinline__ void load_o8(const TO* p, float (&f)[8]) {
  if constexpr (std::is_same<TO, float>::value) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    load8<TO>(p, f);
  }
}

template <typename T, typename TO, int D, bool RAG>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const TO* __restrict__ o, const T* __restrict__ dO,
                                                       const float* __restrict__ lse, float* __restrict__ delta,
                                                       float* __restrict__ l2, int8_t* __restrict__ do_q,
                                                       float* __restrict__ do_scale, float* __restrict__ dq_acc,
                                                       unsigned* __restrict__ dq_flags, IoLayout io, int nT, int N) {
  constexpr int kGroups = D / kVec;            // threads per row
  constexpr int kRowsPerPass = 256 / kGroups;
  constexpr int kIters = kBlk / kRowsPerPass;
  __shared__ float red[8];
  const long long blk = blockIdx.x;
  const int g = threadIdx.x % kGroups, r0 = threadIdx.x / kGroups;
  const size_t base = (size_t)blk * kBlk * D;                      // the contiguous buffers (dO^, dQ accumulator)
  const long long iob = io.row(blk / nT, (blk % nT) * (long long)kBlk);  // O and dO in the I/O layout
  const int nv = RAG ? min(kBlk, N - (int)(blk % nT) * kBlk) : kBlk;  // rows this block holds (A33)
  float v[kIters][kVec];
  float amax = 0.f;
  // dO rows in flight before any arithmetic (kIters 16-byte loads per thread); O's alongside
  uint4 rdo[kIters];
#pragma unroll
  for (int it = 0; it < kIters; ++it)
    rdo[it] = r0 + it * kRowsPerPass < nv ? *reinterpret_cast<const uint4*>(dO + iob + (r0 + it * kRowsPerPass) * io.sn + g * kVec)
                                          : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int r = r0 + it * kRowsPerPass;
    const size_t off = base + (size_t)r * D + g * kVec;
    float fo[kVec];
    unpack8<T>(rdo[it], v[it]);
    if (r < nv) {
      load_o8<TO>(o + iob + r * io.sn + g * kVec, fo);
    } else {
#pragma unroll
      for (int e = 0; e < kVec; ++e) fo[e] = 0.f;
    }
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < kVec; ++e) {
      dot = fma((double)v[it][e], (double)fo[e], dot);
      amax = fmaxf(amax, fabsf(v[it][e]));
    }
#pragma unroll
    for (int s = kGroups / 2; s; s >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, s);
    if (g == 0) {
      // padded rows (A33): delta 0 and L = +inf, so K4's P = 2^{t - L} and dS vanish on them
      const size_t row = (size_t)blk * kBlk + r;
      delta[row] = __double2float_rn(dot);
      l2[row] = r < nv ? lse[(blk / nT) * (long long)N + (blk % nT) * kBlk + r] * 1.4426950408889634f : INFINITY;
    }
    *reinterpret_cast<float4*>(dq_acc + off) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(dq_acc + off + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  amax = warp_max(amax);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) amax = fmaxf(amax, red[w]);
  const float sc = __fdiv_rn(amax, 127.f);
  const float inv = amax > 0.f ? __fdiv_rn(127.f, amax) : 0.f;
  if (threadIdx.x == 0) do_scale[blk] = sc;
  if (dq_flags && threadIdx.x < 4) dq_flags[blk * 4 + threadIdx.x] = 0u;  // SAGE_DETERMINISTIC flags
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int r = r0 + it * kRowsPerPass;
    uint32_t w[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) w[h] = quant4(v[it] + 4 * h, inv);
    *reinterpret_cast<uint2*>(do_q + base + (size_t)r * D + g * kVec) = make_uint2(w[0], w[1]);
  }
}

__global__ void fill_kernel(float* __restrict__ x, size_t n, float v) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// 8 elements per thread, from the contiguous accumulator to dQ in the I/O layout (the I/O type, or fp32)
template <typename T, bool F32, bool RAG>
__global__ void dq_finalize_kernel(const float* __restrict__ acc, void* __restrict__ dq, size_t n8, int N, int d,
                                   IoLayout io) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const size_t e = i * 8, row = e / d;
  // the accumulator has Np rows per head (A33)
  const size_t arow = RAG ? (row / N) * (size_t)padded_len(N) + row % N : row;
  const float4* ap = reinterpret_cast<const float4*>(acc + arow * d + e % d);
  const float4 a = ap[0], b = ap[1];
  const long long off = io.row((long long)(row / N), (long long)(row % N)) + (long long)(e % d);
  if constexpr (F32) {
    reinterpret_cast<float4*>(static_cast<float*>(dq) + off)[0] = a;
    reinterpret_cast<float4*>(static_cast<float*>(dq) + off)[1] = b;
  } else {
    const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    *reinterpret_cast<uint4*>(static_cast<T*>(dq) + off) = pack8<T>(f);
  }
}

// ---------------------------------------------------------------- QK-norm backward
// RMSNorm backward (reading A26) for one 128-row block per CTA, 16 rows per warp, D/32 consecutive
// columns per lane (vector loads), the 16 rows loaded before any reduction so their loads overlap:
// dy = bf16(attention gradient) (from the fp32 dQ accumulator, or the bf16 dK in place),
// g = dy o gamma, xh = x rstd, dx = rstd (g - xh mean(g o xh)) -> bf16;  gpart[block][c] = sum
// over the block's rows of dy o xh (fixed order: rows within a warp, then warps 0..7).
template <typename T, int D>
__global__ void __launch_bounds__(256) norm_bwd_kernel(const float* __restrict__ dy32, const T* dy16,
                                                       const T* __restrict__ x,
                                                       const float* __restrict__ rstd, const float* __restrict__ gamma,
                                                       T* dx, float* __restrict__ gpart, IoLayout io, int N) {
  constexpr int kPer = D / 32;  // 4 or 2
  constexpr int kRows = 16;
  __shared__ float red[8][D];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t blk = blockIdx.x;
  const size_t row0 = blk * kBlk + warp * kRows;  // in the padded row space (Np rows per head, A33)
  const int Np = padded_len(N);
  float gam[kPer], gacc[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    gam[e] = gamma[lane * kPer + e];
    gacc[e] = 0.f;
  }
  float dy[kRows][kPer], xv[kRows][kPer], rs[kRows];
#pragma unroll
  for (int rr = 0; rr < kRows; ++rr) {
    const size_t off = (row0 + rr) * D + lane * kPer;  // the contiguous fp32 dQ accumulator
    const long long ioff = io.row((long long)((row0 + rr) / Np), (long long)((row0 + rr) % Np)) + lane * kPer;
    rs[rr] = rstd[row0 + rr];
    if ((int)((row0 + rr) % Np) >= N) {  // a row the short last block lacks: no contribution
#pragma unroll
      for (int e = 0; e < kPer; ++e) xv[rr][e] = dy[rr][e] = 0.f;
      continue;
    }
    if constexpr (kPer == 4) {
      const uint2 xu = *reinterpret_cast<const uint2*>(x + ioff);
      const float2 x0 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(&xu.x));
      const float2 x1 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(&xu.y));
      xv[rr][0] = x0.x; xv[rr][1] = x0.y; xv[rr][2] = x1.x; xv[rr][3] = x1.y;
      if (dy32) {
        const float4 f = *reinterpret_cast<const float4*>(dy32 + off);
        dy[rr][0] = f.x; dy[rr][1] = f.y; dy[rr][2] = f.z; dy[rr][3] = f.w;
      } else {
        const uint2 du = *reinterpret_cast<const uint2*>(dy16 + ioff);
        const float2 d0 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(&du.x));
        const float2 d1 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(&du.y));
        dy[rr][0] = d0.x; dy[rr][1] = d0.y; dy[rr][2] = d1.x; dy[rr][3] = d1.y;
      }
    } else {
      const float2 x0 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(x + ioff));
      xv[rr][0] = x0.x; xv[rr][1] = x0.y;
      if (dy32) {
        const float2 f = *reinterpret_cast<const float2*>(dy32 + off);
        dy[rr][0] = f.x; dy[rr][1] = f.y;
      } else {
        const float2 d0 = Io<T>::to2(*reinterpret_cast<const typename Io<T>::T2*>(dy16 + ioff));
        dy[rr][0] = d0.x; dy[rr][1] = d0.y;
      }
    }
  }
  float dot[kRows];
#pragma unroll
  for (int rr = 0; rr < kRows; ++rr) {
    dot[rr] = 0.f;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      if (dy32) dy[rr][e] = Io<T>::round(dy[rr][e]);  // A26
      xv[rr][e] *= rs[rr];                                                    // xh
      gacc[e] = fmaf(dy[rr][e], xv[rr][e], gacc[e]);
      dy[rr][e] *= gam[e];                                                    // g
      dot[rr] = fmaf(dy[rr][e], xv[rr][e], dot[rr]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) dot[rr] += __shfl_xor_sync(0xffffffffu, dot[rr], o);
  }
#pragma unroll
  for (int rr = 0; rr < kRows; ++rr) {
    if ((int)((row0 + rr) % Np) >= N) continue;
    const long long off = io.row((long long)((row0 + rr) / Np), (long long)((row0 + rr) % Np)) + lane * kPer;
    const float mean = dot[rr] * (1.f / D);
    typename Io<T>::T2 h[kPer / 2];
#pragma unroll
    for (int e = 0; e < kPer; e += 2)
      h[e / 2] = Io<T>::from2(rs[rr] * fmaf(-xv[rr][e], mean, dy[rr][e]),
                                       rs[rr] * fmaf(-xv[rr][e + 1], mean, dy[rr][e + 1]));
    if constexpr (kPer == 4)
      *reinterpret_cast<uint2*>(dx + off) = *reinterpret_cast<const uint2*>(h);
    else
      *reinterpret_cast<typename Io<T>::T2*>(dx + off) = h[0];
  }
#pragma unroll
  for (int e = 0; e < kPer; ++e) red[warp][lane * kPer + e] = gacc[e];
  __syncthreads();
  if (threadIdx.x < D) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    gpart[blk * D + threadIdx.x] = s;
  }
}

// dgamma[c] = sum over blocks of gpart[block][c], fixed order, coalesced: stage 1 (one CTA per 64
// consecutive blocks, thread = column) sums in block order into part2 (double); stage 2 sums
// part2 in order.
constexpr int kGBlk = 64;
__global__ void dgamma_stage1_kernel(const float* __restrict__ gpart, double* __restrict__ part2, int nblk, int D) {
  const int c = threadIdx.x;
  const int b0 = blockIdx.x * kGBlk, b1 = min(nblk, b0 + kGBlk);
  double s = 0.0;
  for (int b = b0; b < b1; ++b) s += (double)gpart[(size_t)b * D + c];
  part2[(size_t)blockIdx.x * D + c] = s;
}
__global__ void dgamma_stage2_kernel(const double* __restrict__ part2, float* __restrict__ dgamma, int n2, int D) {
  const int c = threadIdx.x;
  double s = 0.0;
  for (int b = 0; b < n2; ++b) s += part2[(size_t)b * D + c];
  dgamma[c] = __double2float_rn(s);
}

}  // namespace

// I/O type dispatch: every launcher takes void pointers and the SAGE_FP16 choice
#define SAGE_IO_DISPATCH(fp16, ...)        \
  do {                                     \
    if (fp16) {                            \
      using IoT = __half;                  \
      __VA_ARGS__;                         \
    } else {                               \
      using IoT = __nv_bfloat16;           \
      __VA_ARGS__;                         \
    }                                      \
  } while (0)

#define SAGE_RAG_DISPATCH(N, ...)          \
  do {                                     \
    if ((N) % kBlk) {                      \
      constexpr bool kRag = true;          \
      __VA_ARGS__;                         \
    } else {                               \
      constexpr bool kRag = false;         \
      __VA_ARGS__;                         \
    }                                      \
  } while (0)

cudaError_t launch_colsum(const void* x, double* part, int BH, int N, int d, cudaStream_t s, NormIn nrm, bool fp16,
                          IoLayout io) {
  const int nT = num_blocks(N);
  const unsigned grid = (unsigned)(BH * nT);
  SAGE_IO_DISPATCH(fp16, SAGE_RAG_DISPATCH(N, {
    const IoT* xt = static_cast<const IoT*>(x);
    if (nrm.gamma) {
      if (d == 128)
        colsum_kernel<IoT, 128, true, kRag><<<grid, 256, 0, s>>>(xt, part, nrm, io, nT, N);
      else
        colsum_kernel<IoT, 64, true, kRag><<<grid, 256, 0, s>>>(xt, part, nrm, io, nT, N);
    } else {
      if (d == 128)
        colsum_kernel<IoT, 128, false, kRag><<<grid, 256, 0, s>>>(xt, part, nrm, io, nT, N);
      else
        colsum_kernel<IoT, 64, false, kRag><<<grid, 256, 0, s>>>(xt, part, nrm, io, nT, N);
    }
  }));
  return cudaGetLastError();
}

cudaError_t launch_norm_bwd(const float* dy32, const void* dy16, const void* x, const float* rstd, const float* gamma,
                            void* dx, float* gpart, float* dgamma, size_t rows, int d, cudaStream_t s, bool fp16,
                            IoLayout io, int N) {
  const unsigned nblk = (unsigned)(rows / kBlk);
  SAGE_IO_DISPATCH(fp16, {
    const IoT* dyt = static_cast<const IoT*>(dy16);
    const IoT* xt = static_cast<const IoT*>(x);
    IoT* dxt = static_cast<IoT*>(dx);
    if (d == 128)
      norm_bwd_kernel<IoT, 128><<<nblk, 256, 0, s>>>(dy32, dyt, xt, rstd, gamma, dxt, gpart, io, N);
    else
      norm_bwd_kernel<IoT, 64><<<nblk, 256, 0, s>>>(dy32, dyt, xt, rstd, gamma, dxt, gpart, io, N);
  });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the stage-1 sums (double) follow the nblk x d block partials in the same workspace slot
  const unsigned n2 = (nblk + kGBlk - 1) / kGBlk;
  double* part2 = reinterpret_cast<double*>(gpart + (size_t)nblk * d + ((size_t)nblk * d & 1));
  dgamma_stage1_kernel<<<n2, d, 0, s>>>(gpart, part2, (int)nblk, d);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  dgamma_stage2_kernel<<<1, d, 0, s>>>(part2, dgamma, (int)n2, d);
  return cudaGetLastError();
}

cudaError_t launch_colmean(const double* part, float* mu, int BH, int N, int d, cudaStream_t s) {
  int n = BH * d;
  colmean_kernel<<<(n + 127) / 128, 128, 0, s>>>(part, mu, N, d, BH);
  return cudaGetLastError();
}

cudaError_t launch_blockmean(const double* part, float* mu_q, int BH, int N, int d, cudaStream_t s) {
  size_t n = (size_t)BH * num_blocks(N) * d;
  blockmean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(part, mu_q, n, d, N);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const QuantJobs& jobs, int njobs, int BH, int N, int d, cudaStream_t s, bool fp16,
                            IoLayout io) {
  int T = num_blocks(N);
  dim3 grid((unsigned)(BH * T), (unsigned)njobs);
  bool qkn = false;
  for (int i = 0; i < njobs; ++i) qkn = qkn || jobs.j[i].gamma;
  SAGE_IO_DISPATCH(fp16, SAGE_RAG_DISPATCH(N, {
    if (qkn) {
      if (d == 128)
        quantize_kernel<IoT, 128, true, kRag><<<grid, 256, 0, s>>>(jobs, T, io, N);
      else
        quantize_kernel<IoT, 64, true, kRag><<<grid, 256, 0, s>>>(jobs, T, io, N);
    } else {
      if (d == 128)
        quantize_kernel<IoT, 128, false, kRag><<<grid, 256, 0, s>>>(jobs, T, io, N);
      else
        quantize_kernel<IoT, 64, false, kRag><<<grid, 256, 0, s>>>(jobs, T, io, N);
    }
  }));
  return cudaGetLastError();
}

cudaError_t launch_qsmooth_bias(const void* k, const float* mu_k, const float* mu_q, float* bias, int BH, int N, int d,
                                cudaStream_t s, NormIn nrm, bool fp16, IoLayout io) {
  const int T = num_blocks(N);
  dim3 grid((unsigned)(BH * T), (unsigned)((T + kBiasI - 1) / kBiasI));
  SAGE_IO_DISPATCH(fp16, SAGE_RAG_DISPATCH(N, {
    const IoT* kt = static_cast<const IoT*>(k);
    if (d == 128)
      qsmooth_bias_kernel<IoT, 128, kRag><<<grid, 128, 0, s>>>(kt, mu_k, mu_q, bias, N, nrm, io);
    else
      qsmooth_bias_kernel<IoT, 64, kRag><<<grid, 128, 0, s>>>(kt, mu_k, mu_q, bias, N, nrm, io);
  }));
  return cudaGetLastError();
}

cudaError_t launch_bwd_prep(const void* o, const void* dO, const float* lse, float* delta, float* l2, int8_t* do_q,
                            float* do_scale, float* dq_acc, int BH, int N, int d, cudaStream_t s, unsigned* dq_flags,
                            bool fp16, bool o_f32, IoLayout io) {
  const int nT = num_blocks(N);
  unsigned grid = (unsigned)(BH * nT);
  SAGE_IO_DISPATCH(fp16, SAGE_RAG_DISPATCH(N, {
    const IoT* dot = static_cast<const IoT*>(dO);
    if (o_f32) {
      const float* ot = static_cast<const float*>(o);
      if (d == 128)
        bwd_prep_kernel<IoT, float, 128, kRag><<<grid, 256, 0, s>>>(ot, dot, lse, delta, l2, do_q, do_scale, dq_acc, dq_flags, io, nT, N);
      else
        bwd_prep_kernel<IoT, float, 64, kRag><<<grid, 256, 0, s>>>(ot, dot, lse, delta, l2, do_q, do_scale, dq_acc, dq_flags, io, nT, N);
    } else {
      const IoT* ot = static_cast<const IoT*>(o);
      if (d == 128)
        bwd_prep_kernel<IoT, IoT, 128, kRag><<<grid, 256, 0, s>>>(ot, dot, lse, delta, l2, do_q, do_scale, dq_acc, dq_flags, io, nT, N);
      else
        bwd_prep_kernel<IoT, IoT, 64, kRag><<<grid, 256, 0, s>>>(ot, dot, lse, delta, l2, do_q, do_scale, dq_acc, dq_flags, io, nT, N);
    }
  }));
  return cudaGetLastError();
}

cudaError_t launch_fill(float* x, size_t n, float v, cudaStream_t s) {
  fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, v);
  return cudaGetLastError();
}

cudaError_t launch_dq_finalize(const float* dq_acc, void* dq, int BH, int N, int d, cudaStream_t s, bool fp16,
                               IoLayout io, bool f32) {
  const size_t n8 = (size_t)BH * N * d / 8;
  const unsigned grid = (unsigned)((n8 + 255) / 256);
  if (f32) {
    SAGE_RAG_DISPATCH(N, dq_finalize_kernel<float, true, kRag><<<grid, 256, 0, s>>>(dq_acc, dq, n8, N, d, io));
    return cudaGetLastError();
  }
  SAGE_IO_DISPATCH(fp16, SAGE_RAG_DISPATCH(N, dq_finalize_kernel<IoT, false, kRag><<<grid, 256, 0, s>>>(dq_acc, dq, n8, N, d, io)));
  return cudaGetLastError();
}

}  // namespace sage
