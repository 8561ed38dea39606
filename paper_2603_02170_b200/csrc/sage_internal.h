// sage_internal.h -- host-side declarations shared by the libsage translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sage {

constexpr int kBlk = 128;  // B_q = B_kv = 128 (reading A5): tcgen05 M = 128 tiles
constexpr int kMaxSeqLen = 32768;  // per-head scale rows are staged in shared memory (T <= 256)
// N need not be a multiple of 128 (reading A33): a head has T = ceil(N / 128) blocks, the last one short.
// The library's own per-row buffers (int8 tiles, L, delta, the Q-smoothing bias, the fp32 dQ accumulator,
// QK-norm rstd) give every head Np = 128 T rows; rows N .. Np-1 hold zeros (or masked values).
__host__ __device__ __forceinline__ int num_blocks(int N) { return (N + kBlk - 1) / kBlk; }
__host__ __device__ __forceinline__ int padded_len(int N) { return num_blocks(N) * kBlk; }

// Layout of the I/O tensors (Q, K, V, O, dO, dQ, dK, dV; X_q, X_k, dX_q, dX_k with QK-norm): element
// strides of the batch, head and token dimensions (the head dimension d is contiguous).  Row (bh, n) of
// head bh = b * H + h starts at element b * sb + h * sh + n * sn.  Contiguous [B, H, N, d]: sb = H N d,
// sh = N d, sn = d.  The library's own buffers (int8 tiles, scales, the fp32 dQ accumulator) stay contiguous.
struct IoLayout {
  long long sb, sh, sn;
  int H;
  __host__ __device__ __forceinline__ long long row(long long bh, long long n) const {
    return (bh / H) * sb + (bh % H) * sh + n * sn;
  }
  __host__ __device__ __forceinline__ bool contiguous(int N, int d) const {
    return sn == d && sh == (long long)N * d && sb == (long long)H * N * d;
  }
};

// ---- memory-bound passes (sage_prep.cu) ----
// QK-norm input transform (readings A24/A25): when gamma is non-null, every kernel that
// reads Q or K sees y = bf16(fl32(fl32(x * rstd[row]) * gamma[c])) instead of x, with
// rstd[row] = fl32(1 / sqrt(mean(x^2) + eps)) computed from the row as it is loaded (K0, K1; K1
// stores it for the backward) or read back (the Q-smoothing bias kernel, after K1).
struct NormIn {
  float* rstd;         // [BH*Np]
  const float* gamma;  // [d] or null (no QK-norm)
  float eps;
};
// RMSNorm backward (reading A26): dx (bf16) from dy (fp32 dy32, or bf16 dy16 -- may alias dx), and
// dgamma[d] via per-block partials gpart [rows/128][d] fp32 followed by [ceil(rows/128/64)][d] fp64
// stage sums in the same buffer (fixed-order reduction).
cudaError_t launch_norm_bwd(const float* dy32, const void* dy16, const void* x, const float* rstd, const float* gamma,
                            void* dx, float* gpart, float* dgamma, size_t rows, int d, cudaStream_t s, bool fp16,
                            IoLayout io, int N);
// K0: per-(head, 128-row chunk) column sums in double, fixed order (reading A17).
// Q, K, V, O, dO, dQ, dK, dV are bf16, or fp16 with SAGE_FP16 (`fp16` in the launchers below).
cudaError_t launch_colsum(const void* x, double* part, int BH, int N, int d, cudaStream_t s, NormIn nrm, bool fp16,
                          IoLayout io);
// K0b: mu[bh][c] = fl32(sum_t part[bh][t][c] / N)  (mu_K).
cudaError_t launch_colmean(const double* part, float* mu, int BH, int N, int d, cudaStream_t s);
// K0c: mu_Q[bh][t][c] = fl32(part[bh][t][c] / 128)  (block-wise mu_Qi).
cudaError_t launch_blockmean(const double* part, float* mu_q, int BH, int N, int d, cudaStream_t s);
// K1: per-block psi of x - mu (mu per column: mu_mode 0 none, 1 per head [BH][d], 2 per block [BH][T][d]),
// up to three tensors in one launch.
struct QuantJob {
  const void* x;
  const float* mu;
  int mu_mode;
  int8_t* xq;
  float* scale;
  float* rstd;         // QK-norm (NormIn): rstd out [BH*N]
  const float* gamma;  // or null
  float eps;
  int fp8;             // SAGE_PV_FP8 (V only): E4M3 values with scale amax/448 instead of INT8 with amax/127
};
struct QuantJobs {
  QuantJob j[3];
};
cudaError_t launch_quantize(const QuantJobs& jobs, int njobs, int BH, int N, int d, cudaStream_t s, bool fp16,
                            IoLayout io);
// Q-smoothing bias_i[n] = mu_Qi . (K[n] - mu_K)  (reading A13), fp32.
cudaError_t launch_qsmooth_bias(const void* k, const float* mu_k, const float* mu_q, float* bias, int BH, int N, int d,
                                cudaStream_t s, NormIn nrm, bool fp16, IoLayout io);
// K3: delta = rowsum(dO o O) (Alg. 2 line 2), psi(dO) (line 6, reading A22), l2 = lse*log2(e),
//     dq_acc = 0.
//     delta = fl32(sum in fp64 of the exact products): bit-exact against the oracle given the stored O.
//     o_f32: O is fp32 (SAGE_FP32_OUT) instead of the I/O type.
cudaError_t launch_bwd_prep(const void* o, const void* dO, const float* lse, float* delta, float* l2, int8_t* do_q,
                            float* do_scale, float* dq_acc, int BH, int N, int d, cudaStream_t s, unsigned* dq_flags,
                            bool fp16, bool o_f32, IoLayout io);
cudaError_t launch_fill(float* x, size_t n, float v, cudaStream_t s);
// K5: dQ fp32 -> bf16.
// (dq_acc contiguous [BH*N][d]; dq in the I/O layout; fp32 out with f32 = true)
cudaError_t launch_dq_finalize(const float* dq_acc, void* dq, int BH, int N, int d, cudaStream_t s, bool fp16,
                               IoLayout io, bool f32);

// ---- fused tensor-core kernels ----
struct FwdArgs {
  CUtensorMap tm_q, tm_k, tm_v;  // int8 [BH*N][d], box [128][d]
  const float *q_scale, *k_scale, *v_scale;
  const float* bias;  // [BH][T][N] or null
  void* o;     // bf16, or fp16 with SAGE_FP16
  float* lse;
  int BH, N, d;
  float tau;
  bool causal, qsmooth;
  bool pu8;    // SAGE_P_U8: P^ in 0..255 (u8 x s8 PV)
  bool fp16;   // SAGE_FP16: fp16 I/O
  bool f32out; // SAGE_FP32_OUT: O written as fp32
  bool pvfp8;  // SAGE_PV_FP8: P^ and V^ in E4M3, P^V^ as a kind::f8f6f4 MMA with fp32 accumulation
  IoLayout io; // layout of O
  int ablate;  // profiling only (SAGE_ABLATE bit 8: timeline, bit 16: sage_debug_fwd_dump)
};
cudaError_t launch_fwd(const FwdArgs& a, cudaStream_t s);
// test-only K2 dump (libsage_trace.so, sage_debug_fwd_dump): S int32 [head][N q][N kv], P^ u8 same
// layout, s_P fp32 [head][N q][T], PV int32 [head][T j][N q][d]; null pointers are skipped
struct FwdDump {
  int32_t* s;
  uint8_t* p;
  float* sp;
  int32_t* pv;
  int heads;
};
cudaError_t set_fwd_dump(const FwdDump& d);
cudaError_t read_fwd_trace(void* host, size_t bytes);  // profiling: K2 event timeline

struct BwdArgs {
  CUtensorMap tm_q, tm_k, tm_doq;  // int8 [BH*N][d], box [128][d]
  CUtensorMap tm_v, tm_do;         // bf16 4-D [B][H][N][d] in the I/O layout, box [1][1][128][64]
  CUtensorMap tm_dq;               // fp32 dQ accumulator [BH*N][d], box [32][32] (TMA reduce-add per warp)
  const float *q_scale, *k_scale, *do_scale;
  const float *l2, *delta;         // [BH][N]
  const float* bias;               // [BH][T][N] or null
  const float* mu_q;               // [BH][T][d] or null
  float* dq_acc;                   // [BH][N][d]
  void *dk, *dv;  // bf16, or fp16 with SAGE_FP16
  int BH, N, d;
  float tau;
  bool causal, qsmooth;
  bool pu8;    // SAGE_P_U8: psi(P) in 0..255 (u8 x s8 dV)
  bool fp16;   // SAGE_FP16: fp16 V, dO (dP MMA kind::f16 with f16 operands) and outputs
  bool f32out; // SAGE_FP32_OUT: dK, dV written as fp32
  IoLayout io; // layout of dK, dV (and of V, dO: the 4-D tensor maps)
  bool pcol;   // SAGE_P_COLSCALE: psi(P) per key row of P^T instead of per tile
  bool fine;   // SAGE_FINE_BWD: pcol + psi(dS) per key for dK and per query for dQ
  unsigned* dq_flags;  // SAGE_DETERMINISTIC: [BH][T][4] zeroed ordering flags, or null
  int ablate;  // profiling only (SAGE_ABLATE): 1 drain math off, 2 compute math off, 4 dQ reduction off
};
cudaError_t launch_bwd(const BwdArgs& a, cudaStream_t s);
cudaError_t read_bwd_trace(void* host, size_t bytes);  // profiling: K4 event timeline
// test-only K4 tile dump (libsage_trace.so, SAGE_ABLATE bit 16): device pointers, [head][N kv][N q]
// for the tiles, [head][T i][T j] for the scales; heads = 0 disables
struct BwdDump {
  int8_t *pt, *dst;
  float *sp, *sds, *ds;
  int heads;
};
cudaError_t set_bwd_dump(const BwdDump& d);
// the int32 accumulators (sage_debug_dump_acc): S^T [head][N kv][N q], dV / dK tiles [head][T i][N kv][d],
// dQ tiles [head][T j][N q][d]; null = not dumped
cudaError_t set_bwd_dump_acc(int32_t* s_t, int32_t* dv_t, int32_t* dk_t, int32_t* dq_t, float* dp_t);

// UMMA tile test (sage_debug_umma)
cudaError_t launch_debug_umma(int mode, int K, int N, const CUtensorMap* tma, const CUtensorMap* tmb,
                              const void* a, void* d, cudaStream_t s);

// Tensor-map helpers (sage_api.cu)
enum TmapType { kU8 = 0, kBF16 = 1, kF32 = 2, kF16 = 3 };
bool make_tmap_2d(CUtensorMap* m, const void* base, TmapType type, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint32_t box_cols);
// 4-D map over an I/O tensor [B][H][N][d] with element strides (io), box [1][1][box_rows][box_cols]
bool make_tmap_io(CUtensorMap* m, const void* base, TmapType type, int B, int N, int d, const IoLayout& io,
                  uint32_t box_rows, uint32_t box_cols);

}  // namespace sage
