/*
 * sage.h -- C ABI of libsage.so: SageBwd trainable INT8 attention (arXiv 2603.02170)
 * forward and backward, hand-written for sm_100a (B200).
 *
 * The operations (PAPER.md line numbers, section/algorithm in brackets):
 *   sage_fwd  Alg. 1, P:638-671 [App. A "Forward pass of the 8-bit attention"]:
 *             K-smoothing K <- K - mean_row(K), optional block-wise
 *             Q-smoothing with the low-rank bias added back, per-block INT8
 *             psi of Q, K, V (Alg. 1 line 3), INT8 S = Q^K^T (line 7),
 *             online softmax (line 8), per-token INT8 P~ (line 9), INT8 P^V^ (line 10),
 *             O and logsumexp L (lines 13-14).
 *   sage_bwd  Alg. 2, P:674-708 [App. A "Backward pass of the 8-bit attention"]:
 *             delta = rowsum(dO o O) (line 2), INT8 S recompute and P = exp(S - L) (line 5),
 *             psi(P), psi(dO) (line 6), INT8 dV (line 7), dP = dO V^T unquantised in
 *             BF16 with FP32 accumulation (line 8), dS = P o (dP - delta) and
 *             psi(dS) (line 9), INT8 dQ (line 10), INT8 dK (line 11) plus the Q-smoothing
 *             dK bias branch.
 * Readings of ambiguous passages (tile size 128, softmax scale 1/sqrt(d), rounding,
 * all-zero blocks, causal masking, ...) are listed in DESIGN.md section 3.
 *
 * Conventions
 *   - Tensors Q, K, V, O, dO, dQ, dK, dV: bf16 (fp16 with SAGE_FP16), [B, H, N, d] with d innermost and the
 *     strides of sage_params (contiguous by default), 16-byte aligned device pointers on the current device.
 *     1 <= N <= 32768, d in {64, 128}.  N need not be a multiple of 128: the last block of a head is then
 *     short, with every per-block statistic taken over the rows it holds (reading A33).  With
 *     SAGE_FP32_OUT the outputs O, dQ, dK, dV are fp32 instead.
 *   - The library's own buffers (ctx, workspace; the views below) pad every head to Np = 128 ceil(N/128)
 *     rows; T = ceil(N/128) is the number of blocks.
 *   - lse: fp32 [B, H, N], natural log (Alg. 1 line 14).
 *   - Ownership: the caller allocates every buffer (device memory), including the
 *     forward->backward context `ctx` (sage_ctx_bytes) and the scratch workspace
 *     (sage_workspace_bytes).  The library never allocates or frees device memory.
 *   - Execution: every call only enqueues kernels on `stream` and returns; errors in
 *     arguments are reported before anything is launched (nothing is written).  Calls are
 *     reentrant and thread-safe as long as concurrent calls use distinct workspaces.
 *     Asynchronous device faults surface at the caller's next synchronisation.
 *   - There is no CPU fallback: without an sm_100 device the calls return SAGE_ERR_ARCH.
 */
#ifndef SAGE_H_
#define SAGE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SAGE_API __attribute__((visibility("default")))
#else
#define SAGE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SAGE_OK = 0,
  SAGE_ERR_INVALID_VALUE = 1, /* null pointer, bad shape/flags, N outside [1, 32768], d not in {64,128} */
  SAGE_ERR_UNSUPPORTED = 2,   /* valid but not implemented combination */
  SAGE_ERR_MISALIGNED = 3,    /* a pointer is not 16-byte aligned */
  SAGE_ERR_WORKSPACE = 4,     /* ctx or workspace smaller than required */
  SAGE_ERR_CUDA = 5,          /* a CUDA runtime call or launch failed (see sage_last_cuda_error) */
  SAGE_ERR_ARCH = 6           /* current device is not sm_100 */
} sage_status;

/* sage_params.flags */
enum {
  SAGE_CAUSAL = 1u << 0,   /* mask key n > query r (reading A14) */
  SAGE_K_SMOOTH = 1u << 1, /* K-smoothing, P:136-147 (the paper's default) */
  SAGE_Q_SMOOTH = 1u << 2, /* block-wise Q-smoothing + bias */
  SAGE_P_U8 = 1u << 3,     /* variant: P^ unsigned in 0..255 with scale max/255,
                              for the per-token P^ of Alg. 1 line 9 and psi(P) of Alg. 2 line 6 (the
                              paper's reading: 0..127, A2); the PV / dV MMAs run u8 x s8.  Halves P^'s
                              rounding step at no cost: lower O and dV error vs full precision. */
  SAGE_QK_NORM = 1u << 4,  /* QK-norm in front of the path: use
                              sage_fwd_qknorm / sage_bwd_qknorm (sage_fwd / sage_bwd reject it) */
  SAGE_DETERMINISTIC = 1u << 5, /* bitwise run-to-run reproducible dQ (reading A19; NEXT-4): the fp32
                              dQ reduction across key blocks happens in a fixed order, enforced by
                              per-(head, query block) flags in the workspace.  Slower backward.
                              Non-causal requires T <= the device's SM count
                              (SAGE_ERR_UNSUPPORTED otherwise).  Every other output is always
                              deterministic. */
  SAGE_P_COLSCALE = 1u << 6, /* variant (the dV half of SURVEY.md 8(f) NEXT-2): the backward's psi(P)
                              (Alg. 2 line 6) takes one scale per key of the tile (the max over its
                              128 queries) instead of one per tile; dV_j's drain applies it per row.
                              dV's error vs full precision drops ~2.6x at Table 1's sigma = 1.
                              Not combinable with SAGE_DETERMINISTIC (SAGE_ERR_INVALID_VALUE). */
  SAGE_FINE_BWD = 1u << 7,  /* variant (the paper's future work on the dS path,
                              P:621-623): SAGE_P_COLSCALE plus psi(dS) (Alg. 2 line 9) taken twice,
                              with one scale per key for the dK operand and one per query for the dQ
                              operand (two int8 copies of the tile).  At Table 1's sigma = 1 it brings
                              dQ / dK / dV to 0.022 / 0.022 / 0.021 vs the paper's 0.018 / 0.022 /
                              0.016 (per-tile: 0.067 / 0.066 / 0.055).  Slower backward.  Not
                              combinable with SAGE_DETERMINISTIC. */
  SAGE_FP16 = 1u << 8,      /* fp16 instead of bf16 for Q, K, V, O, dO, dQ, dK, dV (and X_q, X_k, dX_q,
                              dX_k with QK-norm, whose module output is then fp16): dP = dO V^T runs
                              as an fp16 kind::f16 MMA, the paper's "FP16" option */
  SAGE_FP32_OUT = 1u << 9,  /* O, dQ, dK, dV written as fp32 (no rounding to the I/O type), e.g. to
                              compare against an unrounded reference (reading A18).  delta is then
                              formed from the fp32 O the forward stored (A15).  Not combinable with
                              SAGE_QK_NORM (SAGE_ERR_INVALID_VALUE). */
  SAGE_PV_FP8 = 1u << 10    /* variant: the forward's P^ V^ (Alg. 1 lines 9-10)
                              in FP8 E4M3 -- per-token P^ = e4m3(P~ / s_P) with s_P = e^{rowmax - m}/448,
                              V^ = e4m3(V / s_V) per block with s_V = amax/448 -- as a kind::f8f6f4 MMA
                              accumulating in fp32 (no int32 -> fp32 conversions in the O update).  E4M3's
                              3-bit mantissa makes O 2-4x less accurate than the INT8 path.  The backward is
                              unchanged.  Not combinable with SAGE_P_U8. */
};

typedef struct {
  int32_t batch, heads, seqlen, head_dim; /* B, H, N, d */
  uint32_t flags;                         /* SAGE_* bit set */
  float softmax_scale;                    /* tau; 0 => 1/sqrt(d) (reading A6) */
  /* Element strides of the batch, head and token dimensions of every I/O tensor (Q, K, V, O, dO, dQ, dK, dV,
   * and X_q, X_k, dX_q, dX_k with QK-norm; the head dimension d is contiguous): row (b, h, n) starts at
   * b * stride_b + h * stride_h + n * stride_n.  All three 0 = contiguous [B, H, N, d].  Otherwise each must
   * be a multiple of 8 elements and stride_n >= d (e.g. a [B, N, H, d] tensor: stride_b = N H d,
   * stride_h = d, stride_n = H d).  lse stays contiguous [B, H, N]. */
  int64_t stride_b, stride_h, stride_n;
} sage_params;

/* The forward->backward context (Alg. 2's inputs): a caller-owned device buffer plus a host
 * tag.  sage_fwd fills the buffer and sets params_tag = sage_params_tag(p); sage_bwd refuses
 * (SAGE_ERR_INVALID_VALUE, nothing launched) a ctx whose tag differs from its own params' tag -- a
 * context produced under another shape, softmax scale or flag set (SPEC's "missing retained quantized
 * operands") -- and a ctx never filled by sage_fwd (tag 0). */
typedef struct {
  void* buf;           /* device memory of at least sage_ctx_bytes(p) bytes, 256-byte aligned */
  size_t bytes;        /* size of buf */
  uint64_t params_tag; /* written by sage_fwd; 0 = not filled */
} sage_ctx;

/* Bytes of the context buffer: int8 Q^, K^ [B,H,Np,d]; fp32 s_Q, s_K [B,H,T]; mu_K [B,H,d]; and with
 * SAGE_Q_SMOOTH mu_Q [B,H,T,d] and the bias [B,H,T,Np] (Alg. 2 line 1 inputs).
 * 0 on invalid params. */
SAGE_API size_t sage_ctx_bytes(const sage_params* p);

/* The tag sage_fwd writes into sage_ctx.params_tag for these params (a 64-bit FNV-1a hash of every
 * field; never 0).  0 on invalid params. */
SAGE_API uint64_t sage_params_tag(const sage_params* p);

/* Bytes of scratch for sage_fwd (backward = 0: V^, s_V, partial sums) or sage_bwd
 * (backward = 1: dO^, s_dO, delta, L*log2(e), fp32 dQ accumulator). 0 on invalid params. */
SAGE_API size_t sage_workspace_bytes(const sage_params* p, int backward);

/* Forward (Alg. 1).  Reads q, k, v; writes o, lse, the context buffer ctx->buf and ctx->params_tag.
 * ws must hold sage_workspace_bytes(p, 0) bytes.  stream: a cudaStream_t (NULL = legacy).
 * Errors: SAGE_ERR_INVALID_VALUE (bad params, null pointer, q not on the current device),
 * SAGE_ERR_MISALIGNED, SAGE_ERR_WORKSPACE (ctx->bytes or ws_bytes too small), SAGE_ERR_ARCH,
 * SAGE_ERR_CUDA (a launch failed). */
SAGE_API sage_status sage_fwd(const sage_params* p, const void* q, const void* k, const void* v, void* o, float* lse,
                              sage_ctx* ctx, void* ws, size_t ws_bytes, void* stream);

/* Backward (Alg. 2).  Reads v, the o and lse written by sage_fwd, dO and ctx; writes
 * dq, dk, dv.  ws must hold sage_workspace_bytes(p, 1) bytes.  Errors as sage_fwd, plus
 * SAGE_ERR_INVALID_VALUE when ctx->params_tag != sage_params_tag(p). */
SAGE_API sage_status sage_bwd(const sage_params* p, const void* v, const void* o, const float* lse, const void* dO,
                              const sage_ctx* ctx, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes,
                              void* stream);

/* QK-norm variant ("Stabilizing Outliers with QK-Norm"; eps P:405).  p->flags must hold
 * SAGE_QK_NORM.  Instead of Q and K the caller passes the pre-norm X_q, X_k (bf16 [B,H,N,d]) and the
 * RMSNorm scales gamma_q, gamma_k (fp32 [d], shared by all heads); the path then runs on
 *     Q = bf16(fl32(fl32(X_q * rstd) * gamma_q)),  rstd = fl32(1 / sqrt(mean_c X^2 + eps))
 * (and the same for K), i.e. exactly the BF16 values an unfused RMSNorm module would produce
 * (readings A24-A25).  The normalisation is fused into the smoothing / quantisation
 * passes (Q and K are never written to memory); rstd of every row is kept in ctx for the backward.
 * eps > 0 (the paper uses 1e-6). */
SAGE_API sage_status sage_fwd_qknorm(const sage_params* p, const void* xq, const void* xk, const void* v,
                                     const float* gamma_q, const float* gamma_k, float eps, void* o, float* lse,
                                     sage_ctx* ctx, void* ws, size_t ws_bytes, void* stream);
/* Backward of sage_fwd_qknorm: Alg. 2 as sage_bwd, then the RMSNorm backward (reading A26) fused with
 * the dQ finalisation: writes dX_q, dX_k (bf16 [B,H,N,d]) into dxq, dxk, dV into dv, and
 * dgamma_q, dgamma_k (fp32 [d], summed over all B*H*N rows in a fixed order).  xq, xk, gamma_q,
 * gamma_k must be the forward's. */
SAGE_API sage_status sage_bwd_qknorm(const sage_params* p, const void* xq, const void* xk, const float* gamma_q,
                                     const float* gamma_k, const void* v, const void* o, const float* lse,
                                     const void* dO, const sage_ctx* ctx, void* dxq, void* dxk,
                                     void* dv, float* dgamma_q, float* dgamma_k, void* ws, size_t ws_bytes,
                                     void* stream);

/* Device pointers into a context / workspace buffer (for tests and tracing; no launch). */
typedef struct {
  int8_t *q_i8, *k_i8;        /* [B,H,Np,d] psi(Q_sm or Q), psi(K_sm); rows N..Np-1 zero */
  float *q_scale, *k_scale;   /* [B,H,T] */
  float* mu_k;                /* [B,H,d] */
  float* mu_q;                /* [B,H,T,d] or NULL */
  float* bias;                /* [B,H,T,Np] or NULL: bias_i[n] = mu_Qi . K_sm[n] (0 for n >= N) */
  float *rstd_q, *rstd_k;     /* [B,H,Np] QK-norm rstd of X_q / X_k rows, or NULL */
} sage_ctx_view;
SAGE_API sage_status sage_ctx_get_view(const sage_params* p, void* ctx, sage_ctx_view* out);

typedef struct {
  int8_t* v_i8;   /* fwd: [B,H,Np,d] psi(V) */
  float* v_scale; /* fwd: [B,H,T] */
  int8_t* do_i8;  /* bwd: [B,H,Np,d] psi(dO) */
  float* do_scale;/* bwd: [B,H,T] */
  float* delta;   /* bwd: [B,H,Np] rowsum(dO o O), 0 on the padded rows */
  float* dq_acc;  /* bwd: [B,H,Np,d] fp32 dQ accumulator */
} sage_ws_view;
SAGE_API sage_status sage_ws_get_view(const sage_params* p, int backward, void* ws, sage_ws_view* out);

/* Test entry (Tier B parity): one 128 x N UMMA tile through the same descriptor and
 * TMEM code the fused kernels use.  mode 0: int32 D = A[128][K] . B[N][K]^T with both
 * operands K-major (K in {64,128}, N = 128);  mode 1: A K-major [128][128] written by
 * threads (P^ path), B MN-major [128][N] (N in {64,128}); mode 2: A MN-major [K=128][M=128],
 * B MN-major [128][N]; mode 3: fp32 D = A . B^T, bf16 K-major operands [128][K], [128][K];
 * modes 4 / 5: as 1 / 3 with the A operand read from TMEM (written there by threads);
 * modes 6 / 7: as 1 / 4 with an unsigned u8 A operand (values 0..255, the SAGE_P_U8 P^ paths).
 * a, b, d: device pointers to row-major host-order arrays as described (int8/bf16 in, int32/fp32 out). */
SAGE_API sage_status sage_debug_umma(int mode, int K, int N, const void* a, const void* b, void* d, void* stream);

/* Profiling only (libsage_trace.so): copy the K4 and K2 pipeline timelines (clock64 stamps, uint64
 * [4 CTAs][64 tiles][24 events] each, recorded when the environment variable SAGE_ABLATE has bit 8
 * set) to host memory: K4 in the first half of `bytes`, K2 in the second. */
SAGE_API sage_status sage_debug_trace(void* host_out, size_t bytes);

/* Test only (libsage_trace.so; the production libsage.so returns SAGE_ERR_UNSUPPORTED): make every
 * later sage_bwd dump, for heads bh < `heads` (bh = b*H + h), K4's own backward intermediates
 * (Alg. 2 lines 5-11) into caller-owned device memory (T = N/128; N % 128 == 0 only --
 * a ragged N's backward runs without dumping):
 *   p_hat_t  int8 [heads][N kv][N q]  P^ of tile (i, j) transposed (key-major), psi(P) per tile (A11)
 *   ds_hat_t int8 [heads][N kv][N q]  dS^, same layout
 *   ds_t     fp32 [heads][N kv][N q]  dS = P o (dP - delta) before psi
 *   s_p, s_ds fp32 [heads][T i][T j]  the tile scales fl32(amax / 127)
 *   s_t      int32 [heads][N kv][N q] the recomputed S^T = K^_j Q^_i^T accumulator (line 5)
 *   dv_t     int32 [heads][T i][N kv][d]  the dV tile P^^T dO^_i before its scaling (line 7)
 *   dk_t     int32 [heads][T i][N kv][d]  the dK tile dS^^T Q^_i (line 11)
 *   dq_t     int32 [heads][T j][N q][d]   the dQ tile dS^ K^_j (line 10)
 *   dp_t     fp32  [heads][N kv][N q] dP^T = V_j dO_i^T as the BF16 MMA accumulated it (line 8)
 * Any of the last five may be NULL (not dumped).  Tiles a causal run skips are not written.
 * heads = 0 turns the dump off.  The buffers must stay valid until the dumping sage_bwd has completed.
 * Not thread-safe (process-wide state). */
SAGE_API sage_status sage_debug_dump(void* p_hat_t, float* s_p, void* ds_hat_t, float* s_ds, float* ds_t, int heads);
SAGE_API sage_status sage_debug_dump_acc(int32_t* s_t, int32_t* dv_t, int32_t* dk_t, int32_t* dq_t, float* dp_t);

/* Test only (libsage_trace.so): make every later sage_fwd dump, for heads bh < `heads`, K2's own
 * intermediates (Alg. 1 lines 7-10) into caller-owned device memory (N % 128 == 0 only):
 *   s       int32 [heads][N q][N kv]    the S = Q^_i K^_j^T accumulator of every processed tile (line 7)
 *   p_hat   uint8 [heads][N q][N kv]    the per-token P^ (line 9), 0..127 (0..255 with SAGE_P_U8)
 *   s_p     fp32  [heads][N q][T j]     its per-row scale s_P = e^{rowmax - m_ij} / 127 (line 9)
 *   pv      int32 [heads][T j][N q][d]  the P^ V^_j accumulator before scaling (line 10)
 * Any pointer may be NULL (not dumped).  heads = 0 turns the dump off. */
SAGE_API sage_status sage_debug_fwd_dump(int32_t* s, void* p_hat, float* s_p, int32_t* pv, int heads);

/* Optional instrumentation (calling thread only).  While enabled, sage_fwd / sage_bwd record
 * a CUDA event pair around their fused kernel (K2 / K4) and count every kernel they launch.
 * sage_profile_read synchronises on the recorded events, returns the summed K2 and K4 device
 * times (ms), the number of K2 / K4 launches and of all library kernel launches since the last
 * read, and resets the counters.  Disabled by default: zero cost on the normal path. */
SAGE_API sage_status sage_profile_enable(int enable);
SAGE_API sage_status sage_profile_read(double* fwd_kernel_ms, double* bwd_kernel_ms, int64_t* n_fwd, int64_t* n_bwd,
                                       int64_t* n_launches);

SAGE_API const char* sage_status_string(sage_status s);
SAGE_API int sage_last_cuda_error(void); /* cudaError_t of the last SAGE_ERR_CUDA (per thread) */
SAGE_API int sage_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SAGE_H_ */
