/*
 * sage_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of SageBwd's quantised
 * attention (arXiv 2603.02170), written from the paper:
 *
 *   - Alg. 1 (forward)  PAPER.md:638-671  (Appendix A, "Forward pass of the 8-bit attention")
 *   - Alg. 2 (backward) PAPER.md:674-708  (Appendix A, "Backward pass of the 8-bit attention")
 *   - psi quantiser     PAPER.md:110-114  (Sec. 3 "Quantization": X^ = round(X/delta), delta = max|X|/127, stored in FP32)
 *   - smoothing         PAPER.md:136-162  (Sec. 3 "Q and K Smoothing"), PAPER.md:572-607 (Sec. 6)
 *   - FPA reference     PAPER.md:96-97, 175-186 (Sec. 3 "FlashAttention", "SageBwd" MatMul list)
 *
 * Floating point is double; the integer MatMuls accumulate exactly in int32.
 * Where the paper fixes FP32 (the psi scale "stored in FP32") the FP32
 * operation is emulated exactly (x86-64 SSE single precision, built with
 * -ffp-contract=off, no -ffast-math).  Every reading of an ambiguous or
 * garbled passage is tagged (A#) and listed in DESIGN.md section 3.
 *
 * It shares no code with the CUDA path (paper_2603_02170_b200/csrc) and must
 * never be linked, imported or called by the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it.
 *
 * Layout: every tensor is [BH][N][d] row-major (heads flattened), scales are
 * [BH][T] with T = ceil(N / blk), lse is [BH][N] in natural log.
 *
 * Ragged N (reading A33): when blk does not divide N the last block Q_{T-1} (and
 * K_{T-1}, V_{T-1}, dO_{T-1}) holds the remaining N - (T-1) blk rows; every
 * per-block statistic (psi scale, mu_Qi) is taken over the rows the block holds,
 * and a tile's missing rows / columns are absent (no logits, P = dS = 0).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_CAUSAL    1   /* mask key n > query r (A14) */
#define ORC_K_SMOOTH  2   /* K <- K - mean_row(K) */
#define ORC_Q_SMOOTH  4   /* Q_i <- Q_i - mean_row(Q_i), bias added back */
#define ORC_QUANT_OFF 8   /* psi = identity, no FP32 emulation: tiled full-precision attention */
#define ORC_P_U8     16   /* unsigned 8-bit P^ (0..255, scale max/255) instead of 0..127: the
                             u8 x s8 variant; psi(dS), psi(Q/K/V/dO) unchanged */
#define ORC_P_COL    32   /* backward psi(P) per key column of the tile instead of per tile (the dV half
                             of SURVEY.md 8(f) NEXT-2): dV_j += (P^^T dO^_i) with one scale per key */
#define ORC_DS_FINE  64   /* backward psi(dS) per query row for dQ and per key column for dK, two int8
                             copies of the tile (the dS half of SURVEY.md 8(f) NEXT-2) */
#define ORC_PV_FP8  128   /* forward P^ V^ in FP8 E4M3: per-token P^ = e4m3(P~ / s_P)
                             with s_P = e^{rowmax - m}/448, V^ = e4m3(fl32(V * fl32(448/amax))) per block with
                             s_V = fl32(amax/448); the products are summed exactly.  The backward is unchanged. */

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* psi: per-block INT8 quantisation.                              */
/*   scale = fl32(amax / 127)        ("delta_X = max(|X|)/127, stored in FP32")
 *   inv   = fl32(127 / amax), 0 for an all-zero block              (A3, A4)
 *   q     = clamp(RNE(x * inv), -127, 127)                          (A1, A2)
 * fp32_product != 0: x*inv is an FP32 multiply (inputs Q,K,V,dO are FP32
 * values); otherwise the product is taken in double (P and dS, A4).          */
static void psi_block(const double *x, int n, int fp32_product, int quant_off, double qmax,
                      int8_t *q, double *scale_out, double *xq_out) {
  double amax = 0.0;
  for (int e = 0; e < n; ++e) {
    double a = fabs(x[e]);
    if (a > amax) amax = a;
  }
  if (quant_off) {              /* psi = identity */
    for (int e = 0; e < n; ++e) xq_out[e] = x[e];
    *scale_out = 1.0;
    return;
  }
  float famax = (float)amax;    /* exact: x are FP32 values or amax rounds once */
  float fq = (float)qmax;       /* 127, or 255 for the unsigned P^ variant */
  float scale = famax / fq;
  float inv = famax > 0.0f ? fq / famax : 0.0f;
  for (int e = 0; e < n; ++e) {
    double y;
    if (fp32_product) {
      float yf = (float)x[e] * inv;  /* FP32 multiply, round-to-nearest */
      y = (double)yf;
    } else {
      y = x[e] * (double)inv;
    }
    double r = nearbyint(y);       /* round half to even (default mode) */
    if (r > qmax) r = qmax;
    if (r < -qmax) r = -qmax;
    if (q) q[e] = (int8_t)r;
    if (xq_out) xq_out[e] = r;
  }
  *scale_out = (double)scale;
}

/* FP8 E4M3 (1 sign, 4 exponent bits with bias 7, 3 mantissa bits; largest finite 448, smallest subnormal
 * 2^-9): round to nearest, ties to even, saturating at +-448 (PTX cvt.rn.satfinite.e4m3x2.f32). */
static double e4m3_rne(double x) {
  double a = fabs(x);
  if (a == 0.0) return 0.0;
  if (a >= 448.0) return x < 0 ? -448.0 : 448.0;
  int E;
  frexp(a, &E);                       /* a = f 2^E, f in [0.5, 1): binade 2^(E-1) */
  int e = E - 1;
  if (e < -6) e = -6;                 /* subnormals share the quantum 2^-9 */
  double quantum = ldexp(1.0, e - 3); /* 3 mantissa bits */
  double r = nearbyint(a / quantum) * quantum;
  if (r > 448.0) r = 448.0;
  return x < 0 ? -r : r;
}
double oracle_e4m3(double x) { return e4m3_rne(x); }

/* psi into E4M3 over one block (ORC_PV_FP8): scale = fl32(amax/448), q = e4m3(fl32(x * fl32(448/amax))). */
static void psi_block_e4m3(const double *x, int n, double *xq_out, double *scale_out) {
  double amax = 0.0;
  for (int e = 0; e < n; ++e) if (fabs(x[e]) > amax) amax = fabs(x[e]);
  float famax = (float)amax;
  float scale = famax / 448.0f;
  float inv = famax > 0.0f ? 448.0f / famax : 0.0f;
  for (int e = 0; e < n; ++e) xq_out[e] = e4m3_rne((double)((float)x[e] * inv));
  *scale_out = (double)scale;
}

void oracle_psi_block_e4m3(const double *x, int n, double *q, double *scale) { psi_block_e4m3(x, n, q, scale); }

/* Exported for the worked-example pins. */
void oracle_psi_block(const double *x, int n, int fp32_product, int8_t *q, double *scale) {
  psi_block(x, n, fp32_product, 0, 127.0, q, scale, NULL);
}

/* Per-token P quantisation, Alg. 1 line 9:
 *   s_P = exp(rowmax(S_ij) - m_ij) / 127,  P^_ij = P~_ij / s_P  (rounded, A1/A2)
 * pt: one row of P~ = exp(S - m_ij); rm_minus_m = rowmax(S_ij) - m_ij.       */
static double psi_token_row(const double *pt, int n, double rm_minus_m, double pmax, int16_t *q) {
  double sp = exp(rm_minus_m) / pmax;   /* pmax = 127, or 255 with ORC_P_U8 */
  for (int e = 0; e < n; ++e) {
    double r = nearbyint(pt[e] / sp);
    if (r > pmax) r = pmax;
    if (r < 0.0) r = 0.0;
    q[e] = (int16_t)r;
  }
  return sp;
}

double oracle_psi_token_row(const double *pt, int n, double rm_minus_m, int pmax, int16_t *q) {
  return psi_token_row(pt, n, rm_minus_m, (double)pmax, q);
}

/* rows of block t (reading A33: the last block of a ragged N is short) */
static int rows_in(int N, int blk, int t) {
  int r = N - t * blk;
  return r < blk ? r : blk;
}

/* ------------------------------------------------------------------------ */
/* Smoothing.  Column mean in double, in a fixed order: sequential
 * over the rows of each blk-row chunk, then sequential over chunks (A17);
 * rounded once to FP32 unless quant_off.                                     */
static void column_mean(const double *x, int N, int d, int blk, int quant_off, double *mu) {
  int T = (N + blk - 1) / blk;
  for (int c = 0; c < d; ++c) {
    double total = 0.0;
    for (int t = 0; t < T; ++t) {
      double part = 0.0;
      for (int r = 0; r < rows_in(N, blk, t); ++r) part += x[(size_t)(t * blk + r) * d + c];
      total += part;
    }
    double m = total / (double)N;
    mu[c] = quant_off ? m : (double)(float)m;
  }
}

/* x_sm = x - mu, an FP32 subtraction unless quant_off (A4). */
static double smooth_sub(double x, double mu, int quant_off) {
  return quant_off ? x - mu : (double)((float)x - (float)mu);
}

/* Per-head prologue shared by Alg. 1 and Alg. 2 (Alg. 2 line 1 takes the
 * forward's quantised blocks; recomputing them with this same function
 * reproduces them bit for bit).                                             */
typedef struct {
  int N, d, blk, T, flags;
  double *qs, *ks;        /* smoothed Q (if Q_SMOOTH) and K (if K_SMOOTH) [N][d] */
  double *qx, *kx;        /* psi(Q), psi(K) integer values as doubles (or identity) */
  int8_t *q8, *k8;
  double *sq, *sk;        /* [T] */
  double *mu_k;           /* [d] */
  double *mu_q;           /* [T][d] */
  double *bias;           /* [T][N]  bias_i[n] = mu_Qi . K_sm[n] */
} head_prep;

static void prep_free(head_prep *h) {
  free(h->qs); free(h->ks); free(h->qx); free(h->kx); free(h->q8); free(h->k8);
  free(h->sq); free(h->sk); free(h->mu_k); free(h->mu_q); free(h->bias);
}

static void prep_head(head_prep *h, const double *q, const double *k, int N, int d, int blk, int flags) {
  int T = (N + blk - 1) / blk, qo = (flags & ORC_QUANT_OFF) != 0;
  size_t nd = (size_t)N * d;
  h->N = N; h->d = d; h->blk = blk; h->T = T; h->flags = flags;
  h->qs = malloc(nd * sizeof(double)); h->ks = malloc(nd * sizeof(double));
  h->qx = malloc(nd * sizeof(double)); h->kx = malloc(nd * sizeof(double));
  h->q8 = calloc(nd, 1); h->k8 = calloc(nd, 1);
  h->sq = malloc(T * sizeof(double)); h->sk = malloc(T * sizeof(double));
  h->mu_k = calloc(d, sizeof(double)); h->mu_q = calloc((size_t)T * d, sizeof(double));
  h->bias = calloc((size_t)T * N, sizeof(double));

  /* K-smoothing: mu_K = mean_row(K) over all N tokens (A12). */
  if (flags & ORC_K_SMOOTH) column_mean(k, N, d, blk, qo, h->mu_k);
  for (size_t e = 0; e < nd; ++e) h->ks[e] = smooth_sub(k[e], h->mu_k[e % d], qo);

  /* Q-smoothing: mu_Qi = mean_row(Q_i), block-wise (A12). */
  for (int t = 0; t < T; ++t) {
    double *mq = h->mu_q + (size_t)t * d;
    int nb = rows_in(N, blk, t);
    if (flags & ORC_Q_SMOOTH) column_mean(q + (size_t)t * blk * d, nb, d, blk, qo, mq);
    for (int r = 0; r < nb; ++r)
      for (int c = 0; c < d; ++c) {
        size_t e = (size_t)(t * blk + r) * d + c;
        h->qs[e] = smooth_sub(q[e], mq[c], qo);
      }
  }
  /* bias_i[n] = mu_Qi . K_sm[n] in double from the unquantised K_sm (A13). */
  if (flags & ORC_Q_SMOOTH)
    for (int t = 0; t < T; ++t)
      for (int n = 0; n < N; ++n) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += h->mu_q[(size_t)t * d + c] * h->ks[(size_t)n * d + c];
        h->bias[(size_t)t * N + n] = acc;
      }
  /* Alg. 1 line 3: per-block psi of Q_i, K_j. */
  for (int t = 0; t < T; ++t) {
    size_t off = (size_t)t * blk * d;
    int nbd = rows_in(N, blk, t) * d;
    psi_block(h->qs + off, nbd, 1, qo, 127.0, h->q8 + off, &h->sq[t], h->qx + off);
    psi_block(h->ks + off, nbd, 1, qo, 127.0, h->k8 + off, &h->sk[t], h->kx + off);
  }
}

/* S_ij = MM(Q^_i, K^_j) x s_Q x s_K (Alg. 1 line 7 / Alg. 2 line 5), times the
 * softmax scale tau (A6), plus tau*bias_i with Q-smoothing.  The
 * integer product accumulates in int32; |acc| <= d*127^2 < 2^31.
 * Masked entries (A14), and the rows / columns a short last block lacks (A33),
 * are set to -INFINITY.                                                      */
static void s_tile(const head_prep *h, int i, int j, double tau, double *S) {
  int blk = h->blk, d = h->d, N = h->N, qo = (h->flags & ORC_QUANT_OFF) != 0;
  int causal = (h->flags & ORC_CAUSAL) != 0;
  for (int r = 0; r < blk; ++r) {
    int gr = i * blk + r;
    for (int n = 0; n < blk; ++n) {
      int gn = j * blk + n;
      double s;
      if (gr >= N || gn >= N) {
        S[(size_t)r * blk + n] = -INFINITY;
        continue;
      }
      if (qo) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += h->qs[(size_t)gr * d + c] * h->ks[(size_t)gn * d + c];
        s = acc * tau;
      } else {
        int32_t acc = 0;
        for (int c = 0; c < d; ++c)
          acc += (int32_t)h->q8[(size_t)gr * d + c] * (int32_t)h->k8[(size_t)gn * d + c];
        s = (double)acc * h->sq[i] * h->sk[j] * tau;
      }
      if (h->flags & ORC_Q_SMOOTH) s += tau * h->bias[(size_t)i * N + gn];
      if (causal && gn > gr) s = -INFINITY;
      S[(size_t)r * blk + n] = s;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Alg. 1: forward, per head, with the corrections of reading A7:
 *   m_0 = -inf (size B_q), l_ij = e^{m_{i,j-1}-m_ij} l_{i,j-1} + rowsum(P~_ij),
 *   O_ij = diag(e^{m_{i,j-1}-m_ij}) O_{i,j-1} + MM(P^_ij, V^_j) x s_P x s_V.   */
/* qsel (may be NULL = every block): compute O and L only for the query blocks i with qsel[i] != 0 (the
 * other rows of o / lse are left untouched).  The selected blocks run exactly the same arithmetic. */
static void fwd_head(const double *q, const double *k, const double *v, int N, int d, int blk,
                     int flags, double tau, const uint8_t *qsel, double *o, double *lse,
                     float *mu_k, float *mu_q, double *bias,
                     int8_t *q8o, int8_t *k8o, int8_t *v8o, float *sqo, float *sko, float *svo,
                     uint8_t *p8o, double *spo) {
  head_prep h;
  prep_head(&h, q, k, N, d, blk, flags);
  int T = h.T, qo = (flags & ORC_QUANT_OFF) != 0, causal = (flags & ORC_CAUSAL) != 0;
  size_t nd = (size_t)N * d;
  /* psi(V_j), Alg. 1 line 3. */
  double *vx = malloc(nd * sizeof(double));
  int8_t *v8 = calloc(nd, 1);
  double *sv = malloc(T * sizeof(double));
  int pv8 = (flags & ORC_PV_FP8) && !qo;
  for (int t = 0; t < T; ++t) {
    size_t off = (size_t)t * blk * d;
    int nbd = rows_in(N, blk, t) * d;
    if (pv8)
      psi_block_e4m3(v + off, nbd, vx + off, &sv[t]);   /* v8 (int8) stays zero in this mode */
    else
      psi_block(v + off, nbd, 1, qo, 127.0, v8 + off, &sv[t], vx + off);
  }
  double *S = malloc((size_t)blk * blk * sizeof(double));
  double *Pt = malloc((size_t)blk * blk * sizeof(double));
  int16_t *Ph = malloc((size_t)blk * blk * sizeof(int16_t));
  double pmax = (flags & ORC_P_U8) ? 255.0 : 127.0;
  double *acc = malloc((size_t)blk * d * sizeof(double));
  double *Pq = malloc(blk * sizeof(double));
  double *m = malloc(blk * sizeof(double)), *l = malloc(blk * sizeof(double));

  for (int i = 0; i < T; ++i) {
    if (qsel && !qsel[i]) continue;
    for (int r = 0; r < blk; ++r) { m[r] = -INFINITY; l[r] = 0.0; }
    memset(acc, 0, (size_t)blk * d * sizeof(double));
    int jmax = causal ? i : T - 1, nbi = rows_in(N, blk, i);
    for (int j = 0; j <= jmax; ++j) {
      int nbj = rows_in(N, blk, j);   /* keys this block holds (A33); P~ is 0 beyond them */
      s_tile(&h, i, j, tau, S);
      for (int r = 0; r < nbi; ++r) {
        const double *Sr = S + (size_t)r * blk;
        double rm = -INFINITY;
        for (int n = 0; n < blk; ++n) if (Sr[n] > rm) rm = Sr[n];
        if (rm == -INFINITY) continue;           /* fully masked row (A14) */
        double mnew = m[r] > rm ? m[r] : rm;     /* line 8 */
        double alpha = exp(m[r] - mnew);         /* e^{m_{i,j-1} - m_ij}; 0 when m = -inf */
        double rs = 0.0;
        double *Pr = Pt + (size_t)r * blk;
        for (int n = 0; n < blk; ++n) { Pr[n] = exp(Sr[n] - mnew); rs += Pr[n]; }
        l[r] = alpha * l[r] + rs;                /* A7 */
        double *ar = acc + (size_t)r * d;
        if (qo) {
          for (int c = 0; c < d; ++c) {
            double pv = 0.0;
            for (int n = 0; n < nbj; ++n) pv += Pr[n] * vx[(size_t)(j * blk + n) * d + c];
            ar[c] = alpha * ar[c] + pv;
          }
        } else if (pv8) {
          /* line 9 in FP8: s_P = e^{rowmax - m}/448, P^ = e4m3(P~ / s_P); line 10: exact sum of E4M3 products */
          double sp = exp(rm - mnew) / 448.0;
          for (int n = 0; n < blk; ++n) Pq[n] = e4m3_rne(Pr[n] / sp);
          if (p8o) for (int n = 0; n < nbj; ++n) p8o[(size_t)(i * blk + r) * N + (size_t)j * blk + n] = 0;
          if (spo) spo[(size_t)(i * blk + r) * T + j] = sp;
          for (int c = 0; c < d; ++c) {
            double pv = 0.0;
            for (int n = 0; n < nbj; ++n) pv += Pq[n] * vx[(size_t)(j * blk + n) * d + c];
            ar[c] = alpha * ar[c] + pv * sp * sv[j];
          }
        } else {
          int16_t *Phr = Ph + (size_t)r * blk;
          double sp = psi_token_row(Pr, blk, rm - mnew, pmax, Phr);   /* line 9 */
          /* optional dumps (test infrastructure: Tier-C of the forward), P^ [N q][N kv], s_P [N q][T] */
          if (p8o) for (int n = 0; n < nbj; ++n) p8o[(size_t)(i * blk + r) * N + (size_t)j * blk + n] = (uint8_t)Phr[n];
          if (spo) spo[(size_t)(i * blk + r) * T + j] = sp;
          for (int c = 0; c < d; ++c) {                            /* line 10 */
            int32_t pv = 0;
            for (int n = 0; n < nbj; ++n)
              pv += (int32_t)Phr[n] * (int32_t)v8[(size_t)(j * blk + n) * d + c];
            ar[c] = alpha * ar[c] + (double)pv * sp * sv[j];
          }
        }
        m[r] = mnew;
      }
    }
    for (int r = 0; r < nbi; ++r) {              /* lines 13-14 */
      size_t gr = (size_t)i * blk + r;
      for (int c = 0; c < d; ++c) o[gr * d + c] = l[r] > 0.0 ? acc[(size_t)r * d + c] / l[r] : 0.0;
      lse[gr] = l[r] > 0.0 ? m[r] + log(l[r]) : -INFINITY;
    }
  }
  if (mu_k) for (int c = 0; c < d; ++c) mu_k[c] = (float)h.mu_k[c];
  if (mu_q) for (int e = 0; e < T * d; ++e) mu_q[e] = (float)h.mu_q[e];
  if (bias) memcpy(bias, h.bias, (size_t)T * N * sizeof(double));
  if (q8o) memcpy(q8o, h.q8, nd);
  if (k8o) memcpy(k8o, h.k8, nd);
  if (v8o) memcpy(v8o, v8, nd);
  for (int t = 0; t < T; ++t) {
    if (sqo) sqo[t] = (float)h.sq[t];
    if (sko) sko[t] = (float)h.sk[t];
    if (svo) svo[t] = (float)sv[t];
  }
  free(vx); free(v8); free(sv); free(S); free(Pt); free(Ph); free(acc); free(m); free(l); free(Pq);
  prep_free(&h);
}

/* qsel: NULL, or [BH][T] query-block selection (see fwd_head). */
int oracle_fwd_sel(int BH, int N, int d, int blk, int flags, double tau,
                   const double *q, const double *k, const double *v, const uint8_t *qsel,
                   double *o, double *lse,
                   float *mu_k, float *mu_q, double *bias,
                   int8_t *q8, int8_t *k8, int8_t *v8, float *sq, float *sk, float *sv,
                   uint8_t *p8, double *sp) {
  if (BH <= 0 || N <= 0 || d <= 0 || blk <= 0) return -1;
  int T = (N + blk - 1) / blk;
  size_t nd = (size_t)N * d;
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < BH; ++b) {
    fwd_head(q + b * nd, k + b * nd, v + b * nd, N, d, blk, flags, tau, qsel ? qsel + (size_t)b * T : NULL,
             o + b * nd, lse + (size_t)b * N,
             mu_k ? mu_k + (size_t)b * d : NULL, mu_q ? mu_q + (size_t)b * T * d : NULL,
             bias ? bias + (size_t)b * T * N : NULL,
             q8 ? q8 + b * nd : NULL, k8 ? k8 + b * nd : NULL, v8 ? v8 + b * nd : NULL,
             sq ? sq + (size_t)b * T : NULL, sk ? sk + (size_t)b * T : NULL, sv ? sv + (size_t)b * T : NULL,
             p8 ? p8 + (size_t)b * N * N : NULL, sp ? sp + (size_t)b * N * T : NULL);
  }
  return 0;
}

int oracle_fwd(int BH, int N, int d, int blk, int flags, double tau,
               const double *q, const double *k, const double *v,
               double *o, double *lse,
               float *mu_k, float *mu_q, double *bias,
               int8_t *q8, int8_t *k8, int8_t *v8, float *sq, float *sk, float *sv) {
  return oracle_fwd_sel(BH, N, d, blk, flags, tau, q, k, v, NULL, o, lse, mu_k, mu_q, bias, q8, k8, v8, sq, sk, sv,
                        NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* Alg. 2: backward, per head.  Outer loop over kv blocks j, inner over q
 * blocks i.  o_stored is the O the forward wrote (A15), lse its L.
 * dP = dO_i V_j^T (A8) is exact in double from the I/O values (A9).          */
/* qsel / ksel (both NULL = every block): only tiles (i, j) with qsel[i] or ksel[j] are processed; dQ_i is
 * accumulated for the selected query blocks and dK_j, dV_j for the selected key blocks (the other rows
 * stay zero).  A selected output receives exactly the tiles, in exactly the order, of the full run. */
static void bwd_head(const double *q, const double *k, const double *v, const double *o_stored,
                     const double *dO, const double *lse, const uint8_t *qsel, const uint8_t *ksel,
                     int N, int d, int blk, int flags, double tau,
                     double *dq, double *dk, double *dv, double *delta_out, int8_t *do8_out, float *sdo_out,
                     uint8_t *p8_out, float *sp_out, int8_t *ds8_out, float *sds_out, double *ds_out) {
  head_prep h;
  prep_head(&h, q, k, N, d, blk, flags);
  int T = h.T, qo = (flags & ORC_QUANT_OFF) != 0, causal = (flags & ORC_CAUSAL) != 0;
  size_t nd = (size_t)N * d, bb = (size_t)blk * blk;
  /* Alg. 2 line 2: D = rowsum(dO o O). */
  double *delta = malloc(N * sizeof(double));
  for (int r = 0; r < N; ++r) {
    double s = 0.0;
    for (int c = 0; c < d; ++c) s += dO[(size_t)r * d + c] * o_stored[(size_t)r * d + c];
    delta[r] = s;
  }
  /* Alg. 2 line 6: psi(dO_i), independent of j, so taken once (A22). */
  double *dox = malloc(nd * sizeof(double));
  int8_t *do8 = calloc(nd, 1);
  double *sdo = malloc(T * sizeof(double));
  for (int t = 0; t < T; ++t) {
    size_t off = (size_t)t * blk * d;
    psi_block(dO + off, rows_in(N, blk, t) * d, 1, qo, 127.0, do8 + off, &sdo[t], dox + off);
  }
  double *S = malloc(bb * sizeof(double)), *P = malloc(bb * sizeof(double));
  double *dS = malloc(bb * sizeof(double)), *Px = malloc(bb * sizeof(double)), *dSx = malloc(bb * sizeof(double));
  int8_t *dS8 = malloc(bb);
  double pmax = (flags & ORC_P_U8) ? 255.0 : 127.0;
  int pcol = (flags & ORC_P_COL) != 0;
  double *spcol = malloc(blk * sizeof(double));
  double *colx = malloc(blk * sizeof(double)), *colq = malloc(blk * sizeof(double));
  int dsfine = (flags & ORC_DS_FINE) != 0;
  int8_t *dSq8 = malloc(bb), *dSk8 = malloc(bb);
  double *sq_row = malloc(blk * sizeof(double)), *sk_col = malloc(blk * sizeof(double));
  memset(dq, 0, nd * sizeof(double));
  memset(dk, 0, nd * sizeof(double));
  memset(dv, 0, nd * sizeof(double));

  int all = !qsel && !ksel;
  for (int j = 0; j < T; ++j) {
    for (int i = causal ? j : 0; i < T; ++i) {
      int want_q = all || (qsel && qsel[i]), want_k = all || (ksel && ksel[j]);
      if (!want_q && !want_k) continue;
      /* rows / columns this tile holds (A33); P = dS = 0 beyond them */
      int nbi = rows_in(N, blk, i), nbj = rows_in(N, blk, j);
      /* line 5: S_ij recomputed from Q^, K^; P_ij = exp(S_ij - L_i). */
      s_tile(&h, i, j, tau, S);
      for (int r = 0; r < blk; ++r)
        for (int n = 0; n < blk; ++n) {
          double s = S[(size_t)r * blk + n];
          P[(size_t)r * blk + n] = s == -INFINITY ? 0.0 : exp(s - lse[i * blk + r]);
        }
      /* line 6: psi(P_ij) over the whole B_q x B_kv tile (A11). */
      double sp;
      if (pcol && !qo) {
        /* psi over each key column n of the tile: s_P[n] = fl32(max_r P[r,n] / pmax) */
        sp = 0.0;
        for (int n = 0; n < blk; ++n) {
          for (int r = 0; r < blk; ++r) colx[r] = P[(size_t)r * blk + n];
          psi_block(colx, blk, 0, 0, pmax, NULL, &spcol[n], colq);
          for (int r = 0; r < blk; ++r) Px[(size_t)r * blk + n] = colq[r];
          if (spcol[n] > sp) sp = spcol[n];
        }
      } else {
        psi_block(P, (int)bb, 0, qo, pmax, NULL, &sp, Px);  /* Px: the integer P^ (0..pmax) */
        for (int n = 0; n < blk; ++n) spcol[n] = sp;
      }
      /* line 7: dV_j += MM(P^_ij^T, dO^_i) x s_P x s_dO. */
      for (int n = 0; n < nbj; ++n)
        for (int c = 0; c < d; ++c) {
          double val;
          if (qo) {
            double a = 0.0;
            for (int r = 0; r < nbi; ++r) a += Px[(size_t)r * blk + n] * dox[(size_t)(i * blk + r) * d + c];
            val = a;
          } else {
            int32_t a = 0;
            for (int r = 0; r < nbi; ++r)
              a += (int32_t)Px[(size_t)r * blk + n] * (int32_t)do8[(size_t)(i * blk + r) * d + c];
            val = (double)a * spcol[n] * sdo[i];
          }
          if (want_k) dv[(size_t)(j * blk + n) * d + c] += val;
        }
      /* line 8: dP_ij = MM(dO_i, V_j^T), kept unquantised (A8, A9).
       * line 9: dS_ij = P_ij o (dP_ij - D_i). */
      for (int r = 0; r < blk; ++r)
        for (int n = 0; n < blk; ++n) {
          double a = 0.0;
          if (r >= nbi || n >= nbj) {
            dS[(size_t)r * blk + n] = 0.0;
            continue;
          }
          for (int c = 0; c < d; ++c) a += dO[(size_t)(i * blk + r) * d + c] * v[(size_t)(j * blk + n) * d + c];
          dS[(size_t)r * blk + n] = P[(size_t)r * blk + n] * (a - delta[i * blk + r]);
        }
      double sds;
      psi_block(dS, (int)bb, 0, qo, 127.0, dS8, &sds, dSx);
      /* the dQ operand (scale per query row r) and the dK operand (scale per key column n): the
       * tile's dS^ and s_dS for both, or with ORC_DS_FINE a psi per row and a psi per column */
      if (dsfine && !qo) {
        for (int r = 0; r < blk; ++r) psi_block(dS + (size_t)r * blk, blk, 0, 0, 127.0, dSq8 + (size_t)r * blk, &sq_row[r], NULL);
        for (int n = 0; n < blk; ++n) {
          for (int r = 0; r < blk; ++r) colx[r] = dS[(size_t)r * blk + n];
          psi_block(colx, blk, 0, 0, 127.0, NULL, &sk_col[n], colq);
          for (int r = 0; r < blk; ++r) dSk8[(size_t)r * blk + n] = (int8_t)colq[r];
        }
      } else {
        memcpy(dSq8, dS8, bb);
        memcpy(dSk8, dS8, bb);
        for (int e = 0; e < blk; ++e) sq_row[e] = sk_col[e] = sds;
      }
      /* optional tile dumps (test infrastructure: Tier-C and fidelity reports), [N q][N kv] */
      for (int r = 0; r < nbi; ++r)
        for (int n = 0; n < nbj; ++n) {
          size_t g = (size_t)(i * blk + r) * N + (size_t)j * blk + n, t = (size_t)r * blk + n;
          if (p8_out) p8_out[g] = (uint8_t)Px[t];
          if (ds8_out) ds8_out[g] = dSk8[t];  /* the dK operand (= the tile's dS^ unless ORC_DS_FINE) */
          if (ds_out) ds_out[g] = dS[t];
        }
      if (sp_out) sp_out[(size_t)i * T + j] = (float)sp;
      if (sds_out) sds_out[(size_t)i * T + j] = (float)sds;
      /* line 10: dQ_i += MM(dS^_ij, K^_j) x s_dS x s_K  (x tau, A6). */
      for (int r = 0; r < nbi; ++r)
        for (int c = 0; c < d; ++c) {
          double val;
          if (qo) {
            double a = 0.0;
            for (int n = 0; n < nbj; ++n) a += dSx[(size_t)r * blk + n] * h.kx[(size_t)(j * blk + n) * d + c];
            val = a * tau;
          } else {
            int32_t a = 0;
            for (int n = 0; n < nbj; ++n)
              a += (int32_t)dSq8[(size_t)r * blk + n] * (int32_t)h.k8[(size_t)(j * blk + n) * d + c];
            val = (double)a * sq_row[r] * h.sk[j] * tau;
          }
          if (want_q) dq[(size_t)(i * blk + r) * d + c] += val;
        }
      /* line 11: dK_j += MM(dS^_ij^T, Q^_i) x s_dS x s_Q  (x tau, A6);
       * with Q-smoothing also dK_bias = (dS^T 1) mu_Q^T  (A13). */
      for (int n = 0; n < nbj; ++n) {
        double colsum = 0.0;
        for (int r = 0; r < nbi; ++r) colsum += qo ? dSx[(size_t)r * blk + n] : (double)dSk8[(size_t)r * blk + n];
        for (int c = 0; c < d; ++c) {
          double val;
          if (qo) {
            double a = 0.0;
            for (int r = 0; r < nbi; ++r) a += dSx[(size_t)r * blk + n] * h.qx[(size_t)(i * blk + r) * d + c];
            val = a * tau;
          } else {
            int32_t a = 0;
            for (int r = 0; r < nbi; ++r)
              a += (int32_t)dSk8[(size_t)r * blk + n] * (int32_t)h.q8[(size_t)(i * blk + r) * d + c];
            val = (double)a * sk_col[n] * h.sq[i] * tau;
          }
          if (flags & ORC_Q_SMOOTH) val += tau * (qo ? 1.0 : sk_col[n]) * colsum * h.mu_q[(size_t)i * d + c];
          if (want_k) dk[(size_t)(j * blk + n) * d + c] += val;
        }
      }
    }
  }
  if (delta_out) memcpy(delta_out, delta, N * sizeof(double));
  if (do8_out) memcpy(do8_out, do8, nd);
  if (sdo_out) for (int t = 0; t < T; ++t) sdo_out[t] = (float)sdo[t];
  free(delta); free(dox); free(do8); free(sdo); free(S); free(P); free(dS); free(Px); free(dSx);
  free(dS8); free(spcol); free(colx); free(colq); free(dSq8); free(dSk8); free(sq_row); free(sk_col);
  prep_free(&h);
}

/* qsel, ksel: NULL, or [BH][T] query / key block selections (see bwd_head). */
int oracle_bwd_sel(int BH, int N, int d, int blk, int flags, double tau,
                   const double *q, const double *k, const double *v, const double *o_stored,
                   const double *dO, const double *lse, const uint8_t *qsel, const uint8_t *ksel,
                   double *dq, double *dk, double *dv,
                   double *delta, int8_t *do8, float *sdo,
                   uint8_t *p8, float *sp, int8_t *ds8, float *sds, double *ds) {
  if (BH <= 0 || N <= 0 || d <= 0 || blk <= 0) return -1;
  int T = (N + blk - 1) / blk;
  size_t nd = (size_t)N * d;
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < BH; ++b) {
    bwd_head(q + b * nd, k + b * nd, v + b * nd, o_stored + b * nd, dO + b * nd, lse + (size_t)b * N,
             qsel ? qsel + (size_t)b * T : NULL, ksel ? ksel + (size_t)b * T : NULL,
             N, d, blk, flags, tau, dq + b * nd, dk + b * nd, dv + b * nd,
             delta ? delta + (size_t)b * N : NULL, do8 ? do8 + b * nd : NULL,
             sdo ? sdo + (size_t)b * T : NULL,
             p8 ? p8 + (size_t)b * N * N : NULL, sp ? sp + (size_t)b * T * T : NULL,
             ds8 ? ds8 + (size_t)b * N * N : NULL, sds ? sds + (size_t)b * T * T : NULL,
             ds ? ds + (size_t)b * N * N : NULL);
  }
  return 0;
}

int oracle_bwd(int BH, int N, int d, int blk, int flags, double tau,
               const double *q, const double *k, const double *v, const double *o_stored,
               const double *dO, const double *lse,
               double *dq, double *dk, double *dv,
               double *delta, int8_t *do8, float *sdo,
               uint8_t *p8, float *sp, int8_t *ds8, float *sds, double *ds) {
  return oracle_bwd_sel(BH, N, d, blk, flags, tau, q, k, v, o_stored, dO, lse, NULL, NULL, dq, dk, dv, delta, do8,
                        sdo, p8, sp, ds8, sds, ds);
}

/* ------------------------------------------------------------------------ */
/* Full-precision attention (FPA), materialising N x N, for fidelity reports
 * and pins:
 *   S = tau Q K^T (masked), P = softmax(S), O = P V, L = logsumexp(S)
 *   delta = rowsum(dO o O), dP = dO V^T, dS = P o (dP - delta 1^T),
 *   dQ = tau dS K, dK = tau dS^T Q, dV = P^T dO.
 * Optional intermediates P, dP, dS are [BH][N][N]; delta is [BH][N].         */
static void fpa_head(const double *q, const double *k, const double *v, const double *dO, int N, int d,
                     int flags, double tau, double *o, double *lse, double *dq, double *dk, double *dv,
                     double *Po, double *dPo, double *dSo, double *deltao) {
  int causal = (flags & ORC_CAUSAL) != 0;
  size_t nn = (size_t)N * N;
  double *P = malloc(nn * sizeof(double)), *dS = malloc(nn * sizeof(double));
  double *dP = malloc(nn * sizeof(double)), *delta = malloc(N * sizeof(double));
  for (int r = 0; r < N; ++r) {
    double *Pr = P + (size_t)r * N, mx = -INFINITY;
    for (int n = 0; n < N; ++n) {
      double s = -INFINITY;
      if (!(causal && n > r)) {
        s = 0.0;
        for (int c = 0; c < d; ++c) s += q[(size_t)r * d + c] * k[(size_t)n * d + c];
        s *= tau;
      }
      Pr[n] = s;
      if (s > mx) mx = s;
    }
    double sum = 0.0;
    for (int n = 0; n < N; ++n) { Pr[n] = Pr[n] == -INFINITY ? 0.0 : exp(Pr[n] - mx); sum += Pr[n]; }
    for (int n = 0; n < N; ++n) Pr[n] /= sum;
    lse[r] = mx + log(sum);
    for (int c = 0; c < d; ++c) {
      double a = 0.0;
      for (int n = 0; n < N; ++n) a += Pr[n] * v[(size_t)n * d + c];
      o[(size_t)r * d + c] = a;
    }
  }
  if (dO) {
    for (int r = 0; r < N; ++r) {
      double s = 0.0;
      for (int c = 0; c < d; ++c) s += dO[(size_t)r * d + c] * o[(size_t)r * d + c];
      delta[r] = s;
      for (int n = 0; n < N; ++n) {
        double a = 0.0;
        for (int c = 0; c < d; ++c) a += dO[(size_t)r * d + c] * v[(size_t)n * d + c];
        dP[(size_t)r * N + n] = a;
        dS[(size_t)r * N + n] = P[(size_t)r * N + n] * (a - s);
      }
    }
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < d; ++c) {
        double a = 0.0;
        for (int n = 0; n < N; ++n) a += dS[(size_t)r * N + n] * k[(size_t)n * d + c];
        dq[(size_t)r * d + c] = tau * a;
      }
    for (int n = 0; n < N; ++n)
      for (int c = 0; c < d; ++c) {
        double a = 0.0, b = 0.0;
        for (int r = 0; r < N; ++r) {
          a += dS[(size_t)r * N + n] * q[(size_t)r * d + c];
          b += P[(size_t)r * N + n] * dO[(size_t)r * d + c];
        }
        dk[(size_t)n * d + c] = tau * a;
        dv[(size_t)n * d + c] = b;
      }
    if (dPo) memcpy(dPo, dP, nn * sizeof(double));
    if (dSo) memcpy(dSo, dS, nn * sizeof(double));
    if (deltao) memcpy(deltao, delta, N * sizeof(double));
  }
  if (Po) memcpy(Po, P, nn * sizeof(double));
  free(P); free(dS); free(dP); free(delta);
}

int oracle_fpa(int BH, int N, int d, int flags, double tau,
               const double *q, const double *k, const double *v, const double *dO,
               double *o, double *lse, double *dq, double *dk, double *dv,
               double *P, double *dP, double *dS, double *delta) {
  if (BH <= 0 || N <= 0 || d <= 0) return -1;
  size_t nd = (size_t)N * d, nn = (size_t)N * N;
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < BH; ++b)
    fpa_head(q + b * nd, k + b * nd, v + b * nd, dO ? dO + b * nd : NULL, N, d, flags, tau,
             o + b * nd, lse + (size_t)b * N, dq ? dq + b * nd : NULL, dk ? dk + b * nd : NULL,
             dv ? dv + b * nd : NULL, P ? P + b * nn : NULL, dP ? dP + b * nn : NULL,
             dS ? dS + b * nn : NULL, delta ? delta + (size_t)b * N : NULL);
  return 0;
}
