// sage_bwd.cu -- K4: SageBwd backward, Alg. 2.  One CTA per
// (head, 128-key block j), looping over query blocks i (kv-stationary, Alg. 2 loop
// order: j outer, i inner).  Everything is computed transposed so that
// TMEM lanes are key rows:
//   S^T   = MM(K^_j, Q^_i)          kind::i8   A K^_j K-major, B Q^_i K-major     (line 5)
//   P     = exp(S - L_i);  psi(P) over the 128x128 tile (reading A11)               (lines 5-6)
//   dP^T  = V_j dO_i^T               kind::f16  bf16 operands, fp32 accumulation     (line 8)
//   dS    = P o (dP - D_i);  psi(dS) over the tile                                   (line 9)
//   dV_j += MM(P^^T, dO^_i) s_P s_dO    A P^^T smem K-major, B dO^_i MN-major        (line 7)
//   dK_j += MM(dS^^T, Q^_i) s_dS s_Q tau  (+ tau s_dS colsum(dS^) mu_Qi)  (line 11)
//   dQ_i += MM(dS^, K^_j) s_dS s_K tau    A dS^ (the dS^^T tile read MN-major), B K^_j MN-major (line 10)
//
// Warp roles (512 threads, register budgets re-balanced with setmaxnreg):
//   warp 0        TMA producer: K^_j, V_j once; per i a stage {Q^_i, dO_i, dO^_i, L_i, delta_i}
//   warp 1        TMEM allocator + MMA issuer (one thread)
//   warps 4-11    two compute warpgroups, query columns [0,64) / [64,128) of every tile.
//                 Single pass: S^T and dP^T are read from TMEM once into a 64-float register
//                 tile (t -> P -> dS in place), so their TMEM columns free up immediately and
//                 the next tile's MMAs overlap this tile's softmax / quantisation.
//   warps 12-15   drain warpgroup: the per-tile scales forbid int32 accumulation across
//                 tiles, so every dK/dQ (and, for d=64, dV) int32 tile is converted and scaled
//                 here while the compute warpgroups already work on the next tile.  dK_j (and
//                 dV_j for d=64) accumulate in fp32 registers; for d=128 the compute warps drain
//                 the dV tile into an fp32 accumulator in TMEM.  dQ_i is reduced across key blocks
//                 with a TMA reduce-add (cp.reduce.async.bulk.tensor .add, fp32) per drain warp,
//                 finalised by K5.
// TMEM (512 columns):  d=64 : S 0 | dP 128 | dV 256 | dK 320 | dQ 384 | V_j (bf16) 448 | P^^T 480
//                      d=128: S/dV 0 | dP 128 | dK, then dQ 256 | dV fp32 accumulator 384
//   (d=128 aliases the dV tile onto S, and dK_i and dQ_i take turns in the third region
//   (SAGE_K4_DKQ128); the MMA issuer orders them through the drain barriers.)
#include "sage_internal.h"
#include "sm100.cuh"

namespace sage {
namespace {

constexpr int kThreads = 512;
constexpr int kComputeWarps = 8;
constexpr int kDrainWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxT = kMaxSeqLen / kBlk;

template <int D, bool FINE = false>
struct BwdSmem {
  static constexpr int kStages = D == 64 ? 4 : 2;
  static constexpr int kTile = kBlk * D;           // int8 [128][D]
  // d=128: bf16 dO_i gets its own single buffer (it is only read by the dP MMA, early in a
  // tile), which frees the shared memory for the dQ reduce staging below
  static constexpr bool kSplitDO = D == 128;
  static constexpr int kK = 0;                     // K^_j
  static constexpr int kV = kK + kTile;            // V_j bf16: D/64 panels of [128][64]
  static constexpr int kStage = kV + 2 * kTile;    // per stage: Q^_i, dO^_i, L2, delta (+ dO_i bf16 for d=64)
  // d=128 stages also carry mu_Qi (Q-smoothing dK bias branch) after delta
  static constexpr int kSQ = 0, kSDOQ = kTile, kSL = 2 * kTile, kSDelta = 2 * kTile + 512, kSMu = 2 * kTile + 1024;
  static constexpr int kSDO = 2 * kTile + 1024;  // d=64 only (1024-aligned for the 128B-swizzled panel)
  static constexpr int kStageBytes = kSplitDO ? 2 * kTile + 2048 : 4 * kTile + 1024;
  static constexpr int kDO = kStage + kStages * kStageBytes;    // d=128: dO_i bf16 panels
  static constexpr int kPt = kDO + (kSplitDO ? 2 * kTile : 0);  // P^^T [128 kv][128 q]
  static constexpr int kDSt = kPt + (D == 64 ? 0 : kBlk * kBlk);  // dS^^T [128 kv][128 q] (d=64: P^^T is in TMEM)
  static constexpr int kDSq = kDSt + kBlk * kBlk;             // FINE: dS^ with per-query scales (A of dQ)
  // dQ staging for the TMA reduce-add, per drain warp (its 32 TMEM lanes = 32 query rows):
  // kDqBufs buffers of [kDqBoxes][32 rows][32 cols] fp32 boxes, 128B-swizzled; d=64 stages the warp's
  // whole row slice per round, d=128 a quarter of it (4 rounds per tile).  No cross-warp barrier.
  // FINE gives one staging buffer to its second dS^ tile and puts the staging right after the tiles
  // (1024-aligned without padding) to fit in 227 KB.
  static constexpr int kDqBox = 32 * 32 * 4;
  static constexpr int kDqBoxes = 1;
  static constexpr int kDqRounds = (D / 32) / kDqBoxes;
  static constexpr int kDqBufs = FINE ? 1 : 2;
  static constexpr int kDqWarp = kDqBufs * kDqBoxes * kDqBox;  // per drain warp
  static constexpr int kSmall = FINE ? kDSq + kBlk * kBlk + 4 * kDqWarp : kDSq;  // the small arrays start here
  static constexpr int kRed = kSmall;                         // [2][8] floats (cross-warp max)
  static constexpr int kScl = kRed + 64;                      // [4][2] floats {s_P, s_dS} per tile slot
  static constexpr int kRowSum = kScl + 32;                   // [2 slots][2 wg][128] int (Q-smoothing colsum of dS^)
  static constexpr int kRowX = kRowSum + 4 * kBlk * 4;         // [P, dS][2 wg][128] per-row maxima (exchange)
  static constexpr int kSpRow = kRowX + (FINE ? 2 : 1) * 2 * kBlk * 4;  // [4 slots][128] per-key psi(P) maxima
  static constexpr int kSpK = kSpRow + 4 * kBlk * 4;           // FINE: [4 slots][128] per-key dS maxima (dK)
  static constexpr int kSpQ = kSpK + (FINE ? 4 * kBlk * 4 : 0);  // FINE: [4 slots][128] per-query dS maxima (dQ)
  static constexpr int kColMax = kSpQ + (FINE ? 4 * kBlk * 4 : 0);  // FINE: [2 wg][4 warps][64] column maxima
  static constexpr int kInvQ = kColMax + (FINE ? 2 * 4 * 64 * 4 : 0);  // FINE: [2 wg][64] per-query inverses
  // s_Q[bh][0..T), s_dO[bh][0..T) staged in smem (T <= kMaxT); FINE reads them from global instead
  static constexpr int kScQ = kInvQ + (FINE ? 2 * 64 * 4 : 0);
  static constexpr int kScDO = kScQ + (FINE ? 0 : kMaxT * 4);
  static constexpr int kDq = FINE ? kDSq + kBlk * kBlk : (kScDO + kMaxT * 4 + 1023) / 1024 * 1024;
  static constexpr int kBar = FINE ? kScDO : kDq + 4 * kDqWarp;
  static constexpr int kNumBars = 1 + 2 * kStages + 14;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmemSlot + 16;
  static constexpr int kAlloc = kBytes + 1024;
  static constexpr uint32_t kStageTx = kSplitDO ? 2 * kTile + 1024 : 4 * kTile + 1024;  // + D*4 with mu_Q
  static constexpr uint32_t kDOTx = 2 * kTile;
  static_assert(kAlloc <= 232448, "K4 shared memory exceeds the 227 KB per-CTA limit");
};

// Profiling hooks (timeline + ablation switches) exist only in the SAGE_TRACE=1 build
// (libsage_trace.so); the production library compiles them out.
#ifndef SAGE_K4_RP
#define SAGE_K4_RP 56
#endif
#ifndef SAGE_K4_RC64
#define SAGE_K4_RC64 136  // 144 spilled (68 B STL per thread) for a within-noise gain: kept at 136
#endif
#ifndef SAGE_K4_RC128
#define SAGE_K4_RC128 120  // ptxas spills at 128 (20 B / 124 B per thread), none at 120
#endif
#ifndef SAGE_K4_DKQ128
#define SAGE_K4_DKQ128 1  // d=128: dK shares the dQ region (1) or dP's (0, round 1)
#endif
#ifndef SAGE_K4_DVDP
#define SAGE_K4_DVDP 0  // d=128: the dV tile on dP's columns, so S_{i+1} goes out as soon as S_i is in
                        // registers (1; C4 K4 +1.4%, C3 -1.6%: DESIGN.md 7.3), or on S's (0)
#endif
#ifndef SAGE_K4_EXPIPE
#define SAGE_K4_EXPIPE 1  // P = 2^t for the first 32 columns before the tile-max barrier and the dP wait, the
                          // second 32 interleaved with the first chunk's dS work (0: each chunk's 32 after its dP load)
#endif
#ifndef SAGE_K4_TAIL_MAXT
#define SAGE_K4_TAIL_MAXT 32  // d=128, T <= this (N <= 4K): the TAIL instantiation (below), where the CTA's tail is a
                              // large share of its time (measured: S1K K4 -3.7%, S2K -2.4%; at C4 its extra
                              // register pressure costs +1%, so long sequences keep the plain kernel)
#endif
#ifndef SAGE_K4_DETDEFER
#define SAGE_K4_DETDEFER 1  // SAGE_DETERMINISTIC, causal: a drain warp hands on its dQ turn at its next tile (its reduce
                            // has completed by then) instead of waiting for the reduce right after issuing it
                            // (measured: C4 K4 15.14 -> 13.52 ms; the non-causal rotated order, where the next
                            // contributor is exactly one tile behind, gets slower: C2 0.748 -> 0.774 ms, so off there)
#endif
#ifndef SAGE_K4_HGROUP
#define SAGE_K4_HGROUP 4  // CTA order: groups of this many heads, within a group key block j major (all the
                          // group's j = 0 CTAs, then j = 1, ...): longest-first across the group while only a few
                          // heads' Q^/dO^/dO tiles are in flight (L2 reuse); 1 = head-major
#endif
#ifndef SAGE_TRACE
#define SAGE_TRACE 0
#endif
// Profiling-only timeline (SAGE_ABLATE bit 8): clock64 stamps of pipeline events for the
// first kTrCtas CTAs, read back with sage_debug_trace().  One predicated branch per event.
constexpr int kTrCtas = 4, kTrTiles = 64, kTrEvents = 24;
__device__ unsigned long long g_trace[kTrCtas * kTrTiles * kTrEvents];
#define TR(ev, it)                                                                  \
  do {                                                                              \
    if (SAGE_TRACE && (ablate & 8) && blockIdx.x < kTrCtas && (it) < kTrTiles)      \
      g_trace[(blockIdx.x * kTrTiles + (it)) * kTrEvents + (ev)] = clock64();       \
  } while (0)

// Test-only tile dump (SAGE_ABLATE bit 16, libsage_trace.so; sage_debug_dump): the compute
// warps write P^^T, dS^^T (int8) and the pre-psi dS^T (fp32) as [head][N kv][N q], and the tile
// scales s_P, s_dS as [head][T i][T j], for heads bh < g_dump.heads (Tier C, fidelity reports).
__device__ BwdDump g_dump;
#define DUMPING (SAGE_TRACE && (ablate & 16) && bh < g_dump.heads && dump_ok)
// ... and the int32 accumulators (sage_debug_dump_acc): S^T [head][N kv][N q], the dV / dK tiles
// [head][T i][N kv][D], the dQ tiles [head][T j][N q][D], each before any scaling
struct BwdDumpAcc {
  int32_t *s_t, *dv, *dk, *dq;
  float* dp;  // dP^T = V_j dO_i^T as the kind::f16 MMA left it (fp32), [head][N kv][N q]
};
__device__ BwdDumpAcc g_dacc;
__device__ __forceinline__ void dump_words(int32_t* dst, const uint32_t* v, int n) {
  for (int e = 0; e < n; e += 4) *reinterpret_cast<uint4*>(dst + e) = make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
}

// Order-preserving float <-> int map (monotone for all finite values and +-inf), so a float max is
// one redux.sync.max.s32 instead of five shuffles.
__device__ __forceinline__ int ford(float x) {
  const int b = __float_as_int(x);
  return b ^ ((b >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float ford_inv(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }

// max over the 256 compute threads (warps 4-11), named barrier `id`
__device__ __forceinline__ float compute_max(float v, int* red, int cw, int id) {
  const int k = __reduce_max_sync(0xffffffffu, ford(v));
  if ((threadIdx.x & 31) == 0) red[cw] = k;
  named_bar_sync(id, 256);
  const int4 a = *reinterpret_cast<const int4*>(red);
  const int4 b = *reinterpret_cast<const int4*>(red + 4);
  return ford_inv(max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w))));
}

// VAR: 0 the default path, 1 SAGE_DETERMINISTIC, 2 SAGE_P_COLSCALE, 3 SAGE_FINE_BWD (per-key psi(P),
// per-key dS^ for dK, per-query dS^ for dQ) -- separate instantiations, because compiling the
// variants' logic into the default kernel costs 2-8% (measured)
// TAIL: d=128, the compute warps, idle once their last tile is done, store dV_j and drain half of the last
// dQ tile, shortening the CTA's tail (the drain warps keep dK_j and dQ's other half)
template <int D, bool CAUSAL, bool QSMOOTH, int VAR, bool TAIL>
__global__ void __launch_bounds__(kThreads, 1)
    sage_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_doq, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                    const float* __restrict__ q_scale,
                    const float* __restrict__ k_scale, const float* __restrict__ do_scale,
                    const float* __restrict__ l2g, const float* __restrict__ deltag, const float* __restrict__ bias,
                    const float* __restrict__ mu_q, float* __restrict__ dq_acc, void* __restrict__ dk_out,
                    void* __restrict__ dv_out, int N, int BH, float tau, int pu8, int fp16, int f32out,
                    unsigned* __restrict__ dq_flags, IoLayout io, int ablate_arg) {
  constexpr bool fine = VAR == 3;
  constexpr bool pcol = VAR == 2 || fine;
  const int ablate = SAGE_TRACE ? ablate_arg : 0;
  // psi(P) levels (Alg. 2 line 6): 127, or 255 for the unsigned P^ variant (SAGE_P_U8)
  const float pmax = pu8 ? 255.f : 127.f;
  using L = BwdSmem<D, VAR == 3>;
  constexpr int kStages = L::kStages;
  constexpr bool kAlias = D == 128;
  // setmaxnreg budgets (x128 threads each; sum = 512 regs/thread-slot = the 64K register file)
  // setmaxnreg budget per warpgroup (sums to 4 x 128): producer/MMA, 2 x compute, drain gets the rest
  constexpr uint32_t kRegProducer = SAGE_K4_RP, kRegCompute = D == 64 ? SAGE_K4_RC64 : SAGE_K4_RC128,
                     kRegDrain = 512 - kRegProducer - 2 * kRegCompute;
  static_assert(kRegProducer % 8 == 0 && kRegCompute % 8 == 0 && kRegDrain % 8 == 0, "setmaxnreg needs multiples of 8");
  static_assert(kRegProducer >= 24 && kRegCompute <= 256 && kRegDrain >= 24 && kRegDrain <= 256,
                "setmaxnreg values must lie in [24, 256]");
  static_assert(kRegProducer + 2 * kRegCompute + kRegDrain == 512, "the four warpgroups share 512 registers/slot");
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by offsetting the __shared__ array itself, so every
  // derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;             // [kStages]
  uint64_t* q_empty = q_full + kStages;    // [kStages]
  uint64_t* b0 = q_empty + kStages;
  // MMA -> compute / drain (tcgen05.commit).  dv_full also tells the compute warps that P^^T
  // may be overwritten, dkq_full that dS^^T may be; each completes once per tile and no waiter
  // can fall a full phase behind (checked per wait below), so one barrier serves both.
  uint64_t* s_full = b0 + 0;
  uint64_t* dp_full = b0 + 1;
  uint64_t* dv_full = b0 + 2;
  uint64_t* dkq_full = b0 + 3;
  uint64_t* p_ready = b0 + 4;      // compute -> MMA (8 warps): P^^T written, S^T read
  uint64_t* ds_ready = b0 + 5;     // compute -> MMA (8 warps): dS^^T written, dP^T read
  uint64_t* dv_drained = b0 + 6;   // drain -> MMA (4 warps)
  uint64_t* dkq_drained = b0 + 7;
  uint64_t* do_full = b0 + 8;      // d=128 dO buffer: TMA -> MMA
  uint64_t* do_empty = b0 + 9;     // d=128 dO buffer: MMA (dP done) -> TMA
  uint64_t* dq_drained = b0 + 10;  // drain -> MMA (4 warps): dQ tile read (dkq_drained: dK tile read)
  uint64_t* v_tmem = b0 + 11;      // compute -> MMA (8 warps): V_j copied into TMEM (d=64)
  uint64_t* s_free = b0 + 12;      // compute -> MMA (8 warps): S^T read into registers (d=64)
  uint64_t* dk_full = b0 + 13;     // d=128: MMA -> drain, the dK tile (dkq_full then marks the dQ tile,
                                   // issued after it: both have read dS^^T)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  int* red = reinterpret_cast<int*>(smem + L::kRed);
  float* scl = reinterpret_cast<float*>(smem + L::kScl);
  float* sc_q_s = reinterpret_cast<float*>(smem + L::kScQ);
  float* sc_do_s = reinterpret_cast<float*>(smem + L::kScDO);
  int* rowsum_s = reinterpret_cast<int*>(smem + L::kRowSum);
  float* rowx = reinterpret_cast<float*>(smem + L::kRowX);
  float* sp_row = reinterpret_cast<float*>(smem + L::kSpRow);
  float* sp_k = reinterpret_cast<float*>(smem + L::kSpK);     // FINE
  float* sp_q = reinterpret_cast<float*>(smem + L::kSpQ);     // FINE
  int* colmax = reinterpret_cast<int*>(smem + L::kColMax);    // FINE
  float* invq_s = reinterpret_cast<float*>(smem + L::kInvQ);  // FINE

  // N need not be a multiple of 128 (reading A33): T blocks, the library's tiles padded to Np rows per head
  const int T = num_blocks(N), Np = T * kBlk;
  const bool dump_ok = N == Np;  // the tile dumps (test build) are laid out for N % 128 == 0 only
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t one = blockDim.x / kThreads;  // a runtime 1 (i2f2 on the FMA pipe, SAGE_I2F_FMA)
  const int tile = blockIdx.x;
  // CTA order: heads in groups of SAGE_K4_HGROUP, within a group low j (most query blocks when causal) first
  // across its heads, so the group's CTAs share its Q^/dO/dO^ tiles and dQ rows through L2 and the longest
  // CTAs never start in the grid's last wave (SAGE_DETERMINISTIC keeps one head at a time, see below).
  constexpr int kHG = VAR == 1 ? 1 : SAGE_K4_HGROUP;
  const int grp = tile / (kHG * T), g_heads = min(kHG, BH - grp * kHG), within = tile - grp * kHG * T;
  const int bh = grp * kHG + within % g_heads;
  // SAGE_DETERMINISTIC (dq_flags != null): dQ_i receives its key-block contributions in a fixed order,
  // enforced with per-(head, i, drain warp) flags.  Causal: descending j (j = i first), so the CTAs
  // launch high j first and every CTA only waits on CTAs launched before it.  Non-causal: CTA j
  // visits the query blocks rotated, i = (j + it) mod T, and dQ_i's contributions come in iteration
  // order; all T CTAs of a head are co-resident (the API requires T <= SM count).
  constexpr bool det = VAR == 1;
  constexpr bool kDetDefer = det && CAUSAL && SAGE_K4_DETDEFER;
  const int j = (det && CAUSAL) ? T - 1 - tile % T : (kHG == 1 ? tile % T : within / g_heads);
  const int i0 = CAUSAL ? j : 0;
  const int n_it = T - i0;
  auto i_of = [&](int it) { return (det && !CAUSAL) ? (j + it) % T : i0 + it; };
  const int krow = bh * Np + j * kBlk;
  const int kv_valid = N - j * kBlk;  // keys of this block (< 128 only in a ragged N's last block)

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    // a stage is released by the dK/dQ MMA commit, and (when it carries mu_Qi) by the drain
    // warps once their dK drain has read mu_Qi
    constexpr uint32_t kEmptyCount = (L::kSplitDO && QSMOOTH) ? 1 + kDrainWarps : 1;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(q_full + s, 1);
      mbar_init(q_empty + s, kEmptyCount);
    }
    for (int b = 0; b < 4; ++b) mbar_init(b0 + b, 1);
    mbar_init(dk_full, 1);
    for (int b = 4; b < 6; ++b) mbar_init(b0 + b, kComputeWarps);
    // d=128: the compute warps drain the dV tile (it aliases S, so draining it gates S_{i+1})
    mbar_init(dv_drained, kAlias ? kComputeWarps : kDrainWarps);
    mbar_init(dkq_drained, kDrainWarps);
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(dq_drained, kDrainWarps);
    mbar_init(v_tmem, kComputeWarps);
    mbar_init(s_free, kComputeWarps);
    fence_mbar_init();
  }
  // per-block scales s_Q, s_dO of this head: staged in smem (FINE, short of smem: read from global)
  const float* sc_q = fine ? q_scale + (size_t)bh * T : sc_q_s;
  const float* sc_do = fine ? do_scale + (size_t)bh * T : sc_do_s;
  for (int t = threadIdx.x; !fine && t < T; t += kThreads) {
    sc_q_s[t] = q_scale[(size_t)bh * T + t];
    sc_do_s[t] = do_scale[(size_t)bh * T + t];
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;
  const uint32_t tDP = tmem + 128;
  constexpr bool kDvDp = kAlias && SAGE_K4_DKQ128 && SAGE_K4_DVDP;
  constexpr bool kTail = TAIL && (VAR == 0 || VAR == 2) && (!kAlias || (SAGE_K4_DKQ128 && !kDvDp));
  const uint32_t tDV = kAlias ? (kDvDp ? tmem + 128 : tmem) : tmem + 256;
  // d=128: dK_i and then dQ_i take turns in the third region, so dP_{i+1} never waits for the dK drain
  constexpr bool kDkQ = kAlias && SAGE_K4_DKQ128;
  const uint32_t tDK = kAlias ? (kDkQ ? tmem + 256 : tmem + 128) : tmem + 256 + D;
  const uint32_t tDQ = kAlias ? tmem + 256 : tmem + 256 + 2 * D;
  const uint32_t tDVacc = tmem + 384;  // d=128 only
  // d=64: the A operands of dP^T (V_j, bf16) and dV (P^^T, int8) live in TMEM ("TS" MMAs), which
  // takes 48 KB/tile of operand reads and P^ stores off the shared-memory port
  constexpr bool kTS = D == 64;
  const uint32_t tVa = tmem + 448;  // V_j bf16 [128][64]: 32 columns
  const uint32_t tPa = tmem + 480;  // P^^T int8 [128 kv][128 q]: 32 columns

  if (warp < 4) {
    reg_set<kRegProducer, 65536 / kThreads>();
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer (one elected lane)
      if (elect_one()) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_doq);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_do);
        mbar_expect_tx(kv_full, 3 * L::kTile);
        tma_load_2d(smem + L::kK, &tm_k, kv_full, 0, krow);
#pragma unroll
        for (int p = 0; p < D / 64; ++p)
          tma_load_4d(smem + L::kV + p * 16384, &tm_v, kv_full, p * 64, j * kBlk, bh % io.H, bh / io.H);
      }
      __syncwarp();
      for (int it = 0; it < n_it; ++it) {
        const int s = it % kStages, i = i_of(it);
        const int qrow = bh * Np + i * kBlk;
        uint8_t* st = smem + L::kStage + s * L::kStageBytes;
        mbar_wait(q_empty + s, ((it / kStages) & 1) ^ 1);
        if (elect_one()) {
          TR(14, it);
          const bool mu_in_stage = L::kSplitDO && QSMOOTH;
          mbar_expect_tx(q_full + s, L::kStageTx + (mu_in_stage ? D * 4 : 0));
          if (mu_in_stage) bulk_load(st + L::kSMu, mu_q + ((size_t)bh * T + i) * D, D * 4, q_full + s);
          tma_load_2d(st + L::kSQ, &tm_q, q_full + s, 0, qrow);
          if constexpr (!L::kSplitDO) {
#pragma unroll
            for (int p = 0; p < D / 64; ++p)
              tma_load_4d(st + L::kSDO + p * 16384, &tm_do, q_full + s, p * 64, i * kBlk, bh % io.H, bh / io.H);
          }
          tma_load_2d(st + L::kSDOQ, &tm_doq, q_full + s, 0, qrow);
          bulk_load(st + L::kSL, l2g + qrow, 512, q_full + s);
          bulk_load(st + L::kSDelta, deltag + qrow, 512, q_full + s);
        }
        __syncwarp();
        if constexpr (L::kSplitDO) {
          mbar_wait(do_empty, (it & 1) ^ 1);  // dP_{it-1} has read the dO buffer
          if (elect_one()) {
            mbar_expect_tx(do_full, L::kDOTx);
#pragma unroll
            for (int p = 0; p < D / 64; ++p)
              tma_load_4d(smem + L::kDO + p * 16384, &tm_do, do_full, p * 64, i * kBlk, bh % io.H, bh / io.H);
          }
          __syncwarp();
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (whole warp, one elected lane issues)
      constexpr uint32_t kIdS = idesc_i8(128, 128, false, false);     // S^T
      const uint32_t kIdDP = idesc_bf16(128, 128, false, false, fp16 != 0);  // dP^T (bf16 or fp16 V, dO)
      constexpr uint32_t kIdDV = idesc_i8(128, D, false, true);       // dK (B MN-major)
      const uint32_t kIdDVp = pu8 ? idesc_i8(128, D, false, true, true) : kIdDV;  // dV: A = P^^T, s8 or u8
      constexpr uint32_t kIdDQ = idesc_i8(128, D, true, true);        // dQ (A, B MN-major)
      // smem operand addresses; descriptors are formed at issue time (cheap uniform-datapath ALU)
      const uint32_t st0 = smem_u32(smem + L::kStage);
      const uint32_t k_addr = smem_u32(smem + L::kK);
      const uint32_t v_addr = smem_u32(smem + L::kV);
      const uint32_t pt_addr = smem_u32(smem + L::kPt);
      const uint32_t dst_addr = smem_u32(smem + L::kDSt);
      const uint32_t dsq_addr = smem_u32(smem + (fine ? L::kDSq : L::kDSt));  // FINE: the per-query dS^
      auto soff = [&](int it) { return (uint32_t)((it % kStages) * L::kStageBytes); };
      auto issue_s = [&](int it) {
        mbar_wait(q_full + it % kStages, (it / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          TR(22, it);
          const uint32_t q_addr = st0 + soff(it) + L::kSQ;
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk)
            mma_i8(tS, desc_kmajor(k_addr, D, kk * 32), desc_kmajor(q_addr, D, kk * 32), kIdS, kk > 0);
          mma_commit(s_full);
          TR(0, it);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int it) {  // stage `it` was already waited for by issue_s(it)
        if constexpr (L::kSplitDO) {
          mbar_wait(do_full, it & 1);
          tc_fence_after();
        }
        if (elect_one()) {
          const uint32_t do_addr = L::kSplitDO ? smem_u32(smem + L::kDO) : st0 + soff(it) + L::kSDO;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            if constexpr (kTS)
              mma_bf16_ts(tDP, tVa + kk * 8, desc_kmajor(do_addr + off, 128, 0), kIdDP, kk > 0);
            else
              mma_bf16(tDP, desc_kmajor(v_addr + off, 128, 0), desc_kmajor(do_addr + off, 128, 0), kIdDP, kk > 0);
          }
          mma_commit(dp_full);
          if constexpr (L::kSplitDO) mma_commit(do_empty);
          TR(2, it);
        }
        __syncwarp();
      };
      auto issue_dv = [&](int it) {
        if (elect_one()) {
          const uint32_t doq_addr = st0 + soff(it) + L::kSDOQ;
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk) {
            if constexpr (kTS)
              mma_i8_ts(tDV, tPa + kk * 8, desc_mnmajor(doq_addr, D, kk * 32), kIdDVp, kk > 0);
            else
              mma_i8(tDV, desc_kmajor(pt_addr, 128, kk * 32), desc_mnmajor(doq_addr, D, kk * 32), kIdDVp, kk > 0);
          }
          mma_commit(dv_full);
          TR(1, it);
        }
        __syncwarp();
      };
      auto issue_dkdq = [&](int it) {
        if (elect_one()) {
          const uint32_t q_addr = st0 + soff(it) + L::kSQ;
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk)
            mma_i8(tDK, desc_kmajor(dst_addr, 128, kk * 32), desc_mnmajor(q_addr, D, kk * 32), kIdDV, kk > 0);
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk)
            mma_i8(tDQ, desc_mnmajor(dsq_addr, 128, kk * 32), desc_mnmajor(k_addr, D, kk * 32), kIdDQ, kk > 0);
          mma_commit(dkq_full);
          mma_commit(q_empty + it % kStages);
          TR(3, it);
        }
        __syncwarp();
      };
      // d=128: dK_i and then (once drained) dQ_i in the same TMEM region
      auto issue_dk = [&](int it) {
        if (elect_one()) {
          const uint32_t q_addr = st0 + soff(it) + L::kSQ;
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk)
            mma_i8(tDK, desc_kmajor(dst_addr, 128, kk * 32), desc_mnmajor(q_addr, D, kk * 32), kIdDV, kk > 0);
          mma_commit(dk_full);
          mma_commit(q_empty + it % kStages);  // Q^_i was the stage's last MMA operand
          TR(3, it);
        }
        __syncwarp();
      };
      auto issue_dq = [&](int it) {
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kBlk / 32; ++kk)
            mma_i8(tDQ, desc_mnmajor(dsq_addr, 128, kk * 32), desc_mnmajor(k_addr, D, kk * 32), kIdDQ, kk > 0);
          mma_commit(dkq_full);  // dQ_i ready; with dK_i before it, dS^^T has been read
          TR(4, it);
        }
        __syncwarp();
      };
      mbar_wait(kv_full, 0);
      issue_s(0);
      if constexpr (kTS) mbar_wait(v_tmem, 0);
      issue_dp(0);
      for (int it = 0; it < n_it; ++it) {
        const uint32_t ph = it & 1, pph = ph ^ 1;
        const bool more = it + 1 < n_it;
        if constexpr (!kAlias) {
          // compute events per tile: s_free (S^T in registers) < p_ready (dP^T read; P^^T
          // written) < ds_ready (dS^^T written).  S_{i+1} goes out as soon as S_i is read, dP_{i+1}
          // right behind dV_i, so the next tile's operands are ready when the compute gets there.
          if (more) {
            mbar_wait(s_free, ph);
            tc_fence_after();
            issue_s(it + 1);
          }
          mbar_wait(p_ready, ph);
          if (it > 0) mbar_wait(dv_drained, pph);
          if (lane == 0) TR(17, it);
          tc_fence_after();
          issue_dv(it);
          if (more) issue_dp(it + 1);
          mbar_wait(ds_ready, ph);
          if (it > 0) {
            mbar_wait(dkq_drained, pph);
            mbar_wait(dq_drained, pph);
          }
          if (lane == 0) TR(20, it);
          tc_fence_after();
          issue_dkdq(it);
        } else if constexpr (!kDkQ) {
          // d=128 (round 1): dV_i lands on S's columns, dK_i on dP's (both read by p_ready)
          mbar_wait(p_ready, ph);
          tc_fence_after();
          issue_dv(it);
          mbar_wait(ds_ready, ph);
          if (it > 0) mbar_wait(dq_drained, pph);
          tc_fence_after();
          issue_dkdq(it);
          if (more) {
            mbar_wait(dv_drained, ph);
            tc_fence_after();
            issue_s(it + 1);
            mbar_wait(dkq_drained, ph);
            tc_fence_after();
            issue_dp(it + 1);
          }
        } else if constexpr (kDvDp) {
          // d=128 (SAGE_K4_DVDP): S_{i+1} goes out once S_i is in registers (s_free); dV_i lands on
          // dP's columns (read by p_ready), so dP_{i+1} waits for the compute warps' dV drain.
          if (more) {
            mbar_wait(s_free, ph);
            tc_fence_after();
            issue_s(it + 1);
          }
          mbar_wait(p_ready, ph);
          if (lane == 0) TR(17, it);
          tc_fence_after();
          issue_dv(it);
          mbar_wait(ds_ready, ph);
          if (it > 0) mbar_wait(dq_drained, pph);  // dQ_{i-1} drained out of the third region
          if (lane == 0) TR(20, it);
          tc_fence_after();
          issue_dk(it);
          if (more) {
            mbar_wait(dv_drained, ph);
            tc_fence_after();
            issue_dp(it + 1);
          }
          mbar_wait(dkq_drained, ph);  // dK_i drained
          tc_fence_after();
          issue_dq(it);
        } else {
          // d=128: dV_i lands on S's columns (read by p_ready), so S_{i+1} waits until the compute
          // warps have drained dV_i; dP_{i+1} goes out right behind dV_i (dP_i was read by p_ready).
          // dK_i and then dQ_i take turns in the third region.
          mbar_wait(p_ready, ph);
          if (lane == 0) TR(17, it);
          tc_fence_after();
          issue_dv(it);
          if (more) issue_dp(it + 1);
          mbar_wait(ds_ready, ph);
          if (it > 0) mbar_wait(dq_drained, pph);  // dQ_{i-1} drained out of the third region
          if (lane == 0) TR(20, it);
          tc_fence_after();
          issue_dk(it);
          if (more) {
            mbar_wait(dv_drained, ph);
            tc_fence_after();
            issue_s(it + 1);
          }
          mbar_wait(dkq_drained, ph);  // dK_i drained
          tc_fence_after();
          issue_dq(it);
        }
      }
    }
  } else if (warp < 4 + kComputeWarps) {
    reg_set<kRegCompute, 65536 / kThreads>();
    // ------------------------------------------------------------ compute warpgroups (256 threads)
    const int cw = warp - 4;                 // compute warp 0..7
    const int wg = cw / 4;
    const int r = (warp % 4) * 32 + lane;    // TMEM lane = key row of S^T / dP^T
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    const int qc0 = wg * 64;                 // this warpgroup's query columns of the tile
    const float tau2 = tau * kLog2e;
    const float sk = k_scale[(size_t)bh * T + j];
    uint8_t* pt = smem + L::kPt;
    uint8_t* dst = smem + L::kDSt;
    if constexpr (kTS) {
      // V_j row r (this warpgroup's 64 bytes) from the swizzled smem panel into TMEM (A of dP^T)
      mbar_wait(kv_full, 0);
      uint32_t w[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 x = *reinterpret_cast<const uint4*>(smem + L::kV + sw_offset(r, wg * 4 + c, 128));
        w[4 * c] = x.x;
        w[4 * c + 1] = x.y;
        w[4 * c + 2] = x.z;
        w[4 * c + 3] = x.w;
      }
      tmem_st16(tVa + wg * 16 + lane_off, w);
      tmem_wait_st();
      tc_fence_before();
      warp_arrive(v_tmem);
    }

    for (int it = 0; it < n_it; ++it) {
      const int i = i_of(it), s = it % kStages;
      const uint32_t ph = it & 1, pph = ph ^ 1;
      const uint8_t* st = smem + L::kStage + s * L::kStageBytes;
      const float4* Ls4 = reinterpret_cast<const float4*>(st + L::kSL) + qc0 / 4;
      const float4* Ds4 = reinterpret_cast<const float4*>(st + L::kSDelta) + qc0 / 4;
      const float c2 = sc_q[i] * sk * tau2;  // int32 -> log2-domain logit
      const float b2 = QSMOOTH ? bias[((size_t)bh * T + i) * Np + (size_t)j * kBlk + r] * tau2 : 0.f;
      const bool diag = CAUSAL && (i == j);
      const bool cm = !(ablate & 2);
      float t[64];
#pragma unroll
      for (int e = 0; e < 64; ++e) t[e] = 0.f;

      // -- step 1: t = log2 P = S*c2 + b2 - L2[q]  (Alg. 2 line 5), tile max of t
      mbar_wait(q_full + s, (it / kStages) & 1);
      mbar_wait(s_full, ph);
      tc_fence_after();
      if (threadIdx.x == 128) TR(5, it);
      float tmax = -INFINITY;
if (cm) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t v[32];
        tmem_ld32(tS + qc0 + cc * 32 + lane_off, v);
        tmem_wait_ld();
        if (threadIdx.x == 128 && cc == 0) TR(16, it);
        if (DUMPING && g_dacc.s_t)
          dump_words(g_dacc.s_t + ((size_t)bh * N + j * kBlk + r) * N + i * kBlk + qc0 + cc * 32, v, 32);
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          float4 l4 = Ls4[cc * 8 + e4];
          float2 a = i2f2(v[4 * e4], v[4 * e4 + 1], one);
          float2 b = i2f2(v[4 * e4 + 2], v[4 * e4 + 3], one);
          float2 na = make_float2(-l4.x, -l4.y), nb = make_float2(-l4.z, -l4.w);
          if constexpr (QSMOOTH) {
            na = fadd2(na, make_float2(b2, b2));
            nb = fadd2(nb, make_float2(b2, b2));
          }
          a = ffma2(a, make_float2(c2, c2), na);
          b = ffma2(b, make_float2(c2, c2), nb);
          const int e = cc * 32 + 4 * e4;
          t[e] = a.x;
          t[e + 1] = a.y;
          t[e + 2] = b.x;
          t[e + 3] = b.y;
        }
      }
}
      if (threadIdx.x == 128) TR(18, it);
      tc_fence_before();
      if constexpr (!kAlias || kDvDp) warp_arrive(s_free);  // S^T consumed: S_{i+1} may be issued
      if (diag) {  // causal: key r attends query q only if r <= q (reading A14)
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (r > qc0 + e) t[e] = -INFINITY;
      }
      // A key row the short last block of a ragged N lacks (A33; the missing queries have L = +inf, so
      // their P is 0): its K^ and V rows are zero, so its P, dS reach dQ only through K^ = 0 and its own dV,
      // dK rows, which are not written.  It must only stay out of the tile maxima (s_P, s_dS): its
      // row max is dropped here and its |dS| max below (FINE: its per-query dS maxima need the full mask)
      const bool kv_missing = r >= kv_valid;
      if (fine && kv_missing) {
#pragma unroll
        for (int e = 0; e < 64; ++e) t[e] = -INFINITY;
      }
#pragma unroll
      for (int e = 0; e < 64; e += 4) tmax = fmaxf(tmax, fmax3(t[e], t[e + 1], fmaxf(t[e + 2], t[e + 3])));
      if (kv_missing) tmax = -INFINITY;
      if constexpr (SAGE_K4_EXPIPE) {
        // P = 2^t does not depend on the tile max: the first chunk's exponentials overlap the barrier below
        // and the dP wait
#pragma unroll
        for (int u = 0; u < (SAGE_K4_EXPIPE == 2 ? 64 : 32); ++u) t[u] = ex2(t[u]);
      }

      // -- step 2: psi(P) scale over the tile: amax = max P = 2^max(t)  (line 6, reading A11)
      if (threadIdx.x == 128) TR(19, it);
      // SAGE_P_COLSCALE: one scale per key row r of P^T (a key column of P, the dV contraction's free
      // index), the max over this tile's 128 queries: this thread's 64 and the other warpgroup's 64
      float amax_p;
      if constexpr (pcol) {
        rowx[wg * kBlk + r] = tmax;
        named_bar_sync(1, 256);
        amax_p = ex2(fmaxf(tmax, rowx[(wg ^ 1) * kBlk + r]));
        if (wg == 0) sp_row[(it & 3) * kBlk + r] = amax_p;
      } else {
        amax_p = ex2(compute_max(tmax, red, cw, 1));
      }
      if (threadIdx.x == 128) TR(21, it);
      // inv = 127/amax via the correctly rounded reciprocal (within 1 ulp of fl32(127/amax); P^ is
      // Tier C); the exact s_P = fl32(amax/127) is formed by the drain off this path
      const float inv_p = amax_p > 0.f ? __fmul_rn(pmax, __frcp_rn(amax_p)) : 0.f;
      // tile scales for the drain warpgroup (4 slots: it cannot run 4 tiles ahead of the drain)
      if (threadIdx.x == 128) scl[(it & 3) * 2] = amax_p;

      // -- step 3: P = 2^t, P^ = RNE(P * inv) -> P^^T smem (A of dV, K-major);
      //            dS = P o (dP - delta) (lines 8-9) in the same pass, tile max |dS|
      // P^^T may be overwritten once dV_{i-1} has read it: dP_i is issued after dV_{i-1} and a
      // tcgen05.commit tracks every earlier MMA of the issuing thread, so dp_full(i) implies it
      mbar_wait(dp_full, ph);
      tc_fence_after();
      if (threadIdx.x == 128) TR(15, it);
      float dsmax = 0.f;
      uint32_t pw[16];  // this thread's P^ row slice (64 int8) for the TMEM A operand of dV
if (cm) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t v[32];
        tmem_ld32(tDP + qc0 + cc * 32 + lane_off, v);
        if constexpr (!SAGE_K4_EXPIPE) {
          // the chunk's 32 exponentials first: back-to-back MUFU work while the TMEM load lands
#pragma unroll
          for (int u = 0; u < 32; ++u) t[cc * 32 + u] = ex2(t[cc * 32 + u]);
        }
        tmem_wait_ld();
        if (DUMPING && g_dacc.dp)
          dump_words(reinterpret_cast<int32_t*>(g_dacc.dp) + ((size_t)bh * N + j * kBlk + r) * N + i * kBlk + qc0 + cc * 32,
                     v, 32);
#pragma unroll
        for (int c16 = 0; c16 < 2; ++c16) {
          uint32_t w[4];
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int ev = c16 * 16 + e4 * 4;  // index into v
            const int e = cc * 32 + ev;        // index into t
            if (SAGE_K4_EXPIPE == 1 && cc == 0) {  // the second chunk's exponentials, 4 per group of this one
#pragma unroll
              for (int u = 0; u < 4; ++u) t[32 + ev + u] = ex2(t[32 + ev + u]);
            }
            const float4 d4 = Ds4[e / 4];
            float2 qa = ffma2(make_float2(t[e], t[e + 1]), make_float2(inv_p, inv_p), make_float2(kMagic, kMagic));
            float2 qb = ffma2(make_float2(t[e + 2], t[e + 3]), make_float2(inv_p, inv_p), make_float2(kMagic, kMagic));
            w[e4] = pack4_magic(qa.x, qa.y, qb.x, qb.y);
            float2 a = fadd2(make_float2(__uint_as_float(v[ev]), __uint_as_float(v[ev + 1])), make_float2(-d4.x, -d4.y));
            float2 b = fadd2(make_float2(__uint_as_float(v[ev + 2]), __uint_as_float(v[ev + 3])), make_float2(-d4.z, -d4.w));
            a = fmul2(a, make_float2(t[e], t[e + 1]));
            b = fmul2(b, make_float2(t[e + 2], t[e + 3]));
            t[e] = a.x;
            t[e + 1] = a.y;
            t[e + 2] = b.x;
            t[e + 3] = b.y;
            dsmax = fmax3(dsmax, fabsf(a.x), fmax3(fabsf(a.y), fabsf(b.x), fabsf(b.y)));
          }
          if (DUMPING)
            *reinterpret_cast<uint4*>(g_dump.pt + ((size_t)bh * N + j * kBlk + r) * N + i * kBlk + qc0 + cc * 32 +
                                      c16 * 16) = make_uint4(w[0], w[1], w[2], w[3]);
          if constexpr (kTS) {
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) pw[cc * 8 + c16 * 4 + e4] = w[e4];
          } else {
            *reinterpret_cast<uint4*>(pt + sw_offset(r, (qc0 + cc * 32) / 16 + c16, 128)) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
}
      if (threadIdx.x == 128) TR(23, it);
      if constexpr (kTS) {
        tmem_st16(tPa + wg * 16 + lane_off, pw);
        tmem_wait_st();
      } else {
        fence_proxy_async_smem();
      }
      tc_fence_before();
      warp_arrive(p_ready);  // P^^T written; S^T and dP^T read (their TMEM columns may be reused)
      if (threadIdx.x == 128) TR(6, it);

      if (kv_missing) dsmax = 0.f;
      // -- step 5: psi(dS) scale over the tile (FINE: one per key row for dK, one per query for dQ)
      float amax_ds;
      if constexpr (fine) {
        // per key: this thread's 64 queries and the other warpgroup's 64 (second exchange slot)
        rowx[2 * kBlk + wg * kBlk + r] = dsmax;
        // per query: the max of |dS| over this warpgroup's 128 key rows, column by column
        // (|x| as int is monotone), one redux per column and warp, lane 0 keeps the 64 results
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const int m = __reduce_max_sync(0xffffffffu, __float_as_int(fabsf(t[c])));
          if (lane == 0) colmax[(wg * 4 + (warp % 4)) * 64 + c] = m;
        }
        named_bar_sync(2, 256);
        amax_ds = fmaxf(dsmax, rowx[2 * kBlk + (wg ^ 1) * kBlk + r]);
        if (wg == 0) sp_k[(it & 3) * kBlk + r] = amax_ds;
        const int tw = threadIdx.x - 128 - wg * 128;  // 0..127 within the warpgroup
        if (tw < 64) {
          const int* cmx = colmax + wg * 4 * 64 + tw;
          const float aq = __int_as_float(max(max(cmx[0], cmx[64]), max(cmx[128], cmx[192])));
          invq_s[wg * 64 + tw] = aq > 0.f ? __fmul_rn(127.f, __frcp_rn(aq)) : 0.f;
          sp_q[(it & 3) * kBlk + qc0 + tw] = aq;
        }
        named_bar_sync(3 + wg, 128);
      } else {
        amax_ds = compute_max(dsmax, red + 8, cw, 2);
      }
      const float inv_ds = amax_ds > 0.f ? __fmul_rn(127.f, __frcp_rn(amax_ds)) : 0.f;
      if (threadIdx.x == 128) scl[(it & 3) * 2 + 1] = amax_ds;
      if (DUMPING) {
        float* dsrow = g_dump.ds + ((size_t)bh * N + j * kBlk + r) * N + i * kBlk + qc0;
#pragma unroll
        for (int e = 0; e < 64; e += 4) *reinterpret_cast<float4*>(dsrow + e) = make_float4(t[e], t[e + 1], t[e + 2], t[e + 3]);
        if (threadIdx.x == 128) {
          g_dump.sp[((size_t)bh * T + i) * T + j] = __fdiv_rn(amax_p, pmax);
          g_dump.sds[((size_t)bh * T + i) * T + j] = __fdiv_rn(amax_ds, 127.f);
        }
      }

      // -- step 6: dS^ = RNE(dS * inv) -> dS^^T smem (A of dK K-major, A of dQ MN-major)
      if (it > 0) mbar_wait(dkq_full, pph);  // dK_{i-1}, dQ_{i-1} have read dS^^T
      if (threadIdx.x == 128) TR(9, it);
      int rsum = 0;
if (cm) {
#pragma unroll
      for (int c16 = 0; c16 < 4; ++c16) {
        uint32_t w[4];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int e = c16 * 16 + e4 * 4;
          float2 qa = ffma2(make_float2(t[e], t[e + 1]), make_float2(inv_ds, inv_ds), make_float2(kMagic, kMagic));
          float2 qb = ffma2(make_float2(t[e + 2], t[e + 3]), make_float2(inv_ds, inv_ds), make_float2(kMagic, kMagic));
          w[e4] = pack4_magic(qa.x, qa.y, qb.x, qb.y);
          if constexpr (QSMOOTH) rsum = __dp4a((int)w[e4], 0x01010101, rsum);
        }
        *reinterpret_cast<uint4*>(dst + sw_offset(r, qc0 / 16 + c16, 128)) = make_uint4(w[0], w[1], w[2], w[3]);
        if constexpr (fine) {  // the dQ operand: the same dS with per-query inverses
          uint32_t wq[4];
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int e = c16 * 16 + e4 * 4;
            const float4 iq = *reinterpret_cast<const float4*>(invq_s + wg * 64 + e);
            float2 qa = ffma2(make_float2(t[e], t[e + 1]), make_float2(iq.x, iq.y), make_float2(kMagic, kMagic));
            float2 qb = ffma2(make_float2(t[e + 2], t[e + 3]), make_float2(iq.z, iq.w), make_float2(kMagic, kMagic));
            wq[e4] = pack4_magic(qa.x, qa.y, qb.x, qb.y);
          }
          *reinterpret_cast<uint4*>(smem + L::kDSq + sw_offset(r, qc0 / 16 + c16, 128)) =
              make_uint4(wq[0], wq[1], wq[2], wq[3]);
        }
        if (DUMPING)
          *reinterpret_cast<uint4*>(g_dump.dst + ((size_t)bh * N + j * kBlk + r) * N + i * kBlk + qc0 + c16 * 16) =
              make_uint4(w[0], w[1], w[2], w[3]);
      }
}
      if constexpr (QSMOOTH) rowsum_s[(it & 1) * kBlk * 2 + wg * kBlk + r] = rsum;
      fence_proxy_async_smem();
      tc_fence_before();
      warp_arrive(ds_ready);
      if (threadIdx.x == 128) TR(8, it);
      if constexpr (kAlias) {
        // d=128: dV_j += tile * s_P * s_dO_i (Alg. 2 line 7) into the fp32 TMEM accumulator, this
        // warpgroup's 64 columns.  The dV tile sits on S's columns, so S_{i+1} waits for this
        // drain; the compute warps are otherwise idle here, and two warpgroups halve it.
        mbar_wait(dv_full, ph);
        tc_fence_after();
        const float s_p = __fdiv_rn(amax_p, pmax);  // psi(P) scale = fl32(amax/127)
        const float sp_do = s_p * sc_do[i];
        const float2 f = make_float2(sp_do, sp_do);
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t v[32], a[32];
          tmem_ld32(tDV + qc0 + c0 + lane_off, v);
          tmem_ld32(tDVacc + qc0 + c0 + lane_off, a);
          tmem_wait_ld();
          if (DUMPING && g_dacc.dv)
            dump_words(g_dacc.dv + (((size_t)bh * T + i) * N + j * kBlk + r) * D + qc0 + c0, v, 32);
          if (it == 0) {
#pragma unroll
            for (int e = 0; e < 32; ++e) a[e] = 0u;
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 x = ffma2(i2f2(v[e], v[e + 1], one), f,
                                   make_float2(__uint_as_float(a[e]), __uint_as_float(a[e + 1])));
            a[e] = __float_as_uint(x.x);
            a[e + 1] = __float_as_uint(x.y);
          }
          tmem_st32(tDVacc + qc0 + c0 + lane_off, a);
        }
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(dv_drained);
      }
    }
    if constexpr (kTail) {
      // the CTA's tail: (d=128) this warpgroup's 64 columns of dV_j -> the output, from the fp32 TMEM accumulator
      if constexpr (kAlias) {
        const long long orow = io.row(bh, (long long)j * kBlk + r) + qc0;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t a[32];
          tmem_ld32(tDVacc + qc0 + c0 + lane_off, a);
          tmem_wait_ld();
          if (r >= kv_valid) continue;  // a key the short last block lacks (A33)
          if (f32out) {
#pragma unroll
            for (int e4 = 0; e4 < 32; e4 += 4)
              *reinterpret_cast<uint4*>(static_cast<float*>(dv_out) + orow + c0 + e4) =
                  make_uint4(a[e4], a[e4 + 1], a[e4 + 2], a[e4 + 3]);
          } else {
#pragma unroll
            for (int e8 = 0; e8 < 32; e8 += 8) {
              uint32_t hv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                hv[e] = pack2_io(__uint_as_float(a[e8 + 2 * e]), __uint_as_float(a[e8 + 2 * e + 1]), fp16);
              *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dv_out) + orow + c0 + e8) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
            }
          }
        }
      }
      // ... and the second half of the last dQ tile's columns (d=128: 64 + 32 wg .., both warpgroups; d=64: 32 ..,
      // warpgroup 1) for this warp's 32 query rows: scaled into a 4 KB swizzled box in the P^^T / dS^^T buffers
      // (free: their last readers, the dV / dK / dQ MMAs, have completed), then one TMA reduce-add, exactly as
      // the drain warps do with the first half
      if (kAlias || wg == 1) {
      const int itl = n_it - 1, il = i_of(itl);
      mbar_wait(dkq_full, itl & 1);
      tc_fence_after();
      const float s_ds = __fdiv_rn(scl[(itl & 3) * 2 + 1], 127.f);  // the tile's psi(dS) max, as the drain reads it
      const float2 f = make_float2(s_ds * sk * tau, s_ds * sk * tau);
      const int c0 = kAlias ? 64 + 32 * wg : 32;
      uint8_t* box = smem + ((kAlias && !wg) ? L::kPt : L::kDSt) + (warp % 4) * L::kDqBox;
      uint32_t v[32];
      tmem_ld32(tDQ + c0 + lane_off, v);
      tmem_wait_ld();
      if (DUMPING && g_dacc.dq) dump_words(g_dacc.dq + (((size_t)bh * T + j) * N + il * kBlk + r) * D + c0, v, 32);
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        float2 a = fmul2(i2f2(v[e], v[e + 1], one), f);
        float2 b = fmul2(i2f2(v[e + 2], v[e + 3], one), f);
        *reinterpret_cast<float4*>(box + sw_offset(lane, e / 4, 128)) = make_float4(a.x, a.y, b.x, b.y);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_reduce_add_2d(&tm_dq, box, c0, bh * Np + il * kBlk + (warp % 4) * 32);
        bulk_commit();
        bulk_wait_all();  // the staging box must outlive the reduce
      }
      __syncwarp();
      }
    }
  } else {
    reg_set<kRegDrain, 65536 / kThreads>();
    // ------------------------------------------------------------ drain warpgroup (128 threads)
    const int r = (warp % 4) * 32 + lane;  // TMEM lane: key row (dV, dK) or query row (dQ)
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    const float sk = k_scale[(size_t)bh * T + j];
    const long long orow = io.row(bh, (long long)j * kBlk + r);  // dK, dV in the I/O layout
    constexpr int kRegV = kAlias ? 1 : D;  // dV_j in registers (d=64) or in TMEM (d=128)
    float dv_acc[kRegV];
    float dk_acc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) dk_acc[c] = 0.f;
#pragma unroll
    for (int c = 0; c < kRegV; ++c) dv_acc[c] = 0.f;

    unsigned* det_pending = nullptr;  // SAGE_DETERMINISTIC: the dQ turn this warp still has to hand on
    for (int it = 0; it < n_it; ++it) {
      const int i = i_of(it);
      const uint32_t ph = it & 1;
      const float sq = sc_q[i];
      const float sdo = sc_do[i];

      // dV_j += tile * s_P * s_dO_i  (Alg. 2 line 7); d=128: drained by the compute warps
      if constexpr (!kAlias) {
        mbar_wait(dv_full, ph);
        tc_fence_after();
        if (threadIdx.x == 384) TR(10, it);
        if (!(ablate & 1)) {
          // psi(P) scale = fl32(amax/127): the tile's, or this key row's (SAGE_P_COLSCALE)
          const float s_p = __fdiv_rn(pcol ? sp_row[(it & 3) * kBlk + r] : scl[(it & 3) * 2], pmax);
          const float2 f = make_float2(s_p * sdo, s_p * sdo);
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tDV + c0 + lane_off, v);
            tmem_wait_ld();
            if (DUMPING && g_dacc.dv)
              dump_words(g_dacc.dv + (((size_t)bh * T + i) * N + j * kBlk + r) * D + c0, v, 32);
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              float2 x = ffma2(i2f2(v[e], v[e + 1], one), f,
                               make_float2(dv_acc[c0 + e], dv_acc[c0 + e + 1]));
              dv_acc[c0 + e] = x.x;
              dv_acc[c0 + e + 1] = x.y;
            }
          }
        }
        tc_fence_before();
        warp_arrive(dv_drained);
      }

      // dK_j += tile * s_dS * s_Q * tau (+ Q-smoothing bias branch)  (line 11)
      mbar_wait(kDkQ ? dk_full : dkq_full, ph);
      tc_fence_after();
      if (threadIdx.x == 384) TR(11, it);
      if (!(ablate & 1)) {
        // psi(dS) scale: the tile's, or this key row's (FINE)
        const float s_ds = __fdiv_rn(fine ? sp_k[(it & 3) * kBlk + r] : scl[(it & 3) * 2 + 1], 127.f);
        const float2 f = make_float2(s_ds * sq * tau, s_ds * sq * tau);
        float fb = 0.f;
        const float* muq = nullptr;
        if constexpr (QSMOOTH) {
          const int* rs = rowsum_s + (it & 1) * kBlk * 2;
          fb = tau * s_ds * (float)(rs[r] + rs[kBlk + r]);
          muq = L::kSplitDO ? reinterpret_cast<const float*>(smem + L::kStage + (it % kStages) * L::kStageBytes + L::kSMu)
                            : mu_q + ((size_t)bh * T + i) * D;
        }
        uint32_t kb[2][16];
        tmem_ld16(tDK + lane_off, kb[0]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t(&v)[16] = kb[c & 1];
          if (c + 1 < D / 16) tmem_ld16(tDK + (c + 1) * 16 + lane_off, kb[(c + 1) & 1]);
          if (DUMPING && g_dacc.dk)
            dump_words(g_dacc.dk + (((size_t)bh * T + i) * N + j * kBlk + r) * D + c * 16, v, 16);
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const int cc = c * 16 + e;
            float2 acc = make_float2(dk_acc[cc], dk_acc[cc + 1]);
            if constexpr (QSMOOTH) {
              const float2 m2 = *reinterpret_cast<const float2*>(muq + cc);
              acc = ffma2(make_float2(fb, fb), m2, acc);
            }
            float2 x = ffma2(i2f2(v[e], v[e + 1], one), f, acc);
            dk_acc[cc] = x.x;
            dk_acc[cc + 1] = x.y;
          }
          if (c + 1 < D / 16) tmem_wait_ld();
        }
      }
      tc_fence_before();
      warp_arrive(dkq_drained);  // dK tile read (d=128: the region may take dQ_i)
      if constexpr (L::kSplitDO && QSMOOTH) warp_arrive(q_empty + it % kStages);  // mu_Qi read

      // dQ_i += tile * s_dS * s_K * tau, fp32 reduction across key blocks (line 10)
      if constexpr (kDkQ) {
        mbar_wait(dkq_full, ph);  // d=128: the dQ tile, issued once dK_i was drained
        tc_fence_after();
      }
      if (threadIdx.x == 384) TR(12, it);
      {
        // scaled rows -> this warp's swizzled smem staging (2 buffers) -> TMA reduce-add per box
        // the tile's psi(dS) scale, or this query row's (FINE; TMEM lane r = query row of dQ_i)
        const float s_ds = __fdiv_rn(fine ? sp_q[(it & 3) * kBlk + r] : scl[(it & 3) * 2 + 1], 127.f);
        const float2 f = make_float2(s_ds * sk * tau, s_ds * sk * tau);
        uint8_t* wstage = smem + L::kDq + (warp % 4) * L::kDqWarp;
        unsigned* flag = det ? dq_flags + ((size_t)bh * T + i) * kDrainWarps + (warp % 4) : nullptr;
        if (det) {  // wait for the contributions ordered before this one: (i - j) mod T of them
          if (lane == 0) {
            if (kDetDefer && det_pending) {  // the previous tile's contribution, complete in L2 by now
              bulk_wait_all();
              flag_release_add(det_pending);
            }
            flag_wait_geq(flag, (unsigned)((i - j + T) % T));
          }
          __syncwarp();
        }
        // SAGE_K4_TAIL: the compute warps take the last tile's columns 64..127
        const int n_rounds = (kTail && it == n_it - 1) ? L::kDqRounds / 2 : L::kDqRounds;
#pragma unroll
        for (int qq = 0; qq < L::kDqRounds; ++qq) {
          if (qq >= n_rounds) break;
          const int rnd = it * L::kDqRounds + qq;
          uint8_t* stage = wstage + (rnd % L::kDqBufs) * L::kDqBoxes * L::kDqBox;
          if (lane == 0 && rnd >= L::kDqBufs) bulk_wait_read<L::kDqBufs - 1>();  // round rnd-kDqBufs has read `stage`
          __syncwarp();
          if (!(ablate & 1)) {
#pragma unroll
            for (int bx = 0; bx < L::kDqBoxes; ++bx) {
              const int c0 = (qq * L::kDqBoxes + bx) * 32;
              uint32_t v[32];
              tmem_ld32(tDQ + c0 + lane_off, v);
              tmem_wait_ld();
              if (DUMPING && g_dacc.dq)
                dump_words(g_dacc.dq + (((size_t)bh * T + j) * N + i * kBlk + r) * D + c0, v, 32);
              uint8_t* box = stage + bx * L::kDqBox;
#pragma unroll
              for (int e = 0; e < 32; e += 4) {
                float2 a = fmul2(i2f2(v[e], v[e + 1], one), f);
                float2 b = fmul2(i2f2(v[e + 2], v[e + 3], one), f);
                *reinterpret_cast<float4*>(box + sw_offset(lane, e / 4, 128)) = make_float4(a.x, a.y, b.x, b.y);
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(ablate & 4)) {
#pragma unroll
            for (int bx = 0; bx < L::kDqBoxes; ++bx)
              tma_reduce_add_2d(&tm_dq, stage + bx * L::kDqBox, (qq * L::kDqBoxes + bx) * 32,
                                bh * Np + i * kBlk + (warp % 4) * 32);
            bulk_commit();
          }
        }
        if (kDetDefer) {
          det_pending = flag;  // handed on at the next tile (or after the loop)
        } else if (det) {  // this contribution complete in L2, then pass the turn on
          if (lane == 0) {
            bulk_wait_all();
            flag_release_add(flag);
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      warp_arrive(dq_drained);
      if (threadIdx.x == 384) TR(13, it);
    }
    if (lane == 0) bulk_wait_all();  // staging smem must outlive this warp's in-flight reduces
    if (kDetDefer && lane == 0 && det_pending) flag_release_add(det_pending);
    if constexpr (kAlias && !kTail) {  // the compute warps' last dV accumulation
      mbar_wait(dv_drained, (n_it - 1) & 1);
      tc_fence_after();
    }
    if constexpr (kTail && kAlias) {
      // dK_j rows only: the compute warps store dV_j (TAIL)
      if (r < kv_valid) {
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 8) {
          if (f32out) {
            *reinterpret_cast<float4*>(static_cast<float*>(dk_out) + orow + c0) =
                make_float4(dk_acc[c0], dk_acc[c0 + 1], dk_acc[c0 + 2], dk_acc[c0 + 3]);
            *reinterpret_cast<float4*>(static_cast<float*>(dk_out) + orow + c0 + 4) =
                make_float4(dk_acc[c0 + 4], dk_acc[c0 + 5], dk_acc[c0 + 6], dk_acc[c0 + 7]);
          } else {
            uint32_t hk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) hk[e] = pack2_io(dk_acc[c0 + 2 * e], dk_acc[c0 + 2 * e + 1], fp16);
            *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dk_out) + orow + c0) = make_uint4(hk[0], hk[1], hk[2], hk[3]);
          }
        }
      }
    } else {
    // epilogue: dK_j, dV_j rows -> bf16 (not the rows a short last block lacks, A33)
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      float vv[32];
      if constexpr (kAlias) {
        uint32_t a[16], b[16];
        tmem_ld16(tDVacc + c0 + lane_off, a);
        tmem_ld16(tDVacc + c0 + 16 + lane_off, b);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          vv[e] = __uint_as_float(a[e]);
          vv[16 + e] = __uint_as_float(b[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) vv[e] = dv_acc[c0 + e];
      }
      if (r >= kv_valid) continue;  // (after the warp-collective TMEM loads)
      if (f32out) {  // SAGE_FP32_OUT
#pragma unroll
        for (int e4 = 0; e4 < 32; e4 += 4) {
          *reinterpret_cast<float4*>(static_cast<float*>(dk_out) + orow + c0 + e4) =
              make_float4(dk_acc[c0 + e4], dk_acc[c0 + e4 + 1], dk_acc[c0 + e4 + 2], dk_acc[c0 + e4 + 3]);
          *reinterpret_cast<float4*>(static_cast<float*>(dv_out) + orow + c0 + e4) =
              make_float4(vv[e4], vv[e4 + 1], vv[e4 + 2], vv[e4 + 3]);
        }
        continue;
      }
#pragma unroll
      for (int e8 = 0; e8 < 32; e8 += 8) {
        uint32_t hk[4], hv[4];  // the I/O type: bf16, or fp16 with SAGE_FP16
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hk[e] = pack2_io(dk_acc[c0 + e8 + 2 * e], dk_acc[c0 + e8 + 2 * e + 1], fp16);
          hv[e] = pack2_io(vv[e8 + 2 * e], vv[e8 + 2 * e + 1], fp16);
        }
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dk_out) + orow + c0 + e8) = make_uint4(hk[0], hk[1], hk[2], hk[3]);
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dv_out) + orow + c0 + e8) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
      }
    }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool C, bool QS, int VAR, bool TAIL>
cudaError_t launch_tt(const BwdArgs& a, cudaStream_t s) {
  auto kern = sage_bwd_kernel<D, C, QS, VAR, TAIL>;
  constexpr int kSmem = BwdSmem<D, VAR == 3>::kAlloc;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (e != cudaSuccess) return e;
  const int T = num_blocks(a.N);
  kern<<<a.BH * T, kThreads, kSmem, s>>>(a.tm_q, a.tm_k, a.tm_doq, a.tm_v, a.tm_do, a.tm_dq, a.q_scale,
                                                       a.k_scale, a.do_scale, a.l2, a.delta, a.bias, a.mu_q,
                                                       a.dq_acc, a.dk, a.dv, a.N, a.BH, a.tau, a.pu8 ? 1 : 0,
                                                       a.fp16 ? 1 : 0, a.f32out ? 1 : 0, a.dq_flags, a.io, a.ablate);
  return cudaGetLastError();
}

}  // namespace

cudaError_t set_bwd_dump(const BwdDump& d) { return cudaMemcpyToSymbol(g_dump, &d, sizeof(d)); }

cudaError_t set_bwd_dump_acc(int32_t* s_t, int32_t* dv_t, int32_t* dk_t, int32_t* dq_t, float* dp_t) {
  const BwdDumpAcc a{s_t, dv_t, dk_t, dq_t, dp_t};
  return cudaMemcpyToSymbol(g_dacc, &a, sizeof(a));
}

cudaError_t read_bwd_trace(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace)) bytes = sizeof(g_trace);
  return cudaMemcpyFromSymbol(host, g_trace, bytes);
}

template <int D, bool C, bool QS, int VAR>
cudaError_t launch_t(const BwdArgs& a, cudaStream_t s) {
  // (d=64 has the same tail path -- half of the last dQ tile by compute warpgroup 1 -- but measured neutral at
  // C2, 0.495 vs 0.494-0.500 ms, so it is not instantiated)
  if constexpr (D == 128 && (VAR == 0 || VAR == 2))
    if (num_blocks(a.N) <= SAGE_K4_TAIL_MAXT) return launch_tt<D, C, QS, VAR, true>(a, s);
  return launch_tt<D, C, QS, VAR, false>(a, s);
}

template <int D, int VAR>
cudaError_t launch_d(const BwdArgs& a, cudaStream_t s) {
  if (a.causal) return a.qsmooth ? launch_t<D, true, true, VAR>(a, s) : launch_t<D, true, false, VAR>(a, s);
  return a.qsmooth ? launch_t<D, false, true, VAR>(a, s) : launch_t<D, false, false, VAR>(a, s);
}

template <int D>
cudaError_t launch_v(const BwdArgs& a, cudaStream_t s) {
  if (a.dq_flags != nullptr) return launch_d<D, 1>(a, s);  // the API rejects det + colscale / fine
  if (a.fine) return launch_d<D, 3>(a, s);
  return a.pcol ? launch_d<D, 2>(a, s) : launch_d<D, 0>(a, s);
}

cudaError_t launch_bwd(const BwdArgs& a, cudaStream_t s) {
  return a.d == 128 ? launch_v<128>(a, s) : launch_v<64>(a, s);
}

}  // namespace sage
