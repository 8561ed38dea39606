// sage_api.cu -- the extern "C" boundary of libsage.so (include/sage.h): argument
// validation, carving of the caller-owned ctx / workspace buffers, TMA tensor-map
// encoding and the kernel launch sequence of sage_fwd (K0, K1, [bias], K2) and
// sage_bwd (K3, K4, K5).  No device memory is allocated here.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/sage.h"
#include "sage_internal.h"

namespace sage {
namespace {

thread_local int g_last_cuda_error = 0;

sage_status cuda_fail_at(cudaError_t e, int line) {
  g_last_cuda_error = (int)e;
  if (std::getenv("SAGE_DEBUG"))
    std::fprintf(stderr, "[libsage] cuda error %d (%s) at sage_api.cu:%d\n", (int)e, cudaGetErrorString(e), line);
  return SAGE_ERR_CUDA;
}
#define cuda_fail(e) cuda_fail_at((e), __LINE__)

// ---- cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// Per-device arch check (sm_100 only; there is no fallback path).  Also clears a stale
// error another library left in this thread's runtime state, so that the
// cudaGetLastError() after each of our launches reports only our own launches.
sage_status check_arch() {
  (void)cudaGetLastError();
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  // Bind the device's primary context to this thread (e.g. torch's autograd worker thread):
  // cuTensorMapEncodeTiled needs a current context.
  if ((e = cudaSetDevice(dev)) != cudaSuccess) return cuda_fail(e);
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return SAGE_ERR_ARCH;
  return (major == 10 && minor == 0) ? SAGE_OK : SAGE_ERR_ARCH;
}

constexpr size_t kAlign = 256;
size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Dims {
  size_t BH, N, d, T, Np;  // T = ceil(N / 128) blocks; the library's per-row buffers have Np = 128 T rows per head
  bool causal, ks, qs, pu8, qkn, det, pcol, fine, fp16, f32out, pvfp8;
  float tau;
  IoLayout io;  // element strides of the I/O tensors
};

bool dims_of(const sage_params* p, Dims* o) {
  if (!p) return false;
  if (p->batch <= 0 || p->heads <= 0 || p->seqlen <= 0) return false;
  if (p->head_dim != 64 && p->head_dim != 128) return false;
  if (p->seqlen > kMaxSeqLen) return false;  // any N >= 1: a ragged N has a short last block (reading A33)
  if (p->flags & ~(uint32_t)(SAGE_CAUSAL | SAGE_K_SMOOTH | SAGE_Q_SMOOTH | SAGE_P_U8 | SAGE_QK_NORM | SAGE_DETERMINISTIC |
                             SAGE_P_COLSCALE | SAGE_FINE_BWD | SAGE_FP16 | SAGE_FP32_OUT | SAGE_PV_FP8))
    return false;
  if (!(p->softmax_scale >= 0.f) || std::isinf(p->softmax_scale)) return false;
  const size_t BH = (size_t)p->batch * p->heads;
  if (BH * (size_t)padded_len(p->seqlen) > (size_t)INT32_MAX / 2) return false;  // TMA row coordinates are int32
  o->BH = BH;
  o->N = p->seqlen;
  o->d = p->head_dim;
  o->T = (size_t)num_blocks(p->seqlen);
  o->Np = o->T * kBlk;
  o->causal = p->flags & SAGE_CAUSAL;
  o->ks = p->flags & SAGE_K_SMOOTH;
  o->qs = p->flags & SAGE_Q_SMOOTH;
  o->pu8 = p->flags & SAGE_P_U8;
  o->qkn = p->flags & SAGE_QK_NORM;
  o->det = p->flags & SAGE_DETERMINISTIC;
  o->pcol = p->flags & SAGE_P_COLSCALE;
  o->fine = p->flags & SAGE_FINE_BWD;
  o->fp16 = p->flags & SAGE_FP16;
  o->f32out = p->flags & SAGE_FP32_OUT;
  o->pvfp8 = p->flags & SAGE_PV_FP8;
  if (o->pvfp8 && o->pu8) return false;  // one forward P^ variant at a time
  if (o->det && (o->pcol || o->fine)) return false;  // one backward variant at a time
  if (o->f32out && o->qkn) return false;              // the QK-norm outputs dX are I/O-typed
  o->tau = p->softmax_scale > 0.f ? p->softmax_scale : 1.f / std::sqrt((float)p->head_dim);
  // I/O layout: all strides 0 = contiguous [B, H, N, d]; otherwise every stride >= 1 and a multiple of 8
  // elements (16-byte rows for the vector loads and the TMA maps), the token stride at least d
  const long long sb = p->stride_b, sh = p->stride_h, sn = p->stride_n;
  if (sb == 0 && sh == 0 && sn == 0) {
    o->io = IoLayout{(long long)p->heads * p->seqlen * p->head_dim, (long long)p->seqlen * p->head_dim,
                     (long long)p->head_dim, p->heads};
  } else {
    if (sb <= 0 || sh <= 0 || sn < p->head_dim || (sb | sh | sn) % 8) return false;
    o->io = IoLayout{sb, sh, sn, p->heads};
  }
  return true;
}

// ---- carving.  ctx: q_i8, k_i8, q_scale, k_scale, mu_k, [mu_q, bias]
struct CtxLayout {
  size_t q8, k8, sq, sk, muk, muq, bias, rq, rk, total;
};
CtxLayout ctx_layout(const Dims& D) {
  CtxLayout L{};
  size_t off = 0, nd = D.BH * D.Np * D.d;  // padded rows (A33)
  L.q8 = off; off += up(nd);
  L.k8 = off; off += up(nd);
  L.sq = off; off += up(D.BH * D.T * 4);
  L.sk = off; off += up(D.BH * D.T * 4);
  L.muk = off; off += up(D.BH * D.d * 4);
  L.muq = off; off += D.qs ? up(D.BH * D.T * D.d * 4) : 0;
  L.bias = off; off += D.qs ? up(D.BH * D.T * D.Np * 4) : 0;
  L.rq = off; off += D.qkn ? up(D.BH * D.Np * 4) : 0;  // QK-norm rstd of X_q, X_k rows
  L.rk = off; off += D.qkn ? up(D.BH * D.Np * 4) : 0;
  L.total = off;
  return L;
}
// fwd ws: v_i8, v_scale, colsum partials (K [, Q])
struct FwdWs {
  size_t v8, sv, partk, partq, total;
};
FwdWs fwd_ws(const Dims& D) {
  FwdWs W{};
  size_t off = 0, nd = D.BH * D.Np * D.d;
  W.v8 = off; off += up(nd);
  W.sv = off; off += up(D.BH * D.T * 4);
  W.partk = off; off += up(D.BH * D.T * D.d * 8);
  W.partq = off; off += D.qs ? up(D.BH * D.T * D.d * 8) : 0;
  W.total = off;
  return W;
}
// bwd ws: do_i8, do_scale, delta, l2, dq_acc
struct BwdWs {
  size_t do8, sdo, delta, l2, dq, gq, gk, flags, total;
};
BwdWs bwd_ws(const Dims& D) {
  BwdWs W{};
  size_t off = 0, nd = D.BH * D.Np * D.d;
  W.do8 = off; off += up(nd);
  W.sdo = off; off += up(D.BH * D.T * 4);
  W.delta = off; off += up(D.BH * D.Np * 4);
  W.l2 = off; off += up(D.BH * D.Np * 4);
  W.dq = off; off += up(nd * 4);
  // QK-norm dgamma partials: per 128-row block (fp32), then per 64 blocks (fp64), see launch_norm_bwd
  const size_t gbytes = D.BH * D.T * D.d * 4 + 8 + (D.BH * D.T + 63) / 64 * D.d * 8;
  W.gq = off; off += D.qkn ? up(gbytes) : 0;
  W.gk = off; off += D.qkn ? up(gbytes) : 0;
  W.flags = off; off += D.det ? up(D.BH * D.T * 4 * 4) : 0;  // SAGE_DETERMINISTIC dQ ordering flags
  W.total = off;
  return W;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---- optional instrumentation (sage_profile_enable / sage_profile_read), per thread
struct Prof {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[2];  // [0] K2, [1] K4
  std::vector<cudaEvent_t> pool;
  int64_t launches = 0;
  cudaEvent_t get() {
    cudaEvent_t e = nullptr;
    if (!pool.empty()) {
      e = pool.back();
      pool.pop_back();
    } else if (cudaEventCreate(&e) != cudaSuccess) {
      e = nullptr;
    }
    return e;
  }
};
thread_local Prof g_prof;

// Launch `fn` (the fused kernel) bracketed by events when profiling.
template <typename F>
cudaError_t timed(int which, cudaStream_t s, F&& fn) {
  if (!g_prof.on) return fn();
  cudaEvent_t a = g_prof.get(), b = g_prof.get();
  if (a) cudaEventRecord(a, s);
  cudaError_t e = fn();
  if (b) cudaEventRecord(b, s);
  if (a && b) g_prof.ev[which].emplace_back(a, b);
  return e;
}

// Profiling-only ablation switch for K4 (SAGE_ABLATE=<bits>), read once; 0 in normal use.
int ablate_flags() {
  static int v = [] {
    const char* e = std::getenv("SAGE_ABLATE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// sage_debug_dump / sage_debug_fwd_dump state (libsage_trace.so only): K4 / K2 dumps on while heads > 0
int g_dump_heads = 0;
int g_fwd_dump_heads = 0;

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(base) + off);
}

// A device pointer of another device than the current one would be launched against on the wrong
// GPU: reject it (host or unregistered pointers are left to the launch to fault on).
bool on_current_device(const void* ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return true;
  return a.device == dev;
}

// FNV-1a over every sage_params field (sage_params_tag); never 0.
uint64_t params_tag(const sage_params* p) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint32_t v) {
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xFFu;
      h *= 1099511628211ull;
    }
  };
  uint32_t sc;
  std::memcpy(&sc, &p->softmax_scale, 4);
  mix((uint32_t)p->batch);
  mix((uint32_t)p->heads);
  mix((uint32_t)p->seqlen);
  mix((uint32_t)p->head_dim);
  mix(p->flags);
  mix(sc);
  for (long long v : {(long long)p->stride_b, (long long)p->stride_h, (long long)p->stride_n}) {
    mix((uint32_t)v);
    mix((uint32_t)((unsigned long long)v >> 32));
  }
  return h ? h : 1;
}

}  // namespace

namespace {
// Per-thread cache of encoded tensor maps (the encode is a driver call of a few microseconds; a training
// loop re-uses the same buffers every step).  Keyed by everything the encoding depends on.
struct TmapEntry {
  const void* base;
  uint64_t rows, cols;
  uint32_t box_rows, box_cols, type, device;
  uint64_t stamp;
  CUtensorMap map;
};
constexpr int kTmapCache = 64;
thread_local TmapEntry g_tmaps[kTmapCache];
thread_local uint64_t g_tmap_clock = 0;
}  // namespace

bool make_tmap_2d_uncached(CUtensorMap* m, const void* base, TmapType type, uint64_t rows, uint64_t cols,
                           uint32_t box_rows, uint32_t box_cols);

bool make_tmap_2d(CUtensorMap* m, const void* base, TmapType type, uint64_t rows, uint64_t cols, uint32_t box_rows,
                  uint32_t box_cols) {
  int dev = 0;
  (void)cudaGetDevice(&dev);
  TmapEntry* victim = &g_tmaps[0];
  for (auto& e : g_tmaps) {
    if (e.stamp && e.base == base && e.rows == rows && e.cols == cols && e.box_rows == box_rows &&
        e.box_cols == box_cols && e.type == (uint32_t)type && e.device == (uint32_t)dev) {
      e.stamp = ++g_tmap_clock;
      *m = e.map;
      return true;
    }
    if (e.stamp < victim->stamp) victim = &e;
  }
  if (!make_tmap_2d_uncached(m, base, type, rows, cols, box_rows, box_cols)) return false;
  *victim = TmapEntry{base, rows, cols, box_rows, box_cols, (uint32_t)type, (uint32_t)dev, ++g_tmap_clock, *m};
  return true;
}

bool make_tmap_io(CUtensorMap* m, const void* base, TmapType type, int B, int N, int d, const IoLayout& io,
                  uint32_t box_rows, uint32_t box_cols) {
  // a contiguous tensor is the 2-D map the kernels' 4-D coordinates reduce to; otherwise a 4-D map
  // (d, N, H, B) with the caller's strides.  Cached like the 2-D maps (keyed by base, shape and strides).
  struct Entry {
    const void* base;
    long long sb, sh, sn;
    int B, H, N, d, type, device;
    uint32_t box_rows, box_cols;
    uint64_t stamp;
    CUtensorMap map;
  };
  constexpr int kCache = 16;
  thread_local Entry cache[kCache];
  thread_local uint64_t clock = 0;
  int dev = 0;
  (void)cudaGetDevice(&dev);
  Entry* victim = &cache[0];
  for (auto& e : cache) {
    if (e.stamp && e.base == base && e.sb == io.sb && e.sh == io.sh && e.sn == io.sn && e.B == B && e.H == io.H &&
        e.N == N && e.d == d && e.type == (int)type && e.device == dev && e.box_rows == box_rows && e.box_cols == box_cols) {
      e.stamp = ++clock;
      *m = e.map;
      return true;
    }
    if (e.stamp < victim->stamp) victim = &e;
  }
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const uint32_t esz = type == kF32 ? 4 : (type == kBF16 || type == kF16) ? 2 : 1;
  const CUtensorMapDataType dt = type == kF32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : type == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : type == kF16  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)io.H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)io.sn * esz, (cuuint64_t)io.sh * esz, (cuuint64_t)io.sb * esz};
  cuuint32_t box[4] = {box_cols, box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const uint32_t row_bytes = box_cols * esz;
  CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(m, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (std::getenv("SAGE_DEBUG"))
      std::fprintf(stderr, "[libsage] cuTensorMapEncodeTiled (4-D) -> %d\n", (int)r);
    return false;
  }
  *victim = Entry{base, io.sb, io.sh, io.sn, B, io.H, N, d, (int)type, dev, box_rows, box_cols, ++clock, *m};
  return true;
}

bool make_tmap_2d_uncached(CUtensorMap* m, const void* base, TmapType type, uint64_t rows, uint64_t cols,
                           uint32_t box_rows, uint32_t box_cols) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const uint32_t esz = type == kF32 ? 4 : (type == kBF16 || type == kF16) ? 2 : 1;
  const CUtensorMapDataType dt = type == kF32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : type == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : type == kF16  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const uint32_t row_bytes = box_cols * esz;
  CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && std::getenv("SAGE_DEBUG"))
    std::fprintf(stderr, "[libsage] cuTensorMapEncodeTiled -> %d (base %p rows %llu cols %llu box %u x %u)\n", (int)r,
                 base, (unsigned long long)rows, (unsigned long long)cols, box_rows, box_cols);
  return r == CUDA_SUCCESS;
}

}  // namespace sage

using namespace sage;

extern "C" {

int sage_version(void) { return 1; }

const char* sage_status_string(sage_status s) {
  switch (s) {
    case SAGE_OK: return "SAGE_OK";
    case SAGE_ERR_INVALID_VALUE: return "SAGE_ERR_INVALID_VALUE";
    case SAGE_ERR_UNSUPPORTED: return "SAGE_ERR_UNSUPPORTED";
    case SAGE_ERR_MISALIGNED: return "SAGE_ERR_MISALIGNED";
    case SAGE_ERR_WORKSPACE: return "SAGE_ERR_WORKSPACE";
    case SAGE_ERR_CUDA: return "SAGE_ERR_CUDA";
    case SAGE_ERR_ARCH: return "SAGE_ERR_ARCH";
  }
  return "SAGE_ERR_UNKNOWN";
}

int sage_last_cuda_error(void) { return g_last_cuda_error; }

sage_status sage_profile_enable(int enable) {
  g_prof.on = enable != 0;
  return SAGE_OK;
}

sage_status sage_profile_read(double* fwd_kernel_ms, double* bwd_kernel_ms, int64_t* n_fwd, int64_t* n_bwd,
                              int64_t* n_launches) {
  double ms[2] = {0.0, 0.0};
  int64_t n[2] = {0, 0};
  cudaError_t err = cudaSuccess;
  for (int w = 0; w < 2; ++w) {
    for (auto& pr : g_prof.ev[w]) {
      float t = 0.f;
      cudaError_t e = cudaEventSynchronize(pr.second);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t, pr.first, pr.second);
      if (e != cudaSuccess) err = e;
      ms[w] += t;
      ++n[w];
      g_prof.pool.push_back(pr.first);
      g_prof.pool.push_back(pr.second);
    }
    g_prof.ev[w].clear();
  }
  if (fwd_kernel_ms) *fwd_kernel_ms = ms[0];
  if (bwd_kernel_ms) *bwd_kernel_ms = ms[1];
  if (n_fwd) *n_fwd = n[0];
  if (n_bwd) *n_bwd = n[1];
  if (n_launches) *n_launches = g_prof.launches;
  g_prof.launches = 0;
  return err == cudaSuccess ? SAGE_OK : cuda_fail(err);
}

size_t sage_ctx_bytes(const sage_params* p) {
  Dims D;
  return dims_of(p, &D) ? ctx_layout(D).total : 0;
}

uint64_t sage_params_tag(const sage_params* p) {
  Dims D;
  return dims_of(p, &D) ? params_tag(p) : 0;
}

size_t sage_workspace_bytes(const sage_params* p, int backward) {
  Dims D;
  if (!dims_of(p, &D)) return 0;
  return backward ? bwd_ws(D).total : fwd_ws(D).total;
}

sage_status sage_ctx_get_view(const sage_params* p, void* ctx, sage_ctx_view* out) {
  Dims D;
  if (!dims_of(p, &D) || !ctx || !out) return SAGE_ERR_INVALID_VALUE;
  CtxLayout L = ctx_layout(D);
  out->q_i8 = at<int8_t>(ctx, L.q8);
  out->k_i8 = at<int8_t>(ctx, L.k8);
  out->q_scale = at<float>(ctx, L.sq);
  out->k_scale = at<float>(ctx, L.sk);
  out->mu_k = at<float>(ctx, L.muk);
  out->mu_q = D.qs ? at<float>(ctx, L.muq) : nullptr;
  out->bias = D.qs ? at<float>(ctx, L.bias) : nullptr;
  out->rstd_q = D.qkn ? at<float>(ctx, L.rq) : nullptr;
  out->rstd_k = D.qkn ? at<float>(ctx, L.rk) : nullptr;
  return SAGE_OK;
}

sage_status sage_ws_get_view(const sage_params* p, int backward, void* ws, sage_ws_view* out) {
  Dims D;
  if (!dims_of(p, &D) || !ws || !out) return SAGE_ERR_INVALID_VALUE;
  std::memset(out, 0, sizeof(*out));
  if (backward) {
    BwdWs W = bwd_ws(D);
    out->do_i8 = at<int8_t>(ws, W.do8);
    out->do_scale = at<float>(ws, W.sdo);
    out->delta = at<float>(ws, W.delta);
    out->dq_acc = at<float>(ws, W.dq);
  } else {
    FwdWs W = fwd_ws(D);
    out->v_i8 = at<int8_t>(ws, W.v8);
    out->v_scale = at<float>(ws, W.sv);
  }
  return SAGE_OK;
}

}  // extern "C"

namespace {
// Forward launch sequence; gq/gk non-null <=> QK-norm (q, k are then X_q, X_k).
sage_status fwd_impl(const Dims& D, const void* q, const void* k, const void* v, const float* gq, const float* gk,
                     float eps, void* o, float* lse, void* ctx, size_t ctx_bytes, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!q || !k || !v || !o || !lse || !ctx || !ws) return SAGE_ERR_INVALID_VALUE;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(lse) || !aligned16(ctx) ||
      !aligned16(ws))
    return SAGE_ERR_MISALIGNED;
  const CtxLayout C = ctx_layout(D);
  const FwdWs W = fwd_ws(D);
  if (ctx_bytes < C.total || ws_bytes < W.total) return SAGE_ERR_WORKSPACE;
  sage_status st = check_arch();
  if (st != SAGE_OK) return st;
  if (!on_current_device(q) || !on_current_device(o) || !on_current_device(ctx)) return SAGE_ERR_INVALID_VALUE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int BH = (int)D.BH, N = (int)D.N, d = (int)D.d;
  const void *qb = q, *kb = k, *vb = v;  // bf16, or fp16 with SAGE_FP16
  const bool h = D.fp16;
  int8_t *q8 = at<int8_t>(ctx, C.q8), *k8 = at<int8_t>(ctx, C.k8), *v8 = at<int8_t>(ws, W.v8);
  float *sq = at<float>(ctx, C.sq), *sk = at<float>(ctx, C.sk), *sv = at<float>(ws, W.sv);
  float* muk = at<float>(ctx, C.muk);
  float* muq = D.qs ? at<float>(ctx, C.muq) : nullptr;
  float* bias = D.qs ? at<float>(ctx, C.bias) : nullptr;
  double* partk = at<double>(ws, W.partk);
  double* partq = D.qs ? at<double>(ws, W.partq) : nullptr;
  float* rq = D.qkn ? at<float>(ctx, C.rq) : nullptr;
  float* rk = D.qkn ? at<float>(ctx, C.rk) : nullptr;
  const NormIn nq{rq, gq, eps}, nk{rk, gk, eps};

  FwdArgs a{};
  const uint64_t rows = D.BH * D.Np;
  if (!make_tmap_2d(&a.tm_q, q8, kU8, rows, d, kBlk, d) || !make_tmap_2d(&a.tm_k, k8, kU8, rows, d, kBlk, d) ||
      !make_tmap_2d(&a.tm_v, v8, kU8, rows, d, kBlk, d))
    return cuda_fail(cudaErrorInvalidValue);

  cudaError_t e = cudaSuccess;
  // QK-norm: the row statistics and normalised values are formed on the fly in K0/K1
  // K0: smoothing statistics
  if (D.ks) {
    if ((e = launch_colsum(kb, partk, BH, N, d, s, nk, h, D.io)) != cudaSuccess) return cuda_fail(e);
    if ((e = launch_colmean(partk, muk, BH, N, d, s)) != cudaSuccess) return cuda_fail(e);
  }
  if (D.qs) {
    if ((e = launch_colsum(qb, partq, BH, N, d, s, nq, h, D.io)) != cudaSuccess) return cuda_fail(e);
    if ((e = launch_blockmean(partq, muq, BH, N, d, s)) != cudaSuccess) return cuda_fail(e);
  }
  // K1: per-block psi (Alg. 1 line 3)
  QuantJobs qj{};
  qj.j[0] = QuantJob{qb, muq, D.qs ? 2 : 0, q8, sq, rq, gq, eps};
  qj.j[1] = QuantJob{kb, muk, D.ks ? 1 : 0, k8, sk, rk, gk, eps};
  qj.j[0].fp8 = qj.j[1].fp8 = 0;
  qj.j[2] = QuantJob{vb, nullptr, 0, v8, sv, nullptr, nullptr, 0.f, D.pvfp8 ? 1 : 0};
  if ((e = launch_quantize(qj, 3, BH, N, d, s, h, D.io)) != cudaSuccess) return cuda_fail(e);
  // mu_K is all-zero when K-smoothing is off (ctx is caller memory: make it so)
  if (!D.ks && (e = launch_fill(muk, D.BH * D.d, 0.f, s)) != cudaSuccess) return cuda_fail(e);
  if (D.qs && (e = launch_qsmooth_bias(kb, muk, muq, bias, BH, N, d, s, nk, h, D.io)) != cudaSuccess)
    return cuda_fail(e);
  // K2: fused INT8 forward (Alg. 1 lines 4-14)
  a.q_scale = sq;
  a.k_scale = sk;
  a.v_scale = sv;
  a.bias = bias;
  a.o = o;
  a.fp16 = D.fp16;
  a.f32out = D.f32out;
  a.pvfp8 = D.pvfp8;
  a.io = D.io;
  a.lse = lse;
  a.BH = BH;
  a.N = N;
  a.d = d;
  a.tau = D.tau;
  a.causal = D.causal;
  a.qsmooth = D.qs;
  a.pu8 = D.pu8;
  a.ablate = ablate_flags() | (g_fwd_dump_heads > 0 ? 16 : 0);
  if ((e = timed(0, s, [&] { return launch_fwd(a, s); })) != cudaSuccess) return cuda_fail(e);
  if (g_prof.on) g_prof.launches += (D.ks ? 2 : 1) + (D.qs ? 3 : 0) + 1 + 1;
  return SAGE_OK;
}

// Backward launch sequence; with QK-norm (D.qkn) dq/dk receive dX_q/dX_k and xq, xk, gq, gk, dgq, dgk
// are the RMSNorm inputs and dgamma outputs.
sage_status bwd_impl(const Dims& D, const void* v, const void* o, const float* lse, const void* dO, const void* ctx,
                     size_t ctx_bytes, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, void* stream,
                     const void* xq, const void* xk, const float* gq, const float* gk, float* dgq, float* dgk) {
  if (!v || !o || !lse || !dO || !ctx || !dq || !dk || !dv || !ws) return SAGE_ERR_INVALID_VALUE;
  if (!aligned16(v) || !aligned16(o) || !aligned16(lse) || !aligned16(dO) || !aligned16(ctx) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv) || !aligned16(ws))
    return SAGE_ERR_MISALIGNED;
  const CtxLayout C = ctx_layout(D);
  const BwdWs W = bwd_ws(D);
  if (ctx_bytes < C.total || ws_bytes < W.total) return SAGE_ERR_WORKSPACE;
  sage_status st = check_arch();
  if (st != SAGE_OK) return st;
  if (!on_current_device(dO) || !on_current_device(dq) || !on_current_device(ctx)) return SAGE_ERR_INVALID_VALUE;
  if (D.det && !D.causal) {
    // the rotated non-causal order needs all T key-block CTAs of a head resident at once
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return cuda_fail(cudaErrorInvalidValue);
    if ((int)D.T > sms) return SAGE_ERR_UNSUPPORTED;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int BH = (int)D.BH, N = (int)D.N, d = (int)D.d;
  void* cx = const_cast<void*>(ctx);
  int8_t *q8 = at<int8_t>(cx, C.q8), *k8 = at<int8_t>(cx, C.k8), *do8 = at<int8_t>(ws, W.do8);
  float *sq = at<float>(cx, C.sq), *sk = at<float>(cx, C.sk), *sdo = at<float>(ws, W.sdo);
  float *delta = at<float>(ws, W.delta), *l2 = at<float>(ws, W.l2);
  // SAGE_FP32_OUT with contiguous outputs: dQ is reduced straight into the caller's fp32 dq (zeroed by K3; no K5)
  const bool dq_direct = D.f32out && D.io.contiguous((int)D.N, (int)D.d) && D.Np == D.N;
  float* dqacc = dq_direct ? static_cast<float*>(dq) : at<float>(ws, W.dq);

  BwdArgs a{};
  const uint64_t rows = D.BH * D.Np;
  if (!make_tmap_2d(&a.tm_q, q8, kU8, rows, d, kBlk, d) || !make_tmap_2d(&a.tm_k, k8, kU8, rows, d, kBlk, d) ||
      !make_tmap_2d(&a.tm_doq, do8, kU8, rows, d, kBlk, d) ||
      !make_tmap_io(&a.tm_v, v, D.fp16 ? kF16 : kBF16, BH / D.io.H, N, d, D.io, kBlk, 64) ||
      !make_tmap_io(&a.tm_do, dO, D.fp16 ? kF16 : kBF16, BH / D.io.H, N, d, D.io, kBlk, 64) ||
      !make_tmap_2d(&a.tm_dq, dqacc, kF32, rows, d, 32, 32))
    return cuda_fail(cudaErrorInvalidValue);
  cudaError_t e;
  // K3: delta, psi(dO), L*log2(e), zero dQ accumulator (Alg. 2 lines 2, 6)
  unsigned* dqflags = D.det ? at<unsigned>(ws, W.flags) : nullptr;
  if ((e = launch_bwd_prep(o, dO, lse, delta, l2, do8, sdo, dqacc, BH, N, d, s, dqflags, D.fp16, D.f32out, D.io)) !=
      cudaSuccess)
    return cuda_fail(e);
  // K4: fused INT8 backward (Alg. 2 lines 3-11)
  a.q_scale = sq;
  a.k_scale = sk;
  a.do_scale = sdo;
  a.l2 = l2;
  a.delta = delta;
  a.bias = D.qs ? at<float>(cx, C.bias) : nullptr;
  a.mu_q = D.qs ? at<float>(cx, C.muq) : nullptr;
  a.dq_acc = dqacc;
  a.dk = dk;
  a.dv = dv;
  a.fp16 = D.fp16;
  a.f32out = D.f32out;
  a.io = D.io;
  a.BH = BH;
  a.N = N;
  a.d = d;
  a.tau = D.tau;
  a.causal = D.causal;
  a.qsmooth = D.qs;
  a.pu8 = D.pu8;
  a.dq_flags = dqflags;
  a.pcol = D.pcol;
  a.fine = D.fine;
  a.ablate = ablate_flags() | (g_dump_heads > 0 ? 16 : 0);
  if ((e = timed(1, s, [&] { return launch_bwd(a, s); })) != cudaSuccess) return cuda_fail(e);
  if (g_prof.on) g_prof.launches += 2;  // K3, K4
  if (D.qkn) {
    // RMSNorm backward (reading A26), fused with the dQ finalisation; dK (w.r.t. the normalised K,
    // bf16 from K4) is turned into dX_k in place
    const auto* rq = at<const float>(cx, C.rq);
    const auto* rk = at<const float>(cx, C.rk);
    if ((e = launch_norm_bwd(dqacc, nullptr, xq, rq, gq, dq, at<float>(ws, W.gq),
                             dgq, D.BH * D.Np, d, s, D.fp16, D.io, N)) != cudaSuccess)
      return cuda_fail(e);
    if ((e = launch_norm_bwd(nullptr, dk, xk, rk, gk, dk, at<float>(ws, W.gk),
                             dgk, D.BH * D.Np, d, s, D.fp16, D.io, N)) != cudaSuccess)
      return cuda_fail(e);
    if (g_prof.on) g_prof.launches += 6;  // 2 x (norm_bwd, dgamma stage 1, stage 2)
    return SAGE_OK;
  }
  // K5 (not when dq already holds the fp32 sum)
  if (dq_direct) return SAGE_OK;
  if ((e = launch_dq_finalize(dqacc, dq, BH, N, d, s, D.fp16, D.io, D.f32out)) != cudaSuccess)
    return cuda_fail(e);
  if (g_prof.on) g_prof.launches += 1;  // K5
  return SAGE_OK;
}
}  // namespace

extern "C" {

sage_status sage_fwd(const sage_params* p, const void* q, const void* k, const void* v, void* o, float* lse,
                     sage_ctx* ctx, void* ws, size_t ws_bytes, void* stream) {
  Dims D;
  if (!dims_of(p, &D) || D.qkn || !ctx) return SAGE_ERR_INVALID_VALUE;  // QK-norm: sage_fwd_qknorm
  const sage_status st = fwd_impl(D, q, k, v, nullptr, nullptr, 0.f, o, lse, ctx->buf, ctx->bytes, ws, ws_bytes, stream);
  if (st == SAGE_OK) ctx->params_tag = params_tag(p);
  return st;
}

sage_status sage_fwd_qknorm(const sage_params* p, const void* xq, const void* xk, const void* v, const float* gamma_q,
                            const float* gamma_k, float eps, void* o, float* lse, sage_ctx* ctx, void* ws,
                            size_t ws_bytes, void* stream) {
  Dims D;
  if (!dims_of(p, &D) || !D.qkn || !ctx || !gamma_q || !gamma_k || !(eps > 0.f) || std::isinf(eps))
    return SAGE_ERR_INVALID_VALUE;
  if (!aligned16(gamma_q) || !aligned16(gamma_k)) return SAGE_ERR_MISALIGNED;
  const sage_status st =
      fwd_impl(D, xq, xk, v, gamma_q, gamma_k, eps, o, lse, ctx->buf, ctx->bytes, ws, ws_bytes, stream);
  if (st == SAGE_OK) ctx->params_tag = params_tag(p);
  return st;
}

sage_status sage_bwd(const sage_params* p, const void* v, const void* o, const float* lse, const void* dO,
                     const sage_ctx* ctx, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, void* stream) {
  Dims D;
  if (!dims_of(p, &D) || D.qkn || !ctx) return SAGE_ERR_INVALID_VALUE;  // QK-norm: sage_bwd_qknorm
  if (ctx->params_tag != params_tag(p)) return SAGE_ERR_INVALID_VALUE;   // another forward's context
  return bwd_impl(D, v, o, lse, dO, ctx->buf, ctx->bytes, dq, dk, dv, ws, ws_bytes, stream, nullptr, nullptr,
                  nullptr, nullptr, nullptr, nullptr);
}

sage_status sage_bwd_qknorm(const sage_params* p, const void* xq, const void* xk, const float* gamma_q,
                            const float* gamma_k, const void* v, const void* o, const float* lse, const void* dO,
                            const sage_ctx* ctx, void* dxq, void* dxk, void* dv, float* dgamma_q, float* dgamma_k,
                            void* ws, size_t ws_bytes, void* stream) {
  Dims D;
  if (!dims_of(p, &D) || !D.qkn || !ctx || !xq || !xk || !gamma_q || !gamma_k || !dgamma_q || !dgamma_k)
    return SAGE_ERR_INVALID_VALUE;
  if (ctx->params_tag != params_tag(p)) return SAGE_ERR_INVALID_VALUE;
  if (!aligned16(xq) || !aligned16(xk) || !aligned16(gamma_q) || !aligned16(gamma_k) || !aligned16(dgamma_q) ||
      !aligned16(dgamma_k))
    return SAGE_ERR_MISALIGNED;
  return bwd_impl(D, v, o, lse, dO, ctx->buf, ctx->bytes, dxq, dxk, dv, ws, ws_bytes, stream, xq, xk, gamma_q,
                  gamma_k, dgamma_q, dgamma_k);
}

sage_status sage_debug_trace(void* host_out, size_t bytes) {
  if (!host_out) return SAGE_ERR_INVALID_VALUE;
  // first half: K4 timeline, second half: K2 timeline
  cudaError_t e = read_bwd_trace(host_out, bytes / 2);
  if (e == cudaSuccess) e = read_fwd_trace(static_cast<uint8_t*>(host_out) + bytes / 2, bytes / 2);
  return e == cudaSuccess ? SAGE_OK : cuda_fail(e);
}

sage_status sage_debug_dump(void* p_hat_t, float* s_p, void* ds_hat_t, float* s_ds, float* ds_t, int heads) {
#if SAGE_TRACE
  if (heads < 0 || (heads > 0 && (!p_hat_t || !s_p || !ds_hat_t || !s_ds || !ds_t))) return SAGE_ERR_INVALID_VALUE;
  BwdDump d{static_cast<int8_t*>(p_hat_t), static_cast<int8_t*>(ds_hat_t), s_p, s_ds, ds_t, heads};
  cudaError_t e = set_bwd_dump(d);
  if (e != cudaSuccess) return cuda_fail(e);
  g_dump_heads = heads;
  return SAGE_OK;
#else
  (void)p_hat_t; (void)s_p; (void)ds_hat_t; (void)s_ds; (void)ds_t; (void)heads;
  return SAGE_ERR_UNSUPPORTED;
#endif
}

sage_status sage_debug_dump_acc(int32_t* s_t, int32_t* dv_t, int32_t* dk_t, int32_t* dq_t, float* dp_t) {
#if SAGE_TRACE
  cudaError_t e = set_bwd_dump_acc(s_t, dv_t, dk_t, dq_t, dp_t);
  return e == cudaSuccess ? SAGE_OK : cuda_fail(e);
#else
  (void)s_t; (void)dv_t; (void)dk_t; (void)dq_t; (void)dp_t;
  return SAGE_ERR_UNSUPPORTED;
#endif
}

sage_status sage_debug_fwd_dump(int32_t* s, void* p_hat, float* s_p, int32_t* pv, int heads) {
#if SAGE_TRACE
  if (heads < 0) return SAGE_ERR_INVALID_VALUE;
  FwdDump d{s, static_cast<uint8_t*>(p_hat), s_p, pv, heads};
  cudaError_t e = set_fwd_dump(d);
  if (e != cudaSuccess) return cuda_fail(e);
  g_fwd_dump_heads = heads;
  return SAGE_OK;
#else
  (void)s; (void)p_hat; (void)s_p; (void)pv; (void)heads;
  return SAGE_ERR_UNSUPPORTED;
#endif
}

sage_status sage_debug_umma(int mode, int K, int N, const void* a, const void* b, void* d, void* stream) {
  if (mode < 0 || mode > 7 || !a || !b || !d) return SAGE_ERR_INVALID_VALUE;
  const bool kmode = mode == 0 || mode == 3 || mode == 5;
  if (kmode && K != 64 && K != 128) return SAGE_ERR_INVALID_VALUE;
  if (!kmode && N != 64 && N != 128) return SAGE_ERR_INVALID_VALUE;
  if (!aligned16(a) || !aligned16(b) || !aligned16(d)) return SAGE_ERR_MISALIGNED;
  sage_status st = check_arch();
  if (st != SAGE_OK) return st;
  CUtensorMap ta{}, tb{};
  bool ok = true;
  if (mode == 0) {
    ok = make_tmap_2d(&ta, a, kU8, 128, K, 128, K) && make_tmap_2d(&tb, b, kU8, 128, K, 128, K);
  } else if (mode == 3 || mode == 5) {
    ok = make_tmap_2d(&ta, mode == 3 ? a : b, kBF16, 128, K, 128, 64) && make_tmap_2d(&tb, b, kBF16, 128, K, 128, 64);
  } else {
    ok = make_tmap_2d(&tb, b, kU8, 128, N, 128, N);
    ta = tb;
  }
  if (!ok) return cuda_fail(cudaErrorInvalidValue);
  cudaError_t e = launch_debug_umma(mode, K, N, &ta, &tb, a, d, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE_OK : cuda_fail(e);
}

}  // extern "C"
