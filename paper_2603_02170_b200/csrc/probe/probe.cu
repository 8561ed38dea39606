// probe.cu -- N0 microbenchmarks: the sm_100a rates the SageBwd kernels are
// designed around.  One CTA (per SM when gridDim > 1), clock64 timing inside the kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe probe.cu && ./probe
// Prints one JSON object: per-SM rates in ops (or bytes) per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../sm100.cuh"

using namespace sage;

__device__ unsigned long long g_cyc[64];
__device__ float g_sink[1024];

// ---- ALU-type throughput: each warp runs `iters` x 8 independent ops
template <int OP>
__global__ void alu_kernel(int iters, int seed) {
  float f[8];
  uint32_t u[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    f[e] = (float)(threadIdx.x + e + seed) * 0.001f;
    u[e] = threadIdx.x * 7 + e + seed;
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (OP == 0) f[e] = __int2float_rn((int)u[e]) + f[e] * 0.f, u[e] += 1;            // I2FP (+ FFMA, IADD)
      if (OP == 1) f[e] = ex2(f[e]) * 0.5f;                                              // MUFU.EX2 (+FMUL)
      if (OP == 2) {                                                                     // FFMA2
        float2 r = ffma2(make_float2(f[e], f[(e + 1) & 7]), make_float2(1.0001f, 0.9999f), make_float2(0.1f, 0.2f));
        f[e] = r.x;
        f[(e + 1) & 7] = r.y;
      }
      if (OP == 3) u[e] = __byte_perm(u[e], u[(e + 3) & 7], 0x0040 + it);                // PRMT
      if (OP == 4) f[e] = fmaf(f[e], 1.0001f, 0.1f);                                     // FFMA
    }
  }
  unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) acc += f[e] + (float)u[e];
  g_sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cyc[0] = t1 - t0;
}

// ---- TMEM load throughput: every warp reads its 32 lanes x NCOL columns repeatedly
template <int NCOL>
__global__ void tmem_ld_kernel(int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp % 4) * 32) << 16);
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < NCOL; c += 32) {
      tmem_ld32(base + ((warp / 4) * NCOL + c) % 512, v);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += v[e];
    }
  }
  unsigned long long t1 = clock64();
  g_sink[threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) g_cyc[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

// ---- MMA throughput: one thread issues `iters` x 4 MMAs (K chunks) into TMEM; descriptors are
// precomputed so the loop is issue-light.  MODE: see kModeName.
template <int MODE>
__device__ __forceinline__ void issue(uint32_t d, uint32_t at, uint64_t da, uint64_t db, uint32_t acc) {
  if (MODE == 0) mma_i8(d, da, db, idesc_i8(128, 128, false, false), acc);
  if (MODE == 1) mma_i8(d, da, db, idesc_i8(128, 64, false, true), acc);
  if (MODE == 2) mma_i8(d, da, db, idesc_i8(128, 64, true, true), acc);
  if (MODE == 3) mma_bf16(d, da, db, idesc_bf16(128, 128, false, false), acc);
  if (MODE == 4) mma_i8(d, da, db, idesc_i8(128, 128, false, true), acc);
  if (MODE == 5) mma_i8_ts(d, at, db, idesc_i8(128, 128, false, false), acc);
  if (MODE == 6) mma_i8_ts(d, at, db, idesc_i8(128, 64, false, true), acc);
  if (MODE == 7) mma_bf16_ts(d, at, db, idesc_bf16(128, 128, false, false), acc);
  if (MODE == 8) mma_i8_ts(d, at, db, idesc_i8(128, 128, false, true), acc);
  if (MODE == 9) mma_i8(d, da, db, idesc_i8(128, 256, false, false), acc);
  if (MODE == 10) mma_i8_ts(d, at, db, idesc_i8(128, 256, false, false), acc);
  if (MODE == 11) mma_i8(d, da, db, idesc_i8(128, 128, false, false), acc);
}
template <int MODE, int COMMITS = 0>
__global__ void mma_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, bar2[2];
  const int warp = threadIdx.x / 32;
  for (int e = threadIdx.x; e < 65536 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(smem)[e] = e * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2[0], 1);
    mbar_init(&bar2[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && COMMITS == 3) {
    // latency of one MMA group: issue 4 MMAs, commit, wait
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    unsigned long long tot = 0;
    for (int it = 0; it < 64; ++it) {
      unsigned long long t0 = clock64();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        issue<MODE>(slot, slot + 256 + kk * 8, desc_kmajor(a, 128, kk * 32), desc_kmajor(b, 128, kk * 32), kk > 0);
      mma_commit(&bar2[0]);
      mbar_wait(&bar2[0], it & 1);
      tot += clock64() - t0;
    }
    g_cyc[1] = tot * 4 / 64;  // reported per instruction x4 below -> group latency
  } else if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    uint64_t da[4], db[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const bool amn = MODE == 2, bmn = MODE == 1 || MODE == 2 || MODE == 4 || MODE == 6 || MODE == 8;
      const uint32_t rb = (MODE == 1 || MODE == 2 || MODE == 6) ? 64 : 128;
      da[kk] = amn ? desc_mnmajor(a, 128, kk * 32) : (MODE == 11 ? desc_kmajor(a, 64, (kk * 32) % 64) : desc_kmajor(a, 128, kk * 32));
      db[kk] = bmn ? desc_mnmajor(b, rb, kk * 32) : (MODE == 11 ? desc_kmajor(b, 64, (kk * 32) % 64) : desc_kmajor(b, 128, kk * 32));
    }
    const uint32_t d0 = slot, d1 = (MODE == 9 || MODE == 10) ? slot : slot + 128, at = slot + 256;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it += 2) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        issue<MODE>(d0, at + kk * 8, da[kk], db[kk], kk > 0);
        if (COMMITS == 2) mma_commit(&bar2[kk & 1]);
      }
      if (COMMITS == 1) mma_commit(&bar2[0]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        issue<MODE>(d1, at + kk * 8, da[kk], db[kk], kk > 0);
        if (COMMITS == 2) mma_commit(&bar2[kk & 1]);
      }
      if (COMMITS == 1) mma_commit(&bar2[1]);
    }
    unsigned long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    g_cyc[0] = t1 - t0;
    g_cyc[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

static unsigned long long cyc(int which = 0) {
  unsigned long long h[64];
  cudaMemcpyFromSymbol(h, g_cyc, sizeof(h));
  return h[which];
}

int main() {
  cudaFree(0);
  const char* opname[] = {"i2fp", "ex2", "ffma2_pairs", "prmt", "ffma"};
  printf("{\n");
  for (int op = 0; op < 5; ++op)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: alu_kernel<0><<<1, warps * 32>>>(iters, 1); break;
          case 1: alu_kernel<1><<<1, warps * 32>>>(iters, 1); break;
          case 2: alu_kernel<2><<<1, warps * 32>>>(iters, 1); break;
          case 3: alu_kernel<3><<<1, warps * 32>>>(iters, 1); break;
          case 4: alu_kernel<4><<<1, warps * 32>>>(iters, 1); break;
        }
        cudaDeviceSynchronize();
      }
      const double ops = (double)iters * 8 * warps * 32;
      printf("  \"%s_w%d_thread_ops_per_clk\": %.2f,\n", opname[op], warps, ops / cyc());
    }
  for (int warps : {4, 8, 16}) {
    const int iters = 4096;
    for (int ncol : {32, 64}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (ncol == 32) tmem_ld_kernel<32><<<1, warps * 32>>>(iters);
        else tmem_ld_kernel<64><<<1, warps * 32>>>(iters);
        cudaDeviceSynchronize();
      }
      const double bytes = (double)iters * ncol * 4 * 32 * warps;
      printf("  \"tmem_ld_w%d_x%d_bytes_per_clk\": %.1f,\n", warps, ncol, bytes / cyc());
    }
  }
  const char* mname[] = {"i8_m128n128k32_ss_kk", "i8_m128n64k32_b_mn", "i8_m128n64k32_ab_mn", "bf16_m128n128k16_ss_kk",
                         "i8_m128n128k32_b_mn", "i8_ts_m128n128k32", "i8_ts_m128n64k32_b_mn", "bf16_ts_m128n128k16",
                         "i8_ts_m128n128k32_b_mn", "i8_m128n256k32_ss", "i8_ts_m128n256k32", "i8_m128n128k32_ss_sw64"};
  auto run = [&](auto kern, int mode, int grid) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const int iters = 1024;
    for (int rep = 0; rep < 2; ++rep) {
      kern<<<grid, 128, 70000>>>(iters);
      cudaDeviceSynchronize();
    }
    printf("  \"mma_%s%s_clk_per_instr\": %.2f,\n", mname[mode], grid > 1 ? "_148sm" : "", (double)cyc(1) / (iters * 4));
  };
  run(mma_kernel<0>, 0, 1); run(mma_kernel<1>, 1, 1); run(mma_kernel<2>, 2, 1); run(mma_kernel<3>, 3, 1);
  run(mma_kernel<4>, 4, 1); run(mma_kernel<5>, 5, 1); run(mma_kernel<6>, 6, 1); run(mma_kernel<7>, 7, 1);
  run(mma_kernel<8>, 8, 1); run(mma_kernel<9>, 9, 1); run(mma_kernel<10>, 10, 1); run(mma_kernel<11>, 11, 1);
  run(mma_kernel<0>, 0, 148); run(mma_kernel<3>, 3, 148);
  printf("  \"note\": \"next: mode0 with a commit per 4-MMA group, a commit per MMA, then group latency\",\n");
  run(mma_kernel<0, 1>, 0, 1); run(mma_kernel<0, 2>, 0, 1); run(mma_kernel<0, 3>, 0, 1);
  cudaError_t e = cudaGetLastError();
  printf("  \"cuda\": \"%s\"\n}\n", cudaGetErrorString(e));
  return 0;
}
