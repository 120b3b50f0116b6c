// Microbenchmark probe (diagnostics only): issue rate of tcgen05.mma kind::f16
// M=128 with both operands in shared memory, for a given N and operand layout.
// One CTA, one issuing thread, `iters` dependent-accumulate MMAs into one TMEM
// accumulator; reports clock64 cycles per MMA. Used to size the GEMM tiles.
#include "tc_common.cuh"

namespace sa {
namespace tcp {

using namespace tc;

__global__ void __launch_bounds__(128, 1) mma_probe_kernel(int n, int iters, int layout,
                                                           unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (3 * 8192 + 3 * 256 * 64) / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid < 32) tmem_alloc<256>(&slot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t a = smem_u32(smem), b = a + 128 * 64;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) |
                           (uint32_t(128 >> 4) << 24);
    auto desc = [&](uint32_t s) -> uint64_t {
      if (layout == 0)  // interleaved, LBO 128, SBO 512
        return uint64_t((s >> 4) & 0x3FFFu) | (uint64_t(128 >> 4) << 16) |
               (uint64_t(512 >> 4) << 32) | (uint64_t(1) << 46);
      return smem_desc(s);  // SWIZZLE_64B
    };
    const uint64_t ad = desc(a), bd = desc(b);
    const long long t0 = clock64();
    if (layout < 2) {
      for (int i = 0; i < iters; ++i) mma_bf16(tmem, ad, bd, idesc, i > 0 ? 1u : 0u);
    } else {
      // the GEMM kernels' pattern: 3 A planes (8 KB apart) x 3 B planes, 2 k-steps;
      // layout 3: + a tcgen05.commit after every 12 MMAs; layout 4: + alternate
      // between two accumulators (as fc1 / fc2 do)
      const uint64_t a2 = desc(smem_u32(smem)), b2 = desc(smem_u32(smem) + 3 * 8192);
      for (int i = 0; i < iters / 12; ++i) {
        const uint32_t dt = (layout == 4 && (i & 1)) ? tmem + 128 : tmem;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          mma_split_step<3>(dt, a2 + uint64_t(ks * 16), b2 + uint64_t(ks * 16), 8192,
                            uint32_t(n) * 64, idesc, (i | ks) != 0);
        if (layout >= 3) mma_commit(&bar2);
        if (layout >= 5) tc_fence_after();      // layout 5: + tcgen05.fence::after_thread_sync
        if (layout >= 6) tc_fence_before();     // layout 6: + fence::before_thread_sync
      }
    }
    const long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = (unsigned long long)(t2 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<256>(tmem);
}

}  // namespace tcp
}  // namespace sa

extern "C" int sa_probe_mma(int n, int iters, int layout, unsigned long long* out, void* stream) {
  const int smem = 3 * 8192 + 3 * 256 * 64 + 1024;
  cudaFuncSetAttribute(sa::tcp::mma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  // layout >= 10: the same pattern on every SM at once (full-chip contention)
  const int grid = layout >= 10 ? 148 : 1;
  sa::tcp::mma_probe_kernel<<<grid, 128, smem, sa::as_stream(stream)>>>(n, iters, layout % 10, out);
  return cudaGetLastError() == cudaSuccess ? SA_OK : SA_ERR_CUDA;
}

// ---- A-operand-in-TMEM probe (diagnostics only) ------------------------------
// 1) correctness: D = A·B^T for M=128, N=n, K=16 with A written to TMEM by
//    tcgen05.st (lane = row, column c = bf16 pair k = 2c, 2c+1) and B in smem
//    (interleaved K-major); D copied to `d_out` (128 x n fp32).
// 2) rate: `iters` chained MMAs with A in TMEM; out[0]/out[1] issue/complete cycles.
namespace sa {
namespace tcp {
using namespace tc;

__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) mma_ts_probe_kernel(int n, int iters,
                                                              const uint16_t* a_in,
                                                              const uint16_t* b_in, float* d_out,
                                                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B (n x 16) into the interleaved K-major layout
  for (int i = tid; i < n * 16; i += 128) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<uint16_t*>(smem + plane_offset(r, k)) = b_in[i];
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a_col = 256;   // A at columns 256..263, D at 0..n-1
  {
    uint32_t r[8];
    for (int c = 0; c < 8; ++c)
      r[c] = uint32_t(a_in[tid * 16 + 2 * c]) | (uint32_t(a_in[tid * 16 + 2 * c + 1]) << 16);
    tmem_st8(tmem + (uint32_t(warp * 32) << 16) + a_col, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) |
                           (uint32_t(128 >> 4) << 24);
    const uint64_t bd = smem_desc(smem_u32(smem));
    mma_bf16_ts(tmem, tmem + a_col, bd, idesc, 0u);
    const long long t0 = clock64();
    if (iters > 0) {
      for (int i = 0; i < iters; ++i) mma_bf16_ts(tmem + 128, tmem + a_col, bd, idesc, i > 0);
    }
    const long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = (unsigned long long)(t2 - t0);
  }
  __syncthreads();
  tc_fence_after();
  for (int cb = 0; cb < n; cb += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(cb), v);
    for (int q = 0; q < 16; ++q) d_out[tid * n + cb + q] = v[q];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace tcp
}  // namespace sa

extern "C" int sa_probe_mma_ts(int n, int iters, const void* a_in, const void* b_in, float* d_out,
                               unsigned long long* out, void* stream) {
  const int smem = 256 * 16 * 2 + 1024;
  cudaFuncSetAttribute(sa::tcp::mma_ts_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  sa::tcp::mma_ts_probe_kernel<<<1, 128, smem, sa::as_stream(stream)>>>(
      n, iters, static_cast<const uint16_t*>(a_in), static_cast<const uint16_t*>(b_in), d_out, out);
  return cudaGetLastError() == cudaSuccess ? SA_OK : SA_ERR_CUDA;
}

// ---- MLP-pattern probe (diagnostics only) ------------------------------------
// Replays the fused MLP's MMA issue pattern on one CTA with no other warps:
// per hidden chunk q, fc1 = 2 k-steps x NP plane products into acc1[q % 4]
// (A = x planes in TMEM, B = ring slot q % 4 of W1), fc2 = 2 k-steps x NP into
// acc2 (A = GELU planes A2[q % 4] in TMEM, B = ring slot q % 4 of W2).
// variant bit 0: B of every MMA from slot 0 (no ring); bit 1: every MMA into
// one accumulator; bit 2: commit per chunk to an mbarrier (as the kernel).
namespace sa {
namespace tcp {
__global__ void __launch_bounds__(128, 1) mma_mlp_probe_kernel(int chunks, int np, int variant,
                                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // variant bit 4: pseudo-random bf16 operands (else all ones)
  for (int i = tid; i < (8 * 6144) / 4; i += 128)
    reinterpret_cast<uint32_t*>(smem)[i] =
        (variant & 16) ? ((uint32_t(i) * 2654435761u) & 0xbfffbfffu) | 0x3c003c00u : 0x3f803f80u;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  {  // A planes: ones
    uint32_t r[16];
    for (int c = 0; c < 16; ++c)
      r[c] = (variant & 16) ? ((uint32_t(tid * 16 + c) * 2246822519u) & 0xbfffbfffu) | 0x3c003c00u
                            : 0x3f803f80u;
    for (int col = 192; col < 512; col += 16) tmem_st16(tmem + (uint32_t(warp * 32) << 16) + col, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_m128(32);
    const uint32_t sb = smem_u32(smem);
    const long long t0 = clock64();
    for (int q = 0; q < chunks; ++q) {
      const int s = (variant & 1) ? 0 : (q & 3);
      const uint32_t d1 = tmem + ((variant & 2) ? 0u : uint32_t((q & 3) * 32));
      const uint32_t d2 = tmem + ((variant & 2) ? 0u : 128u);
      const uint32_t w1 = sb + uint32_t(s) * 6144, w2 = sb + 4 * 6144 + uint32_t(s) * 6144;
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t bd = smem_desc(w1 + ks * 256);
        if (np == 1) mma_split_step_ts<1>(d1, tmem + 192 + ks * 8, bd, 16, 2048, idesc, ks != 0);
        else mma_split_step_ts<3>(d1, tmem + 192 + ks * 8, bd, 16, 2048, idesc, ks != 0);
      }
      if (variant & 4) mma_commit(&bar2);
      const uint32_t a2 = tmem + 320 + uint32_t((q & 3) * 48);
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t bd = smem_desc(w2 + ks * 256);
        if (np == 1) mma_split_step_ts<1>(d2, a2 + ks * 8, bd, 16, 2048, idesc, (q | ks) != 0);
        else mma_split_step_ts<3>(d2, a2 + ks * 8, bd, 16, 2048, idesc, (q | ks) != 0);
      }
      if (variant & 4) mma_commit(&bar2);
    }
    const long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = (unsigned long long)(t2 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
}  // namespace tcp
}  // namespace sa

extern "C" int sa_probe_mma_mlp(int chunks, int np, int variant, unsigned long long* out,
                                void* stream) {
  const int smem = 8 * 6144 + 1024;
  cudaFuncSetAttribute(sa::tcp::mma_mlp_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  // variant bit 3: one CTA per SM (full chip)
  sa::tcp::mma_mlp_probe_kernel<<<(variant & 8) ? 148 : 1, 128, smem, sa::as_stream(stream)>>>(
      chunks, np, variant, out);
  return cudaGetLastError() == cudaSuccess ? SA_OK : SA_ERR_CUDA;
}

// ---- operand-pattern probe (diagnostics only) ---------------------------------
// cycles per M=128 K=16 bf16 MMA (N = n) for the operand patterns the fused MLP
// issues: mode 0 one A (TMEM) / one B; 1: A cycles over three TMEM planes;
// 2: A and B cycle over three planes; 3: A from shared memory, cycling;
// 4: as 2, D alternates between two accumulators. rnd: pseudo-random bf16
// operands instead of ones. grid: CTAs (one per SM).
namespace sa {
namespace tcp {
__global__ void __launch_bounds__(128, 1) mma_seq_probe_kernel(int n, int iters, int mode, int rnd,
                                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (6 * 16384) / 4; i += 128)
    reinterpret_cast<uint32_t*>(smem)[i] =
        rnd ? ((uint32_t(i) * 2654435761u) & 0xbfffbfffu) | 0x3c003c00u : 0x3f803f80u;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (tid == 0) {
    mbar_init(&bar, (mode == 16 || mode == 18) ? 2 : 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  {
    uint32_t r[16];
    for (int c = 0; c < 16; ++c)
      r[c] = rnd ? ((uint32_t(tid * 16 + c) * 2246822519u) & 0xbfffbfffu) | 0x3c003c00u : 0x3f803f80u;
    for (int col = 384; col < 512; col += 16) tmem_st16(tmem + (uint32_t(warp * 32) << 16) + col, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (mode == 19 || mode == 20) {
    // mode 19: warp 0 issues the mode-12 MMA stream while warps 1-3 stream
    // tcgen05.ld / st over TMEM columns 256-383 (the GELU pattern); mode 20:
    // the loads / stores alone (warps 1-3), reported as cycles per MMA-slot
    const uint32_t idesc = idesc_bf16_m128(n);
    const uint32_t id32 = idesc_bf16_m128(32);
    const uint32_t sb = smem_u32(smem);
    const uint64_t bpd = (uint32_t(n) * 64) >> 4;
    const long long t0 = clock64();
    if (warp == 0 && mode == 19) {
      for (int i = 0; i < iters; i += 12) {
        const uint64_t b0 = smem_desc(sb + 3 * 16384 + (i & 4) * 64);
        const uint32_t a0 = tmem + 384 + (i & 4) * 2;
        const bool odd = (i / 12) & 1;
#pragma unroll
        for (int u = 0; u < 12; ++u)
          mma_ts_w(tmem + (odd ? 192u : 0u), a0 + uint32_t(u % 3) * 16, b0 + uint64_t(u / 6) * bpd,
                   odd ? id32 : idesc, (i | u) ? 1u : 0u);
      }
      commit_w(&bar);
      mbar_wait(&bar, 0);
    } else if (warp > 0) {
      const uint32_t base = tmem + (uint32_t(warp * 32) << 16) + 256;
      for (int i = 0; i < iters / 4; ++i) {
        float v[16];
        tmem_ld16(base + (i & 3) * 16, v);
        uint32_t r[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) r[t] = __float_as_uint(v[2 * t] + v[2 * t + 1]);
        tmem_st8(base + 64 + (i & 7) * 8, r);
        tmem_st8(base + 96 + (i & 3) * 8, r);
        tmem_st_wait();
      }
    }
    const long long t2 = clock64();
    if (blockIdx.x == 0 && tid == (mode == 19 ? 0 : 32)) {
      out[0] = (unsigned long long)(t2 - t0);
      out[1] = (unsigned long long)(t2 - t0);
    }
  } else if (mode >= 16 && warp < 2) {
    // mode 16: two warps issue concurrently (each 12 MMAs N = n into its own
    // D, then a commit); mode 17: one warp, same stream with the commit;
    // mode 18: two warps, no commits
    const uint32_t idesc = idesc_bf16_m128(n);
    const uint32_t sb = smem_u32(smem);
    const uint64_t bpd = (uint32_t(n) * 64) >> 4;
    __shared__ __align__(8) uint64_t cbar[2];
    if (mode != 17 || warp == 0) {
      const long long t0 = clock64();
      for (int i = 0; i < iters; i += 12) {
        const uint64_t b0 = smem_desc(sb + 3 * 16384 + (i & 4) * 64);
        const uint32_t a0 = tmem + 384 + (i & 4) * 2 + warp * 48;
        const uint32_t d = tmem + warp * 192;
#pragma unroll
        for (int u = 0; u < 12; ++u)
          mma_ts_w(d, a0 + uint32_t(u % 3) * 16, b0 + uint64_t(u / 6) * bpd, idesc, (i | u) ? 1u : 0u);
        if (mode != 18) commit_w(&cbar[warp]);
      }
      const long long t1 = clock64();
      commit_w(&bar);
      if (warp == 0) mbar_wait(&bar, 0);
      const long long t2 = clock64();
      if (blockIdx.x == 0 && tid == 0) {
        out[0] = (unsigned long long)(t1 - t0);
        out[1] = (unsigned long long)(t2 - t0);
      }
    }
  } else if (mode >= 8 && mode < 16 && warp == 0) {
    // warp-wide issue (elect inside the asm), per-MMA operands from the loop
    // counter: mode 8 A / B cycle over three planes; mode 9 + D alternates;
    // mode 10: the same, unrolled x6 from per-iteration base addresses
    const uint32_t idesc = idesc_bf16_m128(n);
    const uint32_t sb = smem_u32(smem);
    const uint32_t bplane = uint32_t(n) * 64;
    const long long t0 = clock64();
    if (mode == 13 || mode == 14 || mode == 15) {
      // mode 12's pattern at the fused MLP's TMEM columns: 13 D = 96 / 288, A at
      // 416 (x planes); 14 D = 0 / 256, A at 416; 15 D = 96 / 288, A at 384
      const uint32_t id32 = idesc_bf16_m128(32);
      const uint32_t dd0 = mode == 14 ? 0u : 96u, dd1 = mode == 14 ? 256u : 288u;
      const uint32_t abase = mode == 15 ? 384u : 416u;
      for (int i = 0; i < iters; i += 12) {
        const uint64_t b0 = smem_desc(sb + 3 * 16384 + (i & 4) * 64);
        const uint32_t a0 = tmem + abase + (i & 4) * 2;
        const uint64_t bpd = bplane >> 4;
#pragma unroll
        for (int u = 0; u < 12; ++u) {
          const bool odd = (i / 12) & 1;
          mma_ts_w(tmem + (odd ? dd1 : dd0), a0 + uint32_t(u % 3) * 16, b0 + uint64_t(u / 6) * bpd,
                   odd ? id32 : idesc, (i | u) ? 1u : 0u);
        }
      }
    } else if (mode == 11 || mode == 12) {
      // mode 11: the same, N alternating n / 32 every MMA; mode 12: 12 MMAs into
      // D0 (N = n) then 12 into D1 (N = 32), as fc1 / fc2 chunks alternate
      const uint32_t id32 = idesc_bf16_m128(32);
      for (int i = 0; i < iters; i += 12) {
        const uint64_t b0 = smem_desc(sb + 3 * 16384 + (i & 4) * 64);
        const uint32_t a0 = tmem + 384 + (i & 4) * 2;
        const uint64_t bpd = bplane >> 4;
#pragma unroll
        for (int u = 0; u < 12; ++u) {
          const bool odd = mode == 11 ? (u & 1) : ((i / 12) & 1);
          mma_ts_w(tmem + (odd ? 192u : 0u), a0 + uint32_t(u % 3) * 16, b0 + uint64_t(u / 6) * bpd,
                   odd ? id32 : idesc, (i | u) ? 1u : 0u);
        }
      }
    } else if (mode == 10) {
      for (int i = 0; i < iters; i += 6) {
        const uint64_t b0 = smem_desc(sb + 3 * 16384 + (i & 2) * 128);
        const uint32_t a0 = tmem + 384 + (i & 2) * 4;
        const uint32_t d = tmem + ((i & 4) ? 192u : 0u);
        const uint64_t bpd = bplane >> 4;
#pragma unroll
        for (int u = 0; u < 6; ++u)
          mma_ts_w(d, a0 + uint32_t(u % 3) * 16, b0 + uint64_t(u / 3) * bpd, idesc, (i | u) ? 1u : 0u);
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        const int pa = i % 3, pb = (i / 3) % 3;
        const uint32_t d = tmem + ((mode == 9 && (i & 1)) ? 192u : 0u);
        const uint64_t bd = smem_desc(sb + 3 * 16384 + uint32_t(pb) * bplane + (i & 1) * 256);
        mma_ts_w(d, tmem + 384 + uint32_t(pa) * 16 + (i & 1) * 8, bd, idesc, i > 0 ? 1u : 0u);
      }
    }
    const long long t1 = clock64();
    commit_w(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0 && (tid & 31) == 0) {
      out[0] = (unsigned long long)(t1 - t0);
      out[1] = (unsigned long long)(t2 - t0);
    }
  } else if (mode < 8 && tid == 0) {
    const uint32_t idesc = idesc_bf16_m128(n);
    const uint32_t sb = smem_u32(smem);
    const uint32_t bplane = uint32_t(n) * 64;   // B plane bytes (n rows x 32 k)
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int pa = (mode >= 1) ? i % 3 : 0;
      const int pb = (mode == 2 || mode == 4) ? (i / 3) % 3 : 0;
      const uint32_t d = tmem + ((mode == 4 && (i & 1)) ? 192u : 0u);
      const uint64_t bd = smem_desc(sb + 3 * 16384 + uint32_t(pb) * bplane + (i & 1) * 256);
      if (mode == 3) {
        const uint64_t ad = smem_desc(sb + uint32_t(pa) * 16384 + (i & 1) * 256);
        mma_bf16(d, ad, bd, idesc, i > 0 ? 1u : 0u);
      } else {
        mma_bf16_ts(d, tmem + 384 + uint32_t(pa) * 16 + (i & 1) * 8, bd, idesc, i > 0 ? 1u : 0u);
      }
    }
    const long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = (unsigned long long)(t1 - t0);
      out[1] = (unsigned long long)(t2 - t0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
}  // namespace tcp
}  // namespace sa

extern "C" int sa_probe_mma_seq(int n, int iters, int mode, int rnd, int grid,
                                unsigned long long* out, void* stream) {
  const int smem = 6 * 16384 + 1024;
  cudaFuncSetAttribute(sa::tcp::mma_seq_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  sa::tcp::mma_seq_probe_kernel<<<grid, 128, smem, sa::as_stream(stream)>>>(n, iters, mode, rnd, out);
  return cudaGetLastError() == cudaSuccess ? SA_OK : SA_ERR_CUDA;
}

// ---- GELU + split throughput probe (diagnostics only) --------------------------
// every thread runs `iters` rounds of 8 GELU pairs (nf of them with the FMA-pipe
// reciprocal) + the bf16 plane split on register data; mode bit 0: skip the
// split, bit 1: skip the GELU. Returns clock cycles of CTA 0.
#include "tc_gemm_kernel.cuh"
namespace sa {
namespace tcp {
template <int NF>
__global__ void __launch_bounds__(512) gelu_probe_kernel(int iters, int mode, float* sink,
                                                         unsigned long long* out) {
  float v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = float(threadIdx.x + t) * 0.001f - 0.3f;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      float g0 = v[2 * t], g1 = v[2 * t + 1];
      if (!(mode & 2)) {
        if (t < NF) tc::gelu_pair<true>(g0, g1);
        else tc::gelu_pair<false>(g0, g1);
      }
      if (!(mode & 1) && (mode & 4)) {   // truncation split (no F2FP)
        const tc::Split3u sp = tc::split3x2_trunc(g0, g1);
        acc += sp.h ^ sp.m ^ sp.l;
      } else if (!(mode & 1)) {
        const tc::Split3 sp = tc::split3x2(g0, g1);
        acc += tc::bf2_bits(sp.h) ^ tc::bf2_bits(sp.m) ^ tc::bf2_bits(sp.l);
      } else {
        acc += __float_as_uint(g0) ^ __float_as_uint(g1);
      }
      v[2 * t] = g0 + 1e-3f;
      v[2 * t + 1] = g1 - 1e-3f;
    }
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u) sink[0] = v[0];
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}
}  // namespace tcp
}  // namespace sa

extern "C" int sa_probe_gelu(int iters, int mode, int nf, int threads, float* sink,
                             unsigned long long* out, void* stream) {
  auto s = sa::as_stream(stream);
  if (nf == 0) sa::tcp::gelu_probe_kernel<0><<<148, threads, 0, s>>>(iters, mode, sink, out);
  else if (nf == 4) sa::tcp::gelu_probe_kernel<4><<<148, threads, 0, s>>>(iters, mode, sink, out);
  else sa::tcp::gelu_probe_kernel<8><<<148, threads, 0, s>>>(iters, mode, sink, out);
  return cudaGetLastError() == cudaSuccess ? SA_OK : SA_ERR_CUDA;
}
