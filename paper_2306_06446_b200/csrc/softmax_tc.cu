// Softmax attention core (the exempt-stage MSA, ref attention.py:92-97) on the
// tensor cores, n <= 256 keys, head dim 32 or 64:
//   out = softmax(q k^T / sqrt(dk)) v      per (image, head)
//
// fp32 parity as in the GEMMs (tcgemm.cu): q, k, p and v enter as exact
// hi/mid/lo bf16 splits and each product is the six plane products whose
// weight is >= 2^-16 (smallest first), accumulated in fp32 in TMEM.
//
// One CTA per (128-query tile, head, image), one CTA per SM (512 TMEM columns):
//   1. q rows → three bf16 planes in TMEM (A of q k^T; thread = query = TMEM
//      lane, warps w / w+4 split the channels); k rows → three K-major planes
//      in shared memory (B; rows = keys).
//   2. S = q k^T: dk/16 K-steps x 6 plane products, N = keys (padded to 32).
//   3. Softmax, thread = query row, the reference's float32 order: s = S /
//      f32(sqrt(dk)); m = max_j s; e_j = exp(s_j - m); t = sum_j e_j;
//      p_j = e_j / t. Pass 1 reads S for the max, pass 2 writes e back over S,
//      pass 3 splits p into three planes per 32-key chunk into a two-slot TMEM
//      ring (A of p v).
//   4. O = p v: per 32-key chunk the v planes (B, K-major: rows = channels)
//      are built in shared memory by warps 4-7 while warps 0-3 write the p
//      planes; 2 K-steps x 6 products per chunk.
//   5. Epilogue: thread = query, O → out (row stride d).
#include "tc_common.cuh"

namespace sa {
namespace smt {

constexpr int kThreads = 256;
constexpr int kMT = 128;
constexpr int kMaxKeys = 256;
constexpr uint32_t kS = 0;        // S / e: columns [0, npad)
// TMEM map: npad <= 96 keys: 256 columns (two CTAs per SM), S [0, 96), q planes
// | p ring [96, 192), O [192, 256); else 512 columns, S [0, 256), q | p ring
// [256, 352), O [384, 448)
__host__ __device__ inline bool small_map(int npad) { return npad <= 96; }

struct Params {
  const float* q;
  const float* k;
  const float* v;
  float* out;
  int n, d, ld, heads;
  float scale_div;   // f32(sqrt(dk)), the reference's divisor
};

template <int DK>
__host__ __device__ inline uint32_t smem_bytes(int n) {
  const uint32_t npad = (uint32_t(n) + 31) & ~31u;
  const uint32_t kpl = 3 * npad * DK * 2;                 // k planes
  const uint32_t vring = 2 * 3 * DK * 64;                 // v planes, two 32-key slots
  return (kpl > vring ? kpl : vring) + 16 * 8;
}

template <int DK>
__global__ void __launch_bounds__(kThreads, 2) softmax_tc_kernel(Params p) {
  constexpr uint32_t kVPlane = DK * 64;       // one v plane of a 32-key chunk
  constexpr uint32_t kVSlot = 3 * kVPlane;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, b = blockIdx.z, n = p.n;
  const int m0 = blockIdx.x * kMT;
  const int npad = (n + 31) & ~31;
  const uint32_t kplane = uint32_t(npad) * DK * 2;   // one k plane
  const uint32_t sb = smem_bytes<DK>(n) - 16 * 8;   // barriers after the operands
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + sb);
  uint64_t* m1 = bars;
  uint64_t* m2 = bars + 1;
  uint64_t* full = bars + 2;    // [2] p planes + v planes of a chunk written
  uint64_t* empty = bars + 4;   // [2] chunk's MMAs done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);
  const size_t row0 = size_t(b) * n;
  const int qq = warp & 3, half = warp >> 2;

  if (tid == 0) {
    tc::mbar_init(m1, 1);
    tc::mbar_init(m2, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(full + s, 4);
      tc::mbar_init(empty + s, 1);
    }
    tc::fence_barrier_init();
  }
  const bool small = small_map(npad);
  const uint32_t kQ = small ? 96u : 256u;      // q planes (MMA1) | p ring (MMA2)
  const uint32_t kO = small ? 192u : 384u;     // O accumulator: dk columns
  if (warp == 0) {
    if (small) tc::tmem_alloc<256>(tslot);
    else tc::tmem_alloc<512>(tslot);
  }
  __shared__ float red[2][kMT];   // cross-warp-group max / sum of each query row
  // ---- k rows → three K-major planes (row = key, K = channels, 32-wide blocks)
  for (int e = tid; e < npad * (DK / 8); e += kThreads) {
    const int kr = e % npad, g = e / npad;   // key, group of 8 channels
    float f[8];
    if (kr < n) {
      const float4* src = reinterpret_cast<const float4*>(p.k + (row0 + kr) * p.ld + h * DK + 8 * g);
      const float4 a = __ldg(src), c = __ldg(src + 1);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = c.x; f[5] = c.y; f[6] = c.z; f[7] = c.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = 0.f;
    }
    uint32_t hw[4], mw[4], lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const tc::Split3 sp = tc::split3x2(f[2 * i], f[2 * i + 1]);
      hw[i] = tc::bf2_bits(sp.h);
      mw[i] = tc::bf2_bits(sp.m);
      lw[i] = tc::bf2_bits(sp.l);
    }
    const uint32_t off = uint32_t(g >> 2) * uint32_t(npad) * 64 + uint32_t(kr >> 3) * 512 +
                         uint32_t(g & 3) * 128 + uint32_t(kr & 7) * 16;
    *reinterpret_cast<uint4*>(smem + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(smem + kplane + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    *reinterpret_cast<uint4*>(smem + 2 * kplane + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t lq = tbase + (uint32_t(32 * qq) << 16);
  const int qi = 32 * qq + lane;            // query in the tile (TMEM lane)
  const bool q_ok = m0 + qi < n;
  // ---- q row (this warp's channel half) → three planes in TMEM --------------
  {
    constexpr int CH = DK / 2;               // channels per warp half
    const float* src = p.q + (row0 + m0 + qi) * p.ld + h * DK + CH * half;
#pragma unroll
    for (int c0 = 0; c0 < CH; c0 += 32) {
      uint32_t hw[16], mw[16], lw[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 a = q_ok && c0 + 4 * i < CH ? __ldg(reinterpret_cast<const float4*>(src + c0) + i)
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        const tc::Split3 s0 = tc::split3x2(a.x, a.y), s1 = tc::split3x2(a.z, a.w);
        hw[2 * i] = tc::bf2_bits(s0.h);
        hw[2 * i + 1] = tc::bf2_bits(s1.h);
        mw[2 * i] = tc::bf2_bits(s0.m);
        mw[2 * i + 1] = tc::bf2_bits(s1.m);
        lw[2 * i] = tc::bf2_bits(s0.l);
        lw[2 * i + 1] = tc::bf2_bits(s1.l);
      }
      // plane pl of channel c at column kQ + pl * DK/2 + c/2
      const uint32_t col = kQ + (CH * half + c0) / 2;
      if (CH - c0 >= 32) {
        tc::tmem_st16(lq + col, hw);
        tc::tmem_st16(lq + DK / 2 + col, mw);
        tc::tmem_st16(lq + DK + col, lw);
      } else {   // CH = 16 (dk = 32): 8 columns per plane
        uint32_t h8[16], m8[16], l8[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          h8[i] = hw[i];
          m8[i] = mw[i];
          l8[i] = lw[i];
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lq + col),
            "r"(h8[0]), "r"(h8[1]), "r"(h8[2]), "r"(h8[3]), "r"(h8[4]), "r"(h8[5]), "r"(h8[6]),
            "r"(h8[7])
            : "memory");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                lq + DK / 2 + col),
            "r"(m8[0]), "r"(m8[1]), "r"(m8[2]), "r"(m8[3]), "r"(m8[4]), "r"(m8[5]), "r"(m8[6]),
            "r"(m8[7])
            : "memory");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lq + DK + col),
            "r"(l8[0]), "r"(l8[1]), "r"(l8[2]), "r"(l8[3]), "r"(l8[4]), "r"(l8[5]), "r"(l8[6]),
            "r"(l8[7])
            : "memory");
      }
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  // ---- S = q k^T (six plane products per K = 16 step) ------------------------
  if (warp == 0) {
    tc::tc_fence_after();
    const uint32_t idS = tc::idesc_bf16_m128(npad);
    const uint32_t s0 = tc::smem_u32(smem);
#pragma unroll
    for (int ks = 0; ks < DK / 16; ++ks) {
      const uint32_t a0 = tbase + kQ + 8 * ks;
      const uint64_t b0 = tc::smem_desc(s0 + uint32_t(ks >> 1) * uint32_t(npad) * 64 + uint32_t(ks & 1) * 256);
      tc::mma_chain6_ts_w(tbase + kS, a0, b0, DK / 2, uint64_t(kplane >> 4), idS, ks > 0 ? 1u : 0u);
    }
    tc::commit_w(m1);
  }
  tc::mbar_wait(m1, 0);
  tc::tc_fence_after();
  const int nch = npad / 32;
  // ---- softmax rows (thread = query); warp group g = warp / 4 takes the
  // 32-key chunks c with c % 2 == g (max and sum combined across the two
  // groups in a fixed order) ------------------------------------------------
  // s = S / f32(sqrt dk): a multiply when the divisor is a power of two (dk 64)
  const bool pow2 = DK == 64;
  const float inv_div = 1.0f / p.scale_div;
  auto scaled = [&](uint32_t bits) {
    return pow2 ? __uint_as_float(bits) * inv_div : __fdiv_rn(__uint_as_float(bits), p.scale_div);
  };
  float mx = -INFINITY;
  for (int c = half; c < nch; c += 2) {
    uint32_t r[32];
    tc::tmem_ld32_nowait(lq + kS + 32 * c, r);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (32 * c + i < n) mx = fmaxf(mx, scaled(r[i]));
  }
  red[half][qi] = mx;
  __syncthreads();
  mx = fmaxf(red[0][qi], red[1][qi]);
  float tot = 0.f;
  for (int c = half; c < nch; c += 2) {
    uint32_t r[32];
    tc::tmem_ld32_nowait(lq + kS + 32 * c, r);
    tc::tmem_ld_wait();
    uint32_t ea[16], eb[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float e = 32 * c + i < n ? expf(scaled(r[i]) - mx) : 0.f;
      tot += e;
      if (i < 16) ea[i] = __float_as_uint(e); else eb[i - 16] = __float_as_uint(e);
    }
    tc::tmem_st16(lq + kS + 32 * c, ea);
    tc::tmem_st16(lq + kS + 32 * c + 16, eb);
  }
  tc::tmem_st_wait();
  __syncthreads();   // (red[][] reads of the max done before the sums overwrite it)
  red[half][qi] = tot;
  __syncthreads();
  tot = red[0][qi] + red[1][qi];
  const float inv = 1.0f / tot;
  // ---- p planes (TMEM ring slot g) + v planes (smem slot g) per chunk; warp 0
  // issues every chunk's p v products in key order --------------------------
  constexpr uint32_t idO = tc::idesc_bf16_m128(DK);
  const int gt = tid & 127;   // thread within the warp group
  for (int c = 0; c < nch; ++c) {
    const int slot = c & 1;
    if (slot == half) {
      if (c >= 2) tc::mbar_wait(empty + slot, uint32_t((c >> 1) - 1) & 1u);
      uint32_t r[32];
      tc::tmem_ld32_nowait(lq + kS + 32 * c, r);
      tc::tmem_ld_wait();
      uint32_t hw[16], mw[16], lw[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const tc::Split3 sp = tc::split3x2(__uint_as_float(r[2 * i]) * inv,
                                           __uint_as_float(r[2 * i + 1]) * inv);
        hw[i] = tc::bf2_bits(sp.h);
        mw[i] = tc::bf2_bits(sp.m);
        lw[i] = tc::bf2_bits(sp.l);
      }
      const uint32_t col = kQ + uint32_t(slot) * 48;
      tc::tmem_st16(lq + col, hw);
      tc::tmem_st16(lq + col + 16, mw);
      tc::tmem_st16(lq + col + 32, lw);
      // v planes of the chunk (rows = channels, K = 32 keys)
      uint8_t* sg = smem + slot * kVSlot;
      for (int e = gt; e < DK * 4; e += 128) {
        const int j = e % DK, tg = e / DK;   // channel, group of 8 keys
        uint32_t vh[4], vm[4], vl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int kr = 32 * c + 8 * tg + 2 * i;
          const float v0 = kr < n ? __ldg(p.v + (row0 + kr) * p.ld + h * DK + j) : 0.f;
          const float v1 = kr + 1 < n ? __ldg(p.v + (row0 + kr + 1) * p.ld + h * DK + j) : 0.f;
          const tc::Split3 sp = tc::split3x2(v0, v1);
          vh[i] = tc::bf2_bits(sp.h);
          vm[i] = tc::bf2_bits(sp.m);
          vl[i] = tc::bf2_bits(sp.l);
        }
        const uint32_t off = uint32_t(j >> 3) * 512 + uint32_t(tg) * 128 + uint32_t(j & 7) * 16;
        *reinterpret_cast<uint4*>(sg + off) = make_uint4(vh[0], vh[1], vh[2], vh[3]);
        *reinterpret_cast<uint4*>(sg + kVPlane + off) = make_uint4(vm[0], vm[1], vm[2], vm[3]);
        *reinterpret_cast<uint4*>(sg + 2 * kVPlane + off) = make_uint4(vl[0], vl[1], vl[2], vl[3]);
      }
      tc::tmem_st_wait();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full + slot);
    }
    if (warp == 0) {
      tc::mbar_wait(full + slot, uint32_t(c >> 1) & 1u);
      tc::tc_fence_after();
      const uint32_t col = kQ + uint32_t(slot) * 48;
      const uint32_t vs = tc::smem_u32(smem + slot * kVSlot);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
        tc::mma_chain6_ts_w(tbase + kO, tbase + col + 8 * ks, tc::smem_desc(vs + ks * 256), 16,
                            uint64_t(kVPlane >> 4), idO, (c > 0 || ks > 0) ? 1u : 0u);
      tc::commit_w(empty + slot);
      if (c == nch - 1) tc::commit_w(m2);
    }
  }
  tc::mbar_wait(m2, 0);
  tc::tc_fence_after();
  // ---- epilogue: thread = query, warp halves split the channels ---------------
  {
    constexpr int CH = DK / 2;
    uint32_t r[32];
    tc::tmem_ld32_nowait(lq + kO + CH * half, r);   // (dk = 32: the upper 16 unused)
    tc::tmem_ld_wait();
    if (q_ok) {
      float* dst = p.out + (row0 + m0 + qi) * p.d + h * DK + CH * half;
#pragma unroll
      for (int i = 0; i < CH / 4; ++i)
        reinterpret_cast<float4*>(dst)[i] =
            make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                        __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    if (small) tc::tmem_dealloc<256>(tbase);
    else tc::tmem_dealloc<512>(tbase);
  }
}

}  // namespace smt

// SA_ERR_VALUE when the shape is outside this kernel's envelope.
int softmax_tc_launch(const float* q, const float* k, const float* v, int64_t ld, float* out,
                      int64_t B, int64_t n, int64_t d, int64_t heads, float scale_div,
                      cudaStream_t s) {
  using namespace smt;
  if (heads <= 0 || d % heads) return SA_ERR_VALUE;
  const int64_t dk = d / heads;
  if ((dk != 32 && dk != 64) || n < 1 || n > kMaxKeys || B > 65535 || heads > 65535)
    return SA_ERR_VALUE;
  if ((ld % 4) || (d % 4) || ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) |
                               reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(out)) &
                              15))
    return SA_ERR_VALUE;
  uint32_t smem = dk == 32 ? smem_bytes<32>(int(n)) : smem_bytes<64>(int(n));
  // 512 TMEM columns per CTA: keep one CTA per SM (a second one would spin in
  // tcgen05.alloc until the first frees its columns)
  if (!small_map(int((n + 31) & ~31)) && smem < 120 * 1024) smem = 120 * 1024;
  Params p{q, k, v, out, int(n), int(d), int(ld), int(heads), scale_div};
  void (*kern)(Params) = dk == 32 ? softmax_tc_kernel<32> : softmax_tc_kernel<64>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  dim3 grid(unsigned((n + kMT - 1) / kMT), unsigned(heads), unsigned(B));
  kern<<<grid, kThreads, smem, s>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("sa_softmax_attn: tensor-core launch failed: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  count_launch(1);
  return SA_OK;
}

}  // namespace sa
