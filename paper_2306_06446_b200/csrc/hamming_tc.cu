// K2b on the tensor cores: quadratic binary (Hamming-space) attention + DWConv
// for the DeiT-T shape (n <= 256 tokens, head dim 32 or 64).
//
// Semantics (the (QK)V order of attention.linear_core on the binary features
// of model.py:355-358 — associativity, ref tests/test_attention.py:72-79 — plus
// the DWConv branch attention.py:170-179 added before W_O, model.py:367-373):
//   S_ij  = popc(cq_i & ck_j)                                  (integer <= dk)
//   out_i = gq*gk * sum_j S_ij v_j / (gq*gk * sum_j S_ij + eps) + dwconv3x3(V)_i
//
// One CTA per (128-query tile, head, image):
//   1. TMA: the head's V (n tokens x dk channels, fp32) as dk/32 boxes of
//      32 channels with the 128-byte swizzle (conflict-free column reads for
//      the transposes and the DWConv); q/k code words by LDG.
//   2. S = Cq · Ck^T on tcgen05: the codes as exact bf16 0/1 operands (K = dk),
//      fp32 accumulator in TMEM (exact integers), converted in place to bf16
//      (exact: S <= 64) — the A operand of the next product, never leaving TMEM.
//   3. O = S · [V_hi | V_mid | V_lo] + S · 1: V as its exact three-plane bf16
//      split (K-major, built per 32-key stage from the staged V, three stages in
//      flight), plus a ones row whose column is the integer row sum of S; the
//      three plane products accumulate in one fp32 accumulator.
//   4. Epilogue (thread = query, warps split the channels): out = O * gq*gk /
//      (gq*gk*rowsum + eps) + DWConv from the swizzled V (taps in the
//      reference's (row, col) order, tensor.py:191-194).
#include "tc_common.cuh"

namespace sa {
namespace ham {

constexpr int kThreads = 256;
constexpr int kMT = 128;           // queries per CTA
constexpr int kNS = 3;             // S·V stages in flight (32 keys each)
constexpr uint32_t kOcol = 128;    // O accumulator: dk value columns + 16 (row-sum column)
constexpr uint32_t kTmemCols = 256;
constexpr int kMaxKeys = 256;

struct Params {
  const uint32_t* cq;
  const uint32_t* ck;
  const float* gq;
  const float* gk;
  const float* dw;
  float* out;
  int n, ld, heads, side;
  float eps;
};

struct Lay {
  uint32_t v, vh, taps, cq, ck, u, b1, bars, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

template <int DK>
__host__ __device__ inline Lay layout(int n) {
  constexpr int W = DK / 32;
  const uint32_t npad = align_up(uint32_t(n), 32);
  Lay L;
  uint32_t o = 0;
  L.v = o;
  L.vh = align_up(uint32_t(n) * 128u, 1024);   // one 32-channel half, 1024-aligned (swizzle)
  o += (DK / 32) * L.vh;
  L.taps = o;
  o += 9 * DK * 4;
  L.cq = o;
  o += kMT * W * 4;
  L.ck = o;
  o += npad * W * 4;
  o = align_up(o, 1024);
  L.u = o;   // union: MMA1 operands | S·V stages
  L.b1 = o + kMT * DK * 2;
  const uint32_t mma1 = kMT * DK * 2 + npad * DK * 2;
  const uint32_t ring = kNS * 3 * (DK + 16) * 64;
  o += mma1 > ring ? mma1 : ring;
  o = align_up(o, 16);
  L.bars = o;
  o += (2 * kNS + 4) * 8;
  L.total = o;
  return L;
}

// two-word (bf16 pair) patterns of code bits
__device__ __forceinline__ uint32_t bits2bf(uint32_t b0, uint32_t b1) {
  return (b0 ? 0x3F80u : 0u) | (b1 ? 0x3F800000u : 0u);
}
__device__ __forceinline__ uint4 byte2bf(uint32_t by) {
  return make_uint4(bits2bf(by & 1u, by & 2u), bits2bf(by & 4u, by & 8u),
                    bits2bf(by & 16u, by & 32u), bits2bf(by & 64u, by & 128u));
}

__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}

template <int DK>
__global__ void __launch_bounds__(kThreads, 2)
    hamming_tc_kernel(Params p, const __grid_constant__ CUtensorMap tmV) {
  constexpr int W = DK / 32;
  constexpr uint32_t kPlane = (DK + 16) * 64;   // one plane of a 32-key stage
  constexpr uint32_t kStage = 3 * kPlane;
  constexpr int kProdWarps = DK * 4 / 32;       // producers of a stage: one item per thread
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, b = blockIdx.z, H = p.heads, n = p.n, side = p.side;
  const int m0 = blockIdx.x * kMT;
  const int nq = min(kMT, n - m0);
  const int npad = (n + 31) & ~31;
  const Lay L = layout<DK>(n);
  uint8_t* Vs = smem + L.v;
  float* taps = reinterpret_cast<float*>(smem + L.taps);
  uint32_t* cqs = reinterpret_cast<uint32_t*>(smem + L.cq);
  uint32_t* cks = reinterpret_cast<uint32_t*>(smem + L.ck);
  uint8_t* U = smem + L.u;
  uint8_t* B1 = smem + L.b1;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + kNS;
  uint64_t* m1 = bars + 2 * kNS;
  uint64_t* m2 = m1 + 1;
  uint64_t* vbar = m1 + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(m1 + 3);

  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(full + s, kProdWarps);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(m1, 1);
    tc::mbar_init(m2, 1);
    tc::mbar_init(vbar, 1);
    tc::fence_barrier_init();
    tc::mbar_expect_tx(vbar, uint32_t(DK / 32) * uint32_t(n) * 128u);
    for (int hf = 0; hf < DK / 32; ++hf)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(Vs + hf * L.vh)),
          "l"(reinterpret_cast<uint64_t>(&tmV)), "r"(h * DK + 32 * hf), "r"(0), "r"(b),
          "r"(tc::smem_u32(vbar))
          : "memory");
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(tslot);
  {
    const size_t base = (size_t(b) * H + h) * n;
    for (int i = tid; i < kMT * W; i += kThreads)
      cqs[i] = i < nq * W ? __ldg(p.cq + (base + m0) * W + i) : 0u;
    for (int i = tid; i < npad * W; i += kThreads)
      cks[i] = i < n * W ? __ldg(p.ck + base * W + i) : 0u;
    for (int i = tid; i < 9 * DK; i += kThreads)
      taps[i] = p.dw ? __ldg(p.dw + (i / DK) * p.ld + h * DK + (i % DK)) : 0.f;
  }
  __syncthreads();
  // ---- MMA1 operands: Cq tile (128 rows) and Ck (npad rows), K = dk bits,
  // K-major in 32-wide K halves; one item = 8 code bits of one row
  for (int e = tid; e < (kMT + npad) * (DK / 8); e += kThreads) {
    const bool isq = e < kMT * (DK / 8);
    const int e2 = isq ? e : e - kMT * (DK / 8);
    const int rows = isq ? kMT : npad;
    const int r = e2 % rows, g = e2 / rows;
    const uint32_t wd = (isq ? cqs : cks)[r * W + (g >> 2)];
    const uint32_t off = uint32_t(g >> 2) * uint32_t(rows) * 64 + uint32_t(r >> 3) * 512 +
                         uint32_t(g & 3) * 128 + uint32_t(r & 7) * 16;
    *reinterpret_cast<uint4*>((isq ? U : B1) + off) = byte2bf((wd >> (8 * (g & 3))) & 0xFFu);
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 0) {
    const uint32_t idS = tc::idesc_bf16_m128(npad);
#pragma unroll
    for (int ks = 0; ks < DK / 16; ++ks) {
      const uint64_t ad = tc::smem_desc(tc::smem_u32(U) + uint32_t(ks >> 1) * (kMT * 64) +
                                        uint32_t(ks & 1) * 256);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(B1) + uint32_t(ks >> 1) * uint32_t(npad) * 64 +
                                        uint32_t(ks & 1) * 256);
      mma_ss_w(tbase, ad, bd, idS, ks > 0 ? 1u : 0u);
    }
    tc::commit_w(m1);
  }
  tc::mbar_wait(m1, 0);
  tc::tc_fence_after();
  // ---- S (fp32, exact integers) → bf16 pairs in place: A operand of S·V ------
  if (warp < 4) {
    const uint32_t lq = tbase + (uint32_t(32 * warp) << 16);
    for (int c = 0; c < npad / 32; ++c) {
      uint32_t r[32], o[16];
      tc::tmem_ld32_nowait(lq + 32 * c, r);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i)
        o[i] = tc::bf2_bits(__floats2bfloat162_rn(__uint_as_float(r[2 * i]),
                                                  __uint_as_float(r[2 * i + 1])));
      tc::tmem_st16(lq + 16 * c, o);
    }
    tc::tmem_st_wait();
  } else {
    // constant rows of every S·V stage: plane 0 row dk = 1.0 (row sums), rows
    // dk+1..dk+15 and planes 1, 2 rows dk.. = 0 (the MMA1 operands are dead)
    for (int i = tid - 128; i < kNS * 3 * 64; i += 128) {
      const int s = i / 192, pl = (i / 64) % 3, e = i % 64;
      const int gr = e >> 5, ch = e & 31;   // row group dk/8 + gr, 16-byte chunk
      const bool one = pl == 0 && gr == 0 && (ch & 7) == 0;
      const uint32_t v = one ? 0x3F803F80u : 0u;
      *reinterpret_cast<uint4*>(U + s * kStage + pl * kPlane + (DK / 8 + gr) * 512 + ch * 16) =
          make_uint4(v, v, v, v);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::mbar_wait(vbar, 0);

  // ---- O = S · V planes (+ row sums), 32-key stages -------------------------
  const int KS = npad / 32;
  constexpr uint32_t idO = tc::idesc_bf16_m128(DK + 16);
  if (warp < kProdWarps) {
    const int j = tid % DK, tg = tid / DK;   // channel, group of 8 keys
    const uint8_t* vcol = Vs + (j >> 5) * L.vh + (j & 3) * 4;
    const int jc = (j & 31) >> 2;            // 16-byte chunk of the channel
#pragma unroll 1
    for (int st = 0; st < KS; ++st) {
      const int slot = st % kNS;
      if (st >= kNS) tc::mbar_wait(empty + slot, uint32_t(st / kNS - 1) & 1u);
      uint8_t* sg = U + slot * kStage;
      uint32_t hw[4], mw[4], lw[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 32 * st + 8 * tg + 2 * i;
        const float v0 =
            k < n ? *reinterpret_cast<const float*>(vcol + k * 128 + ((jc ^ (k & 7)) << 4)) : 0.f;
        const float v1 = k + 1 < n ? *reinterpret_cast<const float*>(
                                         vcol + (k + 1) * 128 + ((jc ^ ((k + 1) & 7)) << 4))
                                   : 0.f;
        const tc::Split3 sp = tc::split3x2(v0, v1);
        hw[i] = tc::bf2_bits(sp.h);
        mw[i] = tc::bf2_bits(sp.m);
        lw[i] = tc::bf2_bits(sp.l);
      }
      const uint32_t off = uint32_t(j >> 3) * 512 + uint32_t(tg) * 128 + uint32_t(j & 7) * 16;
      *reinterpret_cast<uint4*>(sg + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(sg + kPlane + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
      *reinterpret_cast<uint4*>(sg + 2 * kPlane + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(full + slot);
      if (warp == 0) {
        tc::mbar_wait(full + slot, uint32_t(st / kNS) & 1u);
        tc::tc_fence_after();
        const uint32_t sb = tc::smem_u32(sg);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int pl = 2; pl >= 0; --pl)   // lo, mid, hi: smallest products first
            tc::mma_ts_w(tbase + kOcol, tbase + 8 * (2 * st + ks),
                         tc::smem_desc(sb + uint32_t(pl) * kPlane + uint32_t(ks) * 256), idO,
                         (st == 0 && ks == 0 && pl == 2) ? 0u : 1u);
        tc::commit_w(empty + slot);
      }
    }
    if (warp == 0) tc::commit_w(m2);
  }
  tc::mbar_wait(m2, 0);
  tc::tc_fence_after();

  // ---- epilogue: thread = query, warp pair (w, w+4) splits the channels ------
  const int qq = warp & 3, half = warp >> 2;
  if (half < DK / 32) {
    const int qi = 32 * qq + lane;   // query in the tile (TMEM lane)
    const uint32_t lq = tbase + (uint32_t(32 * qq) << 16);
    uint32_t o[32];
    tc::tmem_ld32_nowait(lq + kOcol + 32 * half, o);
    const uint32_t dn = tmem_ld1(lq + kOcol + DK);
    tc::tmem_ld_wait();
    if (qi < nq) {
      const int t = m0 + qi;
      const float gg = __ldg(p.gq + b * H + h) * __ldg(p.gk + b * H + h);
      const float sc = __fdiv_rn(gg, __fadd_rn(__fmul_rn(gg, __uint_as_float(dn)), p.eps));
      const int r = t / side, c = t - r * side;
      int tok[9];
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const int rr = r + di - 1, cc = c + dj - 1;
          const int k = rr * side + cc;
          tok[di * 3 + dj] = (p.dw && rr >= 0 && rr < side && cc >= 0 && cc < side && k < n) ? k : -1;
        }
      const uint8_t* vh = Vs + half * L.vh;
      float* op = p.out + (size_t(b) * n + t) * p.ld + h * DK + 32 * half;
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          const int k = tok[q];
          const float4 v4 = k >= 0 ? *reinterpret_cast<const float4*>(vh + k * 128 + ((c4 ^ (k & 7)) << 4))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 t4 = *reinterpret_cast<const float4*>(taps + q * DK + 32 * half + 4 * c4);
          s[0] = fmaf(v4.x, t4.x, s[0]);
          s[1] = fmaf(v4.y, t4.y, s[1]);
          s[2] = fmaf(v4.z, t4.z, s[2]);
          s[3] = fmaf(v4.w, t4.w, s[3]);
        }
        float4 y;
        y.x = __fadd_rn(__fmul_rn(__uint_as_float(o[4 * c4 + 0]), sc), s[0]);
        y.y = __fadd_rn(__fmul_rn(__uint_as_float(o[4 * c4 + 1]), sc), s[1]);
        y.z = __fadd_rn(__fmul_rn(__uint_as_float(o[4 * c4 + 2]), sc), s[2]);
        y.w = __fadd_rn(__fmul_rn(__uint_as_float(o[4 * c4 + 3]), sc), s[3]);
        *reinterpret_cast<float4*>(op + 4 * c4) = y;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace ham

// SA_ERR_VALUE when the shape is outside this kernel's envelope (the caller
// then uses the CUDA-core kernel of binattn.cu).
int hamming_tc_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                      const float* v, const float* dw, float* out, int64_t B, int64_t n,
                      int64_t d, int64_t heads, float eps, cudaStream_t s) {
  using namespace ham;
  if (heads <= 0 || d % heads) return SA_ERR_VALUE;
  const int64_t dk = d / heads;
  if (dk != 32 && dk != 64) return SA_ERR_VALUE;
  if (n < 1 || n > kMaxKeys || B < 1 || B > 65535 || heads > 65535) return SA_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(v) & 15) != 0) return SA_ERR_VALUE;
  int side = 0;
  while (int64_t(side) * side < n) ++side;
  const Lay L = dk == 32 ? layout<32>(int(n)) : layout<64>(int(n));
  if (L.total > 200 * 1024) return SA_ERR_VALUE;
  Params p{cq, ck, gq, gk, dw, out, int(n), int(d), int(heads), side, eps};
  void (*kern)(Params, CUtensorMap) = dk == 32 ? hamming_tc_kernel<32> : hamming_tc_kernel<64>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
  CUtensorMap tmV;
  memset(&tmV, 0, sizeof(tmV));
  const cuuint64_t dims[3] = {cuuint64_t(d), cuuint64_t(n), cuuint64_t(B)};
  const cuuint64_t strides[2] = {cuuint64_t(d) * 4, cuuint64_t(n) * cuuint64_t(d) * 4};
  const cuuint32_t box[3] = {32u, cuuint32_t(n), 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode_tmap_tiled(&tmV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(v), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SA_ERR_VALUE;
  dim3 grid(unsigned((n + kMT - 1) / kMT), unsigned(heads), unsigned(B));
  kern<<<grid, kThreads, L.total, s>>>(p, tmV);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("sa_hamming_attn: tensor-core launch failed: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  count_launch(1);
  return SA_OK;
}

}  // namespace sa
