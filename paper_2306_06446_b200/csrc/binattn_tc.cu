// K2a on the tensor cores: binary linear attention + DWConv, head dim 32 or 64.
//
// Semantics (ref attention.py:113-120 on the binary features of
// model.py:355-358, DWConv branch attention.py:170-179 added before W_O,
// model.py:367-373), per (image, head):
//   S[j][a]  = sum_{t : ck[t][a]} v_t[j]             (K^T V, additions only)
//   cnt[a]   = sum_t ck[t][a]                         (integer)
//   out_t[j] = gq*gk * sum_{a : cq[t][a]} S[j][a] / (gq*gk*sum_{a : cq[t][a]} cnt[a] + eps)
//              + dwconv3x3(V)_t[j]
//
// Both contractions have a {0,1} operand, so they run on tcgen05 with bf16
// operands and fp32 accumulation: V (fp32) enters as its exact hi/mid/lo bf16
// split, the codes as exact 0.0/1.0. Nothing is rounded before the fp32
// accumulator; the accumulation itself is the tensor core's fp32.
//
// Work unit = (image, head, 32-channel slice of V): the V channels of a head
// are independent in both products, so a dk = 64 head is two units that share
// the code words (each unit contracts all dk code bits). One thread-block
// cluster per unit; CTA `rank` owns a band of BR rows of the token grid
// (side = ceil(sqrt n), row-major, zero padded):
//   1. TMA: the band's V rows (+1 halo row above and below; rows outside the
//      grid and cells past n arrive as zeros) → shared memory, 128 B / token;
//      V is read from HBM exactly once. The band's q/k code words by LDG.
//   2. Phase A (K^T V): 32-token stages, two in flight. Warps 0-3 write the
//      A operand = [V_hi; V_mid; V_lo; ones] (M = 128 rows = plane x channel,
//      K = tokens), warps 4-7 the B operand = K codes as bf16 (N = dk rows,
//      K = tokens); one elected lane issues M=128 x N=dk x K=16 MMAs into
//      TMEM. Lanes 0-95 hold the three plane partials of S, lane 96 (the ones
//      row) the code-bit counts.
//   3. The planes are summed ((hi + mid) + lo) into the band partial; the CL
//      partials are exchanged through distributed shared memory and summed in
//      rank order (deterministic, identical in every CTA of the cluster).
//   4. Phase B (Q (K^T V), transposed so TMEM lanes are channels): A = S split
//      into three bf16 planes in TMEM, replicated in the four lane quarters;
//      B = Q codes of 64 tokens as bf16 (K-major); three plane MMAs per K=16
//      step accumulate num[j][token] in one fp32 accumulator (double-buffered,
//      the next tile's MMAs run under this tile's epilogue).
//   5. Epilogue: warp w reads 8 tokens of its lane quarter (lane = channel),
//      scales by gq*gk / (gq*gk*D + eps) (D = the integer code-count dot,
//      computed once per token), adds the 3x3 DWConv from a register sliding
//      window over the staged band, and stores 128 B per token (coalesced).
#include <cooperative_groups.h>

#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace sa {
namespace bat {

constexpr int kThreads = 256;
constexpr int kNS = 2;             // phase-A stages in flight (32 tokens each)
constexpr int kTileB = 64;         // phase-B tokens per accumulator tile
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kAccA = 0;      // phase-A accumulator: columns [0, dk)
constexpr uint32_t kAccB = 0;      // phase-B accumulators: [0, 64), [64, 128)
constexpr uint32_t kKvCol = 128;   // S planes (A operand of phase B): 3 * dk/2 columns
constexpr uint32_t kStageA = 8192; // 128 rows x 32 tokens bf16
constexpr int kMaxBandTokens = 400;
constexpr int kMaxBandRows = 24;   // per-row V barriers (band rows <= 400 / side or <= side)

struct Params {
  const uint32_t* cq;
  const uint32_t* ck;
  const float* gq;
  const float* gk;
  const float* dw;
  float* out;
  int n, ld, heads, side, rows_total, band_rows;
  float eps;
};

struct Lay {
  uint32_t v, cq, ck, sc, xp, kv, ring, bars, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

template <int DKC>
__host__ __device__ inline Lay layout(int side, int band_rows) {
  constexpr int W = DKC / 32;
  constexpr uint32_t KP = DKC + 4;
  const uint32_t tmax = uint32_t(band_rows) * side;
  Lay L;
  uint32_t o = 0;
  L.v = o;
  o += uint32_t(band_rows + 2) * side * 128u;
  o = align_up(o, 16);
  const uint32_t tpad = align_up(tmax, 64);   // codes zero-padded to whole phase-B tiles
  L.cq = o;
  o += tpad * W * 4;
  L.ck = o;
  o += tpad * W * 4;
  o = align_up(o, 16);
  L.sc = o;                                  // per-token scale (+ slack for 8-token reads)
  o += (tmax + 64) * 4;
  o = align_up(o, 16);
  L.xp = o;                                  // exchange: [32][KP] partial S + [DKC] counts
  o += (32 * KP + DKC) * 4;
  o = align_up(o, 16);
  o = align_up(o, 1024);
  L.ring = o;   // union: phase-A stages | plane scratch | summed S + count masks | B tiles
  L.kv = o;
  const uint32_t ringA = kNS * (kStageA + DKC * 64);
  const uint32_t scr = 2 * 32 * KP * 4;
  const uint32_t tilesB = 2 * kTileB * DKC * 2;
  const uint32_t kvm = (32 * KP + DKC) * 4 + 4 * 24 * W * 4;
  uint32_t u = ringA > scr ? ringA : scr;
  u = u > kvm ? u : kvm;
  u = u > tilesB ? u : tilesB;
  o += u;
  o = align_up(o, 16);
  L.bars = o;
  o += (2 * kNS + 4 + kMaxBandRows + 2) * 8;
  L.total = o;
  return L;
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

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}

// two code bits → bf16 pair (0.0 / 1.0 each), low half = first bit
__device__ __forceinline__ uint32_t bits2bf(uint32_t b0, uint32_t b1) {
  return (b0 ? 0x3F80u : 0u) | (b1 ? 0x3F800000u : 0u);
}

#ifdef BAT_PROF
__device__ unsigned long long* g_bat_prof = nullptr;
#define BAT_PROF_MARK_T(i, th)                                                                 \
  if (tid == (th) && g_bat_prof)                                                                 \
    g_bat_prof[((size_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + \
               (i)] = clock64();
#define BAT_PROF_MARK(i) BAT_PROF_MARK_T(i, 0)
#else
#define BAT_PROF_MARK(i)
#define BAT_PROF_MARK_T(i, th)
#endif

template <int DKC>
__global__ void __launch_bounds__(kThreads, 2)
    binattn_tc_kernel(Params p, const __grid_constant__ CUtensorMap tmV) {
  constexpr int W = DKC / 32;          // code words per token
  constexpr int S = DKC / 32;          // V slices per head
  constexpr int KP = DKC + 4;          // padded fp32 row of the S exchange buffers
  constexpr uint32_t kStageB = DKC * 64;   // K codes of 32 tokens as bf16
  constexpr uint32_t kTileBytes = kTileB * DKC * 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CL = int(cluster.num_blocks());
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  BAT_PROF_MARK(7);
  const int b = blockIdx.z;
  const int h = blockIdx.y / S, sl = blockIdx.y - (blockIdx.y / S) * S;
  const int side = p.side, n = p.n, BR = p.band_rows, H = p.heads;
  const uint32_t ROWB = uint32_t(side) * 128u;
  const Lay L = layout<DKC>(side, BR);
  uint8_t* Vb = smem + L.v;
  uint32_t* cqs = reinterpret_cast<uint32_t*>(smem + L.cq);
  uint32_t* cks = reinterpret_cast<uint32_t*>(smem + L.ck);
  float* scs = reinterpret_cast<float*>(smem + L.sc);
  float* xP = reinterpret_cast<float*>(smem + L.xp);
  float* KVs = reinterpret_cast<float*>(smem + L.kv);
  uint8_t* ring = smem + L.ring;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + kNS;
  uint64_t* accA = bars + 2 * kNS;
  uint64_t* mfull = accA + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mfull + 2);
  uint64_t* vbar = bars + 2 * kNS + 4;   // one per smem row of the V band

  const int r0 = rank * BR;
  const int r1 = min(p.rows_total, r0 + BR);
  const int t_lo = min(n, r0 * side), t_hi = min(n, r1 * side);
  const int T = t_hi - t_lo;

  // ---- 1. V band (TMA), codes, constant operand rows ------------------------
  if (tid == 0) {
    for (int R = 0; R < BR + 2; ++R) tc::mbar_init(vbar + R, 1);
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(full + s, kThreads / 32);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(accA, 1);
    tc::mbar_init(mfull, 1);
    tc::mbar_init(mfull + 1, 1);
    tc::fence_barrier_init();
    // smem row R = grid row r0 - 1 + R: the head slice's 32 channels x side
    // tokens; rows outside the grid / cells past n are out of bounds → zeros.
    // Band rows first (phase A starts on them), the two halo rows last.
    for (int i = 0; i < BR + 2; ++i) {
      const int R = i < BR ? i + 1 : (i == BR ? 0 : BR + 1);
      const int rr = r0 - 1 + R;
      tc::mbar_expect_tx(vbar + R, ROWB);
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(Vb + R * ROWB)),
          "l"(reinterpret_cast<uint64_t>(&tmV)), "r"(h * DKC + 32 * sl), "r"(rr * side), "r"(b),
          "r"(tc::smem_u32(vbar + R))
          : "memory");
    }
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(tslot);
  {
    const size_t c0 = ((size_t(b) * H + h) * n + t_lo) * W;
    const int Tp = (T + 63) & ~63;
    for (int i = tid; i < Tp * W; i += kThreads) {
      const bool in = i < T * W;
      cqs[i] = in ? __ldg(p.cq + c0 + i) : 0u;
      cks[i] = in ? __ldg(p.ck + c0 + i) : 0u;
    }
  }
  // rows 96..127 of every phase-A A stage: bf16 1.0 (the count row; 97..127 unused)
  for (int i = tid; i < kNS * 128; i += kThreads) {
    const int s = i >> 7, e = i & 127;
    reinterpret_cast<uint4*>(ring + s * (kStageA + DKC * 64) + 12 * 512)[e] =
        make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  }
  float tap[9];
  const int ch = h * DKC + 32 * sl + lane;   // model channel of this lane
  const bool has_dw = p.dw != nullptr;
#pragma unroll
  for (int q = 0; q < 9; ++q) tap[q] = has_dw ? __ldg(p.dw + q * p.ld + ch) : 0.f;
  const float gq = __ldg(p.gq + b * H + h), gk = __ldg(p.gk + b * H + h);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  BAT_PROF_MARK(0);

  // ---- 2. phase A: S partial of the band ------------------------------------
  // 32-token stages, kNS in flight: warps 0-3 write the A operand (V planes,
  // rows 32p + j, K = tokens), warps 4-7 the B operand (K codes as bf16, rows
  // = code bit); warp 0 issues the stage's two MMAs when all eight arrived.
  const int KS = (T + 31) >> 5;
  int rows_ok = 0;   // band rows (smem rows 1..) this thread has waited for
  constexpr uint32_t idA = tc::idesc_bf16_m128(DKC);
  const uint8_t* vband = Vb + ROWB;   // band token u at vband + u * 128
#pragma unroll 1
  for (int st = 0; st < KS; ++st) {
    const int slot = st & (kNS - 1);
    if (st >= kNS) tc::mbar_wait(empty + slot, uint32_t((st / kNS) - 1) & 1u);
    uint8_t* sA = ring + slot * (kStageA + kStageB);
    uint8_t* sB = sA + kStageA;
    if (warp < 4) {   // A rows 32p + j (plane p of channel j = lane), tokens 8*warp..+7
      uint32_t hw[4], mw[4], lw[4];
      const int u0 = 32 * st + 8 * warp;
      const bool whole = u0 + 8 <= T;
      const int need = min(BR, (min(u0 + 8, T) - 1) / side + 1);   // band rows of these tokens
      while (rows_ok < need) tc::mbar_wait(vbar + 1 + rows_ok++, 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = u0 + 2 * i;
        const float* vp = reinterpret_cast<const float*>(vband + u * 128) + lane;
        const float v0 = (whole || u < T) ? vp[0] : 0.f;
        const float v1 = (whole || u + 1 < T) ? vp[32] : 0.f;
        const tc::Split3 sp = tc::split3x2(v0, v1);
        hw[i] = tc::bf2_bits(sp.h);
        mw[i] = tc::bf2_bits(sp.m);
        lw[i] = tc::bf2_bits(sp.l);
      }
      const uint32_t off = uint32_t(lane >> 3) * 512 + uint32_t(warp) * 128 + uint32_t(lane & 7) * 16;
      *reinterpret_cast<uint4*>(sA + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(sA + 2048 + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
      *reinterpret_cast<uint4*>(sA + 4096 + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    } else {          // B rows = code bit c, tokens 8*(warp-4)..+7 (codes are zero past T)
      const int tg = warp - 4;
      const int u0 = 32 * st + 8 * tg;
#pragma unroll
      for (int cw = 0; cw < W; ++cw) {
        uint32_t bit[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) bit[i] = (cks[(u0 + i) * W + cw] >> lane) & 1u;
        const int c = 32 * cw + lane;
        const uint32_t off = uint32_t(c >> 3) * 512 + uint32_t(tg) * 128 + uint32_t(c & 7) * 16;
        *reinterpret_cast<uint4*>(sB + off) =
            make_uint4(bits2bf(bit[0], bit[1]), bits2bf(bit[2], bit[3]), bits2bf(bit[4], bit[5]),
                       bits2bf(bit[6], bit[7]));
      }
    }
    tc::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(full + slot);
    if (warp == 0) {
      tc::mbar_wait(full + slot, uint32_t(st / kNS) & 1u);
      tc::tc_fence_after();
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sA));
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sB));
      mma_ss_w(tbase + kAccA, ad, bd, idA, st > 0 ? 1u : 0u);
      mma_ss_w(tbase + kAccA, ad + (256 >> 4), bd + (256 >> 4), idA, 1u);
      tc::commit_w(empty + slot);
      if (st == 0) { BAT_PROF_MARK_T(9, 0); }
    }
  }
  if (warp == 0) tc::commit_w(accA);
  for (int R = 0; R < BR + 2; ++R) tc::mbar_wait(vbar + R, 0);   // halos (+ rows for warps 4-7)
  tc::mbar_wait(accA, 0);
  BAT_PROF_MARK(1);
  tc::tc_fence_after();
  float* scr = reinterpret_cast<float*>(ring);   // [2][32][KP]: mid, lo planes
  if (warp >= 1 && warp < 4) {
#pragma unroll
    for (int cw = 0; cw < W; ++cw) {
      uint32_t r[32];
      tc::tmem_ld32_nowait(tbase + (uint32_t(32 * warp) << 16) + kAccA + 32 * cw, r);
      tc::tmem_ld_wait();
      if (warp < 3) {
        float* row = scr + (warp - 1) * 32 * KP + lane * KP + 32 * cw;
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          *reinterpret_cast<float4*>(row + c) =
              make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                          __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
      } else if (lane == 0) {
#pragma unroll
        for (int c = 0; c < 32; ++c) xP[32 * KP + 32 * cw + c] = __uint_as_float(r[c]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int cw = 0; cw < W; ++cw) {
      uint32_t r[32];
      tc::tmem_ld32_nowait(tbase + kAccA + 32 * cw, r);
      tc::tmem_ld_wait();
      const float* m1 = scr + lane * KP + 32 * cw;
      const float* m2 = scr + 32 * KP + lane * KP + 32 * cw;
      float* dst = xP + lane * KP + 32 * cw;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 a = *reinterpret_cast<const float4*>(m1 + c);
        const float4 z = *reinterpret_cast<const float4*>(m2 + c);
        float4 o;
        o.x = __fadd_rn(__fadd_rn(__uint_as_float(r[c]), a.x), z.x);
        o.y = __fadd_rn(__fadd_rn(__uint_as_float(r[c + 1]), a.y), z.y);
        o.z = __fadd_rn(__fadd_rn(__uint_as_float(r[c + 2]), a.z), z.z);
        o.w = __fadd_rn(__fadd_rn(__uint_as_float(r[c + 3]), a.w), z.w);
        *reinterpret_cast<float4*>(dst + c) = o;
      }
    }
  }
  tc::tc_fence_before();
  // ---- 4. cluster exchange: S = sum over bands in rank order ------------------
  cluster.sync();
  BAT_PROF_MARK(2);
  {
    constexpr int C4 = DKC / 4;
    for (int e = tid; e < 33 * C4; e += kThreads) {
      const int j = e / C4, c4 = e - j * C4;
      const int off = j * KP + 4 * c4;   // j == 32: the count row
      float4 o[8];   // all remote loads in flight before the (rank-ordered) sum
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < CL) o[r] = *reinterpret_cast<const float4*>(cluster.map_shared_rank(xP, r) + off);
      float4 acc = o[0];
#pragma unroll
      for (int r = 1; r < 8; ++r) {
        if (r < CL) {
          acc.x = __fadd_rn(acc.x, o[r].x);
          acc.y = __fadd_rn(acc.y, o[r].y);
          acc.z = __fadd_rn(acc.z, o[r].z);
          acc.w = __fadd_rn(acc.w, o[r].w);
        }
      }
      *reinterpret_cast<float4*>(KVs + off) = acc;
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  BAT_PROF_MARK(3);
  const float gg = gq * gk;
  if (warp < 4) {
    // S (row j = lane) as three bf16 planes into this warp's TMEM lane quarter:
    // column kKvCol + p*dk/2 + c/2 holds the pair (c, c+1) of plane p
    const float* row = KVs + lane * KP;
    const uint32_t tq = tbase + (uint32_t(32 * warp) << 16) + kKvCol;
#pragma unroll
    for (int cw = 0; cw < W; ++cw) {
      uint32_t ph[16], pm[16], pl[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 v2 = *reinterpret_cast<const float2*>(row + 32 * cw + 2 * i);
        const tc::Split3 sp = tc::split3x2(v2.x, v2.y);
        ph[i] = tc::bf2_bits(sp.h);
        pm[i] = tc::bf2_bits(sp.m);
        pl[i] = tc::bf2_bits(sp.l);
      }
      tc::tmem_st16(tq + 16 * cw, ph);
      tc::tmem_st16(tq + DKC / 2 + 16 * cw, pm);
      tc::tmem_st16(tq + DKC + 16 * cw, pl);
    }
    tc::tmem_st_wait();
  } else {
    // per-token scale gq*gk / (gq*gk*D + eps), D = sum of the code-bit counts
    // over the set q bits, bit-sliced: D = sum_k popc(q & mask_k) << k where
    // mask_k = the code bits whose count has bit k (integers, exact)
    const float* cnt = KVs + 32 * KP;
    uint32_t* mk = reinterpret_cast<uint32_t*>(KVs + 32 * KP + DKC) + (warp - 4) * 24 * W;
    uint32_t cmax = 0;
#pragma unroll
    for (int cw = 0; cw < W; ++cw) {
      const uint32_t cv = uint32_t(cnt[32 * cw + lane]);
      cmax = max(cmax, cv);
#pragma unroll
      for (int k = 0; k < 24; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, (cv >> k) & 1u);
        if (lane == 0) mk[k * W + cw] = m;
      }
    }
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    const int nb = 32 - __clz(int(cmax));
    __syncwarp();
    for (int u = tid - 128; u < T; u += 128) {
      uint32_t D = 0;
#pragma unroll
      for (int cw = 0; cw < W; ++cw) {
        const uint32_t wd = cqs[u * W + cw];
        for (int k = 0; k < nb; ++k) D += uint32_t(__popc(wd & mk[k * W + cw])) << k;
      }
      scs[u] = __fdiv_rn(gg, __fadd_rn(__fmul_rn(gg, float(D)), p.eps));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  BAT_PROF_MARK(4);
  // ---- 5. phase B: num[j][token] = sum_a S[j][a] cq[token][a] ----------------
  const int NT = (T + kTileB - 1) / kTileB;
  constexpr uint32_t idB = tc::idesc_bf16_m128(kTileB);
  auto build = [&](int i) {   // Q codes of tile i as bf16, K-major, 32-wide K halves
    uint8_t* dst = ring + (i & 1) * kTileBytes;
    for (int e = tid; e < kTileB * (DKC / 8); e += kThreads) {
      const int ul = e & (kTileB - 1), g = e / kTileB;   // token in tile, group of 8 bits
      const int u = kTileB * i + ul;
      const uint32_t wd = cqs[u * W + (g >> 2)];   // zero past T
      const uint32_t by = (wd >> (8 * (g & 3))) & 0xFFu;
      const uint32_t off = uint32_t(g >> 2) * (kTileB * 64) + uint32_t(ul >> 3) * 512 +
                           uint32_t(g & 3) * 128 + uint32_t(ul & 7) * 16;
      *reinterpret_cast<uint4*>(dst + off) =
          make_uint4(bits2bf(by & 1u, by & 2u), bits2bf(by & 4u, by & 8u),
                     bits2bf(by & 16u, by & 32u), bits2bf(by & 64u, by & 128u));
    }
    tc::fence_proxy_async_smem();
  };
  auto issue = [&](int i) {   // warp 0, whole warp
    const uint32_t acc = tbase + kAccB + uint32_t(i & 1) * kTileB;
    const uint32_t sb = tc::smem_u32(ring + (i & 1) * kTileBytes);
#pragma unroll
    for (int ks = 0; ks < DKC / 16; ++ks) {
      const uint64_t bd = tc::smem_desc(sb + uint32_t(ks >> 1) * (kTileB * 64) + uint32_t(ks & 1) * 256);
#pragma unroll
      for (int pp = 2; pp >= 0; --pp)   // lo, mid, hi: smallest products first
        tc::mma_ts_w(acc, tbase + kKvCol + uint32_t(pp) * (DKC / 2) + 8 * ks, bd, idB,
                     (ks == 0 && pp == 2) ? 0u : 1u);
    }
    tc::commit_w(mfull + (i & 1));
  };
  const int q = warp & 3;   // TMEM lane quarter of this warp
  float* outp = p.out + size_t(b) * n * p.ld + ch;
  if (NT > 0) {
    build(0);
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
      tc::tc_fence_after();
      issue(0);
    }
  }
#pragma unroll 1
  for (int i = 0; i < NT; ++i) {
    if (i + 1 < NT) {
      build(i + 1);   // its buffer was last read by MMA(i-1), waited for in iteration i-1
      tc::tc_fence_before();
      __syncthreads();   // + the epilogue of tile i-1 is done with accumulator (i+1)&1
      if (warp == 0) {
        tc::tc_fence_after();
        issue(i + 1);
      }
    }
    tc::mbar_wait(mfull + (i & 1), uint32_t(i >> 1) & 1u);
    tc::tc_fence_after();
    uint32_t r[8];
    tmem_ld8(tbase + (uint32_t(32 * q) << 16) + kAccB + uint32_t(i & 1) * kTileB + 8 * warp, r);
    tc::tmem_ld_wait();
    const int ub = kTileB * i + 8 * warp;   // this warp's run of 8 band tokens
    const int nk = min(8, T - ub);
    if (nk > 0) {
      float sc8[8];
      *reinterpret_cast<float4*>(sc8) = *reinterpret_cast<const float4*>(scs + ub);
      *reinterpret_cast<float4*>(sc8 + 4) = *reinterpret_cast<const float4*>(scs + ub + 4);
      int t = t_lo + ub;
      const int rr = t / side;
      int cc = t - rr * side;
      float* op = outp + size_t(t) * p.ld;
      if (has_dw) {
        // 3x3 window over grid cells: w0/w1/w2[di] = V(row rr-1+di, col cc-1/cc/cc+1);
        // smem row rr - r0 holds grid row rr - 1 (zero rows/cells outside the grid)
        const uint8_t* rowp = Vb + (rr - r0) * ROWB + 4 * lane;
        if (nk == 8 && cc + 8 <= side) {
          // the whole run lies in one grid row: the 3 x 10 window once, eight
          // independent tap chains
          float w[3][10];
#pragma unroll
          for (int di = 0; di < 3; ++di) {
            const float* rp = reinterpret_cast<const float*>(rowp + di * ROWB) + (cc - 1) * 32;
            w[di][0] = cc > 0 ? rp[0] : 0.f;
#pragma unroll
            for (int x = 1; x < 9; ++x) w[di][x] = rp[32 * x];
            w[di][9] = cc + 8 < side ? rp[32 * 9] : 0.f;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float sdw = 0.f;
#pragma unroll
            for (int di = 0; di < 3; ++di) {
              sdw = fmaf(w[di][k], tap[di * 3 + 0], sdw);
              sdw = fmaf(w[di][k + 1], tap[di * 3 + 1], sdw);
              sdw = fmaf(w[di][k + 2], tap[di * 3 + 2], sdw);
            }
            op[size_t(k) * p.ld] = __fadd_rn(__fmul_rn(__uint_as_float(r[k]), sc8[k]), sdw);
          }
        } else {
        auto vat = [&](int di, int c) -> float {
          return c < side ? *reinterpret_cast<const float*>(rowp + di * ROWB + c * 128) : 0.f;
        };
        float w0[3], w1[3], w2[3];
#pragma unroll
        for (int di = 0; di < 3; ++di) {
          w0[di] = cc > 0 ? *reinterpret_cast<const float*>(rowp + di * ROWB + (cc - 1) * 128) : 0.f;
          w1[di] = *reinterpret_cast<const float*>(rowp + di * ROWB + cc * 128);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k < nk) {
#pragma unroll
            for (int di = 0; di < 3; ++di) w2[di] = vat(di, cc + 1);
            // taps in the reference's (row, col) order (tensor.py:191-194)
            float sdw = 0.f;
#pragma unroll
            for (int di = 0; di < 3; ++di) {
              sdw = fmaf(w0[di], tap[di * 3 + 0], sdw);
              sdw = fmaf(w1[di], tap[di * 3 + 1], sdw);
              sdw = fmaf(w2[di], tap[di * 3 + 2], sdw);
            }
            *op = __fadd_rn(__fmul_rn(__uint_as_float(r[k]), sc8[k]), sdw);
            op += p.ld;
            if (++cc == side) {   // next grid row: window restarts at column 0
              cc = 0;
              rowp += ROWB;
#pragma unroll
              for (int di = 0; di < 3; ++di) {
                w0[di] = 0.f;
                w1[di] = *reinterpret_cast<const float*>(rowp + di * ROWB);
              }
            } else {
#pragma unroll
              for (int di = 0; di < 3; ++di) {
                w0[di] = w1[di];
                w1[di] = w2[di];
              }
            }
          }
        }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k < nk) {
            *op = __fmul_rn(__uint_as_float(r[k]), sc8[k]);
            op += p.ld;
          }
        }
      }
    }
    tc::tc_fence_before();
  }
  __syncthreads();
  BAT_PROF_MARK(5);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tbase);
  BAT_PROF_MARK(6);
}

}  // namespace bat

// Host side: band / cluster geometry and launch; SA_ERR_VALUE when the shape is
// outside this kernel's envelope (the caller then uses another path).
int binattn_tc_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                      const float* v, const float* dw, float* out, int64_t B, int64_t n,
                      int64_t d, int64_t heads, float eps, cudaStream_t s) {
  using namespace bat;
  if (heads <= 0 || d % heads) return SA_ERR_VALUE;
  const int64_t dk = d / heads;
  if (dk != 32 && dk != 64) return SA_ERR_VALUE;
  if (B <= 0 || B > 65535 || n <= 0 || n >= (int64_t(1) << 24)) return SA_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(v) & 15) != 0) return SA_ERR_VALUE;
  int side = 0;
  while (int64_t(side) * side < n) ++side;
  if (side > 256) return SA_ERR_VALUE;
  const int rows_total = int((n + side - 1) / side);
  // bands of <= ~400 tokens, at most 8 CTAs per cluster (portable size)
  int br = kMaxBandTokens / side;
  br = br < 1 ? 1 : (br > rows_total ? rows_total : br);
  int cl = (rows_total + br - 1) / br;
  if (cl > 8) {
    br = (rows_total + 7) / 8;
    cl = (rows_total + br - 1) / br;
  }
  const Lay L = dk == 32 ? layout<32>(side, br) : layout<64>(side, br);
  if (L.total > 200 * 1024 || br > kMaxBandRows) return SA_ERR_VALUE;
  Params p{cq, ck, gq, gk, dw, out, int(n), int(d), int(heads), side, rows_total, br, eps};
  void (*kern)(Params, CUtensorMap) = dk == 32 ? binattn_tc_kernel<32> : binattn_tc_kernel<64>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(cl), unsigned(heads * (dk / 32)), unsigned(B));
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(cl);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // V as a (channel, token, image) tensor: per-image token bounds make the
  // cells past n out of bounds (zero fill), as are halo rows outside the grid
  CUtensorMap tmV;
  memset(&tmV, 0, sizeof(tmV));
  const cuuint64_t dims[3] = {cuuint64_t(d), cuuint64_t(n), cuuint64_t(B)};
  const cuuint64_t strides[2] = {cuuint64_t(d) * 4, cuuint64_t(n) * cuuint64_t(d) * 4};
  const cuuint32_t box[3] = {32u, cuuint32_t(side), 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode_tmap_tiled(&tmV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(v), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SA_ERR_VALUE;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, tmV);
  if (e != cudaSuccess) {
    set_error("sa_linear_binary_attn: tensor-core launch failed: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  count_launch(1);
  return SA_OK;
}

}  // namespace sa

#ifdef BAT_PROF
extern "C" int sa_bat_prof_set(unsigned long long* buf) {
  return cudaMemcpyToSymbol(sa::bat::g_bat_prof, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
extern "C" int sa_bat_prof_launch(const uint32_t* cq, const uint32_t* ck, const float* gq,
                                  const float* gk, const float* v, const float* dw, float* out,
                                  int64_t B, int64_t n, int64_t d, int64_t heads, float eps) {
  return sa::binattn_tc_launch(cq, ck, gq, gk, v, dw, out, B, n, d, heads, eps, 0);
}
#endif
