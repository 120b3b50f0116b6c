// K2a, streaming form: binary linear attention + DWConv on the tensor cores,
// one persistent CTA per SM walking (image, head, 32-channel slice) units.
//
// Semantics (ref attention.py:113-120 on the binary features of
// model.py:355-358, DWConv branch attention.py:170-179 added before W_O,
// model.py:367-373), per unit:
//   S[j][a]  = sum_{t : ck[t][a]} v_t[j]             (K^T V, additions only)
//   cnt[a]   = sum_t ck[t][a]                         (integer)
//   out_t[j] = gq*gk * sum_{a : cq[t][a]} S[j][a] / (gq*gk*sum_{a : cq[t][a]} cnt[a] + eps)
//              + dwconv3x3(V)_t[j]
// Both contractions have a {0,1} operand, so they run on tcgen05 with exact
// bf16 operands (V and S as hi/mid/lo planes, codes as 0.0/1.0) and fp32
// accumulation, as in binattn_tc.cu (same operand layouts and arithmetic
// order per element).
//
// Why a streaming kernel: the tensor-core work is ~1% of the time; what
// costs is moving V twice and the output once. Each CTA keeps a ring of V
// grid rows (TMA, one row of the token grid per copy, zero-filled past the
// image) and walks the unit's tiles (R grid rows, <= 128 tokens) twice:
//   pass A: converter warps turn the tile into the K^T V operands (V planes
//           K-major with a ones row for the code counts, K codes as bf16);
//           the MMA warp accumulates S and cnt over all tiles in TMEM;
//   switch: S is summed ((hi + mid) + lo), split into bf16 planes and stored
//           in TMEM as the A operand of pass B (replicated in the four lane
//           quarters), the code counts become bit-slice masks;
//   pass B: the Q codes of the tile (bf16, K-major) against S in TMEM give
//           num[j][token]; the epilogue scales by gq*gk / (gq*gk*D + eps)
//           (D = integer code-count dot), adds the 3x3 DWConv from the V
//           rows in the ring (rows above / below the tile stay resident) and
//           stores 128 B per token. V is re-read in pass B within a few
//           microseconds of pass A, from L2.
// Every stage hand-off is an mbarrier pair (producer warp: TMA rows; MMA warp:
// tcgen05.mma / commit; 8 worker warps: operands and epilogue), so row loads,
// conversions, MMAs and epilogues of neighbouring tiles and units overlap.
#include "tc_common.cuh"

namespace sa {
namespace bas {

constexpr int kWorkers = 8;                    // warps 0-7
constexpr int kProdWarp = 8, kMmaWarp = 9;
constexpr int kThreads = 10 * 32;
constexpr int kMaxTT = 128;                    // tokens per tile (MMA N of pass B)
constexpr uint32_t kBlkA = 8192;               // A K-block: 128 rows x 32 tokens bf16
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccA = 0;                  // pass A accumulator [0, DK)
constexpr uint32_t kAccB = 64;                 // pass B accumulators [64, 192), [192, 320)
constexpr uint32_t kA2 = 320;                  // S planes (A operand of pass B)

struct Params {
  const uint32_t* cq;
  const uint32_t* ck;
  const float* gq;
  const float* gk;
  const float* dw;
  float* out;
  int B, n, ld, heads, side, RT, R, TTr, TT, NT, NR, units;
  float eps;
  long long* tl;   // debug builds: CTA 0 event clocks [event][slot] (nullptr: off)
  uint32_t hint;   // mbarrier try_wait suspend-time hint (ns)
};

#ifdef SA_DEBUG
#define BAS_TL(ev, i)                                                                   \
  do {                                                                                  \
    if (p.tl && blockIdx.x == 0 && (i) < 256) p.tl[(ev) * 256 + (i)] = clock64();      \
  } while (0)
#else
#define BAS_TL(ev, i) do {} while (0)
#endif

struct Lay {
  uint32_t ring, opa, opb, kv, mk, bars, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

template <int DK>
__host__ __device__ inline Lay layout(int side, int NR, int TT) {
  constexpr int W = DK / 32;
  const uint32_t KB = uint32_t((TT + 31) / 32);
  Lay L;
  uint32_t o = 0;
  L.opa = o;                                   // [2] x KB x (A block | B block)
  o += 2 * KB * (kBlkA + DK * 64);
  L.opb = o;                                   // [2] Q codes tile, bf16 K-major halves
  o += 2 * uint32_t(kMaxTT) * DK * 2;
  L.ring = o;                                  // NR + 1 (zero) rows x (side + 2) tokens x 128 B
  o += uint32_t(NR + 1) * (side + 2) * 128;
  o = align_up(o, 16);
  L.kv = o;                                    // [3 planes + count][32][DK + 4] fp32
  o += (3 * 32 * (DK + 4) + DK) * 4;
  o = align_up(o, 16);
  L.mk = o;                                    // [24][W] count bit-slice masks
  o += 24 * W * 4;
  o = align_up(o, 8);
  L.bars = o;
  o += (2 * NR + 12 + 4) * 8;
  L.total = o;
  return L;
}

// two code bits → bf16 pair (0.0 / 1.0 each), low half = first bit
__device__ __forceinline__ uint32_t bits2bf(uint32_t b0, uint32_t b1) {
  return (b0 ? 0x3F80u : 0u) | (b1 ? 0x3F800000u : 0u);
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

__device__ __forceinline__ void workers_sync() {
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

template <int DK>
__global__ void __launch_bounds__(kThreads, 1)
    binattn_stream_kernel(Params p, const __grid_constant__ CUtensorMap tmV) {
  constexpr int W = DK / 32;
  constexpr int S = DK / 32;                   // 32-channel slices per head
  constexpr int KP = DK + 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int side = p.side, n = p.n, RT = p.RT, R = p.R, TT = p.TT, TTr = p.TTr, NT = p.NT;
  const int NR = p.NR, H = p.heads;
  const uint32_t ROWB = uint32_t(side) * 128u;        // TMA bytes of one grid row
  const uint32_t ROWP = uint32_t(side + 2) * 128u;    // ring slot: zero column | row | zero column
  const int KB = (TT + 31) / 32;
  const Lay L = layout<DK>(side, NR, TT);
  uint8_t* opa = smem + L.opa;
  uint8_t* opb = smem + L.opb;
  uint8_t* ring = smem + L.ring;
  float* kvs = reinterpret_cast<float*>(smem + L.kv);
  uint32_t* mk = reinterpret_cast<uint32_t*>(smem + L.mk);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* row_full = bars;
  uint64_t* row_empty = row_full + NR;
  uint64_t* opa_full = row_empty + NR;   // [2]
  uint64_t* opa_empty = opa_full + 2;    // [2]
  uint64_t* opb_full = opa_empty + 2;    // [2]
  uint64_t* opb_empty = opb_full + 2;    // [2]
  uint64_t* accb_full = opb_empty + 2;   // [2]
  uint64_t* accb_empty = accb_full + 2;  // [2]
  uint64_t* acca_full = accb_empty + 2;
  uint64_t* a2_full = acca_full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(a2_full + 2);
  const uint32_t blkAB = kBlkA + DK * 64;      // one A + B K-block
  const uint32_t opa_bytes = uint32_t(KB) * blkAB;
  const uint32_t opb_bytes = uint32_t(kMaxTT) * DK * 2;

  if (tid == 0) {
    for (int i = 0; i < NR; ++i) {
      tc::mbar_init(row_full + i, 1);
      tc::mbar_init(row_empty + i, kWorkers);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(opa_full + i, kWorkers);
      tc::mbar_init(opa_empty + i, 1);
      tc::mbar_init(opb_full + i, kWorkers);
      tc::mbar_init(opb_empty + i, 1);
      tc::mbar_init(accb_full + i, 1);
      tc::mbar_init(accb_empty + i, kWorkers);
    }
    tc::mbar_init(acca_full, 1);
    tc::mbar_init(a2_full, 4);
    tc::fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc<kTmemCols>(tslot);
  // the ring's zero padding: slot columns 0 and side + 1 and the whole zero row
  // (slot NR); TMA writes only columns 1..side
  for (int i = tid; i < (NR + 1) * (side + 2) * 32; i += kThreads) {
    const int slot = i / ((side + 2) * 32), col = (i / 32) % (side + 2);
    if (slot == NR || col == 0 || col == side + 1)
      reinterpret_cast<float*>(ring)[i] = 0.f;
  }
  // rows 96..127 of every pass-A A block: bf16 1.0 (row 96 = the code counts)
  for (int i = tid; i < 2 * KB * 128; i += kThreads) {
    const int blk = i >> 7, e = i & 127;
    reinterpret_cast<uint4*>(opa + blk * blkAB + 12 * 512)[e] =
        make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == kProdWarp) {
    // ---------------- producer: V grid rows, pass A then pass B, per unit ----------------
    if (lane == 0) {
      uint32_t seq = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int b = u / (H * S), hs = u - b * (H * S);
        const int c0 = (hs / S) * DK + 32 * (hs % S);
        for (int pass = 0; pass < 2; ++pass)
          for (int r = 0; r < RT; ++r, ++seq) {
            const uint32_t slot = seq % uint32_t(NR);
            tc::mbar_wait_s(tc::smem_u32(row_empty + slot), ((seq / uint32_t(NR)) & 1u) ^ 1u, p.hint);
            BAS_TL(6, int(seq));
            tc::mbar_expect_tx(row_full + slot, ROWB);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tc::smem_u32(ring + slot * ROWP + 128)),
                "l"(reinterpret_cast<uint64_t>(&tmV)), "r"(c0), "r"(r * side), "r"(b),
                "r"(tc::smem_u32(row_full + slot))
                : "memory");
          }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    const uint32_t idA = tc::idesc_bf16_m128(DK);
    const uint32_t idB = tc::idesc_bf16_m128(TT);
    const uint32_t sa0 = tc::smem_u32(opa), sb0 = tc::smem_u32(opb);
    uint32_t ta = 0, tb = 0, uc = 0;   // pass-A / pass-B tile counters, unit counter
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++uc) {
      for (int k = 0; k < NT; ++k, ++ta) {
        const uint32_t buf = ta & 1u, ph = (ta >> 1) & 1u;
        tc::mbar_wait_s(tc::smem_u32(opa_full + buf), ph, p.hint);
        if (lane == 0) BAS_TL(2, int(ta));
        tc::tc_fence_after();
        const uint32_t base = sa0 + buf * opa_bytes;
        for (int kb = 0; kb < KB; ++kb) {
          const uint64_t ad = tc::smem_desc(base + kb * blkAB);
          const uint64_t bd = tc::smem_desc(base + kb * blkAB + kBlkA);
          mma_ss_w(tbase + kAccA, ad, bd, idA, (k | kb) ? 1u : 0u);
          mma_ss_w(tbase + kAccA, ad + (256 >> 4), bd + (256 >> 4), idA, 1u);
        }
        tc::commit_w(opa_empty + buf);
      }
      tc::commit_w(acca_full);
      tc::mbar_wait_s(tc::smem_u32(a2_full), uc & 1u, p.hint);   // S planes in TMEM
      tc::tc_fence_after();
      for (int k = 0; k < NT; ++k, ++tb) {
        const uint32_t buf = tb & 1u, ph = (tb >> 1) & 1u;
        tc::mbar_wait_s(tc::smem_u32(opb_full + buf), ph, p.hint);
        tc::mbar_wait_s(tc::smem_u32(accb_empty + buf), ph ^ 1u, p.hint);
        if (lane == 0) BAS_TL(7, int(tb));
        tc::tc_fence_after();
        const uint32_t acc = tbase + kAccB + buf * uint32_t(kMaxTT);
        const uint32_t sb = sb0 + buf * opb_bytes;
#pragma unroll
        for (int ks = 0; ks < DK / 16; ++ks) {
          const uint64_t bd =
              tc::smem_desc(sb + uint32_t(ks >> 1) * uint32_t(TT * 64) + uint32_t(ks & 1) * 256);
#pragma unroll
          for (int pp = 2; pp >= 0; --pp)   // lo, mid, hi: smallest products first
            tc::mma_ts_w(acc, tbase + kA2 + uint32_t(pp) * (DK / 2) + 8 * ks, bd, idB,
                         (ks == 0 && pp == 2) ? 0u : 1u);
        }
        tc::commit_w(opb_empty + buf);
        tc::commit_w(accb_full + buf);
      }
    }
  } else {
    // ---------------- workers (warps 0-7) ----------------
    const int q4 = warp & 3;                   // TMEM lane quarter
    const uint8_t* zrow = ring + NR * ROWP;    // all zeros
    const uint32_t rf0 = tc::smem_u32(row_full), re0 = tc::smem_u32(row_empty);
    uint32_t seq = 0;                          // row sequence number of (unit, pass, row 0)
    uint32_t ta = 0, tb = 0, uc = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++uc) {
      const int b = u / (H * S), hs = u - b * (H * S);
      const int h = hs / S;
      const int ch = h * DK + 32 * (hs % S) + lane;   // model channel of this lane
      const size_t cbase = (size_t(b) * H + h) * size_t(n) * W;
      float tap[9];
#pragma unroll
      for (int t9 = 0; t9 < 9; ++t9) tap[t9] = p.dw ? __ldg(p.dw + t9 * p.ld + ch) : 0.f;
      const float gg = __fmul_rn(__ldg(p.gq + b * H + h), __ldg(p.gk + b * H + h));
      const uint32_t seqA = seq, seqB = seq + uint32_t(RT);
      seq += 2u * uint32_t(RT);

      // ======== pass A ========
      // Every worker warp converts 4 tokens of each 32-token K block (its V
      // values → the A planes, its K codes → the B operand), so the warps are
      // balanced and need no CTA-wide barrier: opa_full counts their arrivals.
      // Lanes 0..4W-1 hold the warp's code words of the tile (one word per K
      // block), loaded one tile ahead.
      auto load_codes = [&](const uint32_t* src, int k, int tok0, int ntok, int nj, uint32_t (&dst)[4]) {
        // tokens tok0 + 32*j + lane / W of tile k (j < nj = register), zero outside
        const int t0 = k * R * side;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= nj) break;
          const int tt = tok0 + 32 * j + lane / W;
          dst[j] = (k < NT && lane < ntok * W && tt < TTr && t0 + tt < n)
                       ? __ldg(src + cbase + size_t(t0 + tt) * W + lane % W)
                       : 0u;
        }
      };
      uint32_t kw[4];
      load_codes(p.ck, 0, 4 * warp, 4, KB, kw);
      uint32_t s_lo = uint32_t(seqA) % uint32_t(NR), p_lo = (uint32_t(seqA) / uint32_t(NR)) & 1u;
      for (int k = 0; k < NT; ++k, ++ta) {
        const uint32_t buf = ta & 1u, ph = (ta >> 1) & 1u;
        if (tid == 0) BAS_TL(0, int(ta));
        const int rlo = k * R, nrow = min(RT, rlo + R) - rlo;   // grid rows of the tile
        uint32_t cw4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) cw4[j] = kw[j];
        load_codes(p.ck, k + 1, 4 * warp, 4, KB, kw);
        auto slot = [&](int j) -> uint32_t {   // ring slot of tile row j
          const uint32_t sj = s_lo + uint32_t(j);
          return sj >= uint32_t(NR) ? sj - uint32_t(NR) : sj;
        };
        auto spar = [&](int j) -> uint32_t { return s_lo + uint32_t(j) >= uint32_t(NR) ? p_lo ^ 1u : p_lo; };
        for (int j = 0; j < nrow; ++j) tc::mbar_wait_s(rf0 + 8 * slot(j), spar(j), p.hint);
        tc::mbar_wait_s(tc::smem_u32(opa_empty + buf), ph ^ 1u, p.hint);   // MMAs of tile ta - 2 done
        if (tid == 0) BAS_TL(8, int(ta));
        uint8_t* base = opa + buf * opa_bytes;
        // first token of this warp in K block 0, and its tile row / column
        int rr = (4 * warp) / side, cc = 4 * warp - rr * side;
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          if (kb >= KB) break;
          uint8_t* sA = base + kb * blkAB;
          uint8_t* sB = sA + kBlkA;
          // A: channel c = lane, planes p at rows 32p + c, tokens 4w..4w+3 of the block
          float vv[4];
          {
            int r2 = rr, c2 = cc;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float* rp = r2 < nrow ? reinterpret_cast<const float*>(ring + slot(r2) * ROWP)
                                          : reinterpret_cast<const float*>(zrow);
              vv[i] = rp[(c2 + 1) * 32 + lane];
              if (++c2 == side) { c2 = 0; ++r2; }
            }
          }
          const tc::Split3 s01 = tc::split3x2(vv[0], vv[1]);
          const tc::Split3 s23 = tc::split3x2(vv[2], vv[3]);
          const uint32_t offA = uint32_t(lane >> 3) * 512 + uint32_t(warp >> 1) * 128 +
                                uint32_t(lane & 7) * 16 + uint32_t(warp & 1) * 8;
          *reinterpret_cast<uint2*>(sA + offA) = make_uint2(tc::bf2_bits(s01.h), tc::bf2_bits(s23.h));
          *reinterpret_cast<uint2*>(sA + 2048 + offA) = make_uint2(tc::bf2_bits(s01.m), tc::bf2_bits(s23.m));
          *reinterpret_cast<uint2*>(sA + 4096 + offA) = make_uint2(tc::bf2_bits(s01.l), tc::bf2_bits(s23.l));
          // B: code bit a = lane (+ 32 per word), the same 4 tokens
#pragma unroll
          for (int w = 0; w < W; ++w) {
            uint32_t bit[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              bit[i] = (__shfl_sync(0xffffffffu, cw4[kb], i * W + w) >> lane) & 1u;
            const int c = 32 * w + lane;
            const uint32_t offB = uint32_t(c >> 3) * 512 + uint32_t(warp >> 1) * 128 +
                                  uint32_t(c & 7) * 16 + uint32_t(warp & 1) * 8;
            *reinterpret_cast<uint2*>(sB + offB) =
                make_uint2(bits2bf(bit[0], bit[1]), bits2bf(bit[2], bit[3]));
          }
          // advance this warp's token by 32
          cc += 32;
          while (cc >= side) { cc -= side; ++rr; }
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (tid == 0) BAS_TL(1, int(ta));
        if (lane == 0) {
          tc::mbar_arrive(opa_full + buf);
          // the tile's rows are converted (pass A is done with them)
          for (int j = 0; j < nrow; ++j) tc::mbar_arrive_s(re0 + 8 * slot(j));
        }
        __syncwarp();
        // next tile's first row
        s_lo += uint32_t(nrow);
        if (s_lo >= uint32_t(NR)) { s_lo -= uint32_t(NR); p_lo ^= 1u; }
      }

      // ======== switch: S = (hi + mid) + lo, counts, S planes → TMEM ========
      tc::mbar_wait_s(tc::smem_u32(acca_full), uc & 1u, p.hint);
      tc::tc_fence_after();
      float* kv3 = kvs;                                 // [3][32][KP] planes, then S
      float* cntf = kvs + 3 * 32 * KP;                  // [DK] counts
      if (warp < 4) {
#pragma unroll
        for (int cw = 0; cw < W; ++cw) {
          uint32_t r[32];
          tc::tmem_ld32_nowait(tbase + (uint32_t(32 * warp) << 16) + kAccA + 32 * cw, r);
          tc::tmem_ld_wait();
          if (warp < 3) {
            float* row = kv3 + warp * 32 * KP + lane * KP + 32 * cw;
#pragma unroll
            for (int c = 0; c < 32; c += 4)
              *reinterpret_cast<float4*>(row + c) =
                  make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                              __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
          } else if (lane == 0) {
#pragma unroll
            for (int c = 0; c < 32; ++c) cntf[32 * cw + c] = __uint_as_float(r[c]);
          }
        }
      }
      tc::tc_fence_before();
      workers_sync();
      if (warp < 4) {
        // S row j = lane as three bf16 planes into this warp's TMEM lane quarter:
        // column kA2 + p*DK/2 + c/2 holds the pair (c, c+1) of plane p
        const uint32_t tq = tbase + (uint32_t(32 * warp) << 16) + kA2;
#pragma unroll
        for (int cw = 0; cw < W; ++cw) {
          uint32_t ph[16], pm[16], pl[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float s2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = 32 * cw + 2 * i + e;
              s2[e] = __fadd_rn(__fadd_rn(kv3[lane * KP + c], kv3[32 * KP + lane * KP + c]),
                                kv3[64 * KP + lane * KP + c]);
            }
            const tc::Split3 sp = tc::split3x2(s2[0], s2[1]);
            ph[i] = tc::bf2_bits(sp.h);
            pm[i] = tc::bf2_bits(sp.m);
            pl[i] = tc::bf2_bits(sp.l);
          }
          tc::tmem_st16(tq + 16 * cw, ph);
          tc::tmem_st16(tq + DK / 2 + 16 * cw, pm);
          tc::tmem_st16(tq + DK + 16 * cw, pl);
        }
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(a2_full);
      } else if (warp == 4) {
        // count bit-slice masks: mask_k = code bits whose count has bit k set
#pragma unroll
        for (int cw = 0; cw < W; ++cw) {
          const uint32_t cv = uint32_t(cntf[32 * cw + lane]);
#pragma unroll
          for (int kk = 0; kk < 24; ++kk) {
            const uint32_t m = __ballot_sync(0xffffffffu, (cv >> kk) & 1u);
            if (lane == 0) mk[kk * W + cw] = m;
          }
        }
      }
      workers_sync();
      uint32_t cmax = 0;
      {
        uint32_t cv = 0;
#pragma unroll
        for (int cw = 0; cw < W; ++cw) cv = max(cv, uint32_t(cntf[32 * cw + lane]));
        cmax = __reduce_max_sync(0xffffffffu, cv);
      }
      const int nb = 32 - __clz(int(cmax));
      if (tid == 0) BAS_TL(3, int(uc));

      // ======== pass B ========
      // Warp w owns tokens [16w, 16w + 16) of every tile: it builds their Q-code
      // rows of the B operand and their scales (lane < 16: token 16w + lane),
      // then runs their epilogue; opb_full / accb_empty count the 8 warps.
      uint32_t qw[4];
      load_codes(p.cq, 0, 16 * warp, 16, 1, qw);
      float scl = 0.f;   // lane < 16: scale of token 16w + lane of the built tile
      auto build = [&](int k, uint32_t tbk) -> float {
        const uint32_t buf = tbk & 1u, ph = (tbk >> 1) & 1u;
        const uint32_t wd = qw[0];   // lane < 16*W: word lane % W of token 16w + lane / W
        load_codes(p.cq, k + 1, 16 * warp, 16, 1, qw);
        tc::mbar_wait_s(tc::smem_u32(opb_empty + buf), ph ^ 1u, p.hint);   // MMAs of tile tbk - 2 done with it
        uint8_t* dst = opb + buf * opb_bytes;
        // chunk e = (token j, byte g of the codes): 16 tokens x DK/8 chunks
#pragma unroll
        for (int i = 0; i < (16 * (DK / 8) + 31) / 32; ++i) {
          const int e = lane + 32 * i;
          const int j = e / (DK / 8), g = e % (DK / 8);
          const uint32_t word = __shfl_sync(0xffffffffu, wd, (j * W + (g >> 2)) & 31);
          const int ul = 16 * warp + j;
          if (e < 16 * (DK / 8) && ul < TT) {
            const uint32_t by = (word >> (8 * (g & 3))) & 0xFFu;
            const uint32_t off = uint32_t(g >> 2) * uint32_t(TT * 64) + uint32_t(ul >> 3) * 512 +
                                 uint32_t(g & 3) * 128 + uint32_t(ul & 7) * 16;
            *reinterpret_cast<uint4*>(dst + off) =
                make_uint4(bits2bf(by & 1u, by & 2u), bits2bf(by & 4u, by & 8u),
                           bits2bf(by & 16u, by & 32u), bits2bf(by & 64u, by & 128u));
          }
        }
        // scale of token 16w + lane: gq*gk / (gq*gk*D + eps), D the integer code-count dot
        uint32_t D = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint32_t cwd = __shfl_sync(0xffffffffu, wd, (lane * W + w) & 31);
          for (int kk = 0; kk < nb; ++kk) D += uint32_t(__popc(cwd & mk[kk * W + w])) << kk;
        }
        const float sc = __fdiv_rn(gg, __fadd_rn(__fmul_rn(gg, float(D)), p.eps));
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(opb_full + buf);
        return sc;
      };
      float* outp = p.out + size_t(b) * n * p.ld + ch;
      scl = build(0, tb);
      uint32_t sb_lo = uint32_t(seqB) % uint32_t(NR), pb_lo = (uint32_t(seqB) / uint32_t(NR)) & 1u;
      for (int k = 0; k < NT; ++k, ++tb) {
        const float sc_cur = scl;
        if (k + 1 < NT) scl = build(k + 1, tb + 1);
        const uint32_t buf = tb & 1u, ph = (tb >> 1) & 1u;
        const int t0 = k * R * side;
        const int rlo = k * R, rhi = min(RT, rlo + R);
        // grid rows g_lo .. g_hi (rlo-1 .. rhi inside the grid) must have landed;
        // sb_lo / pb_lo: slot / parity of grid row g_lo
        const int g_lo = max(0, rlo - 1), g_hi = min(RT - 1, rhi);
        auto slot = [&](int r) -> uint32_t {   // ring slot of grid row r >= g_lo
          const uint32_t sj = sb_lo + uint32_t(r - g_lo);
          return sj >= uint32_t(NR) ? sj - uint32_t(NR) : sj;
        };
        for (int r = g_lo; r <= g_hi; ++r)
          tc::mbar_wait_s(rf0 + 8 * slot(r), sb_lo + uint32_t(r - g_lo) >= uint32_t(NR) ? pb_lo ^ 1u : pb_lo,
                          p.hint);
        auto rowp = [&](int r) -> const float* {   // grid row r (the zero row outside the grid)
          if (r < 0 || r >= RT) return reinterpret_cast<const float*>(zrow) + lane;
          return reinterpret_cast<const float*>(ring + slot(r) * ROWP) + lane;
        };
        tc::mbar_wait_s(tc::smem_u32(accb_full + buf), ph, p.hint);
        if (tid == 0) BAS_TL(4, int(tb));
        tc::tc_fence_after();
        const int ub = 16 * warp;
        const int nk = min(16, min(TTr, n - t0) - ub);
        if (nk > 0) {
          float num[16];
          tc::tmem_ld16(tbase + (uint32_t(32 * q4) << 16) + kAccB + buf * uint32_t(kMaxTT) + ub, num);
          const int t = t0 + ub;
          int rr = t / side;
          int cc = t - rr * side;
          float* op = outp + size_t(t) * p.ld;
          if (nk == 16 && cc + 16 <= side) {
            // one grid row: the 3 x 18 window once (padded rows: no bounds), 16 tap chains
            float w[3][18];
#pragma unroll
            for (int di = 0; di < 3; ++di) {
              const float* rp = rowp(rr - 1 + di) + cc * 32;   // column cc - 1 (+1 pad)
#pragma unroll
              for (int x = 0; x < 18; ++x) w[di][x] = rp[32 * x];
            }
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              // taps in the reference's (row, col) order (tensor.py:191-194)
              float sdw = 0.f;
#pragma unroll
              for (int di = 0; di < 3; ++di) {
                sdw = fmaf(w[di][kk], tap[di * 3 + 0], sdw);
                sdw = fmaf(w[di][kk + 1], tap[di * 3 + 1], sdw);
                sdw = fmaf(w[di][kk + 2], tap[di * 3 + 2], sdw);
              }
              const float sc = __shfl_sync(0xffffffffu, sc_cur, kk);
              op[size_t(kk) * p.ld] = __fadd_rn(__fmul_rn(num[kk], sc), sdw);
            }
          } else {
            const float* rp[3] = {rowp(rr - 1), rowp(rr), rowp(rr + 1)};
            float w0[3], w1[3], w2[3];
#pragma unroll
            for (int di = 0; di < 3; ++di) {
              w0[di] = rp[di][cc * 32];
              w1[di] = rp[di][(cc + 1) * 32];
            }
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
              const float sc = __shfl_sync(0xffffffffu, sc_cur, kk);
              if (kk < nk) {
#pragma unroll
                for (int di = 0; di < 3; ++di) w2[di] = rp[di][(cc + 2) * 32];
                float sdw = 0.f;
#pragma unroll
                for (int di = 0; di < 3; ++di) {
                  sdw = fmaf(w0[di], tap[di * 3 + 0], sdw);
                  sdw = fmaf(w1[di], tap[di * 3 + 1], sdw);
                  sdw = fmaf(w2[di], tap[di * 3 + 2], sdw);
                }
                *op = __fadd_rn(__fmul_rn(num[kk], sc), sdw);
                op += p.ld;
                if (++cc == side) {   // next grid row: window restarts at column 0
                  cc = 0;
                  ++rr;
                  rp[0] = rp[1];
                  rp[1] = rp[2];
                  rp[2] = rowp(rr + 1);
#pragma unroll
                  for (int di = 0; di < 3; ++di) {
                    w0[di] = 0.f;
                    w1[di] = rp[di][32];
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
        }
        tc::tc_fence_before();
        __syncwarp();
        if (tid == 0) BAS_TL(5, int(tb));
        // rows whose last use is this tile: rlo-1 .. rhi-2 (the next tile starts at rhi-1)
        const int last = (k + 1 < NT) ? rhi - 2 : RT - 1;
        if (lane == 0) {
          tc::mbar_arrive(accb_empty + buf);
          for (int r = g_lo; r <= last; ++r) tc::mbar_arrive_s(re0 + 8 * slot(r));
        }
        __syncwarp();
        // the next tile's first row is max(0, rhi - 1)
        if (k + 1 < NT) {
          const int adv = max(0, rhi - 1) - g_lo;
          sb_lo += uint32_t(adv);
          if (sb_lo >= uint32_t(NR)) { sb_lo -= uint32_t(NR); pb_lo ^= 1u; }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace bas

SA_DEBUG_SWITCH(uint32_t, g_bas_hint, 0x100000u, sa_debug_attn_hint)
#ifdef SA_DEBUG
static long long* g_bas_tl = nullptr;
extern "C" void sa_debug_attn_timeline(void* buf) { g_bas_tl = static_cast<long long*>(buf); }
#else
static constexpr long long* g_bas_tl = nullptr;
#endif

// Host side: tile / ring geometry and launch; SA_ERR_VALUE when the shape is
// outside this kernel's envelope (the caller then uses another path).
int binattn_stream_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                          const float* v, const float* dw, float* out, int64_t B, int64_t n,
                          int64_t d, int64_t heads, float eps, cudaStream_t s) {
  using namespace bas;
  if (heads <= 0 || d % heads) return SA_ERR_VALUE;
  const int64_t dk = d / heads;
  if (dk != 32 && dk != 64) return SA_ERR_VALUE;
  if (B <= 0 || n <= 0 || n >= (int64_t(1) << 24)) return SA_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(v) & 15) != 0 || (d * 4) % 16 != 0) return SA_ERR_VALUE;
  int side = 0;
  while (int64_t(side) * side < n) ++side;
  if (side > kMaxTT) return SA_ERR_VALUE;
  const int RT = int((n + side - 1) / side);
  const int R = kMaxTT / side < RT ? kMaxTT / side : RT;
  const int TTr = R * side;
  const int TT = (TTr + 15) / 16 * 16;
  const int NT = (RT + R - 1) / R;
  const int NR = 2 * R + 2;
  const int64_t units = B * heads * (dk / 32);
  if (units >= (int64_t(1) << 31)) return SA_ERR_VALUE;
  const Lay L = dk == 32 ? layout<32>(side, NR, TT) : layout<64>(side, NR, TT);
  const uint32_t smem = L.total + 1024;   // + 1 KB alignment slack
  if (smem > 227 * 1024) return SA_ERR_VALUE;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  Params p{cq, ck, gq, gk, dw, out, int(B), int(n), int(d), int(heads), side, RT, R, TTr, TT, NT,
           NR, int(units), eps, g_bas_tl, g_bas_hint};
  void (*kern)(Params, CUtensorMap) = dk == 32 ? binattn_stream_kernel<32> : binattn_stream_kernel<64>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  // V as a (channel, token, image) tensor: per-image token bounds make the
  // cells past n out of bounds (zero fill)
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
  const int grid = int(units < sms ? units : sms);
  kern<<<grid, kThreads, smem, s>>>(p, tmV);
  count_launch(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("sa_linear_binary_attn: streaming launch failed: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  return SA_OK;
}

}  // namespace sa
