// K5 fused: the whole (MoE) MLP  y = [res +] gate · fc2(GELU(fc1(x)))  in one
// persistent tcgen05 kernel; the hidden activations never leave the SM.
//
// Reference: Mlp.forward (model.py:204-208) inside MoeModule.forward
// (model.py:250-274), experts (Mlp(Linear,Linear), Mlp(Shift,Shift))
// (model.py:514-521). Numerics as in tcgemm.cu: x and GELU(h) are split into
// hi/mid/lo bf16 planes (exact), shift weights are exact bf16, dense weights
// three planes; fp32 accumulation in TMEM.
//
// Per 128-token tile of one expert the hidden dimension runs in chunks of
// HC = 64: fc1(q) → acc1 in TMEM buffer q % 3 → GELU group q % 3: tcgen05.ld,
// GELU, split, tcgen05.st of the three A2 planes into the SAME buffer (over the
// consumed accumulator) → fc2(q) accumulates into acc2[tile % 2]; fc1(q + 3)
// waits until fc2(q) released the buffer. At d = 32 the dense fc2 concatenates
// B planes along N (A_mid·[w_hi|w_mid], A_hi·[w_hi|w_mid] at N = 64 into two
// 32-column partial sums, A_lo·w_hi and A_hi·w_lo at N = 32): 4 MMAs per K
// step instead of 6, the same six products; the epilogue adds the partials.
//
// What paces a kernel like this is instruction issue, not the tensor pipe: a
// 128 x N x 16 tcgen05.mma retires in ~N/2 cycles, but a single issuing warp
// that derives every operand with dependent arithmetic (or waits on an
// mbarrier, ~90 cycles even when the phase is complete) spends far longer per
// MMA (scripts/probe_mma_seq.py). So fc1 and fc2 have an issuing warp each;
// their per-chunk loops hold only the waits, one asm block per K step whose
// operands are per-chunk bases plus compile-time offsets, and the commits.
// Roles (19 warps, one CTA per SM):
//   warps  0-11       GELU groups g = 0..2 (chunks q % 3 == g, buffer g); warp
//                     quad = TMEM lane block
//   warps 12-15       producers: gather x rows (MoE permutation), split,
//                     tcgen05.st → A1 (thread = row = TMEM lane); drain acc2:
//                     × gate, + residual, transpose, scatter to token order
//   warp  16 / 17     fc1 / fc2 MMA issuers
//   warp  18          weights: d = 32 (hidden <= 256): both experts' W1 / W2
//                     resident in shared memory, loaded once; d = 64: W1 / W2
//                     chunk rings (bulk async copy)
// Every hand-off is a full/empty mbarrier pair; parities flip on wrap, so
// tiles of the two experts interleave freely.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace tcm {

using namespace tc;

constexpr int HC = 64;                 // hidden chunk (fc1 N, fc2 K)
#ifndef MLP_NF
#define MLP_NF 0                       // GELU pairs (of 8) whose reciprocal runs on the FMA pipe
#endif
constexpr int kGelu = 16;              // GELU warps 0-15 (column group x lane quad)
// GELU layout: true = two groups of 8 warps on alternate chunks, 32 columns per
// warp; false = all 16 warps on every chunk, 16 columns per warp
#ifndef MLP_GELU_ALT
#define MLP_GELU_ALT 0
#endif
constexpr bool kGeluAlt = MLP_GELU_ALT != 0;
constexpr int kGeluPerChunk = kGeluAlt ? 8 : 16;
constexpr int kProd = 16;              // producers: warps 16 .. 16 + 4·(d/32) - 1
// wide form (d = 128 / 160): hidden chunks of 32, one A1 buffer, a single
// acc2 of d columns, GELU in two groups of 8 warps on alternate chunks, one
// producer warp per TMEM lane quarter walking every K stage
template <int D>
struct Wide {
  static constexpr bool W = D > 64;
  static constexpr int HC = W ? 32 : 64;
};
#ifndef MLP_NA64
#define MLP_NA64 1   // d = 64: A1 buffers (2 leaves two chunk buffers) (A/B knob)
#endif
#ifndef MLP_PG32
#define MLP_PG32 1   // d = 32: producer groups on alternate tiles (A/B knob)
#endif
template <int D>
struct Roles {
  static constexpr int PGN = D == 32 ? MLP_PG32 : 1;                // producer groups
  static constexpr int PPG = Wide<D>::W ? 4 : 4 * (D / 32);         // warps per group
  static constexpr int NPW = PGN * PPG;                             // producer warps
  static constexpr int kMma1 = kProd + NPW, kMma2 = kMma1 + 1, kWld = kMma1 + 2;
  static constexpr int kThreads = (kWld + 1) * 32;
};
constexpr int kResHidden = 256;        // d = 32: weights resident up to this hidden
constexpr uint32_t kPlaneCols = 16;    // TMEM columns of one 32-k bf16 plane
constexpr uint32_t kBufCols = 96;      // acc1 (64 fp32) / A2 (3 planes x 32) buffer

struct MlpParams {
  const float* x;
  const int32_t* perm;       // nullptr: identity rows
  const int32_t* counts;     // nullptr: one group
  const float* gate;
  const float* residual;
  float* y;
  const uint16_t* w1[2];     // packed (bn = HC) planes per expert
  const uint16_t* w2[2];     // packed (bn = d) planes per expert
  int np0, np1;              // planes per expert (3 dense, 1 shift)
  int64_t M;
  int hidden;
  unsigned long long* prof;  // debug builds: cycles per wait site (nullptr: off)
  long long* tl;             // debug builds: CTA 0 event timeline [8][64] (nullptr: off)
  int dbg;                   // debug builds: role isolation bits (see kDbg)
  const float* lnf_g;        // LNF: the stage's final LayerNorm on the output rows
  const float* lnf_b;
  float lnf_eps;
};

#ifdef SA_DEBUG
constexpr bool kDbg = true;    // dbg bit 1: GELU handshakes only; 2: producers handshakes
#else                          // only; 4: no MMAs (commits only); 8: MMA issuers alone,
constexpr bool kDbg = false;   // no waits
#endif

// wait sites of the optional cycle profile (debug builds)
enum { S_OF = 0, S_A1E, S_WR, S_OE, S_HE, S_A1F, S_BF, S_HF, S_W, T_PROD, T_MMA1, T_MMA2,
       T_GELU, S_N };

template <int D, bool RES, bool LNF = false>
struct Layout {
  static constexpr bool W = Wide<D>::W;
  static constexpr int HC = Wide<D>::HC;                      // hidden chunk (fc1 N, fc2 K)
  static constexpr int KC1 = D / 32;                          // fc1 K stages
  // A1 buffers (TMEM); d = 64 can trade a chunk buffer for a second A1
  static constexpr int NA = D == 32 ? 2 : (D == 64 && MLP_NA64 == 2 ? 2 : 1);
  static constexpr int NB = W ? 2 : (D == 64 && NA == 2 ? 2 : 3);   // acc1 / A2 buffers (TMEM)
  // wide: the A1 lo plane lives in shared memory (ss-form MMAs), hi / mid in
  // TMEM; d <= 160 also concatenates the dense fc1 B planes along N (3 MMAs
  // per K step into three 32-column partial sums, added by the GELU warps)
  static constexpr bool CATW = W && D <= 160;
  static constexpr int A1P = W ? 2 : 3;                       // A1 planes in TMEM
  static constexpr uint32_t BUFC = W ? (CATW ? 96 : 48) : 96; // acc1 | A2 (3 planes)
  static constexpr int NO = W ? 1 : 2;                        // acc2 buffers
  static constexpr int GPC = W ? 8 : kGeluPerChunk;           // GELU warps per chunk
  static constexpr bool CAT = D == 32;                        // N-concatenated dense fc2
  static constexpr int NW = W ? (D == 128 ? 3 : 2) : (LNF && D == 64 ? 3 : 4);   // ring slots (RES = false)
  static constexpr uint32_t W1C = KC1 * 3 * (HC * 32 * 2);    // dense W1 chunk bytes
  static constexpr uint32_t W2C = (HC / 32) * 3 * (D * 32 * 2);
  static constexpr uint32_t RW1 = (kResHidden / HC) * W1C;    // resident dense W1
  static constexpr uint32_t RW2 = (kResHidden / HC) * W2C;
  // resident: W1 dense | W1 shift | W2 dense | W2 shift
  __device__ static constexpr uint32_t r_w1(int e) { return e ? RW1 : 0u; }
  __device__ static constexpr uint32_t r_w2(int e) { return RW1 + RW1 / 3 + (e ? RW2 : 0u); }
  static constexpr uint32_t WBYTES = RES ? (RW1 + RW1 / 3 + RW2 + RW2 / 3) : NW * (W1C + W2C);
  static constexpr uint32_t OFF_ALO = WBYTES;                 // wide: [KC1][128 x 32] bf16 lo plane
  static constexpr uint32_t ALO = W ? KC1 * kBM * 32 * 2 : 0;
  static constexpr uint32_t OFF_XB = OFF_ALO + ALO;
  static constexpr int XP = LNF ? D + 4 : kXPitch;            // transpose pitch (LNF: whole rows)
  // producer transpose slots (LNF: one whole-row buffer per TMEM lane quarter,
  // shared by the quarter's producer warps)
  static constexpr uint32_t XB = (LNF ? 4 * Roles<D>::PGN : Roles<D>::NPW) * 32 * XP * 4;
  static constexpr uint32_t OFF_BAR = OFF_XB + XB;
  // barriers: a1 full/empty[NA], w1 full/empty[NW], w2 full/empty[NW],
  //           h_full/h_empty/buf_free[NB], o_full/o_empty[NO], wres
  static constexpr uint32_t NBAR = 2 * NA + 4 * NW + 3 * NB + 2 * NO + 1;
  static constexpr uint32_t TOTAL = OFF_BAR + NBAR * 8 + 16 + 1024;  // + alignment slack
  // TMEM columns: buffers[NB] (acc1 | A2) | acc2[2] | A1[NA] (KC1 x 3 planes)
  static constexpr uint32_t T_BUF = 0;
  static constexpr uint32_t T_ACC2 = NB * BUFC;
  static constexpr uint32_t ACC2C = W ? D : 64;
  static constexpr uint32_t T_A1 = T_ACC2 + NO * ACC2C;
  static constexpr uint32_t A1COLS = KC1 * A1P * kPlaneCols;
  static constexpr uint32_t TCOLS = 512;
  static_assert(T_A1 + NA * A1COLS <= TCOLS, "TMEM budget");
  static_assert(TOTAL <= 232448, "shared memory budget");
};

__device__ __forceinline__ int64_t mlp_tiles(const MlpParams& p, int64_t c0) {
  if (!p.counts) return (p.M + 127) / 128;
  return (c0 + 127) / 128 + (p.M - c0 + 127) / 128;
}
__device__ __forceinline__ bool mlp_tile(const MlpParams& p, int64_t c0, int64_t m, int& e,
                                         int64_t& r0, int64_t& r1) {
  if (!p.counts) {
    e = 0;
    r0 = m * 128;
    r1 = min(p.M, r0 + 128);
  } else {
    const int64_t t0 = (c0 + 127) / 128;
    if (m < t0) {
      e = 0;
      r0 = m * 128;
      r1 = min(c0, r0 + 128);
    } else {
      e = 1;
      r0 = c0 + (m - t0) * 128;
      r1 = min(p.M, r0 + 128);
    }
  }
  return r0 < r1;
}

// ---- one K step of MMAs per asm block (warp-uniform, one elected lane
// issues); every operand is passed in a register, no arithmetic inside.
// shift weights (one exact plane): lo·w, mid·w, hi·w
__device__ __forceinline__ void mma3(uint32_t d, uint32_t ah, uint32_t am, uint32_t al, uint64_t b,
                                     uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "r"(al), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// dense, six products into one accumulator: lo·hi, mid·mid, hi·lo, mid·hi, hi·mid, hi·hi
__device__ __forceinline__ void mma6(uint32_t d, uint32_t ah, uint32_t am, uint32_t al, uint64_t b0,
                                     uint64_t b1, uint64_t b2, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %4, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %5, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %6, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %7, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "r"(al), "l"(b0), "l"(b1), "l"(b2), "r"(id), "r"(acc)
      : "memory");
}
// dense, d = 32, B planes concatenated along N (rows 0-31 w_hi, 32-63 w_mid,
// 64-95 w_lo): columns [0,32) collect mh + lh + hl + hh, [32,64) mm + hm
__device__ __forceinline__ void mma_cat4(uint32_t d, uint32_t ah, uint32_t am, uint32_t al,
                                         uint64_t b0, uint64_t b2, uint32_t id64, uint32_t id32,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %6, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %4, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %6, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "r"(al), "l"(b0), "l"(b2), "r"(id64), "r"(id32), "r"(acc)
      : "memory");
}

// wide form, A lo plane from shared memory (descriptor), hi / mid from TMEM.
// shift: lo·w, mid·w, hi·w (the order of mma3)
__device__ __forceinline__ void mma3_lo(uint32_t d, uint32_t ah, uint32_t am, uint64_t alo, uint64_t b,
                                        uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "l"(alo), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// dense, six products in mma6's order (lo·hi from shared memory)
__device__ __forceinline__ void mma6_lo(uint32_t d, uint32_t ah, uint32_t am, uint64_t alo, uint64_t b0,
                                        uint64_t b1, uint64_t b2, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %5, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %6, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %7, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %7, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "l"(alo), "l"(b0), "l"(b1), "l"(b2), "r"(id), "r"(acc)
      : "memory");
}
// dense, B planes concatenated along N (rows 0-31 w_hi, 32-63 w_mid, 64-95
// w_lo): A_hi·[w_hi|w_mid|w_lo] → columns [0, 96), A_mid·[w_hi|w_mid] →
// [32, 96), A_lo·w_hi → [64, 96): column block j holds the products of
// combined order j (hh; hm + mh; hl + mm + lh)
__device__ __forceinline__ void mma_cat3(uint32_t d, uint32_t ah, uint32_t am, uint64_t alo,
                                         uint64_t b0, uint32_t id96, uint32_t id64, uint32_t id32,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t.reg .b32 d1, d2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %8, 0;\n\t"
      "add.u32 d1, %0, 32;\n\t"
      "add.u32 d2, %0, 64;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [d1], [%2], %4, %6, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [d2], %3, %4, %7, 1;\n\t}" ::"r"(d),
      "r"(ah), "r"(am), "l"(alo), "l"(b0), "r"(id96), "r"(id64), "r"(id32), "r"(acc)
      : "memory");
}

template <int D, bool RES, int NF, bool LNF = false>
__global__ void __launch_bounds__(Roles<D>::kThreads, 1) mlp_kernel(MlpParams p) {
  static_assert(!LNF || D == 32 || D == 64, "final LayerNorm: narrow form (d = 32 / 64)");
  using L = Layout<D, RES, LNF>;
  constexpr int kMma1 = Roles<D>::kMma1, kMma2 = Roles<D>::kMma2, kWld = Roles<D>::kWld;
  constexpr int NPW = Roles<D>::NPW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the swizzle pattern keys on absolute address bits: align the carve-out to 1 KB
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* a1_full = bar;
  uint64_t* a1_empty = a1_full + L::NA;
  uint64_t* w1_full = a1_empty + L::NA;
  uint64_t* w1_empty = w1_full + L::NW;
  uint64_t* w2_full = w1_empty + L::NW;
  uint64_t* w2_empty = w2_full + L::NW;
  uint64_t* h_full = w2_empty + L::NW;      // fc1(q) done
  uint64_t* h_empty = h_full + L::NB;       // GELU(q) wrote A2 (16 warps)
  uint64_t* buf_free = h_empty + L::NB;     // fc2(q) done reading A2: buffer reusable
  uint64_t* o_full = buf_free + L::NB;      // [NO] acc2 ready
  uint64_t* o_empty = o_full + L::NO;       // [NO] acc2 drained (producer warps)
  uint64_t* wres = o_empty + L::NO;         // resident weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + L::NBAR * 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef SA_DEBUG
  __shared__ unsigned long long sprof[S_N];
  if (tid < S_N) sprof[tid] = 0;
  const long long t_start = clock64();
#define PW(site, b, par_)                                                              \
  do {                                                                                 \
    if (p.dbg & 8) {                                                                   \
    } else if (p.prof) {                                                               \
      const long long t0_ = clock64();                                                 \
      mbar_wait(b, par_);                                                              \
      if (lane == 0) atomicAdd(&sprof[site], (unsigned long long)(clock64() - t0_));   \
    } else {                                                                           \
      mbar_wait(b, par_);                                                              \
    }                                                                                  \
  } while (0)
#define TL(ev, q)                                                                        \
  do {                                                                                   \
    if (p.tl && blockIdx.x == 0 && lane == 0 && (q) < 64) p.tl[(ev) * 64 + (q)] = clock64(); \
  } while (0)
#else
#define PW(site, b, par_) mbar_wait(b, par_)
#define TL(ev, q) do {} while (0)
#endif
  if (warp == kMma1) tmem_alloc<L::TCOLS>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < L::NA; ++i) {
      mbar_init(&a1_full[i], Roles<D>::PPG);
      mbar_init(&a1_empty[i], 1);
    }
    for (int i = 0; i < L::NW; ++i) {
      mbar_init(&w1_full[i], 1);
      mbar_init(&w1_empty[i], 1);
      mbar_init(&w2_full[i], 1);
      mbar_init(&w2_empty[i], 1);
    }
    for (int i = 0; i < L::NB; ++i) {
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], L::GPC);
      mbar_init(&buf_free[i], 1);
    }
    for (int i = 0; i < L::NO; ++i) {
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], Roles<D>::PPG);
    }
    mbar_init(wres, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t c0 = p.counts ? int64_t(p.counts[0]) : 0;
  const int64_t ntile = mlp_tiles(p, c0);
  constexpr int HC = L::HC;
  const int nchunk = p.hidden / HC;

  if (kDbg && (p.dbg & 8) && warp != kMma1 && warp != kMma2) {
    // debug: the MMA issuers alone, no waits (raw instruction-stream rate)
  } else if (warp >= kProd && warp < kMma1) {
    // ------- producers: x rows → A1 planes (TMEM); drain acc2 -------
    // warp (quad, kc0): rows quad·32 + lane (= TMEM lanes), K stages / output
    // channel blocks kc0, kc0 + KST, ... (narrow: one stage per warp; wide: one
    // warp per lane quarter walks every stage)
    // (PGN > 1: groups of PPG warps take the CTA's tiles alternately; each
    // group owns one A1 buffer and one acc2 buffer, NA = NO = PGN)
    constexpr int PGN = Roles<D>::PGN, PPG = Roles<D>::PPG;
    constexpr int KST = PPG / 4;
    static_assert(PGN == 1 || (PGN == L::NA && PGN == L::NO), "a group per A1 / acc2 buffer");
    const int pgi = (warp - kProd) / PPG, pwl = (warp - kProd) % PPG;
    const int quad = pwl & 3, kc0 = pwl >> 2;
    const int ptid = quad * 32 + lane;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    float* xb = reinterpret_cast<float*>(smem + L::OFF_XB) +
                (LNF ? pgi * 4 + quad : warp - kProd) * 32 * L::XP;
    // the warp's 16-column output blocks: 2 per owned K stage
    constexpr int NBLK = 2 * (L::KC1 / KST);
    auto blk_col = [&](int bi) { return 32 * (kc0 + (bi >> 1) * KST) + 16 * (bi & 1); };
    auto drain = [&](int64_t jt, int e, int64_t r0, int64_t r1) {
      const int ob = int(jt % L::NO);
      const uint32_t oph = uint32_t(jt / L::NO) & 1u;
      if (kDbg && (p.dbg & 2)) {
        PW(S_OF, &o_full[ob], oph);
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_empty[ob]);
        return;
      }
      const int64_t r = r0 + ptid;
      int64_t orow = -1;
      float gt = 1.f;
      if (r < r1) {
        orow = p.perm ? int64_t(__ldg(p.perm + r)) : r;
        if (p.gate) gt = __ldg(p.gate + orow);
      }
      // the lane's 4 output rows (it * 8 + lane / 4) and 4 channels per 16-wide
      // column block; residual rows prefetched one block ahead
      const int c4 = (lane & 3) * 4;
      int64_t orow_l[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) orow_l[it] = __shfl_sync(0xffffffffu, orow, it * 8 + (lane >> 2));
      float4 res[2][4];
      auto load_res = [&](int cb, float4 (&dst)[4]) {
#pragma unroll
        for (int it = 0; it < 4; ++it)
          dst[it] = (p.residual && orow_l[it] >= 0)
                        ? __ldg(reinterpret_cast<const float4*>(p.residual + orow_l[it] * D + cb + c4))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      load_res(blk_col(0), res[0]);
      const bool two = L::CAT && (e ? p.np1 : p.np0) == 3;   // dense d = 32: two partial sums
      PW(S_OF, &o_full[ob], oph);
      tc_fence_after();
      const uint32_t acc = tmem + lane_base + L::T_ACC2 + uint32_t(ob) * L::ACC2C;
      if constexpr (LNF) {
        // (1) gate · acc2 row-major into xb (thread = row), (2) + residual in
        // the transposed layout (coalesced residual loads), (3) the stage's
        // final LayerNorm per row with layernorm_row_kernel's operation order,
        // (4) coalesced stores of the normalised rows
        constexpr int XP = L::XP;
#pragma unroll
        for (int bi = 0; bi < NBLK; ++bi) {
          const int cb = blk_col(bi);
          float v[16];
          tmem_ld16(acc + uint32_t(cb), v);
          if (two) {
            float w[16];
            tmem_ld16(acc + 32u + uint32_t(cb), w);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = v[t] + w[t];
          }
#pragma unroll
          for (int t = 0; t < 16; t += 4)
            *reinterpret_cast<float4*>(xb + lane * XP + cb + t) =
                make_float4(v[t] * gt, v[t + 1] * gt, v[t + 2] * gt, v[t + 3] * gt);
        }
        __syncwarp();
#pragma unroll
        for (int bi = 0; bi < NBLK; ++bi) {
          const int cb = blk_col(bi);
          const int rb = bi & 1;
          if (bi + 1 < NBLK) load_res(blk_col(bi + 1), res[rb ^ 1]);
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int ri = it * 8 + (lane >> 2);
            float4* q = reinterpret_cast<float4*>(xb + ri * XP + cb + c4);
            float4 o = *q;
            if (p.residual) {
              const float4 rr = res[rb][it];
              o = make_float4(rr.x + o.x, rr.y + o.y, rr.z + o.z, rr.w + o.w);
            }
            *q = o;
          }
        }
        // d = 64: the lane quarter's two producer warps hold half a row each;
        // named barrier (id 1 + quad, 64 threads) before the statistics read
        // the other warp's columns, and again before either overwrites its own
        auto quad_sync = [&]() {
          if (KST > 1) asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
          else __syncwarp();
        };
        quad_sync();
        float mean = 0.f, inv = 0.f;
        const float4* xr = reinterpret_cast<const float4*>(xb + lane * XP);
        if (orow >= 0) {   // layernorm_row_kernel's operation order over the whole row
          float sm = 0.f;
#pragma unroll
          for (int i = 0; i < D / 4; ++i) {
            const float4 w = xr[i];
            sm += (w.x + w.y) + (w.z + w.w);
          }
          mean = sm / float(D);
          float q2 = 0.f;
#pragma unroll
          for (int i = 0; i < D / 4; ++i) {
            float4 w = xr[i];
            w.x -= mean; w.y -= mean; w.z -= mean; w.w -= mean;
            q2 += (w.x * w.x + w.y * w.y) + (w.z * w.z + w.w * w.w);
          }
          inv = 1.0f / sqrtf(q2 / float(D) + p.lnf_eps);
        }
        quad_sync();
        if (orow >= 0) {   // this warp's columns
#pragma unroll
          for (int bi = 0; bi < NBLK; bi += 2) {
            const int c0 = blk_col(bi) / 4;
#pragma unroll
            for (int i = c0; i < c0 + 8; ++i) {
              float4 w = xr[i];
              w.x -= mean; w.y -= mean; w.z -= mean; w.w -= mean;
              const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.lnf_g) + i);
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.lnf_b) + i);
              reinterpret_cast<float4*>(xb + lane * XP)[i] =
                  make_float4(w.x * inv * g4.x + b4.x, w.y * inv * g4.y + b4.y,
                              w.z * inv * g4.z + b4.z, w.w * inv * g4.w + b4.w);
            }
          }
        }
        __syncwarp();
#pragma unroll
        for (int bi = 0; bi < NBLK; ++bi) {
          const int cb = blk_col(bi);
          const int n = cb + c4;
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int ri = it * 8 + (lane >> 2);
            const int64_t orow_i = orow_l[it];
            if (orow_i < 0) continue;
            *reinterpret_cast<float4*>(p.y + orow_i * D + n) =
                *reinterpret_cast<const float4*>(xb + ri * XP + cb + c4);
          }
        }
        __syncwarp();
      } else {
#pragma unroll
      for (int bi = 0; bi < NBLK; ++bi) {
        const int cb = blk_col(bi);
        const int rb = bi & 1;
        if (bi + 1 < NBLK) load_res(blk_col(bi + 1), res[rb ^ 1]);
        float v[16];
        tmem_ld16(acc + uint32_t(cb), v);
        if (two) {
          float w[16];
          tmem_ld16(acc + 32u + uint32_t(cb), w);
#pragma unroll
          for (int t = 0; t < 16; ++t) v[t] = v[t] + w[t];
        }
#pragma unroll
        for (int t = 0; t < 16; t += 4)
          *reinterpret_cast<float4*>(xb + lane * kXPitch + t) =
              make_float4(v[t] * gt, v[t + 1] * gt, v[t + 2] * gt, v[t + 3] * gt);
        __syncwarp();
        const int n = cb + c4;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int ri = it * 8 + (lane >> 2);
          const int64_t orow_i = orow_l[it];
          if (orow_i < 0) continue;
          float4 o = *reinterpret_cast<const float4*>(xb + ri * kXPitch + c4);
          if (p.residual) {
            const float4 rr = res[rb][it];
            o = make_float4(rr.x + o.x, rr.y + o.y, rr.z + o.z, rr.w + o.w);
          }
          *reinterpret_cast<float4*>(p.y + orow_i * D + n) = o;
        }
        __syncwarp();
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ob]);
    };
    // the NA previous tiles (their acc2 is drained NA tiles later)
    int pe1 = 0, pe2 = 0;
    int64_t pa1 = 0, pb1 = 0, pa2 = 0, pb2 = 0;
    int64_t j = 0;   // this group's tile count
    int ab = PGN > 1 ? pgi : 0;   // PGN > 1: the group's own A1 buffer
    uint32_t pab = 0u;
    int64_t jall = 0;   // the CTA's valid-tile index (all groups)
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
      if (PGN > 1 && (jall++ % PGN) != pgi) continue;
      const int64_t row = r0 + ptid;
      const bool live = row < r1 && !(kDbg && (p.dbg & 2));
      const float* xrow = live ? p.x + (p.perm ? int64_t(__ldg(p.perm + row)) : row) * D : nullptr;
      float4 v[8];
      auto load_stage = [&](int kc) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = live ? __ldg(reinterpret_cast<const float4*>(xrow + 32 * kc) + i)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      load_stage(kc0);
      PW(S_A1E, &a1_empty[ab], pab ^ 1u);
      tc_fence_after();
      const uint32_t a1 = tmem + lane_base + L::T_A1 + uint32_t(ab) * L::A1COLS;
#pragma unroll 1
      for (int kc = kc0; kc < L::KC1; kc += KST) {
        if (kc != kc0) load_stage(kc);
        if (!(kDbg && (p.dbg & 2))) {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {   // 16 channels (8 bf16 pairs) at a time
            uint32_t hp[8], mp[8], lp[8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float4 q = v[sub * 4 + t];
              const Split3u a = split3x2_trunc(q.x, q.y);   // (no F2FP, as the GELU planes)
              const Split3u b = split3x2_trunc(q.z, q.w);
              hp[2 * t] = a.h;
              hp[2 * t + 1] = b.h;
              mp[2 * t] = a.m;
              mp[2 * t + 1] = b.m;
              lp[2 * t] = a.l;
              lp[2 * t + 1] = b.l;
            }
            const uint32_t col = a1 + kc * L::A1P * kPlaneCols + sub * 8;
            tmem_st8(col, hp);
            tmem_st8(col + kPlaneCols, mp);
            if constexpr (L::W) {   // lo plane → shared memory, UMMA canonical K-major layout
              uint8_t* lo = smem + L::OFF_ALO + kc * (kBM * 32 * 2);
              *reinterpret_cast<uint4*>(lo + plane_offset(ptid, 16 * sub)) =
                  make_uint4(lp[0], lp[1], lp[2], lp[3]);
              *reinterpret_cast<uint4*>(lo + plane_offset(ptid, 16 * sub + 8)) =
                  make_uint4(lp[4], lp[5], lp[6], lp[7]);
            } else {
              tmem_st8(col + 2 * kPlaneCols, lp);
            }
          }
        }
      }
      if constexpr (L::W) fence_proxy_async_smem();   // the lo plane is read by the tensor cores
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a1_full[ab]);
      if (PGN > 1) {
        // this group's previous tile (global index (j - 1)·PGN + group)
        pab ^= 1u;
        if (j >= 1) drain((j - 1) * PGN + pgi, pe1, pa1, pb1);
        pe1 = e; pa1 = r0; pb1 = r1;
        ++j;
        continue;
      }
      if (++ab == L::NA) { ab = 0; pab ^= 1u; }
      // then drain tile j - NA (its fc2 ends while fc1 works on the tiles between)
      if (L::NA == 1 && j >= 1) drain(j - 1, pe1, pa1, pb1);
      if (L::NA == 2 && j >= 2) drain(j - 2, pe2, pa2, pb2);
      pe2 = pe1; pa2 = pa1; pb2 = pb1;
      pe1 = e; pa1 = r0; pb1 = r1;
      ++j;
    }
    if (PGN > 1) {
      if (j >= 1) drain((j - 1) * PGN + pgi, pe1, pa1, pb1);
    } else {
      if (L::NA == 2 && j >= 2) drain(j - 2, pe2, pa2, pb2);
      if (j >= 1) drain(j - 1, pe1, pa1, pb1);
    }
  } else if (warp == kWld) {
    // ---------------- weights ----------------
    if (lane == 0) {
      if (RES) {
        const int ne = p.counts ? 2 : 1;
        uint32_t total = 0;
        for (int e = 0; e < ne; ++e)
          total += uint32_t(e ? p.np1 : p.np0) * uint32_t(p.hidden) * 64u * uint32_t(L::KC1 + D / 32);
        mbar_expect_tx(wres, total);
        for (int e = 0; e < ne; ++e) {
          const int np = e ? p.np1 : p.np0;
          const uint32_t b1 = uint32_t(L::KC1 * np) * uint32_t(p.hidden) * 64u;
          const uint32_t b2 = uint32_t(np) * uint32_t(p.hidden / 32) * uint32_t(D * 64);
          bulk_g2s(smem + L::r_w1(e), e ? p.w1[1] : p.w1[0], b1, wres);
          bulk_g2s(smem + L::r_w2(e), e ? p.w2[1] : p.w2[0], b2, wres);
        }
      } else {
        // W1 and W2 chunk rings, filled in chunk order (W1(q), W2(q), W1(q+1) ...)
        int s = 0;
        uint32_t ph = 0u;
        for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
          int e;
          int64_t r0, r1;
          if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
          const int np = e ? p.np1 : p.np0;
          const uint32_t by1 = uint32_t(L::KC1 * np) * (HC * 32 * 2);
          const uint32_t by2 = uint32_t((HC / 32) * np) * (D * 32 * 2);
          const uint8_t* s1 = reinterpret_cast<const uint8_t*>(e ? p.w1[1] : p.w1[0]);
          const uint8_t* s2 = reinterpret_cast<const uint8_t*>(e ? p.w2[1] : p.w2[0]);
          for (int c = 0; c < nchunk; ++c) {
            PW(S_WR, &w1_empty[s], ph ^ 1u);
            mbar_expect_tx(&w1_full[s], by1);
            bulk_g2s(smem + s * L::W1C, s1 + size_t(c) * by1, by1, &w1_full[s]);
            PW(S_WR, &w2_empty[s], ph ^ 1u);
            mbar_expect_tx(&w2_full[s], by2);
            bulk_g2s(smem + L::NW * L::W1C + s * L::W2C, s2 + size_t(c) * by2, by2, &w2_full[s]);
            if (++s == L::NW) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMma1) {
    // ---------------- fc1 issuer: x planes (A1) · W1 chunk → acc1 buffer ----------------
    constexpr uint32_t id1 = idesc_bf16_m128(HC);
    constexpr uint64_t BP = (HC * 64) >> 4;   // W1 plane stride (descriptor units)
    const uint32_t sbase = smem_u32(smem);
    if (RES) PW(S_W, wres, 0);
    int b = 0, ab = 0, s = 0, qq = 0;
    uint32_t pb = 0u, pab = 0u, ps = 0u;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
      const bool shift = (e ? p.np1 : p.np0) == 1;
      const uint32_t cstride = uint32_t(L::KC1 * (shift ? 1 : 3) * HC * 64);
      uint32_t wrow = sbase + L::r_w1(e);
      PW(S_A1F, &a1_full[ab], pab);
      const uint32_t a1 = tmem + L::T_A1 + uint32_t(ab) * L::A1COLS;
      for (int c = 0; c < nchunk; ++c, ++qq) {
        if (!RES) PW(S_W, &w1_full[s], ps);
        PW(S_BF, &buf_free[b], pb ^ 1u);   // fc2(q - 3) released the buffer
        TL(0, qq);
        tc_fence_after();
        const uint32_t d1 = tmem + L::T_BUF + uint32_t(b) * L::BUFC;
        const uint64_t bd0 = smem_desc(RES ? wrow : sbase + uint32_t(s) * L::W1C);
        if (!(kDbg && (p.dbg & 4))) {
          if constexpr (L::W) {
            constexpr uint32_t id96 = idesc_bf16_m128(96), id64 = idesc_bf16_m128(64);
            const uint32_t alo0 = smem_u32(smem + L::OFF_ALO);
#pragma unroll
            for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const uint32_t ah = a1 + kc * 2 * kPlaneCols + ks * 8;
                const uint64_t alo = smem_desc(alo0 + kc * (kBM * 32 * 2) + ks * 256);
                const uint32_t acc = (kc | ks) ? 1u : 0u;
                if (shift) {
                  mma3_lo(d1, ah, ah + kPlaneCols, alo,
                          bd0 + uint64_t((kc * (HC * 64) + ks * 256) >> 4), id1, acc);
                } else {
                  const uint64_t bd = bd0 + uint64_t((kc * (3 * HC * 64) + ks * 256) >> 4);
                  if (L::CATW)
                    mma_cat3(d1, ah, ah + kPlaneCols, alo, bd, id96, id64, id1, acc);
                  else
                    mma6_lo(d1, ah, ah + kPlaneCols, alo, bd, bd + BP, bd + 2 * BP, id1, acc);
                }
              }
          } else {
#pragma unroll
          for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ah = a1 + kc * 3 * kPlaneCols + ks * 8;
              const uint32_t acc = (kc | ks) ? 1u : 0u;
              if (shift) {
                mma3(d1, ah, ah + kPlaneCols, ah + 2 * kPlaneCols,
                     bd0 + uint64_t((kc * (HC * 64) + ks * 256) >> 4), id1, acc);
              } else {
                const uint64_t bd = bd0 + uint64_t((kc * (3 * HC * 64) + ks * 256) >> 4);
                mma6(d1, ah, ah + kPlaneCols, ah + 2 * kPlaneCols, bd, bd + BP, bd + 2 * BP, id1, acc);
              }
            }
          }
        }
        commit_w(&h_full[b]);
        TL(1, qq);
        if (!RES) commit_w(&w1_empty[s]);
        if (++b == L::NB) { b = 0; pb ^= 1u; }
        if (++s == L::NW) { s = 0; ps ^= 1u; }
        wrow += cstride;
      }
      commit_w(&a1_empty[ab]);   // A1 fully consumed
      if (++ab == L::NA) { ab = 0; pab ^= 1u; }
    }
  } else if (warp == kMma2) {
    // ---------------- fc2 issuer: GELU planes (A2) · W2 chunk → acc2 ----------------
    constexpr uint32_t id64 = idesc_bf16_m128(64);
    constexpr uint32_t id32 = idesc_bf16_m128(32);
    constexpr uint32_t id2 = idesc_bf16_m128(D);
    constexpr uint64_t BP = (D * 64) >> 4;    // W2 plane stride (descriptor units)
    const uint32_t sbase = smem_u32(smem);
    if (RES) PW(S_W, wres, 0);
    int b = 0, ob = 0, s = 0, qq = 0;
    uint32_t pb = 0u, pob = 0u, ps = 0u;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
      const bool shift = (e ? p.np1 : p.np0) == 1;
      const uint32_t cstride = uint32_t((HC / 32) * (shift ? 1 : 3) * D * 64);
      uint32_t wrow = sbase + L::r_w2(e);
      PW(S_OE, &o_empty[ob], pob ^ 1u);   // acc2[ob] drained
      const uint32_t d2 = tmem + L::T_ACC2 + uint32_t(ob) * L::ACC2C;
      for (int c = 0; c < nchunk; ++c, ++qq) {
        if (!RES) PW(S_W, &w2_full[s], ps);
        PW(S_HE, &h_empty[b], pb);        // GELU(q) wrote A2[b]
        TL(4, qq);
        tc_fence_after();
        const uint32_t bb = tmem + L::T_BUF + uint32_t(b) * L::BUFC;
        const uint64_t bd0 = smem_desc(RES ? wrow : sbase + L::NW * L::W1C + uint32_t(s) * L::W2C);
        const uint32_t a0 = c != 0 ? 1u : 0u;
        if (!(kDbg && (p.dbg & 4))) {
#pragma unroll
          for (int ks = 0; ks < HC / 16; ++ks) {
            // A2 planes of K step ks: kGeluAlt: hi at 32(ks/2) + 8(ks%2), mid 16
            // further, lo at 64 + 16(ks/2) + 8(ks%2); else hi at 16ks, mid at
            // 16ks + 8, lo at 64 + 8ks
            const uint32_t ah = kGeluAlt ? bb + (ks >> 1) * 32u + (ks & 1) * 8u : bb + ks * 16u;
            const uint32_t am = ah + (kGeluAlt ? 16u : 8u);
            const uint32_t al = kGeluAlt ? bb + 64u + (ks >> 1) * 16u + (ks & 1) * 8u
                                : (L::CATW ? bb + 32u + ks * 16u : bb + uint32_t(HC) + ks * 8u);
            const uint32_t acc = ks ? 1u : a0;
            if (shift) {
              mma3(d2, ah, am, al, bd0 + uint64_t(((ks >> 1) * (D * 64) + (ks & 1) * 256) >> 4),
                   id2, acc);
            } else {
              const uint64_t bd = bd0 + uint64_t(((ks >> 1) * (3 * D * 64) + (ks & 1) * 256) >> 4);
              if (L::CAT)
                mma_cat4(d2, ah, am, al, bd, bd + 2 * BP, id64, id32, acc);
              else
                mma6(d2, ah, am, al, bd, bd + BP, bd + 2 * BP, id2, acc);
            }
          }
        }
        commit_w(&buf_free[b]);
        TL(5, qq);
        if (!RES) commit_w(&w2_empty[s]);
        if (++b == L::NB) { b = 0; pb ^= 1u; }
        if (++s == L::NW) { s = 0; ps ^= 1u; }
        wrow += cstride;
      }
      commit_w(&o_full[ob]);
      if (++ob == L::NO) { ob = 0; pob ^= 1u; }
    }
  } else if (warp < kGelu && kGeluAlt && !L::W) {
    // ------- GELU: group gs = warp / 8 takes chunks q % 2 == gs; warp (h, quad)
    // of the group takes hidden columns [32h, 32h + 32) = fc2 K steps 2h, 2h+1.
    // Its planes go over its own consumed accumulator columns (hi [32h, 32h+16),
    // mid [32h+16, 32h+32)) and the free columns [64 + 16h, 80 + 16h) (lo) -------
    const int gs = warp >> 3, h = (warp >> 2) & 1, quad = warp & 3;
    const uint32_t lb = tmem + (uint32_t(quad * 32) << 16) + L::T_BUF;
    int nt = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (mlp_tile(p, c0, m, e, r0, r1)) ++nt;
    }
    const int total_q = nt * nchunk;
    for (int q = gs; q < total_q; q += 2) {
      const int b = q % L::NB;
      const uint32_t ph = uint32_t(q / L::NB) & 1u;
      PW(S_HF, &h_full[b], ph);             // fc1(q) done
      if (warp == 0) TL(2, q);
      tc_fence_after();
      const uint32_t bb = lb + uint32_t(b) * kBufCols;
      if (!(kDbg && (p.dbg & 1))) {
        uint32_t r[32];
        tmem_ld32_nowait(bb + uint32_t(32 * h), r);
        tmem_ld_wait();
        uint32_t hp[16], mp[16], lp[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          float g0 = __uint_as_float(r[2 * t]), g1 = __uint_as_float(r[2 * t + 1]);
          if (kDbg && (p.dbg & 64)) {   // debug: no GELU math
          } else if (t < 2 * NF) {
            gelu_pair<true>(g0, g1);
          } else {
            gelu_pair<false>(g0, g1);
          }
          const Split3u sp = split3x2_trunc(g0, g1);   // no F2FP: the MUFU pipe is the GELU's
          hp[t] = sp.h;
          mp[t] = sp.m;
          lp[t] = sp.l;
        }
        tmem_st16(bb + uint32_t(32 * h), hp);
        tmem_st16(bb + uint32_t(32 * h + 16), mp);
        tmem_st16(bb + uint32_t(64 + 16 * h), lp);
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&h_empty[b]);
      if (warp == 0) TL(3, q);
      if (warp == kGelu - 1) TL(6, q);
    }
  } else if (warp < kGelu) {
    // ------- GELU (kGeluAlt = false): warp (k, quad) takes hidden columns [16k, 16k + 16) of a
    // chunk = K step k of fc2; its planes go over its own consumed accumulator
    // columns (hi [16k, 16k + 8), mid [16k + 8, 16k + 16)) and the free
    // columns [HC + 8k, HC + 8k + 8) (lo). Narrow (HC = 64): all 16 warps on
    // every chunk; wide (HC = 32): groups of 8 warps (gs = warp / 8) on
    // alternate chunks -------
    const int gs = L::W ? warp >> 3 : 0;
    const int k = L::W ? (warp >> 2) & 1 : warp >> 2, quad = warp & 3;
    constexpr int QS = L::W ? 2 : 1;
    const uint32_t lb = tmem + (uint32_t(quad * 32) << 16) + L::T_BUF;
    int nt = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (mlp_tile(p, c0, m, e, r0, r1)) ++nt;
    }
    const int total_q = nt * nchunk;
    if constexpr (L::W) {
      // chunk q (global chunk index of this CTA); cat3: dense wide tile whose
      // acc1 holds three partial sums (mma_cat3)
      auto gelu_chunk = [&](int q, int b, uint32_t ph, bool cat3) {
        PW(S_HF, &h_full[b], ph);             // fc1(q) done
        if (warp == 0) TL(2, q);
        tc_fence_after();
        const uint32_t bb = lb + uint32_t(b) * L::BUFC;
        if (!(kDbg && (p.dbg & 1))) {
          float r[16];
          if (kDbg && (p.dbg & 128)) {   // debug: no TMEM traffic (synthetic inputs, no stores)
  #pragma unroll
            for (int t = 0; t < 16; ++t) r[t] = float(t + q) * 0.01f;
          } else if (L::CATW && cat3) {
            float r1[16], r2[16];
            tmem_ld16(bb + uint32_t(16 * k), r);
            tmem_ld16(bb + uint32_t(32 + 16 * k), r1);
            tmem_ld16(bb + uint32_t(64 + 16 * k), r2);
  #pragma unroll
            for (int t = 0; t < 16; ++t) r[t] = r[t] + (r1[t] + r2[t]);   // hh + (hm+mh + hl+mm+lh)
          } else {
            tmem_ld16(bb + uint32_t(16 * k), r);
          }
          uint32_t hp[8], mp[8], lp[8];
  #pragma unroll
          for (int t = 0; t < 8; ++t) {
            float g0 = r[2 * t], g1 = r[2 * t + 1];
            if (kDbg && (p.dbg & 64)) {   // debug: no GELU math
            } else if (t < NF) {
              gelu_pair<true>(g0, g1);
            } else {
              gelu_pair<false>(g0, g1);
            }
            const Split3u sp = split3x2_trunc(g0, g1);   // no F2FP: the MUFU pipe is the GELU's
            hp[t] = sp.h;
            mp[t] = sp.m;
            lp[t] = sp.l;
          }
          if (kDbg && (p.dbg & 128)) {
            if (hp[0] == 0x12345u && mp[1] == 7u && lp[2] == 9u) mbar_arrive(&h_empty[b]);   // keep the math live
          } else {
            tmem_st8(bb + uint32_t(16 * k), hp);
            tmem_st8(bb + uint32_t(16 * k + 8), mp);
            // lo: over this warp's own consumed columns of block 1 (CATW), else the free columns
            tmem_st8(bb + uint32_t(L::CATW ? 32 + 16 * k : HC + 8 * k), lp);
            tmem_st_wait();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&h_empty[b]);
        if (warp == 0) TL(3, q);
        if (warp == kGelu - 1) TL(6, q);
      };
      int q = 0;
      for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
        int e;
        int64_t r0, r1;
        if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
        const bool dense = (e ? p.np1 : p.np0) == 3;
        for (int c = 0; c < nchunk; ++c, ++q)
          if ((q % QS) == gs) gelu_chunk(q, q % L::NB, uint32_t(q / L::NB) & 1u, dense);
      }
    } else {
      for (int q = 0; q < total_q; ++q) {
        const int b = q % L::NB;
        const uint32_t ph = uint32_t(q / L::NB) & 1u;
        PW(S_HF, &h_full[b], ph);             // fc1(q) done
        if (warp == 0) TL(2, q);
        tc_fence_after();
        const uint32_t bb = lb + uint32_t(b) * L::BUFC;
        if (!(kDbg && (p.dbg & 1))) {
          float r[16];
          if (kDbg && (p.dbg & 128)) {   // debug: no TMEM traffic (synthetic inputs, no stores)
  #pragma unroll
            for (int t = 0; t < 16; ++t) r[t] = float(t + q) * 0.01f;
          } else if (false) {
            float r1[16], r2[16];
            tmem_ld16(bb + uint32_t(16 * k), r);
            tmem_ld16(bb + uint32_t(32 + 16 * k), r1);
            tmem_ld16(bb + uint32_t(64 + 16 * k), r2);
  #pragma unroll
            for (int t = 0; t < 16; ++t) r[t] = r[t] + (r1[t] + r2[t]);   // hh + (hm+mh + hl+mm+lh)
          } else {
            tmem_ld16(bb + uint32_t(16 * k), r);
          }
          uint32_t hp[8], mp[8], lp[8];
  #pragma unroll
          for (int t = 0; t < 8; ++t) {
            float g0 = r[2 * t], g1 = r[2 * t + 1];
            if (kDbg && (p.dbg & 64)) {   // debug: no GELU math
            } else if (t < NF) {
              gelu_pair<true>(g0, g1);
            } else {
              gelu_pair<false>(g0, g1);
            }
            const Split3u sp = split3x2_trunc(g0, g1);   // no F2FP: the MUFU pipe is the GELU's
            hp[t] = sp.h;
            mp[t] = sp.m;
            lp[t] = sp.l;
          }
          if (kDbg && (p.dbg & 128)) {
            if (hp[0] == 0x12345u && mp[1] == 7u && lp[2] == 9u) mbar_arrive(&h_empty[b]);   // keep the math live
          } else {
            tmem_st8(bb + uint32_t(16 * k), hp);
            tmem_st8(bb + uint32_t(16 * k + 8), mp);
            // lo: over this warp's own consumed columns of block 1 (CATW), else the free columns
            tmem_st8(bb + uint32_t(L::CATW ? 32 + 16 * k : HC + 8 * k), lp);
            tmem_st_wait();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&h_empty[b]);
        if (warp == 0) TL(3, q);
        if (warp == kGelu - 1) TL(6, q);
      }
    }
    (void)total_q;
  }
#ifdef SA_DEBUG
  if (p.prof && lane == 0) {
    const int site = warp < kGelu ? T_GELU
                     : (warp < kMma1 ? T_PROD : (warp == kMma1 ? T_MMA1 : (warp == kMma2 ? T_MMA2 : -1)));
    if (site >= 0) atomicAdd(&sprof[site], (unsigned long long)(clock64() - t_start));
  }
#endif
#undef PW
#undef TL
  tc_fence_before();
  __syncthreads();
#ifdef SA_DEBUG
  if (p.prof && tid < S_N) atomicAdd(p.prof + tid, sprof[tid]);
#endif
  if (warp == kMma1) tmem_dealloc<L::TCOLS>(tmem);
}

}  // namespace tcm

// GELU pairs (of 8 per thread and chunk) whose reciprocal runs on the FMA pipe
SA_DEBUG_SWITCH(int, g_mlp_gelu_fma, 0, sa_debug_mlp_mode)
SA_DEBUG_SWITCH(int, g_mlp_dbg, 0, sa_debug_mlp_roles)
#ifdef SA_DEBUG
static unsigned long long* g_mlp_prof = nullptr;
extern "C" void sa_debug_mlp_profile(void* dev_buf) {
  g_mlp_prof = static_cast<unsigned long long*>(dev_buf);
}
static long long* g_mlp_tl = nullptr;
extern "C" void sa_debug_mlp_timeline(void* dev_buf) { g_mlp_tl = static_cast<long long*>(dev_buf); }
#else
static constexpr unsigned long long* g_mlp_prof = nullptr;
static constexpr long long* g_mlp_tl = nullptr;
#endif

static int g_sms_mlp = 0;

template <int D, bool RES, int NF, bool LNF = false>
static void mlp_launch_one(const tcm::MlpParams& p, int grid, cudaStream_t s) {
  const int smem = int(tcm::Layout<D, RES, LNF>::TOTAL);
  cudaFuncSetAttribute(tcm::mlp_kernel<D, RES, NF, LNF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  tcm::mlp_kernel<D, RES, NF, LNF><<<grid, tcm::Roles<D>::kThreads, smem, s>>>(p);
}

template <int D, bool RES>
static void mlp_launch_nf(const tcm::MlpParams& p, int grid, cudaStream_t s) {
  switch (g_mlp_gelu_fma) {
#ifdef SA_DEBUG
    case 2: mlp_launch_one<D, RES, 2>(p, grid, s); break;
    case 4: mlp_launch_one<D, RES, 4>(p, grid, s); break;
#endif
    default: mlp_launch_one<D, RES, MLP_NF>(p, grid, s); break;
  }
}

static int mlp_launch(tcm::MlpParams& p, int d, cudaStream_t s) {
  using namespace tcm;
  if (p.M == 0) return SA_OK;
  p.prof = g_mlp_prof;
  p.tl = g_mlp_tl;
  p.dbg = g_mlp_dbg;
  if (g_sms_mlp == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_mlp, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = cdiv(p.M, 128) + (p.counts ? 1 : 0);
  const int grid = int(tiles < g_sms_mlp ? tiles : g_sms_mlp);
  if (p.lnf_g) {   // the stage's final LayerNorm (d = 32 / 64, checked by the caller)
    if (d == 64)
      mlp_launch_one<64, false, 0, true>(p, grid, s);
    else if (p.hidden <= kResHidden)
      mlp_launch_one<32, true, 0, true>(p, grid, s);
    else
      mlp_launch_one<32, false, 0, true>(p, grid, s);
  } else if (d == 32) {
    if (p.hidden <= kResHidden)
      mlp_launch_nf<32, true>(p, grid, s);
    else
      mlp_launch_nf<32, false>(p, grid, s);
  } else if (d == 64) {
    mlp_launch_nf<64, false>(p, grid, s);
  } else if (d == 128) {
    mlp_launch_nf<128, false>(p, grid, s);
  } else {
    mlp_launch_nf<160, false>(p, grid, s);
  }
  count_launch(1);
  SA_LAUNCH_CHECK("mlp_kernel");
  return SA_OK;
}

}  // namespace sa

using namespace sa;

/* The fused kernels read W1 packed with bn = sa_tc_fused_mlp_chunk(d) (the
 * hidden chunk: 64 for d = 32 / 64, 32 for d = 128 / 160) and W2 packed with
 * bn = d; see sa_weight_pack. */
extern "C" int sa_tc_fused_mlp_chunk(int64_t d) {
  // (d = 192 builds and is exact, but fc1's 72 N = 32 MMAs per chunk make it
  // slower than the two-GEMM path: 391 vs 353 us at the DeiT-T shape)
  return (d == 32 || d == 64) ? 64 : (d == 128 || d == 160) ? 32 : 0;
}

extern "C" int sa_tc_fused_mlp_ok(int64_t d, int64_t hidden) {
  const int hc = sa_tc_fused_mlp_chunk(d);
  return hc > 0 && hidden % hc == 0 && hidden > 0 && hidden <= 8192;
}

extern "C" int sa_tc_fused_mlp_w1_bn(void) { return tcm::HC; }

extern "C" int sa_tc_moe_mlp_fused(const float* x, const int32_t* perm, const int32_t* counts,
                                   const float* gate, const void* w1_dense, const void* w2_dense,
                                   const void* w1_shift, const void* w2_shift, float* y,
                                   const float* residual, int64_t M, int64_t d, int64_t hidden,
                                   void* stream) {
  SA_REQUIRE(sa_tc_fused_mlp_ok(d, hidden), SA_ERR_SHAPE,
             "sa_tc_moe_mlp_fused: d=%lld hidden=%lld unsupported", (long long)d,
             (long long)hidden);
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_tc_moe_mlp_fused: M=%lld out of range",
             (long long)M);
  tcm::MlpParams p;
  memset(&p, 0, sizeof(p));
  p.x = x;
  p.perm = perm;
  p.counts = counts;
  p.gate = gate;
  p.residual = residual;
  p.y = y;
  p.w1[0] = static_cast<const uint16_t*>(w1_dense);
  p.w2[0] = static_cast<const uint16_t*>(w2_dense);
  p.w1[1] = static_cast<const uint16_t*>(w1_shift);
  p.w2[1] = static_cast<const uint16_t*>(w2_shift);
  p.np0 = 3;
  p.np1 = 1;
  p.M = M;
  p.hidden = int(hidden);
  return mlp_launch(p, int(d), as_stream(stream));
}

/* sa_tc_moe_mlp_fused with the stage's final LayerNorm (Model stage norm,
 * model.py:565-577; tensor.py:114-128) applied to the output rows in the same
 * kernel: y = LN(residual + gate · expert(x)), bit-identical to
 * sa_tc_moe_mlp_fused followed by sa_layernorm; d = 32. */
extern "C" int sa_tc_moe_mlp_fused_ln(const float* x, const int32_t* perm, const int32_t* counts,
                                      const float* gate, const void* w1_dense, const void* w2_dense,
                                      const void* w1_shift, const void* w2_shift, float* y,
                                      const float* residual, int64_t M, int64_t d, int64_t hidden,
                                      const float* ln_gain, const float* ln_bias, float eps,
                                      void* stream) {
  SA_REQUIRE((d == 32 || d == 64) && sa_tc_fused_mlp_ok(d, hidden), SA_ERR_SHAPE,
             "sa_tc_moe_mlp_fused_ln: d=%lld hidden=%lld unsupported (d = 32 / 64)", (long long)d,
             (long long)hidden);
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE,
             "sa_tc_moe_mlp_fused_ln: M=%lld out of range", (long long)M);
  SA_REQUIRE(ln_gain != nullptr && ln_bias != nullptr, SA_ERR_VALUE,
             "sa_tc_moe_mlp_fused_ln: LayerNorm gain and bias required");
  tcm::MlpParams p;
  memset(&p, 0, sizeof(p));
  p.x = x;
  p.perm = perm;
  p.counts = counts;
  p.gate = gate;
  p.residual = residual;
  p.y = y;
  p.w1[0] = static_cast<const uint16_t*>(w1_dense);
  p.w2[0] = static_cast<const uint16_t*>(w2_dense);
  p.w1[1] = static_cast<const uint16_t*>(w1_shift);
  p.w2[1] = static_cast<const uint16_t*>(w2_shift);
  p.np0 = 3;
  p.np1 = 1;
  p.M = M;
  p.hidden = int(hidden);
  p.lnf_g = ln_gain;
  p.lnf_b = ln_bias;
  p.lnf_eps = eps;
  return mlp_launch(p, int(d), as_stream(stream));
}

extern "C" int sa_tc_mlp_fused(const float* x, const void* w1pack, int w1_kind,
                               const void* w2pack, int w2_kind, float* y, int64_t M, int64_t d,
                               int64_t hidden, const float* residual, void* stream) {
  SA_REQUIRE(sa_tc_fused_mlp_ok(d, hidden), SA_ERR_SHAPE,
             "sa_tc_mlp_fused: d=%lld hidden=%lld unsupported", (long long)d, (long long)hidden);
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_tc_mlp_fused: M=%lld out of range",
             (long long)M);
  SA_REQUIRE(w1_kind == w2_kind, SA_ERR_VALUE, "sa_tc_mlp_fused: fc1/fc2 kinds differ");
  tcm::MlpParams p;
  memset(&p, 0, sizeof(p));
  p.x = x;
  p.residual = residual;
  p.y = y;
  p.w1[0] = static_cast<const uint16_t*>(w1pack);
  p.w2[0] = static_cast<const uint16_t*>(w2pack);
  p.np0 = w1_kind == SA_W_SHIFT ? 1 : 3;
  p.np1 = p.np0;
  p.M = M;
  p.hidden = int(hidden);
  return mlp_launch(p, int(d), as_stream(stream));
}
