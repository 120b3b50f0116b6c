// Persistent warp-specialized tcgen05 GEMM (see tcgemm.cu for the numerics).
//
// One CTA per SM, 17 warps, tiles of 128 rows x BN columns processed in a
// static stride; the CTA's j-th non-empty tile belongs to "lane" g = j & 1:
//   warps  8-11 / 12-15  producer group g: per 32-wide K stage, gather the
//                        tile's 128 A rows with coalesced 128-bit loads (plain /
//                        MoE-permuted / patchified image), split them into
//                        hi/mid/lo bf16 planes in the UMMA canonical layout; one
//                        thread pulls the weight planes of the stage with a
//                        single bulk async copy (TMA engine, complete_tx);
//   warp  16             MMA issuer: one thread chains tcgen05.mma into TMEM
//                        accumulator g and commits to the mbarriers;
//   warp  17             A loader (plain / MoE-gathered rows): bulk-copies the
//                        tile's fp32 row segments (TMA engine, 128 B per row and
//                        K stage) into staging slots several stages ahead, one
//                        ring per producer group (a ring has exactly one in-order
//                        consumer, so an mbarrier parity can never alias a fill
//                        two phases old), so the producers read A from shared
//                        memory and HBM latency stays off their critical path
//                        (p.nst = 0: producers load A themselves — patchify);
//   warps  0-3 / 4-7     epilogue group g: tcgen05.ld (thread = accumulator
//                        row), GELU / x gate, transpose through shared memory,
//                        then coalesced 64-byte row segments with residual /
//                        position add and MoE scatter back to token order.
// Two producer groups, two TMEM accumulators and two epilogue groups keep
// two tiles' latency chains in flight; each group owns every other stage of
// the shared-memory ring (full/empty mbarriers), tfull/tempty hand the
// accumulators between MMA and epilogue.
#pragma once

#include "tc_common.cuh"

namespace sa {
namespace tc {

constexpr int kBM = 128;
// The A-staging loader (warp 17) measured slower than direct producer loads on
// every projection shape (per-row bulk copies saturate the TMA unit; cp.async
// staging adds a hop without shortening the per-tile latency chain), so it is
// compiled out; the code is kept for reference and A/B runs.
constexpr bool kStaging = false;
constexpr int kThreads = kStaging ? 576 : 544;
constexpr int kMmaWarp = 16;
constexpr int kLoadWarp = 17;
constexpr uint32_t kStgBytes = kBM * kBK * 4;   // one fp32 staging slot (128 rows x 32 k)
constexpr uint32_t kPlaneA = kBM * kBK * 2;  // bytes per A plane
constexpr int kXPitch = 20;                   // transpose buffer pitch (floats, 16B rows)
constexpr int kXPitchW = 36;                  // 32-column transpose pitch (wide tiles)
// per-epilogue-warp smem slot (1 KB multiple): a TMA box (32x32 fp32) or the
// transpose buffer (32 x kXPitch) + residual staging [2][32][16]
constexpr uint32_t kWarpSlot = 7168;

enum AMode { A_PLAIN = 0, A_GATHER = 1, A_PATCH = 2 };

struct TcParams {
  const float* A;
  int64_t lda;
  const int32_t* a_rows;
  int64_t pH, pW, pC, patch, pside;
  float sub;
  const uint16_t* Bp[6];     // packed weights per row group (expert; or problem x expert)
  int nplanes[6];
  int64_t M, K, N;
  int kchunks;
  int ntiles;
  int stages;  // even; group g owns stages g, g+2, ...
  const int32_t* counts;
  float* C;
  const int32_t* c_rows;
  const float* gate;
  const float* residual;
  int act;
  const float* pos;
  int64_t img_tokens;
  int extra;
  int nst;     // A staging slots over both rings (2, 4 or 8; 0 = producers load A directly)
  int rb;      // 1: every weight tile resident in shared memory for the whole kernel
  uint32_t rb_bytes[2];   // resident bytes per expert (packed planes, [n_tile][kc][plane])
  int dbg;     // debug role isolation (0 in production): 1 no A loads, 2 no C stores, 4 no MMAs
  int tma_c;   // 1: C rows are the tile rows (no scatter / position): TMA-store epilogue
  int kq_min;  // K stages alternate between producer groups when kchunks > kq_min (else whole tiles)
  int ngroups;         // > 2: grouped problems — counts[2i], counts[2i+1] are problem i's
                       // expert sizes, its rows are [i·prob_rows, (i+1)·prob_rows) of the
                       // gathered / scattered row space (a_rows, c_rows stacked per problem)
  int64_t prob_rows;
  const float* ln_g;   // LNE instantiation: LayerNorm of each output row (N = BN ∈ {32, 64})
  const float* ln_b;
  float ln_eps;
};

// TMEM accumulators: four buffers when they fit (BN <= 128), so the MMA can run
// two tiles ahead of each epilogue group; else two.
template <int BN>
struct Acc {
  static constexpr int N = 4 * BN <= 512 ? 4 : 2;
  static constexpr uint32_t COLS = N * BN;
  static constexpr uint32_t TCOLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128
                                    : COLS <= 256 ? 256 : 512;   // power of two >= 32
};

struct TileInfo {
  int group;  // expert
  int64_t r0, r1;
  int n_tile;
};

// Row groups of the GEMM (one per expert, or per problem x expert) with their
// first m-tile, first row and size; built once per CTA in shared memory.
struct GroupTab {
  int n;
  int tile0[7];
  int64_t row0[6], cnt[6];
};

__device__ __forceinline__ void build_groups(const TcParams& p, GroupTab& g) {
  if (!p.counts) {
    g.n = 1;
    g.row0[0] = 0;
    g.cnt[0] = p.M;
  } else if (p.ngroups > 2) {
    g.n = p.ngroups;
    for (int i = 0; i < g.n; ++i) {
      const int64_t c = p.counts[i & ~1];   // the problem's expert-0 size
      g.row0[i] = int64_t(i >> 1) * p.prob_rows + ((i & 1) ? c : 0);
      g.cnt[i] = (i & 1) ? p.prob_rows - c : c;
    }
  } else {
    const int64_t c0 = p.counts[0];
    g.n = 2;
    g.row0[0] = 0;
    g.cnt[0] = c0;
    g.row0[1] = c0;
    g.cnt[1] = p.M - c0;
  }
  int t = 0;
  for (int i = 0; i < g.n; ++i) {
    g.tile0[i] = t;
    t += int((g.cnt[i] + kBM - 1) / kBM);
  }
  g.tile0[g.n] = t;
}

__device__ __forceinline__ int64_t num_m_tiles(const GroupTab& g) { return g.tile0[g.n]; }

// m-tiles: group i owns tiles [tile0[i], tile0[i+1]) over its rows.
// t < 2^31 (checked on the host); ntiles == 1 (N <= BN) avoids the division.
// GRP: grouped problems (table walk); otherwise at most two expert groups.
template <bool GRP>
__device__ __forceinline__ TileInfo tile_info(const TcParams& p, const GroupTab& G, int t) {
  TileInfo ti;
  int m = t;
  ti.n_tile = 0;
  if (p.ntiles != 1) {
    m = t / p.ntiles;
    ti.n_tile = t - m * p.ntiles;
  }
  if (!p.counts) {   // one group: no table lookups
    ti.group = 0;
    ti.r0 = int64_t(m) * kBM;
    ti.r1 = min(p.M, ti.r0 + kBM);
    return ti;
  }
  if (!GRP) {        // expert 0 owns ceil(c0/128) tiles, expert 1 the rest
    const int t0 = G.tile0[1];
    const int64_t c0 = G.cnt[0];
    if (m < t0) {
      ti.group = 0;
      ti.r0 = int64_t(m) * kBM;
      ti.r1 = min(c0, ti.r0 + kBM);
    } else {
      ti.group = 1;
      ti.r0 = c0 + (int64_t(m) - t0) * kBM;
      ti.r1 = min(p.M, ti.r0 + kBM);
    }
    return ti;
  }
  int g = 0;
  while (g + 1 < G.n && m >= G.tile0[g + 1]) ++g;
  ti.group = g;
  ti.r0 = G.row0[g] + int64_t(m - G.tile0[g]) * kBM;
  ti.r1 = min(G.row0[g] + G.cnt[g], ti.r0 + kBM);
  return ti;
}

// The next non-empty tile at or after t whose ordinal among the CTA's non-empty
// tiles has parity g (the tiles a producer / epilogue group owns; g < 0: any);
// j counts the ordinals. Returns total when there is none.
template <bool GRP>
__device__ __forceinline__ int next_group_tile(const TcParams& p, const GroupTab& G, int total,
                                               int g, int t, int& j, int& jj, TileInfo& ti) {
  for (; t < total; t += gridDim.x) {
    ti = tile_info<GRP>(p, G, t);
    if (ti.r0 >= ti.r1) continue;
    jj = j++;
    if (g < 0 || (jj & 1) == g) return t;   // g < 0: every non-empty tile
  }
  return total;
}

__device__ __forceinline__ float gelu_fast(float x) {
  // 0.5·x·(1 + tanh(u)) == x / (1 + exp(-2u)); ex2.approx + fast divide keep
  // ~1e-7 relative accuracy (the reference's tanh is itself a float32 libm call)
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float u = c * (x + a * (x * x * x));
  return __fdividef(x, 1.0f + __expf(-2.0f * u));
}

// gelu_fast on a pair with packed f32x2 multiplies / fma / add: per lane the
// same operations as gelu_fast (x·x, x·x², fma(x³, a, x), ·c, ·(-2), ·log2e,
// ex2.approx, +1, div.approx), so the results are bitwise identical
__device__ __forceinline__ void gelu_fast2(float& x0, float& x1) {
  float t0, t1;
  asm("{\n\t.reg .b64 x, q, u, k;\n\t"
      "mov.b64 x, {%2, %3};\n\t"
      "mul.rn.f32x2 q, x, x;\n\t"
      "mul.rn.f32x2 q, x, q;\n\t"
      "mov.b64 k, {%4, %4};\n\t"
      "fma.rn.f32x2 u, q, k, x;\n\t"
      "mov.b64 k, {%5, %5};\n\t"
      "mul.rn.f32x2 u, u, k;\n\t"
      "mov.b64 k, {%6, %6};\n\t"
      "mul.rn.f32x2 u, u, k;\n\t"
      "mov.b64 k, {%7, %7};\n\t"
      "mul.rn.f32x2 u, u, k;\n\t"
      "mov.b64 {%0, %1}, u;\n\t}"
      : "=f"(t0), "=f"(t1)
      : "f"(x0), "f"(x1), "f"(0.044715f), "f"(0.7978845608028654f), "f"(-2.0f),
        "f"(1.4426950408889634f));
  float e0, e1;
  asm("ex2.approx.f32 %0, %1;" : "=f"(e0) : "f"(t0));
  asm("ex2.approx.f32 %0, %1;" : "=f"(e1) : "f"(t1));
  float d0, d1;
  asm("{\n\t.reg .b64 e, o;\n\tmov.b64 e, {%2, %3};\n\tmov.b64 o, {%4, %4};\n\t"
      "add.rn.f32x2 e, e, o;\n\tmov.b64 {%0, %1}, e;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(e0), "f"(e1), "f"(1.0f));
  asm("div.approx.f32 %0, %1, %2;" : "=f"(x0) : "f"(x0), "f"(d0));
  asm("div.approx.f32 %0, %1, %2;" : "=f"(x1) : "f"(x1), "f"(d1));
}

// tanh-form GELU on a pair, as x / (1 + 2^t) with t = -2·log2(e)·c·(x + a·x³)
// folded to t = x·(K1 + K2·x²): packed f32x2 arithmetic, ex2.approx.ftz and
// either rcp.approx.ftz (MUFU) or, with FMA_RCP, 1/(1 + 2^t) from a bit-trick
// seed and three Newton steps on the FMA pipe (the two pipes share the GELU
// load). Relative error ~2e-7 against the float32 tanh form (the reference's
// own tanh is a float32 libm call; tests hold the logits to 1e-5).
template <bool FMA_RCP>
__device__ __forceinline__ void gelu_pair(float& x0, float& x1) {
  constexpr float kL2e = 1.4426950408889634f, kC = 0.7978845608028654f, kA = 0.044715f;
  constexpr float K1 = -2.0f * kL2e * kC, K2 = -2.0f * kL2e * kC * kA;
  float t0, t1;
  asm("{\n\t.reg .b64 x, q, k1, k2;\n\t"
      "mov.b64 x, {%2, %3};\n\t"
      "mov.b64 k1, {%4, %4};\n\t"
      "mov.b64 k2, {%5, %5};\n\t"
      "mul.rn.f32x2 q, x, x;\n\t"
      "fma.rn.f32x2 q, q, k2, k1;\n\t"
      "mul.rn.f32x2 q, q, x;\n\t"
      "mov.b64 {%0, %1}, q;\n\t}"
      : "=f"(t0), "=f"(t1)
      : "f"(x0), "f"(x1), "f"(K1), "f"(K2));
  if (FMA_RCP) {   // keep 1 + 2^t finite for the seed (|result| < 2^-120 there anyway)
    t0 = fminf(t0, 126.f);
    t1 = fminf(t1, 126.f);
  }
  float e0, e1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t1));
  if (!FMA_RCP) {
    float d0, d1;
    asm("{\n\t.reg .b64 e, o;\n\tmov.b64 e, {%2, %3};\n\tmov.b64 o, {%4, %4};\n\t"
        "add.rn.f32x2 e, e, o;\n\tmov.b64 {%0, %1}, e;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(e0), "f"(e1), "f"(1.0f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(d0) : "f"(d0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(d1) : "f"(d1));
    asm("{\n\t.reg .b64 x, r;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 r, {%2, %3};\n\t"
        "mul.rn.f32x2 x, x, r;\n\tmov.b64 {%0, %1}, x;\n\t}"
        : "+f"(x0), "+f"(x1)
        : "f"(d0), "f"(d1));
  } else {
    asm("{\n\t.reg .b64 e, d, r, c, o, one, m1, x;\n\t.reg .b32 d0, d1, r0, r1;\n\t"
        "mov.b64 one, {%4, %4};\n\t"
        "mov.b64 m1, {%5, %5};\n\t"
        "mov.b64 e, {%2, %3};\n\t"
        "add.rn.f32x2 d, e, one;\n\t"
        "sub.rn.f32x2 o, m1, e;\n\t"
        "mov.b64 {d0, d1}, d;\n\t"
        "sub.s32 r0, 0x7EF311C3, d0;\n\t"
        "sub.s32 r1, 0x7EF311C3, d1;\n\t"
        "mov.b64 r, {r0, r1};\n\t"
        "fma.rn.f32x2 c, o, r, one;\n\t"
        "fma.rn.f32x2 r, r, c, r;\n\t"
        "fma.rn.f32x2 c, o, r, one;\n\t"
        "fma.rn.f32x2 r, r, c, r;\n\t"
        "fma.rn.f32x2 c, o, r, one;\n\t"
        "fma.rn.f32x2 r, r, c, r;\n\t"
        "mov.b64 x, {%0, %1};\n\t"
        "mul.rn.f32x2 x, x, r;\n\t"
        "mov.b64 {%0, %1}, x;\n\t}"
        : "+f"(x0), "+f"(x1)
        : "f"(e0), "f"(e1), "f"(1.0f), "f"(-1.0f));
  }
}

__device__ __forceinline__ float gelu_one(float x) {
  float y = 0.f;
  gelu_pair<false>(x, y);
  return x;
}

__host__ __device__ inline size_t tc_fixed_smem() {
  return size_t(8) * kWarpSlot + 1024             // epilogue slots (+ 1 KB alignment)
         + 2 * 128 * sizeof(int64_t)                // per-group row tables
         + (2 * 8 + 4 + 2 * 8) * 8 + 16;            // barriers (+ staging) + TMEM slot
}

// RES: the TMA-store epilogue adds a residual (plain rows only); a separate
// instantiation so kernels without one carry no residual code (register cap 96)
template <int BN, int AM, bool RES = false, bool LNE = false, bool GRP = false>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(TcParams p,
                                                              const __grid_constant__ CUtensorMap tmC) {
  // direct epilogue (thread = row, no shared-memory transpose) for wide tiles
  // (measured: removes the transpose cost but its per-row 16-byte stores halve
  // DRAM write efficiency — 391 vs 283 us on K3 — so the transposed path stays)
  constexpr bool DIRECT = false;
  // (32-column transposes measured slower on the scattered MoE outputs)
  constexpr bool WIDE = false;
  constexpr bool TMA_OK = (BN % 32) == 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the swizzle pattern keys on absolute address bits: align the carve-out to 1 KB
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr uint32_t TCOLS = Acc<BN>::TCOLS;
  constexpr int NACC = Acc<BN>::N;
  constexpr uint32_t kPlaneB = BN * kBK * 2;
  const int S = p.stages;
  const int SG = S / 2;
  const int npb_max = max(p.nplanes[0], p.counts ? p.nplanes[1] : 0);
  // resident weights: B lives in one region loaded at kernel start; stages hold A only
  const uint32_t stage_bytes = 3 * kPlaneA + (p.rb ? 0u : uint32_t(npb_max) * kPlaneB);
  const int NST = p.nst;
  uint8_t* resb = smem + size_t(S) * stage_bytes;                            // resident B
  const uint32_t rb_total = p.rb ? ((p.rb_bytes[0] + p.rb_bytes[1] + 1023u) & ~1023u) : 0u;
  uint8_t* stg = resb + rb_total;                                            // [NST][128][32] f32
  // per-epilogue-warp slot (kWarpSlot bytes, 1 KB aligned): the warp's
  // transpose buffer [32][kXPitch(W)] OR its 4 KB TMA-store box (128-byte
  // swizzle needs the 1 KB alignment); a warp only ever touches its own slot
  uint8_t* slots = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(stg + size_t(NST) * kStgBytes) + 1023) & ~uintptr_t(1023));
  float* xbuf = reinterpret_cast<float*>(slots);
  int64_t* orow_s = reinterpret_cast<int64_t*>(slots + 8 * kWarpSlot);    // [2][128]
  uint8_t* tma_box = slots;
  uint64_t* bars = reinterpret_cast<uint64_t*>(orow_s + 256);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;                 // [NACC] accumulator ready
  uint64_t* tempty = tfull + NACC;                // [NACC] accumulator drained
  const int NSG = NST / 2;                        // staging slots per producer group
  uint64_t* sfull = tempty + NACC;                // [2][NSG] staging slot loaded
  uint64_t* sempty = sfull + NST;                 // [2][NSG] staging slot consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + NST + 1);   // (+ resident-B barrier)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ GroupTab gtab;
  if (warp == kMmaWarp) tmem_alloc<TCOLS>(tmem_slot);
  if (tid == 0) build_groups(p, gtab);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 4);     // the four warps of the owning producer group
      mbar_init(&empty[s], 1);    // one MMA commit
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(&tfull[b], 1);    // one MMA commit
      mbar_init(&tempty[b], 128); // every thread of the epilogue group
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&sfull[i], 32);   // one cp.async completion arrival per loader lane
      mbar_init(&sempty[i], 4);   // the four warps of the consuming producer group
    }
    fence_barrier_init();
    if (p.rb) {   // every weight tile of both experts, once (TMA bulk copies)
      uint64_t* rbar = sempty + NST;
      mbar_init(rbar, 1);
      fence_barrier_init();
      mbar_expect_tx(rbar, p.rb_bytes[0] + p.rb_bytes[1]);
      bulk_g2s(resb, p.Bp[0], p.rb_bytes[0], rbar);
      if (p.rb_bytes[1]) bulk_g2s(resb + p.rb_bytes[0], p.Bp[1], p.rb_bytes[1], rbar);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (p.rb) mbar_wait(sempty + NST, 0);
  const uint32_t tmem = *tmem_slot;
  const GroupTab& gt = gtab;
  const int total = int(num_m_tiles(gtab) * p.ntiles);

  if (warp >= 8 && warp < 16) {
    // ================= producers =================
    const int g = (warp - 8) >> 2;
    const int ptid = tid - 256 - 128 * g;
    const int rsub = ptid >> 3;          // row within each 16-row slab
    const int k4 = (ptid & 7) * 4;       // k offset within the 32-wide stage
    const int64_t pcw = p.patch * p.pC;
    int sg = 0;
    uint32_t phase = 0;
    int j = 0;
    int sidx = 0;   // stages this group has taken from its staging ring
    // MoE gather indices of the group's NEXT tile are loaded while the current
    // tile is processed (their HBM latency would otherwise precede every tile)
    constexpr bool PF = AM == A_GATHER;
    int jj_unused;
    TileInfo ti_n;
    // K stages: with one stage per tile the two groups alternate tiles; with
    // several, consecutive stages of the CTA's whole sequence alternate between
    // the groups, so both keep loads in flight within a deep-K tile
    const bool kq = p.kchunks > p.kq_min;
    const int gsel = kq ? -1 : g;
    int q = 0;
    int t_n = next_group_tile<GRP>(p, gt, total, gsel, blockIdx.x, j, jj_unused, ti_n);
    int idx_n[8];
    auto load_idx = [&](const TileInfo& tq, int (&ix)[8]) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = tq.r0 + rsub + 16 * i;
        ix[i] = (PF && NST == 0 && row < tq.r1) ? __ldg(p.a_rows + row) : 0;
      }
    };
    if (t_n < total) load_idx(ti_n, idx_n);
    while (t_n < total) {
      const TileInfo ti = ti_n;
      int idx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) idx[i] = idx_n[i];
      t_n = next_group_tile<GRP>(p, gt, total, gsel, t_n + gridDim.x, j, jj_unused, ti_n);
      if (t_n < total) load_idx(ti_n, idx_n);
      const int npb = p.nplanes[ti.group];
      const uint16_t* Bg = p.Bp[ti.group] + size_t(ti.n_tile) * p.kchunks * npb * (BN * kBK);
      const uint32_t bbytes = uint32_t(npb) * kPlaneB;
      const float* rowp[8];
      // patchify: (image, patch row, patch col) of this thread's first row by one
      // division set; the other seven rows (16 apart) step it with carries
      int pb = 0, py = 0, px = 0;
      if (AM == A_PATCH && NST == 0) {
        const int tpi = int(p.pside * p.pside), ps = int(p.pside);
        const int r32 = int(ti.r0) + rsub;
        pb = r32 / tpi;
        const int tt = r32 - pb * tpi;
        py = tt / ps;
        px = tt - py * ps;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = ti.r0 + rsub + 16 * i;
        rowp[i] = nullptr;
        if (row < ti.r1) {
          if (AM == A_PLAIN || NST > 0) {
            rowp[i] = p.A + row * p.lda;   // (staged: only the non-null flag is used)
          } else if (AM == A_GATHER) {
            rowp[i] = p.A + int64_t(idx[i]) * p.lda;
          } else {
            rowp[i] = p.A + ((int64_t(pb) * p.pH + int64_t(py) * p.patch) * p.pW +
                             int64_t(px) * p.patch) * p.pC;
          }
        }
        if (AM == A_PATCH && NST == 0) {   // next row: 16 tokens on
          const int ps = int(p.pside);
          px += 16;
          while (px >= ps) {
            px -= ps;
            if (++py == ps) {
              py = 0;
              ++pb;
            }
          }
        }
      }
      for (int kc = 0; kc < p.kchunks; ++kc) {
        if (kq && ((q++ & 1) != g)) continue;
        const int s = g + 2 * sg;
        const int64_t k = int64_t(kc) * kBK + k4;
        float4 v[8];
        if (kStaging && NST > 0) {   // A rows from the loader's staging slot
          const int ss = g * NSG + (sidx % NSG);
          mbar_wait(&sfull[ss], uint32_t(sidx / NSG) & 1u);
          ++sidx;
          const float* sp = reinterpret_cast<const float*>(stg + size_t(ss) * kStgBytes);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rowp[i] != nullptr && k < p.K)
              v[i] = *reinterpret_cast<const float4*>(sp + (rsub + 16 * i) * kBK + k4);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sempty[ss]);
        } else {
          // patch offset of this thread's k: one division per stage, not per row
          int64_t koff = k;
          if (AM == A_PATCH) {
            const int kq = int(k) / int(pcw);
            koff = int64_t(kq) * (p.pW * p.pC) + (int(k) - kq * int(pcw));
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {   // issue the global loads before waiting for the slot
            v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (rowp[i] != nullptr && k < p.K) {
              const float* src = rowp[i] + koff;
              if (!(p.dbg & 1)) v[i] = __ldg(reinterpret_cast<const float4*>(src));
            }
          }
        }
        mbar_wait(&empty[s], phase ^ 1u);
        uint8_t* st = smem + size_t(s) * stage_bytes;
        if (ptid == 0 && !p.rb) {
          mbar_add_tx(&full[s], bbytes);
          bulk_g2s(st + 3 * kPlaneA, Bg + size_t(kc) * npb * (BN * kBK), bbytes, &full[s]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (p.dbg & 32) break;   // debug: no conversion / stage stores
          if (AM == A_PATCH && rowp[i] != nullptr && k < p.K) {
            v[i].x -= p.sub; v[i].y -= p.sub; v[i].z -= p.sub; v[i].w -= p.sub;
          }
          const Split3u a = split3x2_trunc(v[i].x, v[i].y);   // (no F2FP, see split3x2_trunc)
          const Split3u b = split3x2_trunc(v[i].z, v[i].w);
          const uint32_t off = plane_offset(rsub + 16 * i, k4);
          *reinterpret_cast<uint2*>(st + off) = make_uint2(a.h, b.h);
          *reinterpret_cast<uint2*>(st + kPlaneA + off) = make_uint2(a.m, b.m);
          *reinterpret_cast<uint2*>(st + 2 * kPlaneA + off) = make_uint2(a.l, b.l);
        }
        if (!(p.dbg & 8)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++sg == SG) {
          sg = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == kLoadWarp) {
    // ================= A loader (staged mode) =================
    if (kStaging && NST > 0 && AM != A_PATCH) {
      // lane = (16-byte chunk c, row sub-slab rs): one warp instruction copies
      // four full 128-byte row segments (coalesced cp.async); completion is
      // tracked per lane by cp.async.mbarrier.arrive.noinc (32 arrivals). The
      // row indices (MoE gather) of the next tile are loaded one tile ahead.
      const int c = lane & 7, rs = lane >> 3;
      auto next_tile = [&](int t) {
        for (; t < total; t += gridDim.x) {
          const TileInfo ti = tile_info<GRP>(p, gt, t);
          if (ti.r0 < ti.r1) break;
        }
        return t;
      };
      auto rows_of = [&](int t, int (&src)[32], int& nrows) {
        nrows = 0;
        if (t >= total) return;
        const TileInfo ti = tile_info<GRP>(p, gt, t);
        nrows = int(ti.r1 - ti.r0);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int r = rs + 4 * i;
          const int64_t row = ti.r0 + r;
          src[i] = r < nrows ? (AM == A_GATHER ? __ldg(p.a_rows + row) : int(row)) : -1;
        }
      };
      int t = next_tile(blockIdx.x);
      int cur[32], nxt[32];
      int ncur = 0, nnxt = 0;
      rows_of(t, cur, ncur);
      int fills[2] = {0, 0};   // stages loaded into each group's ring
      int jt = 0;              // non-empty tiles so far (group = jt & 1)
      while (t < total) {
        const int tn = next_tile(t + gridDim.x);
        rows_of(tn, nxt, nnxt);
        const int gg = jt++ & 1;
        for (int kc = 0; kc < p.kchunks; ++kc) {
          const int fi = fills[gg]++;
          const int ss = gg * NSG + (fi % NSG);
          mbar_wait(&sempty[ss], (uint32_t(fi / NSG) & 1u) ^ 1u);
          const bool c_ok = int64_t(kc) * kBK + c * 4 < p.K;
          const uint32_t dst = smem_u32(stg + size_t(ss) * kStgBytes) + uint32_t(rs * kBK * 4 + c * 16);
          const float* base = p.A + int64_t(kc) * kBK + c * 4;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (cur[i] >= 0 && c_ok) {
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(i * 4 * kBK * 4)),
                           "l"(base + int64_t(cur[i]) * p.lda)
                           : "memory");
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sfull[ss]))
                       : "memory");
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) cur[i] = nxt[i];
        ncur = nnxt;
        t = tn;
      }
      (void)ncur;
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer (whole warp; one elected lane issues) =================
    constexpr uint32_t idesc = idesc_bf16_m128(BN);
    const uint32_t smem_base = smem_u32(smem);
    int sg[2] = {0, 0};
    uint32_t phase[2] = {0, 0};
    uint32_t acc_phase[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) acc_phase[a] = 0u;
    const bool kq_mma = p.kchunks > p.kq_min;
    int qm = 0;
    int j = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const TileInfo ti = tile_info<GRP>(p, gt, t);
      if (ti.r0 >= ti.r1) continue;
      const int jj = j++;
      const int acc = jj & (NACC - 1);      // TMEM accumulator
      const int npb = p.nplanes[ti.group];
      mbar_wait(&tempty[acc], acc_phase[acc] ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem + uint32_t(acc * BN);
      for (int kc = 0; kc < p.kchunks; ++kc) {
        // producer group of this stage (alternating tiles, or alternating
        // stages when the tile has several)
        const int g = kq_mma ? (qm++ & 1) : (jj & 1);
        const int s = g + 2 * sg[g];
        mbar_wait(&full[s], phase[g]);
        tc_fence_after();
        const uint32_t sa = smem_base + uint32_t(s) * stage_bytes;
        const uint32_t sb = p.rb ? smem_u32(resb) + (ti.group ? p.rb_bytes[0] : 0u) +
                                       uint32_t((ti.n_tile * p.kchunks + kc) * npb) * kPlaneB
                                 : sa + 3 * kPlaneA;
#pragma unroll
        for (int ks = 0; ks < kBK / 16; ++ks) {
          const uint64_t ad = smem_desc(sa + ks * 256);
          const uint64_t bd = smem_desc(sb + ks * 256);
          const uint32_t acc = (kc | ks) != 0;
          if (p.dbg & 4) continue;
          if (npb == 1)
            mma_chain3_ss_w(d_tmem, ad, bd, kPlaneA >> 4, idesc, acc);
          else
            mma_chain6_ss_w(d_tmem, ad, bd, kPlaneA >> 4, kPlaneB >> 4, idesc, acc);
        }
        commit_w(&empty[s]);
        if (++sg[g] == SG) {
          sg[g] = 0;
          phase[g] ^= 1u;
        }
      }
      commit_w(&tfull[acc]);
      acc_phase[acc] ^= 1u;
    }
  } else {
    // ===== epilogue group g (warps 4g..4g+3): warp reads TMEM lanes 32*(warp%4) =====
    const int g = warp >> 2, quad = warp & 3;
    float* xb = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xbuf) + warp * kWarpSlot);
    int64_t* orow_t = orow_s + g * 128;
    uint32_t acc_phase[NACC / 2];   // this group owns accumulators g, g + 2, ...
#pragma unroll
    for (int a = 0; a < NACC / 2; ++a) acc_phase[a] = 0u;
    const bool vec4 = (p.N & 3) == 0;
    int j = 0;
    const int rl = quad * 32 + lane;             // row within the tile
    // Row metadata is software-pipelined over the group's tiles: the scatter
    // row of tile B (next) and its gate, and the scatter row of tile C (after
    // next), are in flight while tile A is drained (dependent HBM loads).
    auto scatter_row = [&](const TileInfo& tq) -> int64_t {
      const int64_t r = tq.r0 + rl;
      if (r >= tq.r1) return -1;
      // grouped problems: c_rows holds problem-local rows; the problem's block of C
      const int64_t off = GRP ? int64_t(tq.group >> 1) * p.prob_rows : 0;
      return p.c_rows ? int64_t(__ldg(p.c_rows + r)) + off : r;
    };
    TileInfo tiA, tiB, tiC;
    int jjA = 0, jjB = 0, jjC = 0;
    int tA = next_group_tile<GRP>(p, gt, total, g, blockIdx.x, j, jjA, tiA);
    int tB = tA < total ? next_group_tile<GRP>(p, gt, total, g, tA + gridDim.x, j, jjB, tiB) : total;
    int64_t crA = tA < total ? scatter_row(tiA) : -1;
    int64_t crB = tB < total ? scatter_row(tiB) : -1;
    float gA = (p.gate && crA >= 0 && p.img_tokens == 0) ? __ldg(p.gate + crA) : 1.f;
    while (tA < total) {
      const int tC = tB < total ? next_group_tile<GRP>(p, gt, total, g, tB + gridDim.x, j, jjC, tiC)
                                : total;
      const int64_t crC = tC < total ? scatter_row(tiC) : -1;
      const float gB = (p.gate && crB >= 0 && p.img_tokens == 0) ? __ldg(p.gate + crB) : 1.f;
      const TileInfo ti = tiA;
      const int jj = jjA;
      const int acc = jj & (NACC - 1), ah = acc >> 1;
      const int64_t r = ti.r0 + rl;
      const bool r_ok = r < ti.r1;
      int64_t orow = -1, pos_idx = 0;
      float gt = 1.f;
      if (r_ok) {
        orow = crA;
        if (p.img_tokens > 0 && (p.extra != 0 || p.pos != nullptr)) {
          const int b = int(r) / int(p.img_tokens), tt = int(r) - b * int(p.img_tokens);
          orow = b * (p.img_tokens + p.extra) + p.extra + tt;
          pos_idx = p.extra + tt;
          if (p.gate) gt = __ldg(p.gate + orow);
        } else if (p.gate) {
          gt = gA;
        }
      }
      // the row table of the previous tile of this group has been consumed by
      // every warp of the group once they all reach this barrier
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
      orow_t[rl] = r_ok ? (p.pos ? (orow | (pos_idx << 40)) : orow) : int64_t(-1);
      // the residual row (one contiguous N-float run) is pulled into L2 by the
      // TMA engine while the accumulator is still being computed: the
      // epilogue's per-block residual loads then hit L2 instead of HBM
      if (p.residual && r_ok && (p.N & 3) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.residual + orow * p.N),
                     "r"(uint32_t(p.N) * 4u)
                     : "memory");
      mbar_wait(&tfull[acc], acc_phase[ah]);
      acc_phase[ah] ^= 1u;
      tc_fence_after();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
      const uint32_t t_base = tmem + (uint32_t(quad * 32) << 16) + uint32_t(acc * BN);
      const int64_t n_base = int64_t(ti.n_tile) * BN;
      // a TMA box writes whole 32-row slabs: only tiles that end at a 128-row
      // boundary or at M (not the partial tile before an expert boundary)
      const bool tma_tile = TMA_OK && p.tma_c && !(p.dbg & 16) &&
                            (ti.r1 - ti.r0 == kBM || ti.r1 == p.M);
      if (TMA_OK && p.tma_c && !tma_tile) {   // the slot may still feed a TMA store
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      }
      if (p.dbg & 16) {
        // debug: epilogue reduced to the accumulator handshake
      } else if (tma_tile) {
        // TMA-store epilogue: 32 accumulator columns per TMEM load, written by
        // the thread (= row) into a 32 x 32 fp32 box in shared memory with the
        // 128-byte swizzle (16-byte chunk c of row r at c ^ (r & 7): the eight
        // lanes of a bank group hit distinct banks), then one elected lane
        // stores the box with cp.async.bulk.tensor (full-line writes, rows past
        // M clipped by the tensor map).
        uint8_t* box = tma_box + warp * kWarpSlot;
        const int row0 = int(ti.r0) + quad * 32;
        // plain rows: the residual row of this thread is row r itself (L2-prefetched)
        const float* rres = (RES && r_ok) ? p.residual + r * p.N + n_base : nullptr;
        // LNE: LayerNorm of the thread's output row (the whole row is this tile,
        // N = BN) with layernorm_row_kernel's arithmetic: sums over float4
        // groups in column order, two passes over TMEM for mean and variance
        float ln_mean = 0.f, ln_inv = 0.f;
        if (LNE) {
          float sum = 0.f;
#pragma unroll 1
          for (int cb = 0; cb < BN; cb += 32) {
            uint32_t raw[32];
            tmem_ld32_nowait(t_base + uint32_t(cb), raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i)
              sum += (__uint_as_float(raw[4 * i]) + __uint_as_float(raw[4 * i + 1])) +
                     (__uint_as_float(raw[4 * i + 2]) + __uint_as_float(raw[4 * i + 3]));
          }
          ln_mean = sum / float(BN);
          float q = 0.f;
#pragma unroll 1
          for (int cb = 0; cb < BN; cb += 32) {
            uint32_t raw[32];
            tmem_ld32_nowait(t_base + uint32_t(cb), raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float x0 = __uint_as_float(raw[4 * i]) - ln_mean;
              const float x1 = __uint_as_float(raw[4 * i + 1]) - ln_mean;
              const float x2 = __uint_as_float(raw[4 * i + 2]) - ln_mean;
              const float x3 = __uint_as_float(raw[4 * i + 3]) - ln_mean;
              q += (x0 * x0 + x1 * x1) + (x2 * x2 + x3 * x3);
            }
          }
          ln_inv = 1.0f / sqrtf(q / float(BN) + p.ln_eps);
        }
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          if (lane == 0) bulk_wait_read0();   // the box's previous store has read it
          __syncwarp();
          // residual: the row's 32-column segment is copied straight into this
          // thread's swizzled box row (cp.async, no registers), then added in place
          const bool has_res = rres != nullptr;   // (tma_c with a residual implies N % 32 == 0)
          if (has_res) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                               smem_u32(box + lane * 128 + ((c ^ (lane & 7)) * 16))),
                           "l"(rres + cb + 4 * c)
                           : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
          }
          uint32_t raw[32];
          tmem_ld32_nowait(t_base + uint32_t(cb), raw);
          tmem_ld_wait();
          if (cb + 32 >= BN) {   // accumulator fully in registers: hand it back
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          if (has_res) asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float4 o = make_float4(__uint_as_float(raw[4 * c]), __uint_as_float(raw[4 * c + 1]),
                                   __uint_as_float(raw[4 * c + 2]), __uint_as_float(raw[4 * c + 3]));
            if (p.act == 1) {
              gelu_pair<false>(o.x, o.y);
              gelu_pair<false>(o.z, o.w);
            }
            if (p.gate) { o.x *= gt; o.y *= gt; o.z *= gt; o.w *= gt; }
            if (LNE) {
              const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.ln_g + cb + 4 * c));
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.ln_b + cb + 4 * c));
              o.x -= ln_mean; o.y -= ln_mean; o.z -= ln_mean; o.w -= ln_mean;
              o = make_float4(o.x * ln_inv * g4.x + b4.x, o.y * ln_inv * g4.y + b4.y,
                              o.z * ln_inv * g4.z + b4.z, o.w * ln_inv * g4.w + b4.w);
            }
            float4* slot = reinterpret_cast<float4*>(box + lane * 128 + ((c ^ (lane & 7)) * 16));
            if (has_res) {
              const float4 q = *slot;
              o = make_float4(q.x + o.x, q.y + o.y, q.z + o.z, q.w + o.w);
            }
            *slot = o;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(p.dbg & 2)) {
            tma_store_2d(&tmC, box, int(n_base) + cb, row0);
            bulk_commit();
          }
        }
      } else if (DIRECT && false) {
        // thread = output row: 16 columns per TMEM load (issued one chunk
        // ahead), then four 16-byte stores of the row's contiguous 64-byte
        // segment (no shared-memory transpose)
        const bool full4 = vec4 && n_base + BN <= p.N;
        float* crow = (r_ok && orow >= 0) ? p.C + orow * p.N + n_base : nullptr;
        const float* rrow = (crow && p.residual) ? p.residual + orow * p.N + n_base : nullptr;
        const float* prow = (crow && p.pos) ? p.pos + pos_idx * p.N + n_base : nullptr;
        float v[16];
        tmem_ld16(t_base, v);
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 16) {
          float o[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) o[q] = v[q];
          if (cb + 16 < BN) tmem_ld16(t_base + uint32_t(cb + 16), v);
          if (crow == nullptr) continue;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float e = o[q];
            if (p.act == 1) e = gelu_one(e);
            if (p.gate) e = e * gt;
            o[q] = e;
          }
          if (full4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4 w = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
              if (prow) {
                const float4 pp = __ldg(reinterpret_cast<const float4*>(prow + cb) + q);
                w.x += pp.x; w.y += pp.y; w.z += pp.z; w.w += pp.w;
              }
              if (rrow) {
                const float4 rq = __ldg(reinterpret_cast<const float4*>(rrow + cb) + q);
                w = make_float4(rq.x + w.x, rq.y + w.y, rq.z + w.z, rq.w + w.w);
              }
              if (!(p.dbg & 2)) *reinterpret_cast<float4*>(crow + cb + 4 * q) = w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int64_t n = n_base + cb + q;
              if (n >= p.N) break;
              float e = o[q];
              if (prow) e = e + __ldg(prow + cb + q);
              if (rrow) e = __ldg(rrow + cb + q) + e;
              crow[cb + q] = e;
            }
          }
        }
      } else if (WIDE) {
        // 32 columns per TMEM load; the warp's 32 x 32 block is transposed in
        // shared memory and written as four full 128-byte row segments per
        // store instruction (8 lanes per row)
        const int rq = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 32) {
          uint32_t raw[32];
          tmem_ld32_nowait(t_base + uint32_t(cb), raw);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            float4 o = make_float4(__uint_as_float(raw[q]), __uint_as_float(raw[q + 1]),
                                   __uint_as_float(raw[q + 2]), __uint_as_float(raw[q + 3]));
            if (p.act == 1) {
              gelu_pair<false>(o.x, o.y);
              gelu_pair<false>(o.z, o.w);
            }
            if (p.gate) { o.x *= gt; o.y *= gt; o.z *= gt; o.w *= gt; }
            *reinterpret_cast<float4*>(xb + lane * kXPitchW + q) = o;
          }
          __syncwarp();
          const int64_t n = n_base + cb + c4;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int ri = it * 4 + rq;
            const int64_t meta = orow_t[quad * 32 + ri];
            if (meta < 0) continue;
            const int64_t orow_i = p.pos ? (meta & ((int64_t(1) << 40) - 1)) : meta;
            const int64_t pos_i = p.pos ? (meta >> 40) : 0;
            float4 o = *reinterpret_cast<const float4*>(xb + ri * kXPitchW + c4);
            if (vec4 && n + 3 < p.N) {
              if (p.pos) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(p.pos + pos_i * p.N + n));
                o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
              }
              if (p.residual) {
                const float4 q =
                    __ldg(reinterpret_cast<const float4*>(p.residual + orow_i * p.N + n));
                o = make_float4(q.x + o.x, q.y + o.y, q.z + o.z, q.w + o.w);
              }
              if (!(p.dbg & 2)) *reinterpret_cast<float4*>(p.C + orow_i * p.N + n) = o;
            } else {
              const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (n + q >= p.N) break;
                float e = ov[q];
                if (p.pos) e = e + __ldg(p.pos + pos_i * p.N + n + q);
                if (p.residual) e = __ldg(p.residual + orow_i * p.N + n + q) + e;
                p.C[orow_i * p.N + n + q] = e;
              }
            }
          }
          __syncwarp();
        }
      } else {
      // residual rows (scattered MoE rows) staged one 16-column block ahead in
      // the warp's slot with cp.async: each lane copies exactly the (row, 4
      // columns) pieces it adds below, so no cross-lane synchronisation
      float* rs = xb + 32 * kXPitch;   // [2][32][16]
      const int c4r = (lane & 3) * 4;
      const bool stage_res = p.residual != nullptr && vec4;
      int64_t orow_r[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int64_t meta = orow_t[quad * 32 + it * 8 + (lane >> 2)];
        orow_r[it] = meta < 0 ? int64_t(-1) : (p.pos ? (meta & ((int64_t(1) << 40) - 1)) : meta);
      }
      auto issue_res = [&](int cb, int buf) {
        const int64_t n = n_base + cb + c4r;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          if (orow_r[it] >= 0 && n + 3 < p.N)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                             smem_u32(rs + (buf * 32 + it * 8 + (lane >> 2)) * 16 + c4r)),
                         "l"(p.residual + orow_r[it] * p.N + n)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      if (stage_res) issue_res(0, 0);
#pragma unroll 1
      for (int cb = 0; cb < BN; cb += 16) {
        const int rbuf = (cb >> 4) & 1;
        if (stage_res) {
          if (cb + 16 < BN) {
            issue_res(cb + 16, rbuf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
        }
        float v[16];
        tmem_ld16(t_base + uint32_t(cb), v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float o = v[q];
          if (p.act == 1) o = gelu_one(o);
          if (p.gate) o = o * gt;
          v[q] = o;
        }
#pragma unroll
        for (int q = 0; q < 16; q += 4)
          *reinterpret_cast<float4*>(xb + lane * kXPitch + q) =
              make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        __syncwarp();
        // 8 rows x 4 float4 per instruction: each row segment is 64 contiguous bytes
        const int c4 = (lane & 3) * 4;
        const int64_t n = n_base + cb + c4;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int ri = it * 8 + (lane >> 2);
          const int64_t meta = orow_t[quad * 32 + ri];
          if (meta < 0) continue;
          const int64_t orow_i = p.pos ? (meta & ((int64_t(1) << 40) - 1)) : meta;
          const int64_t pos_i = p.pos ? (meta >> 40) : 0;
          float4 o = *reinterpret_cast<const float4*>(xb + ri * kXPitch + c4);
          if (vec4 && n + 3 < p.N) {
            if (p.pos) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(p.pos + pos_i * p.N + n));
              o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
            }
            if (p.residual) {
              const float4 q = *reinterpret_cast<const float4*>(rs + (rbuf * 32 + ri) * 16 + c4);
              o = make_float4(q.x + o.x, q.y + o.y, q.z + o.z, q.w + o.w);
            }
            if (!(p.dbg & 2)) *reinterpret_cast<float4*>(p.C + orow_i * p.N + n) = o;
          } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (n + q >= p.N) break;
              float e = ov[q];
              if (p.pos) e = e + __ldg(p.pos + pos_i * p.N + n + q);
              if (p.residual) e = __ldg(p.residual + orow_i * p.N + n + q) + e;
              p.C[orow_i * p.N + n + q] = e;
            }
          }
        }
        __syncwarp();
      }
      }
      if (!tma_tile) {
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
      tA = tB;
      tiA = tiB;
      jjA = jjB;
      crA = crB;
      gA = gB;
      tB = tC;
      tiB = tiC;
      jjB = jjC;
      crB = crC;
    }
  }
  if (warp < 8 && lane == 0) bulk_wait0();   // TMA stores of this warp retired
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<TCOLS>(tmem);
}

}  // namespace tc
}  // namespace sa
