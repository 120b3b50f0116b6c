// K5 fused: the whole (MoE) MLP  y = [res +] gate · fc2(GELU(fc1(x)))  in one
// persistent tcgen05 kernel; the hidden activations never leave the SM.
//
// Reference: Mlp.forward (model.py:204-208) inside MoeModule.forward
// (model.py:250-274), experts (Mlp(Linear,Linear), Mlp(Shift,Shift))
// (model.py:514-521). Numerics as in tcgemm.cu: x and GELU(h) are split into
// hi/mid/lo bf16 planes (exact), shift weights are exact bf16, dense weights
// three planes; fp32 accumulation in TMEM.
//
// Per 128-token tile of one expert the hidden dimension is walked in chunks of
// HC = 32 columns, counted globally by q:
//   fc1(q) → acc1[q % NB] (TMEM) → GELU group (q % 2): tcgen05.ld, GELU, split,
//   tcgen05.st → A2[q % NB] (TMEM) → fc2(q) accumulates into acc2[tile % 2].
// Both A operands (the x planes A1 and the GELU planes A2) live in TMEM and
// feed tcgen05.mma in its A-from-TMEM form, so shared-memory bandwidth is
// spent only on the weight tiles (B operands): with A in shared memory every
// narrow (N = 32) MMA re-reads a 4 KB A tile and the issue rate collapses
// under the GELU / producer traffic.
// Roles (15 warps, one CTA per SM):
//   warps  0-3 / 4-7  GELU groups 0 / 1 (alternate chunks; warp quad = TMEM
//                     lane block); group (tile % 2) also runs the final epilogue
//                     of the tile: tcgen05.ld acc2, x gate, + residual, scatter
//   warps  8-11       producers: gather x rows (MoE permutation), split,
//                     tcgen05.st → A1 (thread = row = TMEM lane)
//   warp  12          MMA issuer (one thread): fc1 runs LOOK chunks ahead of fc2
//   warps 13 / 14     weight streamers: W1 / W2 chunk rings (bulk async copy)
// Every ring carries full/empty mbarriers; parities derive from the running
// counters, so tiles of the two experts interleave freely.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace tcm {

using namespace tc;

constexpr int HC = 32;                 // hidden chunk (fc1 N, fc2 K)
constexpr int kThreads = 480;
constexpr int kMma = 12, kW1 = 13, kW2 = 14;
constexpr int kMaxTiles = 1024;               // per-CTA tile table of the MMA issuer
constexpr uint32_t kPlaneCols = 16;           // TMEM columns of one 32-k bf16 plane

struct MlpParams {
  const float* x;
  const int32_t* perm;       // nullptr: identity rows
  const int32_t* counts;     // nullptr: one group
  const float* gate;
  const float* residual;
  float* y;
  const uint16_t* w1[2];     // packed (bn = 32) planes per expert
  const uint16_t* w2[2];     // packed (bn = d) planes per expert
  int np[2];                 // planes per expert (3 dense, 1 shift)
  int64_t M;
  int hidden;
  unsigned long long* prof;  // optional: cycles per wait site (debug builds of the timeline)
  int dbg;                   // debug experiments (0 in production)
};

// wait-site ids for the optional cycle profile
enum { P_A1E = 0, P_W1E, P_W2E, P_A1F, P_W1F, P_HE1, P_OE, P_W2F, P_HE2, P_HF, P_A2E, P_OF,
       P_T_PROD, P_T_MMA, P_T_GELU, P_ISS1, P_ISS2, P_NSITE };

template <int D>
struct Layout {
  static constexpr int KC1 = D / 32;                         // fc1 K stages
  static constexpr int NA = D == 32 ? 2 : 1;                 // A1 buffers (TMEM)
  static constexpr int NB = D == 32 ? 4 : 3;                 // acc1 / A2 buffers (TMEM)
  static constexpr int LOOK = NB - 1;                        // fc1 lookahead over fc2
  static constexpr int NW = D == 32 ? 4 : 2;                 // W1 / W2 ring slots
  static constexpr uint32_t W1C = KC1 * 3 * (HC * 32 * 2);   // max W1 chunk bytes
  static constexpr uint32_t W2C = 3 * (D * 32 * 2);          // max W2 chunk bytes
  static constexpr uint32_t XB = 8 * 32 * kXPitch * 4;
  static constexpr uint32_t OFF_W1 = 0;
  static constexpr uint32_t OFF_W2 = OFF_W1 + NW * W1C;
  static constexpr uint32_t OFF_XB = OFF_W2 + NW * W2C;
  static constexpr uint32_t OFF_ROW = OFF_XB + XB;            // [2][128] int64
  static constexpr uint32_t OFF_BAR = OFF_ROW + 2 * 128 * 8;
  // barriers: a1 full/empty[NA], w1 full/empty[NW], w2 full/empty[NW],
  //           h_full/h_empty/a2_empty[NB], o_full/o_empty[2]
  static constexpr uint32_t NBAR = 2 * NA + 4 * NW + 3 * NB + 4;
  static constexpr uint32_t TOTAL = OFF_BAR + NBAR * 8 + 16 + 1024;  // + alignment slack
  // TMEM columns: acc1[NB] | acc2[2] | A1[NA] (KC1 x 3 planes) | A2[NB] (3 planes)
  static constexpr uint32_t T_ACC1 = 0;
  static constexpr uint32_t T_ACC2 = NB * HC;
  static constexpr uint32_t T_A1 = T_ACC2 + 2 * D;
  static constexpr uint32_t A1COLS = KC1 * 3 * kPlaneCols;
  static constexpr uint32_t T_A2 = T_A1 + NA * A1COLS;
  static constexpr uint32_t A2COLS = 3 * kPlaneCols;
  static constexpr uint32_t TCOLS = 512;
  static_assert(T_A2 + NB * A2COLS <= TCOLS, "TMEM budget");
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

__device__ __forceinline__ uint32_t par(int64_t use) { return uint32_t(use) & 1u; }

template <int D, bool DBG>
__global__ void __launch_bounds__(kThreads, 1) mlp_kernel(MlpParams p) {
  using L = Layout<D>;
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
  uint64_t* h_empty = h_full + L::NB;       // GELU(q) read acc1 and wrote A2 (128 threads)
  uint64_t* a2_empty = h_empty + L::NB;     // fc2(q) done reading A2
  uint64_t* o_full = a2_empty + L::NB;      // [2] acc2 ready
  uint64_t* o_empty = o_full + 2;           // [2] acc2 drained (128 threads)
  int64_t* rowtab = reinterpret_cast<int64_t*>(smem + L::OFF_ROW);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + L::NBAR * 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ unsigned long long sprof[P_NSITE];
  __shared__ uint8_t tile_e[kMaxTiles];
  if (tid < P_NSITE) sprof[tid] = 0;
  const long long t_start = clock64();
#define PWAIT(site, b, par_)                                        \
  do {                                                              \
    if (!DBG) {                                                     \
      mbar_wait(b, par_);                                           \
    } else if (p.dbg & 8) {                                         \
    } else if (p.prof) {                                            \
      const long long t0_ = clock64();                              \
      mbar_wait(b, par_);                                           \
      if (lane == 0) atomicAdd(&sprof[site], (unsigned long long)(clock64() - t0_)); \
    } else {                                                        \
      mbar_wait(b, par_);                                           \
    }                                                               \
  } while (0)
  // debug bit 64 (with 16): plain arrivals instead of tcgen05.commit
  auto commit = [&](uint64_t* b) {   // whole MMA warp calls this
    if (DBG && (p.dbg & 80) == 80) {
      if (lane == 0) mbar_arrive(b);
    } else {
      commit_w(b);
    }
  };
  if (warp == kMma) tmem_alloc<L::TCOLS>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < L::NA; ++i) {
      mbar_init(&a1_full[i], 4);
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
      mbar_init(&h_empty[i], 128);
      mbar_init(&a2_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t c0 = p.counts ? int64_t(p.counts[0]) : 0;
  const int64_t ntile = mlp_tiles(p, c0);
  const int nchunk = p.hidden / HC;

  if (DBG && (p.dbg & 8) && warp != kMma) {
    // debug: only the MMA issuer runs (no handshakes)
  } else if (warp >= 8 && warp < 12) {
    // ---------------- producers: x rows → A1 planes (TMEM) ----------------
    const int ptid = tid - 256;                  // = tile row = TMEM lane
    const uint32_t lane_base = uint32_t((warp - 8) * 32) << 16;
    int64_t j = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
      const int buf = int(j % L::NA);
      const uint32_t ph = par(j / L::NA);
      ++j;
      const int64_t row = r0 + ptid;
      float4 v[D / 4];
      if (!(DBG && (p.dbg & 2)) && row < r1) {
        const float* src = p.x + (p.perm ? int64_t(__ldg(p.perm + row)) : row) * D;
#pragma unroll
        for (int i = 0; i < D / 4; ++i) v[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
      } else {
#pragma unroll
        for (int i = 0; i < D / 4; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      PWAIT(P_A1E, &a1_empty[buf], ph ^ 1u);
      tc_fence_after();
      const uint32_t a1 = tmem + lane_base + L::T_A1 + uint32_t(buf) * L::A1COLS;
#pragma unroll
      for (int kc = 0; kc < L::KC1; ++kc) {
        if (DBG && (p.dbg & 2)) break;   // debug: no A1 stores
        uint32_t hp[16], mp[16], lp[16];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float4 q = v[kc * 8 + t];
          const Split3 a = split3x2(q.x, q.y);
          const Split3 b = split3x2(q.z, q.w);
          hp[2 * t] = bf2_bits(a.h);
          hp[2 * t + 1] = bf2_bits(b.h);
          mp[2 * t] = bf2_bits(a.m);
          mp[2 * t + 1] = bf2_bits(b.m);
          lp[2 * t] = bf2_bits(a.l);
          lp[2 * t + 1] = bf2_bits(b.l);
        }
        tmem_st16(a1 + kc * 3 * kPlaneCols, hp);
        tmem_st16(a1 + kc * 3 * kPlaneCols + kPlaneCols, mp);
        tmem_st16(a1 + kc * 3 * kPlaneCols + 2 * kPlaneCols, lp);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a1_full[buf]);
    }
  } else if (warp == kW1 || warp == kW2) {
    // ---------------- weight streamers (one thread each) ----------------
    if (lane == 0) {
      const bool first = warp == kW1;
      uint64_t* full = first ? w1_full : w2_full;
      uint64_t* empty = first ? w1_empty : w2_empty;
      uint8_t* ring = smem + (first ? L::OFF_W1 : L::OFF_W2);
      const uint32_t slot_bytes = first ? L::W1C : L::W2C;
      int64_t q = 0;
      for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
        int e;
        int64_t r0, r1;
        if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
        const int np = p.np[e];
        const uint32_t bytes = first ? uint32_t(L::KC1 * np) * (HC * 32 * 2)
                                     : uint32_t(np) * (D * 32 * 2);
        const uint16_t* src0 = first ? p.w1[e] : p.w2[e];
        for (int c = 0; c < nchunk; ++c, ++q) {
          const int s = int(q % L::NW);
          PWAIT(first ? P_W1E : P_W2E, &empty[s], par(q / L::NW) ^ 1u);
          if (DBG && (p.dbg & 32)) {   // debug: no weight copies (slot contents stale)
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(ring + s * slot_bytes, src0 + size_t(c) * (bytes / 2), bytes, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMma) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    constexpr uint32_t id1 = idesc_bf16_m128(HC);
    constexpr uint32_t id2 = idesc_bf16_m128(D);
    const uint32_t sbase = smem_u32(smem);
    // The CTA's non-empty tiles in order (expert of each). fc1 runs LOOK
    // chunks ahead of fc2 across tile boundaries (no per-tile drain). Two
    // cursors walk (tile, chunk) with incremental counters: buffer indices
    // and mbarrier parities flip on wrap, no divisions in the loop.
    int nt = 0;
    if (lane == 0) {
      for (int64_t m = blockIdx.x; m < ntile && nt < kMaxTiles; m += gridDim.x) {
        int e;
        int64_t r0, r1;
        if (mlp_tile(p, c0, m, e, r0, r1)) tile_e[nt++] = uint8_t(e);
      }
    }
    nt = __shfl_sync(0xffffffffu, nt, 0);
    __syncwarp();
    struct Cur {
      int c, jt, np;     // chunk within tile, tile index, planes of the tile's expert
      int b, ws;         // acc1 / A2 buffer, weight ring slot
      uint32_t pb, pw;   // parities of b and ws (flip on wrap)
    };
    const int np0 = p.np[0], np1 = p.np[1];
    auto start_tile = [&](Cur& k) { k.np = (k.jt < nt && tile_e[k.jt]) ? np1 : np0; };
    auto advance = [&](Cur& k) {
      if (++k.b == L::NB) { k.b = 0; k.pb ^= 1u; }
      if (++k.ws == L::NW) { k.ws = 0; k.pw ^= 1u; }
      if (++k.c == nchunk) { k.c = 0; ++k.jt; start_tile(k); }
    };
    Cur f1{0, 0, 0, 0, 0, 0u, 0u}, f2{0, 0, 0, 0, 0, 0u, 0u};
    start_tile(f1);
    start_tile(f2);
    int ab1 = 0;                 // A1 buffer of f1's tile
    uint32_t pab1 = 0u;
    int ab2 = 0;                 // A1 buffer of f2's tile (released after its last fc1)
    int ob2 = 0;                 // acc2 buffer of f2's tile
    uint32_t pob2 = 0u;
    const int total_q = nt * nchunk;
    constexpr int LOOK = L::LOOK;
    for (int step = 0; step < total_q + LOOK; ++step) {
      if (step < total_q) {  // ---- fc1(f1)
        if (f1.c == 0) PWAIT(P_A1F, &a1_full[ab1], pab1);
        PWAIT(P_W1F, &w1_full[f1.ws], f1.pw);
        PWAIT(P_HE1, &h_empty[f1.b], f1.pb ^ 1u);   // acc1[b] drained (GELU(q - NB))
        if (!(DBG && (p.dbg & 128))) tc_fence_after();
        const uint32_t a1 = tmem + L::T_A1 + uint32_t(ab1) * L::A1COLS;
        const uint32_t w1 = sbase + L::OFF_W1 + f1.ws * L::W1C;
        const uint32_t d1 = tmem + L::T_ACC1 + uint32_t(f1.b * HC);
        if (!(DBG && (p.dbg & 16))) {
#pragma unroll
          for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ad = a1 + kc * 3 * kPlaneCols + ks * 8;
              const uint64_t bd = smem_desc(w1 + kc * f1.np * (HC * 32 * 2) + ks * 256);
              const uint32_t acc = (kc | ks) != 0;
              if (f1.np == 1)
                mma_chain3_ts_w(d1, ad, bd, kPlaneCols, id1, acc);
              else
                mma_chain6_ts_w(d1, ad, bd, kPlaneCols, (HC * 32 * 2) >> 4, id1, acc);
            }
        }
        commit(&h_full[f1.b]);
        commit(&w1_empty[f1.ws]);
        const bool last1 = f1.c == nchunk - 1;
        if (last1) commit(&a1_empty[ab1]);   // A1 fully consumed
        advance(f1);
        if (last1) {
          if (++ab1 == L::NA) { ab1 = 0; pab1 ^= 1u; }
        }
      }
      if (step >= LOOK) {   // ---- fc2(f2)
        if (f2.c == 0) PWAIT(P_OE, &o_empty[ob2], pob2 ^ 1u);   // acc2[ob] drained
        PWAIT(P_W2F, &w2_full[f2.ws], f2.pw);
        PWAIT(P_HE2, &h_empty[f2.b], f2.pb);            // GELU(q) wrote A2[b]
        if (!(DBG && (p.dbg & 128))) tc_fence_after();
        const uint32_t a2 = tmem + L::T_A2 + uint32_t(f2.b) * L::A2COLS;
        const uint32_t w2 = sbase + L::OFF_W2 + f2.ws * L::W2C;
        const uint32_t d2 = tmem + L::T_ACC2 + uint32_t(ob2 * D);
        if (!(DBG && (p.dbg & 16))) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t bd = smem_desc(w2 + ks * 256);
            const uint32_t acc = (f2.c | ks) != 0;
            if (f2.np == 1)
              mma_chain3_ts_w(d2, a2 + ks * 8, bd, kPlaneCols, id2, acc);
            else
              mma_chain6_ts_w(d2, a2 + ks * 8, bd, kPlaneCols, (D * 32 * 2) >> 4, id2, acc);
          }
        }
        commit(&a2_empty[f2.b]);
        commit(&w2_empty[f2.ws]);
        const bool last2 = f2.c == nchunk - 1;
        if (last2) commit(&o_full[ob2]);
        advance(f2);
        if (last2) {
          if (++ob2 == 2) { ob2 = 0; pob2 ^= 1u; }
        }
      }
    }
    (void)ab2;
  } else {
    // ---------------- GELU groups + final epilogue (warps 0-7) ----------------
    const int g = warp >> 2, quad = warp & 3;
    const int rl = quad * 32 + lane;
    float* xb = reinterpret_cast<float*>(smem + L::OFF_XB) + warp * 32 * kXPitch;
    int64_t q0 = 0;
    int64_t j = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      if (!mlp_tile(p, c0, m, e, r0, r1)) continue;
      const int ob = int(j & 1);
      const uint32_t oph = par(j >> 1);
      ++j;
      // the draining group's row metadata (dependent perm → gate loads) is
      // issued before the tile's GELU chunks so its latency overlaps them
      const int64_t r = r0 + rl;
      const bool r_ok = r < r1;
      int64_t orow = -1;
      float gt = 1.f;
      if (ob == g && r_ok) {
        orow = p.perm ? int64_t(__ldg(p.perm + r)) : r;
        if (p.gate) gt = __ldg(p.gate + orow);
      }
      for (int c = 0; c < nchunk; ++c) {
        const int64_t q = q0 + c;
        if (int(q & 1) != g) continue;
        const int b = int(q % L::NB);
        const uint32_t ph = par(q / L::NB);
        PWAIT(P_HF, &h_full[b], ph);            // fc1(q) done
        PWAIT(P_A2E, &a2_empty[b], ph ^ 1u);     // fc2(q - NB) finished reading A2[b]
        tc_fence_after();
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        float v[32];
        if (!(DBG && (p.dbg & 4))) {   // (debug switch: skip the GELU pass)
        {
          float lo[16], hi[16];
          const uint32_t ta = tmem + lane_base + L::T_ACC1 + uint32_t(b * HC);
          tmem_ld16(ta, lo);
          tmem_ld16(ta + 16, hi);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            v[t] = lo[t];
            v[16 + t] = hi[t];
          }
        }
        {
          uint32_t hp[16], mp[16], lp[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            float g0 = v[2 * t], g1 = v[2 * t + 1];
            gelu_fast2(g0, g1);
            const Split3 sp = split3x2(g0, g1);
            hp[t] = bf2_bits(sp.h);
            mp[t] = bf2_bits(sp.m);
            lp[t] = bf2_bits(sp.l);
          }
          const uint32_t a2 = tmem + lane_base + L::T_A2 + uint32_t(b) * L::A2COLS;
          tmem_st16(a2, hp);
          tmem_st16(a2 + kPlaneCols, mp);
          tmem_st16(a2 + 2 * kPlaneCols, lp);
          tmem_st_wait();
        }
        }
        tc_fence_before();
        mbar_arrive(&h_empty[b]);
      }
      q0 += nchunk;
      if (ob != g) continue;   // the other group drains this tile's acc2
      // ---- final epilogue: acc2 (128 x D) → × gate → + residual → scatter ----
      int64_t* rt = rowtab + g * 128;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");   // previous table consumed
      rt[rl] = orow;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");   // table published
      // the lane's 4 output rows (it * 8 + lane / 4) and 4 channels per 16-wide
      // column block; residual rows are prefetched one block ahead, the first
      // block before waiting for the accumulator
      const int c4 = (lane & 3) * 4;
      int64_t orow_l[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) orow_l[it] = rt[quad * 32 + it * 8 + (lane >> 2)];
      float4 res[2][4];
      auto load_res = [&](int cb, float4 (&dst)[4]) {
#pragma unroll
        for (int it = 0; it < 4; ++it)
          dst[it] = (p.residual && orow_l[it] >= 0)
                        ? __ldg(reinterpret_cast<const float4*>(p.residual + orow_l[it] * D + cb + c4))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      load_res(0, res[0]);
      PWAIT(P_OF, &o_full[ob], oph);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < D; cb += 16) {
        const int rb = (cb >> 4) & 1;
        if (cb + 16 < D) load_res(cb + 16, res[rb ^ 1]);
        float v[16];
        tmem_ld16(tmem + (uint32_t(quad * 32) << 16) + L::T_ACC2 + uint32_t(ob * D + cb), v);
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
      tc_fence_before();
      mbar_arrive(&o_empty[ob]);
    }
  }
  if (DBG && p.prof && lane == 0) {
    const int site = warp < 8 ? P_T_GELU : (warp < 12 ? P_T_PROD : (warp == kMma ? P_T_MMA : -1));
    if (site >= 0) atomicAdd(&sprof[site], (unsigned long long)(clock64() - t_start));
  }
#undef PWAIT
  tc_fence_before();
  __syncthreads();
  if (DBG && p.prof && tid < P_NSITE) atomicAdd(p.prof + tid, sprof[tid]);
  if (warp == kMma) tmem_dealloc<L::TCOLS>(tmem);
}

}  // namespace tcm

#ifdef SA_DEBUG
static unsigned long long* g_mlp_prof = nullptr;
extern "C" void sa_debug_mlp_profile(void* dev_buf) {
  g_mlp_prof = static_cast<unsigned long long*>(dev_buf);
}
#else
static constexpr unsigned long long* g_mlp_prof = nullptr;
#endif
SA_DEBUG_SWITCH(int, g_mlp_dbg, 0, sa_debug_mlp_mode)

static int g_sms_mlp = 0;

static int mlp_launch(tcm::MlpParams& p, int d, cudaStream_t s) {
  using namespace tcm;
  if (p.M == 0) return SA_OK;
  p.prof = g_mlp_prof;
  p.dbg = g_mlp_dbg;
  if (g_sms_mlp == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_mlp, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = cdiv(p.M, 128) + (p.counts ? 1 : 0);
  const int grid = int(tiles < g_sms_mlp ? tiles : g_sms_mlp);
  const bool dbg = p.prof != nullptr || p.dbg != 0;
#define SA_MLP_LAUNCH(DV, DB)                                                               \
  {                                                                                         \
    const int smem = int(Layout<DV>::TOTAL);                                                \
    cudaFuncSetAttribute(mlp_kernel<DV, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    mlp_kernel<DV, DB><<<grid, tcm::kThreads, smem, s>>>(p);                                \
  }
  if (d == 32) {
    if (dbg) SA_MLP_LAUNCH(32, true) else SA_MLP_LAUNCH(32, false)
  } else {
    if (dbg) SA_MLP_LAUNCH(64, true) else SA_MLP_LAUNCH(64, false)
  }
#undef SA_MLP_LAUNCH
  count_launch(1);
  SA_LAUNCH_CHECK("mlp_kernel");
  return SA_OK;
}

}  // namespace sa

using namespace sa;

/* The fused kernels read W1 packed with bn = 32 (hidden chunks) and W2 packed
 * with bn = d; see sa_weight_pack. */
extern "C" int sa_tc_fused_mlp_ok(int64_t d, int64_t hidden) {
  return (d == 32 || d == 64) && hidden % tcm::HC == 0 && hidden > 0;
}

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
  p.np[0] = 3;
  p.np[1] = 1;
  p.M = M;
  p.hidden = int(hidden);
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
  p.np[0] = w1_kind == SA_W_SHIFT ? 1 : 3;
  p.M = M;
  p.hidden = int(hidden);
  return mlp_launch(p, int(d), as_stream(stream));
}
