// Fused attention input: LayerNorm + the three q/k/v routers +
// both experts of each q/k/v MoE projection on the tensor cores + the sign-hash
// epilogue, for model dims 32 and 64 (head dim 32).
//
// Reference composition (Block.forward → AttentionLayer.forward,
// model.py:454-459, 340-358): y = LN1(x) (tensor.py:114-128); for r in q,k,v:
// route(y, W_g^r) (moe.py:81-92), proj_r(y) = gate · expert_e(y) with experts
// Linear / ShiftLinearLayer (model.py:250-274, 499-502); q, k are then binarised
// per (image, head) (quantize.py:123-140 via model.py:355-358).
//
// One persistent CTA per SM walks 128-token tiles of the flat (B·n, d) input:
//   warps 4-7  producers (thread = token row; d = 32 q/k/v: a second group,
//              warps 8-11, takes alternate tiles): the x row, LayerNorm in fp32
//              (the exact arithmetic of sa_ln_route), three fp64 router dots →
//              winner / gate (numpy-exp tie rule), written to the dispatch
//              arrays and to a shared route table; the normalised row split
//              into hi/mid/lo bf16 planes and stored to TMEM (A operand);
//   last warp  MMA issuer: per projection the dense expert (6 plane products)
//              and the shift expert (3, exact bf16 weights) into TMEM
//              accumulators — both experts for every token, so no
//              permutation / gather / scatter exists (the selection is a per-row
//              choice in the epilogue); all weights resident in shared memory;
//   warps 0-3  epilogue (thread = row): picks its expert's accumulator, × gate;
//              q and k → 32-bit sign codes (!(y < 0)) and fp64 |y| partials per
//              32-row segment (→ γ by sa_gamma_finalize), v → a 32 x 32 box in
//              128-byte-swizzled shared memory stored by TMA.
// Products per row are computed by the same split-precision MMA chains as the
// unfused path (sa_tc_moe_linear), so the projections agree bit for bit.
//
// The same kernel in its one-projection form (NP = 1) is the attention output
// projection W_O (AttentionLayer.forward, model.py:374, with the residual of
// Block.forward, model.py:454-459): no LayerNorm, one router on the merged
// heads, out = residual + gate · expert(merged), stored by TMA.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace qkv {

using namespace tc;

// Warp roles: Cfg::EG epilogue groups of 4 warps (warps 0 .. 4·EG-1), then
// Cfg::PG producer groups of 4 warps, then the MMA issuer (Cfg::MMA_WARP).
// Producer group g takes the CTA's tiles j = g, g + PG, ...; the A-operand
// buffers (NA) are a ring over tiles; the accumulators are a ring of NACC
// "units" — one (tile, projection) pair for the q/k/v form (both experts,
// 2·D columns), one tile for W_O — and epilogue group e takes units
// u = e, e + EG, ... All handshakes are mbarrier rings whose waiters can be at
// most one phase ahead (EG <= NACC, producer lag bounded by the A ring; see
// the wait sites).
constexpr uint32_t kPlaneCols = 16;
constexpr int kRT = 8;           // route-table ring slots (tiles)
constexpr int kAD = 8;           // "A buffer consumed" barrier ring (tiles)

#ifndef QKV_PG32
#define QKV_PG32 3   // q/k/v producer groups at d = 32
#endif
#ifndef QKV_EG32
#define QKV_EG32 2   // q/k/v epilogue groups at d = 32 (3: 107.0 vs 104.8 us)
#endif
#ifndef QKV_PG64
#define QKV_PG64 2   // q/k/v producer groups at d = 64
#endif
#ifndef QKV_RI64
#define QKV_RI64 3   // q/k/v router chains interleaved per pass at d = 64
#endif
#ifndef QKV_WO_PG
#define QKV_WO_PG 1
#endif
#ifndef QKV_WO_EG
#define QKV_WO_EG 1
#endif
template <int D, int NP, bool LNR = false>   // NP projections: 3 (q, k, v with LN1 + hash) or 1 (W_O)
struct Cfg {
  static constexpr int KC1 = D / 32;                // K stages of 32
  static constexpr int H = D / 32;                  // heads (dk = 32)
  // the q/k/v form is CUDA-core bound (LN, three fp64 router dots per row,
  // sign-hash / γ epilogue): several groups per role keep enough warps in
  // flight to hide their dependent chains
  static constexpr int PG = NP == 3 ? (D == 32 ? QKV_PG32 : QKV_PG64) : QKV_WO_PG;
  // (LNR: the W_O epilogue also runs the LayerNorm + fp64 router: two groups)
  static constexpr int EG = NP == 3 ? (D == 32 ? QKV_EG32 : 2) : (LNR ? 2 : QKV_WO_EG);
  static constexpr int NA = 2;                      // A buffers in TMEM
  static constexpr uint32_t ACC_COLS = 2 * D;       // one unit: dense | shift expert
  static constexpr int NACC = D == 32 ? 4 : 2;
  static constexpr int PROD0 = 4 * EG;
  static constexpr int MMA_WARP = PROD0 + 4 * PG;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr bool PREFETCH = PG <= 2 && (D == 32 || NP == 1);   // register budget
  static constexpr uint32_t A_COLS = KC1 * 3 * kPlaneCols;
  static constexpr uint32_t T_A = 0;
  static constexpr uint32_t T_ACC = (NA * A_COLS + 31) / 32 * 32;
  static_assert(T_ACC + NACC * ACC_COLS <= 512, "TMEM budget");
  static_assert(EG <= NACC, "epilogue groups may run at most one accumulator phase ahead");
  static_assert(PG <= 4, "route-table / A-ring phase bound");
  // resident weights: per projection dense (3 planes) then shift (1 plane)
  static constexpr uint32_t WD = uint32_t(D) * D * 2 * 3;
  static constexpr uint32_t WS = uint32_t(D) * D * 2;
  static constexpr uint32_t W_BYTES = NP * (WD + WS);
};

struct Params {
  const float* x;
  const float* gain;
  const float* bias;
  float eps;
  const float* wg[3];
  const uint16_t* wd[3];      // dense packed planes (bn = d)
  const uint16_t* wsh[3];     // shift packed plane (bn = d)
  float tie;
  int64_t M;
  int n;
  int32_t* expert_of;         // [3][M]
  float* gate;                // [3][M]
  uint32_t* codes[2];         // q, k: [B][H][n]
  float* rsum;                // [2][H][M] per-row Σ|y| (fp32 pairwise over the head's 32 columns)
  const float* residual;      // NP = 1: out = residual + gate · expert(x)
  // W_O form with the next LayerNorm + router in the epilogue (LNR): y2 =
  // LN2(out) (tmV2), the MLP router's (expert, gate) per row
  const float* ln_g;
  const float* ln_b;
  float ln_eps;
  const float* wg2;
  int32_t* expert_of2;
  float* gate2;
  int dbg;                    // debug builds: 1 producers skip LN / routers, 2 epilogue skips
                              // its work (handshakes only), 4 no MMAs, 8 producers skip loads,
                              // 32 skip routers only, 64 skip LN only
};
#ifdef SA_DEBUG
constexpr bool kQDbg = true;
#else
constexpr bool kQDbg = false;
#endif

// smem layout (bytes)
template <int D, int NP, bool LNR = false>
struct Smem {
  using C = Cfg<D, NP, LNR>;
  static constexpr uint32_t W = 0;
  static constexpr uint32_t WG = C::W_BYTES;                       // [NP (+1)][D][2] double
  static constexpr uint32_t RT_E = WG + (NP + (LNR ? 1 : 0)) * 2 * D * 8;   // [kRT][NP][128] int
  static constexpr uint32_t RT_G = RT_E + kRT * NP * 128 * 4;      // [kRT][NP][128] float
  static constexpr uint32_t BOX = (RT_G + kRT * NP * 128 * 4 + 1023) & ~1023u;  // [4·EG warps][H][4 KB]
  static constexpr uint32_t BOX2 = BOX + 4 * C::EG * C::H * 4096;   // LNR: y2 boxes
  static constexpr uint32_t BAR = BOX2 + (LNR ? 4 * C::EG * C::H * 4096 : 0);
  static constexpr uint32_t NBAR = C::NA + kAD + 2 * C::NACC + 2 * kRT + 1;
  static constexpr uint32_t TOTAL = BAR + NBAR * 8 + 16 + 1024;    // + alignment slack
  static_assert(TOTAL <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ int decide2(float l0, float l1, float tie_thresh, float& gate) {
  // same rule as moe.cu decide() (ref moe.py:81-92)
  const float m = fmaxf(l0, l1);
  const float sh0 = l0 - m, sh1 = l1 - m;
  const int e = (l1 > l0 && sh0 < -tie_thresh) ? 1 : 0;
  const float e0 = (sh0 >= -tie_thresh) ? 1.f : expf(sh0);
  const float e1 = (sh1 >= -tie_thresh) ? 1.f : expf(sh1);
  gate = (e ? e1 : e0) / (e0 + e1);
  return e;
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int D, int NP, bool LNR = false>
__global__ void __launch_bounds__(Cfg<D, NP, LNR>::THREADS, 1) qkv_kernel(Params p, const __grid_constant__ CUtensorMap tmV,
                                                                         const __grid_constant__ CUtensorMap tmV2) {
  static_assert(!LNR || NP == 1, "LN + router epilogue: W_O form only");
  using C = Cfg<D, NP, LNR>;
  using S = Smem<D, NP, LNR>;
  constexpr int kMma = C::MMA_WARP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* swg = reinterpret_cast<double*>(smem + S::WG);
  int* rt_e = reinterpret_cast<int*>(smem + S::RT_E);
  float* rt_g = reinterpret_cast<float*>(smem + S::RT_G);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::BAR);
  uint64_t* a_full = bar;
  uint64_t* a_done = a_full + C::NA;
  uint64_t* acc_full = a_done + kAD;
  uint64_t* acc_empty = acc_full + C::NACC;
  uint64_t* rt_full = acc_empty + C::NACC;
  uint64_t* rt_empty = rt_full + kRT;
  uint64_t* wbar = rt_empty + kRT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kMma) tmem_alloc<512>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < C::NA; ++i) mbar_init(&a_full[i], 4);
    for (int i = 0; i < kAD; ++i) mbar_init(&a_done[i], 1);
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    for (int i = 0; i < kRT; ++i) {
      mbar_init(&rt_full[i], 4);
      mbar_init(&rt_empty[i], 4 * NP);   // every unit of the tile reads its route
    }
    mbar_init(wbar, 1);
    fence_barrier_init();
    // every weight tile, once: per projection dense (3 planes) then shift
    mbar_expect_tx(wbar, C::W_BYTES);
    for (int r = 0; r < NP; ++r) {
      bulk_g2s(smem + S::W + r * (C::WD + C::WS), p.wd[r], C::WD, wbar);
      bulk_g2s(smem + S::W + r * (C::WD + C::WS) + C::WD, p.wsh[r], C::WS, wbar);
    }
  }
  for (int i = tid; i < NP * 2 * D; i += C::THREADS) swg[i] = double(p.wg[i / (2 * D)][i % (2 * D)]);
  if (LNR)
    for (int i = tid; i < 2 * D; i += C::THREADS) swg[NP * 2 * D + i] = double(p.wg2[i]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntile = int((p.M + 127) / 128);

  if (warp >= C::PROD0 && warp < kMma) {
    // ---------------- producers: LN + routers + A planes ----------------
    constexpr int NPG = C::PG;
    const int pg = (warp - C::PROD0) >> 2, pw = (warp - C::PROD0) & 3;
    const int rl = pw * 32 + lane;
    const uint32_t lane_base = uint32_t(pw * 32) << 16;
    float4 xn[C::PREFETCH ? D / 4 : 1];
    auto load_row = [&](int mm, float4* dst) {
      const int64_t rr = int64_t(mm) * 128 + rl;
      const float4* xr = reinterpret_cast<const float4*>(p.x + rr * D);
#pragma unroll
      for (int i = 0; i < D / 4; ++i)
        dst[i] = (mm < ntile && rr < p.M && !(kQDbg && (p.dbg & 8))) ? __ldg(xr + i)
                                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    if (C::PREFETCH) load_row(blockIdx.x + pg * gridDim.x, xn);
    int j = pg;
    for (int m = blockIdx.x + pg * gridDim.x; m < ntile; m += NPG * gridDim.x, j += NPG) {
      const int64_t row = int64_t(m) * 128 + rl;
      const bool ok = row < p.M;
      float v[D];
      {
        float4 xc[C::PREFETCH ? 1 : D / 4];
        const float4* src = xn;
        if (!C::PREFETCH) {
          load_row(m, xc);
          src = xc;
        }
#pragma unroll
        for (int i = 0; i < D / 4; ++i) {
          v[4 * i] = src[i].x; v[4 * i + 1] = src[i].y; v[4 * i + 2] = src[i].z; v[4 * i + 3] = src[i].w;
        }
      }
      if (C::PREFETCH) load_row(m + NPG * gridDim.x, xn);
      if (NP == 3 && ok && !(kQDbg && (p.dbg & 65))) {
        // LayerNorm: the exact operation sequence of ln_route_kernel (moe.cu)
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < D / 4; ++i) s += (v[4 * i] + v[4 * i + 1]) + (v[4 * i + 2] + v[4 * i + 3]);
        const float mean = s / float(D);
        float q2 = 0.f;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          v[i] -= mean;
          q2 += v[i] * v[i];
        }
        const float inv = 1.0f / sqrtf(q2 / float(D) + p.eps);
#pragma unroll
        for (int i = 0; i < D / 4; ++i) {
          const float4 g = __ldg(reinterpret_cast<const float4*>(p.gain) + i);
          const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias) + i);
          v[4 * i] = v[4 * i] * inv * g.x + b.x;
          v[4 * i + 1] = v[4 * i + 1] * inv * g.y + b.y;
          v[4 * i + 2] = v[4 * i + 2] * inv * g.z + b.z;
          v[4 * i + 3] = v[4 * i + 3] * inv * g.w + b.w;
        }
      }
      // routers (fp64 dots in channel order, as ln_route_kernel / route_kernel).
      // Slot rs was last used by tile j - kRT; this group's previous tile
      // passed its A-ring wait, so tile j - kRT's release is the only
      // outstanding phase (one-phase-ahead bound).
      const int rs = j % kRT;
      mbar_wait(&rt_empty[rs], (uint32_t(j / kRT) & 1u) ^ 1u);
      // the NP routers' chains are interleaved (2·NP independent fp64 chains
      // in flight, each in channel order, so the logits are unchanged)
      constexpr int RI = (NP == 3 && D == 64) ? QKV_RI64 : NP;
#pragma unroll 1
      for (int r0 = 0; r0 < NP; r0 += RI) {
        if (kQDbg && (p.dbg & 33)) {   // debug: no router dots (route table: expert 0, gate 1)
#pragma unroll
          for (int i = 0; i < RI; ++i) {
            rt_e[(rs * NP + r0 + i) * 128 + rl] = 0;
            rt_g[(rs * NP + r0 + i) * 128 + rl] = 1.f;
          }
        } else {
        double s0[RI], s1[RI];
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          s0[i] = 0.0;
          s1[i] = 0.0;
        }
        // weights of channel c + 1 are loaded while channel c's DFMAs run
        // (warp-uniform shared-memory broadcasts)
        const double2* wrow = reinterpret_cast<const double2*>(swg) + r0 * D;
        double2 wc[RI];
#pragma unroll
        for (int i = 0; i < RI; ++i) wc[i] = wrow[i * D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double2 wn[RI];
#pragma unroll
          for (int i = 0; i < RI; ++i) wn[i] = wrow[i * D + (c + 1 < D ? c + 1 : c)];
          const double vc = double(v[c]);
#pragma unroll
          for (int i = 0; i < RI; ++i) {
            s0[i] = fma(vc, wc[i].x, s0[i]);
            s1[i] = fma(vc, wc[i].y, s1[i]);
          }
#pragma unroll
          for (int i = 0; i < RI; ++i) wc[i] = wn[i];
        }
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          const int r = r0 + i;
          float g = 1.f;
          int e = 0;
          if (ok) {
            e = decide2(float(s0[i]), float(s1[i]), p.tie, g);
            p.expert_of[r * p.M + row] = e;
            p.gate[r * p.M + row] = g;
          }
          rt_e[(rs * NP + r) * 128 + rl] = e;
          rt_g[(rs * NP + r) * 128 + rl] = g;
        }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rt_full[rs]);
      // A planes → TMEM: buffer ab was last read by tile j - NA's MMAs
      const int ab = j % C::NA;
      if (j >= C::NA) mbar_wait(&a_done[(j - C::NA) % kAD], uint32_t((j - C::NA) / kAD) & 1u);
      tc_fence_after();
      const uint32_t a1 = tmem + lane_base + C::T_A + uint32_t(ab) * C::A_COLS;
#pragma unroll
      for (int kc = 0; kc < C::KC1; ++kc) {
        uint32_t hp[16], mp[16], lp[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const Split3u sp = split3x2_trunc(v[kc * 32 + 2 * t], v[kc * 32 + 2 * t + 1]);
          hp[t] = sp.h;
          mp[t] = sp.m;
          lp[t] = sp.l;
        }
        tmem_st16(a1 + kc * 3 * kPlaneCols, hp);
        tmem_st16(a1 + kc * 3 * kPlaneCols + kPlaneCols, mp);
        tmem_st16(a1 + kc * 3 * kPlaneCols + 2 * kPlaneCols, lp);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[ab]);
    }
  } else if (warp == kMma) {
    // ---------------- MMA issuer (whole warp; one elected lane issues) ----------------
    mbar_wait(wbar, 0);   // resident weights landed
    constexpr uint32_t idesc = idesc_bf16_m128(D);
    const uint32_t wbase = smem_u32(smem + S::W);
    int u = 0;
    int j = 0;
    for (int m = blockIdx.x; m < ntile; m += gridDim.x, ++j) {
      const int ab = j % C::NA;
      mbar_wait(&a_full[ab], uint32_t(j / C::NA) & 1u);
      tc_fence_after();
      const uint32_t a0 = tmem + C::T_A + uint32_t(ab) * C::A_COLS;
#pragma unroll
      for (int r = 0; r < NP; ++r, ++u) {
        const int cb = u % C::NACC;
        mbar_wait(&acc_empty[cb], (uint32_t(u / C::NACC) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + C::T_ACC + uint32_t(cb) * C::ACC_COLS;
        if (!(kQDbg && (p.dbg & 4))) {
          const uint32_t wd = wbase + r * (C::WD + C::WS);
          const uint32_t ws = wd + C::WD;
#pragma unroll
          for (int kc = 0; kc < C::KC1; ++kc)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ad = a0 + kc * 3 * kPlaneCols + ks * 8;
              const uint32_t accf = (kc | ks) != 0;
              mma_chain6_ts_w(acc, ad, smem_desc(wd + kc * 3 * (D * 32 * 2) + ks * 256), kPlaneCols,
                              (D * 32 * 2) >> 4, idesc, accf);
              mma_chain3_ts_w(acc + uint32_t(D), ad, smem_desc(ws + kc * (D * 32 * 2) + ks * 256),
                              kPlaneCols, idesc, accf);
            }
        }
        commit_w(&acc_full[cb]);
      }
      commit_w(&a_done[j % kAD]);
    }
  } else if (warp < C::PROD0) {
    // ---------------- epilogue (thread = row), group eg takes units eg, eg + EG, ... ----------------
    const int eg = warp >> 2, quad = warp & 3;
    const int rl = quad * 32 + lane;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    uint8_t* box = smem + S::BOX + (eg * 4 + quad) * C::H * 4096;
    const int nunit = ((ntile - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x)) * NP;
    for (int u = eg; u < nunit; u += C::EG) {
      const int j = u / NP, r = u % NP;
      const int m = int(blockIdx.x) + j * int(gridDim.x);
      const int64_t row = int64_t(m) * 128 + rl;
      const bool ok = row < p.M;
      const int rs = j % kRT, cb = u % C::NACC;
      // one-phase-ahead: this group's previous unit u - EG >= u - NACC was
      // already committed, and tile j - 1's route (or older) was already read
      mbar_wait(&rt_full[rs], uint32_t(j / kRT) & 1u);
      const int e = rt_e[(rs * NP + r) * 128 + rl];
      const float g = rt_g[(rs * NP + r) * 128 + rl];
      // W_O: the residual row is loaded before the accumulator wait
      float4 res[NP == 1 ? D / 4 : 1];
      if (NP == 1) {
#pragma unroll
        for (int i = 0; i < (NP == 1 ? D / 4 : 0); ++i)
          res[i] = ok ? __ldg(reinterpret_cast<const float4*>(p.residual + row * D) + i)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rt_empty[rs]);
      mbar_wait(&acc_full[cb], uint32_t(u / C::NACC) & 1u);
      tc_fence_after();
      if (kQDbg && (p.dbg & 2)) {
        tc_fence_before();
        mbar_arrive(&acc_empty[cb]);
        continue;
      }
      const uint32_t acc = tmem + lane_base + C::T_ACC + uint32_t(cb) * C::ACC_COLS;
      // image / segment bookkeeping of this warp's 32 rows
      const int64_t wrow0 = int64_t(m) * 128 + quad * 32;
      const int b = int(row / p.n), t = int(row - int64_t(b) * p.n);
      const float2 g2 = make_float2(g, g);
      float hrow[LNR ? D : 1];   // LNR: the output row, for the LayerNorm + router below
#pragma unroll
      for (int hh = 0; hh < C::H; ++hh) {
        uint32_t code = 0u;
        float hs[2];
        uint8_t* bx = box + hh * 4096;
        if (!(NP == 3 && r < 2)) {   // v / W_O: the box is free once its last TMA store read it
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t rd[16], rsft[16];
          tmem_ld16_nowait(acc + hh * 32 + half * 16, rd);
          tmem_ld16_nowait(acc + uint32_t(D) + hh * 32 + half * 16, rsft);
          tmem_ld_wait();
          // gate and residual are two float32 roundings, as the reference's
          // y * gate then residual + y (no FMA contraction)
          float y[16];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            const float2 a2 = make_float2(__uint_as_float(e ? rsft[c] : rd[c]),
                                          __uint_as_float(e ? rsft[c + 1] : rd[c + 1]));
            const float2 y2 = __fmul2_rn(g2, a2);
            y[c] = y2.x;
            y[c + 1] = y2.y;
          }
          if (NP == 1) {   // W_O: + residual
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const int cc = hh * 32 + half * 16 + c;
              const float4 q4 = res[NP == 1 ? cc / 4 : 0];
              const float rv = (c & 3) == 0 ? q4.x : (c & 3) == 1 ? q4.y : (c & 3) == 2 ? q4.z : q4.w;
              y[c] = __fadd_rn(rv, y[c]);
              if (LNR) hrow[LNR ? cc : 0] = y[c];
            }
          }
          if (NP == 3 && r < 2) {
#pragma unroll
            for (int c = 0; c < 16; ++c) code |= (y[c] < 0.f ? 0u : 1u) << (half * 16 + c);
            // |y| row sum: fixed pairwise fp32 tree over the 32 columns
            // (error <= 5 ulp of the row sum), fp64 across rows below
            float tsum[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) tsum[c] = fabsf(y[2 * c]) + fabsf(y[2 * c + 1]);
#pragma unroll
            for (int w = 4; w > 0; w >>= 1)
#pragma unroll
              for (int c = 0; c < w; ++c) tsum[c] += tsum[c + w];
            hs[half] = tsum[0];
          } else {
            // v / W_O: half of a 32 x 32 box (128-byte swizzle) → TMA store
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int ch = half * 4 + c;
              *reinterpret_cast<float4*>(bx + lane * 128 + ((ch ^ (lane & 7)) * 16)) =
                  make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
            }
          }
        }
        if (NP == 3 && r < 2) {
          if (ok) {
            p.codes[r][(int64_t(b) * C::H + hh) * p.n + t] = code;
            p.rsum[(int64_t(r) * C::H + hh) * p.M + row] = hs[0] + hs[1];
          }
        } else {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmV, bx, hh * 32, int(wrow0));
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[cb]);
      if (LNR) {
        // LayerNorm of the output row + the next MoE router on it: the exact
        // operation sequence of ln_route_kernel (moe.cu), so y2 and the route
        // are bit-identical to sa_ln_route on the stored output
        if (ok) {
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < D / 4; ++i)
            s += (hrow[4 * i] + hrow[4 * i + 1]) + (hrow[4 * i + 2] + hrow[4 * i + 3]);
          const float mean = s / float(D);
          float q2 = 0.f;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            hrow[i] -= mean;
            q2 += hrow[i] * hrow[i];
          }
          const float inv = 1.0f / sqrtf(q2 / float(D) + p.ln_eps);
#pragma unroll
          for (int i = 0; i < D / 4; ++i) {
            const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.ln_g) + i);
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.ln_b) + i);
            hrow[4 * i] = hrow[4 * i] * inv * g4.x + b4.x;
            hrow[4 * i + 1] = hrow[4 * i + 1] * inv * g4.y + b4.y;
            hrow[4 * i + 2] = hrow[4 * i + 2] * inv * g4.z + b4.z;
            hrow[4 * i + 3] = hrow[4 * i + 3] * inv * g4.w + b4.w;
          }
          const double2* w2r = reinterpret_cast<const double2*>(swg + NP * 2 * D);
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const double2 w = w2r[c];
            const double vc = double(hrow[c]);
            s0 = fma(vc, w.x, s0);
            s1 = fma(vc, w.y, s1);
          }
          float g2v;
          const int e2 = decide2(float(s0), float(s1), p.tie, g2v);
          p.expert_of2[row] = e2;
          p.gate2[row] = g2v;
        }
        // y2 boxes: free once their previous stores (issued before this
        // unit's H output-box stores) were read
        uint8_t* box2 = smem + S::BOX2 + (eg * 4 + quad) * C::H * 4096;
        if (lane == 0) {
          if (C::H == 1)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
        }
        __syncwarp();
#pragma unroll
        for (int hh = 0; hh < C::H; ++hh)
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(box2 + hh * 4096 + lane * 128 + ((c ^ (lane & 7)) * 16)) =
                make_float4(hrow[(hh * 32 + 4 * c) % (LNR ? D : 1)],
                            hrow[(hh * 32 + 4 * c + 1) % (LNR ? D : 1)],
                            hrow[(hh * 32 + 4 * c + 2) % (LNR ? D : 1)],
                            hrow[(hh * 32 + 4 * c + 3) % (LNR ? D : 1)]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int hh = 0; hh < C::H; ++hh) {
            tma_store_2d(&tmV2, box2 + hh * 4096, hh * 32, int(wrow0));
            bulk_commit();
          }
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) tmem_dealloc<512>(tmem);
}

// γ[r][b·H + h] = Σ |y| over image b's rows of head h / (n · 32): one
// 128-thread CTA per (r, b, h); thread t sums the per-row fp32 sums of rows
// t, t + 128, ... in fp64 (four independent loads in flight), each warp meets
// in a fixed xor tree and thread 0 adds the four warp sums in order
// (deterministic, no atomics).
constexpr int kGfThreads = 128;
__global__ void __launch_bounds__(kGfThreads) gamma_finalize_qkv(const float* __restrict__ rsum,
                                                               int64_t M, int H, int64_t B, int n,
                                                               float* __restrict__ gq,
                                                               float* __restrict__ gk) {
  __shared__ double ws[kGfThreads / 32];
  const int64_t i = blockIdx.x;   // (r, b, h)
  const int tid = threadIdx.x, lane = tid & 31;
  const int r = int(i / (B * H));
  const int64_t bh = i % (B * H);
  const int64_t b = bh / H;
  const int h = int(bh % H);
  const float* src = rsum + (int64_t(r) * H + h) * M + b * n;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int t = tid;
  for (; t + 3 * kGfThreads < n; t += 4 * kGfThreads) {
    s0 += double(__ldg(src + t));
    s1 += double(__ldg(src + t + kGfThreads));
    s2 += double(__ldg(src + t + 2 * kGfThreads));
    s3 += double(__ldg(src + t + 3 * kGfThreads));
  }
  for (; t < n; t += kGfThreads) s0 += double(__ldg(src + t));
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ws[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    const double tot = (ws[0] + ws[1]) + (ws[2] + ws[3]);
    (r == 0 ? gq : gk)[bh] = float(tot / (double(n) * 32.0));
  }
}

}  // namespace qkv
}  // namespace sa

using namespace sa;

SA_DEBUG_SWITCH(int, g_qkv_dbg, 0, sa_debug_qkv_mode)


extern "C" int sa_ln_qkv_hash_ok(int64_t d, int64_t n) {
  return (d == 32 || d == 64) && n >= 32;
}

extern "C" size_t sa_ln_qkv_hash_workspace(int64_t B, int64_t n, int64_t d) {
  const int64_t M = B * n;
  return size_t(2 * M * (d / 32)) * sizeof(float) + 256;
}

extern "C" int sa_ln_qkv_hash(const float* x, const float* gain, const float* bias, float eps,
                              const float* wg_q, const float* wg_k, const float* wg_v,
                              const void* wq_dense, const void* wq_shift, const void* wk_dense,
                              const void* wk_shift, const void* wv_dense, const void* wv_shift,
                              float tie_thresh, int64_t B, int64_t n, int64_t d,
                              int32_t* expert_of, float* gate, uint32_t* codes_q,
                              uint32_t* codes_k, float* gamma_q, float* gamma_k, float* v,
                              void* ws, size_t ws_bytes, void* stream) {
  using namespace qkv;
  SA_REQUIRE(sa_ln_qkv_hash_ok(d, n), SA_ERR_SHAPE, "sa_ln_qkv_hash: d=%lld n=%lld unsupported",
             (long long)d, (long long)n);
  SA_REQUIRE(B > 0 && B * n < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_ln_qkv_hash: bad batch");
  SA_REQUIRE(ws_bytes >= sa_ln_qkv_hash_workspace(B, n, d), SA_ERR_VALUE,
             "sa_ln_qkv_hash: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t M = B * n;
  Params p;
  memset(&p, 0, sizeof(p));
  p.dbg = g_qkv_dbg;
  p.x = x;
  p.gain = gain;
  p.bias = bias;
  p.eps = eps;
  p.wg[0] = wg_q; p.wg[1] = wg_k; p.wg[2] = wg_v;
  p.wd[0] = static_cast<const uint16_t*>(wq_dense);
  p.wd[1] = static_cast<const uint16_t*>(wk_dense);
  p.wd[2] = static_cast<const uint16_t*>(wv_dense);
  p.wsh[0] = static_cast<const uint16_t*>(wq_shift);
  p.wsh[1] = static_cast<const uint16_t*>(wk_shift);
  p.wsh[2] = static_cast<const uint16_t*>(wv_shift);
  p.tie = tie_thresh;
  p.M = M;
  p.n = int(n);
  p.expert_of = expert_of;
  p.gate = gate;
  p.codes[0] = codes_q;
  p.codes[1] = codes_k;
  p.rsum = static_cast<float*>(ws);
  CUtensorMap tmV;
  memset(&tmV, 0, sizeof(tmV));
  {
    const cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(M)};
    const cuuint64_t strides[1] = {cuuint64_t(d) * 4};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tmap_tiled(
        &tmV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, v, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SA_REQUIRE(r == CUDA_SUCCESS, SA_ERR_CUDA, "sa_ln_qkv_hash: tensor map for v failed (%d)", int(r));
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (M + 127) / 128;
  const int grid = int(tiles < sms ? tiles : sms);
  if (d == 32) {
    const int smem = int(Smem<32, 3>::TOTAL);
    cudaFuncSetAttribute(qkv_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    qkv_kernel<32, 3><<<grid, qkv::Cfg<32, 3>::THREADS, smem, s>>>(p, tmV, tmV);
  } else {
    const int smem = int(Smem<64, 3>::TOTAL);
    cudaFuncSetAttribute(qkv_kernel<64, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    qkv_kernel<64, 3><<<grid, qkv::Cfg<64, 3>::THREADS, smem, s>>>(p, tmV, tmV);
  }
  const int64_t H = d / 32;
  gamma_finalize_qkv<<<unsigned(2 * B * H), kGfThreads, 0, s>>>(p.rsum, M, int(H), B,
                                                                 int(n), gamma_q, gamma_k);
  count_launch(2);
  SA_LAUNCH_CHECK("sa_ln_qkv_hash");
  return SA_OK;
}

/* MoeModule.forward of a (Linear, ShiftLinearLayer) projection with d -> d and
 * the block residual (the attention output projection, model.py:250-274, 374,
 * 454-459): route (fp64 dot, numpy tie rule), both experts on the tensor cores,
 * out = residual + gate · expert(x); expert_of / gate [M] for the lazy plan. */
extern "C" int sa_fused_moe_linear_ok(int64_t d) { return d == 32 || d == 64; }

namespace {

int encode_rows_map(CUtensorMap* tm, float* base, int64_t M, int64_t d) {
  memset(tm, 0, sizeof(*tm));
  const cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(M)};
  const cuuint64_t strides[1] = {cuuint64_t(d) * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  return int(encode_tmap_tiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

template <int D, bool LNR>
void launch_wo(const qkv::Params& p, const CUtensorMap& tmY, const CUtensorMap& tmY2, int grid,
               cudaStream_t s) {
  using namespace qkv;
  const int smem = int(Smem<D, 1, LNR>::TOTAL);
  cudaFuncSetAttribute(qkv_kernel<D, 1, LNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  qkv_kernel<D, 1, LNR><<<grid, Cfg<D, 1, LNR>::THREADS, smem, s>>>(p, tmY, tmY2);
}

int fused_moe_linear_impl(const char* who, const float* x, const float* wg, const void* w_dense,
                          const void* w_shift, const float* residual, float tie_thresh, int64_t M,
                          int64_t d, int32_t* expert_of, float* gate, float* y,
                          const float* ln_gain, const float* ln_bias, float eps,
                          const float* wg2, float* y2, int32_t* expert_of2, float* gate2,
                          void* stream) {
  using namespace qkv;
  SA_REQUIRE(sa_fused_moe_linear_ok(d), SA_ERR_SHAPE, "%s: d=%lld unsupported", who, (long long)d);
  SA_REQUIRE(M > 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "%s: bad M", who);
  SA_REQUIRE(residual != nullptr, SA_ERR_VALUE, "%s: residual required", who);
  const bool lnr = y2 != nullptr;
  SA_REQUIRE(!lnr || (ln_gain && ln_bias && wg2 && expert_of2 && gate2), SA_ERR_VALUE,
             "%s: LayerNorm / router outputs need gain, bias, router weights and route arrays", who);
  cudaStream_t s = as_stream(stream);
  Params p;
  memset(&p, 0, sizeof(p));
  p.dbg = g_qkv_dbg;
  p.x = x;
  p.wg[0] = wg;
  p.wd[0] = static_cast<const uint16_t*>(w_dense);
  p.wsh[0] = static_cast<const uint16_t*>(w_shift);
  p.tie = tie_thresh;
  p.M = M;
  p.n = int(M);   // (no image structure needed: no hashing)
  p.expert_of = expert_of;
  p.gate = gate;
  p.residual = residual;
  p.ln_g = ln_gain;
  p.ln_b = ln_bias;
  p.ln_eps = eps;
  p.wg2 = wg2;
  p.expert_of2 = expert_of2;
  p.gate2 = gate2;
  CUtensorMap tmY, tmY2;
  int r = encode_rows_map(&tmY, y, M, d);
  SA_REQUIRE(r == CUDA_SUCCESS, SA_ERR_CUDA, "%s: tensor map failed (%d)", who, r);
  if (lnr) {
    r = encode_rows_map(&tmY2, y2, M, d);
    SA_REQUIRE(r == CUDA_SUCCESS, SA_ERR_CUDA, "%s: tensor map for y2 failed (%d)", who, r);
  } else {
    tmY2 = tmY;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (M + 127) / 128;
  const int grid = int(tiles < sms ? tiles : sms);
  if (d == 32) {
    if (lnr) launch_wo<32, true>(p, tmY, tmY2, grid, s);
    else launch_wo<32, false>(p, tmY, tmY2, grid, s);
  } else {
    if (lnr) launch_wo<64, true>(p, tmY, tmY2, grid, s);
    else launch_wo<64, false>(p, tmY, tmY2, grid, s);
  }
  count_launch(1);
  SA_LAUNCH_CHECK(who);
  return SA_OK;
}

}  // namespace

extern "C" int sa_fused_moe_linear(const float* x, const float* wg, const void* w_dense,
                                   const void* w_shift, const float* residual, float tie_thresh,
                                   int64_t M, int64_t d, int32_t* expert_of, float* gate,
                                   float* y, void* stream) {
  return fused_moe_linear_impl("sa_fused_moe_linear", x, wg, w_dense, w_shift, residual,
                               tie_thresh, M, d, expert_of, gate, y, nullptr, nullptr, 0.f,
                               nullptr, nullptr, nullptr, nullptr, stream);
}

/* The same W_O kernel with the block's second LayerNorm and the MLP router in
 * its epilogue (Block.forward, model.py:454-459: h = x + attn(LN1 x); the MLP
 * input LN2(h) and its route, moe.py:81-92): y = h, y2 = LN2(h) and the MLP's
 * (expert, gate) per row — what sa_ln_route computes from h, bit for bit,
 * without re-reading h. */
extern "C" int sa_fused_moe_linear_ln_route(const float* x, const float* wg, const void* w_dense,
                                            const void* w_shift, const float* residual,
                                            float tie_thresh, int64_t M, int64_t d,
                                            int32_t* expert_of, float* gate, float* y,
                                            const float* ln_gain, const float* ln_bias, float eps,
                                            const float* wg2, float* y2, int32_t* expert_of2,
                                            float* gate2, void* stream) {
  SA_REQUIRE(y2 != nullptr, SA_ERR_VALUE, "sa_fused_moe_linear_ln_route: y2 required");
  return fused_moe_linear_impl("sa_fused_moe_linear_ln_route", x, wg, w_dense, w_shift, residual,
                               tie_thresh, M, d, expert_of, gate, y, ln_gain, ln_bias, eps, wg2,
                               y2, expert_of2, gate2, stream);
}
