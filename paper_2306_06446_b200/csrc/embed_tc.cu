// Patch embedding + the stage's embedding LayerNorm in one warp-specialised
// tcgen05 kernel (d = 32 / 64, K = patch·patch·C <= 128, no cls / pos: the
// PVTv2 stages).
//
// Reference: Model.patchify + patch_embed.forward (model.py:557-570) followed by
// LayerNorm.forward (model.py:174-178, tensor.py:114-128). Same arithmetic as
// the GEMM path's LNE instantiation (tc_gemm_kernel<BN, A_PATCH, false, true>):
// x − sub split into hi/mid/lo bf16 planes, dense weights in three planes, the
// six plane products per K step in the same order, then the row LayerNorm with
// layernorm_row_kernel's summation order — bit-identical outputs.
//
// Why a separate kernel: the embedding GEMM is N = d = 32 / 64 wide and 2-4 K
// stages deep, so the generic GEMM's per-stage handshakes (producer group →
// stage ring → MMA → commit) and its K-stage-granular A staging dominate; here
// a producer thread owns a token row for the whole tile (the patch's image
// rows, contiguous p·C floats each), stores all its K planes to TMEM at once,
// and the MMA warp issues the tile's K steps back to back:
//   warps 0-3   epilogue (thread = token row): LayerNorm from TMEM (two passes
//               for mean and variance, a third to normalise), shared-memory
//               transpose, coalesced row stores;
//   warps 4..   producers, groups of 4 warps: K <= 64: four groups on
//               alternate tiles (four tiles' image loads in flight, one TMEM A
//               buffer each); deeper K: two groups splitting each row's K
//               stages;
//   last warp   MMA issuer; the packed weights stay resident in shared memory.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace emb {

using namespace tc;

constexpr uint32_t kPlaneCols = 16;

#ifndef EMB_SPLIT_MINKC
#define EMB_SPLIT_MINKC 2   // K stages above which the producers split K instead of alternating tiles
#endif
#ifndef EMB_SPLIT_PG
#define EMB_SPLIT_PG 4   // split-K producer groups (each converts KC / PG stages of every tile)
#endif
template <int D, int KC>
struct Cfg {
  // producer groups: K <= 64: two groups on alternate tiles (two tiles' image
  // loads in flight); deeper K: two groups splitting each row's K stages
  static constexpr bool SPLITK = KC > EMB_SPLIT_MINKC;
  static constexpr int PG = SPLITK ? (KC < EMB_SPLIT_PG ? KC : EMB_SPLIT_PG) : 4;
  static_assert(!SPLITK || KC % PG == 0, "split K: whole K stages per group");
  static constexpr int MMA_WARP = 4 + 4 * PG;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr int NA = SPLITK ? 2 : 4, NACC = 2;
  static constexpr uint32_t A_COLS = KC * 3 * kPlaneCols;
  static constexpr uint32_t T_A = 0;
  static constexpr uint32_t T_ACC = NA * A_COLS;
  static constexpr uint32_t TCOLS = 512;
  static_assert(T_ACC + NACC * D <= TCOLS, "TMEM budget");
  static constexpr uint32_t W_BYTES = uint32_t(KC) * 3 * D * 64;   // resident packed weights
  static constexpr uint32_t XB = W_BYTES;                          // [4 warps][32][kXPitch] fp32
  static constexpr uint32_t BAR = XB + 4 * 32 * kXPitch * 4;
  static constexpr uint32_t TOTAL = BAR + 16 * 8 + 16 + 1024;
};

struct Params {
  const float* grid;          // NHWC (B, H, W, C)
  int64_t H, W, C;
  int patch, side;
  float sub;
  const uint16_t* w;          // packed (bn = d), 3 planes
  const float* gain;
  const float* bias;
  float eps;
  float* y;                   // (B·side², d)
  int64_t M;
  int n;                      // tokens per image
  int K;                      // patch·patch·C
};

template <int D, int KC>
__global__ void __launch_bounds__(Cfg<D, KC>::THREADS, 1) embed_ln_kernel(Params p) {
  using CF = Cfg<D, KC>;
  constexpr int kMma = CF::MMA_WARP;
  constexpr int KV = KC * 8;   // float4 per row (zero past K)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + CF::BAR);
  uint64_t* a_full = bar;                // [NA] producer group's 4 warps
  uint64_t* a_empty = a_full + CF::NA;   // [NA] MMA commit
  uint64_t* acc_full = a_empty + CF::NA; // [NACC] MMA commit
  uint64_t* acc_empty = acc_full + CF::NACC;   // [NACC] 128 epilogue threads
  uint64_t* wbar = acc_empty + CF::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kMma) tmem_alloc<CF::TCOLS>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < CF::NA; ++i) {
      mbar_init(&a_full[i], CF::SPLITK ? 4 * CF::PG : 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < CF::NACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    mbar_init(wbar, 1);
    fence_barrier_init();
    mbar_expect_tx(wbar, CF::W_BYTES);
    bulk_g2s(smem, p.w, CF::W_BYTES, wbar);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntile = int((p.M + 127) / 128);

  if (warp >= 4 && warp < kMma) {
    // ---------------- producers: patch rows → A planes (TMEM) ----------------
    const int pg = (warp - 4) >> 2, pw = (warp - 4) & 3;
    const int rl = pw * 32 + lane;
    const uint32_t lane_base = uint32_t(pw * 32) << 16;
    const int rowf4 = int(p.patch * p.C) / 4;   // float4 per image row of the patch
    constexpr int KCG = CF::SPLITK ? KC / CF::PG : KC;   // K stages this group converts
    const int kc0 = CF::SPLITK ? pg * KCG : 0;
    const int mstep = CF::SPLITK ? gridDim.x : CF::PG * gridDim.x;
    int j = CF::SPLITK ? 0 : pg;
    for (int m = blockIdx.x + (CF::SPLITK ? 0 : pg) * gridDim.x; m < ntile;
         m += mstep, j += CF::SPLITK ? 1 : CF::PG) {
      const int64_t t = int64_t(m) * 128 + rl;
      float4 v[KCG * 8];
#pragma unroll
      for (int i = 0; i < KCG * 8; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < p.M) {
        const int b = int(t / p.n), tt = int(t - int64_t(b) * p.n);
        const int py = tt / p.side, px = tt - py * p.side;
        const float* base = p.grid + ((int64_t(b) * p.H + int64_t(py) * p.patch) * p.W +
                                      int64_t(px) * p.patch) * p.C;
#pragma unroll
        for (int i = 0; i < KCG * 8; ++i) {
          const int ig = kc0 * 8 + i;                          // float4 index in the row's K
          const int ir = ig / rowf4, ic = ig - ir * rowf4;   // image row of the patch, float4 in it
          if (ir < p.patch) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(base + int64_t(ir) * p.W * p.C) + ic);
            v[i] = make_float4(q.x - p.sub, q.y - p.sub, q.z - p.sub, q.w - p.sub);
          }
        }
      }
      const int ab = j % CF::NA;
      mbar_wait(&a_empty[ab], (uint32_t(j / CF::NA) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t a1 = tmem + lane_base + CF::T_A + uint32_t(ab) * CF::A_COLS;
#pragma unroll
      for (int kcl = 0; kcl < KCG; ++kcl)
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int kc = kc0 + kcl;
          uint32_t hp[8], mp[8], lp[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 q = v[kcl * 8 + sub * 4 + i];
            const Split3u a = split3x2_trunc(q.x, q.y);
            const Split3u c = split3x2_trunc(q.z, q.w);
            hp[2 * i] = a.h;
            hp[2 * i + 1] = c.h;
            mp[2 * i] = a.m;
            mp[2 * i + 1] = c.m;
            lp[2 * i] = a.l;
            lp[2 * i + 1] = c.l;
          }
          const uint32_t col = a1 + kc * 3 * kPlaneCols + sub * 8;
          tmem_st8(col, hp);
          tmem_st8(col + kPlaneCols, mp);
          tmem_st8(col + 2 * kPlaneCols, lp);
        }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[ab]);
    }
  } else if (warp == kMma) {
    // ---------------- MMA issuer ----------------
    mbar_wait(wbar, 0);
    constexpr uint32_t id = idesc_bf16_m128(D);
    constexpr uint64_t BP = (D * 64) >> 4;
    const uint64_t wd0 = smem_desc(smem_u32(smem));
    int j = 0;
    for (int m = blockIdx.x; m < ntile; m += gridDim.x, ++j) {
      const int ab = j % CF::NA, cb = j % CF::NACC;
      mbar_wait(&a_full[ab], uint32_t(j / CF::NA) & 1u);
      mbar_wait(&acc_empty[cb], (uint32_t(j / CF::NACC) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t a0 = tmem + CF::T_A + uint32_t(ab) * CF::A_COLS;
      const uint32_t acc = tmem + CF::T_ACC + uint32_t(cb) * D;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ah = a0 + kc * 3 * kPlaneCols + ks * 8;
          const uint64_t bd = wd0 + uint64_t((kc * 3 * (D * 64) + ks * 256) >> 4);
          // lo·hi, mid·mid, hi·lo, mid·hi, hi·mid, hi·hi (the GEMM path's order)
          mma_ts_w(acc, ah + 2 * kPlaneCols, bd, id, (kc | ks) ? 1u : 0u);
          mma_ts_w(acc, ah + kPlaneCols, bd + BP, id, 1u);
          mma_ts_w(acc, ah, bd + 2 * BP, id, 1u);
          mma_ts_w(acc, ah + kPlaneCols, bd, id, 1u);
          mma_ts_w(acc, ah, bd + BP, id, 1u);
          mma_ts_w(acc, ah, bd, id, 1u);
        }
      commit_w(&a_empty[ab]);
      commit_w(&acc_full[cb]);
    }
  } else {
    // ---------------- epilogue (warps 0-3, thread = token row) ----------------
    const int quad = warp;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    float* xb = reinterpret_cast<float*>(smem + CF::XB) + quad * 32 * kXPitch;
    const int c4 = (lane & 3) * 4;
    int j = 0;
    for (int m = blockIdx.x; m < ntile; m += gridDim.x, ++j) {
      const int cb = j % CF::NACC;
      mbar_wait(&acc_full[cb], uint32_t(j / CF::NACC) & 1u);
      tc_fence_after();
      const uint32_t tb = tmem + lane_base + CF::T_ACC + uint32_t(cb) * D;
      // LayerNorm with layernorm_row_kernel's arithmetic: sums over float4
      // groups in column order, two TMEM passes for mean and variance
      float sum = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t raw[32];
        tmem_ld32_nowait(tb + uint32_t(c0), raw);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          sum += (__uint_as_float(raw[4 * i]) + __uint_as_float(raw[4 * i + 1])) +
                 (__uint_as_float(raw[4 * i + 2]) + __uint_as_float(raw[4 * i + 3]));
      }
      const float ln_mean = sum / float(D);
      float q = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t raw[32];
        tmem_ld32_nowait(tb + uint32_t(c0), raw);
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
      const float ln_inv = 1.0f / sqrtf(q / float(D) + p.eps);
      const int64_t row0 = int64_t(m) * 128 + quad * 32;
      // the lane's 4 output rows (it * 8 + lane / 4) and 4 channels per 16-wide block
#pragma unroll
      for (int cbk = 0; cbk < D; cbk += 16) {
        float v[16];
        tmem_ld16(tb + uint32_t(cbk), v);
        if (cbk + 16 >= D) {   // accumulator fully read: hand it back
          tc_fence_before();
          mbar_arrive(&acc_empty[cb]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 g4 = __ldg(reinterpret_cast<const float4*>(p.gain + cbk + 4 * c));
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + cbk + 4 * c));
          float4 o = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          o.x -= ln_mean; o.y -= ln_mean; o.z -= ln_mean; o.w -= ln_mean;
          o = make_float4(o.x * ln_inv * g4.x + b4.x, o.y * ln_inv * g4.y + b4.y,
                          o.z * ln_inv * g4.z + b4.z, o.w * ln_inv * g4.w + b4.w);
          *reinterpret_cast<float4*>(xb + lane * kXPitch + 4 * c) = o;
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int ri = it * 8 + (lane >> 2);
          const int64_t row = row0 + ri;
          if (row < p.M)
            *reinterpret_cast<float4*>(p.y + row * D + cbk + c4) =
                *reinterpret_cast<const float4*>(xb + ri * kXPitch + c4);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) tmem_dealloc<CF::TCOLS>(tmem);
}

}  // namespace emb

// Launch when the shape is inside this kernel's envelope; SA_ERR_VALUE
// otherwise (the caller uses the GEMM path).
int embed_ln_launch(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C, int64_t patch,
                    float sub, const void* wpack, int bn, int64_t d, const float* gain,
                    const float* bias, float eps, float* y, cudaStream_t s) {
  using namespace emb;
  const int64_t K = patch * patch * C;
  if (!(d == 32 || d == 64) || bn != d || K > 128 || (patch * C) % 4 != 0 || H != W || H % patch)
    return SA_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(grid) & 15) != 0 || (reinterpret_cast<uintptr_t>(y) & 15) != 0)
    return SA_ERR_VALUE;
  const int KC = int((K + 31) / 32);
  const int64_t side = H / patch, n = side * side;
  Params p{grid, H, W, C, int(patch), int(side), sub, static_cast<const uint16_t*>(wpack), gain, bias,
           eps, y, B * n, int(n), int(K)};
  if (p.M == 0) return SA_OK;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = (p.M + 127) / 128;
  const int grid_n = int(tiles < sms ? tiles : sms);
#define SA_EMB_CASE(DV, KCV)                                                                  \
  if (d == DV && KC == KCV) {                                                                 \
    const int smem = int(Cfg<DV, KCV>::TOTAL);                                                \
    cudaFuncSetAttribute(embed_ln_kernel<DV, KCV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         smem);                                                              \
    embed_ln_kernel<DV, KCV><<<grid_n, Cfg<DV, KCV>::THREADS, smem, s>>>(p);                  \
    count_launch(1);                                                                          \
    SA_LAUNCH_CHECK("embed_ln_kernel");                                                       \
    return SA_OK;                                                                             \
  }
  SA_EMB_CASE(32, 1)
  SA_EMB_CASE(32, 2)
  SA_EMB_CASE(32, 4)
  SA_EMB_CASE(64, 1)
  SA_EMB_CASE(64, 2)
  SA_EMB_CASE(64, 4)
#undef SA_EMB_CASE
  return SA_ERR_VALUE;
}

}  // namespace sa
