// K5 fused: the whole (MoE) MLP  y = [res +] gate · fc2(GELU(fc1(x)))  in one
// persistent tcgen05 kernel; the hidden activations never leave the SM.
//
// Reference: Mlp.forward (model.py:204-208) inside MoeModule.forward
// (model.py:250-274), experts (Mlp(Linear,Linear), Mlp(Shift,Shift))
// (model.py:514-521). Numerics as in tcgemm.cu: x and GELU(h) are split into
// hi/mid/lo bf16 planes (exact), shift weights are exact bf16, dense weights
// three planes; fp32 accumulation in TMEM.
//
// Per 128-token tile of one expert, the hidden dimension is walked in chunks
// of HC = 32: fc1(c) → acc1[c%2] (TMEM) → GELU warps: tcgen05.ld, GELU, split,
// st.shared → A2[c%2] → fc2(c) accumulates acc2[tile%2] (TMEM, d columns).
// Roles (14 warps, one CTA per SM):
//   warps  0-7  GELU + final epilogue (warp e: TMEM lanes 32*(e%4), column half e/4)
//   warps  8-11 producers: gather x rows (MoE permutation), split → A1[tile%2]
//   warp  12    MMA issuer (one thread), order fc1(0) fc1(1) fc2(0) fc1(2) fc2(1) …
//   warp  13    weight streamer: per chunk one bulk copy of the W1 chunk and
//               one of the W2 chunk (pre-packed planes) into a 2-slot ring.
// All double buffers carry full/empty mbarriers; the running chunk counter
// q drives the parities, so tiles of different experts interleave freely.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace tcm {

using namespace tc;

constexpr int HC = 32;                 // hidden chunk (fc1 N, fc2 K)
constexpr int kThreads = 448;
constexpr int kMma = 12, kWarpW = 13;
constexpr uint32_t kPlane32 = 128 * 32 * 2;   // one 128-row x 32-k bf16 plane

struct MlpParams {
  const float* x;
  const int32_t* perm;       // nullptr: identity rows, no grouping
  const int32_t* counts;     // nullptr: one group
  const float* gate;
  const float* residual;
  float* y;
  const uint16_t* w1[2];     // packed (bn = 32) planes per expert
  const uint16_t* w2[2];     // packed (bn = d) planes per expert
  int np[2];                 // planes per expert (3 dense, 1 shift)
  int64_t M;
  int hidden;
};

template <int D>
struct Layout {
  static constexpr int KC1 = D / 32;                                  // fc1 K stages
  static constexpr uint32_t A1 = KC1 * 3 * kPlane32;                  // one A1 buffer
  static constexpr uint32_t W1C = KC1 * 3 * (HC * 32 * 2);            // max W1 chunk bytes
  static constexpr uint32_t W2C = 3 * (D * 32 * 2);                   // max W2 chunk bytes
  static constexpr uint32_t WSLOT = W1C + W2C;
  static constexpr uint32_t A2 = 3 * kPlane32;
  static constexpr uint32_t XB = 8 * 32 * kXPitch * 4;
  static constexpr uint32_t OFF_A1 = 0;
  static constexpr uint32_t OFF_W = OFF_A1 + 2 * A1;
  static constexpr uint32_t OFF_A2 = OFF_W + 2 * WSLOT;
  static constexpr uint32_t OFF_XB = OFF_A2 + 2 * A2;
  static constexpr uint32_t OFF_ROW = OFF_XB + XB;                    // [2][128] int64
  static constexpr uint32_t OFF_BAR = OFF_ROW + 2 * 128 * 8;
  static constexpr uint32_t NBAR = 18;
  static constexpr uint32_t TOTAL = OFF_BAR + NBAR * 8 + 16;
  static constexpr uint32_t TCOLS = 2 * HC + 2 * D <= 128 ? 128 : 256;  // acc1[2] + acc2[2]
};

__device__ __forceinline__ int64_t mlp_tiles(const MlpParams& p, int64_t c0) {
  if (!p.counts) return (p.M + 127) / 128;
  return (c0 + 127) / 128 + (p.M - c0 + 127) / 128;
}
__device__ __forceinline__ void mlp_tile(const MlpParams& p, int64_t c0, int64_t m, int& e,
                                         int64_t& r0, int64_t& r1) {
  if (!p.counts) {
    e = 0;
    r0 = m * 128;
    r1 = min(p.M, r0 + 128);
    return;
  }
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

template <int D>
__global__ void __launch_bounds__(kThreads, 1) mlp_kernel(MlpParams p) {
  using L = Layout<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* a1_full = bar + 0;    // [2] producers → MMA (count 4)
  uint64_t* a1_empty = bar + 2;   // [2] MMA commit → producers
  uint64_t* w_full = bar + 4;     // [2] weight copies (count 1 + tx)
  uint64_t* w_empty = bar + 6;    // [2] MMA commit
  uint64_t* h_full = bar + 8;     // [2] fc1 done (MMA commit)
  uint64_t* h_empty = bar + 10;   // [2] GELU warps finished reading acc1 + wrote A2 (count 256)
  uint64_t* a2_empty = bar + 12;  // [2] fc2 done reading A2 (MMA commit)
  uint64_t* o_full = bar + 14;    // [2] acc2[b] ready (MMA commit)
  uint64_t* o_empty = bar + 16;   // [2] acc2[b] drained by the epilogue (count 256)
  int64_t* rowtab = reinterpret_cast<int64_t*>(smem + L::OFF_ROW);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + L::NBAR * 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kMma) tmem_alloc<L::TCOLS>(tmem_slot);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a1_full[i], 4);
      mbar_init(&a1_empty[i], 1);
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], 256);
      mbar_init(&a2_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 256);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: acc1[s] @ s*HC, acc2[b] @ 2*HC + b*D
  const int64_t c0 = p.counts ? int64_t(p.counts[0]) : 0;
  const int64_t ntile = mlp_tiles(p, c0);
  const int nchunk = p.hidden / HC;

  if (warp >= 8 && warp < 12) {
    // ---------------- producers: x rows → A1 planes ----------------
    const int ptid = tid - 256;
    const int rsub = ptid >> 3, k4 = (ptid & 7) * 4;
    int j = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      mlp_tile(p, c0, m, e, r0, r1);
      if (r0 >= r1) continue;
      const int buf = j & 1;
      const uint32_t ph = uint32_t(j >> 1) & 1u;
      ++j;
      const float* rowp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = r0 + rsub + 16 * i;
        rowp[i] = nullptr;
        if (row < r1) rowp[i] = p.x + (p.perm ? int64_t(__ldg(p.perm + row)) : row) * D;
      }
      float4 v[L::KC1][8];
#pragma unroll
      for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[kc][i] = rowp[i] ? __ldg(reinterpret_cast<const float4*>(rowp[i] + kc * 32 + k4))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
      mbar_wait(&a1_empty[buf], ph ^ 1u);
      uint8_t* a1 = smem + L::OFF_A1 + buf * L::A1;
#pragma unroll
      for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const Split3 a = split3x2(v[kc][i].x, v[kc][i].y);
          const Split3 b = split3x2(v[kc][i].z, v[kc][i].w);
          uint8_t* st = a1 + kc * 3 * kPlane32 + plane_offset(rsub + 16 * i, k4);
          *reinterpret_cast<uint2*>(st) = make_uint2(bf2_bits(a.h), bf2_bits(b.h));
          *reinterpret_cast<uint2*>(st + kPlane32) = make_uint2(bf2_bits(a.m), bf2_bits(b.m));
          *reinterpret_cast<uint2*>(st + 2 * kPlane32) = make_uint2(bf2_bits(a.l), bf2_bits(b.l));
        }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a1_full[buf]);
    }
  } else if (warp == kWarpW) {
    // ---------------- weight streamer ----------------
    if (lane == 0) {
      int64_t q = 0;
      for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
        int e;
        int64_t r0, r1;
        mlp_tile(p, c0, m, e, r0, r1);
        if (r0 >= r1) continue;
        const int np = p.np[e];
        const uint32_t b1 = uint32_t(L::KC1 * np) * (HC * 32 * 2);
        const uint32_t b2 = uint32_t(np) * (D * 32 * 2);
        for (int c = 0; c < nchunk; ++c, ++q) {
          const int s = int(q & 1);
          mbar_wait(&w_empty[s], (uint32_t(q >> 1) & 1u) ^ 1u);
          uint8_t* dst = smem + L::OFF_W + s * L::WSLOT;
          mbar_expect_tx(&w_full[s], b1 + b2);
          bulk_g2s(dst, p.w1[e] + size_t(c) * L::KC1 * np * (HC * 32), b1, &w_full[s]);
          bulk_g2s(dst + L::W1C, p.w2[e] + size_t(c) * np * (D * 32), b2, &w_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMma) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_bf16_m128(HC);
      constexpr uint32_t id2 = idesc_bf16_m128(D);
      const uint8_t pa_tab[6] = {2, 1, 0, 1, 0, 0};
      const uint8_t pb_dense[6] = {0, 1, 2, 0, 1, 0};
      const uint32_t sbase = smem_u32(smem);
      int64_t q = 0;
      int j = 0;
      for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
        int e;
        int64_t r0, r1;
        mlp_tile(p, c0, m, e, r0, r1);
        if (r0 >= r1) continue;
        const int buf = j & 1;                 // A1 buffer and acc2 buffer of this tile
        const uint32_t tph = uint32_t(j >> 1) & 1u;
        ++j;
        const int np = p.np[e];
        const int npairs = np == 1 ? 3 : 6;
        const uint32_t a1 = sbase + L::OFF_A1 + buf * L::A1;
        mbar_wait(&a1_full[buf], tph);
        tc_fence_after();
        auto issue_fc1 = [&](int64_t qq) {
          const int s = int(qq & 1);
          const uint32_t ph = uint32_t(qq >> 1) & 1u;
          mbar_wait(&w_full[s], ph);
          mbar_wait(&h_empty[s], ph ^ 1u);    // acc1[s] read by the GELU warps
          tc_fence_after();
          const uint32_t w1 = sbase + L::OFF_W + s * L::WSLOT;
          const uint32_t d1 = tmem + uint32_t(s * HC);
          for (int kc = 0; kc < L::KC1; ++kc)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              for (int i = 0; i < npairs; ++i) {
                const int pb = np == 1 ? 0 : pb_dense[i];
                const uint64_t ad = smem_desc(a1 + (kc * 3 + pa_tab[i]) * kPlane32 + ks * 256);
                const uint64_t bd =
                    smem_desc(w1 + (kc * np + pb) * (HC * 32 * 2) + ks * 256);
                mma_bf16(d1, ad, bd, id1, (kc | ks | i) != 0 ? 1u : 0u);
              }
          mma_commit(&h_full[s]);
        };
        auto issue_fc2 = [&](int64_t qq, bool first) {
          const int s = int(qq & 1);
          const uint32_t ph = uint32_t(qq >> 1) & 1u;
          if (first) mbar_wait(&o_empty[buf], tph ^ 1u);  // acc2[buf] drained (tile j-2)
          // A2[s] written: the GELU warps arrive h_empty[s] after their A2 stores
          mbar_wait(&h_empty[s], ph);
          tc_fence_after();
          const uint32_t a2 = sbase + L::OFF_A2 + s * L::A2;
          const uint32_t w2 = sbase + L::OFF_W + s * L::WSLOT + L::W1C;
          const uint32_t d2 = tmem + uint32_t(2 * HC + buf * D);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            for (int i = 0; i < npairs; ++i) {
              const int pb = np == 1 ? 0 : pb_dense[i];
              const uint64_t ad = smem_desc(a2 + pa_tab[i] * kPlane32 + ks * 256);
              const uint64_t bd = smem_desc(w2 + pb * (D * 32 * 2) + ks * 256);
              mma_bf16(d2, ad, bd, id2, (!first || ks | i) ? 1u : 0u);
            }
          mma_commit(&a2_empty[s]);
          mma_commit(&w_empty[s]);
        };
        const int64_t q0 = q;
        issue_fc1(q0);
        for (int c = 1; c < nchunk; ++c) {
          issue_fc1(q0 + c);
          issue_fc2(q0 + c - 1, c == 1);
        }
        mma_commit(&a1_empty[buf]);            // all fc1 of the tile issued
        issue_fc2(q0 + nchunk - 1, nchunk == 1);
        mma_commit(&o_full[buf]);
        q += nchunk;
      }
    }
    __syncwarp();
  } else {
    // ---------------- GELU warps + final epilogue (warps 0-7) ----------------
    const int quad = warp & 3, half = warp >> 2;
    const int rl = quad * 32 + lane;
    float* xb = reinterpret_cast<float*>(smem + L::OFF_XB) + warp * 32 * kXPitch;
    int64_t q = 0;
    int j = 0;
    for (int64_t m = blockIdx.x; m < ntile; m += gridDim.x) {
      int e;
      int64_t r0, r1;
      mlp_tile(p, c0, m, e, r0, r1);
      if (r0 >= r1) continue;
      const int ob = j & 1;
      const uint32_t ph_o = uint32_t(j >> 1) & 1u;
      ++j;
      for (int c = 0; c < nchunk; ++c, ++q) {
        const int s = int(q & 1);
        const uint32_t ph = uint32_t(q >> 1) & 1u;
        mbar_wait(&h_full[s], ph);            // fc1(q) done
        mbar_wait(&a2_empty[s], ph ^ 1u);     // fc2(q-2) finished reading A2[s]
        tc_fence_after();
        float v[16];
        tmem_ld16(tmem + (uint32_t(quad * 32) << 16) + uint32_t(s * HC + half * 16), v);
        uint32_t hp[8], mp[8], lp[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const Split3 sp = split3x2(gelu_fast(v[2 * t]), gelu_fast(v[2 * t + 1]));
          hp[t] = bf2_bits(sp.h);
          mp[t] = bf2_bits(sp.m);
          lp[t] = bf2_bits(sp.l);
        }
        uint8_t* a2 = smem + L::OFF_A2 + s * L::A2;
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8) {
          const uint32_t off = plane_offset(rl, half * 16 + h8 * 8);
          *reinterpret_cast<uint4*>(a2 + off) =
              make_uint4(hp[4 * h8], hp[4 * h8 + 1], hp[4 * h8 + 2], hp[4 * h8 + 3]);
          *reinterpret_cast<uint4*>(a2 + kPlane32 + off) =
              make_uint4(mp[4 * h8], mp[4 * h8 + 1], mp[4 * h8 + 2], mp[4 * h8 + 3]);
          *reinterpret_cast<uint4*>(a2 + 2 * kPlane32 + off) =
              make_uint4(lp[4 * h8], lp[4 * h8 + 1], lp[4 * h8 + 2], lp[4 * h8 + 3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&h_empty[s]);
      }
      // ---- final epilogue: acc2 (128 x D) → ×gate → +residual → scatter ----
      const int64_t r = r0 + rl;
      const bool r_ok = r < r1;
      int64_t orow = -1;
      float gt = 1.f;
      if (r_ok) {
        orow = p.perm ? int64_t(__ldg(p.perm + r)) : r;
        if (p.gate) gt = __ldg(p.gate + orow);
      }
      int64_t* rt = rowtab + ob * 128;
      if (half == 0) rt[rl] = orow;
      mbar_wait(&o_full[ob], ph_o);
      tc_fence_after();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      constexpr int HALF = D / 2;
#pragma unroll 1
      for (int cb = 0; cb < HALF; cb += 16) {
        float v[16];
        tmem_ld16(tmem + (uint32_t(quad * 32) << 16) +
                      uint32_t(2 * HC + ob * D + half * HALF + cb), v);
#pragma unroll
        for (int t = 0; t < 16; t += 4)
          *reinterpret_cast<float4*>(xb + lane * kXPitch + t) =
              make_float4(v[t] * gt, v[t + 1] * gt, v[t + 2] * gt, v[t + 3] * gt);
        __syncwarp();
        const int c4 = (lane & 3) * 4;
        const int n = half * HALF + cb + c4;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int ri = it * 8 + (lane >> 2);
          const int64_t orow_i = rt[quad * 32 + ri];
          if (orow_i < 0) continue;
          float4 o = *reinterpret_cast<const float4*>(xb + ri * kXPitch + c4);
          if (p.residual) {
            const float4 rr = __ldg(reinterpret_cast<const float4*>(p.residual + orow_i * D + n));
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
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) tmem_dealloc<L::TCOLS>(tmem);
}

}  // namespace tcm

static int g_sms_mlp = 0;

static int mlp_launch(tcm::MlpParams& p, int d, cudaStream_t s) {
  using namespace tcm;
  if (p.M == 0) return SA_OK;
  if (g_sms_mlp == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_mlp, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = cdiv(p.M, 128) + (p.counts ? 1 : 0);
  const int grid = int(tiles < g_sms_mlp ? tiles : g_sms_mlp);
  if (d == 32) {
    const int smem = int(Layout<32>::TOTAL);
    cudaFuncSetAttribute(mlp_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mlp_kernel<32><<<grid, tcm::kThreads, smem, s>>>(p);
  } else {
    const int smem = int(Layout<64>::TOTAL);
    cudaFuncSetAttribute(mlp_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mlp_kernel<64><<<grid, tcm::kThreads, smem, s>>>(p);
  }
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
