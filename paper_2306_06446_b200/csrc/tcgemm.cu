// K3 / K5 / K6 on the 5th-generation tensor cores: tcgen05.mma with TMEM
// accumulators, float32-faithful.
//
// Precision: every float32 activation is split into hi+mid+lo bf16 planes
// (exact: 3 × 8 significant bits = the 24-bit float32 significand). Shift
// weights s·2^P are EXACT in bf16 (one plane), so a shift-Linear needs three
// bf16 MMAs and every product is exact (ref tests/test_quantize.py:79-85 asks
// for the FakeShift product). Dense (mult-expert) weights are split the same
// way and six plane products (lh, mm, hl, mh, hm, hh) are accumulated,
// dropping only terms below 2^-24 relative. Accumulation is float32 in TMEM.
//
// Kernel (persistent, warp-specialized, one CTA per SM, 288 threads):
//   warps 4-7  producers: per 32-wide K stage, gather their 128 A rows with
//              coalesced 128-bit loads (plain / MoE-permuted / patchified
//              image), split to bf16 planes, store them in the UMMA canonical
//              layout; lane 0 of warp 4 pulls the pre-packed weight planes of
//              the stage with ONE bulk async copy (TMA engine, complete_tx).
//   warp 8     MMA issuer: one elected thread chains tcgen05.mma into a
//              double-buffered TMEM accumulator and commits to mbarriers.
//   warps 0-3  epilogue: tcgen05.ld (thread = accumulator row), GELU / ×gate,
//              transpose through shared memory so every store (and residual /
//              position-embedding load) is a coalesced row segment, scatter
//              the MoE rows back to token order.
// A ring of S shared-memory stages (full/empty mbarriers) and two TMEM
// accumulators (tfull/tempty) let loads, MMAs and epilogues of successive
// tiles overlap. The tile list is a static stride over (m-tile, n-tile);
// with MoE grouping the m-tiles of each expert are derived from the device
// counts, so nothing syncs the host (CUDA-graph capturable).
//
// Weight packing (sa_weight_pack): for n-tile nt, K stage kc, plane p the
// packed image is the exact shared-memory layout (see tc_common.cuh), so a
// stage is one contiguous bulk copy.
#include "tc_common.cuh"

namespace sa {
namespace tc {

constexpr int kBM = 128;
constexpr int kThreads = 416;
constexpr uint32_t kPlaneA = kBM * kBK * 2;  // bytes per A plane
constexpr int kXPitch = 20;                   // transpose buffer pitch (floats, 16B rows)

enum AMode { A_PLAIN = 0, A_GATHER = 1, A_PATCH = 2 };

struct TcParams {
  const float* A;
  int64_t lda;
  const int32_t* a_rows;
  int64_t pH, pW, pC, patch, pside;
  float sub;
  const uint16_t* Bp[2];
  int nplanes[2];
  int64_t M, K, N;
  int kchunks;
  int ntiles;
  int stages;
  const int32_t* counts;
  float* C;
  const int32_t* c_rows;
  const float* gate;
  const float* residual;
  int act;
  const float* pos;
  int64_t img_tokens;
  int extra;
};

template <int BN>
struct TmemCols {  // two accumulator buffers, power of two >= 32
  static constexpr uint32_t value = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                    : 2 * BN <= 256 ? 256 : 512;
};

struct TileInfo {
  int group;
  int64_t r0, r1;
  int n_tile;
};

// m-tiles: with grouping, expert 0 owns ceil(c0/128) tiles, expert 1 the rest
__device__ __forceinline__ int64_t num_m_tiles(const TcParams& p, int64_t c0) {
  if (!p.counts) return (p.M + kBM - 1) / kBM;
  return (c0 + kBM - 1) / kBM + (p.M - c0 + kBM - 1) / kBM;
}
__device__ __forceinline__ TileInfo tile_info(const TcParams& p, int64_t c0, int64_t t) {
  TileInfo ti;
  const int64_t m = t / p.ntiles;
  ti.n_tile = int(t % p.ntiles);
  if (!p.counts) {
    ti.group = 0;
    ti.r0 = m * kBM;
    ti.r1 = min(p.M, ti.r0 + kBM);
    return ti;
  }
  const int64_t t0 = (c0 + kBM - 1) / kBM;
  if (m < t0) {
    ti.group = 0;
    ti.r0 = m * kBM;
    ti.r1 = min(c0, ti.r0 + kBM);
  } else {
    ti.group = 1;
    ti.r0 = c0 + (m - t0) * kBM;
    ti.r1 = min(p.M, ti.r0 + kBM);
  }
  return ti;
}

__device__ __forceinline__ float gelu_fast(float x) {
  // 0.5·x·(1 + tanh(u)) == x / (1 + exp(-2u)); ex2.approx + fast divide keep
  // ~1e-7 relative accuracy (the reference's tanh is itself a float32 libm call)
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float u = c * (x + a * (x * x * x));
  return __fdividef(x, 1.0f + __expf(-2.0f * u));
}

template <int BN, int AM>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm_kernel(TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  constexpr uint32_t kPlaneB = BN * kBK * 2;
  const int S = p.stages;
  const int npb_max = max(p.nplanes[0], p.counts ? p.nplanes[1] : 0);
  const uint32_t stage_bytes = 3 * kPlaneA + uint32_t(npb_max) * kPlaneB;
  float* xbuf = reinterpret_cast<float*>(smem + size_t(S) * stage_bytes);      // [4][32][33]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<int64_t*>(xbuf + 8 * 32 * kXPitch) + 256);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = bars + 2 * S + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 12) tmem_alloc<TCOLS>(tmem_slot);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 4);     // four producer warps
      mbar_init(&empty[s], 1);    // one MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);    // one MMA commit
      mbar_init(&tempty[b], 256); // every epilogue thread
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t c0 = p.counts ? int64_t(p.counts[0]) : 0;
  const int64_t total = num_m_tiles(p, c0) * p.ntiles;

  if (warp >= 8 && warp < 12) {
    // ================= producers =================
    const int ptid = tid - 256;
    const int rsub = ptid >> 3;          // row within each 16-row slab
    const int k4 = (ptid & 7) * 4;       // k offset within the 32-wide stage
    const int64_t pcw = p.patch * p.pC;
    int s = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const TileInfo ti = tile_info(p, c0, t);
      if (ti.r0 >= ti.r1) continue;
      const int npb = p.nplanes[ti.group];
      const uint16_t* Bg = p.Bp[ti.group] + size_t(ti.n_tile) * p.kchunks * npb * (BN * kBK);
      const uint32_t bbytes = uint32_t(npb) * kPlaneB;
      const float* rowp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = ti.r0 + rsub + 16 * i;
        rowp[i] = nullptr;
        if (row < ti.r1) {
          if (AM == A_PLAIN) {
            rowp[i] = p.A + row * p.lda;
          } else if (AM == A_GATHER) {
            rowp[i] = p.A + int64_t(__ldg(p.a_rows + row)) * p.lda;
          } else {
            const int64_t tpi = p.pside * p.pside;
            const int64_t b = row / tpi, tt = row % tpi;
            const int64_t py = tt / p.pside, px = tt % p.pside;
            rowp[i] = p.A + ((b * p.pH + py * p.patch) * p.pW + px * p.patch) * p.pC;
          }
        }
      }
      for (int kc = 0; kc < p.kchunks; ++kc) {
        mbar_wait(&empty[s], phase ^ 1u);
        uint8_t* st = smem + size_t(s) * stage_bytes;
        if (ptid == 0) {
          mbar_add_tx(&full[s], bbytes);
          bulk_g2s(st + 3 * kPlaneA, Bg + size_t(kc) * npb * (BN * kBK), bbytes, &full[s]);
        }
        const int64_t k = int64_t(kc) * kBK + k4;
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rowp[i] != nullptr && k < p.K) {
            const float* src = (AM == A_PATCH)
                                   ? rowp[i] + (k / pcw) * (p.pW * p.pC) + (k % pcw)
                                   : rowp[i] + k;
            v[i] = __ldg(reinterpret_cast<const float4*>(src));
            if (AM == A_PATCH) {
              v[i].x -= p.sub; v[i].y -= p.sub; v[i].z -= p.sub; v[i].w -= p.sub;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const Split3 a = split3x2(v[i].x, v[i].y);
          const Split3 b = split3x2(v[i].z, v[i].w);
          const uint32_t off = plane_offset(rsub + 16 * i, k4);
          *reinterpret_cast<uint2*>(st + off) = make_uint2(bf2_bits(a.h), bf2_bits(b.h));
          *reinterpret_cast<uint2*>(st + kPlaneA + off) = make_uint2(bf2_bits(a.m), bf2_bits(b.m));
          *reinterpret_cast<uint2*>(st + 2 * kPlaneA + off) =
              make_uint2(bf2_bits(a.l), bf2_bits(b.l));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (++s == S) {
          s = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 12) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_m128(BN);
      const uint8_t pa_tab[6] = {2, 1, 0, 1, 0, 0};
      const uint8_t pb_dense[6] = {0, 1, 2, 0, 1, 0};
      const uint32_t smem_base = smem_u32(smem);
      int s = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        const TileInfo ti = tile_info(p, c0, t);
        if (ti.r0 >= ti.r1) continue;
        const int npb = p.nplanes[ti.group];
        const int npairs = npb == 1 ? 3 : 6;
        mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(acc * BN);
        for (int kc = 0; kc < p.kchunks; ++kc) {
          mbar_wait(&full[s], phase);
          tc_fence_after();
          const uint32_t sa = smem_base + uint32_t(s) * stage_bytes;
          const uint32_t sb = sa + 3 * kPlaneA;
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {
            for (int i = 0; i < npairs; ++i) {
              const int pb = npb == 1 ? 0 : pb_dense[i];
              const uint64_t ad = smem_desc(sa + pa_tab[i] * kPlaneA + ks * 256);
              const uint64_t bd = smem_desc(sb + pb * kPlaneB + ks * 256);
              mma_bf16(d_tmem, ad, bd, idesc, (kc | ks | i) != 0 ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (++s == S) {
            s = 0;
            phase ^= 1u;
          }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue (warps 0-7): warp e reads TMEM lanes 32*(e%4).. (its rows)
    // and the column half e/4 of the tile; thread = accumulator row. =====
    const int quad = warp & 3, half = warp >> 2;
    float* xb = xbuf + warp * 32 * kXPitch;                 // [32 rows][kXPitch]
    int64_t* orow_s = reinterpret_cast<int64_t*>(xbuf + 8 * 32 * kXPitch);  // [2][128]
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec4 = (p.N & 3) == 0;
    constexpr int HALF = BN / 2;   // columns per warp (multiple of 16)
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const TileInfo ti = tile_info(p, c0, t);
      if (ti.r0 >= ti.r1) continue;
      const int rl = quad * 32 + lane;             // row within the tile
      const int64_t r = ti.r0 + rl;
      const bool r_ok = r < ti.r1;
      int64_t orow = -1, pos_idx = 0;
      float g = 1.f;
      if (r_ok) {
        orow = p.c_rows ? int64_t(__ldg(p.c_rows + r)) : r;
        if (p.img_tokens > 0) {
          const int64_t b = r / p.img_tokens, tt = r % p.img_tokens;
          orow = b * (p.img_tokens + p.extra) + p.extra + tt;
          pos_idx = p.extra + tt;
        }
        if (p.gate) g = __ldg(p.gate + orow);
      }
      int64_t* orow_t = orow_s + acc * 128;
      if (half == 0) orow_t[rl] = p.pos ? (orow | (pos_idx << 40)) : orow;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_base =
          tmem + (uint32_t(quad * 32) << 16) + uint32_t(acc * BN + half * HALF);
      const int64_t n_base = int64_t(ti.n_tile) * BN + half * HALF;
      // the orow table of this tile is complete once all epilogue warps are here
      asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll 1
      for (int cb = 0; cb < HALF; cb += 16) {
        float v[16];
        tmem_ld16(t_base + uint32_t(cb), v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float o = v[j];
          if (p.act == 1) o = gelu_fast(o);
          if (p.gate) o = o * g;
          v[j] = o;
        }
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(xb + lane * kXPitch + j) =
              make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
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
              const float4 q =
                  __ldg(reinterpret_cast<const float4*>(p.residual + orow_i * p.N + n));
              o = make_float4(q.x + o.x, q.y + o.y, q.z + o.z, q.w + o.w);
            }
            *reinterpret_cast<float4*>(p.C + orow_i * p.N + n) = o;
          } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (n + j >= p.N) break;
              float e = ov[j];
              if (p.pos) e = e + __ldg(p.pos + pos_i * p.N + n + j);
              if (p.residual) e = __ldg(p.residual + orow_i * p.N + n + j) + e;
              p.C[orow_i * p.N + n + j] = e;
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) tmem_dealloc<TCOLS>(tmem);
}

// ---- weight packing ---------------------------------------------------------
__global__ void weight_pack_kernel(const void* __restrict__ w, int kind, int64_t K, int64_t N,
                                   int p_min, int BN, int kchunks, int np, int64_t total,
                                   uint16_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  // i enumerates (nt, kc, plane, n_local, k_local) in natural order
  const int64_t k_local = i % kBK;
  int64_t t = i / kBK;
  const int64_t n_local = t % BN;
  t /= BN;
  const int pl = int(t % np);
  t /= np;
  const int64_t kc = t % kchunks;
  const int64_t nt = t / kchunks;
  const int64_t k = kc * kBK + k_local, n = nt * BN + n_local;
  float val = 0.f;
  if (k < K && n < N) {
    if (kind == SA_W_SHIFT) {
      val = decode_shift(static_cast<const uint8_t*>(w)[k * N + n], p_min);
    } else {
      val = static_cast<const float*>(w)[k * N + n];
    }
  }
  __nv_bfloat16 h = __float2bfloat16_rn(val);
  float r1 = val - __bfloat162float(h);
  __nv_bfloat16 m = __float2bfloat16_rn(r1);
  __nv_bfloat16 l = __float2bfloat16_rn(r1 - __bfloat162float(m));
  const __nv_bfloat16 sel = pl == 0 ? h : (pl == 1 ? m : l);
  const size_t stage = size_t((nt * kchunks + kc) * np + pl) * (size_t(BN) * kBK);
  const size_t off = stage + plane_offset(int(n_local), int(k_local)) / 2;
  out[off] = *reinterpret_cast<const uint16_t*>(&sel);
}

}  // namespace tc

static int tc_tile_n_ok(int bn) {
  return bn == 32 || bn == 64 || bn == 128 || bn == 160 || bn == 256;
}

static int g_num_sms = 0;

static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

static int launch_tc(tc::TcParams& p, int amode, int bn, int64_t m_tiles_max, cudaStream_t s) {
  using namespace tc;
  if (p.M == 0) return SA_OK;
  p.ntiles = int(cdiv(p.N, bn));
  const int npb_max = max(p.nplanes[0], p.counts ? p.nplanes[1] : 0);
  const size_t stage_bytes = 3 * size_t(kPlaneA) + size_t(npb_max) * bn * kBK * 2;
  const size_t fixed = 8 * 32 * kXPitch * sizeof(float) + 256 * 8 + (2 * 8 + 4) * 8 + 16;
  const size_t budget = 220 * 1024;
  int stages = int((budget - fixed) / stage_bytes);
  stages = stages > 4 ? 4 : stages;
  if (stages < 2) {
    set_error("tensor-core stage does not fit shared memory (bn=%d)", bn);
    return SA_ERR_VALUE;
  }
  p.stages = stages;
  const size_t smem = size_t(stages) * stage_bytes + fixed;
  const int64_t tiles = m_tiles_max * p.ntiles;
  const int grid = int(tiles < num_sms() ? tiles : num_sms());
#define SA_TC_CASE(BNV)                                                                          \
  case BNV: {                                                                                    \
    auto kfn = amode == A_PLAIN    ? tc_gemm_kernel<BNV, A_PLAIN>                               \
               : amode == A_GATHER ? tc_gemm_kernel<BNV, A_GATHER>                              \
                                   : tc_gemm_kernel<BNV, A_PATCH>;                              \
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));          \
    kfn<<<grid, kThreads, smem, s>>>(p);                                                         \
  } break;
  switch (bn) {
    SA_TC_CASE(32)
    SA_TC_CASE(64)
    SA_TC_CASE(128)
    SA_TC_CASE(160)
    SA_TC_CASE(256)
    default:
      set_error("tensor-core tile N=%d unsupported", bn);
      return SA_ERR_VALUE;
  }
#undef SA_TC_CASE
  count_launch(1);
  SA_LAUNCH_CHECK("tc_gemm_kernel");
  return SA_OK;
}

static tc::TcParams tc_base(int64_t M, int64_t K, int64_t N) {
  tc::TcParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.K = K;
  p.N = N;
  p.lda = K;
  p.kchunks = int(cdiv(K, tc::kBK));
  return p;
}

static int nplanes_of(int kind) { return kind == SA_W_SHIFT ? 1 : 3; }

}  // namespace sa

using namespace sa;

extern "C" int sa_tc_tile_n(int64_t N) {
  if (N <= 256) {
    for (int bn : {32, 64, 128, 160, 256})
      if (N <= bn) return bn;
  }
  if (N % 256 == 0) return 256;
  if (N % 160 == 0) return 160;
  if (N % 128 == 0) return 128;
  return 256;
}

extern "C" size_t sa_weight_pack_bytes(int64_t K, int64_t N, int w_kind, int bn) {
  const int64_t kchunks = cdiv(K, tc::kBK), ntiles = cdiv(N, bn);
  return size_t(ntiles * kchunks * nplanes_of(w_kind)) * size_t(bn) * tc::kBK * 2;
}

extern "C" int sa_weight_pack(const void* w, int w_kind, int64_t K, int64_t N, int p_min, int bn,
                              void* out, void* stream) {
  SA_REQUIRE(w_kind == SA_W_DENSE || w_kind == SA_W_SHIFT, SA_ERR_VALUE,
             "sa_weight_pack: unknown weight kind %d", w_kind);
  SA_REQUIRE(tc_tile_n_ok(bn), SA_ERR_VALUE, "sa_weight_pack: tile N=%d unsupported", bn);
  SA_REQUIRE(K > 0 && N > 0, SA_ERR_SHAPE, "sa_weight_pack: empty weight");
  const int kchunks = int(cdiv(K, tc::kBK));
  const int np = nplanes_of(w_kind);
  const int64_t total = cdiv(N, bn) * kchunks * np * int64_t(bn) * tc::kBK;
  tc::weight_pack_kernel<<<unsigned(cdiv(total, 256)), 256, 0, as_stream(stream)>>>(
      w, w_kind, K, N, p_min, bn, kchunks, np, total, static_cast<uint16_t*>(out));
  count_launch(1);
  SA_LAUNCH_CHECK("sa_weight_pack");
  return SA_OK;
}

static int tc_check(const char* who, int64_t M, int64_t K, int64_t N, int bn) {
  SA_REQUIRE(M >= 0 && K > 0 && N > 0, SA_ERR_SHAPE, "%s: bad extents", who);
  SA_REQUIRE(K % 4 == 0, SA_ERR_SHAPE, "%s: K=%lld must be a multiple of 4", who, (long long)K);
  SA_REQUIRE(tc_tile_n_ok(bn), SA_ERR_VALUE, "%s: tile N=%d unsupported", who, bn);
  return SA_OK;
}

extern "C" int sa_tc_linear(const float* x, const void* wpack, int w_kind, int bn, float* y,
                            int64_t M, int64_t K, int64_t N, const float* residual, int act,
                            void* stream) {
  if (int st = tc_check("sa_tc_linear", M, K, N, bn)) return st;
  tc::TcParams p = tc_base(M, K, N);
  p.A = x;
  p.Bp[0] = static_cast<const uint16_t*>(wpack);
  p.nplanes[0] = nplanes_of(w_kind);
  p.C = y;
  p.residual = residual;
  p.act = act;
  return launch_tc(p, tc::A_PLAIN, bn, cdiv(M, tc::kBM), as_stream(stream));
}

extern "C" int sa_tc_moe_linear(const float* x, const int32_t* perm, const int32_t* counts,
                                const float* gate, const void* wpack_dense,
                                const void* wpack_shift, int bn, float* y, const float* residual,
                                int64_t M, int64_t K, int64_t N, void* stream) {
  if (int st = tc_check("sa_tc_moe_linear", M, K, N, bn)) return st;
  tc::TcParams p = tc_base(M, K, N);
  p.A = x;
  p.a_rows = perm;
  p.Bp[0] = static_cast<const uint16_t*>(wpack_dense);
  p.nplanes[0] = 3;
  p.Bp[1] = static_cast<const uint16_t*>(wpack_shift);
  p.nplanes[1] = 1;
  p.counts = counts;
  p.C = y;
  p.c_rows = perm;
  p.gate = gate;
  p.residual = residual;
  return launch_tc(p, tc::A_GATHER, bn, cdiv(M, tc::kBM) + 1, as_stream(stream));
}

extern "C" size_t sa_tc_mlp_workspace(int64_t M, int64_t hidden) {
  return size_t(M) * size_t(hidden) * sizeof(float);
}

extern "C" int sa_tc_mlp(const float* x, const void* w1pack, int w1_kind, int bn1,
                         const void* w2pack, int w2_kind, int bn2, float* y, int64_t M, int64_t d,
                         int64_t hidden, const float* residual, void* ws, size_t ws_bytes,
                         void* stream) {
  SA_REQUIRE(ws_bytes >= sa_tc_mlp_workspace(M, hidden), SA_ERR_VALUE,
             "sa_tc_mlp: workspace too small");
  float* h = static_cast<float*>(ws);
  int st = sa_tc_linear(x, w1pack, w1_kind, bn1, h, M, d, hidden, nullptr, 1, stream);
  if (st) return st;
  return sa_tc_linear(h, w2pack, w2_kind, bn2, y, M, hidden, d, residual, 0, stream);
}

extern "C" int sa_tc_moe_mlp(const float* x, const int32_t* perm, const int32_t* counts,
                             const float* gate, const void* w1_dense, const void* w2_dense,
                             const void* w1_shift, const void* w2_shift, int bn1, int bn2,
                             float* y, const float* residual, int64_t M, int64_t d, int64_t hidden,
                             void* ws, size_t ws_bytes, void* stream) {
  if (int st = tc_check("sa_tc_moe_mlp", M, d, hidden, bn1)) return st;
  if (int st = tc_check("sa_tc_moe_mlp", M, hidden, d, bn2)) return st;
  SA_REQUIRE(ws_bytes >= sa_tc_mlp_workspace(M, hidden), SA_ERR_VALUE,
             "sa_tc_moe_mlp: workspace too small");
  float* h = static_cast<float*>(ws);
  cudaStream_t s = as_stream(stream);
  tc::TcParams p1 = tc_base(M, d, hidden);
  p1.A = x;
  p1.a_rows = perm;
  p1.Bp[0] = static_cast<const uint16_t*>(w1_dense);
  p1.nplanes[0] = 3;
  p1.Bp[1] = static_cast<const uint16_t*>(w1_shift);
  p1.nplanes[1] = 1;
  p1.counts = counts;
  p1.C = h;
  p1.act = 1;
  int st = launch_tc(p1, tc::A_GATHER, bn1, cdiv(M, tc::kBM) + 1, s);
  if (st) return st;
  tc::TcParams p2 = tc_base(M, hidden, d);
  p2.A = h;
  p2.Bp[0] = static_cast<const uint16_t*>(w2_dense);
  p2.nplanes[0] = 3;
  p2.Bp[1] = static_cast<const uint16_t*>(w2_shift);
  p2.nplanes[1] = 1;
  p2.counts = counts;
  p2.C = y;
  p2.c_rows = perm;
  p2.gate = gate;
  p2.residual = residual;
  return launch_tc(p2, tc::A_PLAIN, bn2, cdiv(M, tc::kBM) + 1, s);
}

extern "C" int sa_tc_patch_embed(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                                 int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                                 const float* cls, const float* pos, float* y, void* stream) {
  SA_REQUIRE(B > 0 && H > 0 && W > 0 && C > 0 && patch > 0 && d > 0, SA_ERR_SHAPE,
             "sa_tc_patch_embed: bad extents");
  SA_REQUIRE(H % patch == 0 && W % patch == 0 && H == W, SA_ERR_SHAPE,
             "sa_tc_patch_embed: square image side %lld not divisible by patch %lld",
             (long long)H, (long long)patch);
  SA_REQUIRE((patch * C) % 4 == 0, SA_ERR_SHAPE,
             "sa_tc_patch_embed: patch*C must be a multiple of 4");
  const int64_t side = H / patch;
  const int64_t n = side * side;
  const int64_t K = patch * patch * C;
  if (int st = tc_check("sa_tc_patch_embed", B * n, K, d, bn)) return st;
  tc::TcParams p = tc_base(B * n, K, d);
  p.A = grid;
  p.pH = H;
  p.pW = W;
  p.pC = C;
  p.patch = patch;
  p.pside = side;
  p.sub = sub;
  p.Bp[0] = static_cast<const uint16_t*>(wpack);
  p.nplanes[0] = 3;
  p.C = y;
  p.pos = pos;
  p.img_tokens = n;
  p.extra = cls ? 1 : 0;
  cudaStream_t s = as_stream(stream);
  int st = launch_tc(p, tc::A_PATCH, bn, cdiv(B * n, tc::kBM), s);
  if (st) return st;
  if (cls) return write_cls_rows(cls, pos, y, B, n + 1, d, s);
  return SA_OK;
}
