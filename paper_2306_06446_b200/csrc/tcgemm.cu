// K3 / K5 / K6 on the 5th-generation tensor cores: tcgen05.mma with TMEM
// accumulators, float32-faithful.
//
// Precision: every float32 activation is split into hi+mid+lo bf16 planes
// (exact: 3 × 8 significant bits = the 24-bit float32 significand). Shift
// weights s·2^P are EXACT in bf16 (one plane), so a shift-Linear needs three
// bf16 MMAs and every product is exact — the result equals the float32 sum of
// exact products (ref tests/test_quantize.py:79-85 asks for exactly that).
// Dense (mult-expert) weights are split the same way and six plane products
// (hh, hm, mh, hl, mm, lh) are accumulated, dropping only terms below 2^-24
// relative. Accumulation is float32 in TMEM.
//
// Kernel: one 128-row output tile per CTA (4 warps). Per 32-wide K stage:
// thread 0 pulls the pre-packed weight planes into shared memory with one
// bulk async copy (TMA engine, mbarrier complete_tx) while all 128 threads
// gather their A row (plain / MoE-permuted / patchified image), split it and
// store the three planes in the UMMA canonical layout; one elected thread then
// issues the tcgen05.mma chain and commits to an mbarrier. The epilogue reads
// the accumulator with tcgen05.ld (thread = row) and applies GELU / ×gate /
// +residual / +pos / row scatter before the store. Several CTAs per SM overlap
// one tile's epilogue with another tile's MMAs.
//
// Weight packing (sa_weight_pack): for n-tile nt, K stage kc, plane p the
// packed image is the exact shared-memory layout (see tc_common.cuh), so a
// stage is one contiguous bulk copy.
#include "tc_common.cuh"

namespace sa {
namespace tc {

constexpr int kThreads = 128;
constexpr int kBM = 128;
constexpr uint32_t kPlaneA = kBM * kBK * 2;  // bytes per A plane

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
struct TmemCols {
  static constexpr uint32_t value = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

template <int BN, int AM>
__global__ void __launch_bounds__(kThreads) tc_gemm_kernel(TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 3 * kPlaneA;
  __shared__ __align__(8) uint64_t bar_b;
  __shared__ __align__(8) uint64_t bar_mma;
  __shared__ uint32_t tmem_slot;
  constexpr uint32_t TCOLS = TmemCols<BN>::value;
  constexpr uint32_t kPlaneB = BN * kBK * 2;

  // ---- tile scheduling (MoE grouping reads the device-side counts) ----
  int group = 0;
  int64_t r0, r1;
  if (p.counts) {
    const int64_t c0 = p.counts[0];
    const int64_t t0 = (c0 + kBM - 1) / kBM;
    if (blockIdx.x < t0) {
      r0 = int64_t(blockIdx.x) * kBM;
      r1 = min(c0, r0 + kBM);
    } else {
      group = 1;
      r0 = c0 + (int64_t(blockIdx.x) - t0) * kBM;
      r1 = min(p.M, r0 + kBM);
    }
  } else {
    r0 = int64_t(blockIdx.x) * kBM;
    r1 = min(p.M, r0 + kBM);
  }
  if (r0 >= r1) return;  // uniform for the whole CTA, before any TMEM use

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<TCOLS>(&tmem_slot);
  if (tid == 0) {
    mbar_init(&bar_b, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  // ---- A row source ----
  const int64_t arow = r0 + tid;
  const bool a_ok = arow < r1;
  const float* abase = nullptr;
  int64_t prs = 0;
  if (a_ok) {
    if (AM == A_PLAIN) {
      abase = p.A + arow * p.lda;
    } else if (AM == A_GATHER) {
      abase = p.A + int64_t(p.a_rows[arow]) * p.lda;
    } else {
      const int64_t tpi = p.pside * p.pside;
      const int64_t b = arow / tpi, t = arow % tpi;
      const int64_t py = t / p.pside, px = t % p.pside;
      abase = p.A + ((b * p.pH + py * p.patch) * p.pW + px * p.patch) * p.pC;
      prs = p.pW * p.pC;
    }
  }
  const int64_t pcw = p.patch * p.pC;
  const int npb = p.nplanes[group];
  const int64_t n_tile = blockIdx.y;
  const uint16_t* Bg = p.Bp[group] + size_t(n_tile) * p.kchunks * npb * (BN * kBK);
  const uint32_t bbytes = uint32_t(npb) * kPlaneB;
  constexpr uint32_t idesc = idesc_bf16_m128(BN);
  // plane products: shift (1 B plane) → (0,0),(1,0),(2,0); dense → 6 terms
  const int npairs = npb == 1 ? 3 : 6;
  const uint8_t pa_tab[6] = {2, 1, 0, 1, 0, 0};
  const uint8_t pb_dense[6] = {0, 1, 2, 0, 1, 0};

  const uint32_t sA_u32 = smem_u32(sA), sB_u32 = smem_u32(sB);
  for (int kc = 0; kc < p.kchunks; ++kc) {
    const uint32_t ph = uint32_t(kc) & 1u;
    if (tid == 0) {
      mbar_expect_tx(&bar_b, bbytes);
      bulk_g2s(sB, Bg + size_t(kc) * npb * (BN * kBK), bbytes, &bar_b);
    }
    // A: this thread's row, 32 k values → 3 bf16 planes
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float f[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t k = int64_t(kc) * kBK + q * 8 + h * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a_ok && k < p.K) {
          const float* src = (AM == A_PATCH) ? abase + (k / pcw) * prs + (k % pcw) : abase + k;
          v = __ldg(reinterpret_cast<const float4*>(src));
          if (AM == A_PATCH) {
            v.x -= p.sub; v.y -= p.sub; v.z -= p.sub; v.w -= p.sub;
          }
        }
        f[h * 4 + 0] = v.x; f[h * 4 + 1] = v.y; f[h * 4 + 2] = v.z; f[h * 4 + 3] = v.w;
      }
      uint4 ph4[3];
      uint32_t* hp = reinterpret_cast<uint32_t*>(&ph4[0]);
      uint32_t* mp = reinterpret_cast<uint32_t*>(&ph4[1]);
      uint32_t* lp = reinterpret_cast<uint32_t*>(&ph4[2]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const Split3 s = split3x2(f[2 * j], f[2 * j + 1]);
        hp[j] = bf2_bits(s.h);
        mp[j] = bf2_bits(s.m);
        lp[j] = bf2_bits(s.l);
      }
      const uint32_t off = plane_offset(tid, q * 8);
#pragma unroll
      for (int pl = 0; pl < 3; ++pl)
        *reinterpret_cast<uint4*>(sA + pl * kPlaneA + off) = ph4[pl];
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&bar_b, ph);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kBK / 16; ++ks) {
        for (int i = 0; i < npairs; ++i) {
          const int pa = pa_tab[i];
          const int pb = npb == 1 ? 0 : pb_dense[i];
          const uint64_t ad = smem_desc(sA_u32 + pa * kPlaneA + ks * 256);
          const uint64_t bd = smem_desc(sB_u32 + pb * kPlaneB + ks * 256);
          mma_bf16(tmem, ad, bd, idesc, (kc | ks | i) != 0 ? 1u : 0u);
        }
      }
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph);
  }
  tc_fence_after();

  // ---- epilogue: thread = accumulator row ----
  const int64_t r = r0 + warp * 32 + lane;
  const bool r_ok = r < r1;
  int64_t orow = 0, pos_idx = 0;
  float g = 1.f;
  if (r_ok) {
    orow = p.c_rows ? int64_t(p.c_rows[r]) : r;
    if (p.img_tokens > 0) {
      const int64_t b = r / p.img_tokens, t = r % p.img_tokens;
      orow = b * (p.img_tokens + p.extra) + p.extra + t;
      pos_idx = p.extra + t;
    }
    if (p.gate) g = p.gate[orow];
  }
  const int64_t n_base = n_tile * BN;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
    if (!r_ok) continue;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t n = n_base + c0 + j;
      if (n >= p.N) continue;
      float o = v[j];
      if (p.act == 1) o = gelu_tanh(o);
      if (p.gate) o = o * g;
      if (p.pos) o = o + p.pos[pos_idx * p.N + n];
      if (p.residual) o = p.residual[orow * p.N + n] + o;
      p.C[orow * p.N + n] = o;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<TCOLS>(tmem);
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

static int launch_tc(tc::TcParams& p, int amode, int bn, int64_t m_tiles, cudaStream_t s) {
  using namespace tc;
  if (p.M == 0) return SA_OK;
  const int ntiles = int(cdiv(p.N, bn));
  dim3 grid((unsigned)m_tiles, (unsigned)ntiles, 1u);
  const int npb_max = max(p.nplanes[0], p.counts ? p.nplanes[1] : 0);
  size_t smem = 3 * size_t(kPlaneA) + size_t(npb_max) * bn * kBK * 2;
  if (bn > 128) smem = max(smem, size_t(80 * 1024));  // ≤ 2 CTAs/SM: 2 × 256 TMEM columns
  else if (bn == 128) smem = max(smem, size_t(50 * 1024));  // ≤ 4 CTAs/SM: 4 × 128 columns
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
      if (N <= bn && (bn == N || bn >= N)) return bn;
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
