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
// Kernel: persistent and warp-specialized (tc_gemm_kernel.cuh) — two producer
// groups gather/split A and bulk-copy B into a shared-memory ring, one thread
// issues tcgen05.mma into two TMEM accumulators, two epilogue groups drain
// them; alternate tiles go to alternate groups so two tiles are in flight.
// The tile list is a static stride over (m-tile, n-tile); with MoE grouping
// the m-tiles of each expert are derived from the device counts, so nothing
// syncs the host (CUDA-graph capturable).
//
// Weight packing (sa_weight_pack): for n-tile nt, K stage kc, plane p the
// packed image is the exact shared-memory layout (see tc_common.cuh), so a
// stage is one contiguous bulk copy.
#include "tc_gemm_kernel.cuh"

namespace sa {
namespace tc {

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

#ifdef SA_DEBUG
// debug: gelu_fast2 / split3x2 against their scalar forms on n patterned
// inputs spanning [-16, 16] and the float edge values; counts mismatching bits
__global__ void gelu_pair_check_kernel(int64_t n, unsigned long long* bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t h = uint32_t(i) * 2654435761u;
  float a = (float(h >> 8) / 16777216.0f - 0.5f) * 32.0f;
  float b = __uint_as_float(h);   // arbitrary bit patterns (incl. huge / tiny / inf / nan)
  if (!isfinite(b)) b = -a;
  float p0 = a, p1 = b;
  tc::gelu_fast2(p0, p1);
  const float s0 = tc::gelu_fast(a), s1 = tc::gelu_fast(b);
  const tc::Split3 sp = tc::split3x2(a, b);
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h2);
  const float ra = a - hf.x, rb = b - hf.y;
  const __nv_bfloat162 m2 = __floats2bfloat162_rn(ra, rb);
  const float2 mf = __bfloat1622float2(m2);
  const __nv_bfloat162 l2 = __floats2bfloat162_rn(ra - mf.x, rb - mf.y);
  const bool ok = __float_as_uint(p0) == __float_as_uint(s0) &&
                  __float_as_uint(p1) == __float_as_uint(s1) &&
                  tc::bf2_bits(sp.h) == tc::bf2_bits(h2) && tc::bf2_bits(sp.m) == tc::bf2_bits(m2) &&
                  tc::bf2_bits(sp.l) == tc::bf2_bits(l2);
  if (!ok) atomicAdd(bad, 1ull);
}

extern "C" int sa_debug_gelu_pair_check(int64_t n, unsigned long long* bad_dev, void* stream) {
  gelu_pair_check_kernel<<<unsigned(cdiv(n, 256)), 256, 0, as_stream(stream)>>>(n, bad_dev);
  SA_LAUNCH_CHECK("sa_debug_gelu_pair_check");
  return SA_OK;
}
#endif

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

SA_DEBUG_SWITCH(int, g_tc_dbg, 0, sa_debug_tc_mode)
// TMA-store epilogue for plain outputs
SA_DEBUG_SWITCH(int, g_tc_tma, 1, sa_debug_tc_tma)
// weights resident in shared memory when they fit
SA_DEBUG_SWITCH(int, g_tc_resident, 1, sa_debug_tc_resident)
// stage alternation when kchunks > 4 (measured: whole tiles per group win below)
SA_DEBUG_SWITCH(int, g_tc_kq, 4, sa_debug_tc_kq)
// A staging: 0 = direct A path (default), 1 = auto, 2/4/8 = force slots
SA_DEBUG_SWITCH(int, g_tc_stage, 0, sa_debug_tc_stage)

static int launch_tc(tc::TcParams& p, int amode, int bn, int64_t m_tiles_max, cudaStream_t s) {
  using namespace tc;
  if (p.M == 0) return SA_OK;
  p.ntiles = int(cdiv(p.N, bn));
  const int ng = p.ngroups > 2 ? p.ngroups : (p.counts ? 2 : 1);
  int npb_max = 0;
  for (int i = 0; i < ng; ++i) npb_max = max(npb_max, p.nplanes[i]);
  // resident weights when both experts' packed tiles fit in 48 KB
  p.ntiles = int(cdiv(p.N, bn));
  const size_t wb0 = size_t(p.ntiles) * p.kchunks * p.nplanes[0] * bn * kBK * 2;
  const size_t wb1 = p.counts ? size_t(p.ntiles) * p.kchunks * p.nplanes[1] * bn * kBK * 2 : 0;
  p.rb = (g_tc_resident && p.ngroups <= 2 && wb0 + wb1 <= 48 * 1024) ? 1 : 0;
  p.dbg = g_tc_dbg;
  p.kq_min = g_tc_kq;
  p.rb_bytes[0] = p.rb ? uint32_t(wb0) : 0u;
  p.rb_bytes[1] = p.rb ? uint32_t(wb1) : 0u;
  const size_t rb_total = p.rb ? ((wb0 + wb1 + 1023) & ~size_t(1023)) : 0;
  const size_t stage_bytes = 3 * size_t(kPlaneA) + (p.rb ? 0 : size_t(npb_max) * bn * kBK * 2);
  const size_t fixed = tc_fixed_smem() + 1024;   // + 1 KB alignment slack
  const size_t budget = 220 * 1024;
  // A staging (loader warp + bulk copies) for plain / gathered rows whose 16-byte
  // segments the TMA engine can copy; patchify keeps the direct loads
  const bool stageable = tc::kStaging && g_tc_stage && amode != A_PATCH && (p.K % 4) == 0 && (p.lda % 4) == 0 &&
                         (reinterpret_cast<uintptr_t>(p.A) & 15) == 0;
  int stages = 0, nst = 0;
  for (int cand_nst : {8, 4, 2, 0}) {
    if (cand_nst > 0 && !stageable) continue;
    if (g_tc_stage >= 2 && cand_nst > g_tc_stage) continue;
    const size_t room = budget - fixed - rb_total - size_t(cand_nst) * kStgBytes;
    int st = int(room / stage_bytes);
    st = st > 4 ? 4 : (st & ~1);  // even: the two producer groups alternate
    if (st >= 2) {
      stages = st;
      nst = cand_nst;
      break;
    }
  }
  if (stages < 2) {
    set_error("tensor-core stage does not fit shared memory (bn=%d)", bn);
    return SA_ERR_VALUE;
  }
  p.stages = stages;
  p.nst = nst;
  const size_t smem = size_t(stages) * stage_bytes + rb_total + size_t(nst) * kStgBytes + fixed;
  const int64_t tiles = m_tiles_max * p.ntiles;
  if (tiles >= (int64_t(1) << 31)) {
    set_error("tensor-core GEMM: %lld tiles exceed the 32-bit tile index", (long long)tiles);
    return SA_ERR_SHAPE;
  }
  const int grid = int(tiles < num_sms() ? tiles : num_sms());
  // TMA-store epilogue when C's rows are exactly the tile rows
  CUtensorMap tmC;
  memset(&tmC, 0, sizeof(tmC));
  p.tma_c = 0;
  if (g_tc_tma && bn % 32 == 0 && p.c_rows == nullptr &&
      (p.residual == nullptr ||
       ((reinterpret_cast<uintptr_t>(p.residual) & 15) == 0 && p.N % 32 == 0)) &&
      p.pos == nullptr && (p.img_tokens == 0 || p.extra == 0) && (p.N % 4) == 0 &&
      (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && p.M < (int64_t(1) << 31)) {
    const cuuint64_t dims[2] = {cuuint64_t(p.N), cuuint64_t(p.M)};
    const cuuint64_t strides[1] = {cuuint64_t(p.N) * 4};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tmap_tiled(
        &tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p.C, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) p.tma_c = 1;
  }
  // a residual on the TMA path needs the RES instantiation (plain A rows only)
  const bool res_tma = p.tma_c && p.residual != nullptr;
  if (res_tma && amode != A_PLAIN) p.tma_c = 0;
  // the fused LayerNorm lives in the TMA epilogue of a single-column-tile patch GEMM
  if (p.ln_g && !(p.tma_c && amode == A_PATCH && p.ntiles == 1 && p.N == bn && (bn == 32 || bn == 64))) {
    set_error("fused LayerNorm epilogue needs one 32/64-wide column tile on the TMA path");
    return SA_ERR_VALUE;
  }
#define SA_TC_CASE(BNV)                                                                          \
  case BNV: {                                                                                    \
    auto kfn = amode == A_PLAIN                                                                  \
                   ? (res_tma ? tc_gemm_kernel<BNV, A_PLAIN, true> : tc_gemm_kernel<BNV, A_PLAIN>) \
               : amode == A_GATHER                                                             \
                   ? (p.ngroups > 2 ? tc_gemm_kernel<BNV, A_GATHER, false, false, true>            \
                                    : tc_gemm_kernel<BNV, A_GATHER>)                               \
               : (p.ln_g ? tc_gemm_kernel<BNV, A_PATCH, false, (BNV == 32 || BNV == 64)>         \
                         : tc_gemm_kernel<BNV, A_PATCH>);                                       \
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));          \
    kfn<<<grid, kThreads, smem, s>>>(p, tmC);                                                    \
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
  // GEMM tile widths, plus d = 192 (the wide fused MLP reads W2 packed with bn = d)
  SA_REQUIRE(tc_tile_n_ok(bn) || bn == 192, SA_ERR_VALUE, "sa_weight_pack: tile N=%d unsupported", bn);
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
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31) && K > 0 && N > 0, SA_ERR_SHAPE, "%s: bad extents",
             who);
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

// The q/k/v projections of one attention layer routed by one fused LN+router
// pass (stacked plans: perm [nprob][M], counts [nprob][2], gate [nprob][M]) in
// ONE launch: 2·nprob row groups (problem x expert) over the same input x, y
// stacked [nprob][M][N]. Per problem identical to sa_tc_moe_linear.
extern "C" int sa_tc_moe_linear_grouped(const float* x, const int32_t* perm, const int32_t* counts,
                                        const float* gate, const void* const* wpack_dense,
                                        const void* const* wpack_shift, int nprob, int bn,
                                        float* y, int64_t M, int64_t K, int64_t N, void* stream) {
  SA_REQUIRE(nprob >= 1 && nprob <= 3, SA_ERR_VALUE, "sa_tc_moe_linear_grouped: 1..3 problems");
  SA_REQUIRE(M * nprob < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_tc_moe_linear_grouped: too many rows");
  if (int st = tc_check("sa_tc_moe_linear_grouped", M * nprob, K, N, bn)) return st;
  tc::TcParams p = tc_base(M * nprob, K, N);
  p.A = x;
  p.a_rows = perm;
  for (int i = 0; i < nprob; ++i) {
    p.Bp[2 * i] = static_cast<const uint16_t*>(wpack_dense[i]);
    p.nplanes[2 * i] = 3;
    p.Bp[2 * i + 1] = static_cast<const uint16_t*>(wpack_shift[i]);
    p.nplanes[2 * i + 1] = 1;
  }
  p.ngroups = 2 * nprob;
  p.prob_rows = M;
  p.counts = counts;
  p.C = y;
  p.c_rows = perm;
  p.gate = gate;
  return launch_tc(p, tc::A_GATHER, bn, nprob * (cdiv(M, tc::kBM) + 1), as_stream(stream));
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

static int tc_patch_embed_impl(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                               int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                               const float* cls, const float* pos, float* y, const float* ln_g,
                               const float* ln_b, float ln_eps, void* stream);
namespace sa {
int embed_ln_launch(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C, int64_t patch,
                    float sub, const void* wpack, int bn, int64_t d, const float* gain,
                    const float* bias, float eps, float* y, cudaStream_t s);
}
// patch embed + LN: 0 = the dedicated kernel (embed_tc.cu) when the shape
// allows, 1 = the GEMM path's LNE epilogue (bit-identical)
SA_DEBUG_SWITCH(int, g_embed_mode, 0, sa_debug_embed_mode)

extern "C" int sa_tc_patch_embed(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                                 int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                                 const float* cls, const float* pos, float* y, void* stream) {
  return tc_patch_embed_impl(grid, B, H, W, C, patch, sub, wpack, bn, d, cls, pos, y, nullptr,
                             nullptr, 0.f, stream);
}

extern "C" int sa_tc_patch_embed_ln_ok(int64_t d, int has_cls, int has_pos) {
  return (d == 32 || d == 64) && !has_cls && !has_pos;
}

extern "C" int sa_tc_patch_embed_ln(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                                    int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                                    const float* gain, const float* bias, float eps, float* y,
                                    void* stream) {
  SA_REQUIRE(gain != nullptr && bias != nullptr && sa_tc_patch_embed_ln_ok(d, 0, 0), SA_ERR_VALUE,
             "sa_tc_patch_embed_ln: d=%lld unsupported (32 or 64)", (long long)d);
  if (g_embed_mode == 0 && B > 0 && H > 0 && W > 0 && C > 0 && patch > 0 && H % patch == 0 &&
      B * (H / patch) * (W / patch) < (int64_t(1) << 31)) {
    const int st = embed_ln_launch(grid, B, H, W, C, patch, sub, wpack, bn, d, gain, bias, eps, y,
                                   as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  return tc_patch_embed_impl(grid, B, H, W, C, patch, sub, wpack, bn, d, nullptr, nullptr, y, gain,
                             bias, eps, stream);
}

static int tc_patch_embed_impl(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                               int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                               const float* cls, const float* pos, float* y, const float* ln_g,
                               const float* ln_b, float ln_eps, void* stream) {
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
  SA_REQUIRE(B * n < (int64_t(1) << 31), SA_ERR_SHAPE,
             "sa_tc_patch_embed: %lld tokens exceed the 32-bit token index", (long long)(B * n));
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
  p.ln_g = ln_g;
  p.ln_b = ln_b;
  p.ln_eps = ln_eps;
  cudaStream_t s = as_stream(stream);
  int st = launch_tc(p, tc::A_PATCH, bn, cdiv(B * n, tc::kBM), s);
  if (st) return st;
  if (cls) return write_cls_rows(cls, pos, y, B, n + 1, d, s);
  return SA_OK;
}
