// Linear layers: dense (mult) and shift (power-of-two) weights, plain GEMM,
// patch embedding, MLPs and the two-expert MoE launch, all on one fp32 GEMM
// core with fused prologues (row gather / patchify) and epilogues (GELU,
// ×gate, scatter, residual, position embedding).
//
// This is the first-generation CUDA-core (FFMA) path: 128×BN×16 tiles, 256
// threads, 8×(BN/16) register micro-tiles, double-buffered shared memory.
// Shift weights stay packed (1 byte/weight) in HBM and are decoded into exact
// float32 s·2^P in shared memory by writing the exponent field
// (ref quantize.py:99-101) — every x·2^P product is exact, so the result equals
// a dense product against the reconstruction up to summation order
// (ref tests/test_quantize.py:79-85).
//
// MoE (ref model.py:250-274): rows are addressed in the PERMUTED order of
// sa_moe_route (expert-0 tokens ascending | expert-1 tokens ascending); the
// tile scheduler reads counts[0] on the device, so both experts run in ONE grid
// sized for the worst case (no host sync, CUDA-graph capturable). Tile t
// belongs to expert 0 if t < ceil(c0/BM), else expert 1; out-of-range tiles exit.
#include "common.cuh"

namespace sa {

constexpr int kBM = 128, kBK = 16, kGemmThreads = 256;

enum AMode { A_PLAIN = 0, A_GATHER = 1, A_PATCH = 2 };

struct GemmParams {
  // A operand
  const float* A;
  int64_t lda;
  const int32_t* a_rows;  // A_GATHER: virtual row -> source row
  int64_t pH, pW, pC, patch, pside;  // A_PATCH geometry (grid B,H,W,C; patch; tokens/side)
  float sub;                          // A_PATCH: value subtracted from every element
  // B operand per expert (index 0 when no grouping)
  const void* B[2];
  int bkind[2];  // SA_W_DENSE / SA_W_SHIFT
  int p_min;
  int64_t M, K, N;
  const int32_t* counts;  // non-null: two-expert grouping on permuted rows
  // epilogue
  float* C;
  const int32_t* c_rows;  // scatter: virtual row -> output row
  const float* gate;      // per output row
  const float* residual;  // per output row (ld = N)
  int act;                // 0 none, 1 gelu
  const float* pos;       // (pos_rows, N), indexed by token-in-image + extra
  int64_t img_tokens;     // tokens per image for pos / cls remapping (0 = off)
  int extra;              // 1 when a cls token precedes the patch tokens
};

template <int BN, int AM>
__global__ void __launch_bounds__(kGemmThreads) gemm_f32_kernel(GemmParams p) {
  constexpr int TN = BN / 16;
  __shared__ __align__(16) float As[2][kBK][kBM + 4];
  __shared__ __align__(16) float Bs[2][kBK][BN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;

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
  if (r0 >= r1) return;
  const int64_t n0 = int64_t(blockIdx.y) * BN;
  const bool shiftB = p.bkind[group] == SA_W_SHIFT;
  const void* Bp = p.B[group];
  const int64_t K = p.K, N = p.N;

  // ---- A loader: thread -> (row am, k offsets ak, ak+4) ----
  const int am = tid >> 1, ak = (tid & 1) * 8;
  const int64_t arow = r0 + am;
  const bool arow_ok = arow < r1;
  const float* abase = nullptr;
  int64_t patch_row_stride = 0;
  if (arow_ok) {
    if (AM == A_PLAIN) {
      abase = p.A + arow * p.lda;
    } else if (AM == A_GATHER) {
      abase = p.A + int64_t(p.a_rows[arow]) * p.lda;
    } else {
      const int64_t tpi = p.pside * p.pside;
      const int64_t b = arow / tpi, t = arow % tpi;
      const int64_t py = t / p.pside, px = t % p.pside;
      abase = p.A + ((b * p.pH + py * p.patch) * p.pW + px * p.patch) * p.pC;
      patch_row_stride = p.pW * p.pC;
    }
  }
  const int64_t pcw = p.patch * p.pC;  // contiguous run per image row of a patch

  auto load_a = [&](int64_t k0, float4 (&ra)[2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t k = k0 + ak + i * 4;
      if (arow_ok && k < K) {
        const float* src;
        if (AM == A_PATCH) src = abase + (k / pcw) * patch_row_stride + (k % pcw);
        else src = abase + k;
        float4 v = __ldg(reinterpret_cast<const float4*>(src));
        if (AM == A_PATCH) {
          v.x -= p.sub; v.y -= p.sub; v.z -= p.sub; v.w -= p.sub;
        }
        ra[i] = v;
      } else {
        ra[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  auto store_a = [&](int buf, const float4 (&ra)[2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      As[buf][ak + i * 4 + 0][am] = ra[i].x;
      As[buf][ak + i * 4 + 1][am] = ra[i].y;
      As[buf][ak + i * 4 + 2][am] = ra[i].z;
      As[buf][ak + i * 4 + 3][am] = ra[i].w;
    }
  };

  // ---- B loader: BN/4 float4 per k row; threads [0, 4*BN) active ----
  constexpr int BQ = BN / 4;
  const int bk = tid / BQ, bn = (tid % BQ) * 4;
  const bool b_act = tid < kBK * BQ;
  const bool nvec = (N & 3) == 0;
  auto load_b = [&](int64_t k0, float4& rb) {
    rb = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!b_act) return;
    const int64_t k = k0 + bk, n = n0 + bn;
    if (k >= K || n >= N) return;
    if (!shiftB) {
      const float* src = static_cast<const float*>(Bp) + k * N + n;
      if (nvec) {
        rb = __ldg(reinterpret_cast<const float4*>(src));
      } else {
        rb.x = __ldg(src);
        if (n + 1 < N) rb.y = __ldg(src + 1);
        if (n + 2 < N) rb.z = __ldg(src + 2);
        if (n + 3 < N) rb.w = __ldg(src + 3);
      }
    } else {
      const uint8_t* src = static_cast<const uint8_t*>(Bp) + k * N + n;
      if (nvec) {
        const uint32_t q = __ldg(reinterpret_cast<const uint32_t*>(src));
        rb.x = decode_shift(q & 0xffu, p.p_min);
        rb.y = decode_shift((q >> 8) & 0xffu, p.p_min);
        rb.z = decode_shift((q >> 16) & 0xffu, p.p_min);
        rb.w = decode_shift(q >> 24, p.p_min);
      } else {
        rb.x = decode_shift(__ldg(src), p.p_min);
        if (n + 1 < N) rb.y = decode_shift(__ldg(src + 1), p.p_min);
        if (n + 2 < N) rb.z = decode_shift(__ldg(src + 2), p.p_min);
        if (n + 3 < N) rb.w = decode_shift(__ldg(src + 3), p.p_min);
      }
    }
  };
  auto store_b = [&](int buf, const float4& rb) {
    if (b_act) *reinterpret_cast<float4*>(&Bs[buf][bk][bn]) = rb;
  };

  float acc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const int64_t ktiles = (K + kBK - 1) / kBK;
  float4 ra[2], rb;
  load_a(0, ra);
  load_b(0, rb);
  store_a(0, ra);
  store_b(0, rb);
  __syncthreads();

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int buf = int(kt & 1);
    const bool more = kt + 1 < ktiles;
    if (more) {
      load_a((kt + 1) * kBK, ra);
      load_b((kt + 1) * kBK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[TN];
      if (TN == 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
        bv[0] = b4.x; bv[1] = b4.y; bv[2] = b4.z; bv[3] = b4.w;
      } else {
        const float2 b2 = *reinterpret_cast<const float2*>(&Bs[buf][kk][tx * TN]);
        bv[0] = b2.x; bv[1] = b2.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      store_a(buf ^ 1, ra);
      store_b(buf ^ 1, rb);
    }
    __syncthreads();
  }

  // ---- epilogue ----
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + ty * 8 + i;
    if (r >= r1) continue;
    int64_t orow = p.c_rows ? int64_t(p.c_rows[r]) : r;
    int64_t pos_idx = 0;
    if (p.img_tokens > 0) {
      const int64_t b = r / p.img_tokens, t = r % p.img_tokens;
      orow = b * (p.img_tokens + p.extra) + p.extra + t;
      pos_idx = p.extra + t;
    }
    const float g = p.gate ? p.gate[orow] : 1.f;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx * TN + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (p.act == 1) v = gelu_tanh(v);
      if (p.gate) v = v * g;
      if (p.pos) v = v + p.pos[pos_idx * N + n];
      if (p.residual) v = p.residual[orow * N + n] + v;
      p.C[orow * N + n] = v;
    }
  }
}

static int launch_gemm(GemmParams& p, int amode, int64_t m_tiles, cudaStream_t s) {
  if (p.M == 0) return SA_OK;
  const bool narrow = p.N <= 32;
  const int BN = narrow ? 32 : 64;
  dim3 grid(unsigned(m_tiles), unsigned(cdiv(p.N, BN)));
#define SA_GEMM_LAUNCH(BNV, AMV) gemm_f32_kernel<BNV, AMV><<<grid, kGemmThreads, 0, s>>>(p)
  if (narrow) {
    if (amode == A_PLAIN) SA_GEMM_LAUNCH(32, A_PLAIN);
    else if (amode == A_GATHER) SA_GEMM_LAUNCH(32, A_GATHER);
    else SA_GEMM_LAUNCH(32, A_PATCH);
  } else {
    if (amode == A_PLAIN) SA_GEMM_LAUNCH(64, A_PLAIN);
    else if (amode == A_GATHER) SA_GEMM_LAUNCH(64, A_GATHER);
    else SA_GEMM_LAUNCH(64, A_PATCH);
  }
#undef SA_GEMM_LAUNCH
  count_launch(1);
  SA_LAUNCH_CHECK("gemm_f32_kernel");
  return SA_OK;
}

static GemmParams base_params(int64_t M, int64_t K, int64_t N) {
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.K = K;
  p.N = N;
  p.lda = K;
  p.p_min = -15;
  return p;
}

// ---- quantize_shift (ref quantize.py:83-96) --------------------------------
// P = rint(log2|w|) computed exactly without a transcendental: for |w| = m·2^e
// (m in [1,2)), log2|w| rounds up iff m > sqrt(2) (m == sqrt(2) is impossible
// in binary floating point), so P = e + (m > sqrt2). Zeros, subnormals below
// 2^p_min and non-finite magnitudes follow the reference's nan_to_num/clip.
__global__ void quantize_shift_kernel(const float* __restrict__ w, int64_t count, int p_min,
                                      int p_max, uint8_t* __restrict__ packed,
                                      float* __restrict__ s_out, int32_t* __restrict__ p_out) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const float x = w[i];
  const bool neg = x < 0.f;
  const double a = fabs(double(x));
  int P;
  if (a == 0.0 || isnan(a)) {
    P = p_min;                       // log2(0) = -inf → p_min; NaN → p_min
  } else if (isinf(a)) {
    P = p_max;
  } else {
    int e;
    const double m = frexp(a, &e);   // a = m·2^e, m in [0.5, 1)
    // log2 a = (e-1) + log2(2m); rounds up iff 2m > sqrt(2)
    P = (e - 1) + ((2.0 * m) > 1.4142135623730951 ? 1 : 0);
    P = P < p_min ? p_min : (P > p_max ? p_max : P);
  }
  packed[i] = uint8_t((neg ? 0x80u : 0u) | uint32_t(P - p_min));
  if (s_out) s_out[i] = neg ? -1.f : 1.f;
  if (p_out) p_out[i] = P;
}

// ---- literal MatShift (variant 1): exponent-field add + fp32 add ------------
// y[m][n] = sum_k shift(x[m][k], s[k][n], P[k][n]) where shift() flips the sign
// bit and adds P to the exponent field of a normal float (no multiply). Zero,
// subnormal, inf/nan inputs or exponent overflow fall back to ldexpf.
__device__ __forceinline__ float shift_apply(float x, uint32_t code, int p_min) {
  const uint32_t bits = __float_as_uint(x);
  const int P = int(code & 31u) + p_min;
  const uint32_t sgn = (code & 0x80u) << 24;
  const int e = int((bits >> 23) & 0xffu);
  const int ne = e + P;
  if (e != 0 && e != 0xff && ne > 0 && ne < 0xff)
    return __uint_as_float((bits + (uint32_t(P) << 23)) ^ sgn);
  return __uint_as_float(__float_as_uint(ldexpf(x, P)) ^ sgn);
}

constexpr int kMsBM = 64, kMsBN = 64, kMsBK = 32;
__global__ void __launch_bounds__(256) matshift_kernel(const float* __restrict__ x,
                                                       const uint8_t* __restrict__ packed,
                                                       float* __restrict__ y, int64_t M,
                                                       int64_t K, int64_t N, int p_min) {
  __shared__ float xs[kMsBK][kMsBM + 1];
  __shared__ uint8_t ws[kMsBK][kMsBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 4x4 outputs per thread
  const int64_t m0 = int64_t(blockIdx.x) * kMsBM, n0 = int64_t(blockIdx.y) * kMsBN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += kMsBK) {
    for (int idx = tid; idx < kMsBM * kMsBK; idx += 256) {
      const int mm = idx / kMsBK, kk = idx % kMsBK;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      xs[kk][mm] = (gm < M && gk < K) ? x[gm * K + gk] : 0.f;
    }
    for (int idx = tid; idx < kMsBK * kMsBN; idx += 256) {
      const int kk = idx / kMsBN, nn = idx % kMsBN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      ws[kk][nn] = (gk < K && gn < N) ? packed[gk * N + gn] : uint8_t(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kMsBK; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float xv = xs[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += shift_apply(xv, ws[kk][tx * 4 + j], p_min);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn < N) y[gm * N + gn] = acc[i][j];
    }
  }
}

// ---- MatAdd (AddLinear): signed accumulation under binary weights ----------
// y[m][n] = gamma · sum_k (b[k][n] < 0 ? -x[m][k] : x[m][k]): adds and subtracts
// only, one multiply by gamma at the end (ref quantize.py:143-160). The sum runs
// in fp64 like the reference (fp64 sums of fp32 terms, exact whenever the
// terms' exponents span < 29 bits), then one fp64 product and one rounding to
// fp32, so results are bit-identical to the reference in that regime.
// signs: one byte per weight, bit 7 set = negative (the shift-code sign bit).
__global__ void __launch_bounds__(256) matadd_kernel(const float* __restrict__ x,
                                                     const uint8_t* __restrict__ signs,
                                                     double gamma, float* __restrict__ y, int64_t M,
                                                     int64_t K, int64_t N) {
  __shared__ float xs[kMsBK][kMsBM + 1];
  __shared__ uint8_t ws[kMsBK][kMsBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 4x4 outputs per thread
  const int64_t m0 = int64_t(blockIdx.x) * kMsBM, n0 = int64_t(blockIdx.y) * kMsBN;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += kMsBK) {
    for (int idx = tid; idx < kMsBM * kMsBK; idx += 256) {
      const int mm = idx / kMsBK, kk = idx % kMsBK;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      xs[kk][mm] = (gm < M && gk < K) ? x[gm * K + gk] : 0.f;
    }
    for (int idx = tid; idx < kMsBK * kMsBN; idx += 256) {
      const int kk = idx / kMsBN, nn = idx % kMsBN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      ws[kk][nn] = (gk < K && gn < N) ? signs[gk * N + gn] : uint8_t(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kMsBK; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double xv = double(xs[kk][ty * 4 + i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += (ws[kk][tx * 4 + j] & 0x80u) ? -xv : xv;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn < N) y[gm * N + gn] = float(acc[i][j] * gamma);
    }
  }
}

static int check_k4(const char* who, int64_t K) {
  SA_REQUIRE(K % 4 == 0, SA_ERR_SHAPE, "%s: inner extent %lld must be a multiple of 4", who,
             (long long)K);
  return SA_OK;
}

}  // namespace sa

using namespace sa;

extern "C" int sa_quantize_shift(const float* w, int64_t count, int p_min, int p_max,
                                 uint8_t* packed, float* s_out, int32_t* p_out, void* stream) {
  SA_REQUIRE(p_min < p_max, SA_ERR_VALUE, "p_min %d must be below p_max %d", p_min, p_max);
  SA_REQUIRE(p_max - p_min <= 31 && p_min >= -126 && p_max <= 127, SA_ERR_VALUE,
             "exponent range [%d, %d] does not fit the 5-bit shift code", p_min, p_max);
  if (count == 0) return SA_OK;
  quantize_shift_kernel<<<unsigned(cdiv(count, 256)), 256, 0, as_stream(stream)>>>(
      w, count, p_min, p_max, packed, s_out, p_out);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_quantize_shift");
  return SA_OK;
}

extern "C" int sa_linear(const float* x, const void* w, int w_kind, float* y, int64_t M,
                         int64_t K, int64_t N, int p_min, const float* residual, int act,
                         void* stream) {
  SA_REQUIRE(M >= 0 && K > 0 && N > 0, SA_ERR_SHAPE, "sa_linear: bad extents");
  if (int st = check_k4("sa_linear", K)) return st;
  SA_REQUIRE(w_kind == SA_W_DENSE || w_kind == SA_W_SHIFT, SA_ERR_VALUE,
             "sa_linear: unknown weight kind %d", w_kind);
  GemmParams p = base_params(M, K, N);
  p.A = x;
  p.B[0] = w;
  p.bkind[0] = w_kind;
  p.p_min = p_min;
  p.C = y;
  p.residual = residual;
  p.act = act;
  return launch_gemm(p, A_PLAIN, cdiv(M, kBM), as_stream(stream));
}

extern "C" int sa_gemm(const float* a, const float* b, float* c, int64_t M, int64_t K, int64_t N,
                       void* stream) {
  return sa_linear(a, b, SA_W_DENSE, c, M, K, N, -15, nullptr, 0, stream);
}

extern "C" int sa_shift_linear(const float* x, const uint8_t* packed, float* y, int64_t M,
                               int64_t K, int64_t N, int p_min, int variant, void* stream) {
  if (variant == 0) return sa_linear(x, packed, SA_W_SHIFT, y, M, K, N, p_min, nullptr, 0, stream);
  SA_REQUIRE(variant == 1, SA_ERR_VALUE, "sa_shift_linear: unknown variant %d", variant);
  SA_REQUIRE(M >= 0 && K > 0 && N > 0, SA_ERR_SHAPE, "sa_shift_linear: bad extents");
  if (M == 0) return SA_OK;
  dim3 grid(unsigned(cdiv(M, kMsBM)), unsigned(cdiv(N, kMsBN)));
  matshift_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, packed, y, M, K, N, p_min);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_shift_linear");
  return SA_OK;
}

extern "C" int sa_add_linear(const float* x, const uint8_t* signs, double gamma, float* y,
                             int64_t M, int64_t K, int64_t N, void* stream) {
  SA_REQUIRE(M >= 0 && K > 0 && N > 0, SA_ERR_SHAPE, "sa_add_linear: bad extents");
  SA_REQUIRE(cdiv(M, kMsBM) < (int64_t(1) << 31) && cdiv(N, kMsBN) < 65536, SA_ERR_SHAPE,
             "sa_add_linear: extents too large");
  if (M == 0) return SA_OK;
  dim3 grid(unsigned(cdiv(M, kMsBM)), unsigned(cdiv(N, kMsBN)));
  matadd_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, signs, gamma, y, M, K, N);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_add_linear");
  return SA_OK;
}

extern "C" size_t sa_mlp_workspace(int64_t M, int64_t hidden) {
  return size_t(M) * size_t(hidden) * sizeof(float);
}

extern "C" int sa_mlp(const float* x, const void* w1, int w1_kind, const void* w2, int w2_kind,
                      float* y, int64_t M, int64_t d, int64_t hidden, int p_min,
                      const float* residual, void* ws, size_t ws_bytes, void* stream) {
  SA_REQUIRE(ws_bytes >= sa_mlp_workspace(M, hidden), SA_ERR_VALUE, "sa_mlp: workspace too small");
  float* h = static_cast<float*>(ws);
  int st = sa_linear(x, w1, w1_kind, h, M, d, hidden, p_min, nullptr, 1, stream);
  if (st) return st;
  return sa_linear(h, w2, w2_kind, y, M, hidden, d, p_min, residual, 0, stream);
}

extern "C" int sa_moe_linear(const float* x, const int32_t* perm, const int32_t* counts,
                             const float* gate, const float* w_dense, const uint8_t* w_shift,
                             int p_min, float* y, const float* residual, int64_t M, int64_t K,
                             int64_t N, void* stream) {
  SA_REQUIRE(M >= 0 && K > 0 && N > 0, SA_ERR_SHAPE, "sa_moe_linear: bad extents");
  if (int st = check_k4("sa_moe_linear", K)) return st;
  GemmParams p = base_params(M, K, N);
  p.A = x;
  p.a_rows = perm;
  p.B[0] = w_dense;
  p.bkind[0] = SA_W_DENSE;
  p.B[1] = w_shift;
  p.bkind[1] = SA_W_SHIFT;
  p.p_min = p_min;
  p.counts = counts;
  p.C = y;
  p.c_rows = perm;
  p.gate = gate;
  p.residual = residual;
  return launch_gemm(p, A_GATHER, cdiv(M, kBM) + 1, as_stream(stream));
}

extern "C" size_t sa_moe_mlp_workspace(int64_t M, int64_t hidden) {
  return size_t(M) * size_t(hidden) * sizeof(float);
}

extern "C" int sa_moe_mlp(const float* x, const int32_t* perm, const int32_t* counts,
                          const float* gate, const float* w1_dense, const float* w2_dense,
                          const uint8_t* w1_shift, const uint8_t* w2_shift, int p_min, float* y,
                          const float* residual, int64_t M, int64_t d, int64_t hidden, void* ws,
                          size_t ws_bytes, void* stream) {
  SA_REQUIRE(M >= 0 && d > 0 && hidden > 0, SA_ERR_SHAPE, "sa_moe_mlp: bad extents");
  if (int st = check_k4("sa_moe_mlp", d)) return st;
  if (int st = check_k4("sa_moe_mlp", hidden)) return st;
  SA_REQUIRE(ws_bytes >= sa_moe_mlp_workspace(M, hidden), SA_ERR_VALUE,
             "sa_moe_mlp: workspace too small");
  float* h = static_cast<float*>(ws);  // hidden activations in permuted row order
  cudaStream_t s = as_stream(stream);
  GemmParams p1 = base_params(M, d, hidden);
  p1.A = x;
  p1.a_rows = perm;
  p1.B[0] = w1_dense;
  p1.bkind[0] = SA_W_DENSE;
  p1.B[1] = w1_shift;
  p1.bkind[1] = SA_W_SHIFT;
  p1.p_min = p_min;
  p1.counts = counts;
  p1.C = h;
  p1.act = 1;
  int st = launch_gemm(p1, A_GATHER, cdiv(M, kBM) + 1, s);
  if (st) return st;
  GemmParams p2 = base_params(M, hidden, d);
  p2.A = h;
  p2.B[0] = w2_dense;
  p2.bkind[0] = SA_W_DENSE;
  p2.B[1] = w2_shift;
  p2.bkind[1] = SA_W_SHIFT;
  p2.p_min = p_min;
  p2.counts = counts;
  p2.C = y;
  p2.c_rows = perm;
  p2.gate = gate;
  p2.residual = residual;
  return launch_gemm(p2, A_PLAIN, cdiv(M, kBM) + 1, s);
}

extern "C" int sa_patch_embed(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                              int64_t patch, float sub, const float* w, int64_t d,
                              const float* cls, const float* pos, float* y, void* stream) {
  SA_REQUIRE(B > 0 && H > 0 && W > 0 && C > 0 && patch > 0 && d > 0, SA_ERR_SHAPE,
             "sa_patch_embed: bad extents");
  SA_REQUIRE(H % patch == 0 && W % patch == 0 && H == W, SA_ERR_SHAPE,
             "sa_patch_embed: square image side %lld not divisible by patch %lld", (long long)H,
             (long long)patch);
  SA_REQUIRE((patch * C) % 4 == 0, SA_ERR_SHAPE, "sa_patch_embed: patch*C must be a multiple of 4");
  const int64_t side = H / patch;
  const int64_t n = side * side;
  const int64_t K = patch * patch * C;
  GemmParams p = base_params(B * n, K, d);
  p.A = grid;
  p.pH = H;
  p.pW = W;
  p.pC = C;
  p.patch = patch;
  p.pside = side;
  p.sub = sub;
  p.B[0] = w;
  p.bkind[0] = SA_W_DENSE;
  p.C = y;
  p.pos = pos;
  p.img_tokens = n;
  p.extra = cls ? 1 : 0;
  cudaStream_t s = as_stream(stream);
  int st = launch_gemm(p, A_PATCH, cdiv(B * n, kBM), s);
  if (st) return st;
  if (cls) {
    // cls rows: y[b*(n+1)] = cls (+ pos[0])
    return write_cls_rows(cls, pos, y, B, n + 1, d, s);
  }
  return SA_OK;
}
