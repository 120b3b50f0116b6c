// Glue kernels around the hot path: LayerNorm, softmax attention of the
// exempt (MSA) stage, pooling, cls-token rows.
#include "common.cuh"

namespace sa {

// LayerNorm over the last axis, biased variance, eps inside the sqrt
// (ref tensor.py:114-128). One warp per row, d <= 512 held in registers.
template <int PER>
__global__ void __launch_bounds__(256) layernorm_kernel(const float* __restrict__ x,
                                                       const float* __restrict__ gain,
                                                       const float* __restrict__ bias,
                                                       float* __restrict__ y, int64_t M, int d,
                                                       float eps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + warp;
  if (row >= M) return;
  const float* xr = x + row * d;
  float v[PER];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < d ? xr[c] : 0.f;
    s += v[i];
  }
  const float mean = warp_sum(s) / float(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < d ? v[i] - mean : 0.f;
    q += v[i] * v[i];
  }
  const float var = warp_sum(q) / float(d);
  const float inv = 1.0f / sqrtf(var + eps);
  float* yr = y + row * d;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int c = lane + 32 * i;
    if (c < d) yr[c] = v[i] * inv * gain[c] + bias[c];
  }
}

// narrow rows (d = 32 / 64): one thread per row, the whole row in registers
// via 128-bit loads — d/4 independent loads in flight per thread.
// Each warp's 32 rows are staged through shared memory (coalesced 128-bit
// loads and stores of the contiguous 32·D block, row pitch D + 4: conflict-free
// 128-bit row reads), the arithmetic stays per thread = row.
template <int D>
__global__ void __launch_bounds__(128) layernorm_row_kernel(const float* __restrict__ x,
                                                           const float* __restrict__ gain,
                                                           const float* __restrict__ bias,
                                                           float* __restrict__ y, int64_t M,
                                                           float eps) {
  constexpr int P = D + 4;
  __shared__ __align__(16) float tile[4][32 * P];   // 4 warps per block
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = int64_t(blockIdx.x) * blockDim.x + warp * 32;
  const int nrows = int(min(int64_t(32), M - row0));
  if (nrows <= 0) return;
  float* tw = tile[warp];
  {
    const float4* src = reinterpret_cast<const float4*>(x + row0 * D);
    float4 buf[D / 4];
#pragma unroll
    for (int u = 0; u < D / 4; ++u) {
      const int i = lane + 32 * u;   // float4 index in the warp's block
      buf[u] = i < nrows * (D / 4) ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < D / 4; ++u) {
      const int i = lane + 32 * u;
      *reinterpret_cast<float4*>(tw + (i / (D / 4)) * P + 4 * (i % (D / 4))) = buf[u];
    }
  }
  __syncwarp();
  const int64_t row = row0 + lane;
  const float4* xr = reinterpret_cast<const float4*>(tw + lane * P);
  float4 v[D / 4];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < D / 4; ++i) {
    v[i] = xr[i];
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = s / float(D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < D / 4; ++i) {
    v[i].x -= mean; v[i].y -= mean; v[i].z -= mean; v[i].w -= mean;
    q += (v[i].x * v[i].x + v[i].y * v[i].y) + (v[i].z * v[i].z + v[i].w * v[i].w);
  }
  const float inv = 1.0f / sqrtf(q / float(D) + eps);
  float4* yr = reinterpret_cast<float4*>(tw + lane * P);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int i = 0; i < D / 4; ++i) {
    const float4 g = __ldg(g4 + i), bb = __ldg(b4 + i);
    yr[i] = make_float4(v[i].x * inv * g.x + bb.x, v[i].y * inv * g.y + bb.y,
                        v[i].z * inv * g.z + bb.z, v[i].w * inv * g.w + bb.w);
  }
  (void)row;
  __syncwarp();
  float4* dst = reinterpret_cast<float4*>(y + row0 * D);
#pragma unroll
  for (int u = 0; u < D / 4; ++u) {
    const int i = lane + 32 * u;
    if (i < nrows * (D / 4))
      dst[i] = *reinterpret_cast<const float4*>(tw + (i / (D / 4)) * P + 4 * (i % (D / 4)));
  }
}

// softmax attention per (image, head) (ref attention.py:92-97): K (padded) and
// V of the head in shared memory, one warp per query row, lanes over keys for
// the scores and over channels for P·V.
__global__ void __launch_bounds__(256) softmax_attn_kernel(const float* __restrict__ q,
                                                          const float* __restrict__ k,
                                                          const float* __restrict__ v,
                                                          float* __restrict__ out, int n, int d,
                                                          int heads, int dk, float scale_div,
                                                          int ld) {
  extern __shared__ __align__(16) float sm[];
  const int kp = dk + 1;
  float* sk = sm;                         // [n][dk+1]
  float* sv = sk + n * kp;                // [n][dk]
  float* sq = sv + n * dk;                // [8][dk]
  float* sp = sq + 8 * dk;                // [8][n]
  const int bh = blockIdx.x, b = bh / heads, h = bh % heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t rowbase = size_t(b) * n;
  for (int idx = threadIdx.x; idx < n * dk; idx += blockDim.x) {
    const int j = idx / dk, c = idx % dk;
    sk[j * kp + c] = k[(rowbase + j) * ld + h * dk + c];
    sv[j * dk + c] = v[(rowbase + j) * ld + h * dk + c];
  }
  __syncthreads();
  float* myq = sq + warp * dk;
  float* myp = sp + warp * n;
  for (int i = warp; i < n; i += 8) {
    for (int c = lane; c < dk; c += 32) myq[c] = q[(rowbase + i) * ld + h * dk + c];
    __syncwarp();
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) {
      float s = 0.f;
      for (int c = 0; c < dk; ++c) s = fmaf(myq[c], sk[j * kp + c], s);
      s = s / scale_div;
      myp[j] = s;
      mx = fmaxf(mx, s);
    }
    mx = warp_max(mx);
    float tot = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float e = expf(myp[j] - mx);
      myp[j] = e;
      tot += e;
    }
    tot = warp_sum(tot);
    __syncwarp();
    // p_j = e_j / sum (the reference's float32 division, once per key)
    for (int j = lane; j < n; j += 32) myp[j] = myp[j] / tot;
    __syncwarp();
    for (int c = lane; c < dk; c += 32) {
      float acc = 0.f;
#pragma unroll 4
      for (int j = 0; j < n; ++j) acc = fmaf(myp[j], sv[j * dk + c], acc);
      out[(rowbase + i) * d + h * dk + c] = acc;
    }
    __syncwarp();
  }
}

// dk = 32, n <= 32*NJ (PVT stage 4: n = 49): the same arithmetic as
// softmax_attn_kernel, re-laid for instruction-level parallelism — lane =
// key (NJ keys per lane) for the scores and lane = channel for P·V, the query
// rows and probabilities are smem broadcasts, and each warp carries QB queries
// at once (independent FMA chains); key rows and V are read from shared memory
// per 4-channel chunk, so registers stay ~72 (seven CTAs per SM).
// Per key the score is the same fma chain over c = 0..31, the softmax the same
// warp reductions, and P·V the same fma chain over j (zero-padded keys add
// exact zeros), so the output is bit-identical to the generic kernel.
// W warps × QB queries per round: W = QB = 7 covers n = 49 (the PVT stage-4
// grid) in one round instead of four rounds of 4 × 4 with a 1-query tail.
template <int NJ, int QB, int W>
__global__ void __launch_bounds__(32 * W) softmax_attn32_kernel(const float* __restrict__ q,
                                                            const float* __restrict__ k,
                                                            const float* __restrict__ v,
                                                            float* __restrict__ out, int n, int d,
                                                            int heads, float scale_div, int ld) {
  constexpr int NK = 32 * NJ;
  __shared__ __align__(16) float sk[NK][36];   // pitch 36: conflict-free 128-bit row reads
  __shared__ __align__(16) float sv[NK][32];
  __shared__ __align__(16) float sq[NK][32];
  __shared__ __align__(16) float sp[W][QB][NK];
  const int bh = blockIdx.x, b = bh / heads, h = bh % heads;
  const size_t rowbase = size_t(b) * n;
  for (int idx = threadIdx.x; idx < NK * 8; idx += 32 * W) {
    const int j = idx >> 3, c4 = (idx & 7) * 4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), bk = a, cv = a;
    if (j < n) {
      const size_t off = (rowbase + j) * ld + h * 32 + c4;   // inputs: row stride ld
      a = __ldg(reinterpret_cast<const float4*>(q + off));
      bk = __ldg(reinterpret_cast<const float4*>(k + off));
      cv = __ldg(reinterpret_cast<const float4*>(v + off));
    }
    *reinterpret_cast<float4*>(&sq[j][c4]) = a;
    *reinterpret_cast<float4*>(&sk[j][c4]) = bk;
    *reinterpret_cast<float4*>(&sv[j][c4]) = cv;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // queries i0 + W·r (r < QB) per warp iteration; a missing query recomputes i0
  const int nk4 = (n + 3) & ~3;   // P·V stops at the last 4-key group holding a real key
  for (int i0 = warp; i0 < n; i0 += W * QB) {
    float s[QB][NJ];
#pragma unroll
    for (int r = 0; r < QB; ++r)
#pragma unroll
      for (int u = 0; u < NJ; ++u) s[r][u] = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      float4 kk[NJ];   // the lane's key rows, 4 channels at a time (shared by the QB queries)
#pragma unroll
      for (int u = 0; u < NJ; ++u)
        kk[u] = *reinterpret_cast<const float4*>(&sk[lane + 32 * u][4 * m]);
#pragma unroll
      for (int r = 0; r < QB; ++r) {
        const int i = i0 + W * r < n ? i0 + W * r : i0;
        const float4 qq = *reinterpret_cast<const float4*>(&sq[i][4 * m]);
#pragma unroll
        for (int u = 0; u < NJ; ++u) {
          s[r][u] = fmaf(qq.x, kk[u].x, s[r][u]);
          s[r][u] = fmaf(qq.y, kk[u].y, s[r][u]);
          s[r][u] = fmaf(qq.z, kk[u].z, s[r][u]);
          s[r][u] = fmaf(qq.w, kk[u].w, s[r][u]);
        }
      }
    }
    float mx[QB], tot[QB];
#pragma unroll
    for (int r = 0; r < QB; ++r) {
      mx[r] = -INFINITY;
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        s[r][u] = s[r][u] / scale_div;
        if (lane + 32 * u < n) mx[r] = fmaxf(mx[r], s[r][u]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < QB; ++r) mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], o));
#pragma unroll
    for (int r = 0; r < QB; ++r) {
      tot[r] = 0.f;
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        if (lane + 32 * u < n) {
          s[r][u] = expf(s[r][u] - mx[r]);
          tot[r] += s[r][u];
        } else {
          s[r][u] = 0.f;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < QB; ++r) tot[r] += __shfl_xor_sync(0xffffffffu, tot[r], o);
#pragma unroll
    for (int r = 0; r < QB; ++r)
#pragma unroll
      for (int u = 0; u < NJ; ++u) sp[warp][r][lane + 32 * u] = s[r][u] / tot[r];   // padded keys: 0
    __syncwarp();
    float acc[QB];
#pragma unroll
    for (int r = 0; r < QB; ++r) acc[r] = 0.f;
#pragma unroll 4
    for (int j4 = 0; j4 < nk4; j4 += 4) {
      const float v0 = sv[j4][lane], v1 = sv[j4 + 1][lane], v2 = sv[j4 + 2][lane],
                  v3 = sv[j4 + 3][lane];
#pragma unroll
      for (int r = 0; r < QB; ++r) {
        const float4 pp = *reinterpret_cast<const float4*>(&sp[warp][r][j4]);
        acc[r] = fmaf(pp.x, v0, acc[r]);
        acc[r] = fmaf(pp.y, v1, acc[r]);
        acc[r] = fmaf(pp.z, v2, acc[r]);
        acc[r] = fmaf(pp.w, v3, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < QB; ++r)
      if (i0 + W * r < n) out[(rowbase + i0 + W * r) * d + h * 32 + lane] = acc[r];
    __syncwarp();
  }
}

// tokens.mean(axis=1) (ref model.py:574): numpy reduces a non-contiguous axis
// sequentially in float32, so a sequential per-channel sum reproduces it.
__global__ void pool_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t B, int n,
                            int d, int mode) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= B * d) return;
  const int64_t b = i / d;
  const int c = int(i % d);
  const float* xb = x + b * n * d;
  if (mode == 1) {
    y[i] = xb[c];
    return;
  }
  float s = 0.f;
  for (int t = 0; t < n; ++t) s += xb[int64_t(t) * d + c];
  y[i] = s / float(n);
}

__global__ void cls_rows_kernel(const float* __restrict__ cls, const float* __restrict__ pos,
                                float* __restrict__ y, int64_t B, int64_t rows, int d) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= B * d) return;
  const int64_t b = i / d;
  const int c = int(i % d);
  y[b * rows * d + c] = pos ? cls[c] + pos[c] : cls[c];
}

int write_cls_rows(const float* cls, const float* pos, float* y, int64_t B, int64_t rows,
                   int64_t d, cudaStream_t s) {
  cls_rows_kernel<<<unsigned(cdiv(B * d, 256)), 256, 0, s>>>(cls, pos, y, B, rows, int(d));
  count_launch(1);
  SA_LAUNCH_CHECK("cls_rows_kernel");
  return SA_OK;
}

}  // namespace sa

using namespace sa;

extern "C" int sa_layernorm(const float* x, const float* gain, const float* bias, float* y,
                            int64_t M, int64_t d, float eps, void* stream) {
  SA_REQUIRE(M >= 0 && d > 0 && d <= 1024, SA_ERR_SHAPE, "sa_layernorm: d=%lld unsupported",
             (long long)d);
  if (M == 0) return SA_OK;
  cudaStream_t s = as_stream(stream);
  if (d == 32 || d == 64) {
    const unsigned g = unsigned(cdiv(M, 128));
    if (d == 32) layernorm_row_kernel<32><<<g, 128, 0, s>>>(x, gain, bias, y, M, eps);
    else layernorm_row_kernel<64><<<g, 128, 0, s>>>(x, gain, bias, y, M, eps);
    count_launch(1);
    SA_LAUNCH_CHECK("sa_layernorm");
    return SA_OK;
  }
  const unsigned grid = unsigned(cdiv(M, 8));
  const int per = int(cdiv(d, 32));
  if (per <= 1) layernorm_kernel<1><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  else if (per <= 2) layernorm_kernel<2><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  else if (per <= 4) layernorm_kernel<4><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  else if (per <= 8) layernorm_kernel<8><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  else if (per <= 16) layernorm_kernel<16><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  else layernorm_kernel<32><<<grid, 256, 0, s>>>(x, gain, bias, y, M, int(d), eps);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_layernorm");
  return SA_OK;
}

SA_DEBUG_SWITCH(int, g_softmax_generic, 0, sa_debug_softmax_generic)
// 0: tensor-core kernel (softmax_tc.cu) for dk = 64, or dk = 32 with n > 64
SA_DEBUG_SWITCH(int, g_softmax_tc, 0, sa_debug_softmax_tc)
namespace sa {
int softmax_tc_launch(const float* q, const float* k, const float* v, int64_t ld, float* out,
                      int64_t B, int64_t n, int64_t d, int64_t heads, float scale_div,
                      cudaStream_t s);
}
// queries per warp iteration (debug sweep)
SA_DEBUG_SWITCH(int, g_softmax_qb, 4, sa_debug_softmax_qb)

extern "C" int sa_softmax_attn_strided(const float* q, const float* k, const float* v,
                                       int64_t ld, float* out, int64_t B, int64_t n, int64_t d,
                                       int64_t heads, void* stream);

extern "C" int sa_softmax_attn(const float* q, const float* k, const float* v, float* out,
                               int64_t B, int64_t n, int64_t d, int64_t heads, void* stream) {
  return sa_softmax_attn_strided(q, k, v, d, out, B, n, d, heads, stream);
}

extern "C" int sa_softmax_attn_strided(const float* q, const float* k, const float* v,
                                       int64_t ld, float* out, int64_t B, int64_t n, int64_t d,
                                       int64_t heads, void* stream) {
  SA_REQUIRE(B > 0 && n > 0 && d > 0 && heads > 0 && d % heads == 0 && ld >= d, SA_ERR_SHAPE,
             "sa_softmax_attn: bad extents");
  const int64_t dk = d / heads;
  const float scale_div0 = sqrtf(float(dk));  // python float math.sqrt(dk) → f32
  if (!g_softmax_generic && dk == 32 && n <= 64 && (d % 4) == 0 && (ld % 4) == 0 &&
      (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(k) & 15) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    const unsigned grid = unsigned(B * heads);
    cudaStream_t st = as_stream(stream);
#define SA_SM32(NJ, QB) \
  softmax_attn32_kernel<NJ, QB, 4><<<grid, 128, 0, st>>>(q, k, v, out, int(n), int(d), int(heads), \
                                                      scale_div0, int(ld))
    if (n > 42 && n <= 49 && g_softmax_qb == 4) {
      softmax_attn32_kernel<2, 7, 7><<<grid, 224, 0, st>>>(q, k, v, out, int(n), int(d),
                                                          int(heads), scale_div0, int(ld));
    } else if (n <= 32) {
      if (g_softmax_qb == 2) SA_SM32(1, 2);
      else if (g_softmax_qb == 8) SA_SM32(1, 8);
      else SA_SM32(1, 4);
    } else {
      if (g_softmax_qb == 2) SA_SM32(2, 2);
      else if (g_softmax_qb == 8) SA_SM32(2, 8);
      else SA_SM32(2, 4);
    }
#undef SA_SM32
    count_launch(1);
    SA_LAUNCH_CHECK("sa_softmax_attn");
    return SA_OK;
  }
  if (!g_softmax_generic && g_softmax_tc == 0 && (dk == 64 || (dk == 32 && n > 64))) {
    const int st = softmax_tc_launch(q, k, v, ld, out, B, n, d, heads, scale_div0,
                                     as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  const size_t smem = size_t(n * (dk + 1) + n * dk + 8 * dk + 8 * n) * sizeof(float);
  SA_REQUIRE(smem <= 220 * 1024, SA_ERR_SHAPE, "sa_softmax_attn: n=%lld dk=%lld too large",
             (long long)n, (long long)dk);
  cudaFuncSetAttribute(softmax_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const float scale_div = sqrtf(float(dk));  // python float math.sqrt(dk) → f32
  softmax_attn_kernel<<<unsigned(B * heads), 256, smem, as_stream(stream)>>>(
      q, k, v, out, int(n), int(d), int(heads), int(dk), scale_div, int(ld));
  count_launch(1);
  SA_LAUNCH_CHECK("sa_softmax_attn");
  return SA_OK;
}

extern "C" int sa_pool(const float* x, float* y, int64_t B, int64_t n, int64_t d, int mode,
                       void* stream) {
  SA_REQUIRE(B > 0 && n > 0 && d > 0, SA_ERR_SHAPE, "sa_pool: bad extents");
  pool_kernel<<<unsigned(cdiv(B * d, 256)), 256, 0, as_stream(stream)>>>(x, y, B, int(n), int(d),
                                                                          mode);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_pool");
  return SA_OK;
}
