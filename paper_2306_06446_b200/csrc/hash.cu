// K1 — Q/K sign-hash to bit-packed codes + per-(image, head) mean-|x| scale.
//
// Semantics (ref quantize.py:78-80, 123-140 as called at model.py:355-358):
//   code = !(x < 0)        (so -0.0 and NaN hash to 1; built WITHOUT fast-math/FTZ)
//   gamma[b, h] = mean |x| over the n tokens x dk channels of head h of image b.
//
// Layout: x is the flat projection output (B*n, d); codes are written
// [B][heads][n][W], W = ceil(dk/32), bit j of word w = channel 32w+j of the head.
//
// Each CTA owns a chunk of kTokPerCta tokens of one image: warps walk rows with
// 128-bit loads (lane = 4 channels), build 32-bit words with an 8-lane OR
// butterfly, stage them in shared memory and write them out coalesced in the
// [head][token][word] order. |x| is accumulated per channel in registers,
// reduced across warps in a fixed order and emitted as float64 partials per
// (image, chunk, head); a second tiny kernel sums the partials in chunk order,
// so gamma is deterministic (no atomics).
#include "common.cuh"

namespace sa {

constexpr int kHashThreads = 256;
constexpr int kTokPerCta = 64;

template <int NBLK>  // NBLK = ceil(d / 128)
__global__ void __launch_bounds__(kHashThreads) sign_hash_kernel(
    const float* __restrict__ x, int n, int d, int heads, int dk, int W, int chunks,
    uint32_t* __restrict__ codes, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int dwords = d >> 5;                                    // words per row
  uint32_t* sm_codes = reinterpret_cast<uint32_t*>(smem_raw);   // [kTokPerCta][dwords]
  float* sm_cs = reinterpret_cast<float*>(sm_codes + kTokPerCta * dwords);  // [8][d]

  const int b = blockIdx.y, chunk = blockIdx.x;
  const int t0 = chunk * kTokPerCta;
  const int rows = min(kTokPerCta, n - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  float acc[NBLK][4];
#pragma unroll
  for (int j = 0; j < NBLK; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

  for (int r = warp; r < rows; r += kHashThreads / 32) {
    const float* row = x + (size_t(b) * n + t0 + r) * d;
#pragma unroll
    for (int j = 0; j < NBLK; ++j) {
      const int c0 = j * 128 + lane * 4;
      const bool act = c0 < d;  // uniform within each 8-lane group (d % 32 == 0)
      float4 v = act ? __ldg(reinterpret_cast<const float4*>(row + c0)) : make_float4(0, 0, 0, 0);
      acc[j][0] += fabsf(v.x);
      acc[j][1] += fabsf(v.y);
      acc[j][2] += fabsf(v.z);
      acc[j][3] += fabsf(v.w);
      uint32_t nib = uint32_t(!(v.x < 0.f)) | (uint32_t(!(v.y < 0.f)) << 1) |
                     (uint32_t(!(v.z < 0.f)) << 2) | (uint32_t(!(v.w < 0.f)) << 3);
      uint32_t w = nib << (4 * (lane & 7));
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if (act && (lane & 7) == 0) sm_codes[r * dwords + (c0 >> 5)] = w;
    }
  }
  // per-channel |x| sums of this warp → smem
#pragma unroll
  for (int j = 0; j < NBLK; ++j) {
    const int c0 = j * 128 + lane * 4;
    if (c0 < d) {
#pragma unroll
      for (int i = 0; i < 4; ++i) sm_cs[warp * d + c0 + i] = acc[j][i];
    }
  }
  __syncthreads();

  // codes out: [head][token][word] order for coalescing
  const int total = heads * rows * W;
  for (int idx = threadIdx.x; idx < total; idx += kHashThreads) {
    const int wi = idx % W;
    const int r = (idx / W) % rows;
    const int h = idx / (W * rows);
    uint32_t word;
    if (dk >= 32) {
      word = sm_codes[r * dwords + h * (dk >> 5) + wi];
    } else {
      const int bit0 = h * dk;
      word = (sm_codes[r * dwords + (bit0 >> 5)] >> (bit0 & 31)) & ((1u << dk) - 1u);
    }
    codes[((size_t(b) * heads + h) * n + t0 + r) * W + wi] = word;
  }

  // per-head partial sums: fixed-order float64 reduction (warps, then channels)
  for (int h = warp; h < heads; h += kHashThreads / 32) {
    double s = 0.0;
    for (int c = h * dk + lane; c < (h + 1) * dk; c += 32) {
      double cs = 0.0;
      for (int w8 = 0; w8 < kHashThreads / 32; ++w8) cs += double(sm_cs[w8 * d + c]);
      s += cs;
    }
    s = warp_sum(s);
    if (lane == 0) partial[(size_t(b) * chunks + chunk) * heads + h] = s;
  }
}

// Fast path for d dividing 1024 (d = 32, 64, 128, 256, 512): the CTA's token
// chunk is one contiguous run of float4s; thread t always lands on channels
// 4t mod d, so |x| accumulates in four registers, and every warp-load covers
// whole 32-channel words (8-lane OR butterfly). All 32 lanes are busy for
// every d, each thread keeps d/4 independent 128-bit loads in flight.
constexpr int kStreamTok = 256;

// T threads per CTA with 4·T a multiple of D (T = 256 when D divides 1024;
// T = lcm(D/4, 32) scaled to >= 128 otherwise, e.g. 160 for D = 160), so each
// thread's channel 4t mod D is the same in every iteration.
template <int D, int T = kHashThreads, int R = kStreamTok>   // R tokens per CTA
__global__ void __launch_bounds__(T) sign_hash_stream_kernel(
    const float* __restrict__ x, int n, int heads, int dk, int W, int chunks,
    uint32_t* __restrict__ codes, double* __restrict__ partial) {
  static_assert((4 * T) % D == 0 && T % 32 == 0, "fixed channel per thread");
  constexpr int DW = D / 32;
  __shared__ uint32_t sm_codes[R * DW];
  __shared__ double red[T];
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int t0 = chunk * R;
  const int rows = min(R, n - t0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float4* src = reinterpret_cast<const float4*>(x + (size_t(b) * n + t0) * D);
  const int nf4 = rows * (D / 4);
  const int c = (4 * tid) % D;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  // the loop bound is CTA-uniform, so every lane reaches the shuffles; nf4 is a
  // multiple of 8 (D/4 >= 8), so an 8-lane word group is either fully active
  // or fully past the end (and then never stored).
#pragma unroll 4
  for (int base = 0; base < nf4; base += T) {
    const int f = base + tid;
    const bool act = f < nf4;
    const float4 v = act ? __ldg(src + f) : make_float4(0.f, 0.f, 0.f, 0.f);
    a0 += fabsf(v.x);
    a1 += fabsf(v.y);
    a2 += fabsf(v.z);
    a3 += fabsf(v.w);
    uint32_t nib = uint32_t(!(v.x < 0.f)) | (uint32_t(!(v.y < 0.f)) << 1) |
                   (uint32_t(!(v.z < 0.f)) << 2) | (uint32_t(!(v.w < 0.f)) << 3);
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    if (act && (lane & 7) == 0) {
      const int r = (4 * f) / D;
      sm_codes[r * DW + c / 32] = w;
    }
  }
  red[tid] = double(a0) + double(a1) + double(a2) + double(a3);
  __syncthreads();

  const int total = heads * rows * W;
  for (int idx = tid; idx < total; idx += T) {
    const int wi = idx % W;
    const int r = (idx / W) % rows;
    const int h = idx / (W * rows);
    uint32_t word;
    if (dk >= 32) {
      word = sm_codes[r * DW + h * (dk >> 5) + wi];
    } else {
      const int bit0 = h * dk;
      word = (sm_codes[r * DW + (bit0 >> 5)] >> (bit0 & 31)) & ((1u << dk) - 1u);
    }
    codes[((size_t(b) * heads + h) * n + t0 + r) * W + wi] = word;
  }
  // per head: fixed-order sum over the threads whose 4 channels lie in the head
  // (dk >= 4 so a thread's channels never straddle two heads)
  for (int h = warp; h < heads; h += T / 32) {
    double s = 0.0;
    for (int j = lane; j < T; j += 32)
      if (((4 * j) % D) / dk == h) s += red[j];
    s = warp_sum(s);
    if (lane == 0) partial[(size_t(b) * chunks + chunk) * heads + h] = s;
  }
}

__global__ void gamma_finalize_kernel(const double* __restrict__ partial, int BH, int heads,
                                      int chunks, double inv_count, float* __restrict__ gamma) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BH) return;
  const int b = i / heads, h = i % heads;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += partial[(size_t(b) * chunks + c) * heads + h];
  gamma[i] = float(s * inv_count);
}

}  // namespace sa

using namespace sa;

extern "C" size_t sa_sign_hash_workspace(int64_t B, int64_t n, int64_t d, int64_t heads) {
  (void)d;
  return size_t(B) * size_t(cdiv(n, kTokPerCta)) * size_t(heads) * sizeof(double);   // >= stream chunks
}

extern "C" int sa_sign_hash(const float* x, int64_t B, int64_t n, int64_t d, int64_t heads,
                            uint32_t* codes, float* gamma, void* ws, size_t ws_bytes,
                            void* stream) {
  SA_REQUIRE(B > 0 && n > 0 && d > 0 && heads > 0, SA_ERR_SHAPE,
             "sa_sign_hash: empty extents B=%lld n=%lld d=%lld", (long long)B, (long long)n,
             (long long)d);
  SA_REQUIRE(d % heads == 0, SA_ERR_SHAPE, "sa_sign_hash: d %lld not divisible by heads %lld",
             (long long)d, (long long)heads);
  const int64_t dk = d / heads;
  SA_REQUIRE(d % 32 == 0 && d <= 512 && (dk % 32 == 0 || 32 % dk == 0), SA_ERR_SHAPE,
             "sa_sign_hash: unsupported d=%lld dk=%lld (need d%%32==0, d<=512, dk|32 or 32|dk)",
             (long long)d, (long long)dk);
  SA_REQUIRE(ws_bytes >= sa_sign_hash_workspace(B, n, d, heads), SA_ERR_VALUE,
             "sa_sign_hash: workspace too small");
  const int W = int(cdiv(dk, 32));
  double* partial = static_cast<double*>(ws);
  cudaStream_t s = as_stream(stream);
  int chunks;
  if (1024 % d == 0) {
    chunks = int(cdiv(n, kStreamTok));
    dim3 grid(chunks, unsigned(B));
#define SA_HASH_STREAM(DV)                                                                \
  case DV:                                                                                \
    sign_hash_stream_kernel<DV><<<grid, kHashThreads, 0, s>>>(x, int(n), int(heads), int(dk), \
                                                              W, chunks, codes, partial); \
    break;
    switch (d) {
      SA_HASH_STREAM(32)
      SA_HASH_STREAM(64)
      SA_HASH_STREAM(128)
      SA_HASH_STREAM(256)
      SA_HASH_STREAM(512)
    }
#undef SA_HASH_STREAM
  } else if (d == 96 || d == 160 || d == 192 || d == 320 || d == 384) {
    constexpr int R = 64;   // wide rows: 64 tokens per CTA (enough CTAs at small n)
    chunks = int(cdiv(n, R));
    dim3 grid(chunks, unsigned(B));
#define SA_HASH_STREAM_T(DV, TV)                                                            \
  case DV:                                                                                  \
    sign_hash_stream_kernel<DV, TV, R><<<grid, TV, 0, s>>>(x, int(n), int(heads), int(dk), \
                                                           W, chunks, codes, partial);     \
    break;
    switch (d) {
      SA_HASH_STREAM_T(96, 192)
      SA_HASH_STREAM_T(160, 160)
      SA_HASH_STREAM_T(192, 192)
      SA_HASH_STREAM_T(320, 160)
      SA_HASH_STREAM_T(384, 192)
    }
#undef SA_HASH_STREAM_T
  } else {
    chunks = int(cdiv(n, kTokPerCta));
    const size_t smem = size_t(kTokPerCta) * (d / 32) * 4 + size_t(kHashThreads / 32) * d * 4;
    dim3 grid(chunks, unsigned(B));
    const int nblk = int(cdiv(d, 128));
    switch (nblk) {
      case 1:
        sign_hash_kernel<1><<<grid, kHashThreads, smem, s>>>(x, int(n), int(d), int(heads),
                                                            int(dk), W, chunks, codes, partial);
        break;
      case 2:
        sign_hash_kernel<2><<<grid, kHashThreads, smem, s>>>(x, int(n), int(d), int(heads),
                                                            int(dk), W, chunks, codes, partial);
        break;
      default:
        sign_hash_kernel<4><<<grid, kHashThreads, smem, s>>>(x, int(n), int(d), int(heads),
                                                            int(dk), W, chunks, codes, partial);
        break;
    }
  }
  const int BH = int(B * heads);
  gamma_finalize_kernel<<<int(cdiv(BH, 256)), 256, 0, s>>>(partial, BH, int(heads), chunks,
                                                           1.0 / double(n * dk), gamma);
  count_launch(2);
  SA_LAUNCH_CHECK("sa_sign_hash");
  return SA_OK;
}
