// K2a / K2b — additive binary attention over packed {0,1} Q/K codes.
//
// Reference semantics (attention.py:113-120 with binary features from
// model.py:355-358): with features qf = gq*c_q, kf = gk*c_k,
//   kv[a][:] = gk * sum_{j : c_k[j][a] = 1} v_j          (additions only)
//   cnt[a]   = popcount over tokens of code bit a        (integer)
//   num_i    = gq * sum_{a : c_q[i][a] = 1} kv[a]        (additions only)
//   D_i      = sum_{a : c_q[i][a] = 1} cnt[a]            (integer)
//   out_i    = num_i / (gq*gk*D_i + eps)
// plus the DWConv branch on V over the ceil(sqrt(n))^2 token grid
// (attention.py:170-179), added before W_O (model.py:367-373).
//
// Linear (K^T V first) order, three kernels:
//   1. kv_partial: grid (split, B*heads); a CTA stages a token chunk of V and
//      the K codes in shared memory and accumulates S[a][c] with predicated
//      adds (no multiplies); writes per-split partials.
//   2. kv_reduce: fixed-order sum of the splits (deterministic), scale by gk.
//   3. attn_out: grid (token chunk, B); kv of each head in shared memory, one
//      warp per token walks the SET bits of the query code (warp-uniform loop)
//      and adds kv rows; DWConv taps read V from L2; one store per output.
// Quadratic (QK first, DeiT-T): S_ij = popc(cq_i & ck_j) in registers/SMEM,
// then out_i = sum_j S_ij v_j (S never leaves the SM).
#include "common.cuh"

namespace sa {

constexpr int kAttnThreads = 256;
constexpr int kKvElems = 8192; // V floats staged per kv_partial CTA (32 KB)
__host__ __device__ constexpr int kv_tok(int dk) { return kKvElems / dk; }
constexpr int kOutTok = 64;    // tokens per attn_out CTA

template <int DK>
__global__ void __launch_bounds__(kAttnThreads) kv_partial_kernel(
    const uint32_t* __restrict__ codes_k, const float* __restrict__ v, int n, int d, int heads,
    int nsplit, float* __restrict__ part, int* __restrict__ cnt_part) {
  constexpr int W = (DK + 31) / 32;
  constexpr int ROWS = DK / 8;             // rows a per warp
  constexpr int COLS = (DK + 31) / 32;     // columns per lane
  constexpr int kKvTok = kv_tok(DK);
  __shared__ __align__(16) float sv[kKvTok * DK];
  __shared__ uint32_t sc[kKvTok * W];
  __shared__ int scnt[8][DK];

  const int bh = blockIdx.y, split = blockIdx.x;
  const int b = bh / heads, h = bh % heads;
  const int j0 = split * kKvTok;
  const int rows = min(kKvTok, n - j0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // stage V chunk (head slice) and K codes
  for (int idx = threadIdx.x; idx < rows * (DK / 4); idx += kAttnThreads) {
    const int r = idx / (DK / 4), q = idx % (DK / 4);
    const float4 val = __ldg(reinterpret_cast<const float4*>(
        v + (size_t(b) * n + j0 + r) * d + h * DK + q * 4));
    *reinterpret_cast<float4*>(&sv[r * DK + q * 4]) = val;
  }
  for (int idx = threadIdx.x; idx < rows * W; idx += kAttnThreads)
    sc[idx] = codes_k[(size_t(bh) * n + j0) * W + idx];
  __syncthreads();

  float acc[ROWS][COLS];
#pragma unroll
  for (int i = 0; i < ROWS; ++i)
#pragma unroll
    for (int c = 0; c < COLS; ++c) acc[i][c] = 0.f;

  if (DK >= 32) {
    const int a0 = warp * ROWS;          // rows a0 .. a0+ROWS-1 (within one word)
    const int wi = a0 >> 5, sh = a0 & 31;
    for (int r = 0; r < rows; ++r) {
      const uint32_t bits = sc[r * W + wi] >> sh;
      float vv[COLS];
#pragma unroll
      for (int c = 0; c < COLS; ++c) vv[c] = sv[r * DK + c * 32 + lane];
#pragma unroll
      for (int i = 0; i < ROWS; ++i) {
        if ((bits >> i) & 1u) {
#pragma unroll
          for (int c = 0; c < COLS; ++c) acc[i][c] += vv[c];
        }
      }
    }
  } else {  // DK == 16: lane -> (row half, column)
    const int a = warp * ROWS + (lane >> 4);
    const int c = lane & 15;
    for (int r = 0; r < rows; ++r) {
      const uint32_t bits = sc[r];
      if ((bits >> a) & 1u) acc[0][0] += sv[r * DK + c];
    }
  }

  // popcounts of K code bits over the chunk (bit a = lane + 32*word)
  for (int a = lane; a < DK; a += 32) {
    int cc = 0;
    for (int r = warp; r < rows; r += kAttnThreads / 32) cc += (sc[r * W + (a >> 5)] >> (a & 31)) & 1;
    scnt[warp][a] = cc;
  }

  float* dst = part + (size_t(bh) * nsplit + split) * DK * DK;
  if (DK >= 32) {
#pragma unroll
    for (int i = 0; i < ROWS; ++i)
#pragma unroll
      for (int c = 0; c < COLS; ++c) dst[(warp * ROWS + i) * DK + c * 32 + lane] = acc[i][c];
  } else {
    dst[(warp * ROWS + (lane >> 4)) * DK + (lane & 15)] = acc[0][0];
  }
  __syncthreads();
  if (threadIdx.x < DK) {
    int cc = 0;
    for (int w8 = 0; w8 < kAttnThreads / 32; ++w8) cc += scnt[w8][threadIdx.x];
    cnt_part[(size_t(bh) * nsplit + split) * DK + threadIdx.x] = cc;
  }
}

__global__ void kv_reduce_kernel(const float* __restrict__ part, const int* __restrict__ cnt_part,
                                 const float* __restrict__ gamma_k, int dk, int nsplit,
                                 float* __restrict__ kv, int* __restrict__ cnt) {
  const int bh = blockIdx.x;
  const int dd = dk * dk;
  const float g = gamma_k[bh];
  for (int e = threadIdx.x; e < dd; e += blockDim.x) {
    float s = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) s += part[(size_t(bh) * nsplit + sp) * dd + e];
    kv[size_t(bh) * dd + e] = g * s;
  }
  for (int a = threadIdx.x; a < dk; a += blockDim.x) {
    int c = 0;
    for (int sp = 0; sp < nsplit; ++sp) c += cnt_part[(size_t(bh) * nsplit + sp) * dk + a];
    cnt[bh * dk + a] = c;
  }
}

__device__ __forceinline__ float dwconv_at(const float* __restrict__ vb, const float* __restrict__ dw,
                                           int n, int side, int d, int t, int ch) {
  // zero-padded 3x3 taps in the reference's (row, col) tap order (tensor.py:191-194)
  const int r = t / side, c = t % side;
  float s = 0.f;
#pragma unroll
  for (int di = 0; di < 3; ++di) {
#pragma unroll
    for (int dj = 0; dj < 3; ++dj) {
      const int rr = r + di - 1, cc = c + dj - 1;
      if (rr < 0 || rr >= side || cc < 0 || cc >= side) continue;
      const int idx = rr * side + cc;
      if (idx >= n) continue;
      s = fmaf(__ldg(vb + size_t(idx) * d + ch), __ldg(dw + (di * 3 + dj) * d + ch), s);
    }
  }
  return s;
}

template <int DK>
__global__ void __launch_bounds__(kAttnThreads) attn_out_kernel(
    const uint32_t* __restrict__ codes_q, const float* __restrict__ gamma_q,
    const float* __restrict__ gamma_k, const float* __restrict__ kv, const int* __restrict__ cnt,
    const float* __restrict__ v, const float* __restrict__ dw, float* __restrict__ out, int n,
    int d, int heads, int side, float eps) {
  constexpr int W = (DK + 31) / 32;
  constexpr int COLS = (DK + 31) / 32;
  __shared__ __align__(16) float skv[DK * DK];
  __shared__ int scnt[DK];
  const int b = blockIdx.y;
  const int t0 = blockIdx.x * kOutTok;
  const int rows = min(kOutTok, n - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* vb = v + size_t(b) * n * d;

  for (int h = 0; h < heads; ++h) {
    const int bh = b * heads + h;
    __syncthreads();
    for (int e = threadIdx.x; e < DK * DK; e += kAttnThreads) skv[e] = kv[size_t(bh) * DK * DK + e];
    if (threadIdx.x < DK) scnt[threadIdx.x] = cnt[bh * DK + threadIdx.x];
    __syncthreads();
    const float gq = gamma_q[bh], gk = gamma_k[bh];
    for (int r = warp; r < rows; r += kAttnThreads / 32) {
      const int t = t0 + r;
      float acc[COLS];
#pragma unroll
      for (int c = 0; c < COLS; ++c) acc[c] = 0.f;
      int D = 0;
#pragma unroll
      for (int wi = 0; wi < W; ++wi) {
        uint32_t m = codes_q[(size_t(bh) * n + t) * W + wi];
        while (m) {  // warp-uniform: every lane walks the same set bits
          const int a = wi * 32 + __ffs(m) - 1;
          m &= m - 1;
          D += scnt[a];
#pragma unroll
          for (int c = 0; c < COLS; ++c) {
            const int col = c * 32 + lane;
            if (col < DK) acc[c] += skv[a * DK + col];
          }
        }
      }
      const float den = gq * gk * float(D) + eps;
#pragma unroll
      for (int c = 0; c < COLS; ++c) {
        const int col = c * 32 + lane;
        if (col >= DK) continue;
        const int ch = h * DK + col;
        float o = (gq * acc[c]) / den;
        if (dw) o += dwconv_at(vb, dw, n, side, d, t, ch);
        out[(size_t(b) * n + t) * d + ch] = o;
      }
    }
  }
}

// Output pass for dk <= 32, one CTA per (band of token-grid rows, image):
//  - the V rows of the band plus one halo row above/below are staged in shared
//    memory with contiguous 128-bit copies, so the 9 DWConv taps are smem reads;
//  - per head, kv is folded into Four-Russians nibble tables
//      T[g][m][c] = sum_{i in m} kv[4g+i][c],  Tc[g][m] = sum_{i in m} cnt[4g+i]
//    (each entry one addition from a smaller subset), so a token's additive
//    Q·(K^T V) is dk/4 independent table lookups + adds (no multiplies);
//  - one warp per token, lane = channel of the head: coalesced 128 B stores.
template <int DK>
__global__ void __launch_bounds__(kAttnThreads) attn_out_band_kernel(
    const uint32_t* __restrict__ codes_q, const float* __restrict__ gamma_q,
    const float* __restrict__ gamma_k, const float* __restrict__ kv, const int* __restrict__ cnt,
    const float* __restrict__ v, const float* __restrict__ dw, float* __restrict__ out, int n,
    int d, int heads, int side, int band_rows, float eps) {
  constexpr int G = DK / 4;                 // nibble groups
  extern __shared__ __align__(16) float sm[];
  float* T = sm;                            // [G][16][DK]
  int* Tc = reinterpret_cast<int*>(T + G * 16 * DK);     // [G][16]
  uint32_t* Cs = reinterpret_cast<uint32_t*>(Tc + G * 16);  // [heads][band tokens]
  const int b = blockIdx.y;
  const int r0 = blockIdx.x * band_rows;
  const int t_lo = r0 * side, t_hi = min(n, (r0 + band_rows) * side);
  const int h_lo = max(0, (r0 - 1) * side), h_hi = min(n, (r0 + band_rows + 1) * side);
  const int nt = t_hi - t_lo;
  // V band on a zero-padded grid: (band_rows+2) x (side+2) cells of d floats;
  // cell (R, C) holds token (r0-1+R)*side + (C-1) when it exists, else zeros
  float* Vs = reinterpret_cast<float*>(Cs + ((heads * band_rows * side + 3) & ~3));
  const int pw = side + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* vb = v + size_t(b) * n * d;
  if (dw) {
    const int d4 = d / 4;
    float4* dst = reinterpret_cast<float4*>(Vs);
    const int ncell4 = (band_rows + 2) * pw * d4;
    for (int i = threadIdx.x; i < ncell4; i += kAttnThreads) {
      const int c4 = i % d4, cell = i / d4;
      const int R = cell / pw, C = cell % pw;
      const int rr = r0 - 1 + R, cc = C - 1;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rr >= 0 && rr < side && cc >= 0 && cc < side) {
        const int idx = rr * side + cc;
        if (idx < n) val = __ldg(reinterpret_cast<const float4*>(vb + size_t(idx) * d) + c4);
      }
      dst[i] = val;
    }
  }
  for (int i = threadIdx.x; i < heads * nt; i += kAttnThreads) {  // query codes of the band
    const int h = i / nt, t = i % nt;
    Cs[h * nt + t] = __ldg(codes_q + (size_t(b) * heads + h) * n + t_lo + t);
  }
  for (int h = 0; h < heads; ++h) {
    const int bh = b * heads + h;
    __syncthreads();  // previous head's tables are no longer read
    if (threadIdx.x < G * DK) {
      const int g = threadIdx.x / DK, c = threadIdx.x % DK;
      const float* kvh = kv + size_t(bh) * DK * DK;
      float row[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) row[i] = kvh[(4 * g + i) * DK + c];
      float val[16];
      val[0] = 0.f;
#pragma unroll
      for (int m = 1; m < 16; ++m) val[m] = val[m & (m - 1)] + row[__ffs(m) - 1];
#pragma unroll
      for (int m = 0; m < 16; ++m) T[(g * 16 + m) * DK + c] = val[m];
    }
    if (threadIdx.x < G) {
      const int g = threadIdx.x;
      int cr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cr[i] = cnt[bh * DK + 4 * g + i];
      int val[16];
      val[0] = 0;
#pragma unroll
      for (int m = 1; m < 16; ++m) val[m] = val[m & (m - 1)] + cr[__ffs(m) - 1];
#pragma unroll
      for (int m = 0; m < 16; ++m) Tc[g * 16 + m] = val[m];
    }
    float tap[9];
    const bool lane_ok = lane < DK;
    const int ch = h * DK + (lane_ok ? lane : 0);
#pragma unroll
    for (int q = 0; q < 9; ++q) tap[q] = dw ? __ldg(dw + q * d + ch) : 0.f;
    __syncthreads();
    const float gq = gamma_q[bh], gk = gamma_k[bh];
    const float gg = gq * gk;
    const uint32_t* cq = Cs + h * nt - t_lo;
#pragma unroll 2
    for (int t = t_lo + warp; t < t_hi; t += kAttnThreads / 32) {
      const uint32_t w = cq[t];
      float acc = 0.f;
      int D = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int m = (w >> (4 * g)) & 15;
        if (lane_ok) acc += T[(g * 16 + m) * DK + lane];
        D += Tc[g * 16 + m];
      }
      float o = (gq * acc) * __frcp_rn(gg * float(D) + eps);
      if (dw) {
        // token (r, c) sits at padded cell (r - r0 + 1, c + 1); taps in the
        // reference's (row, col) order (tensor.py:191-194), zeros outside
        const int r = t / side, cc = t % side;
        const float* base = Vs + ((r - r0) * pw + cc) * d + ch;   // cell (R-1, C-1)
        float s = 0.f;
#pragma unroll
        for (int di = 0; di < 3; ++di)
#pragma unroll
          for (int dj = 0; dj < 3; ++dj) s = fmaf(base[(di * pw + dj) * d], tap[di * 3 + dj], s);
        o += s;
      }
      if (lane_ok) out[(size_t(b) * n + t) * d + ch] = o;
    }
  }
}

// quadratic Hamming form: one CTA per (query chunk, b*heads)
constexpr int kHamQ = 32;
template <int DK>
__global__ void __launch_bounds__(kAttnThreads) hamming_attn_kernel(
    const uint32_t* __restrict__ codes_q, const uint32_t* __restrict__ codes_k,
    const float* __restrict__ gamma_q, const float* __restrict__ gamma_k,
    const float* __restrict__ v, const float* __restrict__ dw, float* __restrict__ out, int n,
    int d, int heads, int side, float eps) {
  constexpr int W = (DK + 31) / 32;
  constexpr int COLS = (DK + 31) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sv = reinterpret_cast<float*>(smem_raw);                 // [n][DK]
  uint32_t* sk = reinterpret_cast<uint32_t*>(sv + size_t(n) * DK);  // [n][W]
  int* sS = reinterpret_cast<int*>(sk + size_t(n) * W);           // [8 warps][n]
  const int bh = blockIdx.y, b = bh / heads, h = bh % heads;
  const int i0 = blockIdx.x * kHamQ;
  const int rows = min(kHamQ, n - i0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* vb = v + size_t(b) * n * d;
  for (int idx = threadIdx.x; idx < n * (DK / 4); idx += kAttnThreads) {
    const int r = idx / (DK / 4), q = idx % (DK / 4);
    *reinterpret_cast<float4*>(&sv[r * DK + q * 4]) =
        __ldg(reinterpret_cast<const float4*>(vb + size_t(r) * d + h * DK + q * 4));
  }
  for (int idx = threadIdx.x; idx < n * W; idx += kAttnThreads)
    sk[idx] = codes_k[size_t(bh) * n * W + idx];
  __syncthreads();
  const float gq = gamma_q[bh], gk = gamma_k[bh];
  const float g = gq * gk;
  int* myS = sS + warp * n;
  for (int r = warp; r < rows; r += kAttnThreads / 32) {
    const int i = i0 + r;
    uint32_t q[W];
#pragma unroll
    for (int wi = 0; wi < W; ++wi) q[wi] = codes_q[(size_t(bh) * n + i) * W + wi];
    int Dl = 0;
    for (int j = lane; j < n; j += 32) {
      int s = 0;
#pragma unroll
      for (int wi = 0; wi < W; ++wi) s += __popc(q[wi] & sk[j * W + wi]);
      myS[j] = s;
      Dl += s;
    }
    int D = Dl;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) D += __shfl_xor_sync(0xffffffffu, D, o);
    __syncwarp();
    float acc[COLS];
#pragma unroll
    for (int c = 0; c < COLS; ++c) acc[c] = 0.f;
    for (int j = 0; j < n; ++j) {
      const float s = float(myS[j]);   // integer <= dk, exact
#pragma unroll
      for (int c = 0; c < COLS; ++c) {
        const int col = c * 32 + lane;
        if (col < DK) acc[c] = fmaf(s, sv[j * DK + col], acc[c]);
      }
    }
    __syncwarp();
    const float den = g * float(D) + eps;
#pragma unroll
    for (int c = 0; c < COLS; ++c) {
      const int col = c * 32 + lane;
      if (col >= DK) continue;
      const int ch = h * DK + col;
      float o = (g * acc[c]) / den;
      if (dw) o += dwconv_at(vb, dw, n, side, d, i, ch);
      out[(size_t(b) * n + i) * d + ch] = o;
    }
  }
}

__global__ void dwconv_tokens_kernel(const float* __restrict__ v, const float* __restrict__ dw,
                                     float* __restrict__ out, int64_t total, int n, int d,
                                     int side, int accumulate) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int ch = int(i % d);
  const int64_t tok = i / d;
  const int t = int(tok % n);
  const int64_t b = tok / n;
  const float s = dwconv_at(v + b * n * d, dw, n, side, d, t, ch);
  out[i] = accumulate ? out[i] + s : s;
}

__global__ void popc_cnt_kernel(const uint32_t* __restrict__ codes_k, int n, int dk, int W,
                                int BH, int* __restrict__ cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BH * dk) return;
  const int bh = i / dk, a = i % dk;
  int c = 0;
  for (int j = 0; j < n; ++j) c += (codes_k[(size_t(bh) * n + j) * W + (a >> 5)] >> (a & 31)) & 1;
  cnt[i] = c;
}

__global__ void popc_D_kernel(const uint32_t* __restrict__ codes_q, const int* __restrict__ cnt,
                              int n, int dk, int W, int BH, int* __restrict__ D) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BH * n) return;
  const int bh = i / n;
  int s = 0;
  for (int a = 0; a < dk; ++a)
    if ((codes_q[size_t(i) * W + (a >> 5)] >> (a & 31)) & 1) s += cnt[bh * dk + a];
  D[i] = s;
}

__global__ void popc_S_kernel(const uint32_t* __restrict__ codes_q,
                              const uint32_t* __restrict__ codes_k, int n, int W, int64_t total,
                              int* __restrict__ S) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int j = int(i % n);
  const int64_t qi = i / n;          // bh*n + query
  const int64_t bh = qi / n;
  int s = 0;
  for (int w = 0; w < W; ++w) s += __popc(codes_q[qi * W + w] & codes_k[(bh * n + j) * W + w]);
  S[i] = s;
}

static int grid_side(int64_t n) {
  int64_t s = 0;
  while (s * s < n) ++s;
  return int(s);
}

static int check_attn_shapes(const char* who, int64_t B, int64_t n, int64_t d, int64_t heads) {
  SA_REQUIRE(B > 0 && n > 0 && d > 0 && heads > 0, SA_ERR_SHAPE, "%s: empty extents", who);
  SA_REQUIRE(d % heads == 0, SA_ERR_SHAPE, "%s: model_dim %lld not divisible by heads %lld", who,
             (long long)d, (long long)heads);
  const int64_t dk = d / heads;
  SA_REQUIRE(dk == 16 || dk == 32 || dk == 64, SA_ERR_SHAPE,
             "%s: head dim %lld unsupported (16, 32 or 64)", who, (long long)dk);
  return SA_OK;
}

int binattn_tc_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                      const float* v, const float* dw, float* out, int64_t B, int64_t n,
                      int64_t d, int64_t heads, float eps, cudaStream_t s);
int hamming_tc_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                      const float* v, const float* dw, float* out, int64_t B, int64_t n,
                      int64_t d, int64_t heads, float eps, cudaStream_t s);
int binattn_fused_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                         const float* v, const float* dw, float* out, int64_t B, int64_t n,
                         int64_t d, int64_t heads, float eps, cudaStream_t s);
size_t binattn_split_ws_bytes(int64_t B, int64_t heads);
int binattn_split_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                         const float* v, const float* dw, float* out, int64_t B, int64_t n,
                         int64_t d, int64_t heads, float eps, void* ws, size_t ws_bytes,
                         cudaStream_t s);
int binattn_stream_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                          const float* v, const float* dw, float* out, int64_t B, int64_t n,
                          int64_t d, int64_t heads, float eps, cudaStream_t s);
// 0: product choice — dk = 64: tensor-core cluster kernel (binattn_tc.cu);
// dk = 32: CUDA-core single-pass cluster kernel (binattn_fused.cu), measured
// faster at dk = 32 (profiles/r2_attn_bench.txt); 1: multi-kernel; 2: split
// two-kernel form of the CUDA-core fused kernel (bit-identical to it); 3: the
// tensor-core cluster kernel at any dk it supports; 4: = 0; 5 (debug build
// only): the streaming tensor-core kernel (binattn_stream.cu, measured slower:
// DESIGN.md §5)

}  // namespace sa

using namespace sa;

SA_DEBUG_SWITCH(int, g_attn_mode, 0, sa_debug_attn_mode)
// quadratic form: 0 = tensor-core kernel (hamming_tc.cu) when the shape allows,
// 1 = the CUDA-core kernel below
SA_DEBUG_SWITCH(int, g_ham_mode, 0, sa_debug_ham_mode)

extern "C" size_t sa_linear_binary_attn_workspace(int64_t B, int64_t n, int64_t d, int64_t heads) {
  if (heads <= 0 || d % heads) return 0;
  const int64_t dk = d / heads;
  const int64_t nsplit = cdiv(n, kv_tok(int(dk)));
  const int64_t BH = B * heads;
  size_t bytes = 0;
  bytes += size_t(BH * nsplit * dk * dk) * 4;  // partial S
  bytes += size_t(BH * nsplit * dk) * 4;       // partial counts
  bytes += size_t(BH * dk * dk) * 4;           // kv
  bytes += size_t(BH * dk) * 4;                // cnt
  if (dk == 32 && binattn_split_ws_bytes(B, heads) > bytes) bytes = binattn_split_ws_bytes(B, heads);
  return bytes + 256;
}

extern "C" int sa_linear_binary_attn(const uint32_t* codes_q, const uint32_t* codes_k,
                                     const float* gamma_q, const float* gamma_k, const float* v,
                                     const float* dw, float* out, int64_t B, int64_t n, int64_t d,
                                     int64_t heads, float eps, void* ws, size_t ws_bytes,
                                     void* stream) {
  int st = check_attn_shapes("sa_linear_binary_attn", B, n, d, heads);
  if (st) return st;
  SA_REQUIRE(ws_bytes >= sa_linear_binary_attn_workspace(B, n, d, heads), SA_ERR_VALUE,
             "sa_linear_binary_attn: workspace too small");
  const int64_t dk = d / heads;
#ifdef SA_DEBUG
  if (g_attn_mode == 5) {
    st = binattn_stream_launch(codes_q, codes_k, gamma_q, gamma_k, v, dw, out, B, n, d, heads, eps,
                               as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
#endif
  if (dk == 32 && g_attn_mode == 2) {
    st = binattn_split_launch(codes_q, codes_k, gamma_q, gamma_k, v, dw, out, B, n, d, heads, eps,
                              ws, ws_bytes, as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  if ((dk == 64 && (g_attn_mode == 0 || g_attn_mode == 4)) || g_attn_mode == 3) {
    st = binattn_tc_launch(codes_q, codes_k, gamma_q, gamma_k, v, dw, out, B, n, d, heads, eps,
                           as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  if (dk == 32 && (g_attn_mode == 0 || g_attn_mode == 4)) {
    st = binattn_fused_launch(codes_q, codes_k, gamma_q, gamma_k, v, dw, out, B, n, d, heads, eps,
                              as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  const int nsplit = int(cdiv(n, kv_tok(int(dk))));
  const int64_t BH = B * heads;
  float* part = static_cast<float*>(ws);
  int* cnt_part = reinterpret_cast<int*>(part + BH * nsplit * dk * dk);
  float* kv = reinterpret_cast<float*>(cnt_part + BH * nsplit * dk);
  int* cnt = reinterpret_cast<int*>(kv + BH * dk * dk);
  cudaStream_t s = as_stream(stream);
  dim3 g1(nsplit, unsigned(BH));
  dim3 g3(unsigned(cdiv(n, kOutTok)), unsigned(B));
  const int side = grid_side(n);
  // band geometry for the dk <= 32 output pass: rows of the token grid per CTA
  // so that the staged V band (+2 halo rows) stays within ~64 KB
  const int64_t row_bytes = int64_t(side + 2) * d * 4;   // padded grid row
  int band_rows = int(64 * 1024 / row_bytes) - 2;
  band_rows = band_rows < 1 ? 1 : (band_rows > side ? side : band_rows);
  const int nbands = int(cdiv(cdiv(n, side), band_rows));
  const size_t band_smem = (dk / 4) * 16 * (dk + 1) * 4 +
                           size_t((heads * band_rows * side + 3) & ~3) * 4 +
                           (dw ? size_t(band_rows + 2) * row_bytes : 0);
#define SA_ATTN_CASE(DKV)                                                                     \
  case DKV:                                                                                   \
    kv_partial_kernel<DKV><<<g1, kAttnThreads, 0, s>>>(codes_k, v, int(n), int(d), int(heads), \
                                                       nsplit, part, cnt_part);              \
    kv_reduce_kernel<<<unsigned(BH), 256, 0, s>>>(part, cnt_part, gamma_k, DKV, nsplit, kv,  \
                                                  cnt);                                       \
    if (DKV <= 32) {                                                                          \
      cudaFuncSetAttribute(attn_out_band_kernel<DKV <= 32 ? DKV : 32>,                        \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(band_smem));      \
      attn_out_band_kernel<DKV <= 32 ? DKV : 32>                                              \
          <<<dim3(unsigned(nbands), unsigned(B)), kAttnThreads, band_smem, s>>>(              \
              codes_q, gamma_q, gamma_k, kv, cnt, v, dw, out, int(n), int(d), int(heads),     \
              side, band_rows, eps);                                                          \
    } else {                                                                                  \
      attn_out_kernel<DKV><<<g3, kAttnThreads, 0, s>>>(codes_q, gamma_q, gamma_k, kv, cnt, v, \
                                                       dw, out, int(n), int(d), int(heads),   \
                                                       side, eps);                            \
    }                                                                                         \
    break;
  switch (dk) {
    SA_ATTN_CASE(16)
    SA_ATTN_CASE(32)
    SA_ATTN_CASE(64)
  }
#undef SA_ATTN_CASE
  count_launch(3);
  SA_LAUNCH_CHECK("sa_linear_binary_attn");
  return SA_OK;
}

extern "C" int sa_hamming_attn(const uint32_t* codes_q, const uint32_t* codes_k,
                               const float* gamma_q, const float* gamma_k, const float* v,
                               const float* dw, float* out, int64_t B, int64_t n, int64_t d,
                               int64_t heads, float eps, void* stream) {
  int st = check_attn_shapes("sa_hamming_attn", B, n, d, heads);
  if (st) return st;
  if (g_ham_mode == 0) {
    st = hamming_tc_launch(codes_q, codes_k, gamma_q, gamma_k, v, dw, out, B, n, d, heads, eps,
                           as_stream(stream));
    if (st != SA_ERR_VALUE) return st;
  }
  const int64_t dk = d / heads;
  const int64_t W = cdiv(dk, 32);
  const size_t smem = size_t(n) * dk * 4 + size_t(n) * W * 4 + size_t(kAttnThreads / 32) * n * 4;
  SA_REQUIRE(smem <= 200 * 1024, SA_ERR_SHAPE,
             "sa_hamming_attn: n=%lld too large for the quadratic form (use the linear order)",
             (long long)n);
  dim3 grid(unsigned(cdiv(n, kHamQ)), unsigned(B * heads));
  cudaStream_t s = as_stream(stream);
  const int side = grid_side(n);
#define SA_HAM_CASE(DKV)                                                                       \
  case DKV:                                                                                    \
    cudaFuncSetAttribute(hamming_attn_kernel<DKV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         int(smem));                                                           \
    hamming_attn_kernel<DKV><<<grid, kAttnThreads, smem, s>>>(codes_q, codes_k, gamma_q,       \
                                                              gamma_k, v, dw, out, int(n),     \
                                                              int(d), int(heads), side, eps);  \
    break;
  switch (dk) {
    SA_HAM_CASE(16)
    SA_HAM_CASE(32)
    SA_HAM_CASE(64)
  }
#undef SA_HAM_CASE
  count_launch(1);
  SA_LAUNCH_CHECK("sa_hamming_attn");
  return SA_OK;
}

extern "C" int sa_dwconv_tokens(const float* v, const float* dw, float* out, int64_t B, int64_t n,
                                int64_t d, int accumulate, void* stream) {
  SA_REQUIRE(B > 0 && n > 0 && d > 0, SA_ERR_SHAPE, "sa_dwconv_tokens: empty extents");
  const int64_t total = B * n * d;
  dwconv_tokens_kernel<<<unsigned(cdiv(total, 256)), 256, 0, as_stream(stream)>>>(
      v, dw, out, total, int(n), int(d), grid_side(n), accumulate);
  count_launch(1);
  SA_LAUNCH_CHECK("sa_dwconv_tokens");
  return SA_OK;
}

extern "C" int sa_binary_popcounts(const uint32_t* codes_q, const uint32_t* codes_k, int64_t B,
                                   int64_t n, int64_t dk, int64_t heads, int32_t* cnt, int32_t* D,
                                   int32_t* S, void* stream) {
  SA_REQUIRE(B > 0 && n > 0 && dk > 0 && heads > 0, SA_ERR_SHAPE,
             "sa_binary_popcounts: empty extents");
  const int W = int(cdiv(dk, 32));
  const int BH = int(B * heads);
  cudaStream_t s = as_stream(stream);
  popc_cnt_kernel<<<unsigned(cdiv(int64_t(BH) * dk, 256)), 256, 0, s>>>(codes_k, int(n), int(dk), W,
                                                                        BH, cnt);
  popc_D_kernel<<<unsigned(cdiv(int64_t(BH) * n, 256)), 256, 0, s>>>(codes_q, cnt, int(n), int(dk),
                                                                     W, BH, D);
  int launches = 2;
  if (S) {
    const int64_t total = int64_t(BH) * n * n;
    popc_S_kernel<<<unsigned(cdiv(total, 256)), 256, 0, s>>>(codes_q, codes_k, int(n), W, total, S);
    ++launches;
  }
  count_launch(launches);
  SA_LAUNCH_CHECK("sa_binary_popcounts");
  return SA_OK;
}
