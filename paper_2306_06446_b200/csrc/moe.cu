// K4 — top-1 two-expert router + stable token partition (ref moe.py:81-92).
//
//   logits = f32(fp64 x·W_g)        one warp per token, fp64 FMA + fixed shuffle tree;
//                                   every product of two floats is exact in fp64, so the
//                                   f32-rounded logits equal the reference's (ref tensor.py:68-75)
//   winner = argmax(softmax(logits)) with ties → expert 0. For two experts the
//            softmax argmax differs from the logit argmax only when the deficit is
//            so small that numpy's f32 exp rounds to 1 (ref moe.py:89):
//            expert 1 iff l1 > l0 and f32(l0 - l1) < -tie_thresh.
//   gate   = p[winner] = e_w / (e_0 + e_1) in f32 (e of the max logit is exactly 1).
//   perm   = stable partition [expert-0 tokens ascending | expert-1 tokens ascending]
//            = concatenate(index_of) (ref moe.py:91), via block counts → one-CTA
//            scan → block-local ballot ranks. counts[] stay on the device.
#include "common.cuh"

namespace sa {

constexpr int kRouteTok = 256;  // tokens per route / partition block

// winner + gate from the two f32 logits (see the file comment)
__device__ __forceinline__ int decide(float l0, float l1, float tie_thresh, float& gate) {
  const float m = fmaxf(l0, l1);
  const float sh0 = l0 - m, sh1 = l1 - m;  // f32 max-shift (ref tensor.py:100)
  // numpy-exp tie rule decides the winner bit-exactly
  const int e = (l1 > l0 && sh0 < -tie_thresh) ? 1 : 0;
  // e of the max is exp(0) = 1 exactly; a deficit inside the tie band has
  // numpy exp == 1 as well
  const float e0 = (sh0 >= -tie_thresh) ? 1.f : expf(sh0);
  const float e1 = (sh1 >= -tie_thresh) ? 1.f : expf(sh1);
  gate = (e ? e1 : e0) / (e0 + e1);
  return e;
}

// dispatch from precomputed logits (M, 2): one thread per token
__global__ void __launch_bounds__(kRouteTok) dispatch_kernel(const float* __restrict__ logits,
                                                            int64_t M, float tie_thresh,
                                                            int32_t* __restrict__ expert_of,
                                                            float* __restrict__ gate,
                                                            int32_t* __restrict__ block_cnt1) {
  __shared__ int wcnt[kRouteTok / 32];
  const int64_t t = int64_t(blockIdx.x) * kRouteTok + threadIdx.x;
  int e = 0;
  if (t < M) {
    float g;
    e = decide(logits[2 * t], logits[2 * t + 1], tie_thresh, g);
    expert_of[t] = e;
    gate[t] = g;
  }
  const unsigned b = __ballot_sync(0xffffffffu, e == 1);
  if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < kRouteTok / 32; ++w) c += wcnt[w];
    block_cnt1[blockIdx.x] = c;
  }
}

// logits + decision: G threads per token (G = 1 for d <= 64, else 8), each
// thread streams its slice of the row with 128-bit loads and fp64 FMAs; the G
// partial sums meet in a fixed xor-shuffle tree (deterministic).
template <int G>
__global__ void __launch_bounds__(256) route_kernel(const float* __restrict__ x,
                                                   const float* __restrict__ wg, int64_t M, int d,
                                                   float tie_thresh, float* __restrict__ logits,
                                                   int32_t* __restrict__ expert_of,
                                                   float* __restrict__ gate,
                                                   int32_t* __restrict__ block_cnt1) {
  constexpr int TPP = 256 / G;  // tokens per pass
  __shared__ double sw[2 * 512];
  __shared__ int wcnt[8];
  for (int i = threadIdx.x; i < 2 * d; i += blockDim.x) sw[i] = double(wg[i]);
  __syncthreads();
  const int sub = threadIdx.x % G, slot = threadIdx.x / G;
  const int64_t base = int64_t(blockIdx.x) * kRouteTok;
  const int d4 = d >> 2;
  int mine = 0;
#pragma unroll 1
  for (int pass = 0; pass < G; ++pass) {
    const int64_t t = base + pass * TPP + slot;
    const bool ok = t < M;
    double s0 = 0.0, s1 = 0.0;
    if (ok) {
      const float4* row = reinterpret_cast<const float4*>(x + t * d);
      // the row slice in chunks of 16 float4: each chunk's loads are all in
      // flight before its first FMA (one memory latency per 64 channels)
      constexpr int PF = 16;
      for (int cb = 0; cb < d4; cb += PF * G) {
      float4 pre[PF];
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int c4 = cb + sub + u * G;
        pre[u] = c4 < d4 ? __ldg(row + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int c4 = cb + sub + u * G;
        if (c4 >= d4) break;
        const float4 v = pre[u];
        const double* w = sw + 8 * c4;
        s0 = fma(double(v.x), w[0], s0);
        s1 = fma(double(v.x), w[1], s1);
        s0 = fma(double(v.y), w[2], s0);
        s1 = fma(double(v.y), w[3], s1);
        s0 = fma(double(v.z), w[4], s0);
        s1 = fma(double(v.z), w[5], s1);
        s0 = fma(double(v.w), w[6], s0);
        s1 = fma(double(v.w), w[7], s1);
      }
      }
    }
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (ok && sub == 0) {
      const float l0 = float(s0), l1 = float(s1);
      float g;
      const int e = decide(l0, l1, tie_thresh, g);
      gate[t] = g;
      expert_of[t] = e;
      if (logits) {
        logits[2 * t] = l0;
        logits[2 * t + 1] = l1;
      }
      mine += e;
    }
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < 8; ++w) c += wcnt[w];
    block_cnt1[blockIdx.x] = c;
  }
}

// one CTA per router (blockIdx.x): exclusive scan of per-block expert-1
// counts; counts[2r..2r+1]
__global__ void __launch_bounds__(1024) route_scan_kernel(const int32_t* __restrict__ block_cnt1,
                                                          int nblocks, int64_t M,
                                                          int32_t* __restrict__ block_off1,
                                                          int32_t* __restrict__ counts) {
  block_cnt1 += size_t(blockIdx.x) * nblocks;
  block_off1 += size_t(blockIdx.x) * nblocks;
  counts += 2 * blockIdx.x;
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < nblocks ? block_cnt1[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = warp_tot[lane];
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      warp_tot[lane] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    const int excl = carry + warp_tot[warp] + incl - v;
    if (i < nblocks) block_off1[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[1] = carry;
    counts[0] = int32_t(M - carry);
  }
}

__global__ void __launch_bounds__(kRouteTok) partition_kernel(const int32_t* __restrict__ expert_of,
                                                             const int32_t* __restrict__ block_off1,
                                                             const int32_t* __restrict__ counts,
                                                             int64_t M, int32_t* __restrict__ perm) {
  // router r = blockIdx.y (stacked plans of a fused multi-router pass)
  expert_of += size_t(blockIdx.y) * M;
  perm += size_t(blockIdx.y) * M;
  block_off1 += size_t(blockIdx.y) * gridDim.x;
  counts += 2 * blockIdx.y;
  __shared__ int wc[kRouteTok / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t = int64_t(blockIdx.x) * kRouteTok + threadIdx.x;
  const int e = t < M ? expert_of[t] : 0;
  const bool valid = t < M;
  const unsigned b1 = __ballot_sync(0xffffffffu, valid && e == 1);
  if (lane == 0) wc[warp] = __popc(b1);
  __syncthreads();
  int before1 = 0;
  for (int w = 0; w < warp; ++w) before1 += wc[w];
  before1 += __popc(b1 & ((1u << lane) - 1u));
  if (!valid) return;
  const int64_t off1 = block_off1[blockIdx.x];
  const int64_t blk0 = int64_t(blockIdx.x) * kRouteTok;
  const int64_t local = threadIdx.x;
  int64_t pos;
  if (e == 1) {
    pos = int64_t(counts[0]) + off1 + before1;
  } else {
    pos = (blk0 - off1) + (local - before1);
  }
  perm[pos] = int32_t(t);
}

// Stable partition with the block-count scan folded in: each CTA sums the
// expert-1 counts of the blocks before it (and of all blocks, for counts[]),
// integer adds in a fixed tree, so the result equals route_scan_kernel +
// partition_kernel while saving the single-CTA scan launch.
__global__ void __launch_bounds__(kRouteTok) partition_scan_kernel(
    const int32_t* __restrict__ expert_of, const int32_t* __restrict__ block_cnt1, int64_t M,
    int32_t* __restrict__ counts, int32_t* __restrict__ perm) {
  const int nb = gridDim.x;
  expert_of += size_t(blockIdx.y) * M;
  perm += size_t(blockIdx.y) * M;
  block_cnt1 += size_t(blockIdx.y) * nb;
  counts += 2 * blockIdx.y;
  __shared__ int wpre[kRouteTok / 32], wtot[kRouteTok / 32];
  __shared__ int wc[kRouteTok / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int pre = 0, tot = 0;
  for (int i = threadIdx.x; i < nb; i += kRouteTok) {
    const int c = __ldg(block_cnt1 + i);
    tot += c;
    if (i < int(blockIdx.x)) pre += c;
  }
  pre = __reduce_add_sync(0xffffffffu, pre);
  tot = __reduce_add_sync(0xffffffffu, tot);
  if (lane == 0) {
    wpre[warp] = pre;
    wtot[warp] = tot;
  }
  const int64_t t = int64_t(blockIdx.x) * kRouteTok + threadIdx.x;
  const bool valid = t < M;
  const int e = valid ? expert_of[t] : 0;
  const unsigned b1 = __ballot_sync(0xffffffffu, valid && e == 1);
  if (lane == 0) wc[warp] = __popc(b1);
  __syncthreads();
  int off1 = 0, c1 = 0;
#pragma unroll
  for (int w = 0; w < kRouteTok / 32; ++w) {
    off1 += wpre[w];
    c1 += wtot[w];
  }
  const int64_t c0 = M - c1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    counts[0] = int32_t(c0);
    counts[1] = c1;
  }
  int before1 = 0;
  for (int w = 0; w < warp; ++w) before1 += wc[w];
  before1 += __popc(b1 & ((1u << lane) - 1u));
  if (!valid) return;
  const int64_t blk0 = int64_t(blockIdx.x) * kRouteTok;
  const int64_t pos = (e == 1) ? c0 + off1 + before1 : (blk0 - off1) + (threadIdx.x - before1);
  perm[pos] = int32_t(t);
}

SA_DEBUG_SWITCH(int, g_fused_partition, 1, sa_debug_fused_partition)

// scan + partition of nr stacked plans
#ifndef SA_FUSED_PARTITION_MAX_NB
#define SA_FUSED_PARTITION_MAX_NB 1024
#endif
// block counts up to which each partition CTA folds the scan of all block
// counts itself (nb reads per CTA) instead of a separate scan kernel
constexpr int kFusedPartitionMaxNb = SA_FUSED_PARTITION_MAX_NB;
static void launch_partition(const int32_t* expert_of, int32_t* block_cnt1, int32_t* block_off1,
                             int32_t* counts, int32_t* perm, int64_t M, int nb, int nr,
                             cudaStream_t s) {
  // each folded-scan CTA reads all nb block counts (nb² work): only for
  // moderate block counts; large M keeps the single-CTA scan kernel
  if (g_fused_partition && nb <= kFusedPartitionMaxNb) {
    partition_scan_kernel<<<dim3(nb, nr), kRouteTok, 0, s>>>(expert_of, block_cnt1, M, counts, perm);
  } else {
    route_scan_kernel<<<nr, 1024, 0, s>>>(block_cnt1, nb, M, block_off1, counts);
    partition_kernel<<<dim3(nb, nr), kRouteTok, 0, s>>>(expert_of, block_off1, counts, M, perm);
  }
}

// LayerNorm (ref tensor.py:114-128) fused with up to three routers reading the
// normalized rows (the q/k/v projections of an AttentionLayer share one input,
// ref model.py:342-345): one thread per row holds the D floats in registers,
// writes y and, per router, the fp64 logits → winner / gate → block counts.
constexpr int kMaxRouters = 3;

constexpr int kLrThreads = 128;   // ln_route_kernel: 4 warps, each staging its own 32 rows

template <int D, bool LN = true>   // LN = false: routers on x itself (sa_moe_route), no y
__global__ void __launch_bounds__(kLrThreads) ln_route_kernel(
    const float* __restrict__ x, const float* __restrict__ gain, const float* __restrict__ bias,
    float* __restrict__ y, int64_t M, float eps, int nr, const float* __restrict__ wg0,
    const float* __restrict__ wg1, const float* __restrict__ wg2, float tie_thresh,
    int32_t* __restrict__ expert_of, float* __restrict__ gate, int32_t* __restrict__ block_cnt1) {
  constexpr int PITCH = D + 4;  // floats; conflict-free 128-bit row reads
  __shared__ double sw[kMaxRouters][2 * D];
  __shared__ int wcnt[kMaxRouters][kLrThreads / 32];
  extern __shared__ __align__(16) float tile[];  // [kLrThreads][PITCH]
  const float* wgs[kMaxRouters] = {wg0, wg1, wg2};
  for (int r = 0; r < nr; ++r)
    for (int i = threadIdx.x; i < 2 * D; i += kLrThreads) sw[r][i] = double(wgs[r][i]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // each warp stages its 32 rows (one contiguous run of float4s) with
  // coalesced loads, all issued before the first store
  const int64_t row0 = int64_t(blockIdx.x) * kLrThreads + warp * 32;
  const int nrows = int(max(int64_t(0), min(int64_t(32), M - row0)));
  float* tw = tile + warp * 32 * PITCH;
  {
    const float4* src = reinterpret_cast<const float4*>(x + row0 * D);
    constexpr int PER = D / 4;
    float4 buf[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = lane + 32 * u;
      buf[u] = i < nrows * (D / 4) ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = lane + 32 * u;
      *reinterpret_cast<float4*>(tw + (i / (D / 4)) * PITCH + 4 * (i % (D / 4))) = buf[u];
    }
  }
  __syncwarp();
  const int64_t row = row0 + lane;
  const bool ok = row < M;
  float v[D];
  float* trow = tw + lane * PITCH;
  if (LN && ok) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < D / 4; ++i) {
      const float4 q = *reinterpret_cast<const float4*>(trow + 4 * i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
      s += (q.x + q.y) + (q.z + q.w);
    }
    const float mean = s / float(D);
    float q2 = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      v[i] -= mean;
      q2 += v[i] * v[i];
    }
    const float inv = 1.0f / sqrtf(q2 / float(D) + eps);
#pragma unroll
    for (int i = 0; i < D / 4; ++i) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(gain) + i);
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias) + i);
      v[4 * i] = v[4 * i] * inv * g.x + b.x;
      v[4 * i + 1] = v[4 * i + 1] * inv * g.y + b.y;
      v[4 * i + 2] = v[4 * i + 2] * inv * g.z + b.z;
      v[4 * i + 3] = v[4 * i + 3] * inv * g.w + b.w;
      *reinterpret_cast<float4*>(trow + 4 * i) =
          make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  __syncwarp();
  if (LN) {  // coalesced write-back of the warp's normalized rows
    float4* dst = reinterpret_cast<float4*>(y + row0 * D);
#pragma unroll
    for (int u = 0; u < D / 4; ++u) {
      const int i = lane + 32 * u;
      if (i < nrows * (D / 4))
        dst[i] = *reinterpret_cast<const float4*>(tw + (i / (D / 4)) * PITCH + 4 * (i % (D / 4)));
    }
  }
  for (int r = 0; r < nr; ++r) {
    int e = 0;
    if (ok) {
      // router dot on the normalized row, re-read from the tile
      double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
      for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 q = *reinterpret_cast<const float4*>(trow + 4 * c4);
        const double* w = &sw[r][8 * c4];
        s0 = fma(double(q.x), w[0], s0);
        s1 = fma(double(q.x), w[1], s1);
        s0 = fma(double(q.y), w[2], s0);
        s1 = fma(double(q.y), w[3], s1);
        s0 = fma(double(q.z), w[4], s0);
        s1 = fma(double(q.z), w[5], s1);
        s0 = fma(double(q.w), w[6], s0);
        s1 = fma(double(q.w), w[7], s1);
      }
      float g;
      e = decide(float(s0), float(s1), tie_thresh, g);
      expert_of[size_t(r) * M + row] = e;
      gate[size_t(r) * M + row] = g;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, e == 1);
    if (lane == 0) wcnt[r][warp] = __popc(bal);
  }
  __syncthreads();
  // this CTA's share of its 256-token block count (zeroed by the host;
  // integer adds, order-independent)
  if (threadIdx.x < nr) {
    int c = 0;
    for (int w = 0; w < kLrThreads / 32; ++w) c += wcnt[threadIdx.x][w];
    const int nb = int((M + kRouteTok - 1) / kRouteTok);
    atomicAdd(&block_cnt1[size_t(threadIdx.x) * nb + blockIdx.x / (kRouteTok / kLrThreads)], c);
  }
}

// Wide rows (d = 32·PER, e.g. 160): one warp per row, lane l holds channels
// l + 32i. The LayerNorm is layernorm_kernel's arithmetic (lane partials in
// channel order, the same xor-shuffle reductions), so y is bit-identical to
// sa_layernorm; each router's fp64 dot is a per-lane chain over the lane's
// channels followed by a fixed xor tree (deterministic; the f32-rounded
// logits match route_kernel's sequential fp64 chain unless the two fp64 sums
// straddle an f32 rounding boundary). A CTA covers kRouteTok tokens (the block
// counts feed the shared scan / partition kernels); each warp carries RB rows
// at once so their loads are in flight together.
template <int PER>
__global__ void __launch_bounds__(1024, 1) ln_route_warp_kernel(
    const float* __restrict__ x, const float* __restrict__ gain, const float* __restrict__ bias,
    float* __restrict__ y, int64_t M, float eps, int nr, const float* __restrict__ wg0,
    const float* __restrict__ wg1, const float* __restrict__ wg2, float tie_thresh,
    int32_t* __restrict__ expert_of, float* __restrict__ gate, int32_t* __restrict__ block_cnt1) {
  constexpr int D = 32 * PER;
  constexpr int RB = 2;                      // rows per warp step (64-register cap)
  constexpr int kWarps = 32;                 // 1024 threads: 8 rows per warp
  constexpr int ROWS_PER_WARP = kRouteTok / kWarps;
  __shared__ int wcnt[kMaxRouters][kWarps];
  __shared__ double sw[kMaxRouters][2][D];   // [router][expert][channel]: lane reads are contiguous
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* wgs[kMaxRouters] = {wg0, wg1, wg2};
  for (int r = 0; r < nr; ++r)
    for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) sw[r][i & 1][i >> 1] = double(wgs[r][i]);
  float g[PER], bb[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    g[i] = __ldg(gain + lane + 32 * i);
    bb[i] = __ldg(bias + lane + 32 * i);
  }
  __syncthreads();
  const int64_t row0 = int64_t(blockIdx.x) * kRouteTok + int64_t(warp) * ROWS_PER_WARP;
  int cnt[kMaxRouters] = {0, 0, 0};
#pragma unroll 1
  for (int rb = 0; rb < ROWS_PER_WARP; rb += RB) {
    // the RB rows' reductions are interleaved (independent shuffle chains)
    float v[RB][PER];
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      const int64_t row = row0 + rb + k;
#pragma unroll
      for (int i = 0; i < PER; ++i)
        v[k][i] = row < M ? __ldg(x + row * D + lane + 32 * i) : 0.f;
    }
    float st[RB];
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) s += v[k][i];
      st[k] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < RB; ++k) st[k] += __shfl_xor_sync(0xffffffffu, st[k], o);
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      const float mean = st[k] / float(D);
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        v[k][i] = v[k][i] - mean;
        q += v[k][i] * v[k][i];
      }
      st[k] = q;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int k = 0; k < RB; ++k) st[k] += __shfl_xor_sync(0xffffffffu, st[k], o);
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      const int64_t row = row0 + rb + k;
      const float var = st[k] / float(D);
      const float inv = 1.0f / sqrtf(var + eps);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        v[k][i] = v[k][i] * inv * g[i] + bb[i];
        if (row < M) y[row * D + lane + 32 * i] = v[k][i];
      }
    }
#pragma unroll
    for (int r = 0; r < kMaxRouters; ++r) {
      if (r >= nr) break;   // uniform
      double s0[RB], s1[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        s0[k] = 0.0;
        s1[k] = 0.0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          s0[k] = fma(double(v[k][i]), sw[r][0][lane + 32 * i], s0[k]);
          s1[k] = fma(double(v[k][i]), sw[r][1][lane + 32 * i], s1[k]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          s0[k] += __shfl_xor_sync(0xffffffffu, s0[k], o);
          s1[k] += __shfl_xor_sync(0xffffffffu, s1[k], o);
        }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int64_t row = row0 + rb + k;
        float gt;
        const int e = decide(float(s0[k]), float(s1[k]), tie_thresh, gt);
        if (row < M) {
          if (lane == 0) {
            expert_of[size_t(r) * M + row] = e;
            gate[size_t(r) * M + row] = gt;
          }
          cnt[r] += e;
        }
      }
    }
  }
  if (lane == 0)
    for (int r = 0; r < nr; ++r) wcnt[r][warp] = cnt[r];
  __syncthreads();
  if (threadIdx.x < nr) {
    int c = 0;
    for (int ww = 0; ww < kWarps; ++ww) c += wcnt[threadIdx.x][ww];
    block_cnt1[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = c;
  }
}

// Wide rows, 8 lanes per row (4 rows per warp step): lane t of a row's group
// holds channels 32i + 4t .. 32i + 4t + 3 (i < PER), i.e. the partials of the
// 32 "virtual lanes" l = 4t + j of layernorm_kernel. Its xor butterfly over
// 16, 8, 4 becomes shuffles by 4, 2, 1 inside the group, and over 2, 1 adds
// inside the thread: y is bit-identical to sa_layernorm, with ~3x fewer
// instructions per row than one warp per row. Routers: fp64 lane chains over
// the lane's channels + a fixed xor tree. LN = false: routers on x itself.
constexpr int kOctThreads = 128, kOctRows = 64;   // 4 warps x 4 steps x 4 rows

// RT rows per thread and step (row (step·RT + rr)·4 + sub): the RT rows'
// shuffle / fp64 chains interleave and share each weight load; every row's
// arithmetic is the RT = 1 sequence. RT = 1 prefetches the next step's row.
template <int PER, bool LN, int RT>
__global__ void __launch_bounds__(kOctThreads, RT == 1 ? 6 : 4) ln_route_oct_kernel(
    const float* __restrict__ x, const float* __restrict__ gain, const float* __restrict__ bias,
    float* __restrict__ y, int64_t M, float eps, int nr, const float* __restrict__ wg0,
    const float* __restrict__ wg1, const float* __restrict__ wg2, float tie_thresh,
    int32_t* __restrict__ expert_of, float* __restrict__ gate, int32_t* __restrict__ block_cnt1) {
  constexpr int D = 32 * PER;
  constexpr int kRows = kOctRows * RT;   // rows per CTA (RT = 2: 128, one wave at 4 CTAs/SM)
  constexpr int kSteps = kRows / (kOctThreads / 32 * 4 * RT);
  constexpr bool PF = RT == 1;
  // [router][channel block i][k][lane t]: the k-th 16-byte weight pair of lane
  // t (k = 0/1: expert 0 channels c, c+1 / c+2, c+3; k = 2/3: expert 1), so the
  // 8 lanes of a row group read 128 contiguous bytes per load (no bank conflicts)
  __shared__ __align__(16) double2 sw[kMaxRouters][PER][4][8];
  __shared__ int wcnt[kMaxRouters][kOctThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 3, t = lane & 7;
  const float* wgs[kMaxRouters] = {wg0, wg1, wg2};
  for (int r = 0; r < nr; ++r)
    for (int idx = threadIdx.x; idx < PER * 32; idx += kOctThreads) {
      const int i = idx >> 5, k = (idx >> 3) & 3, tt = idx & 7;
      const int c = 32 * i + 4 * tt + 2 * (k & 1), e = k >> 1;   // wg layout [channel][expert]
      sw[r][i][k][tt] = make_double2(double(wgs[r][2 * c + e]), double(wgs[r][2 * c + 2 + e]));
    }
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kRows + warp * (kSteps * 4 * RT);
  int cnt[kMaxRouters] = {0, 0, 0};
  auto row_of = [&](int step, int rr) { return base + (step * RT + rr) * 4 + sub; };
  auto load_rows = [&](int step, float4 (&dst)[RT][PER]) {
#pragma unroll
    for (int rr = 0; rr < RT; ++rr) {
      const int64_t row = row_of(step, rr);
#pragma unroll
      for (int i = 0; i < PER; ++i)
        dst[rr][i] = row < M ? __ldg(reinterpret_cast<const float4*>(x + row * D + 32 * i + 4 * t))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 vn[PF ? RT : 1][PF ? PER : 1];
  if constexpr (PF) load_rows(0, vn);
#pragma unroll 1
  for (int step = 0; step < kSteps; ++step) {
    float4 v[RT][PER];
    if constexpr (PF) {
#pragma unroll
      for (int i = 0; i < PER; ++i) v[0][i] = vn[0][i];
      if (step + 1 < kSteps) load_rows(step + 1, vn);   // next rows in flight
    } else {
      load_rows(step, v);
    }
    if (LN) {
      // virtual-lane partials (channel order within each virtual lane)
      float p[RT][4], q[RT][4], mean[RT], inv[RT];
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) {
        p[rr][0] = p[rr][1] = p[rr][2] = p[rr][3] = 0.f;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          p[rr][0] += v[rr][i].x;
          p[rr][1] += v[rr][i].y;
          p[rr][2] += v[rr][i].z;
          p[rr][3] += v[rr][i].w;
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int rr = 0; rr < RT; ++rr)
#pragma unroll
          for (int j = 0; j < 4; ++j) p[rr][j] += __shfl_xor_sync(0xffffffffu, p[rr][j], o);
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) {
        mean[rr] = ((p[rr][0] + p[rr][2]) + (p[rr][1] + p[rr][3])) / float(D);
        q[rr][0] = q[rr][1] = q[rr][2] = q[rr][3] = 0.f;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          v[rr][i].x = v[rr][i].x - mean[rr];
          v[rr][i].y = v[rr][i].y - mean[rr];
          v[rr][i].z = v[rr][i].z - mean[rr];
          v[rr][i].w = v[rr][i].w - mean[rr];
          q[rr][0] += v[rr][i].x * v[rr][i].x;
          q[rr][1] += v[rr][i].y * v[rr][i].y;
          q[rr][2] += v[rr][i].z * v[rr][i].z;
          q[rr][3] += v[rr][i].w * v[rr][i].w;
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int rr = 0; rr < RT; ++rr)
#pragma unroll
          for (int j = 0; j < 4; ++j) q[rr][j] += __shfl_xor_sync(0xffffffffu, q[rr][j], o);
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) {
        const float var = ((q[rr][0] + q[rr][2]) + (q[rr][1] + q[rr][3])) / float(D);
        inv[rr] = 1.0f / sqrtf(var + eps);
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(gain + 32 * i + 4 * t));
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + 32 * i + 4 * t));
#pragma unroll
        for (int rr = 0; rr < RT; ++rr) {
          const int64_t row = row_of(step, rr);
          v[rr][i].x = v[rr][i].x * inv[rr] * g4.x + b4.x;
          v[rr][i].y = v[rr][i].y * inv[rr] * g4.y + b4.y;
          v[rr][i].z = v[rr][i].z * inv[rr] * g4.z + b4.z;
          v[rr][i].w = v[rr][i].w * inv[rr] * g4.w + b4.w;
          if (row < M) *reinterpret_cast<float4*>(y + row * D + 32 * i + 4 * t) = v[rr][i];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kMaxRouters; ++r) {
      if (r >= nr) break;   // uniform
      double s0[RT], s1[RT];
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) s0[rr] = s1[rr] = 0.0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const double2 a0 = sw[r][i][0][t];
        const double2 a1 = sw[r][i][1][t];
        const double2 b0 = sw[r][i][2][t];
        const double2 b1 = sw[r][i][3][t];
#pragma unroll
        for (int rr = 0; rr < RT; ++rr) {
          s0[rr] = fma(double(v[rr][i].x), a0.x, s0[rr]);
          s1[rr] = fma(double(v[rr][i].x), b0.x, s1[rr]);
          s0[rr] = fma(double(v[rr][i].y), a0.y, s0[rr]);
          s1[rr] = fma(double(v[rr][i].y), b0.y, s1[rr]);
          s0[rr] = fma(double(v[rr][i].z), a1.x, s0[rr]);
          s1[rr] = fma(double(v[rr][i].z), b1.x, s1[rr]);
          s0[rr] = fma(double(v[rr][i].w), a1.y, s0[rr]);
          s1[rr] = fma(double(v[rr][i].w), b1.y, s1[rr]);
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int rr = 0; rr < RT; ++rr) {
          s0[rr] += __shfl_xor_sync(0xffffffffu, s0[rr], o);
          s1[rr] += __shfl_xor_sync(0xffffffffu, s1[rr], o);
        }
#pragma unroll
      for (int rr = 0; rr < RT; ++rr) {
        const int64_t row = row_of(step, rr);
        float gt;
        const int e = decide(float(s0[rr]), float(s1[rr]), tie_thresh, gt);
        if (t == 0 && row < M) {
          expert_of[size_t(r) * M + row] = e;
          gate[size_t(r) * M + row] = gt;
          cnt[r] += e;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kMaxRouters; ++r) {
    const int c = __reduce_add_sync(0xffffffffu, cnt[r]);
    if (lane == 0 && r < nr) wcnt[r][warp] = c;
  }
  __syncthreads();
  // the 256-token block count (zeroed by the host) gets this CTA's share:
  // integer adds, so the result is order-independent
  if (threadIdx.x < nr) {
    int c = 0;
    for (int w = 0; w < kOctThreads / 32; ++w) c += wcnt[threadIdx.x][w];
    const int nb = int((M + kRouteTok - 1) / kRouteTok);
    atomicAdd(&block_cnt1[size_t(threadIdx.x) * nb + blockIdx.x / (kRouteTok / kRows)], c);
  }
}

SA_DEBUG_SWITCH(int, g_route_oct, 1, sa_debug_route_oct)
// rows per thread of the 8-lanes-per-row kernel (debug: 1)
SA_DEBUG_SWITCH(int, g_oct_rt, 2, sa_debug_oct_rows)

}  // namespace sa

using namespace sa;

extern "C" size_t sa_ln_route_workspace(int64_t M, int nr) {
  return size_t(2 * cdiv(M, kRouteTok) * nr) * sizeof(int32_t) + 64;
}

extern "C" int sa_ln_route(const float* x, const float* gain, const float* bias, float* y,
                           int64_t M, int64_t d, float eps, int nr, const float* wg0,
                           const float* wg1, const float* wg2, float tie_thresh,
                           int32_t* expert_of, float* gate, int32_t* counts, int32_t* perm,
                           void* ws, size_t ws_bytes, void* stream) {
  SA_REQUIRE(d > 0 && d % 32 == 0 && d <= 256, SA_ERR_SHAPE,
             "sa_ln_route: d=%lld unsupported (a multiple of 32 up to 256)", (long long)d);
  SA_REQUIRE(nr >= 1 && nr <= kMaxRouters, SA_ERR_VALUE, "sa_ln_route: 1..3 routers, got %d", nr);
  SA_REQUIRE(M > 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_ln_route: bad token count");
  SA_REQUIRE(ws_bytes >= sa_ln_route_workspace(M, nr), SA_ERR_VALUE,
             "sa_ln_route: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int nb = int(cdiv(M, kRouteTok));
  int32_t* block_cnt1 = static_cast<int32_t*>(ws);
  int32_t* block_off1 = block_cnt1 + size_t(nb) * nr;
  if (d == 32 || d == 64) {
    cudaMemsetAsync(block_cnt1, 0, size_t(nb) * nr * sizeof(int32_t), s);
    const unsigned g = unsigned(cdiv(M, kLrThreads));
    if (d == 32) {
      const int smem = kLrThreads * (32 + 4) * 4;
      ln_route_kernel<32><<<g, kLrThreads, smem, s>>>(x, gain, bias, y, M, eps, nr, wg0, wg1,
                                                      wg2, tie_thresh, expert_of, gate, block_cnt1);
    } else {
      const int smem = kLrThreads * (64 + 4) * 4;
      ln_route_kernel<64><<<g, kLrThreads, smem, s>>>(x, gain, bias, y, M, eps, nr, wg0, wg1,
                                                      wg2, tie_thresh, expert_of, gate, block_cnt1);
    }
  } else if (g_route_oct) {
    cudaMemsetAsync(block_cnt1, 0, size_t(nb) * nr * sizeof(int32_t), s);
#define SA_LNRO_RT(P, RT)                                                                      \
  ln_route_oct_kernel<P, true, RT><<<unsigned(cdiv(M, kOctRows * RT)), kOctThreads, 0, s>>>(       \
      x, gain, bias, y, M, eps, nr, wg0, wg1, wg2, tie_thresh, expert_of, gate, block_cnt1)
#define SA_LNRO(P)                                                                             \
  case P:                                                                                      \
    if (g_oct_rt == 2) SA_LNRO_RT(P, 2);                                                       \
    else SA_LNRO_RT(P, 1);                                                                     \
    break;
    switch (d / 32) {
      SA_LNRO(1) SA_LNRO(2) SA_LNRO(3) SA_LNRO(4) SA_LNRO(5) SA_LNRO(6) SA_LNRO(7) SA_LNRO(8)
    }
#undef SA_LNRO
#undef SA_LNRO_RT
  } else {
#define SA_LNRW(P)                                                                             \
  case P:                                                                                      \
    ln_route_warp_kernel<P><<<nb, 1024, 0, s>>>(x, gain, bias, y, M, eps, nr, wg0, wg1,      \
                                                     wg2, tie_thresh, expert_of, gate,       \
                                                     block_cnt1);                            \
    break;
    switch (d / 32) {
      SA_LNRW(1) SA_LNRW(2) SA_LNRW(3) SA_LNRW(4) SA_LNRW(5) SA_LNRW(6) SA_LNRW(7) SA_LNRW(8)
    }
#undef SA_LNRW
  }
  launch_partition(expert_of, block_cnt1, block_off1, counts, perm, M, nb, nr, s);
  count_launch(g_fused_partition && nb <= kFusedPartitionMaxNb ? 2 : 3);
  SA_LAUNCH_CHECK("sa_ln_route");
  return SA_OK;
}

extern "C" size_t sa_moe_route_workspace(int64_t M) {
  const int64_t nb = cdiv(M, kRouteTok);
  return size_t(2 * nb) * sizeof(int32_t) + 64;
}

extern "C" int sa_moe_route(const float* x, const float* wg, int64_t M, int64_t d,
                            float tie_thresh, float* logits, int32_t* expert_of, float* gate,
                            int32_t* counts, int32_t* perm, void* ws, size_t ws_bytes,
                            void* stream) {
  SA_REQUIRE(M >= 0 && d > 0 && d <= 512 && d % 4 == 0, SA_ERR_SHAPE,
             "sa_moe_route: d=%lld unsupported", (long long)d);
  SA_REQUIRE(M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_moe_route: too many tokens");
  SA_REQUIRE(ws_bytes >= sa_moe_route_workspace(M), SA_ERR_VALUE,
             "sa_moe_route: workspace too small");
  cudaStream_t s = as_stream(stream);
  if (M == 0) {
    cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s);
    return SA_OK;
  }
  const int nb = int(cdiv(M, kRouteTok));
  int32_t* block_cnt1 = static_cast<int32_t*>(ws);
  int32_t* block_off1 = block_cnt1 + nb;
  if (logits == nullptr && (d == 32 || d == 64)) {
    // narrow rows: the warp-staged LN+router kernel without its LayerNorm
    // (coalesced row staging; the same sequential fp64 channel order as
    // route_kernel, so identical logits)
    cudaMemsetAsync(block_cnt1, 0, size_t(nb) * sizeof(int32_t), s);
    const unsigned g = unsigned(cdiv(M, kLrThreads));
    if (d == 32)
      ln_route_kernel<32, false><<<g, kLrThreads, kLrThreads * (32 + 4) * 4, s>>>(
          x, nullptr, nullptr, nullptr, M, 0.f, 1, wg, nullptr, nullptr, tie_thresh, expert_of,
          gate, block_cnt1);
    else
      ln_route_kernel<64, false><<<g, kLrThreads, kLrThreads * (64 + 4) * 4, s>>>(
          x, nullptr, nullptr, nullptr, M, 0.f, 1, wg, nullptr, nullptr, tie_thresh, expert_of,
          gate, block_cnt1);
  } else if (g_route_oct && logits == nullptr && d % 32 == 0 && d >= 96 && d <= 256) {
    // wide rows: 8 lanes per row (the LN+router kernel without its LayerNorm)
    cudaMemsetAsync(block_cnt1, 0, size_t(nb) * sizeof(int32_t), s);
#define SA_RO_RT(P, RT)                                                                        \
  ln_route_oct_kernel<P, false, RT><<<unsigned(cdiv(M, kOctRows * RT)), kOctThreads, 0, s>>>(      \
      x, nullptr, nullptr, nullptr, M, 0.f, 1, wg, nullptr, nullptr, tie_thresh, expert_of,    \
      gate, block_cnt1)
#define SA_RO(P)                                                                               \
  case P:                                                                                      \
    if (g_oct_rt == 2) SA_RO_RT(P, 2);                                                         \
    else SA_RO_RT(P, 1);                                                                       \
    break;
    switch (d / 32) { SA_RO(3) SA_RO(4) SA_RO(5) SA_RO(6) SA_RO(7) SA_RO(8) }
#undef SA_RO
#undef SA_RO_RT
  } else {
    // one thread per token: the row streams in 64-channel chunks with all
    // loads of a chunk in flight
    route_kernel<1><<<nb, 256, 0, s>>>(x, wg, M, int(d), tie_thresh, logits, expert_of, gate,
                                       block_cnt1);
  }
  launch_partition(expert_of, block_cnt1, block_off1, counts, perm, M, nb, 1, s);
  count_launch(g_fused_partition && nb <= kFusedPartitionMaxNb ? 2 : 3);
  SA_LAUNCH_CHECK("sa_moe_route");
  return SA_OK;
}

extern "C" int sa_moe_dispatch(const float* logits, int64_t M, float tie_thresh,
                               int32_t* expert_of, float* gate, int32_t* counts, int32_t* perm,
                               void* ws, size_t ws_bytes, void* stream) {
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_moe_dispatch: bad token count");
  SA_REQUIRE(ws_bytes >= sa_moe_route_workspace(M), SA_ERR_VALUE,
             "sa_moe_dispatch: workspace too small");
  cudaStream_t s = as_stream(stream);
  if (M == 0) {
    cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s);
    return SA_OK;
  }
  const int nb = int(cdiv(M, kRouteTok));
  int32_t* block_cnt1 = static_cast<int32_t*>(ws);
  int32_t* block_off1 = block_cnt1 + nb;
  dispatch_kernel<<<nb, kRouteTok, 0, s>>>(logits, M, tie_thresh, expert_of, gate, block_cnt1);
  launch_partition(expert_of, block_cnt1, block_off1, counts, perm, M, nb, 1, s);
  count_launch(g_fused_partition && nb <= kFusedPartitionMaxNb ? 2 : 3);
  SA_LAUNCH_CHECK("sa_moe_dispatch");
  return SA_OK;
}

// per-block expert-1 counts from winners already on the device
__global__ void __launch_bounds__(kRouteTok) count_kernel(const int32_t* __restrict__ expert_of,
                                                         int64_t M, int32_t* __restrict__ block_cnt1) {
  __shared__ int wcnt[kRouteTok / 32];
  const int64_t t = int64_t(blockIdx.x) * kRouteTok + threadIdx.x;
  const int e = t < M ? expert_of[t] : 0;
  const unsigned b = __ballot_sync(0xffffffffu, e == 1);
  if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < kRouteTok / 32; ++w) c += wcnt[w];
    block_cnt1[blockIdx.x] = c;
  }
}

extern "C" size_t sa_moe_partition_workspace(int64_t M) { return sa_moe_route_workspace(M); }

extern "C" int sa_moe_partition(const int32_t* expert_of, int64_t M, int32_t* counts,
                                int32_t* perm, void* ws, size_t ws_bytes, void* stream) {
  SA_REQUIRE(M >= 0 && M < (int64_t(1) << 31), SA_ERR_SHAPE, "sa_moe_partition: bad token count");
  SA_REQUIRE(ws_bytes >= sa_moe_partition_workspace(M), SA_ERR_VALUE,
             "sa_moe_partition: workspace too small");
  cudaStream_t s = as_stream(stream);
  if (M == 0) {
    cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s);
    return SA_OK;
  }
  const int nb = int(cdiv(M, kRouteTok));
  int32_t* block_cnt1 = static_cast<int32_t*>(ws);
  int32_t* block_off1 = block_cnt1 + nb;
  count_kernel<<<nb, kRouteTok, 0, s>>>(expert_of, M, block_cnt1);
  launch_partition(expert_of, block_cnt1, block_off1, counts, perm, M, nb, 1, s);
  count_launch(g_fused_partition && nb <= kFusedPartitionMaxNb ? 2 : 3);
  SA_LAUNCH_CHECK("sa_moe_partition");
  return SA_OK;
}
