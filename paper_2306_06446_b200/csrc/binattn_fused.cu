// K2a, single pass over V: binary linear attention + DWConv for head dim 32,
// one thread-block cluster per image.
//
// Semantics are those of binattn.cu (ref attention.py:113-120 on the binary
// features of model.py:355-358, DWConv branch attention.py:170-179 added
// before W_O, model.py:367-373):
//   kv[a][:] = gk * sum_{j : ck[j][a]} v_j,  cnt[a] = sum_j ck[j][a]
//   out_i    = gq * sum_{a : cq[i][a]} kv[a] / (gq*gk*sum_{a : cq[i][a]} cnt[a] + eps)
//              + dwconv3x3(V)_i
//
// Layout of the work. The token grid (side = ceil(sqrt n), row-major) of one
// image is cut into CL bands of BR grid rows; CTA `rank` of the image's
// cluster owns band `rank`:
//  1. one thread bulk-copies the band's V rows plus one halo row above and
//     below (each grid row is one contiguous (side x d) fp32 run in HBM) into
//     shared memory; V is read from HBM exactly once per image;
//  2. pass 1 (K^T V partial of the band): 16 threads per token stream
//     (4 row groups of 8 code bits x 4 column groups of 8 channels), 16
//     streams; per token a thread adds its 8 V channels into the rows whose
//     K code bit is set (packed f32x2 masked adds: v*1 / v*0 are exact, so
//     the accumulators only ever receive selected V entries); streams are
//     combined in a fixed order (shuffle, then shared memory); the code-bit
//     counts use bit-sliced vertical counters (one warp) and a ballot tree;
//  3. the CL band partials are exchanged through distributed shared memory
//     and summed in rank order (deterministic, identical in every CTA);
//  4. pass 2: per head, kv is folded into Four-Russians nibble tables
//     T[g][m][c] = sum_{i in m} kv[4g+i][c]; a thread owns 4 channels and
//     walks a segment of a grid row: 8 table lookups (float4) per token for
//     the additive Q·(K^T V), the integer D from 8 lanes' count-table lookups
//     and a shuffle tree, and the 3x3 DWConv from a register sliding window
//     over the shared-memory band (3 new float4 per token).
#include <cooperative_groups.h>

#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace sa {
namespace baf {

constexpr int DK = 32;
constexpr int kThreads = 256;
#ifndef K2A_BAND_TOKENS
#define K2A_BAND_TOKENS 400   // ~tokens per cluster CTA (sets the cluster size)
#endif
constexpr int kStreams = 16;        // pass-1 token streams (16 threads each)
constexpr int kMaxCluster = 8;
// pass-2 tokens per row segment (a multiple of 3: the window ring), chosen per
// grid side so a band's (row, segment) units fill the 32 thread slots in one
// round where possible (side 56: 4 segments x 7 rows = 28 units)
__host__ __device__ constexpr int seg_len(int side) {
  return side >= 28 ? 15 : (side >= 14 ? 9 : 6);
}
constexpr int kMaxBandRows = 32;    // split out kernel: static mbarrier array bound

struct Params {
  const uint32_t* cq;
  const uint32_t* ck;
  const float* gq;
  const float* gk;
  const float* v;
  const float* dw;
  float* out;
  int n, d, heads, side, rows_total, band_rows;
  float eps;
  int ld;     // global row stride of V / out in floats (= model dim); head = blockIdx.z
  int pull;   // debug builds: 1 = the pull exchange (cluster barrier + DSMEM loads)
};

struct Smem {
  // byte offsets into the dynamic shared memory carve-out
  uint32_t v, cq, ck, part, cntp, cntw, tab, tcb, mt, cb, bar, total;
};

__host__ __device__ inline Smem smem_layout(int d, int heads, int side, int band_rows) {
  Smem s;
  const uint32_t band_tok = uint32_t(band_rows) * side;
  uint32_t o = 0;
  s.v = o;
  o += uint32_t(band_rows + 2) * side * d * 4;
  s.cq = o;
  o += heads * band_tok * 4;
  s.ck = o;
  o += heads * band_tok * 4;
  o = (o + 15) & ~15u;
  s.part = o;                                  // [heads][DK][DK] band partial of kv
  o += heads * DK * DK * 4;
  s.cntp = o;                                  // [heads][DK] band partial of cnt
  o += heads * DK * 4;
  s.cntw = o;                                  // [DK] bit counts of the current head
  o += DK * 4;
  s.tab = o;                                   // union: pass-1 scratch [4][DK][DK] | tables
  const uint32_t scratch = 4 * DK * DK * 4 + kStreams * DK * 4;
  const uint32_t tables = heads * (DK / 4) * 16 * DK * 4;
  o += scratch > tables ? scratch : tables;
  s.tcb = o;                                   // [heads][4][256] float: byte tables of cnt
  o += heads * 4 * 256 * 4;
  s.mt = o;                                    // [256][8] float: 0/1 masks of a code byte
  o += 256 * 8 * 4;
  s.cb = o;                                    // [kMaxCluster][DK] int: pushed band counts
  o += kMaxCluster * DK * 4;
  s.bar = o;                                   // one mbarrier per smem row (+ codes), then
  o += (band_rows + 3) * 8 + 16;               // the two exchange barriers (xbar, tbar)
  s.total = o;
  return s;
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// acc (two packed fp32) += v * m with m = 1.0 or 0.0 (a code bit, broadcast to
// both lanes): an exact masked add — v*1 and v*0 are exact, so the
// accumulator only ever receives additions of selected V entries. One FFMA2
// per channel pair (a predicated add.f32x2 compiles to FADD2 + 2 SEL).
__device__ __forceinline__ void add2_mask(unsigned long long& acc, unsigned long long v, float m) {
  asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%2, %2};\n\tfma.rn.f32x2 %0, %1, t, %0;\n\t}"
      : "+l"(acc)
      : "l"(v), "f"(m));
}
__device__ __forceinline__ void add2(unsigned long long& acc, unsigned long long v) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(v));
}
__device__ __forceinline__ void fma2(unsigned long long& acc, unsigned long long a,
                                     unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 unpack2(unsigned long long u) {
  return make_float2(__uint_as_float(uint32_t(u)), __uint_as_float(uint32_t(u >> 32)));
}
__device__ __forceinline__ ulonglong2 lds128(const void* p) {
  return *reinterpret_cast<const ulonglong2*>(p);
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct Win {   // one window column: 4 channels of 3 grid rows (packed pairs)
  ulonglong2 r[3];
};

// D = model dim (heads = D / 32), SIDE = token-grid side: every shared-memory
// stride is a compile-time constant.
template <int D, int SIDE>
__global__ void __launch_bounds__(kThreads, 2) binattn_fused_kernel(Params p,
                                                                    const __grid_constant__ CUtensorMap tmV) {
  constexpr int HEADS = D / DK;
  constexpr uint32_t ROWB = uint32_t(SIDE) * D * 4;   // bytes per smem grid row
  constexpr uint32_t TOKB = uint32_t(D) * 4;          // bytes per token
  extern __shared__ __align__(16) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = int(cluster.block_rank());
  const int CL = int(cluster.num_blocks());
  const int b = blockIdx.y;
  const int hz = blockIdx.z, H = p.heads;    // this CTA's head of the image
  const int ld = p.ld;
  const int n = p.n, BR = p.band_rows;
  const Smem L = smem_layout(D, HEADS, SIDE, BR);
  uint8_t* Vb = smem + L.v;
  uint32_t* cqs = reinterpret_cast<uint32_t*>(smem + L.cq);
  uint32_t* cks = reinterpret_cast<uint32_t*>(smem + L.ck);
  float* part = reinterpret_cast<float*>(smem + L.part);
  int* cntp = reinterpret_cast<int*>(smem + L.cntp);
  int* cntw = reinterpret_cast<int*>(smem + L.cntw);
  float* tab = reinterpret_cast<float*>(smem + L.tab);
  float* tcb = reinterpret_cast<float*>(smem + L.tcb);
  float* mt = reinterpret_cast<float*>(smem + L.mt);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = rank * BR;
  const int r1 = min(p.rows_total, r0 + BR);
  const int t_lo = min(n, r0 * SIDE), t_hi = min(n, r1 * SIDE);
  const int nt = t_hi - t_lo;
  // ---- 1. band of V (+ halo rows) → shared memory ----------------------------
  // smem row R holds grid row r0 - 1 + R; cells past n and rows outside the
  // grid are zero (the reference's zero-padded token grid, attention.py:170-179)
  // one mbarrier per smem row, so pass 1 starts on the first rows while the
  // rest of the band is still in flight
  // the band's q / k codes (one head per CTA: contiguous runs) by bulk copy
  // when 16-byte aligned, completing on bar[BR + 2]
  const size_t code0 = (size_t(b) * H + hz) * n + t_lo;
  const bool code_bulk = HEADS == 1 && nt > 0 && (nt * 4) % 16 == 0 && (code0 * 4) % 16 == 0 &&
                         (reinterpret_cast<uintptr_t>(p.cq) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(p.ck) & 15) == 0 &&
                         (su32(cqs) & 15u) == 0 && (su32(cks) & 15u) == 0;
  if (tid == 0) {
    for (int R = 0; R < BR + 5; ++R)   // rows, codes, xbar, tbar
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + R)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (code_bulk) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + BR + 2)),
                   "r"(uint32_t(2 * nt * 4))
                   : "memory");
      tc::bulk_g2s(cqs, p.cq + code0, uint32_t(nt * 4), bar + BR + 2);
      tc::bulk_g2s(cks, p.ck + code0, uint32_t(nt * 4), bar + BR + 2);
    }
    // one TMA copy per grid row from the (channel, token, image) tensor map:
    // box = the head's 32 channels x SIDE tokens; rows outside the grid and
    // cells past n are out of bounds and arrive as zeros (the reference's
    // zero-padded token grid, attention.py:170-179). Band rows first, halos last.
    for (int i = 0; i < BR + 2; ++i) {
      const int R = i < BR ? i + 1 : (i == BR ? 0 : BR + 1);
      const int rr = r0 - 1 + R;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + R)),
                   "r"(ROWB)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(Vb + R * ROWB)),
          "l"(reinterpret_cast<uint64_t>(&tmV)), "r"(hz * DK), "r"(rr * SIDE), "r"(b),
          "r"(su32(bar + R))
          : "memory");
    }
  }
  if (!code_bulk) {
    for (int i = tid; i < HEADS * nt; i += kThreads) {   // codes of the band, [head][token]
      const int h = i / nt, t = i - h * nt;
      const size_t g = (size_t(b) * H + hz + h) * n + t_lo + t;
      cqs[h * nt + t] = __ldg(p.cq + g);
      cks[h * nt + t] = __ldg(p.ck + g);
    }
  }
  for (int i = tid; i < 256 * 8; i += kThreads)          // byte → 8 masks
    mt[i] = ((i >> 3) >> (i & 7)) & 1 ? 1.0f : 0.0f;
  __syncthreads();  // barrier init, codes, masks visible
  // push exchange (below): every CTA's exchange barriers must be initialised
  // before a peer's first remote store; the matching wait sits just before it
  const bool push = HEADS == 1 && (kMaxCluster % CL) == 0 && !p.pull;
  // a one-CTA cluster exchanges nothing: plain shared-memory stores (st.async
  // into the cluster window needs a cluster of at least two CTAs)
  const bool solo = CL == 1;
  if (push && !solo) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  auto wait_row = [&](int R) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t"
        "@!q bra W_%=;\n\t}" ::"r"(su32(bar + R))
        : "memory");
  };

  if (code_bulk) {   // the band's codes have landed
    asm volatile(
        "{\n\t.reg .pred q;\n\tWC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t"
        "@!q bra WC_%=;\n\t}" ::"r"(su32(bar + BR + 2))
        : "memory");
  }
  // ---- 2. pass 1: band partial of K^T V and of the code-bit counts -----------
  const int s_id = tid >> 4;               // stream 0..15 (two per warp)
  const int rg = (tid >> 2) & 3;           // code bits 8rg .. 8rg+7
  const int cgp = tid & 3;                 // channels 8cgp .. 8cgp+7
#pragma unroll 1
  for (int h = 0; h < HEADS; ++h) {
    unsigned long long acc[8][4], cacc[4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) cacc[j] = 0ull;
    const uint8_t* vp = Vb + ROWB + (h * DK + cgp * 8) * 4 + s_id * TOKB;
    const uint32_t* kp = cks + h * nt + s_id;
    const uint8_t* mtb = reinterpret_cast<const uint8_t*>(mt);
    int next_row = 0;   // first band-local token of the next unwaited smem row
    int R_w = 1;
#pragma unroll 2
    for (int t = s_id; t < nt; t += kStreams) {
      if (h == 0 && t >= next_row) {   // band row of token t has landed
        while (t >= next_row) {
          wait_row(R_w);
          ++R_w;
          next_row += SIDE;
        }
      }
      const ulonglong2 va = lds128(vp);
      const ulonglong2 vc = lds128(vp + 16);
      const uint8_t* mrow = mtb + (((*kp) >> (rg * 8)) & 0xffu) * 32;
      const ulonglong2 mp0 = lds128(mrow);
      const ulonglong2 mp1 = lds128(mrow + 16);
      const float2 m01 = unpack2(mp0.x), m23 = unpack2(mp0.y);
      const float2 m45 = unpack2(mp1.x), m67 = unpack2(mp1.y);
      const float m[8] = {m01.x, m01.y, m23.x, m23.y, m45.x, m45.y, m67.x, m67.y};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        add2_mask(acc[i][0], va.x, m[i]);
        add2_mask(acc[i][1], va.y, m[i]);
        add2_mask(acc[i][2], vc.x, m[i]);
        add2_mask(acc[i][3], vc.y, m[i]);
      }
      // code-bit counts: the same 0/1 masks summed (exact small integers)
      add2(cacc[0], mp0.x);
      add2(cacc[1], mp0.y);
      add2(cacc[2], mp1.x);
      add2(cacc[3], mp1.y);
      vp += kStreams * TOKB;
      kp += kStreams;
    }
    if (h == 0) {   // streams with few tokens still own rows later threads read
      while (R_w <= BR) {
        wait_row(R_w);
        ++R_w;
      }
    }
    // combine: the warp's two streams (lanes l, l+16) by shuffle, then warps
    // 4-7 store, warps 0-3 add their own and store, one 4-way sum (fixed order)
    float2 cmb[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack2(acc[i][j]);
        cmb[i][j] = make_float2(a.x + __shfl_down_sync(0xffffffffu, a.x, 16),
                                a.y + __shfl_down_sync(0xffffffffu, a.y, 16));
      }
    float* scr = tab + (warp & 3) * DK * DK + rg * 8 * DK + cgp * 8;
    if (warp >= 4 && lane < 16) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<float2*>(scr + i * DK + 2 * j) = cmb[i][j];
    }
    // counts: lanes with cgp == 0 hold them for rows 8rg..8rg+7 of their
    // stream; fold the 16 streams in a fixed order through shared memory
    if (cgp == 0) {
      float* cs = tab + 4 * DK * DK + s_id * DK + rg * 8;   // after the kv scratch
#pragma unroll
      for (int j = 0; j < 4; ++j) *reinterpret_cast<float2*>(cs + 2 * j) = unpack2(cacc[j]);
    }
    __syncthreads();
    if (warp < 4 && lane < 16) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2* q = reinterpret_cast<float2*>(scr + i * DK + 2 * j);
          const float2 o = *q;
          *q = make_float2(cmb[i][j].x + o.x, cmb[i][j].y + o.y);
        }
    }
    __syncthreads();
    {
      const int e = tid * 4;   // 256 threads x 4 = DK*DK
      float4 s4 = *reinterpret_cast<const float4*>(tab + e);
#pragma unroll
      for (int w4 = 1; w4 < 4; ++w4) {
        const float4 q4 = *reinterpret_cast<const float4*>(tab + w4 * DK * DK + e);
        s4.x += q4.x;
        s4.y += q4.y;
        s4.z += q4.z;
        s4.w += q4.w;
      }
      *reinterpret_cast<float4*>(part + h * DK * DK + e) = s4;
    }
    if (tid < DK) {
      const float* cs = tab + 4 * DK * DK + tid;
      float c = 0.f;
#pragma unroll
      for (int st = 0; st < kStreams; ++st) c += cs[st * DK];
      cntp[h * DK + tid] = int(c);
    }
    __syncthreads();
  }

  // ---- 3. exchange band partials across the cluster (rank order) -------------
  if (push) {
    // Push form (one head per CTA, CL | 8): CTA o owns nibble groups
    // [o·G, o·G + G) (G = 8 / CL, 4 kv rows each). Every CTA stores its band
    // partial rows into the owners' receive slots and its counts into every
    // CTA (st.async, completing on the receiver's xbar); each owner sums its
    // rows in rank order, builds its groups' nibble tables and stores them
    // into every peer's table region (completing on tbar). No cluster-wide
    // barrier and no remote loads: each CTA only waits for the bytes it needs.
    const int G = kMaxCluster / CL;
    uint64_t* xbar = bar + BR + 3;
    uint64_t* tbar = bar + BR + 4;
    float* rbuf = tcb;                                   // [CL][G][4][DK] (tcb is built after)
    int* cbuf = reinterpret_cast<int*>(smem + L.cb);     // [CL][DK]
    if (tid == 0 && !solo) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(xbar)),
                   "r"(uint32_t(CL * G * 4 * DK * 4 + CL * DK * 4))
                   : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(tbar)),
                   "r"(uint32_t((CL - 1) * G * 16 * DK * 4))
                   : "memory");
    }
    if (!solo) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    auto remote = [&](const void* local, int r) {
      uint32_t a;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(local)), "r"(r));
      return a;
    };
    auto st_async4 = [&](uint32_t raddr, uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                         uint32_t rbar) {
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
              raddr),
          "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(rbar)
          : "memory");
    };
    {   // thread → kv row tid / 8, columns 4 (tid % 8) .. + 3 of this band's partial
      const int row = tid >> 3, q = tid & 7;
      const uint4 v4 = *reinterpret_cast<const uint4*>(part + row * DK + 4 * q);
      const int grp = row >> 2, o = grp / G, gi = grp - o * G;
      const float* slot = rbuf + ((rank * G + gi) * 4 + (row & 3)) * DK + 4 * q;
      if (solo) *reinterpret_cast<uint4*>(const_cast<float*>(slot)) = v4;
      else st_async4(remote(slot, o), v4.x, v4.y, v4.z, v4.w, remote(xbar, o));
      if (tid < CL * (DK / 4)) {   // counts → every CTA: thread → (rank dr, 4 counts)
        const int dr = tid / (DK / 4), k = tid % (DK / 4);
        const uint4 c4 = *reinterpret_cast<const uint4*>(cntp + 4 * k);
        if (solo) *reinterpret_cast<uint4*>(cbuf + rank * DK + 4 * k) = c4;
        else st_async4(remote(cbuf + rank * DK + 4 * k, dr), c4.x, c4.y, c4.z, c4.w, remote(xbar, dr));
      }
    }
    if (solo) {
      __syncthreads();
    } else {
      asm volatile(
          "{\n\t.reg .pred q;\n\tWX_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t"
          "@!q bra WX_%=;\n\t}" ::"r"(su32(xbar))
          : "memory");
    }
    if (tid < G * DK) {   // owner: thread = (own group, column)
      const float g = __ldg(p.gk + b * H + hz);
      const int gi = tid / DK, c = tid % DK, grp = rank * G + gi;
      float row[4] = {0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < CL; ++r) {   // rank order, as the pull form
        const float* pr = rbuf + ((r * G + gi) * 4) * DK + c;
        row[0] += pr[0];
        row[1] += pr[DK];
        row[2] += pr[2 * DK];
        row[3] += pr[3 * DK];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) row[i] = __fmul_rn(row[i], g);   // not contracted into the table sums
      float val[16];
      val[0] = 0.f;
      val[1] = row[0];
      val[2] = row[1];
      val[4] = row[2];
      val[8] = row[3];
#pragma unroll
      for (int m = 3; m < 16; ++m)
        if (m & (m - 1)) val[m] = val[m & (m - 1)] + val[m & -m];
#pragma unroll
      for (int m = 0; m < 16; ++m) tab[(grp * 16 + m) * DK + c] = val[m];
    }
    if (tid < DK) {   // total counts (rank order)
      int sc = 0;
      for (int r = 0; r < CL; ++r) sc += cbuf[r * DK + tid];
      cntw[tid] = sc;
    }
    __syncthreads();
    // this CTA's table groups → every peer (G × 16 × DK floats, contiguous)
    const float* mine = tab + rank * G * 16 * DK;
    for (int i = tid; i < (CL - 1) * G * 4 * DK; i += kThreads) {
      const int pr = i / (G * 4 * DK), k = i - pr * (G * 4 * DK);
      const int dr = pr < rank ? pr : pr + 1;
      const uint4 v4 = *reinterpret_cast<const uint4*>(mine + 4 * k);
      st_async4(remote(mine + 4 * k, dr), v4.x, v4.y, v4.z, v4.w, remote(tbar, dr));
    }
    // byte tables of the counts as exact floats: tcb[g][m] = sum_{i in m} cnt[8g+i]
    for (int e = tid; e < 4 * 256; e += kThreads) {
      const int g8 = e >> 8, m = e & 255;
      int sc = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((m >> i) & 1) sc += cntw[8 * g8 + i];
      tcb[e] = float(sc);
    }
    if (!solo)
      asm volatile(
          "{\n\t.reg .pred q;\n\tWT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t"
          "@!q bra WT_%=;\n\t}" ::"r"(su32(tbar))
          : "memory");
    __syncthreads();
  } else {
  cluster.sync();
#pragma unroll 1
  for (int h = 0; h < HEADS; ++h) {
    const float g = __ldg(p.gk + b * H + hz + h);
    const int grp = tid / DK, c = tid % DK;       // tables: thread = (nibble group, column)
    float x[kMaxCluster][4];
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r) {   // issue every peer's loads before summing
      if (r < CL) {
        const float* pr = cluster.map_shared_rank(part, r) + h * DK * DK + 4 * grp * DK + c;
        x[r][0] = pr[0];
        x[r][1] = pr[DK];
        x[r][2] = pr[2 * DK];
        x[r][3] = pr[3 * DK];
      }
    }
    float row[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r)
      if (r < CL) {
        row[0] += x[r][0];
        row[1] += x[r][1];
        row[2] += x[r][2];
        row[3] += x[r][3];
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) row[i] = __fmul_rn(row[i], g);   // not contracted into the table sums
    float val[16];
    val[0] = 0.f;
    val[1] = row[0];
    val[2] = row[1];
    val[4] = row[2];
    val[8] = row[3];
#pragma unroll
    for (int m = 3; m < 16; ++m)
      if (m & (m - 1)) val[m] = val[m & (m - 1)] + val[m & -m];
    float* T = tab + size_t(h) * (DK / 4) * 16 * DK;
#pragma unroll
    for (int m = 0; m < 16; ++m) T[(grp * 16 + m) * DK + c] = val[m];
    if (tid < DK) {   // this head's total counts (rank order), 1 per lane
      int s = 0;
      for (int r = 0; r < CL; ++r) s += cluster.map_shared_rank(cntp, r)[h * DK + tid];
      cntw[tid] = s;
    }
    __syncthreads();
    // byte tables of the counts as exact floats: tcb[h][g][m] = sum_{i in m} cnt[8g+i]
    for (int e = tid; e < 4 * 256; e += kThreads) {
      const int g8 = e >> 8, m = e & 255;
      int s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((m >> i) & 1) s += cntw[8 * g8 + i];
      tcb[h * 1024 + e] = float(s);
    }
    __syncthreads();
  }
  // this CTA has read every peer's partials: arrive now, wait only before
  // exiting (peers may still be reading this CTA's part / cntp, which pass 2
  // does not touch), so an early CTA goes straight on to its outputs
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  }
  // ---- 4. pass 2: outputs ------------------------------------------------------
  wait_row(0);
  wait_row(BR + 1);
  constexpr int NCG = D / 4;                 // channel groups of 4
  constexpr int SLOTS = kThreads / NCG;      // (row, segment) units per round
  constexpr int kSeg = seg_len(SIDE);
  constexpr int SEGS = (SIDE + kSeg - 1) / kSeg;
  static_assert(kThreads % NCG == 0, "every thread has a pass-2 slot");
  const int cgi = tid % NCG, slot = tid / NCG;
  const int h = cgi / (DK / 4), cgl = cgi % (DK / 4);
  const int ch = cgi * 4;
  const float gq = __ldg(p.gq + b * H + hz + h), gk = __ldg(p.gk + b * H + hz + h);
  const float gg = gq * gk;
  ulonglong2 tapu[9];
#pragma unroll
  for (int q = 0; q < 9; ++q)
    tapu[q] = p.dw ? __ldg(reinterpret_cast<const ulonglong2*>(p.dw + q * ld + hz * DK + ch))
                   : make_ulonglong2(0ull, 0ull);
  const bool has_dw = p.dw != nullptr;
  const uint8_t* T = reinterpret_cast<const uint8_t*>(tab + size_t(h) * (DK / 4) * 16 * DK + cgl * 4);
  const float* Tb = tcb + h * 1024;
  const uint32_t* cqh = cqs + h * nt;
  const int units = (r1 - r0) * SEGS;
  float* ob = p.out + size_t(b) * n * ld + hz * DK + ch;
  const ulonglong2 z2 = make_ulonglong2(0ull, 0ull);
  for (int u = slot; u < units; u += SLOTS) {
    const int rl = u / SEGS, sg = u - rl * SEGS;
    const int r = r0 + rl;
    const int c0 = sg * kSeg;
    const int c1 = min(SIDE, c0 + kSeg);
    // column c of smem rows rl..rl+2 (grid rows r-1..r+1) at colb + c*TOKB + R*ROWB
    const uint8_t* colb = Vb + rl * ROWB + ch * 4;
    auto load_col = [&](Win& w, int c) {
      if (c >= 0 && c < SIDE) {
        const uint8_t* q = colb + c * TOKB;
        w.r[0] = lds128(q);
        w.r[1] = lds128(q + ROWB);
        w.r[2] = lds128(q + 2 * ROWB);
      } else {
        w.r[0] = z2;
        w.r[1] = z2;
        w.r[2] = z2;
      }
    };
    // ring of three window columns; roles rotate with the (unrolled) step index
    Win wr[3];
    load_col(wr[0], c0 - 1);
    load_col(wr[1], c0);
    const int tb = r * SIDE + c0;
    const int kmax = min(c1 - c0, n - tb);
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
      if (k >= kmax) break;
      const int c = c0 + k;
      Win& wl = wr[k % 3];
      Win& wc = wr[(k + 1) % 3];
      Win& wn = wr[(k + 2) % 3];
      load_col(wn, c + 1);
      const int t = tb + k;
      const uint32_t q = cqh[t - t_lo];
      // additive Q·(K^T V): 8 nibble-table rows, packed f32x2 adds
      unsigned long long a01 = 0ull, a23 = 0ull;
#pragma unroll
      for (int g = 0; g < DK / 4; ++g) {
        const uint32_t off = (g >= 2 ? (q >> (4 * g - 7)) : (q << (7 - 4 * g))) & 0x780u;
        const ulonglong2 tv = lds128(T + g * 16 * DK * 4 + off);
        add2(a01, tv.x);
        add2(a23, tv.y);
      }
      // D = sum of the counts of the query's set bits: 4 byte-table lookups
      const float D_ = (Tb[q & 255] + Tb[256 + ((q >> 8) & 255)]) +
                       (Tb[512 + ((q >> 16) & 255)] + Tb[768 + (q >> 24)]);
      const float sc = gq * rcp_approx(fmaf(gg, D_, p.eps));
      const float2 x01 = unpack2(a01), x23 = unpack2(a23);
      float4 o = make_float4(__fmul_rn(x01.x, sc), __fmul_rn(x01.y, sc), __fmul_rn(x23.x, sc),
                             __fmul_rn(x23.y, sc));
      if (has_dw) {
        unsigned long long s01 = 0ull, s23 = 0ull;
#pragma unroll
        for (int R = 0; R < 3; ++R) {
          fma2(s01, wl.r[R].x, tapu[R * 3 + 0].x);
          fma2(s23, wl.r[R].y, tapu[R * 3 + 0].y);
          fma2(s01, wc.r[R].x, tapu[R * 3 + 1].x);
          fma2(s23, wc.r[R].y, tapu[R * 3 + 1].y);
          fma2(s01, wn.r[R].x, tapu[R * 3 + 2].x);
          fma2(s23, wn.r[R].y, tapu[R * 3 + 2].y);
        }
        const float2 y01 = unpack2(s01), y23 = unpack2(s23);
        o.x = __fadd_rn(o.x, y01.x);
        o.y = __fadd_rn(o.y, y01.y);
        o.z = __fadd_rn(o.z, y23.x);
        o.w = __fadd_rn(o.w, y23.y);
      }
      *reinterpret_cast<float4*>(ob + size_t(t) * ld) = o;
    }
  }
  if (!push) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Split form (two kernels, no cluster): the same band geometry and the same
// arithmetic in the same order as binattn_fused_kernel, so the output is
// bit-identical; the band partials travel through global memory (L2) instead
// of distributed shared memory. Without the cluster barriers each kernel runs
// at its own occupancy: pass 1 is FP32-pipe work over a shared-memory V band,
// pass 2 streams outputs with the DWConv window read through L1.

// shared-memory layout of the pass-1 kernel (byte offsets): two band buffers
// (V rows, K codes) so the next band's copies overlap this band's FMA work
struct KvSmem {
  uint32_t v[2], ck[2], scr, mt, bar, total;
};
__host__ __device__ inline KvSmem kv_smem_layout(int side, int band_rows, int nbuf) {
  KvSmem s;
  uint32_t o = 0;
  for (int i = 0; i < 2; ++i) {
    s.v[i] = o;                                          // band rows, no halo
    if (i < nbuf) o += uint32_t(band_rows) * side * DK * 4;
  }
  for (int i = 0; i < 2; ++i) {
    s.ck[i] = o;
    if (i < nbuf) o += (uint32_t(band_rows) * side * 4 + 15) & ~15u;
  }
  s.scr = o;                                             // [4][DK][DK] + [kStreams][DK]
  o += 4 * DK * DK * 4 + kStreams * DK * 4;
  s.mt = o;                                              // [256][8] 0/1 masks
  o += 256 * 8 * 4;
  s.bar = o;                                             // [2][band_rows] mbarriers
  o += 2 * band_rows * 8;
  s.total = o;
  return s;
}

// pass 1, persistent: CTA c takes work items c, c + G, ... (item = (image,
// head, band)); per item the band partial of K^T V (un-scaled) and of the
// code-bit counts → part[item][DK*DK], cntp[item][DK]
template <int SIDE>
__global__ void __launch_bounds__(kThreads, 2) binattn_kv_kernel(Params p, float* __restrict__ part_g,
                                                                 int* __restrict__ cnt_g, int CL,
                                                                 int items) {
  constexpr uint32_t ROWB = uint32_t(SIDE) * DK * 4;
  constexpr uint32_t TOKB = uint32_t(DK) * 4;
  extern __shared__ __align__(16) uint8_t smem[];
  const int H = p.heads, ld = p.ld, n = p.n, BR = p.band_rows;
  // one item per CTA (grid = items): a single band buffer; persistent: two
  const KvSmem L = kv_smem_layout(SIDE, BR, int(gridDim.x) >= items ? 1 : 2);
  float* tab = reinterpret_cast<float*>(smem + L.scr);
  float* mt = reinterpret_cast<float*>(smem + L.mt);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool bulk = ld == DK;   // contiguous rows: bulk copies; head slices: cp.async
  struct Item {
    int b, hz, rank, r0, r1, t_lo, nt;
  };
  auto geom = [&](int it) {
    Item I;
    I.rank = it % CL;
    const int bh = it / CL;
    I.b = bh / H;
    I.hz = bh - I.b * H;
    I.r0 = I.rank * BR;
    I.r1 = min(p.rows_total, I.r0 + BR);
    I.t_lo = min(n, I.r0 * SIDE);
    I.nt = min(n, I.r1 * SIDE) - I.t_lo;
    return I;
  };
  // V of item I into buffer `buf` (rows arrive on bar[buf][R] in bulk mode)
  auto issue = [&](const Item& I, int buf) {
    const float* vb = p.v + size_t(I.b) * n * ld + I.hz * DK;
    uint8_t* Vb = smem + L.v[buf];
    if (bulk) {
      if (tid == 0) {
        for (int R = 0; R < BR; ++R) {
          const int rr = I.r0 + R;
          const int ntok = rr < p.rows_total ? max(0, min(SIDE, n - rr * SIDE)) : 0;
          const uint32_t bytes = uint32_t(ntok) * TOKB;
          uint64_t* br = bar + buf * BR + R;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(br)),
                       "r"(bytes)
                       : "memory");
          if (bytes == 0) continue;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(Vb + R * ROWB)),
              "l"(vb + size_t(rr) * SIDE * DK), "r"(bytes), "r"(su32(br))
              : "memory");
        }
      }
    } else {
      for (int i = tid; i < I.nt * (DK / 4); i += kThreads) {
        const int t = i / (DK / 4), c4 = i % (DK / 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(Vb) + uint32_t(t) * TOKB + c4 * 16),
                     "l"(vb + size_t(I.t_lo + t) * ld + c4 * 4)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  constexpr int kCodesPerThread = (kMaxCluster * 64 + kThreads - 1) / kThreads;   // unused bound
  (void)kCodesPerThread;
  if (tid == 0) {
    for (int i = 0; i < 2 * BR; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int i = tid; i < 256 * 8; i += kThreads) mt[i] = ((i >> 3) >> (i & 7)) & 1 ? 1.0f : 0.0f;
  int it = blockIdx.x;
  if (it < items) {
    const Item I0 = geom(it);
    issue(I0, 0);
    uint32_t* ck0 = reinterpret_cast<uint32_t*>(smem + L.ck[0]);
    for (int i = tid; i < I0.nt; i += kThreads)
      ck0[i] = __ldg(p.ck + (size_t(I0.b) * H + I0.hz) * n + I0.t_lo + i);
  }
  __syncthreads();
  uint32_t use_par[2] = {0u, 0u};
  const int s_id = tid >> 4, rg = (tid >> 2) & 3, cgp = tid & 3;
  const uint8_t* mtb = reinterpret_cast<const uint8_t*>(mt);
  for (int k = 0; it < items; it += gridDim.x, ++k) {
    const int buf = k & 1;
    const Item I = geom(it);
    const int it_n = it + gridDim.x;
    Item In;
    uint32_t ckn[2] = {0u, 0u};   // next item's codes, held in registers until this band is done
    if (it_n < items) {
      In = geom(it_n);
      issue(In, buf ^ 1);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = tid + u * kThreads;
        if (i < In.nt) ckn[u] = __ldg(p.ck + (size_t(In.b) * H + In.hz) * n + In.t_lo + i);
      }
    }
    if (!bulk) {   // this band's cp.async group (the next band's may stay in flight)
      if (it_n < items) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    const uint8_t* Vb = smem + L.v[buf];
    const uint32_t* cks = reinterpret_cast<const uint32_t*>(smem + L.ck[buf]);
    auto wait_row = [&](int R) {
      asm volatile(
          "{\n\t.reg .pred q;\n\tW_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n\t"
          "@!q bra W_%=;\n\t}" ::"r"(su32(bar + buf * BR + R)),
          "r"(use_par[buf])
          : "memory");
    };
    unsigned long long acc[8][4], cacc[4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) cacc[j] = 0ull;
    const uint8_t* vp = Vb + (cgp * 8) * 4 + s_id * TOKB;
    const uint32_t* kp = cks + s_id;
    int next_row = 0, R_w = 0;
#pragma unroll 2
    for (int t = s_id; t < I.nt; t += kStreams) {
      if (bulk) {
        while (t >= next_row) {
          wait_row(R_w);
          ++R_w;
          next_row += SIDE;
        }
      }
      const ulonglong2 va = lds128(vp);
      const ulonglong2 vc = lds128(vp + 16);
      const uint8_t* mrow = mtb + (((*kp) >> (rg * 8)) & 0xffu) * 32;
      const ulonglong2 mp0 = lds128(mrow);
      const ulonglong2 mp1 = lds128(mrow + 16);
      const float2 m01 = unpack2(mp0.x), m23 = unpack2(mp0.y);
      const float2 m45 = unpack2(mp1.x), m67 = unpack2(mp1.y);
      const float m[8] = {m01.x, m01.y, m23.x, m23.y, m45.x, m45.y, m67.x, m67.y};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        add2_mask(acc[i][0], va.x, m[i]);
        add2_mask(acc[i][1], va.y, m[i]);
        add2_mask(acc[i][2], vc.x, m[i]);
        add2_mask(acc[i][3], vc.y, m[i]);
      }
      add2(cacc[0], mp0.x);
      add2(cacc[1], mp0.y);
      add2(cacc[2], mp1.x);
      add2(cacc[3], mp1.y);
      vp += kStreams * TOKB;
      kp += kStreams;
    }
    if (bulk) {   // consume every row's phase (streams with few tokens skip rows)
      while (R_w < BR) {
        wait_row(R_w);
        ++R_w;
      }
    }
    use_par[buf] ^= 1u;
    // same fixed-order combine as binattn_fused_kernel
    float2 cmb[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 a = unpack2(acc[i][j]);
        cmb[i][j] = make_float2(a.x + __shfl_down_sync(0xffffffffu, a.x, 16),
                                a.y + __shfl_down_sync(0xffffffffu, a.y, 16));
      }
    float* scr = tab + (warp & 3) * DK * DK + rg * 8 * DK + cgp * 8;
    if (warp >= 4 && lane < 16) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<float2*>(scr + i * DK + 2 * j) = cmb[i][j];
    }
    if (cgp == 0) {
      float* cs = tab + 4 * DK * DK + s_id * DK + rg * 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) *reinterpret_cast<float2*>(cs + 2 * j) = unpack2(cacc[j]);
    }
    __syncthreads();
    if (warp < 4 && lane < 16) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2* q = reinterpret_cast<float2*>(scr + i * DK + 2 * j);
          const float2 o = *q;
          *q = make_float2(cmb[i][j].x + o.x, cmb[i][j].y + o.y);
        }
    }
    __syncthreads();
    {
      const int e = tid * 4;
      float4 s4 = *reinterpret_cast<const float4*>(tab + e);
#pragma unroll
      for (int w4 = 1; w4 < 4; ++w4) {
        const float4 q4 = *reinterpret_cast<const float4*>(tab + w4 * DK * DK + e);
        s4.x += q4.x;
        s4.y += q4.y;
        s4.z += q4.z;
        s4.w += q4.w;
      }
      *reinterpret_cast<float4*>(part_g + size_t(it) * DK * DK + e) = s4;
    }
    if (tid < DK) {
      const float* cs = tab + 4 * DK * DK + tid;
      float c = 0.f;
#pragma unroll
      for (int st = 0; st < kStreams; ++st) c += cs[st * DK];
      cnt_g[size_t(it) * DK + tid] = int(c);
    }
    if (it_n < items) {   // next band's codes into the other buffer
      uint32_t* ckb = reinterpret_cast<uint32_t*>(smem + L.ck[buf ^ 1]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = tid + u * kThreads;
        if (i < In.nt) ckb[i] = ckn[u];
      }
      for (int i = tid + 2 * kThreads; i < In.nt; i += kThreads)
        ckb[i] = __ldg(p.ck + (size_t(In.b) * H + In.hz) * n + In.t_lo + i);
    }
    __syncthreads();   // scratch, this buffer and the codes may be reused
  }
}

// pass 2: rank-order sum of the CL band partials, nibble / byte tables, and the
// output loop of binattn_fused_kernel with the DWConv window read from global
template <int SIDE>
__global__ void __launch_bounds__(kThreads, 2) binattn_out_kernel(Params p, const float* __restrict__ part_g,
                                                                  const int* __restrict__ cnt_g, int CL) {
  constexpr int NCG = DK / 4;
  constexpr int SLOTS = kThreads / NCG;
  constexpr int kSeg = seg_len(SIDE);
  constexpr int SEGS = (SIDE + kSeg - 1) / kSeg;
  constexpr uint32_t ROWB = uint32_t(SIDE) * DK * 4;
  constexpr uint32_t TOKB = uint32_t(DK) * 4;
  __shared__ __align__(16) float tab[(DK / 4) * 16 * DK];   // 16 KB nibble tables
  __shared__ __align__(16) float tcb[4 * 256];
  __shared__ int cntw[DK];
  __shared__ __align__(8) uint64_t bar[kMaxBandRows + 2];
  extern __shared__ __align__(16) uint8_t dsm[];            // V band + halo rows, then q codes
  const int rank = blockIdx.x, b = blockIdx.y, hz = blockIdx.z, H = p.heads;
  const int ld = p.ld, n = p.n, BR = p.band_rows;
  const int tid = threadIdx.x;
  const int r0 = rank * BR;
  const int r1 = min(p.rows_total, r0 + BR);
  const int t_lo = min(n, r0 * SIDE), t_hi = min(n, r1 * SIDE);
  const int nt = t_hi - t_lo;
  const size_t slot0 = (size_t(b) * H + hz) * CL;
  uint8_t* Vb = dsm;
  uint32_t* cqs = reinterpret_cast<uint32_t*>(dsm + size_t(BR + 2) * ROWB);
  {
    // V rows r0-1 .. r0+BR (smem row R = grid row r0-1+R), as binattn_fused_kernel
    const float* vb = p.v + size_t(b) * n * ld + hz * DK;
    if (tid == 0) {
      for (int R = 0; R < BR + 2; ++R)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + R)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int i = 0; i < BR + 2; ++i) {
        const int R = i < BR ? i + 1 : (i == BR ? 0 : BR + 1);
        const int rr = r0 - 1 + R;
        const int ntok = (rr >= 0 && rr < p.rows_total) ? max(0, min(SIDE, n - rr * SIDE)) : 0;
        const uint32_t bytes = ld == DK ? uint32_t(ntok) * TOKB : 0u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + R)),
                     "r"(bytes)
                     : "memory");
        if (bytes == 0) continue;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(Vb + R * ROWB)),
            "l"(vb + size_t(rr) * SIDE * DK), "r"(bytes), "r"(su32(bar + R))
            : "memory");
      }
    }
    if (ld != DK) {
      const int tok_lo = max(0, (r0 - 1) * SIDE);
      const int tok_hi = min(n, (r0 + BR + 1) * SIDE);
      const int smem_tok0 = (r0 - 1) * SIDE;
      for (int i = tid; i < (tok_hi - tok_lo) * (DK / 4); i += kThreads) {
        const int t = tok_lo + i / (DK / 4), c4 = i % (DK / 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(Vb) + uint32_t(t - smem_tok0) * TOKB + c4 * 16),
                     "l"(vb + size_t(t) * ld + c4 * 4)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int R = 0; R < BR + 2; ++R) {   // zero the cells no copy fills
      const int rr = r0 - 1 + R;
      const int ntok = (rr >= 0 && rr < p.rows_total) ? max(0, min(SIDE, n - rr * SIDE)) : 0;
      float4* z = reinterpret_cast<float4*>(Vb + R * ROWB + ntok * TOKB);
      const int nz = (SIDE - ntok) * DK / 4;
      for (int i = tid; i < nz; i += kThreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  for (int i = tid; i < nt; i += kThreads) cqs[i] = __ldg(p.cq + (size_t(b) * H + hz) * n + t_lo + i);
  {
    const float g = __ldg(p.gk + b * H + hz);
    const int grp = tid / DK, c = tid % DK;
    float x[kMaxCluster][4];
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r) {
      if (r < CL) {
        const float* pr = part_g + (slot0 + r) * DK * DK + 4 * grp * DK + c;
        x[r][0] = __ldg(pr);
        x[r][1] = __ldg(pr + DK);
        x[r][2] = __ldg(pr + 2 * DK);
        x[r][3] = __ldg(pr + 3 * DK);
      }
    }
    float row[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < kMaxCluster; ++r)
      if (r < CL) {
        row[0] += x[r][0];
        row[1] += x[r][1];
        row[2] += x[r][2];
        row[3] += x[r][3];
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) row[i] = __fmul_rn(row[i], g);   // not contracted into the table sums
    float val[16];
    val[0] = 0.f;
    val[1] = row[0];
    val[2] = row[1];
    val[4] = row[2];
    val[8] = row[3];
#pragma unroll
    for (int m = 3; m < 16; ++m)
      if (m & (m - 1)) val[m] = val[m & (m - 1)] + val[m & -m];
#pragma unroll
    for (int m = 0; m < 16; ++m) tab[(grp * 16 + m) * DK + c] = val[m];
    if (tid < DK) {
      int s = 0;
      for (int r = 0; r < CL; ++r) s += __ldg(cnt_g + (slot0 + r) * DK + tid);
      cntw[tid] = s;
    }
  }
  __syncthreads();
  for (int e = tid; e < 4 * 256; e += kThreads) {
    const int g8 = e >> 8, m = e & 255;
    int s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if ((m >> i) & 1) s += cntw[8 * g8 + i];
    tcb[e] = float(s);
  }
  __syncthreads();
  const int cgi = tid % NCG, slot = tid / NCG;
  const int ch = cgi * 4;
  const float gq = __ldg(p.gq + b * H + hz), gk = __ldg(p.gk + b * H + hz);
  const float gg = gq * gk;
  ulonglong2 tapu[9];
#pragma unroll
  for (int q = 0; q < 9; ++q)
    tapu[q] = p.dw ? __ldg(reinterpret_cast<const ulonglong2*>(p.dw + q * ld + hz * DK + ch))
                   : make_ulonglong2(0ull, 0ull);
  const bool has_dw = p.dw != nullptr;
  const uint8_t* T = reinterpret_cast<const uint8_t*>(tab + ch);
  float* ob = p.out + size_t(b) * n * ld + hz * DK + ch;
  const ulonglong2 z2 = make_ulonglong2(0ull, 0ull);
  const int units = (r1 - r0) * SEGS;
  if (ld != DK) asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();   // zero fill and strided copies visible
  for (int R = 0; R < BR + 2; ++R) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t"
        "@!q bra W_%=;\n\t}" ::"r"(su32(bar + R))
        : "memory");
  }
  for (int u = slot; u < units; u += SLOTS) {
    const int rl = u / SEGS, sg = u - rl * SEGS;
    const int r = r0 + rl;
    const int c0 = sg * kSeg;
    const int c1 = min(SIDE, c0 + kSeg);
    const uint8_t* colb = Vb + rl * ROWB + ch * 4;
    auto load_col = [&](Win& w, int c) {
      if (c >= 0 && c < SIDE) {
        const uint8_t* q = colb + c * TOKB;
        w.r[0] = lds128(q);
        w.r[1] = lds128(q + ROWB);
        w.r[2] = lds128(q + 2 * ROWB);
      } else {
        w.r[0] = z2;
        w.r[1] = z2;
        w.r[2] = z2;
      }
    };
    Win wr[3];
    load_col(wr[0], c0 - 1);
    load_col(wr[1], c0);
    const int tb = r * SIDE + c0;
    const int kmax = min(c1 - c0, n - tb);
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
      if (k >= kmax) break;
      const int c = c0 + k;
      Win& wl = wr[k % 3];
      Win& wc = wr[(k + 1) % 3];
      Win& wn = wr[(k + 2) % 3];
      load_col(wn, c + 1);
      const int t = tb + k;
      const uint32_t q = cqs[t - t_lo];
      unsigned long long a01 = 0ull, a23 = 0ull;
#pragma unroll
      for (int g = 0; g < DK / 4; ++g) {
        const uint32_t off = (g >= 2 ? (q >> (4 * g - 7)) : (q << (7 - 4 * g))) & 0x780u;
        const ulonglong2 tv = lds128(T + g * 16 * DK * 4 + off);
        add2(a01, tv.x);
        add2(a23, tv.y);
      }
      const float D_ = (tcb[q & 255] + tcb[256 + ((q >> 8) & 255)]) +
                       (tcb[512 + ((q >> 16) & 255)] + tcb[768 + (q >> 24)]);
      const float sc = gq * rcp_approx(fmaf(gg, D_, p.eps));
      const float2 x01 = unpack2(a01), x23 = unpack2(a23);
      float4 o = make_float4(__fmul_rn(x01.x, sc), __fmul_rn(x01.y, sc), __fmul_rn(x23.x, sc),
                             __fmul_rn(x23.y, sc));
      if (has_dw) {
        unsigned long long s01 = 0ull, s23 = 0ull;
#pragma unroll
        for (int R = 0; R < 3; ++R) {
          fma2(s01, wl.r[R].x, tapu[R * 3 + 0].x);
          fma2(s23, wl.r[R].y, tapu[R * 3 + 0].y);
          fma2(s01, wc.r[R].x, tapu[R * 3 + 1].x);
          fma2(s23, wc.r[R].y, tapu[R * 3 + 1].y);
          fma2(s01, wn.r[R].x, tapu[R * 3 + 2].x);
          fma2(s23, wn.r[R].y, tapu[R * 3 + 2].y);
        }
        const float2 y01 = unpack2(s01), y23 = unpack2(s23);
        o.x = __fadd_rn(o.x, y01.x);
        o.y = __fadd_rn(o.y, y01.y);
        o.z = __fadd_rn(o.z, y23.x);
        o.w = __fadd_rn(o.w, y23.y);
      }
      *reinterpret_cast<float4*>(ob + size_t(t) * ld) = o;
    }
  }
}

}  // namespace baf

// Host side: picks the cluster geometry and launches; returns SA_ERR_VALUE when
// the shape is outside this kernel's envelope (the caller then uses the
// multi-kernel path of binattn.cu).
SA_DEBUG_SWITCH(int, g_attn_pull, 0, sa_debug_attn_pull)

int binattn_fused_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                         const float* v, const float* dw, float* out, int64_t B, int64_t n,
                         int64_t d, int64_t heads, float eps, cudaStream_t s) {
  using namespace baf;
  if (d != heads * DK || d % 4 != 0) return SA_ERR_VALUE;
  int side = 0;
  while (int64_t(side) * side < n) ++side;
  const int rows_total = int((n + side - 1) / side);
  // one CTA per (band, image, head): bands of ~400 tokens amortise the table
  // work; a head slice of a wider model is a strided view (row stride d)
  // (16-CTA non-portable clusters measured 1.8x slower: GPC packing)
  int cl = int((n + K2A_BAND_TOKENS - 1) / K2A_BAND_TOKENS);
  cl = cl < 1 ? 1 : (cl > kMaxCluster ? kMaxCluster : cl);
  cl = cl > rows_total ? rows_total : cl;
  const int br = (rows_total + cl - 1) / cl;
  cl = (rows_total + br - 1) / br;
  const Smem L = smem_layout(DK, 1, side, br);
  if (L.total > 220 * 1024) return SA_ERR_VALUE;
  if (br * side > 32 * 63) return SA_ERR_VALUE;   // bit-sliced counters hold 63 tokens/lane
  Params p{cq, ck, gq, gk, v, dw, out, int(n), DK, int(heads), side, rows_total, br, eps, int(d),
           g_attn_pull};
  void (*kern)(Params, CUtensorMap) = nullptr;
  switch (side) {
    case 56: kern = binattn_fused_kernel<DK, 56>; break;
    case 28: kern = binattn_fused_kernel<DK, 28>; break;
    case 14: kern = binattn_fused_kernel<DK, 14>; break;
    case 7: kern = binattn_fused_kernel<DK, 7>; break;
    case 15: kern = binattn_fused_kernel<DK, 15>; break;
    case 18: kern = binattn_fused_kernel<DK, 18>; break;
    case 3: kern = binattn_fused_kernel<DK, 3>; break;
    default: return SA_ERR_VALUE;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
  if (cl > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(cl), unsigned(B), unsigned(heads));
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(cl);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // V as a (channel, token, image) tensor: per-image token bounds make the
  // cells past n out of bounds (zero fill), the halo rows negative / past n
  CUtensorMap tmV;
  memset(&tmV, 0, sizeof(tmV));
  {
    const cuuint64_t dims[3] = {cuuint64_t(d), cuuint64_t(n), cuuint64_t(B)};
    const cuuint64_t strides[2] = {cuuint64_t(d) * 4, cuuint64_t(n) * cuuint64_t(d) * 4};
    const cuuint32_t box[3] = {cuuint32_t(DK), cuuint32_t(side), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if ((reinterpret_cast<uintptr_t>(v) & 15) != 0 ||
        encode_tmap_tiled(&tmV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(v), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return SA_ERR_VALUE;   // (the caller falls back to the multi-kernel path)
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, tmV);
  if (e != cudaSuccess) {
    set_error("sa_linear_binary_attn: fused launch failed: %s", cudaGetErrorString(e));
    return SA_ERR_CUDA;
  }
  count_launch(1);
  return SA_OK;
}

// Split launch (see binattn_kv_kernel / binattn_out_kernel): same geometry as
// binattn_fused_launch; the band partials go to `ws` ([B*H][CL][DK*DK] floats,
// then [B*H][CL][DK] ints). Returns SA_ERR_VALUE outside the envelope.
SA_DEBUG_SWITCH(int, g_kv_persistent, 0, sa_debug_attn_kv_persistent)

size_t binattn_split_ws_bytes(int64_t B, int64_t heads) {
  using namespace baf;
  return size_t(B * heads * kMaxCluster) * (DK * DK + DK) * 4;
}

int binattn_split_launch(const uint32_t* cq, const uint32_t* ck, const float* gq, const float* gk,
                         const float* v, const float* dw, float* out, int64_t B, int64_t n,
                         int64_t d, int64_t heads, float eps, void* ws, size_t ws_bytes,
                         cudaStream_t s) {
  using namespace baf;
  if (d != heads * DK || d % 4 != 0) return SA_ERR_VALUE;
  if (ws_bytes < binattn_split_ws_bytes(B, heads)) return SA_ERR_VALUE;
  int side = 0;
  while (int64_t(side) * side < n) ++side;
  const int rows_total = int((n + side - 1) / side);
  int cl = int((n + K2A_BAND_TOKENS - 1) / K2A_BAND_TOKENS);
  cl = cl < 1 ? 1 : (cl > kMaxCluster ? kMaxCluster : cl);
  cl = cl > rows_total ? rows_total : cl;
  const int br = (rows_total + cl - 1) / cl;
  cl = (rows_total + br - 1) / br;
  const int items = int(B * heads * cl);
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one band per CTA (two CTAs per SM) measured faster than a persistent,
  // double-buffered grid of one CTA per SM (8 warps cannot hide the per-token
  // shared-memory chain); g_kv_persistent selects the latter for A/B runs
  const int g1 = g_kv_persistent ? (items < sms ? items : sms) : items;
  const KvSmem L = kv_smem_layout(side, br, g1 >= items ? 1 : 2);
  if (L.total > 220 * 1024) return SA_ERR_VALUE;
  Params p{cq, ck, gq, gk, v, dw, out, int(n), DK, int(heads), side, rows_total, br, eps, int(d),
           g_attn_pull};
  float* part = static_cast<float*>(ws);
  int* cntp = reinterpret_cast<int*>(part + size_t(B * heads * cl) * DK * DK);
  if (br > kMaxBandRows) return SA_ERR_VALUE;
  const size_t out_smem = size_t(br + 2) * side * DK * 4 + size_t(br) * side * 4;
  void (*k1)(Params, float*, int*, int, int) = nullptr;
  void (*k2)(Params, const float*, const int*, int) = nullptr;
  switch (side) {
#define SA_SPLIT_CASE(S)                   \
  case S:                                  \
    k1 = binattn_kv_kernel<S>;             \
    k2 = binattn_out_kernel<S>;            \
    break;
    SA_SPLIT_CASE(56) SA_SPLIT_CASE(28) SA_SPLIT_CASE(14) SA_SPLIT_CASE(7)
    SA_SPLIT_CASE(15) SA_SPLIT_CASE(18) SA_SPLIT_CASE(3)
#undef SA_SPLIT_CASE
    default: return SA_ERR_VALUE;
  }
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(out_smem));
  const dim3 grid{unsigned(cl), unsigned(B), unsigned(heads)};
  k1<<<g1, kThreads, L.total, s>>>(p, part, cntp, cl, items);
  k2<<<grid, kThreads, out_smem, s>>>(p, part, cntp, cl);
  count_launch(2);
  SA_LAUNCH_CHECK("sa_linear_binary_attn (split)");
  return SA_OK;
}

}  // namespace sa
