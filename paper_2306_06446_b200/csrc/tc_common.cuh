// sm_100a tensor-core plumbing: mbarriers, bulk async copies, TMEM allocation,
// tcgen05.mma issue / commit, TMEM loads, UMMA shared-memory descriptors, and
// the float32 → 3×bf16 split used for float32-faithful products.
//
// Operand layout (both A and B, K-major, SWIZZLE_NONE "interleaved" canonical
// form): a tile of R rows × BK bf16 is stored as core matrices of 8 rows × 16 B;
// element (r, k) lives at byte
//     (r / 8) * SBO + (k / 8) * LBO + (r % 8) * 16 + (k % 8) * 2
// with LBO = 128 B (next 8 k) and SBO = BK * 16 B (next 8 rows). One MMA
// consumes K = 16, i.e. two core matrices along K, so the descriptor start
// address advances by 2 * LBO = 256 B per k-step.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace sa {

// cuTensorMapEncodeTiled resolved through the runtime's driver entry point, so
// the library has no link-time dependency on libcuda (it loads on machines
// without a driver; the call itself needs one).
inline CUresult encode_tmap_tiled(CUtensorMap* map, CUtensorMapDataType dt, cuuint32_t rank,
                                  void* gaddr, const cuuint64_t* dims, const cuuint64_t* strides,
                                  const cuuint32_t* box, const cuuint32_t* estr,
                                  CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                                  CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || f == nullptr)
      return CUDA_ERROR_NOT_FOUND;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn(map, dt, rank, gaddr, dims, strides, box, estr, il, sw, l2, oob);
}

namespace tc {

constexpr int kBK = 32;            // K per shared-memory stage
constexpr uint32_t kLBO = 128;
constexpr uint32_t kSBO = kBK * 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Interleaved (SWIZZLE_NONE) K-major layout: core matrices of 8 rows x 16 B.
// (A probe, scripts/probe_mma.py, measured the same tcgen05.mma rate for this
// layout and for SWIZZLE_64B: ~46 cycles per 128x32x16 MMA, 64 at N=128,
// 128 at N=256 — the per-instruction floor, not shared-memory bandwidth.)
__host__ __device__ __forceinline__ uint32_t plane_offset(int r, int k) {
  return uint32_t(r >> 3) * kSBO + uint32_t(k >> 3) * kLBO + uint32_t(r & 7) * 16 +
         uint32_t(k & 7) * 2;
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// tx bytes only, no arrival (the phase still needs its arrivals)
__device__ __forceinline__ void mbar_add_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the same on a shared-space address, with a suspend-time hint: a waiting
// thread sleeps until the phase completes (or the hint elapses) instead of
// spinning through issue slots its neighbours need
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity, uint32_t hint_ns = 0x100000u) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(hint_ns)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- bulk async copy global → shared (TMA engine, no tensor map) ----------
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- TMEM -----------------------------------------------------------------
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] · B[smem]^T   (both K-major), kind::f16 (bf16 in, f32 acc)
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` once every previously issued tcgen05.mma of this thread is done
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 16 consecutive fp32 columns → 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 consecutive fp32 columns → 32 registers per thread (no wait)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- TMA tensor store (2D box from shared memory) ---------------------------
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_box, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
      "r"(smem_u32(smem_box)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- descriptors ----------------------------------------------------------
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  // start >> 4 | LBO = 128 B (next 8 k) | SBO = 512 B (next 8 rows) | version 1 |
  // layout type 0 = SWIZZLE_NONE
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(kLBO >> 4) << 16) |
         (uint64_t(kSBO >> 4) << 32) | (uint64_t(1) << 46);
}
// kind::f16, A = B = BF16, D = F32, K-major A and B, M = 128
__host__ __device__ constexpr uint32_t idesc_bf16_m128(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

// One 16-deep K step of a split-precision product: every (A plane, B plane)
// pair whose combined weight is >= 2^-16, accumulated into d_tmem.
// NPB = 1 (shift weights, exact in bf16): lo·w, mid·w, hi·w.
// NPB = 3 (dense weights): lo·hi, mid·mid, hi·lo, mid·hi, hi·mid, hi·hi.
// Descriptors are pre-built for plane 0 of A and B; the other planes are
// constant byte offsets added to the 14-bit start-address field (addr >> 4),
// so the unrolled chain is just 64-bit adds and UTCHMMA issues.
template <int NPB>
__device__ __forceinline__ void mma_split_step(uint32_t d_tmem, uint64_t a0, uint64_t b0,
                                               uint32_t a_plane_bytes, uint32_t b_plane_bytes,
                                               uint32_t idesc, bool accumulate) {
  constexpr int NP = NPB == 1 ? 3 : 6;
  constexpr int pa[6] = {2, 1, 0, 1, 0, 0};
  constexpr int pb1[6] = {0, 0, 0, 0, 0, 0};
  constexpr int pb3[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int bpl = NPB == 1 ? pb1[i] : pb3[i];
    mma_bf16(d_tmem, a0 + uint64_t((pa[i] * a_plane_bytes) >> 4),
             b0 + uint64_t((bpl * b_plane_bytes) >> 4), idesc, (accumulate || i > 0) ? 1u : 0u);
  }
}

// ---- A operand in TMEM ("ts" form) -------------------------------------------
// D[tmem] (+)= A[tmem] · B[smem]^T. The A tile (M = 128) lives in TMEM with
// lane = row and 32-bit column c holding the bf16 pair (k = 2c, 2c+1), so one
// K = 16 step reads 8 columns (layout verified against torch by
// scripts/probe_mma_ts.py). Only B is read from shared memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns ← 16 registers per thread
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 32 lanes x 8 consecutive 32-bit columns ← 8 registers per thread
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Split-precision K = 16 step with A planes in TMEM (plane p at a0 + p *
// a_plane_cols columns) and B planes in shared memory (as mma_split_step).
template <int NPB>
__device__ __forceinline__ void mma_split_step_ts(uint32_t d_tmem, uint32_t a0, uint64_t b0,
                                                  uint32_t a_plane_cols, uint32_t b_plane_bytes,
                                                  uint32_t idesc, bool accumulate) {
  constexpr int NP = NPB == 1 ? 3 : 6;
  constexpr int pa[6] = {2, 1, 0, 1, 0, 0};
  constexpr int pb1[6] = {0, 0, 0, 0, 0, 0};
  constexpr int pb3[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int bpl = NPB == 1 ? pb1[i] : pb3[i];
    mma_bf16_ts(d_tmem, a0 + uint32_t(pa[i]) * a_plane_cols,
                b0 + uint64_t((bpl * b_plane_bytes) >> 4), idesc,
                (accumulate || i > 0) ? 1u : 0u);
  }
}

// ---- warp-uniform issue: the whole warp executes these, one elected lane
// issues (no compiler-generated per-instruction election loop) ------------
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
template <int NPB>
__device__ __forceinline__ void mma_split_step_ts_w(uint32_t d_tmem, uint32_t a0, uint64_t b0,
                                                    uint32_t a_plane_cols, uint32_t b_plane_bytes,
                                                    uint32_t idesc, bool accumulate) {
  constexpr int NP = NPB == 1 ? 3 : 6;
  constexpr int pa[6] = {2, 1, 0, 1, 0, 0};
  constexpr int pb1[6] = {0, 0, 0, 0, 0, 0};
  constexpr int pb3[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int bpl = NPB == 1 ? pb1[i] : pb3[i];
    mma_ts_w(d_tmem, a0 + uint32_t(pa[i]) * a_plane_cols, b0 + uint64_t((bpl * b_plane_bytes) >> 4),
             idesc, (accumulate || i > 0) ? 1u : 0u);
  }
}

// One K = 16 split-precision step as a single asm block: one elect.sync, the
// plane operands derived with PTX adds (uniform datapath), then the 3 (shift
// weights: lo·w, mid·w, hi·w) or 6 (dense: lo·hi, mid·mid, hi·lo, mid·hi,
// hi·mid, hi·hi) tcgen05.mma, smallest products first. A planes in TMEM at
// a0 + {0, 1, 2} * apc columns; B planes at b0 + {0, 1, 2} * (bpb >> 4).
__device__ __forceinline__ void mma_chain3_ts_w(uint32_t d, uint32_t a0, uint64_t b0, uint32_t apc,
                                                uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 a1, a2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 a1, %1, %3;\n\t"
      "add.u32 a2, a1, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], %2, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], %2, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, t;\n\t}" ::"r"(d),
      "r"(a0), "l"(b0), "r"(apc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_chain6_ts_w(uint32_t d, uint32_t a0, uint64_t b0, uint32_t apc,
                                                uint64_t bpd, uint32_t idesc, uint32_t acc) {
  // bpd = B plane stride already in descriptor units (bytes >> 4)
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b32 a1, a2;\n\t.reg .b64 b1, b2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u32 a1, %1, %3;\n\t"
      "add.u32 a2, a1, %3;\n\t"
      "add.u64 b1, %2, %4;\n\t"
      "add.u64 b2, b1, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], %2, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b2, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], %2, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %5, t;\n\t}" ::"r"(d),
      "r"(a0), "l"(b0), "r"(apc), "l"(bpd), "r"(idesc), "r"(acc)
      : "memory");
}

// Same chains with A in shared memory (descriptor a0, plane stride apd in
// descriptor units).
__device__ __forceinline__ void mma_chain3_ss_w(uint32_t d, uint64_t a0, uint64_t b0, uint64_t apd,
                                                uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a1, a2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u64 a1, %1, %3;\n\t"
      "add.u64 a2, a1, %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, %2, %4, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, %2, %4, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, t;\n\t}" ::"r"(d),
      "l"(a0), "l"(b0), "l"(apd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_chain6_ss_w(uint32_t d, uint64_t a0, uint64_t b0, uint64_t apd,
                                                uint64_t bpd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a1, a2, b1, b2;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.u32 t, 0, 0;\n\t"
      "add.u64 a1, %1, %3;\n\t"
      "add.u64 a2, a1, %3;\n\t"
      "add.u64 b1, %2, %4;\n\t"
      "add.u64 b2, b1, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, %2, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, b2, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, %2, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, b1, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, t;\n\t}" ::"r"(d),
      "l"(a0), "l"(b0), "l"(apd), "l"(bpd), "r"(idesc), "r"(acc)
      : "memory");
}

// ---- float32 → hi/mid/lo bf16 (hi+mid+lo == x for normal x) ---------------
struct Split3 {
  __nv_bfloat162 h, m, l;
};
// packed fp32 pair helpers (one f32x2 instruction, each lane rounded as the
// scalar operation would be)
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("{\n\t.reg .b64 ta, tb;\n\tmov.b64 ta, {%1, %2};\n\tmov.b64 tb, {%3, %4};\n\t"
      "sub.rn.f32x2 %0, ta, tb;\n\t}"
      : "=l"(r)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return make_float2(__uint_as_float(uint32_t(r)), __uint_as_float(uint32_t(r >> 32)));
}
__device__ __forceinline__ Split3 split3x2(float a, float b) {
  Split3 s;
  s.h = __floats2bfloat162_rn(a, b);
  const float2 r = sub2(make_float2(a, b), __bfloat1622float2(s.h));
  s.m = __floats2bfloat162_rn(r.x, r.y);
  const float2 l = sub2(r, __bfloat1622float2(s.m));
  s.l = __floats2bfloat162_rn(l.x, l.y);
  return s;
}
// The same exact three-plane split by TRUNCATION, with integer / fp32-add
// instructions only: hi = the upper 16 bits of x, mid = the upper 16 bits of
// r = x - hi (exact), lo = r - mid (exact; <= 8 significant bits, so its
// upper 16 bits are the whole value). hi + mid + lo == x as the RN split, but
// no F2FP conversion: those issue on the same 16-lane pipe as MUFU, which the
// GELU already saturates. Returns the three packed bf16x2 words.
struct Split3u {
  uint32_t h, m, l;
};
__device__ __forceinline__ Split3u split3x2_trunc(float a, float b) {
  Split3u s;
  const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  s.h = __byte_perm(ua, ub, 0x7632);
  const float2 r = sub2(make_float2(a, b), make_float2(__uint_as_float(ua & 0xffff0000u),
                                                       __uint_as_float(ub & 0xffff0000u)));
  const uint32_t ra = __float_as_uint(r.x), rb = __float_as_uint(r.y);
  s.m = __byte_perm(ra, rb, 0x7632);
  const float2 l = sub2(r, make_float2(__uint_as_float(ra & 0xffff0000u),
                                       __uint_as_float(rb & 0xffff0000u)));
  s.l = __byte_perm(__float_as_uint(l.x), __float_as_uint(l.y), 0x7632);
  return s;
}
__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 v) {
  return *reinterpret_cast<uint32_t*>(&v);
}

}  // namespace tc
}  // namespace sa
