/*
 * shiftadd_b200.h — C-ABI of libshiftadd_b200.so, the sm_100a implementation of
 * the ShiftAddViT (arXiv 2306.06446) inference hot path.
 *
 * The reference (/root/reference/pkg/src/shiftadd) is a pure-numpy package with
 * no FFI; each entry point below replaces the numpy function cited beside it,
 * and the Python package `paper_2306_06446_b200` binds these symbols through
 * ctypes behind the reference's own module API.
 *
 * Conventions
 *  - every tensor argument is a DEVICE pointer to a contiguous row-major array;
 *    activations are float32 "flat token" matrices (tokens, channels) exactly
 *    like the reference's (batch*n, d) layout (ref model.py:340-345);
 *  - heads are contiguous channel blocks, head i = channels [i*dk, (i+1)*dk)
 *    (ref attention.py:74-78);
 *  - binary codes are packed uint32 words laid out [B][heads][n][ceil(dk/32)];
 *    bit j of word w is the code of channel 32w+j; code = !(x < 0)
 *    (ref quantize.py:78-80, model.py:357-358);
 *  - shift weights are one byte per weight: bit7 = (s < 0), bits0-4 = P - p_min
 *    (ref quantize.py:44-59, 83-101);
 *  - `stream` is a cudaStream_t passed as void*; nothing synchronises the host;
 *  - the library never allocates: callers pass workspace of at least the size
 *    returned by the matching *_workspace() query;
 *  - return value 0 = ok; otherwise an SA_ERR_* code and a thread-local message
 *    from sa_last_error(). The Python shim maps SA_ERR_SHAPE → ShapeError,
 *    SA_ERR_VALUE → ValueError, SA_ERR_STATE → StateError, SA_ERR_CUDA →
 *    RuntimeError (ref tensor.py:25-30).
 */
#ifndef SHIFTADD_B200_H
#define SHIFTADD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA_OK 0
#define SA_ERR_SHAPE 1
#define SA_ERR_VALUE 2
#define SA_ERR_CUDA 3
#define SA_ERR_STATE 4

/* weight kinds for sa_linear / sa_mlp */
#define SA_W_DENSE 0 /* float32 (K, N) */
#define SA_W_SHIFT 1 /* packed shift bytes (K, N) */

/* ---- library ----------------------------------------------------------- */
const char* sa_version(void);
const char* sa_last_error(void);
int sa_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* number of kernels this library has launched since load (for bench evidence) */
uint64_t sa_launch_count(void);

/* ---- K1 sign-hash: replaces quantize.binarize(x, "per-head") + sign_unit as
 * called at model.py:355-358 (module form attention.binarize_qk,
 * attention.py:155-167). x: (B*n, d) projection output. Writes codes
 * [B][heads][n][ceil(dk/32)] and gamma[B*heads] = mean|x| per (image, head). */
size_t sa_sign_hash_workspace(int64_t B, int64_t n, int64_t d, int64_t heads);
int sa_sign_hash(const float* x, int64_t B, int64_t n, int64_t d, int64_t heads,
                 uint32_t* codes, float* gamma, void* ws, size_t ws_bytes, void* stream);

/* ---- K2a linear binary attention: replaces attention.linear_core on the
 * {0,1}·gamma features (attention.py:113-120) plus the DWConv V-branch
 * (attention._dwconv_tokens, attention.py:170-179) as composed by
 * AttentionLayer.forward (model.py:354-373). v: (B*n, d). dw: (3,3,d) or NULL.
 * out: (B*n, d) = merged heads (+ dwconv(v)), i.e. the input of W_O. */
size_t sa_linear_binary_attn_workspace(int64_t B, int64_t n, int64_t d, int64_t heads);
int sa_linear_binary_attn(const uint32_t* codes_q, const uint32_t* codes_k,
                          const float* gamma_q, const float* gamma_k, const float* v,
                          const float* dw, float* out, int64_t B, int64_t n, int64_t d,
                          int64_t heads, float eps, void* ws, size_t ws_bytes, void* stream);

/* ---- K2b quadratic Hamming attention: the (QK)V order of the same function
 * (associativity, ref tests/test_attention.py:72-79): S_ij = popc(cq_i & ck_j),
 * out_i = gq*gk*sum_j S_ij v_j / (gq*gk*sum_j S_ij + eps). Same arguments. */
int sa_hamming_attn(const uint32_t* codes_q, const uint32_t* codes_k, const float* gamma_q,
                    const float* gamma_k, const float* v, const float* dw, float* out,
                    int64_t B, int64_t n, int64_t d, int64_t heads, float eps, void* stream);

/* integer popcount statistics of the binary attention (parity evidence):
 * cnt[B*heads][dk] = sum_j c_k[j][a]; D[B*heads][n] = sum_a c_q[i][a]*cnt[a];
 * S (optional, may be NULL) [B*heads][n][n] = popc(cq_i & ck_j). */
int sa_binary_popcounts(const uint32_t* codes_q, const uint32_t* codes_k, int64_t B,
                        int64_t n, int64_t dk, int64_t heads, int32_t* cnt, int32_t* D,
                        int32_t* S, void* stream);

/* depthwise 3x3 over the ceil(sqrt(n))^2 token grid, zero padded
 * (attention._dwconv_tokens, attention.py:170-179): out = (accumulate ? out : 0)
 * + dwconv(v) */
int sa_dwconv_tokens(const float* v, const float* dw, float* out, int64_t B, int64_t n,
                     int64_t d, int accumulate, void* stream);

/* ---- K3 shift-Linear -------------------------------------------------------
 * sa_quantize_shift replaces quantize.quantize_shift (quantize.py:83-96): for
 * each of `count` weights, s = sign_unit(w), P = clip(rint(log2|w|)), zeros →
 * p_min; writes the packed byte and optionally s (float) and P (int32). */
int sa_quantize_shift(const float* w, int64_t count, int p_min, int p_max, uint8_t* packed,
                      float* s_out, int32_t* p_out, void* stream);
/* sa_shift_linear replaces quantize.shift_forward (quantize.py:104-109) /
 * ShiftLinearLayer.forward (model.py:145-148): y = x @ (s * 2^P).
 * variant 0: decoded weights on the GEMM path; variant 1: literal
 * exponent-field add + fp32 add (no multiply). */
int sa_shift_linear(const float* x, const uint8_t* packed, float* y, int64_t M, int64_t K,
                    int64_t N, int p_min, int variant, void* stream);

/* sa_add_linear replaces quantize.add_matmul (quantize.py:143-160) for an
 * AddLinear(b, gamma) layer (quantize.py:62-75): y = gamma * (x @ b) with b in
 * {-1, +1}, computed by signed fp64 accumulation (adds and subtracts only)
 * and one multiply by gamma. signs: K x N bytes, bit 7 set where b < 0. */
int sa_add_linear(const float* x, const uint8_t* signs, double gamma, float* y, int64_t M,
                  int64_t K, int64_t N, void* stream);

/* ---- dense / shift linear with fused epilogue: replaces Linear.forward
 * (model.py:104-107) and ShiftLinearLayer.forward; y = [residual +] act(x @ W).
 * act: 0 none, 1 gelu (tanh form). residual may be NULL. */
int sa_linear(const float* x, const void* w, int w_kind, float* y, int64_t M, int64_t K,
              int64_t N, int p_min, const float* residual, int act, void* stream);

/* two-layer MLP (Mlp.forward, model.py:204-208): y = [residual +] fc2(gelu(fc1(x)));
 * fc1/fc2 each dense or shift (w*_kind). */
size_t sa_mlp_workspace(int64_t M, int64_t hidden);
int sa_mlp(const float* x, const void* w1, int w1_kind, const void* w2, int w2_kind,
           float* y, int64_t M, int64_t d, int64_t hidden, int p_min,
           const float* residual, void* ws, size_t ws_bytes, void* stream);

/* ---- K4 top-1 two-expert router + stable partition: replaces moe.route
 * (moe.py:81-84) + moe.dispatch (moe.py:87-92). logits = f32(fp64 x·W_g);
 * expert 1 wins iff l1 > l0 and f32(l0 - l1) < -tie_thresh (numpy-exp rule,
 * SURVEY §8a-10); gate = p[winner]; perm = [expert-0 tokens ascending |
 * expert-1 tokens ascending]; counts[2]. logits (M,2) may be NULL. */
size_t sa_moe_route_workspace(int64_t M);
int sa_moe_route(const float* x, const float* wg, int64_t M, int64_t d, float tie_thresh,
                 float* logits, int32_t* expert_of, float* gate, int32_t* counts,
                 int32_t* perm, void* ws, size_t ws_bytes, void* stream);

/* LayerNorm.forward (model.py:174-178) fused with 1..3 routers reading its output
 * (the q/k/v MoE projections share one input, model.py:342-345; the MLP router
 * reads ln2): y = LN(x); for router r: logits from wg_r (d, 2), then the same
 * winner / gate / stable partition as sa_moe_route into expert_of[r*M..],
 * gate[r*M..], counts[2r..], perm[r*M..]. d = 32 or 64. */
size_t sa_ln_route_workspace(int64_t M, int nr);
int sa_ln_route(const float* x, const float* gain, const float* bias, float* y, int64_t M,
                int64_t d, float eps, int nr, const float* wg0, const float* wg1,
                const float* wg2, float tie_thresh, int32_t* expert_of, float* gate,
                int32_t* counts, int32_t* perm, void* ws, size_t ws_bytes, void* stream);

/* the stable partition only (moe.dispatch's index_of, moe.py:91) from winners
 * already on the device: counts[2], perm = [expert-0 ascending | expert-1
 * ascending]. Used to materialise dispatch plans lazily. */
size_t sa_moe_partition_workspace(int64_t M);
int sa_moe_partition(const int32_t* expert_of, int64_t M, int32_t* counts, int32_t* perm,
                     void* ws, size_t ws_bytes, void* stream);

/* dispatch only (moe.dispatch, moe.py:87-92) from precomputed logits (M, 2) */
int sa_moe_dispatch(const float* logits, int64_t M, float tie_thresh, int32_t* expert_of,
                    float* gate, int32_t* counts, int32_t* perm, void* ws, size_t ws_bytes,
                    void* stream);

/* ---- K5 MoE expert launch (gather → expert → ×gate → scatter), replacing
 * MoeModule.forward (model.py:250-274) / moe.moe_forward (moe.py:95-108) with
 * expert 0 = mult (dense) and expert 1 = shift. Both experts run in ONE grid;
 * counts are read on the device (no host sync, CUDA-graph capturable).
 * y[tok] = [residual[tok] +] gate[tok] * expert(x[tok]). */
int sa_moe_linear(const float* x, const int32_t* perm, const int32_t* counts,
                  const float* gate, const float* w_dense, const uint8_t* w_shift, int p_min,
                  float* y, const float* residual, int64_t M, int64_t K, int64_t N,
                  void* stream);
size_t sa_moe_mlp_workspace(int64_t M, int64_t hidden);
int sa_moe_mlp(const float* x, const int32_t* perm, const int32_t* counts, const float* gate,
               const float* w1_dense, const float* w2_dense, const uint8_t* w1_shift,
               const uint8_t* w2_shift, int p_min, float* y, const float* residual,
               int64_t M, int64_t d, int64_t hidden, void* ws, size_t ws_bytes, void* stream);

/* ---- K6 plain GEMM (tensor.matmul, tensor.py:68-75): c = a @ b, float32. */
int sa_gemm(const float* a, const float* b, float* c, int64_t M, int64_t K, int64_t N,
            void* stream);

/* ---- tensor-core (tcgen05 / TMEM) path, float32-faithful ---------------------
 * Activations are split into hi+mid+lo bf16 planes (exact); shift weights are
 * exact in bf16 (1 plane, 3 MMAs per product), dense weights use 3 planes
 * (6 MMAs per product). Weights are packed once into the shared-memory image
 * the kernels copy with one bulk async copy per 32-wide K stage. `bn` is the
 * N tile (32, 64, 128, 160 or 256; sa_tc_tile_n picks it for an N). */
int sa_tc_tile_n(int64_t N);
size_t sa_weight_pack_bytes(int64_t K, int64_t N, int w_kind, int bn);
/* w: float32 (K,N) for SA_W_DENSE or packed shift bytes (K,N) for SA_W_SHIFT */
int sa_weight_pack(const void* w, int w_kind, int64_t K, int64_t N, int p_min, int bn,
                   void* out, void* stream);
/* Linear.forward / ShiftLinearLayer.forward (model.py:104-107, 145-148) */
int sa_tc_linear(const float* x, const void* wpack, int w_kind, int bn, float* y, int64_t M,
                 int64_t K, int64_t N, const float* residual, int act, void* stream);
/* MoeModule.forward with (Linear, ShiftLinearLayer) experts (model.py:250-274, 499-502) */
int sa_tc_moe_linear(const float* x, const int32_t* perm, const int32_t* counts,
                     const float* gate, const void* wpack_dense, const void* wpack_shift, int bn,
                     float* y, const float* residual, int64_t M, int64_t K, int64_t N,
                     void* stream);
/* the q/k/v MoE projections of one AttentionLayer (model.py:342-345) in ONE
 * launch, from stacked plans (perm / gate [nprob][M], counts [nprob][2]);
 * wpack_dense / wpack_shift: nprob packed weight pointers; y [nprob][M][N] */
int sa_tc_moe_linear_grouped(const float* x, const int32_t* perm, const int32_t* counts,
                             const float* gate, const void* const* wpack_dense,
                             const void* const* wpack_shift, int nprob, int bn, float* y,
                             int64_t M, int64_t K, int64_t N, void* stream);
size_t sa_tc_mlp_workspace(int64_t M, int64_t hidden);
/* Mlp.forward (model.py:204-208) */
int sa_tc_mlp(const float* x, const void* w1pack, int w1_kind, int bn1, const void* w2pack,
              int w2_kind, int bn2, float* y, int64_t M, int64_t d, int64_t hidden,
              const float* residual, void* ws, size_t ws_bytes, void* stream);
/* MoeModule.forward with (Mlp(Linear,Linear), Mlp(Shift,Shift)) experts (model.py:514-521) */
int sa_tc_moe_mlp(const float* x, const int32_t* perm, const int32_t* counts, const float* gate,
                  const void* w1_dense, const void* w2_dense, const void* w1_shift,
                  const void* w2_shift, int bn1, int bn2, float* y, const float* residual,
                  int64_t M, int64_t d, int64_t hidden, void* ws, size_t ws_bytes, void* stream);
/* Fused MLP on the tensor cores: fc1 → GELU → fc2 in ONE kernel, the hidden
 * activations stay on chip (TMEM → registers → TMEM); d = 32, 64 (hidden
 * chunks of 64) or d = 128, 160 (chunks of 32), hidden a multiple of the
 * chunk. W1 must be packed with bn = sa_tc_fused_mlp_chunk(d), W2 with bn = d.
 * sa_tc_fused_mlp_w1_bn() is the d <= 64 chunk (64), kept for callers of the
 * narrow form. */
int sa_tc_fused_mlp_ok(int64_t d, int64_t hidden);
int sa_tc_fused_mlp_chunk(int64_t d);
int sa_tc_fused_mlp_w1_bn(void);
int sa_tc_moe_mlp_fused(const float* x, const int32_t* perm, const int32_t* counts,
                        const float* gate, const void* w1_dense, const void* w2_dense,
                        const void* w1_shift, const void* w2_shift, float* y,
                        const float* residual, int64_t M, int64_t d, int64_t hidden,
                        void* stream);
/* sa_tc_moe_mlp_fused with the stage's final LayerNorm (model.py:565-577,
 * tensor.py:114-128) on the output rows in the same kernel, bit-identical to
 * sa_tc_moe_mlp_fused + sa_layernorm; d = 32 or 64. */
int sa_tc_moe_mlp_fused_ln(const float* x, const int32_t* perm, const int32_t* counts,
                           const float* gate, const void* w1_dense, const void* w2_dense,
                           const void* w1_shift, const void* w2_shift, float* y,
                           const float* residual, int64_t M, int64_t d, int64_t hidden,
                           const float* ln_gain, const float* ln_bias, float eps, void* stream);
int sa_tc_mlp_fused(const float* x, const void* w1pack, int w1_kind, const void* w2pack,
                    int w2_kind, float* y, int64_t M, int64_t d, int64_t hidden,
                    const float* residual, void* stream);
/* Fused attention input for d = 32 / 64 (head dim 32), n >= 32:
 * LayerNorm.forward (model.py:174-178) → the q, k, v routers (moe.py:81-92) →
 * MoeModule.forward of the three (Linear, ShiftLinearLayer) projections
 * (model.py:250-274, 499-502; both experts computed, the routed one kept) →
 * quantize.binarize per (image, head) of q and k (quantize.py:123-140 via
 * model.py:355-358). Writes expert_of / gate [3][M] (q, k, v), codes_q / codes_k
 * [B][d/32][n], gamma_q / gamma_k [B*d/32] and v (M, d). Weights packed with
 * sa_weight_pack (bn = d): dense (3 planes) and shift (1 plane) per projection. */
int sa_ln_qkv_hash_ok(int64_t d, int64_t n);
size_t sa_ln_qkv_hash_workspace(int64_t B, int64_t n, int64_t d);
int sa_ln_qkv_hash(const float* x, const float* gain, const float* bias, float eps,
                   const float* wg_q, const float* wg_k, const float* wg_v, const void* wq_dense,
                   const void* wq_shift, const void* wk_dense, const void* wk_shift,
                   const void* wv_dense, const void* wv_shift, float tie_thresh, int64_t B,
                   int64_t n, int64_t d, int32_t* expert_of, float* gate, uint32_t* codes_q,
                   uint32_t* codes_k, float* gamma_q, float* gamma_k, float* v, void* ws,
                   size_t ws_bytes, void* stream);

/* MoeModule.forward of a (Linear, ShiftLinearLayer) d -> d projection plus the
 * block residual (the attention output projection, model.py:250-274, 374,
 * 454-459) in one kernel, d = 32 / 64: router (moe.py:81-92) in the producer,
 * both experts on the tensor cores, y = residual + gate · expert(x). Writes
 * expert_of / gate [M] (the plan's partition is computed on demand with
 * sa_moe_partition). Weights packed with bn = d. */
int sa_fused_moe_linear_ok(int64_t d);
int sa_fused_moe_linear(const float* x, const float* wg, const void* w_dense, const void* w_shift,
                        const float* residual, float tie_thresh, int64_t M, int64_t d,
                        int32_t* expert_of, float* gate, float* y, void* stream);
/* sa_fused_moe_linear with the block's second LayerNorm and the MLP router in
 * the epilogue (Block.forward, model.py:454-459; moe.py:81-92): y = the block
 * residual stream h, y2 = LN2(h) and the MLP's (expert, gate) per row, each
 * bit-identical to sa_ln_route on h; d = 32 or 64. */
int sa_fused_moe_linear_ln_route(const float* x, const float* wg, const void* w_dense,
                                 const void* w_shift, const float* residual, float tie_thresh,
                                 int64_t M, int64_t d, int32_t* expert_of, float* gate, float* y,
                                 const float* ln_gain, const float* ln_bias, float eps,
                                 const float* wg2, float* y2, int32_t* expert_of2, float* gate2,
                                 void* stream);

/* patchify (model.py:557-563) + patch-embed Linear on the tensor cores */
int sa_tc_patch_embed(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                      int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                      const float* cls, const float* pos, float* y, void* stream);
/* the same followed by the stage's embedding LayerNorm (model.py:565-570 →
 * LayerNorm.forward, model.py:174-178) in the GEMM epilogue: y = LN(embed) with
 * sa_layernorm's arithmetic; d = 32 or 64, no cls / pos rows */
int sa_tc_patch_embed_ln_ok(int64_t d, int has_cls, int has_pos);
int sa_tc_patch_embed_ln(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                         int64_t patch, float sub, const void* wpack, int bn, int64_t d,
                         const float* gain, const float* bias, float eps, float* y, void* stream);

/* ---- glue ------------------------------------------------------------------ */
/* LayerNorm.forward (model.py:174-178 → tensor.layernorm, tensor.py:114-128) */
int sa_layernorm(const float* x, const float* gain, const float* bias, float* y, int64_t M,
                 int64_t d, float eps, void* stream);
/* patchify (model.py:557-563) + patch-embed Linear (+cls token, +pos):
 * grid (B,H,W,C) - sub  → y (B*(n+has_cls), d). cls (1,d) and pos ((n+has_cls),d)
 * may be NULL. */
int sa_patch_embed(const float* grid, int64_t B, int64_t H, int64_t W, int64_t C,
                   int64_t patch, float sub, const float* w, int64_t d, const float* cls,
                   const float* pos, float* y, void* stream);
/* softmax attention core on flat projections (attention.softmax_core,
 * attention.py:92-97, folded as at model.py:346-351): out (B*n, d) merged. */
int sa_softmax_attn(const float* q, const float* k, const float* v, float* out, int64_t B,
                    int64_t n, int64_t d, int64_t heads, void* stream);
/* the same on q / k / v with input row stride ld >= d (e.g. column blocks of
 * one concatenated q|k|v projection); out is (B*n, d) */
int sa_softmax_attn_strided(const float* q, const float* k, const float* v, int64_t ld,
                            float* out, int64_t B, int64_t n, int64_t d, int64_t heads,
                            void* stream);
/* tokens.mean(axis=1) (model.py:574) or the cls token (mode 1): y (B, d) */
int sa_pool(const float* x, float* y, int64_t B, int64_t n, int64_t d, int mode, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SHIFTADD_B200_H */
