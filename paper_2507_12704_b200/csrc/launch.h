// launch.h — host-side launchers of the DCAT B200 kernels.
//
// Every kernel file exposes plain host functions taking device pointers and a
// stream; dcat_api.cu orchestrates them into rank_forward_batch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace dcat {

// ---------------------------------------------------------------- dedup.cu
struct DedupIn {
    int64_t B;
    const int64_t* row_offset;
    const int32_t* row_valid;
    int64_t n_events;
    const uint64_t* ts;
    const uint8_t* action;
    const uint8_t* surface;
    const uint64_t* item;
    int n_actions, n_surfaces, max_len, pos_learned;
    int window;  // fixed-window variant: keep the newest min(valid, window - 1) events (0 = off)
    int lt_token;  // AuxLt: the learnable token is appended to every unique's context (0 / 1)
};

// Events of a row's span the sequence module uses: all of them, or the newest window - 1
// (context_forward_fixed, dcat.cpp:301-302); `skip` = leading events dropped.
__host__ __device__ __forceinline__ int seq_kept(const DedupIn& in, int valid) {
    return in.window > 0 ? (valid < in.window - 1 ? valid : in.window - 1) : valid;
}
// context tokens of a unique: its kept events, plus AuxLt's learnable token (finetune.cpp:186-191)
__host__ __device__ __forceinline__ int seq_tokens(const DedupIn& in, int valid) {
    return seq_kept(in, valid) + in.lt_token;
}

// query rows per context-attention tile of the mma.sync flash kernel (attention.cu)
#ifndef DCAT_CTX_BQ
#define DCAT_CTX_BQ 64
#endif
constexpr int kCtxTile = DCAT_CTX_BQ;
// candidate rows per crossing-attention tile (mma.sync kernel: 2 m-tiles of 16 rows per warp)
#ifndef DCAT_CROSS_BQ
#define DCAT_CROSS_BQ 128
#endif
constexpr int kCrossTile = DCAT_CROSS_BQ;

struct Tile {  // one attention work item: <= BM query rows of one unique
    int q0, nq;     // first query row, number of query rows
    int kv0, nkv;   // first context K/V row, number of keys visible to the tile
    int qloc;       // causal: local position of the first query within its unique
    int u;          // unique id
    int pad0, pad1;
};

struct DedupOut {  // device buffers, sized for B rows
    uint64_t* hash;
    uint64_t* tab_key;
    int32_t* tab_val;
    int64_t tab_cap;
    int32_t* slot;
    int32_t* head;
    int32_t* collided;
    int32_t* list;       // compacted row list for the collision rounds
    int32_t* list_n;     // device counter
    int64_t* scan_tmp;   // B + 1
    int64_t* scan_blk;   // block sums
    int64_t* uid;        // B + 1 (exclusive scan of first flags)
    int32_t* rep;        // B
    int32_t* first;      // B (b_u used)
    int32_t* cnt;        // B: candidates per unique
    int32_t* cursor;     // B
    int64_t* goff;       // B + 1: candidate group offsets
    int32_t* perm;       // B: permuted position -> original row
    int64_t* tok_off;    // B + 1: context token offsets per unique
    int64_t* ctx_toff;   // B + 1: context tile offsets
    int64_t* cross_toff; // B + 1: cross tile offsets
    Status* st;
};

// Stage 1: hash / verify / first-appearance ids / groups / token offsets.
// Leaves counts in st (host reads after a sync).
void dedup_plan(const DedupIn& in, const DedupOut& o, uint64_t hash_mask, int tile_m_ctx, int tile_m_cross,
                cudaStream_t s);
// Collision repair rounds (only when st->collisions > 0): returns when fixed.
void dedup_repair(const DedupIn& in, const DedupOut& o, int n_collided, int tile_m_ctx, int tile_m_cross,
                  uint64_t hash_mask, cudaStream_t s);
// Stage 2 (after the host knows b_u / tile counts): tile lists + token map.
void build_tiles(const DedupIn& in, const DedupOut& o, int b_u, int tile_m_ctx, int tile_m_cross, Tile* ctx_tiles,
                 Tile* cross_tiles, int32_t* tok_unique, cudaStream_t s);
// Exclusive scan of n int64 values; out[n] = total; optionally copies total to *total_dst.
void scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* blk, cudaStream_t s);

// ---------------------------------------------------------------- gather.cu
struct EmbParams {
    const float* table;       // J x R x d_sub (fp32 table) or null
    const uint8_t* q;         // quantized table rows (QuantizedTable payload) or null
    int bits, row_bytes, code_bytes;
    const uint64_t* seed_mix; // J: mix64(seed_j)
    int J, R, d_sub;
    const float* action_emb;  // n_actions x d_emb
    const float* surface_emb; // n_surfaces x d_emb
    const float* pos_emb;     // max_len x d_emb or null
    int d_emb;
    const float* lt;          // AuxLt learnable token row (d_emb) or null
    // bf16 path: (action_emb[a] + surface_emb[s]) + pos_emb[i] precombined, row (a * n_surf + s) *
    // max_len + i, or null (fp32 parity path, no learned positions)
    const float* cmb;
    int n_surf, max_len;
};
// the precombined action / surface / position rows of EmbParams::cmb (n_act * n_surf * max_len x d_emb)
void build_combined_emb(const float* action_emb, const float* surface_emb, const float* pos_emb, int n_act,
                        int n_surf, int max_len, int d_emb, float* cmb, cudaStream_t s);
template <typename T>
void gather_context(const DedupIn& in, const DedupOut& o, const EmbParams& ep, const int32_t* tok_unique,
                    int64_t T_ctx, T* E, int ldE, cudaStream_t s);
struct CandParams {
    const uint64_t* candidate;
    const double* age;
    const float* aux;       // B x d_aux or null
    const float* aux_proj;  // d_aux x d_emb
    int d_aux;
    int variant_aux;
    int max_events;
    double fresh_days, mid_days;
    int d_model;            // feat column offset of cand_emb
    int feat_ld;            // feat leading dimension (0 = no feat)
    int aux_first;          // 1: (lookup + aux) + pos as build_input (finetune.cpp:193-203, AuxLt);
                            // 0: (lookup + pos) + aux as the batched Aux path (finetune.cpp:468-479)
};
// candidate_inputs (dcat.cpp:180-197): e[n x d_emb] fp32 = lookup(items) + pos_emb[pos]
void candidate_inputs(const EmbParams& ep, const uint64_t* items, const int32_t* pos, int64_t n, float* e, Status* st,
                      cudaStream_t s);
template <typename T>
void gather_candidates(const DedupIn& in, const DedupOut& o, const EmbParams& ep, const CandParams& cp, int64_t B,
                       T* E, int ldE, T* feat, cudaStream_t s);

// ---------------------------------------------------------------- gemm
enum EpiMode : int {
    EPI_BIAS = 0,       // out = act(acc + bias), split across up to 3 column segments
    EPI_RESID_LN = 1,   // x = acc + bias + resid; x_out fp32; ln_out = LN(x) (or copy of x)
    EPI_L2NORM = 2,     // y = l2norm(acc + bias); x_out fp32; ln_out = LN(y) or copy; mlogits
    EPI_HEAD = 3,       // z = gelu(acc + bias); logits = z . w2 + b2
};

struct Epi {
    int mode;
    int act;                 // EPI_BIAS: 0 none, 1 gelu
    const float* bias;       // [N]
    void* out[3];            // EPI_BIAS: activation outputs per segment
    int out_ld[3];
    int out_trans[3];        // 1: segment stored transposed, [seg_cols][out_ld] (V^T of the K/V cache)
    int seg_cols;            // columns per output segment
    const float* resid;      // EPI_RESID_LN: fp32 residual [M x ld_x]
    float* x_out;            // fp32 [M x ld_x]
    int ld_x;
    const float* ln_g;       // LN gain (null: ln_out = plain copy)
    const float* ln_b;
    void* ln_out;            // activation type
    int ln_ld;
    void* out2;              // EPI_L2NORM: second activation copy (feat), may be null
    int out2_ld;
    const float* mod_w;      // EPI_L2NORM: N x 3 module head (null = none)
    const float* mod_b;
    float* mlogits;          // [M x 3]
    const float* w2;         // EPI_HEAD: hidden x 3
    const float* b2;
    float* logits;           // [M x 3]
    Status* st;
    int layer_idx;           // for non-finite reporting (-1: no check)
    const float* o_bias;     // layer_tail_tc: attention output projection bias [d]
    const float* ln2_g;      // layer_tail_tc: LN2 (pre-FFN) gain / bias [d]
    const float* ln2_b;
};

// bf16 tensor-core GEMM (tcgen05 + TMEM + TMA): C[M x N] = A[M x K] . W^T,
// A bf16 row-major (lda), W bf16 [N x K] row-major, fused epilogue.
void gemm_tc(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K, const Epi& e, cudaStream_t s);
// Fused FFN (tcgen05): x_out = resid + gelu(A . W1t^T + bias) . W2t^T + b2, then LN -> ln_out
// (e.bias = b1 [F], e.b2 = b2 [D], resid / x_out / ld_x / ln_g / ln_b / ln_out / ln_ld as EPI_RESID_LN).
// W1t = W1^T [F x D], W2t = W2^T [D x F] (bf16, K-major).
bool ffn_tc_supported(int D, int F);
// Fused layer tail (tcgen05, one kernel): x_mid = x + (A_o . Wot^T + o_bias); h = LN2(x_mid);
// x_out = x_mid + gelu(h . W1t^T + bias) . W2t^T + b2; ln_out = LN(x_out) (next LN1) or a copy.
// e as for ffn_tc (resid = x) plus o_bias / ln2_g / ln2_b; Wot = Wo^T [D x D] (K-major).
// x_mid and h stay on the SM.
bool layer_tail_tc_supported(int D, int F);
void layer_tail_tc(const bf16* A_o, int lda, const bf16* Wot, const bf16* W1t, const bf16* W2t, int M, int D, int F,
                   const Epi& e, cudaStream_t s);
void ffn_tc(const bf16* A, int lda, const bf16* W1t, const bf16* W2t, int M, int D, int F, const Epi& e,
            cudaStream_t s);
// fp32 parity path: SIMT GEMM (W in reference in x out layout, ldw) + row epilogue.
void gemm_f32(const float* A, int lda, const float* W, int ldw, int M, int N, int K, const Epi& e, float* tmp,
              cudaStream_t s);

// ---------------------------------------------------------------- attention.cu
struct AttnArgs {
    const void* q; int ldq;        // query rows (head h at cols h*dh)
    const void* k; const void* v; int ldkv;  // context K (rows) and V (rows; bf16 path: V^T, see ldvt)
    int ldvt;                      // bf16 path: V cache is V^T [d][ldvt] (keys contiguous); 0 = row-major V
    const void* kself; const void* vself; int ldself;  // crossing: per-row own key/value
    void* out; int ldo;
    const Tile* tiles; int n_tiles;
    int n_heads, dh;
    float scale;
    int causal;                     // 1: context pass, 0: crossing (with self term)
    int max_keys;                   // fp32 path: upper bound on keys per query
    int sparse_tiles;               // crossing: tiles average under half full (k_flash skips idle warps)
    unsigned* dbg;                  // debug counters (DCAT_DEBUG_COUNTERS) or null: [0] causal / [1] crossing
                                    // online-softmax rescale events
};
void attention_bf16(const AttnArgs& a, cudaStream_t s);
void attention_f32(const AttnArgs& a, cudaStream_t s);
// FA4-style tcgen05 attention (attn_fa.cu): bf16, head dim 16 / 32 / 64, V cache transposed
// (ldvt > 0); q_rows = rows of the Q (and k_self / v_self) tensors, kv_rows = context tokens
// actually written (keys past it read as zeros).
bool attention_fa_supported(int dh);
void attention_fa(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s);

// ---------------------------------------------------------------- head / scatter
void scatter_outputs(const int32_t* perm, int64_t B, const float* logits_p, const float* mlog_p, const float* h_p,
                     int d, float* logits, float* mlogits, float* h_cand, cudaStream_t s);
// dst[p] = src[perm[p]] (fp32 rows -> activation type); scatter_rows: dst[perm[p]] = src[p]
template <typename T>
void gather_rows(const float* src, const int32_t* perm, int64_t B, int d, T* dst, cudaStream_t s);
void scatter_rows(const float* src, const int32_t* perm, int64_t B, int d, float* dst, cudaStream_t s);
// Lite selectors (gather_selectors, finetune.cpp:258-274): per unique, the mean (row-order sum,
// then one division) or the last of its token rows of H (fp32, ld d); zeros when it has none.
void pool_selectors(const int64_t* tok_off, int b_u, const float* H, int d, int last, float* sel, cudaStream_t s);
// row tok_off[u + 1] - 1 (a unique's last context token) of src -> dst row u
template <typename T>
void gather_last_rows(const int64_t* tok_off, int b_u, const T* src, int d, T* dst, cudaStream_t s);
// candidate row p (unique-grouped order) <- selector of its unique: feat[p][col0, col0 + d) (activation
// type) and, when hc is non-null, hc[p][0, d) (fp32)
template <typename T>
void broadcast_selectors(const int32_t* perm, const int32_t* rep, int64_t B, const float* sel, int d, T* feat,
                         int ld, int col0, float* hc, cudaStream_t s);
// module logits (crossing_forward, finetune.cpp:317-323) of the flattened selectors [sel_u | hc_p]
// (either part may be null): sum over k ascending of s_k * mod_w[k][j], then + mod_b[j]
void module_logits(const int32_t* perm, const int32_t* rep, int64_t B, const float* sel_u, const float* hc, int d,
                   const float* mod_w, const float* mod_b, float* mlog, cudaStream_t s);

}  // namespace dcat
