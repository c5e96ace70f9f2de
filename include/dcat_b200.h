/*
 * dcat_b200.h — C ABI of the B200-native DCAT scoring path.
 *
 * This is the drop-in boundary for the reference's batch scorer
 *   std::vector<RankingOutputs> seqfm::rank_forward_batch(
 *       const TransformerParams&, const IdEmbSource&, const RankingHeadParams&,
 *       const std::vector<RankingExample>&, const FinetuneConfig&)
 *   (/root/reference/proj/include/seqfm/finetune.hpp:150-154, body finetune.cpp:414-493)
 * and for the DCAT sub-API it is built from
 *   dedup_segments   (dcat.hpp:22,   dcat.cpp:91-108)
 *   context_forward  (dcat.hpp:47-49, dcat.cpp:137-178)
 *   candidate_inputs (dcat.hpp:53-54, dcat.cpp:180-197)
 *   cross_forward    (dcat.hpp:59-60, dcat.cpp:199-271).
 *
 * Plain C types only: pointers, sizes, status codes. No torch, no C++ types.
 * Every entry point returns 0 on success or a negative DCAT_E* code; the
 * message of the last failure on the calling thread is dcat_last_error().
 * The reference throws std::runtime_error (common.hpp:9-16) where this ABI
 * returns DCAT_EINVAL; the C++ shim maps one to the other.
 *
 * Devices and threads: an entry point makes its handle's GPU current for the
 * call and restores the calling thread's current device before returning.
 * Calls on one handle must be serialised by the caller (one handle = one set
 * of streams, CUDA graphs and work buffers); different handles run
 * concurrently. Destroy entry points never fail on a shutting-down runtime.
 *
 * The same structs are consumed by the CPU oracle (oracle/dcat_oracle.h) and
 * by the reference bridge (oracle/ref_bridge.cpp), so one set of host buffers
 * feeds all three implementations.
 */
#ifndef DCAT_B200_H
#define DCAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DCAT_OK 0
#define DCAT_EINVAL (-1)      /* input violates a reference SEQFM_CHECK      */
#define DCAT_ECUDA (-2)       /* CUDA runtime / launch failure               */
#define DCAT_EUNSUPPORTED (-3) /* shape outside the device kernels (e.g. head dim) */
#define DCAT_ENOMEM (-4)
#define DCAT_ENONFINITE (-5)  /* non-finite activation (model.cpp:25-28)     */

/* ModelConfig (model.hpp:84-102). pos_learned: 1 = PosMode::Learned, 0 = None. */
typedef struct dcat_model_config {
    int32_t d_model;
    int32_t n_layers;
    int32_t n_heads;
    int32_t mlp_ratio;
    int32_t max_len;
    int32_t d_emb;
    int32_t n_actions;
    int32_t n_surfaces;
    int32_t pos_learned;
} dcat_model_config;

/* TransformerParams tensors, fp32 row-major, in the exact order of
 * TransformerParams::all_params() (model.cpp:268-286):
 *   log_tau, action_emb, surface_emb, [pos_emb if learned],
 *   phi_in.{w1,b1,w2,b2}, phi_out.{w1,b1,w2,b2}, psi.{w1,b1,w2,b2},
 *   per layer: ln1_g, ln1_b, wq, bq, wk, bk, wv, bv, wo, bo, ln2_g, ln2_b,
 *              fw1, fb1, fw2, fb2.
 * Linear weights are stored in x out (linear_forward: y = x*W + b, model.hpp:44). */
typedef struct dcat_params {
    const float* const* tensors;
    int32_t n_tensors;
} dcat_params;

/* HashedEmbeddingTable (embed.hpp:25-57): J sub-tables of R x d_sub fp32. */
typedef struct dcat_table {
    int32_t num_subtables;
    int32_t rows;
    int32_t d_sub;
    const uint64_t* seeds;          /* [J] per-subtable hash seeds          */
    const float* const* subtables;  /* [J] pointers, each R x d_sub (bits == 0) */
    /* QuantizedTable (embed.hpp:80-125): bits = 4 or 8 selects `packed`, the
     * J x R rows of ceil(d_sub * bits / 8) code bytes (int4: element e in byte
     * e / 2, low nibble first) followed by fp16 scale and fp16 bias, exactly
     * the reference's payload (and PQTB1 body, embed.cpp:212-240). Rows are
     * dequantized on the fly in the gathers: (float)code * scale + bias
     * (dequantize_row, embed.cpp:99-103). bits = 0: fp32 `subtables`. */
    int32_t bits;
    const uint8_t* packed;
} dcat_table;

/* RankingHeadParams (finetune.hpp:70-85). d_feat = d_module + d_emb + n_ctx. */
typedef struct dcat_head {
    int32_t d_module;
    int32_t d_emb;
    int32_t n_ctx;
    int32_t hidden;
    int32_t d_aux;
    const float* w1;       /* d_feat x hidden   */
    const float* b1;       /* hidden            */
    const float* w2;       /* hidden x 3        */
    const float* b2;       /* 3                 */
    const float* mod_w;    /* d_module x 3      */
    const float* mod_b;    /* 3                 */
    const float* aux_proj; /* d_aux x d_emb     */
    const float* lt;       /* d_emb             */
} dcat_head;

/* FusionVariant (finetune.hpp:29). */
enum {
    DCAT_VARIANT_BASE = 0,
    DCAT_VARIANT_AUX = 1,
    DCAT_VARIANT_AUXLT = 2,
    DCAT_VARIANT_LITE_MEAN = 3,
    DCAT_VARIANT_LITE_LAST = 4
};

/* The inference-relevant part of FinetuneConfig (finetune.hpp:87-103). */
typedef struct dcat_finetune_config {
    int32_t variant;
    int32_t use_seq_module;
    int32_t max_events;
    int32_t d_aux;
    double fresh_days;
    double mid_days;
    /* Fixed-window variant of the sequence module (context_forward_fixed /
     * cross_forward_fixed, dcat.cpp:281-415): 0 = off; window W >= 1 keeps each
     * unique's newest min(valid, W - 1) events with positions restarting at 0
     * and puts the candidate at position kept (the ring's free slot). Results
     * are the ring's (which are rotation invariant, test_dcat.cpp:341-361);
     * dedup still keys on the full event prefix; the ranking-head context
     * features use the full row. */
    int32_t window;
    int32_t reserved;
} dcat_finetune_config;

/* A request batch: the std::vector<RankingExample> of the reference
 * (finetune.hpp:36-42) as structure-of-arrays. Row i's valid event prefix
 * (Segment::valid, seqdata.hpp:62-68) is events [row_offset[i],
 * row_offset[i] + row_valid[i]) of the event pool. Rows may share storage;
 * padding past `valid` is not represented (it never affects a score).
 * Event fields follow seqdata.hpp:39-44. aux is n_rows x d_aux or NULL. */
typedef struct dcat_batch {
    int64_t n_rows;
    const int64_t* row_offset;
    const int32_t* row_valid;
    int64_t n_events;
    const uint64_t* ev_ts;
    const uint8_t* ev_action;
    const uint8_t* ev_surface;
    const uint64_t* ev_item;
    const uint64_t* candidate;
    const double* age_seconds;
    const float* aux;
    int32_t d_aux;
} dcat_batch;

/* Flags for dcat_rank_forward_batch / dcat_dedup. */
#define DCAT_INPUT_DEVICE 0x1   /* batch and output pointers are device pointers    */
#define DCAT_PRECISION_FP32 0x2 /* fp32 storage + SIMT math (parity/debug mode)     */
#define DCAT_PROFILE 0x4        /* record per-stage CUDA events (dcat_stage_times)  */
#define DCAT_OUTPUT_DEVICE 0x8  /* output pointers are device pointers (inputs per DCAT_INPUT_DEVICE) */

typedef struct dcat_model dcat_model;

const char* dcat_last_error(void);
const char* dcat_version(void);

/* Uploads parameters to `device` (fp32 -> bf16 for the tensor-core path, fp32
 * kept for the parity path). All host buffers may be freed after return. */
int dcat_model_create(const dcat_model_config* cfg, const dcat_params* params,
                      const dcat_table* table, const dcat_head* head, int32_t device,
                      dcat_model** out);
int dcat_model_destroy(dcat_model* m);

/* Bit-exact replacement of dedup_segments (dcat.cpp:91-108): rep[n_rows],
 * first[b_u] (first-appearance order), *b_u. */
int dcat_dedup(dcat_model* m, const dcat_batch* batch, int32_t* rep, int32_t* first,
               int32_t* b_u, int32_t flags, void* stream);

/* rank_forward_batch (finetune.cpp:414-493): logits[n_rows*3] and
 * module_logits[n_rows*3] in fp32 (the reference converts the fp32 values to
 * double, finetune.cpp:353-356), h_cand[n_rows*d_model] (cross_forward output,
 * unit-norm rows) when non-NULL. Every fusion variant runs on the device:
 *   Base / Aux: cross_forward rows;
 *   AuxLt: the learnable token joins each unique's context (selectors [H_lt | H_cand],
 *     ranking head d_module = 2 d_model);
 *   LiteMean / LiteLast: the pooled per-unique selector (h_cand = that selector);
 *   use_seq_module = 0: ranking head on [cand_emb | ctx] only. */
int dcat_rank_forward_batch(dcat_model* m, const dcat_batch* batch,
                            const dcat_finetune_config* cfg, float* logits,
                            float* module_logits, float* h_cand, int32_t flags, void* stream);

/* Per-layer K/V of unique u from the last dcat_rank_forward_batch call
 * (context_forward's KVCache::seqs[u], dcat.hpp:30-41), as fp32 host arrays of
 * n_u x d_model. *n receives n_u. */
int dcat_debug_kv(dcat_model* m, int32_t layer, int32_t unique, float* k, float* v, int32_t* n);

/* Stage times (ms) of the last call made with DCAT_PROFILE. Up to `cap`
 * entries; names[i] points to static strings. Returns the entry count. */
int dcat_stage_times(dcat_model* m, const char** names, float* ms, int32_t cap);

/* Counters of the last call: kernels launched, unique users, context tokens. */
typedef struct dcat_call_stats {
    int64_t kernel_launches;
    int64_t b_u;
    int64_t ctx_tokens;
    int64_t gemm_launches;
    double gemm_flops;      /* algorithmic flops of all GEMM launches */
    double attn_flops;      /* algorithmic flops of the attention kernels */
} dcat_call_stats;
int dcat_last_stats(dcat_model* m, dcat_call_stats* out);

/* Page-locked host memory for staging batches (cudaHostAlloc): copies from it to the device are
 * asynchronous DMA. Used by the C++ shim to pack std::vector<RankingExample> batches. */
int dcat_host_alloc(uint64_t bytes, void** out);
int dcat_host_free(void* p);

/* ---- The DCAT sub-API (dcat.hpp:47-78) with a device-resident K/V cache ----------------------
 * context_forward (dcat.hpp:47-49, dcat.cpp:137-178) / context_forward_fixed (dcat.hpp:95-98,
 * dcat.cpp:281-336) -> dcat_kv (KVCache / FixedKVCache, dcat.hpp:30-41, 65-78, kept on the device),
 * candidate_inputs (dcat.hpp:53-54, dcat.cpp:180-197), cross_forward / cross_forward_fixed
 * (dcat.hpp:59-60, 100-101, dcat.cpp:199-271, 338-415). A cache computed once can be crossed with
 * any number of candidate batches. Pointers are host memory unless DCAT_INPUT_DEVICE; a cache and
 * the crosses over it use one precision (DCAT_PRECISION_FP32 or not). */
typedef struct dcat_kv dcat_kv;

/* One unique sequence per batch row (row_offset / row_valid / ev_*; candidate / age / aux
 * unused). window = 0: the full valid prefix (context_forward); window >= 1: the newest window - 1
 * events with positions from 0 (context_forward_fixed; the ring rotation does not change results).
 * emit_hidden = 1 runs the last layer in full; h_user (NULL or sum_u n_u x d_model fp32, row u's
 * tokens after rows 0..u-1) then receives phi_out of every token. *out owns the device cache. */
int dcat_context_forward(dcat_model* m, const dcat_batch* uniques, int32_t window, int32_t emit_hidden,
                         float* h_user, int32_t flags, void* stream, dcat_kv** out);
int dcat_kv_destroy(dcat_kv* kv);
/* n_uniques, n_layers, d_model and the per-unique token counts (SeqKV::n / FixedSeqKV::kept) of
 * a cache; n may be NULL. */
int dcat_kv_info(const dcat_kv* kv, int32_t* n_uniques, int32_t* n_layers, int32_t* d_model, int32_t* n);
/* Layer `layer` K and V of unique u (SeqKV::k[layer], v[layer]) as fp32 host n_u x d_model. */
int dcat_kv_read(const dcat_kv* kv, int32_t layer, int32_t unique, float* k, float* v);
/* e_cand[n x d_emb] fp32 = id embedding of items[i] + pos_emb[pos[i]] (candidate_inputs). */
int dcat_candidate_inputs(dcat_model* m, const uint64_t* items, const int32_t* pos, int64_t n, float* e_cand,
                          int32_t flags, void* stream);
/* cross_forward: h[n x d_model] (unit-norm rows) for candidate rows b whose unique is rep[b] (an
 * index into the rows given to dcat_context_forward, DedupPlan::rep) with inputs e_cand[n x d_emb]
 * (fp32, candidate_inputs). The fixed-window cache gives cross_forward_fixed. */
int dcat_cross_forward(dcat_model* m, const dcat_kv* kv, const int32_t* rep, const float* e_cand, int64_t n,
                       float* h, int32_t flags, void* stream);

/* ---- rank_forward_batch over several GPUs of one box from one process -----------------------
 * Rows are split user-disjoint by a content hash of their event span (equal sequences always on one
 * device, so each device's dedup equals the global one), uniques assigned longest-processing-time
 * first on a config-aware cost; every device scores its rows in its own host thread; the scores
 * are gathered to devices[0] with one NCCL group (send / recv over NVLink) and returned in the
 * caller's row order. Host buffers; errors via dcat_multi_last_error(). */
typedef struct dcat_multi dcat_multi;
const char* dcat_multi_last_error(void);
int dcat_multi_create(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                      const dcat_head* head, const int32_t* devices, int32_t n_devices, dcat_multi** out);
int dcat_multi_destroy(dcat_multi* mh);
int dcat_multi_rank_forward_batch(dcat_multi* mh, const dcat_batch* batch, const dcat_finetune_config* cfg,
                                  float* logits, float* module_logits, int32_t flags);
/* the device index (into devices[]) each row of `batch` is scored on */
int dcat_multi_shard(dcat_multi* mh, const dcat_batch* batch, int32_t* owner);

/* Test instrumentation: device counters of a model created with the environment variable
 * DCAT_DEBUG_COUNTERS set (none otherwise). out[0] = online-softmax rescale events of the causal
 * (context) attention kernel, out[1] = of the crossing kernel. Reads and resets them; returns the
 * number of counters written (0 when the model has none). */
int dcat_debug_counters(dcat_model* m, uint64_t* out, int32_t cap);

#ifdef __cplusplus
}
#endif

#endif /* DCAT_B200_H */
