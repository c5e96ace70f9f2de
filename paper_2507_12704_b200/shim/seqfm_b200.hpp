// seqfm_b200.hpp — drop-in B200 scorer with the reference's C++ API.
//
// Compile inside the reference tree (needs its proj/include headers):
//   seqfm::b200::rank_forward_batch has exactly the signature of
//   seqfm::rank_forward_batch (finetune.hpp:150-154) and returns the same
//   RankingOutputs (prob via double sigmoid, finetune.cpp:355). Failures throw
//   std::runtime_error like SEQFM_CHECK (common.hpp:9-16).
//   The DCAT sub-API (dcat.hpp:47-101) is mirrored by context_forward /
//   candidate_inputs / cross_forward (and the fixed-window pair) over a
//   DeviceKVCache that stays resident on the GPU between calls.
// The device work happens in libdcat_b200.so through include/dcat_b200.h.
//
// Threading: every Scorer entry point takes the Scorer's own mutex (one handle = one set of
// streams and work buffers), so a Scorer may be shared by many threads; calls on
// different Scorers run concurrently. The free functions share a process-wide cache of Scorers
// held by shared_ptr (see rank_forward_batch below).
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "seqfm/dcat.hpp"
#include "seqfm/finetune.hpp"

struct dcat_model;
struct dcat_table;
struct dcat_kv;
struct dcat_multi;

namespace seqfm {
namespace b200 {

// context_forward's KVCache / FixedKVCache (dcat.hpp:30-41, 65-78), resident on the device.
class Scorer;

class DeviceKVCache {
public:
    DeviceKVCache() = default;
    ~DeviceKVCache();
    DeviceKVCache(DeviceKVCache&& o) noexcept;
    DeviceKVCache& operator=(DeviceKVCache&& o) noexcept;
    DeviceKVCache(const DeviceKVCache&) = delete;
    DeviceKVCache& operator=(const DeviceKVCache&) = delete;

    int n_uniques() const { return static_cast<int>(n_.size()); }
    int n_layers() const { return n_layers_; }
    int d_model() const { return d_model_; }
    int window() const { return window_; }  // 0: KVCache, >= 1: FixedKVCache
    const std::vector<int>& lengths() const { return n_; }  // SeqKV::n / FixedSeqKV::kept
    // host copy in the reference's KVCache layout (SeqKV::k / v per layer, n x d_model)
    KVCache to_host() const;

private:
    friend class Scorer;
    friend Mat cross_forward(const TransformerParams&, const DeviceKVCache&, const DedupPlan&, const Mat&, int);
    friend Mat cross_forward_fixed(const TransformerParams&, const DeviceKVCache&, const DedupPlan&, const Mat&, int);
    friend DeviceKVCache context_forward(const TransformerParams&, const IdEmbSource&, const std::vector<Segment>&, bool,
                                         std::vector<Mat>*, int);
    friend DeviceKVCache context_forward_fixed(const TransformerParams&, const IdEmbSource&, const std::vector<Segment>&,
                                               int, int, bool, std::vector<Mat>*, int);
    dcat_kv* kv_ = nullptr;
    const Scorer* owner_ = nullptr;         // the Scorer whose GPU holds the cache
    std::shared_ptr<const Scorer> keep_;    // free-function caches keep their cached Scorer alive
    bool fp32_ = false;
    int n_layers_ = 0, d_model_ = 0, window_ = 0;
    std::vector<int> n_;
};

// Owns one set of weights resident on one GPU.
class Scorer {
public:
    Scorer(const TransformerParams& p, const HashedEmbeddingTable& table, const RankingHeadParams& rp,
           int device = 0);
    // QuantizedTable id source (int4 / int8 rows, fp16 scale / bias; embed.hpp:80-125), e.g. from
    // load_quantized (PQTB1, embed.cpp:242-287): rows are dequantized on the device
    Scorer(const TransformerParams& p, const QuantizedTable& table, const RankingHeadParams& rp, int device = 0);
    ~Scorer();
    Scorer(const Scorer&) = delete;
    Scorer& operator=(const Scorer&) = delete;

    // rank_forward_batch (finetune.cpp:414-493) on the device.
    std::vector<RankingOutputs> rank_forward_batch(const std::vector<RankingExample>& batch,
                                                   const FinetuneConfig& cfg) const;
    // dedup_segments (dcat.cpp:91-108), bit-exact; fills uniques when non-null.
    DedupPlan dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques) const;
    // cross_forward output rows (unit-norm H_cand) of the DCAT path, B x d_model.
    Mat candidate_outputs(const std::vector<RankingExample>& batch, const FinetuneConfig& cfg) const;
    // The fixed-window variant (window >= 1): dedup_segments -> context_forward_fixed ->
    // candidate_inputs(pos = kept) -> cross_forward_fixed (dcat.cpp:281-415), B x d_model.
    // Scores equal the reference ring at any rotation (test_dcat.cpp:341-361).
    Mat candidate_outputs_fixed(const std::vector<RankingExample>& batch, const FinetuneConfig& cfg,
                                int window) const;

    // ---- the DCAT sub-API (dcat.hpp:47-101); the cache never leaves the GPU
    // context_forward (dcat.cpp:137-178): h_user (requires emit_hidden) receives phi_out of every
    // token of each unique
    DeviceKVCache context_forward(const std::vector<Segment>& uniques, bool emit_hidden = false,
                                  std::vector<Mat>* h_user = nullptr) const;
    // context_forward_fixed (dcat.cpp:281-336); results do not depend on the ring rotation
    DeviceKVCache context_forward_fixed(const std::vector<Segment>& uniques, int window, int rotation = 0,
                                        bool emit_hidden = false, std::vector<Mat>* h_user = nullptr) const;
    // candidate_inputs (dcat.cpp:180-197)
    Mat candidate_inputs(const std::vector<u64>& items, const std::vector<int>& pos_index) const;
    // cross_forward (dcat.cpp:199-271) / cross_forward_fixed (dcat.cpp:338-415) by the cache's kind
    Mat cross_forward(const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand) const;
    Mat cross_forward_fixed(const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand) const;

    // true: fp32 storage + CUDA-core math (parity mode, DCAT_PRECISION_FP32)
    void set_fp32(bool on) { flags_ = on ? 0x2 : 0; }

private:
    void init(const TransformerParams& p, const struct dcat_table& tab, const RankingHeadParams& rp, int device);
    DeviceKVCache context_impl(const std::vector<Segment>& uniques, int window, bool emit_hidden,
                               std::vector<Mat>* h_user, const char* fn) const;
    dcat_model* m_ = nullptr;
    int d_model_ = 0, d_emb_ = 0, n_layers_ = 0;
    int flags_ = 0;
    mutable std::mutex mu_;
    mutable void* stage_ = nullptr;  // page-locked staging for packed batches (grown on demand)
    mutable size_t stage_bytes_ = 0;
};

// rank_forward_batch over several GPUs of one box from one process: the multi-device drop-in for
// score_groups (finetune.cpp:766-786). Rows are split user-disjoint by a content hash of their
// events (equal sequences on one GPU, so each GPU's dedup equals the global one), uniques assigned
// longest-processing-time first on a config-aware cost, every GPU scores its rows in its own host
// thread, and the scores come back through one NCCL gather (dcat_multi_*, csrc/multi.cu). One
// device behaves exactly like a Scorer on it.
class MultiScorer {
public:
    MultiScorer(const TransformerParams& p, const HashedEmbeddingTable& table, const RankingHeadParams& rp,
                const std::vector<int>& devices);
    ~MultiScorer();
    MultiScorer(const MultiScorer&) = delete;
    MultiScorer& operator=(const MultiScorer&) = delete;
    std::vector<RankingOutputs> rank_forward_batch(const std::vector<RankingExample>& batch,
                                                   const FinetuneConfig& cfg) const;
    // the index into `devices` each example is scored on
    std::vector<int> shard(const std::vector<RankingExample>& batch) const;
    void set_fp32(bool on) { flags_ = on ? 0x2 : 0; }

private:
    struct dcat_multi* mh_ = nullptr;
    int flags_ = 0;
    mutable std::mutex mu_;
    mutable void* stage_ = nullptr;
    mutable size_t stage_bytes_ = 0;
};

// Free function with the reference signature. The ids source must be a HashedEmbeddingTable or
// a QuantizedTable. Weights are uploaded once per (p, ids, rp) and cached. The cache key is the
// three addresses plus a fingerprint of the weights (sizes and a strided sample of every tensor),
// so objects freed and reallocated at the same address with different weights get a new upload;
// invalidate() drops the cache (Scorers still in use by other threads stay alive until they return).
std::vector<RankingOutputs> rank_forward_batch(const TransformerParams& p, const IdEmbSource& ids,
                                               const RankingHeadParams& rp,
                                               const std::vector<RankingExample>& batch,
                                               const FinetuneConfig& cfg);
DedupPlan dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques);
// The sub-API with the reference signatures (n_threads is accepted and ignored: the device runs
// every unique / candidate in parallel). The returned caches live on the GPU of the Scorer the
// (p, ids) pair maps to.
DeviceKVCache context_forward(const TransformerParams& p, const IdEmbSource& ids, const std::vector<Segment>& uniques,
                              bool emit_hidden, std::vector<Mat>* h_user = nullptr, int n_threads = 1);
Mat candidate_inputs(const TransformerParams& p, const IdEmbSource& ids, const std::vector<u64>& items,
                     const std::vector<int>& pos_index);
Mat cross_forward(const TransformerParams& p, const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand,
                  int n_threads = 1);
DeviceKVCache context_forward_fixed(const TransformerParams& p, const IdEmbSource& ids,
                                    const std::vector<Segment>& uniques, int window, int rotation = 0,
                                    bool emit_hidden = false, std::vector<Mat>* h_user = nullptr, int n_threads = 1);
Mat cross_forward_fixed(const TransformerParams& p, const DeviceKVCache& cache, const DedupPlan& plan,
                        const Mat& e_cand, int n_threads = 1);
void invalidate();

}  // namespace b200
}  // namespace seqfm
