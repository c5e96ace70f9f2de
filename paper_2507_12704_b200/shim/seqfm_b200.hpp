// seqfm_b200.hpp — drop-in B200 scorer with the reference's C++ API.
//
// Compile inside the reference tree (needs its proj/include headers):
//   seqfm::b200::rank_forward_batch has exactly the signature of
//   seqfm::rank_forward_batch (finetune.hpp:150-154) and returns the same
//   RankingOutputs (prob via double sigmoid, finetune.cpp:355). Failures throw
//   std::runtime_error like SEQFM_CHECK (common.hpp:9-16).
// The device work happens in libdcat_b200.so through include/dcat_b200.h.
#pragma once

#include <memory>
#include <vector>

#include "seqfm/dcat.hpp"
#include "seqfm/finetune.hpp"

struct dcat_model;
struct dcat_table;

namespace seqfm {
namespace b200 {

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

    // true: fp32 storage + CUDA-core math (parity mode, DCAT_PRECISION_FP32)
    void set_fp32(bool on) { flags_ = on ? 0x2 : 0; }

private:
    void init(const TransformerParams& p, const struct dcat_table& tab, const RankingHeadParams& rp, int device);
    dcat_model* m_ = nullptr;
    int d_model_ = 0;
    int flags_ = 0;
};

// Free function with the reference signature. The ids source must be a
// HashedEmbeddingTable or a QuantizedTable. Weights are uploaded once per (p, ids, rp) address
// triple and cached; call invalidate() after changing weights in place.
std::vector<RankingOutputs> rank_forward_batch(const TransformerParams& p, const IdEmbSource& ids,
                                               const RankingHeadParams& rp,
                                               const std::vector<RankingExample>& batch,
                                               const FinetuneConfig& cfg);
DedupPlan dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques);
void invalidate();

}  // namespace b200
}  // namespace seqfm
