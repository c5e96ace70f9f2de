// seqfm_b200.cpp — the reference-facing C++ shim over the C ABI (include/dcat_b200.h).
#include "seqfm_b200.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "../../include/dcat_b200.h"

namespace seqfm {
namespace b200 {

namespace {

void check(int rc) {
    if (rc != DCAT_OK) throw std::runtime_error(dcat_last_error());
}

dcat_model_config to_c(const ModelConfig& c) {
    dcat_model_config o{};
    o.d_model = c.d_model;
    o.n_layers = c.n_layers;
    o.n_heads = c.n_heads;
    o.mlp_ratio = c.mlp_ratio;
    o.max_len = c.max_len;
    o.d_emb = c.d_emb;
    o.n_actions = c.n_actions;
    o.n_surfaces = c.n_surfaces;
    o.pos_learned = c.pos_mode == ModelConfig::PosMode::Learned ? 1 : 0;
    return o;
}

// SoA view of a std::vector<RankingExample>; one event span per row (rows of a
// request that carry the same Segment object could share one, this keeps it simple)
struct BatchSoA {
    std::vector<int64_t> off;
    std::vector<int32_t> valid;
    std::vector<uint64_t> ts, item, cand;
    std::vector<uint8_t> action, surface;
    std::vector<double> age;
    std::vector<float> aux;
    dcat_batch c{};

    BatchSoA(const std::vector<RankingExample>& b, bool with_aux) {
        size_t B = b.size(), E = 0;
        for (const auto& ex : b) E += static_cast<size_t>(std::max(0, ex.seq.valid));
        off.resize(B);
        valid.resize(B);
        cand.resize(B);
        age.resize(B);
        ts.reserve(E);
        item.reserve(E);
        action.reserve(E);
        surface.reserve(E);
        int d_aux = 0;
        if (with_aux && B) d_aux = static_cast<int>(b[0].aux.size());
        for (size_t i = 0; i < B; i++) {
            const RankingExample& ex = b[i];
            SEQFM_CHECK(ex.seq.valid >= 0 && ex.seq.valid <= ex.seq.length(), "segment valid out of range");
            off[i] = static_cast<int64_t>(ts.size());
            valid[i] = ex.seq.valid;
            for (int e = 0; e < ex.seq.valid; e++) {
                const Event& ev = ex.seq.events[static_cast<size_t>(e)];
                ts.push_back(ev.timestamp);
                action.push_back(static_cast<uint8_t>(ev.action));
                surface.push_back(static_cast<uint8_t>(ev.surface));
                item.push_back(ev.item_id);
            }
            cand[i] = ex.candidate;
            age[i] = ex.age_seconds;
            if (d_aux) {
                SEQFM_CHECK(static_cast<int>(ex.aux.size()) == d_aux, "aux dim mismatch in batch");
                aux.insert(aux.end(), ex.aux.begin(), ex.aux.end());
            }
        }
        c.n_rows = static_cast<int64_t>(B);
        c.row_offset = off.data();
        c.row_valid = valid.data();
        c.n_events = static_cast<int64_t>(ts.size());
        c.ev_ts = ts.data();
        c.ev_action = action.data();
        c.ev_surface = surface.data();
        c.ev_item = item.data();
        c.candidate = cand.data();
        c.age_seconds = age.data();
        c.aux = d_aux ? aux.data() : nullptr;
        c.d_aux = d_aux;
    }
};

dcat_finetune_config to_c(const FinetuneConfig& f) {
    dcat_finetune_config o{};
    o.variant = static_cast<int32_t>(f.variant);
    o.use_seq_module = f.use_seq_module ? 1 : 0;
    o.max_events = f.max_events;
    o.d_aux = f.d_aux;
    o.fresh_days = f.cold.fresh_days;
    o.mid_days = f.cold.mid_days;
    return o;
}

}  // namespace

Scorer::Scorer(const TransformerParams& p, const HashedEmbeddingTable& table, const RankingHeadParams& rp,
               int device) {
    std::vector<const float*> subs;
    for (int j = 0; j < table.num_subtables(); j++) subs.push_back(table.subtable(j).a.data());
    dcat_table tab{table.num_subtables(), table.rows(), table.d_sub(), table.seeds().data(), subs.data(), 0, nullptr};
    init(p, tab, rp, device);
}

// QuantizedTable id source (embed.hpp:80-125): its packed payload goes to the device as is
Scorer::Scorer(const TransformerParams& p, const QuantizedTable& table, const RankingHeadParams& rp, int device) {
    dcat_table tab{table.num_subtables(), table.rows(), table.d_sub(), table.seeds().data(), nullptr,
                   table.bits(),          table.packed_row(0, 0)};
    init(p, tab, rp, device);
}

void Scorer::init(const TransformerParams& p, const dcat_table& tab, const RankingHeadParams& rp, int device) {
    std::vector<const Param*> all = p.all_params();
    std::vector<const float*> tensors;
    for (const Param* q : all) tensors.push_back(q->v.a.data());
    dcat_params prm{tensors.data(), static_cast<int32_t>(tensors.size())};
    dcat_head head{};
    head.d_module = rp.d_module;
    head.d_emb = p.cfg.d_emb;
    head.n_ctx = rp.d_feat - rp.d_module - p.cfg.d_emb;
    head.hidden = rp.w1.v.cols;
    head.d_aux = rp.aux_proj.v.rows;
    head.w1 = rp.w1.v.a.data();
    head.b1 = rp.b1.v.a.data();
    head.w2 = rp.w2.v.a.data();
    head.b2 = rp.b2.v.a.data();
    head.mod_w = rp.mod_w.v.a.data();
    head.mod_b = rp.mod_b.v.a.data();
    head.aux_proj = rp.aux_proj.v.a.data();
    head.lt = rp.lt.v.a.data();
    dcat_model_config cfg = to_c(p.cfg);
    check(dcat_model_create(&cfg, &prm, &tab, &head, device, &m_));
    d_model_ = p.cfg.d_model;
}

Scorer::~Scorer() {
    if (m_) dcat_model_destroy(m_);
}

std::vector<RankingOutputs> Scorer::rank_forward_batch(const std::vector<RankingExample>& batch,
                                                       const FinetuneConfig& cfg) const {
    std::vector<RankingOutputs> out(batch.size());
    if (batch.empty()) return out;
    BatchSoA b(batch, cfg.variant == FusionVariant::Aux);
    dcat_finetune_config fc = to_c(cfg);
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    check(dcat_rank_forward_batch(m_, &b.c, &fc, logits.data(), mlog.data(), nullptr, flags_, nullptr));
    for (size_t i = 0; i < batch.size(); i++)
        for (int j = 0; j < kRankHeadCount; j++) {
            double l = logits[i * 3 + j];  // outputs_from, finetune.cpp:350-359
            out[i].logit[static_cast<size_t>(j)] = l;
            out[i].prob[static_cast<size_t>(j)] = 1.0 / (1.0 + std::exp(-l));
            out[i].module_logit[static_cast<size_t>(j)] = mlog[i * 3 + j];
        }
    return out;
}

Mat Scorer::candidate_outputs(const std::vector<RankingExample>& batch, const FinetuneConfig& cfg) const {
    Mat h(static_cast<int>(batch.size()), d_model_);
    if (batch.empty()) return h;
    BatchSoA b(batch, cfg.variant == FusionVariant::Aux);
    dcat_finetune_config fc = to_c(cfg);
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    check(dcat_rank_forward_batch(m_, &b.c, &fc, logits.data(), mlog.data(), h.a.data(), flags_, nullptr));
    return h;
}

Mat Scorer::candidate_outputs_fixed(const std::vector<RankingExample>& batch, const FinetuneConfig& cfg,
                                    int window) const {
    SEQFM_CHECK(window >= 1, "context_forward_fixed: window must be >= 1, got " << window);
    Mat h(static_cast<int>(batch.size()), d_model_);
    if (batch.empty()) return h;
    BatchSoA b(batch, cfg.variant == FusionVariant::Aux);
    dcat_finetune_config fc = to_c(cfg);
    fc.window = window;
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    check(dcat_rank_forward_batch(m_, &b.c, &fc, logits.data(), mlog.data(), h.a.data(), flags_, nullptr));
    return h;
}

DedupPlan Scorer::dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques) const {
    std::vector<RankingExample> ex(batch.size());
    for (size_t i = 0; i < batch.size(); i++) ex[i].seq = batch[i];
    BatchSoA b(ex, false);
    DedupPlan plan;
    plan.b = static_cast<int>(batch.size());
    plan.rep.resize(batch.size());
    plan.first.resize(batch.size());
    int32_t b_u = 0;
    if (!batch.empty()) check(dcat_dedup(m_, &b.c, plan.rep.data(), plan.first.data(), &b_u, 0, nullptr));
    plan.b_u = b_u;
    plan.first.resize(static_cast<size_t>(b_u));
    if (uniques) {
        uniques->clear();
        for (int u = 0; u < b_u; u++) uniques->push_back(batch[static_cast<size_t>(plan.first[static_cast<size_t>(u)])]);
    }
    return plan;
}

namespace {
std::mutex g_mu;
std::map<std::tuple<const void*, const void*, const void*>, std::unique_ptr<Scorer>> g_cache;

Scorer& cached(const TransformerParams& p, const IdEmbSource& ids, const RankingHeadParams& rp) {
    const auto* table = dynamic_cast<const HashedEmbeddingTable*>(&ids);
    const auto* qtable = dynamic_cast<const QuantizedTable*>(&ids);
    SEQFM_CHECK(table != nullptr || qtable != nullptr,
                "B200 scorer needs a HashedEmbeddingTable or QuantizedTable id source");
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_tuple(static_cast<const void*>(&p), static_cast<const void*>(&ids),
                               static_cast<const void*>(&rp));
    auto it = g_cache.find(key);
    if (it == g_cache.end())
        it = g_cache
                 .emplace(key, table ? std::make_unique<Scorer>(p, *table, rp) : std::make_unique<Scorer>(p, *qtable, rp))
                 .first;
    return *it->second;
}
}  // namespace

std::vector<RankingOutputs> rank_forward_batch(const TransformerParams& p, const IdEmbSource& ids,
                                               const RankingHeadParams& rp,
                                               const std::vector<RankingExample>& batch,
                                               const FinetuneConfig& cfg) {
    return cached(p, ids, rp).rank_forward_batch(batch, cfg);
}

DedupPlan dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques) {
    // the plan needs no weights: a 1-layer stub model carries the enum / position limits
    static std::mutex mu;
    static std::unique_ptr<Scorer> s;
    std::lock_guard<std::mutex> lk(mu);
    if (!s) {
        ModelConfig c;
        c.d_model = 16;
        c.n_layers = 1;
        c.n_heads = 1;
        c.d_emb = 16;
        c.max_len = 8;
        c.pos_mode = ModelConfig::PosMode::None;
        TransformerParams p;
        p.init(c, 0);
        HashedEmbeddingTable t(1, 1, 16, 0);
        RankingHeadParams rp;
        rp.init(16, 16, 1, 8, 8, 1, 0);
        s = std::make_unique<Scorer>(p, t, rp);
    }
    return s->dedup_segments(batch, uniques);
}

void invalidate() {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache.clear();
}

}  // namespace b200
}  // namespace seqfm
