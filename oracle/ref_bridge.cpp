// ref_bridge.cpp — C entry points into the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together with
// the reference's own sources under /root/reference/proj/src into
// oracle/_ref/libseqfm_ref.so. Nothing here re-implements reference math: each
// function adapts the shared C structs (include/dcat_b200.h) to the reference
// C++ types and calls the reference API:
//   TransformerParams::init        model.cpp:219
//   HashedEmbeddingTable(...)      embed.cpp:16
//   RankingHeadParams::init        finetune.cpp:77
//   dedup_segments                 dcat.cpp:91
//   context_forward                dcat.cpp:137
//   candidate_inputs / cross_forward dcat.cpp:180 / :199
//   naive_candidate_outputs        dcat.cpp:417
//   rank_forward_batch             finetune.cpp:414
// Used to generate the golden fixtures (tests/golden/make_golden.py) and as the
// reference arm of bench.py (--impl reference).
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "../include/dcat_b200.h"
#include "seqfm/dcat.hpp"
#include "seqfm/finetune.hpp"

using namespace seqfm;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        g_err.clear();
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

ModelConfig to_cfg(const dcat_model_config* c) {
    ModelConfig m;
    m.d_model = c->d_model;
    m.n_layers = c->n_layers;
    m.n_heads = c->n_heads;
    m.mlp_ratio = c->mlp_ratio;
    m.max_len = c->max_len;
    m.d_emb = c->d_emb;
    m.n_actions = c->n_actions;
    m.n_surfaces = c->n_surfaces;
    m.pos_mode = c->pos_learned ? ModelConfig::PosMode::Learned : ModelConfig::PosMode::None;
    return m;
}

TransformerParams make_params(const dcat_model_config* c, const dcat_params* prm) {
    TransformerParams p;
    p.init(to_cfg(c), 0);
    auto all = p.all_params();
    SEQFM_CHECK(static_cast<int>(all.size()) == prm->n_tensors,
                "bridge: expected " << all.size() << " tensors, got " << prm->n_tensors);
    for (size_t i = 0; i < all.size(); i++)
        std::memcpy(all[i]->v.a.data(), prm->tensors[i], sizeof(float) * all[i]->v.a.size());
    return p;
}

HashedEmbeddingTable make_table(const dcat_table* t) {
    std::vector<u64> seeds(t->seeds, t->seeds + t->num_subtables);
    HashedEmbeddingTable tab(t->rows, t->d_sub, seeds);
    for (int j = 0; j < t->num_subtables; j++)
        std::memcpy(tab.subtable(j).a.data(), t->subtables[j],
                    sizeof(float) * static_cast<size_t>(t->rows) * t->d_sub);
    return tab;
}

// The id source a call scores with: the fp32 HashedEmbeddingTable, or (bits 4 / 8) the
// reference's own quantize() of it (embed.cpp:124-171) as a QuantizedTable.
struct IdSource {
    HashedEmbeddingTable fp;
    QuantizedTable q;
    bool quant;
    explicit IdSource(const dcat_table* t) : fp(make_table(t)), quant(t->bits != 0) {
        if (quant) q = quantize(fp, t->bits);
    }
    const IdEmbSource& get() const {
        if (quant) return q;
        return fp;
    }
};

RankingHeadParams make_head(const dcat_head* h, int d_model) {
    RankingHeadParams rp;
    int sel = d_model > 0 ? h->d_module / d_model : 0;
    rp.init(d_model, h->d_emb, h->d_aux, h->n_ctx, h->hidden, sel, 0);
    auto put = [](Param& p, const float* src) {
        if (src) std::memcpy(p.v.a.data(), src, sizeof(float) * p.v.a.size());
    };
    put(rp.w1, h->w1);
    put(rp.b1, h->b1);
    put(rp.w2, h->w2);
    put(rp.b2, h->b2);
    put(rp.mod_w, h->mod_w);
    put(rp.mod_b, h->mod_b);
    put(rp.aux_proj, h->aux_proj);
    put(rp.lt, h->lt);
    return rp;
}

FinetuneConfig make_ft(const dcat_finetune_config* f, const dcat_head* h) {
    FinetuneConfig c;
    c.variant = static_cast<FusionVariant>(f->variant);
    c.use_seq_module = f->use_seq_module != 0;
    c.max_events = f->max_events;
    c.d_aux = f->d_aux;
    c.crossing_hidden = h->hidden;
    c.cold.fresh_days = f->fresh_days;
    c.cold.mid_days = f->mid_days;
    return c;
}

Segment make_segment(const dcat_batch* b, int64_t i) {
    Segment s;
    s.user_id = static_cast<u64>(i);
    s.valid = b->row_valid[i];
    s.events.resize(static_cast<size_t>(s.valid));
    int64_t o = b->row_offset[i];
    for (int e = 0; e < s.valid; e++) {
        Event& ev = s.events[static_cast<size_t>(e)];
        ev.timestamp = b->ev_ts[o + e];
        ev.action = static_cast<Action>(b->ev_action[o + e]);
        ev.surface = static_cast<Surface>(b->ev_surface[o + e]);
        ev.item_id = b->ev_item[o + e];
    }
    return s;
}

std::vector<RankingExample> make_examples(const dcat_batch* b, const std::vector<int64_t>& rows) {
    std::vector<RankingExample> out(rows.size());
    for (size_t k = 0; k < rows.size(); k++) {
        int64_t i = rows[k];
        RankingExample& ex = out[k];
        ex.seq = make_segment(b, i);
        ex.candidate = b->candidate[i];
        ex.age_seconds = b->age_seconds[i];
        if (b->aux && b->d_aux > 0)
            ex.aux.assign(b->aux + static_cast<size_t>(i) * b->d_aux,
                          b->aux + static_cast<size_t>(i + 1) * b->d_aux);
    }
    return out;
}

void copy_out(const std::vector<RankingOutputs>& r, const std::vector<int64_t>& rows, double* logits,
              double* mlogits, double* probs) {
    for (size_t k = 0; k < rows.size(); k++)
        for (int j = 0; j < 3; j++) {
            logits[rows[k] * 3 + j] = r[k].logit[static_cast<size_t>(j)];
            mlogits[rows[k] * 3 + j] = r[k].module_logit[static_cast<size_t>(j)];
            probs[rows[k] * 3 + j] = r[k].prob[static_cast<size_t>(j)];
        }
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_init_transformer(const dcat_model_config* c, uint64_t seed, float tau_init, float* const* out) {
    return guard([&] {
        TransformerParams p;
        p.init(to_cfg(c), seed, tau_init);
        auto all = p.all_params();
        for (size_t i = 0; i < all.size(); i++)
            std::memcpy(out[i], all[i]->v.a.data(), sizeof(float) * all[i]->v.a.size());
    });
}

int ref_init_table(int32_t J, int32_t R, int32_t d_sub, uint64_t seed, float stddev, uint64_t* seeds,
                   float* data) {
    return guard([&] {
        HashedEmbeddingTable t(J, R, d_sub, seed, stddev);
        for (int j = 0; j < J; j++) {
            seeds[j] = t.seeds()[static_cast<size_t>(j)];
            std::memcpy(data + static_cast<size_t>(j) * R * d_sub, t.subtable(j).a.data(),
                        sizeof(float) * static_cast<size_t>(R) * d_sub);
        }
    });
}

int ref_init_head(int32_t d_model, int32_t d_emb, int32_t d_aux, int32_t n_ctx, int32_t hidden, int32_t sel,
                  uint64_t seed, float* w1, float* b1, float* w2, float* b2, float* mod_w, float* mod_b,
                  float* aux_proj, float* lt) {
    return guard([&] {
        RankingHeadParams rp;
        rp.init(d_model, d_emb, d_aux, n_ctx, hidden, sel, seed);
        auto get = [](const Param& p, float* dst) {
            std::memcpy(dst, p.v.a.data(), sizeof(float) * p.v.a.size());
        };
        get(rp.w1, w1);
        get(rp.b1, b1);
        get(rp.w2, w2);
        get(rp.b2, b2);
        get(rp.mod_w, mod_w);
        get(rp.mod_b, mod_b);
        get(rp.aux_proj, aux_proj);
        get(rp.lt, lt);
    });
}

uint32_t ref_hash_id(uint64_t id, uint64_t seed, uint32_t rows) { return hash_id(id, seed, rows); }

int ref_dedup(const dcat_batch* b, int32_t* rep, int32_t* first, int32_t* b_u) {
    return guard([&] {
        std::vector<Segment> segs;
        segs.reserve(static_cast<size_t>(b->n_rows));
        for (int64_t i = 0; i < b->n_rows; i++) segs.push_back(make_segment(b, i));
        DedupPlan plan = dedup_segments(segs, nullptr);
        for (int i = 0; i < plan.b; i++) rep[i] = plan.rep[static_cast<size_t>(i)];
        for (int u = 0; u < plan.b_u; u++) first[u] = plan.first[static_cast<size_t>(u)];
        *b_u = plan.b_u;
    });
}

// rank_forward_batch as shipped (single-threaded, finetune.cpp:414-493).
int ref_rank_forward_batch(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                           const dcat_head* h, const dcat_finetune_config* f, const dcat_batch* b,
                           double* logits, double* mlogits, double* probs) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        RankingHeadParams rp = make_head(h, c->d_model);
        FinetuneConfig ft = make_ft(f, h);
        ft.validate(p.cfg);
        std::vector<int64_t> rows(static_cast<size_t>(b->n_rows));
        for (int64_t i = 0; i < b->n_rows; i++) rows[static_cast<size_t>(i)] = i;
        auto out = rank_forward_batch(p, tab, rp, make_examples(b, rows), ft);
        copy_out(out, rows, logits, mlogits, probs);
    });
}

// The same reference call fanned out over n_threads std::threads, each on a
// user-disjoint slice of the batch (rank_forward_batch is reentrant, its
// per-row math independent of other users: dcat.cpp:214-268).
int ref_rank_forward_batch_mt(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                              const dcat_head* h, const dcat_finetune_config* f, const dcat_batch* b,
                              double* logits, double* mlogits, double* probs, int32_t n_threads) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        RankingHeadParams rp = make_head(h, c->d_model);
        FinetuneConfig ft = make_ft(f, h);
        ft.validate(p.cfg);
        std::vector<Segment> segs;
        for (int64_t i = 0; i < b->n_rows; i++) segs.push_back(make_segment(b, i));
        DedupPlan plan = dedup_segments(segs, nullptr);
        int T = std::max(1, std::min<int>(n_threads, plan.b_u));
        std::vector<std::vector<int64_t>> slices(static_cast<size_t>(T));
        for (int64_t i = 0; i < b->n_rows; i++)
            slices[static_cast<size_t>(plan.rep[static_cast<size_t>(i)] % T)].push_back(i);
        std::vector<std::thread> th;
        std::vector<std::string> errs(static_cast<size_t>(T));
        for (int k = 0; k < T; k++)
            th.emplace_back([&, k] {
                try {
                    auto& rows = slices[static_cast<size_t>(k)];
                    if (rows.empty()) return;
                    auto out = rank_forward_batch(p, tab, rp, make_examples(b, rows), ft);
                    copy_out(out, rows, logits, mlogits, probs);
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(k)] = e.what();
                }
            });
        for (auto& x : th) x.join();
        for (auto& e : errs) SEQFM_CHECK(e.empty(), e);
    });
}

int ref_context_kv(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                   const dcat_batch* uniques, int32_t layer, int32_t unique, float* k, float* v) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        std::vector<Segment> u = {make_segment(uniques, unique)};
        KVCache cache = context_forward(p, tab, u, false);
        const SeqKV& s = cache.seqs[0];
        std::memcpy(k, s.k[static_cast<size_t>(layer)].a.data(),
                    sizeof(float) * s.k[static_cast<size_t>(layer)].a.size());
        std::memcpy(v, s.v[static_cast<size_t>(layer)].a.data(),
                    sizeof(float) * s.v[static_cast<size_t>(layer)].a.size());
    });
}

int ref_naive_candidate_outputs(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                                const dcat_batch* b, float* out) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        std::vector<Segment> segs;
        std::vector<u64> items;
        for (int64_t i = 0; i < b->n_rows; i++) {
            segs.push_back(make_segment(b, i));
            items.push_back(b->candidate[i]);
        }
        Mat h = naive_candidate_outputs(p, tab, segs, items);
        std::memcpy(out, h.a.data(), sizeof(float) * h.a.size());
    });
}

// dedup -> context_forward -> candidate_inputs -> cross_forward (dcat.cpp:531-537).
int ref_dcat_outputs(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                     const dcat_batch* b, float* h_cand) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        std::vector<Segment> segs;
        std::vector<u64> items;
        for (int64_t i = 0; i < b->n_rows; i++) {
            segs.push_back(make_segment(b, i));
            items.push_back(b->candidate[i]);
        }
        std::vector<Segment> uniques;
        DedupPlan plan = dedup_segments(segs, &uniques);
        KVCache cache = context_forward(p, tab, uniques, false);
        std::vector<int> pos;
        for (int i = 0; i < plan.b; i++) pos.push_back(uniques[static_cast<size_t>(plan.rep[static_cast<size_t>(i)])].valid);
        Mat e = candidate_inputs(p, tab, items, pos);
        Mat h = cross_forward(p, cache, plan, e);
        std::memcpy(h_cand, h.a.data(), sizeof(float) * h.a.size());
    });
}

// dedup -> context_forward_fixed(window, rotation) -> candidate_inputs(pos = kept) ->
// cross_forward_fixed (dcat.cpp:281-415), the composition test_dcat.cpp:300-339 checks.
int ref_dcat_outputs_fixed(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                           const dcat_batch* b, int32_t window, int32_t rotation, float* h_cand) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        IdSource ids(t);
        const IdEmbSource& tab = ids.get();
        std::vector<Segment> segs;
        std::vector<u64> items;
        for (int64_t i = 0; i < b->n_rows; i++) {
            segs.push_back(make_segment(b, i));
            items.push_back(b->candidate[i]);
        }
        std::vector<Segment> uniques;
        DedupPlan plan = dedup_segments(segs, &uniques);
        FixedKVCache cache = context_forward_fixed(p, tab, uniques, window, rotation);
        std::vector<int> pos;
        for (int i = 0; i < plan.b; i++)
            pos.push_back(cache.seqs[static_cast<size_t>(plan.rep[static_cast<size_t>(i)])].kept);
        Mat e = candidate_inputs(p, tab, items, pos);
        Mat h = cross_forward_fixed(p, cache, plan, e);
        std::memcpy(h_cand, h.a.data(), sizeof(float) * h.a.size());
    });
}

// quantize (embed.cpp:124-171): the QuantizedTable payload (J x R packed rows)
int ref_quantize_table(const dcat_table* t, int32_t bits, uint8_t* packed) {
    return guard([&] {
        QuantizedTable q = quantize(make_table(t), bits);
        std::memcpy(packed, q.packed_row(0, 0), q.payload_bytes());
    });
}

// save_quantized (embed.cpp:212-240): a PQTB1 file of the quantized table, with an
// optional config trailer
int ref_save_quantized(const dcat_table* t, int32_t bits, const char* config_text, const char* path) {
    return guard([&] {
        QuantizedTable q = quantize(make_table(t), bits);
        if (config_text) q.set_config_text(config_text);
        save_quantized(q, path);
    });
}

// save_checkpoint (model.cpp:645-666): PFMC1 file of the model + table, with extra config
// text and the ranking head as extra "rank.*" blobs when `head` is non-null
int ref_save_checkpoint(const dcat_model_config* c, const dcat_params* prm, const dcat_table* t,
                        const dcat_head* head, const char* extra_config, const char* path) {
    return guard([&] {
        TransformerParams p = make_params(c, prm);
        HashedEmbeddingTable tab = make_table(t);
        std::vector<std::pair<std::string, Mat>> extra;
        if (head) {
            RankingHeadParams rp = make_head(head, c->d_model);
            for (const Param* q : rp.all_params()) extra.emplace_back(q->name, q->v);
        }
        save_checkpoint(p, tab, path, extra_config ? extra_config : "", extra);
    });
}

// write_sequences (seqdata.cpp:235-259): PSEQ1 file of n_users users; user u's events are
// [offset[u], offset[u + 1]) of the pool
int ref_write_sequences(int32_t n_users, const uint64_t* user_ids, const int64_t* offsets, const uint64_t* ts,
                        const uint8_t* action, const uint8_t* surface, const uint64_t* item,
                        const char* config_text, const char* path) {
    return guard([&] {
        std::vector<UserSequence> seqs(static_cast<size_t>(n_users));
        for (int u = 0; u < n_users; u++) {
            seqs[u].user_id = user_ids[u];
            for (int64_t e = offsets[u]; e < offsets[u + 1]; e++) {
                Event ev;
                ev.timestamp = ts[e];
                ev.action = static_cast<Action>(action[e]);
                ev.surface = static_cast<Surface>(surface[e]);
                ev.item_id = item[e];
                seqs[u].events.push_back(ev);
            }
        }
        write_sequences(seqs, path, config_text ? config_text : "");
    });
}

} // extern "C"
