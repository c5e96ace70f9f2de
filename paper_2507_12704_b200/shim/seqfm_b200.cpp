// seqfm_b200.cpp — the reference-facing C++ shim over the C ABI (include/dcat_b200.h).
#include "seqfm_b200.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>

#include "../../include/dcat_b200.h"
#include "../csrc/host_pool.hpp"

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

size_t align16(size_t n) { return (n + 15) & ~size_t(15); }

// process-wide host workers for batch packing (created on first use, joined at exit)
dcat::ThreadPool& host_pool() {
    static dcat::ThreadPool pool(std::max(1u, std::min(16u, std::thread::hardware_concurrency())) - 1);
    return pool;
}

// a row's valid events: equal sequences (the reference's segment_key content, dcat.cpp:45-56)
bool same_events(const Segment& a, const Segment& b) {
    return a.valid == b.valid && std::equal(a.events.begin(), a.events.begin() + a.valid, b.events.begin());
}
// cheap grouping key of a row's sequence (a few of its events); equality is always verified
uint64_t seq_key(const Segment& s) {
    auto mix = [](uint64_t x) {
        x ^= x >> 30;
        x *= 0xbf58476d1ce4e5b9ULL;
        x ^= x >> 27;
        x *= 0x94d049bb133111ebULL;
        return x ^ (x >> 31);
    };
    uint64_t k = mix(static_cast<uint64_t>(s.valid) + 0x9e3779b97f4a7c15ULL);
    if (s.valid > 0) {
        const Event* e = s.events.data();
        for (int i : {0, s.valid / 2, s.valid - 1})
            k = mix(k ^ e[i].timestamp ^ (e[i].item_id << 7) ^
                    (static_cast<uint64_t>(e[i].action) << 56 | static_cast<uint64_t>(e[i].surface) << 60));
    }
    return k | 1;  // non-zero map key
}

// open-addressing map, non-zero 64-bit key -> int32 (single-threaded scratch)
struct KeyMap {
    std::vector<uint64_t> key;
    std::vector<int32_t> val;
    size_t mask = 0;
    explicit KeyMap(size_t n) {
        size_t cap = 16;
        while (cap < 2 * n) cap <<= 1;
        key.assign(cap, 0);
        val.assign(cap, -1);
        mask = cap - 1;
    }
    int32_t& slot(uint64_t k, bool* fresh) {
        size_t i = (k * 0x9e3779b97f4a7c15ULL) >> 20 & mask;
        while (key[i] != 0 && key[i] != k) i = (i + 1) & mask;
        *fresh = key[i] == 0;
        key[i] = k;
        return val[i];
    }
};

// Structure-of-arrays view of a batch (std::vector<RankingExample>, or bare Segments), packed into
// the Scorer's page-locked staging buffer so the device copies are asynchronous DMA. Every
// RankingExample owns its Segment, but rows of one user carry equal sequences: rows are grouped
// by content (a cheap key, then an exact event-by-event comparison with the group's first row, in
// parallel) and each distinct sequence is packed once, its rows sharing the span (offset, valid).
// The device dedup then settles those rows by span identity; results are the same as with a
// private copy per row, and the host copies ~1/C of the events. Up to 16 host threads.
struct BatchSoA {
    dcat_batch c{};

    template <typename SegAt, typename RowAt>
    BatchSoA(size_t B, SegAt seg_at, RowAt row_at, int d_aux, void*& stage, size_t& stage_bytes) {
        for (size_t i = 0; i < B; i++) {
            const Segment& s = seg_at(i);
            SEQFM_CHECK(s.valid >= 0 && s.valid <= s.length(), "segment valid out of range");
        }
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const size_t T = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, B / 4096));
        auto parallel = [&](size_t n, auto&& f) {  // f(lo, hi) over [0, n) in T slices, on the shim's pool
            if (T <= 1 || n < 2 * T) {
                f(size_t(0), n);
                return;
            }
            host_pool().run(static_cast<unsigned>(T),
                            [&](unsigned t) { f(n * t / T, n * (t + 1) / T); });
        };
        // 1. grouping keys (parallel), 2. provisional groups by key (first row = representative)
        std::vector<uint64_t> key(B);
        parallel(B, [&](size_t lo, size_t hi) {
            for (size_t i = lo; i < hi; i++) key[i] = seq_key(seg_at(i));
        });
        std::vector<int32_t> grp(B);
        std::vector<int64_t> rep;  // representative row of each group
        {
            KeyMap km(B);
            for (size_t i = 0; i < B; i++) {
                bool fresh;
                int32_t& g = km.slot(key[i], &fresh);
                if (fresh) {
                    g = static_cast<int32_t>(rep.size());
                    rep.push_back(static_cast<int64_t>(i));
                }
                grp[i] = g;
            }
        }
        // 3. exact verification against the representative (parallel); rows that differ (a key
        // collision) are regrouped serially among the groups of their key
        std::vector<uint8_t> odd(B, 0);
        parallel(B, [&](size_t lo, size_t hi) {
            for (size_t i = lo; i < hi; i++) {
                const int64_t r = rep[static_cast<size_t>(grp[i])];
                if (static_cast<size_t>(r) != i && !same_events(seg_at(i), seg_at(static_cast<size_t>(r)))) odd[i] = 1;
            }
        });
        std::map<uint64_t, std::vector<int32_t>> extra;  // further groups of a colliding key
        for (size_t i = 0; i < B; i++) {
            if (!odd[i]) continue;
            std::vector<int32_t>& gs = extra[key[i]];
            int32_t found = -1;
            for (int32_t g : gs)
                if (same_events(seg_at(i), seg_at(static_cast<size_t>(rep[static_cast<size_t>(g)])))) {
                    found = g;
                    break;
                }
            if (found < 0) {
                found = static_cast<int32_t>(rep.size());
                rep.push_back(static_cast<int64_t>(i));
                gs.push_back(found);
            }
            grp[i] = found;
        }
        // 4. one span per group
        const size_t G = rep.size();
        std::vector<int64_t> goff(G + 1, 0);
        for (size_t g = 0; g < G; g++) goff[g + 1] = goff[g] + seg_at(static_cast<size_t>(rep[g])).valid;
        const size_t E = static_cast<size_t>(goff[G]);
        // layout: off | valid | ts | item | cand | age | aux | action | surface
        size_t o_off = 0, o_valid = align16(o_off + 8 * B), o_ts = align16(o_valid + 4 * B), o_item = align16(o_ts + 8 * E),
               o_cand = align16(o_item + 8 * E), o_age = align16(o_cand + 8 * B), o_aux = align16(o_age + 8 * B),
               o_act = align16(o_aux + 4 * B * static_cast<size_t>(d_aux)), o_surf = align16(o_act + E),
               total = align16(o_surf + E);
        if (total > stage_bytes) {
            if (stage) dcat_host_free(stage);
            stage = nullptr;
            stage_bytes = 0;
            const size_t want = total + total / 4;
            check(dcat_host_alloc(want, &stage));
            stage_bytes = want;
        }
        uint8_t* base = static_cast<uint8_t*>(stage);
        int64_t* p_off = reinterpret_cast<int64_t*>(base + o_off);
        int32_t* p_valid = reinterpret_cast<int32_t*>(base + o_valid);
        uint64_t* p_ts = reinterpret_cast<uint64_t*>(base + o_ts);
        uint64_t* p_item = reinterpret_cast<uint64_t*>(base + o_item);
        uint64_t* p_cand = reinterpret_cast<uint64_t*>(base + o_cand);
        double* p_age = reinterpret_cast<double*>(base + o_age);
        float* p_aux = reinterpret_cast<float*>(base + o_aux);
        uint8_t* p_act = base + o_act;
        uint8_t* p_surf = base + o_surf;
        parallel(G, [&](size_t lo, size_t hi) {  // the distinct sequences' events
            for (size_t g = lo; g < hi; g++) {
                const Segment& s = seg_at(static_cast<size_t>(rep[g]));
                const size_t e0 = static_cast<size_t>(goff[g]);
                for (int e = 0; e < s.valid; e++) {
                    const Event& ev = s.events[static_cast<size_t>(e)];
                    p_ts[e0 + e] = ev.timestamp;
                    p_item[e0 + e] = ev.item_id;
                    p_act[e0 + e] = static_cast<uint8_t>(ev.action);
                    p_surf[e0 + e] = static_cast<uint8_t>(ev.surface);
                }
            }
        });
        parallel(B, [&](size_t lo, size_t hi) {  // the rows
            for (size_t i = lo; i < hi; i++) {
                p_off[i] = goff[static_cast<size_t>(grp[i])];
                p_valid[i] = seg_at(i).valid;
                row_at(i, p_cand + i, p_age + i, p_aux + i * static_cast<size_t>(d_aux));
            }
        });
        c.n_rows = static_cast<int64_t>(B);
        c.row_offset = p_off;
        c.row_valid = p_valid;
        c.n_events = static_cast<int64_t>(E);
        c.ev_ts = p_ts;
        c.ev_action = p_act;
        c.ev_surface = p_surf;
        c.ev_item = p_item;
        c.candidate = p_cand;
        c.age_seconds = p_age;
        c.aux = d_aux ? p_aux : nullptr;
        c.d_aux = d_aux;
    }
};

BatchSoA pack_examples(const std::vector<RankingExample>& b, bool with_aux, void*& stage, size_t& bytes) {
    int d_aux = with_aux && !b.empty() ? static_cast<int>(b[0].aux.size()) : 0;
    for (const auto& ex : b)
        if (d_aux) SEQFM_CHECK(static_cast<int>(ex.aux.size()) == d_aux, "aux dim mismatch in batch");
    return BatchSoA(
        b.size(), [&](size_t i) -> const Segment& { return b[i].seq; },
        [&](size_t i, uint64_t* cand, double* age, float* aux) {
            *cand = b[i].candidate;
            *age = b[i].age_seconds;
            if (d_aux) std::memcpy(aux, b[i].aux.data(), sizeof(float) * static_cast<size_t>(d_aux));
        },
        d_aux, stage, bytes);
}

BatchSoA pack_segments(const std::vector<Segment>& b, void*& stage, size_t& bytes) {
    return BatchSoA(
        b.size(), [&](size_t i) -> const Segment& { return b[i]; },
        [](size_t, uint64_t* cand, double* age, float*) {
            *cand = 0;
            *age = 0.0;
        },
        0, stage, bytes);
}

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

// Aux and AuxLt read the examples' aux features (finetune.cpp:173, 195-201, 468-479)
bool uses_aux(const FinetuneConfig& cfg) {
    return cfg.variant == FusionVariant::Aux || cfg.variant == FusionVariant::AuxLt;
}

}  // namespace

// ---------------------------------------------------------------- DeviceKVCache
DeviceKVCache::~DeviceKVCache() {
    if (kv_) dcat_kv_destroy(kv_);
}
DeviceKVCache::DeviceKVCache(DeviceKVCache&& o) noexcept { *this = std::move(o); }
DeviceKVCache& DeviceKVCache::operator=(DeviceKVCache&& o) noexcept {
    if (this != &o) {
        if (kv_) dcat_kv_destroy(kv_);
        kv_ = o.kv_;
        o.kv_ = nullptr;
        owner_ = o.owner_;
        keep_ = std::move(o.keep_);
        fp32_ = o.fp32_;
        n_layers_ = o.n_layers_;
        d_model_ = o.d_model_;
        window_ = o.window_;
        n_ = std::move(o.n_);
    }
    return *this;
}

KVCache DeviceKVCache::to_host() const {
    KVCache c;
    c.n_layers = n_layers_;
    c.d_model = d_model_;
    c.seqs.resize(n_.size());
    for (size_t u = 0; u < n_.size(); u++) {
        SeqKV& s = c.seqs[u];
        s.n = n_[u];
        s.k.assign(static_cast<size_t>(n_layers_), Mat(n_[u], d_model_));
        s.v.assign(static_cast<size_t>(n_layers_), Mat(n_[u], d_model_));
        for (int l = 0; l < n_layers_; l++)
            check(dcat_kv_read(kv_, l, static_cast<int32_t>(u), s.k[static_cast<size_t>(l)].a.data(),
                               s.v[static_cast<size_t>(l)].a.data()));
    }
    return c;
}

// ---------------------------------------------------------------- Scorer
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

namespace {
// The reference objects as the C ABI's weight description (pointers into p / rp).
struct CWeights {
    std::vector<const float*> tensors;
    dcat_params prm{};
    dcat_head head{};
    dcat_model_config cfg{};
    CWeights(const TransformerParams& p, const RankingHeadParams& rp) {
        for (const Param* q : p.all_params()) tensors.push_back(q->v.a.data());
        prm = dcat_params{tensors.data(), static_cast<int32_t>(tensors.size())};
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
        cfg = to_c(p.cfg);
    }
};

void to_outputs(const std::vector<float>& logits, const std::vector<float>& mlog, std::vector<RankingOutputs>& out) {
    const size_t B = out.size();
    auto rows = [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; i++)
            for (int j = 0; j < kRankHeadCount; j++) {
                double l = logits[i * 3 + j];  // outputs_from, finetune.cpp:350-359
                out[i].logit[static_cast<size_t>(j)] = l;
                out[i].prob[static_cast<size_t>(j)] = 1.0 / (1.0 + std::exp(-l));
                out[i].module_logit[static_cast<size_t>(j)] = mlog[i * 3 + j];
            }
    };
    const unsigned T = static_cast<unsigned>(std::min<size_t>(host_pool().size(), std::max<size_t>(1, B / 8192)));
    if (T <= 1) {
        rows(0, B);
        return;
    }
    host_pool().run(T, [&](unsigned t) { rows(B * t / T, B * (t + 1) / T); });
}
}  // namespace

void Scorer::init(const TransformerParams& p, const dcat_table& tab, const RankingHeadParams& rp, int device) {
    CWeights w(p, rp);
    check(dcat_model_create(&w.cfg, &w.prm, &tab, &w.head, device, &m_));
    d_model_ = p.cfg.d_model;
    d_emb_ = p.cfg.d_emb;
    n_layers_ = p.cfg.n_layers;
}

Scorer::~Scorer() {
    if (m_) dcat_model_destroy(m_);
    if (stage_) dcat_host_free(stage_);
}

std::vector<RankingOutputs> Scorer::rank_forward_batch(const std::vector<RankingExample>& batch,
                                                       const FinetuneConfig& cfg) const {
    // SEQFM_B200_TIMING=1: host wall time of pack / device call / outputs on stderr (investigation aid)
    static const bool timing = std::getenv("SEQFM_B200_TIMING") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    std::vector<RankingOutputs> out(batch.size());
    if (batch.empty()) return out;
    std::lock_guard<std::mutex> lk(mu_);
    BatchSoA b = pack_examples(batch, uses_aux(cfg), stage_, stage_bytes_);
    const auto t1 = clk::now();
    dcat_finetune_config fc = to_c(cfg);
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    check(dcat_rank_forward_batch(m_, &b.c, &fc, logits.data(), mlog.data(), nullptr, flags_, nullptr));
    const auto t2 = clk::now();
    to_outputs(logits, mlog, out);
    if (timing) {
        auto ms = [](clk::time_point a, clk::time_point z) { return std::chrono::duration<double, std::milli>(z - a).count(); };
        std::fprintf(stderr, "seqfm::b200 rank_forward_batch: alloc+pack %.3f ms (%lld distinct spans of %zu rows), "
                     "device call %.3f ms, outputs %.3f ms\n", ms(t0, t1), static_cast<long long>(b.c.n_events),
                     batch.size(), ms(t1, t2), ms(t2, clk::now()));
    }
    return out;
}

// ---------------------------------------------------------------- MultiScorer
namespace {
void mcheck(int rc) {
    if (rc != DCAT_OK) throw std::runtime_error(dcat_multi_last_error());
}
}  // namespace

MultiScorer::MultiScorer(const TransformerParams& p, const HashedEmbeddingTable& table, const RankingHeadParams& rp,
                         const std::vector<int>& devices) {
    SEQFM_CHECK(!devices.empty(), "MultiScorer: no devices");
    std::vector<const float*> subs;
    for (int j = 0; j < table.num_subtables(); j++) subs.push_back(table.subtable(j).a.data());
    dcat_table tab{table.num_subtables(), table.rows(), table.d_sub(), table.seeds().data(), subs.data(), 0, nullptr};
    CWeights w(p, rp);
    std::vector<int32_t> dev(devices.begin(), devices.end());
    mcheck(dcat_multi_create(&w.cfg, &w.prm, &tab, &w.head, dev.data(), static_cast<int32_t>(dev.size()), &mh_));
}

MultiScorer::~MultiScorer() {
    if (mh_) dcat_multi_destroy(mh_);
    if (stage_) dcat_host_free(stage_);
}

std::vector<RankingOutputs> MultiScorer::rank_forward_batch(const std::vector<RankingExample>& batch,
                                                            const FinetuneConfig& cfg) const {
    std::vector<RankingOutputs> out(batch.size());
    if (batch.empty()) return out;
    std::lock_guard<std::mutex> lk(mu_);
    BatchSoA b = pack_examples(batch, uses_aux(cfg), stage_, stage_bytes_);
    dcat_finetune_config fc = to_c(cfg);
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    mcheck(dcat_multi_rank_forward_batch(mh_, &b.c, &fc, logits.data(), mlog.data(), flags_));
    to_outputs(logits, mlog, out);
    return out;
}

std::vector<int> MultiScorer::shard(const std::vector<RankingExample>& batch) const {
    std::vector<int> owner(batch.size());
    if (batch.empty()) return owner;
    std::lock_guard<std::mutex> lk(mu_);
    BatchSoA b = pack_examples(batch, false, stage_, stage_bytes_);
    std::vector<int32_t> o(batch.size());
    mcheck(dcat_multi_shard(mh_, &b.c, o.data()));
    owner.assign(o.begin(), o.end());
    return owner;
}

Mat Scorer::candidate_outputs(const std::vector<RankingExample>& batch, const FinetuneConfig& cfg) const {
    Mat h(static_cast<int>(batch.size()), d_model_);
    if (batch.empty()) return h;
    std::lock_guard<std::mutex> lk(mu_);
    BatchSoA b = pack_examples(batch, uses_aux(cfg), stage_, stage_bytes_);
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
    std::lock_guard<std::mutex> lk(mu_);
    BatchSoA b = pack_examples(batch, uses_aux(cfg), stage_, stage_bytes_);
    dcat_finetune_config fc = to_c(cfg);
    fc.window = window;
    std::vector<float> logits(batch.size() * 3), mlog(batch.size() * 3);
    check(dcat_rank_forward_batch(m_, &b.c, &fc, logits.data(), mlog.data(), h.a.data(), flags_, nullptr));
    return h;
}

DedupPlan Scorer::dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques) const {
    DedupPlan plan;
    plan.b = static_cast<int>(batch.size());
    plan.rep.resize(batch.size());
    plan.first.resize(batch.size());
    int32_t b_u = 0;
    if (!batch.empty()) {
        std::lock_guard<std::mutex> lk(mu_);
        BatchSoA b = pack_segments(batch, stage_, stage_bytes_);
        check(dcat_dedup(m_, &b.c, plan.rep.data(), plan.first.data(), &b_u, 0, nullptr));
    }
    plan.b_u = b_u;
    plan.first.resize(static_cast<size_t>(b_u));
    if (uniques) {
        uniques->clear();
        for (int u = 0; u < b_u; u++) uniques->push_back(batch[static_cast<size_t>(plan.first[static_cast<size_t>(u)])]);
    }
    return plan;
}

// ---------------------------------------------------------------- the DCAT sub-API
DeviceKVCache Scorer::context_impl(const std::vector<Segment>& uniques, int window, bool emit_hidden,
                                   std::vector<Mat>* h_user, const char* fn) const {
    SEQFM_CHECK(!h_user || emit_hidden, fn << ": h_user requires emit_hidden");
    DeviceKVCache out;
    std::vector<float> hbuf;
    {
        std::lock_guard<std::mutex> lk(mu_);
        BatchSoA b = pack_segments(uniques, stage_, stage_bytes_);
        if (h_user) {
            size_t tokens = 0;
            for (const Segment& s : uniques)
                tokens += static_cast<size_t>(window > 0 ? std::min(s.valid, window - 1) : s.valid);
            hbuf.resize(std::max<size_t>(tokens, 1) * static_cast<size_t>(d_model_));
        }
        check(dcat_context_forward(m_, &b.c, window, emit_hidden ? 1 : 0, h_user ? hbuf.data() : nullptr, flags_,
                                   nullptr, &out.kv_));
    }
    out.owner_ = this;
    out.fp32_ = flags_ != 0;
    out.window_ = window;
    int32_t nu = 0, nl = 0, d = 0;
    check(dcat_kv_info(out.kv_, &nu, &nl, &d, nullptr));
    out.n_layers_ = nl;
    out.d_model_ = d;
    out.n_.assign(static_cast<size_t>(nu), 0);
    if (nu) check(dcat_kv_info(out.kv_, nullptr, nullptr, nullptr, out.n_.data()));
    if (h_user) {  // per unique, its n_u x d rows (the ABI packs them back to back)
        h_user->assign(uniques.size(), Mat());
        size_t at = 0;
        for (size_t u = 0; u < uniques.size(); u++) {
            Mat& m = (*h_user)[u];
            m = Mat(out.n_[u], d_model_);
            std::memcpy(m.a.data(), hbuf.data() + at, sizeof(float) * m.a.size());
            at += m.a.size();
        }
    }
    return out;
}

DeviceKVCache Scorer::context_forward(const std::vector<Segment>& uniques, bool emit_hidden,
                                      std::vector<Mat>* h_user) const {
    return context_impl(uniques, 0, emit_hidden, h_user, "context_forward");
}

DeviceKVCache Scorer::context_forward_fixed(const std::vector<Segment>& uniques, int window, int rotation,
                                            bool emit_hidden, std::vector<Mat>* h_user) const {
    // the device keeps the newest window - 1 tokens contiguously (positions from 0): the ring's
    // rotation is a storage choice the results do not depend on (test_dcat.cpp:341-361)
    SEQFM_CHECK(window >= 1, "context_forward_fixed: window must be >= 1, got " << window);
    SEQFM_CHECK(rotation >= 0, "context_forward_fixed: rotation must be >= 0");
    return context_impl(uniques, window, emit_hidden, h_user, "context_forward_fixed");
}

Mat Scorer::candidate_inputs(const std::vector<u64>& items, const std::vector<int>& pos_index) const {
    SEQFM_CHECK(items.size() == pos_index.size(), "candidate_inputs: size mismatch");
    Mat e(static_cast<int>(items.size()), d_emb_);
    if (items.empty()) return e;
    std::vector<int32_t> pos(pos_index.begin(), pos_index.end());
    std::lock_guard<std::mutex> lk(mu_);
    check(dcat_candidate_inputs(m_, items.data(), pos.data(), static_cast<int64_t>(items.size()), e.a.data(), 0,
                                nullptr));
    return e;
}

Mat Scorer::cross_forward(const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand) const {
    const char* fn = cache.window_ > 0 ? "cross_forward_fixed" : "cross_forward";
    // cross_forward's checks (dcat.cpp:202-208, 341-347)
    SEQFM_CHECK(cache.kv_ && cache.owner_ == this && cache.n_layers_ == n_layers_ && cache.d_model_ == d_model_,
                fn << ": cache/model config mismatch");
    SEQFM_CHECK(cache.n_uniques() == plan.b_u, fn << ": cache has " << cache.n_uniques() << " uniques, plan " << plan.b_u);
    SEQFM_CHECK(e_cand.rows == plan.b, fn << ": " << e_cand.rows << " candidate rows for " << plan.b << " batch rows");
    SEQFM_CHECK(e_cand.cols == d_emb_, fn << ": candidate dim mismatch");
    SEQFM_CHECK(static_cast<int>(plan.rep.size()) == plan.b, fn << ": plan rep size mismatch");
    Mat h(plan.b, d_model_);
    if (plan.b == 0) return h;
    std::vector<int32_t> rep(plan.rep.begin(), plan.rep.end());
    std::lock_guard<std::mutex> lk(mu_);
    check(dcat_cross_forward(m_, cache.kv_, rep.data(), e_cand.a.data(), plan.b, h.a.data(), cache.fp32_ ? 0x2 : 0,
                             nullptr));
    return h;
}

Mat Scorer::cross_forward_fixed(const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand) const {
    SEQFM_CHECK(cache.window_ >= 1, "cross_forward_fixed: the cache is not a fixed-window cache");
    return cross_forward(cache, plan, e_cand);
}

// ---------------------------------------------------------------- free functions
namespace {
std::mutex g_mu;
// key: object addresses + weight fingerprint (guards against a freed object's address being
// reused for different weights)
using Key = std::tuple<const void*, const void*, const void*, uint64_t>;
std::map<Key, std::shared_ptr<Scorer>> g_cache;

uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; i++) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
uint64_t fingerprint_mat(uint64_t h, const Mat& m) {
    h = fnv(h, &m.rows, sizeof m.rows);
    h = fnv(h, &m.cols, sizeof m.cols);
    const size_t n = m.a.size(), step = std::max<size_t>(1, n / 64);
    for (size_t i = 0; i < n; i += step) h = fnv(h, &m.a[i], sizeof(float));
    if (n) h = fnv(h, &m.a[n - 1], sizeof(float));
    return h;
}
uint64_t fingerprint(const TransformerParams& p, const IdEmbSource& ids, const RankingHeadParams* rp) {
    uint64_t h = 1469598103934665603ull;
    for (const Param* q : p.all_params()) h = fingerprint_mat(h, q->v);
    if (const auto* t = dynamic_cast<const HashedEmbeddingTable*>(&ids)) {
        for (int j = 0; j < t->num_subtables(); j++) h = fingerprint_mat(h, t->subtable(j));
        h = fnv(h, t->seeds().data(), t->seeds().size() * sizeof(t->seeds()[0]));
    } else if (const auto* q = dynamic_cast<const QuantizedTable*>(&ids)) {
        const int bits = q->bits();
        h = fnv(h, &bits, sizeof bits);
        const size_t total = static_cast<size_t>(q->num_subtables()) * q->rows() * q->packed_row_bytes();
        const size_t step = std::max<size_t>(1, total / 256);
        const uint8_t* pk = q->packed_row(0, 0);
        for (size_t i = 0; i < total; i += step) h = fnv(h, pk + i, 1);
        h = fnv(h, q->seeds().data(), q->seeds().size() * sizeof(q->seeds()[0]));
    }
    if (rp)
        for (const Mat* m : {&rp->w1.v, &rp->b1.v, &rp->w2.v, &rp->b2.v, &rp->mod_w.v, &rp->mod_b.v, &rp->aux_proj.v,
                             &rp->lt.v})
            h = fingerprint_mat(h, *m);
    return h;
}

std::shared_ptr<Scorer> make_scorer(const TransformerParams& p, const IdEmbSource& ids, const RankingHeadParams& rp) {
    const auto* table = dynamic_cast<const HashedEmbeddingTable*>(&ids);
    const auto* qtable = dynamic_cast<const QuantizedTable*>(&ids);
    SEQFM_CHECK(table != nullptr || qtable != nullptr,
                "B200 scorer needs a HashedEmbeddingTable or QuantizedTable id source");
    return table ? std::make_shared<Scorer>(p, *table, rp) : std::make_shared<Scorer>(p, *qtable, rp);
}

std::shared_ptr<Scorer> cached(const TransformerParams& p, const IdEmbSource& ids, const RankingHeadParams& rp) {
    const Key key{&p, &ids, &rp, fingerprint(p, ids, &rp)};
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) it = g_cache.emplace(key, make_scorer(p, ids, rp)).first;
    return it->second;
}

// the sub-API has no ranking head: a minimal head (hidden 8, no aux) satisfies model creation
std::shared_ptr<Scorer> cached_model(const TransformerParams& p, const IdEmbSource& ids) {
    const Key key{&p, &ids, nullptr, fingerprint(p, ids, nullptr)};
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
        RankingHeadParams rp;
        rp.init(p.cfg.d_model, p.cfg.d_emb, 0, 8, 8, 1, 0);
        it = g_cache.emplace(key, make_scorer(p, ids, rp)).first;
    }
    return it->second;
}
}  // namespace

std::vector<RankingOutputs> rank_forward_batch(const TransformerParams& p, const IdEmbSource& ids,
                                               const RankingHeadParams& rp,
                                               const std::vector<RankingExample>& batch,
                                               const FinetuneConfig& cfg) {
    std::shared_ptr<Scorer> s = cached(p, ids, rp);  // stays alive across a concurrent invalidate()
    return s->rank_forward_batch(batch, cfg);
}

DedupPlan dedup_segments(const std::vector<Segment>& batch, std::vector<Segment>* uniques) {
    // the plan needs no weights: a 1-layer stub model carries the enum / position limits
    static std::mutex mu;
    static std::unique_ptr<Scorer> s;
    {
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
    }
    return s->dedup_segments(batch, uniques);
}

DeviceKVCache context_forward(const TransformerParams& p, const IdEmbSource& ids, const std::vector<Segment>& uniques,
                              bool emit_hidden, std::vector<Mat>* h_user, int /*n_threads*/) {
    std::shared_ptr<Scorer> s = cached_model(p, ids);
    DeviceKVCache c = s->context_forward(uniques, emit_hidden, h_user);
    c.keep_ = s;
    return c;
}

Mat candidate_inputs(const TransformerParams& p, const IdEmbSource& ids, const std::vector<u64>& items,
                     const std::vector<int>& pos_index) {
    SEQFM_CHECK(ids.emb_dim() == p.cfg.d_emb, "candidate_inputs: embedding dim mismatch");
    return cached_model(p, ids)->candidate_inputs(items, pos_index);
}

Mat cross_forward(const TransformerParams& p, const DeviceKVCache& cache, const DedupPlan& plan, const Mat& e_cand,
                  int /*n_threads*/) {
    SEQFM_CHECK(cache.owner_ != nullptr && cache.n_layers_ == p.cfg.n_layers && cache.d_model_ == p.cfg.d_model,
                "cross_forward: cache/model config mismatch");
    return cache.owner_->cross_forward(cache, plan, e_cand);
}

DeviceKVCache context_forward_fixed(const TransformerParams& p, const IdEmbSource& ids,
                                    const std::vector<Segment>& uniques, int window, int rotation, bool emit_hidden,
                                    std::vector<Mat>* h_user, int /*n_threads*/) {
    std::shared_ptr<Scorer> s = cached_model(p, ids);
    DeviceKVCache c = s->context_forward_fixed(uniques, window, rotation, emit_hidden, h_user);
    c.keep_ = s;
    return c;
}

Mat cross_forward_fixed(const TransformerParams& p, const DeviceKVCache& cache, const DedupPlan& plan,
                        const Mat& e_cand, int /*n_threads*/) {
    SEQFM_CHECK(cache.owner_ != nullptr && cache.n_layers_ == p.cfg.n_layers && cache.d_model_ == p.cfg.d_model,
                "cross_forward_fixed: cache/model config mismatch");
    return cache.owner_->cross_forward_fixed(cache, plan, e_cand);
}

void invalidate() {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache.clear();
}

}  // namespace b200
}  // namespace seqfm
