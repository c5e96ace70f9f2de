// test_shim.cpp — the drop-in shim against the UNMODIFIED reference, in one binary.
//
// Links the reference library (oracle/_ref/libseqfm_ref.so, built from
// /root/reference/proj/src) and the B200 shim (seqfm::b200, over
// libdcat_b200.so). Mirrors the reference's own parity tests:
//   test_finetune.cpp:327-364  rank_forward_batch vs the single scorer (rel 1e-4)
//   test_dcat.cpp:84-137       dedup plans exact
//   test_dcat.cpp:215-229      DCAT rows vs naive (1e-4)
// Exit code 0 = all checks pass. Run by tests/test_gpu_shim.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "seqfm/dcat.hpp"
#include "seqfm/finetune.hpp"
#include "../../paper_2507_12704_b200/shim/seqfm_b200.hpp"

using namespace seqfm;

static int failures = 0;
#define EXPECT(c, ...)                                  \
    do {                                                \
        if (!(c)) {                                     \
            failures++;                                 \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                   \
            std::printf("\n");                          \
        }                                               \
    } while (0)

static Segment random_segment(u64 user, int valid, int L, Rng& rng) {
    Segment s;
    s.user_id = user;
    s.valid = valid;
    s.events.resize(static_cast<size_t>(L));
    u64 ts = 10000 + rng.uniform_u64(100);
    for (int i = 0; i < valid; i++) {
        ts += 1 + rng.uniform_u64(20);
        Event& e = s.events[static_cast<size_t>(i)];
        e.timestamp = ts;
        e.action = static_cast<Action>(rng.uniform_u64(kActionCount));
        e.surface = static_cast<Surface>(rng.uniform_u64(kSurfaceCount));
        e.item_id = rng.next_u64() % 100000;
    }
    return s;
}

static std::vector<RankingExample> make_batch(int users, int cands, int L, int d_aux, Rng& rng, bool with_empty) {
    std::vector<Segment> uniq;
    for (int u = 0; u < users; u++) {
        int v = with_empty && u == 0 ? 0 : 1 + static_cast<int>(rng.uniform_u64(static_cast<u64>(L)));
        uniq.push_back(random_segment(static_cast<u64>(u), v, L, rng));
    }
    std::vector<RankingExample> b;
    for (int i = 0; i < users * cands; i++) {
        RankingExample ex;
        ex.seq = uniq[static_cast<size_t>(i % users)];
        ex.seq.user_id = static_cast<u64>(i);
        ex.candidate = rng.next_u64() % 100000;
        ex.age_seconds = rng.uniform(0.0, 60 * 86400.0);
        for (int k = 0; k < d_aux; k++) ex.aux.push_back(static_cast<float>(rng.normal()));
        b.push_back(ex);
    }
    return b;
}

static double rel(double a, double b, double scale) { return std::fabs(a - b) / std::max(1e-3, scale); }

static void check_rank(const char* name, const ModelConfig& mc, int L, int users, int cands, FusionVariant v,
                       bool with_empty) {
    TransformerParams p;
    p.init(mc, 51, 0.3f);
    HashedEmbeddingTable table(4, 64, mc.d_emb / 4, 52);
    FinetuneConfig cfg;
    cfg.variant = v;
    cfg.max_events = L;
    cfg.crossing_hidden = 8;
    cfg.d_aux = 4;
    cfg.validate(mc);
    RankingHeadParams rp;
    rp.init(mc.d_model, mc.d_emb, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, cfg.sel_per_example(), 53);
    Rng ar(5);
    for (auto& x : rp.aux_proj.v.a) x = 0.3f * static_cast<float>(ar.normal());
    Rng rng(77);
    auto batch = make_batch(users, cands, L, v == FusionVariant::Aux || v == FusionVariant::AuxLt ? 4 : 0, rng, with_empty);
    auto ref = seqfm::rank_forward_batch(p, table, rp, batch, cfg);
    b200::Scorer sc(p, table, rp);
    for (int fp32 = 1; fp32 >= 0; fp32--) {
        sc.set_fp32(fp32 != 0);
        auto got = sc.rank_forward_batch(batch, cfg);
        double scale = 0, scale_m = 0, err = 0, err_m = 0;
        for (auto& r : ref)
            for (int h = 0; h < 3; h++) {
                scale = std::max(scale, std::fabs(r.logit[h]));
                scale_m = std::max(scale_m, std::fabs(r.module_logit[h]));
            }
        for (size_t i = 0; i < ref.size(); i++)
            for (int h = 0; h < 3; h++) {
                err = std::max(err, rel(got[i].logit[h], ref[i].logit[h], scale));
                err_m = std::max(err_m, rel(got[i].module_logit[h], ref[i].module_logit[h], scale_m));
                EXPECT(std::fabs(got[i].prob[h] - 1.0 / (1.0 + std::exp(-got[i].logit[h]))) < 1e-12, "prob");
            }
        double tol = fp32 ? 1e-4 : 3e-2;  // test_finetune.cpp:359-361 / bf16 storage
        std::printf("%-28s %s  max rel err logits %.3e  module %.3e  (tol %.0e)\n", name, fp32 ? "fp32" : "bf16", err,
                    err_m, tol);
        EXPECT(err <= tol && err_m <= tol, "%s rank_forward_batch parity", name);
    }
}

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);  // progress survives an abort
    // 1. rank_forward_batch parity (test_finetune.cpp:327-364 analogue)
    ModelConfig tiny;
    tiny.d_model = 16;
    tiny.n_layers = 1;
    tiny.n_heads = 2;
    tiny.mlp_ratio = 2;
    tiny.max_len = 8;
    tiny.d_emb = 8;
    check_rank("tiny base", tiny, 4, 5, 3, FusionVariant::Base, false);
    check_rank("tiny aux", tiny, 4, 5, 3, FusionVariant::Aux, false);
    check_rank("tiny aux-lt", tiny, 4, 5, 3, FusionVariant::AuxLt, false);
    check_rank("tiny base + empty seq", tiny, 4, 5, 3, FusionVariant::Base, true);
    ModelConfig base;
    base.d_model = 256;
    base.n_layers = 4;
    base.n_heads = 8;
    base.max_len = 66;
    base.d_emb = 256;
    check_rank("PinFM-base dims, L=64", base, 64, 3, 40, FusionVariant::Base, false);

    // 2. dedup plans (test_dcat.cpp:84-137)
    Rng rng(3);
    std::vector<Segment> segs;
    for (int i = 0; i < 50; i++) segs.push_back(random_segment(static_cast<u64>(i), static_cast<int>(rng.uniform_u64(9)), 8, rng));
    for (int i = 0; i < 200; i++) {
        Segment s = segs[static_cast<size_t>(rng.uniform_u64(50))];
        s.user_id = 1000 + static_cast<u64>(i);
        if (s.valid < 8) s.events[static_cast<size_t>(s.valid)].item_id = 999999;  // padding is ignored
        segs.push_back(s);
    }
    std::vector<Segment> ur, ub;
    DedupPlan pr = seqfm::dedup_segments(segs, &ur);
    DedupPlan pb = b200::dedup_segments(segs, &ub);
    EXPECT(pr.b_u == pb.b_u && pr.rep == pb.rep && pr.first == pb.first, "dedup plan differs");
    std::printf("dedup: b=%d b_u=%d (reference %d) %s\n", pb.b, pb.b_u, pr.b_u, pr.rep == pb.rep ? "exact" : "DIFF");

    // 3. DCAT candidate rows vs the reference naive forward (test_dcat.cpp:215-229)
    for (int layers : {1, 2})
        for (int heads : {1, 4}) {
            ModelConfig c;
            c.d_model = 16;
            c.n_layers = layers;
            c.n_heads = heads;
            c.d_emb = 16;
            c.max_len = 16;
            TransformerParams p;
            p.init(c, static_cast<u64>(100 + layers * 10 + heads));
            HashedEmbeddingTable table(4, 64, 4, 21);
            RankingHeadParams rp;
            rp.init(16, 16, 16, 8, 64, 1, 11);
            Rng r2(7);
            auto batch = make_batch(4, 4, 10, 0, r2, false);
            std::vector<Segment> bs;
            std::vector<u64> items;
            for (auto& ex : batch) {
                bs.push_back(ex.seq);
                items.push_back(ex.candidate);
            }
            Mat naive = naive_candidate_outputs(p, table, bs, items);
            b200::Scorer sc(p, table, rp);
            sc.set_fp32(true);
            FinetuneConfig cfg;
            cfg.max_events = 10;
            Mat h = sc.candidate_outputs(batch, cfg);
            double m = 0;
            for (size_t i = 0; i < h.a.size(); i++) m = std::max(m, static_cast<double>(std::fabs(h.a[i] - naive.a[i])));
            std::printf("cross vs naive l%d h%d: max abs %.3e\n", layers, heads, m);
            EXPECT(m <= 1e-4, "cross vs naive");
        }

    // 3b. fixed-window variant against the reference ring (dcat.cpp:281-415) at a non-zero rotation
    for (int window : {1, 4, 8, 64}) {
        ModelConfig c;
        c.d_model = 16;
        c.n_layers = 2;
        c.n_heads = 4;
        c.d_emb = 16;
        c.max_len = 16;
        TransformerParams p;
        p.init(c, 101);
        HashedEmbeddingTable table(4, 64, 4, 15);
        RankingHeadParams rp;
        rp.init(16, 16, 16, 8, 64, 1, 11);
        Rng r2(12);
        auto batch = make_batch(4, 3, 12, 0, r2, false);
        std::vector<Segment> segs, uniques;
        std::vector<u64> items;
        for (auto& ex : batch) {
            segs.push_back(ex.seq);
            items.push_back(ex.candidate);
        }
        DedupPlan plan = dedup_segments(segs, &uniques);
        FixedKVCache cache = context_forward_fixed(p, table, uniques, window, 3);
        std::vector<int> pos;
        for (int i = 0; i < plan.b; i++) pos.push_back(cache.seqs[static_cast<size_t>(plan.rep[static_cast<size_t>(i)])].kept);
        Mat ref = cross_forward_fixed(p, cache, plan, candidate_inputs(p, table, items, pos));
        b200::Scorer sc(p, table, rp);
        sc.set_fp32(true);
        FinetuneConfig cfg;
        cfg.max_events = 12;
        Mat h = sc.candidate_outputs_fixed(batch, cfg, window);
        double m = 0;
        for (size_t i = 0; i < h.a.size(); i++) m = std::max(m, static_cast<double>(std::fabs(h.a[i] - ref.a[i])));
        std::printf("fixed window %d vs reference ring (rotation 3): max abs %.3e\n", window, m);
        EXPECT(m <= 1e-4, "fixed window vs cross_forward_fixed");
    }

    // 3c. QuantizedTable id source (int4 / int8): the free function with ids = quantize(table)
    for (int bits : {4, 8}) {
        ModelConfig c;
        c.d_model = 16;
        c.n_layers = 2;
        c.n_heads = 4;
        c.d_emb = 16;
        c.max_len = 16;
        TransformerParams p;
        p.init(c, 141);
        HashedEmbeddingTable table(4, 64, 4, 23);
        QuantizedTable qt = quantize(table, bits);
        RankingHeadParams rp;
        FinetuneConfig cfg;
        cfg.max_events = 12;
        rp.init(16, 16, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, 1, 11);
        Rng r4(19);
        auto batch = make_batch(4, 3, 12, 0, r4, false);
        auto ref = rank_forward_batch(p, qt, rp, batch, cfg);
        b200::Scorer sc(p, qt, rp);
        sc.set_fp32(true);
        auto got = sc.rank_forward_batch(batch, cfg);
        double m = 0;
        for (size_t i = 0; i < ref.size(); i++)
            for (int k = 0; k < kRankHeadCount; k++)
                m = std::max(m, std::fabs(got[i].logit[k] - ref[i].logit[k]) / (std::fabs(ref[i].logit[k]) + 1e-3));
        std::printf("quantized int%d table vs reference: max rel %.3e\n", bits, m);
        EXPECT(m <= 1e-4, "quantized table vs rank_forward_batch(QuantizedTable)");
        auto free_fn = b200::rank_forward_batch(p, qt, rp, batch, cfg);  // bf16 via the free function
        double mb = 0;
        for (size_t i = 0; i < ref.size(); i++)
            for (int k = 0; k < kRankHeadCount; k++) mb = std::max(mb, std::fabs(free_fn[i].logit[k] - ref[i].logit[k]));
        EXPECT(mb <= 3e-2, "quantized table via the free function");
    }

    // 3d. the DCAT sub-API with a device cache: context_forward -> candidate_inputs ->
    // cross_forward (+ the fixed pair) against the reference's own functions (dcat.hpp:47-101)
    {
        ModelConfig c;
        c.d_model = 64;
        c.n_layers = 2;
        c.n_heads = 4;
        c.d_emb = 64;
        c.max_len = 40;
        TransformerParams p;
        p.init(c, 303, 0.3f);
        HashedEmbeddingTable table(8, 256, 8, 31);
        RankingHeadParams rp;
        rp.init(64, 64, 16, 8, 64, 1, 11);
        Rng r5(41);
        auto batch = make_batch(5, 4, 30, 0, r5, true);
        std::vector<Segment> segs, uniques;
        std::vector<u64> items;
        for (auto& ex : batch) {
            segs.push_back(ex.seq);
            items.push_back(ex.candidate);
        }
        DedupPlan plan = dedup_segments(segs, &uniques);
        std::vector<Mat> h_ref;
        KVCache ref_cache = context_forward(p, table, uniques, true, &h_ref);
        std::vector<int> pos;
        for (int i = 0; i < plan.b; i++) pos.push_back(uniques[static_cast<size_t>(plan.rep[static_cast<size_t>(i)])].valid);
        Mat e_ref = candidate_inputs(p, table, items, pos);
        Mat x_ref = cross_forward(p, ref_cache, plan, e_ref);
        b200::Scorer sc(p, table, rp);
        sc.set_fp32(true);
        std::vector<Mat> h_dev;
        b200::DeviceKVCache dc = sc.context_forward(uniques, true, &h_dev);
        KVCache got = dc.to_host();
        double mk = 0, mh = 0;
        for (size_t u = 0; u < uniques.size(); u++) {
            EXPECT(got.seqs[u].n == ref_cache.seqs[u].n, "SeqKV::n");
            for (int l = 0; l < c.n_layers; l++)
                for (size_t i = 0; i < got.seqs[u].k[static_cast<size_t>(l)].a.size(); i++) {
                    mk = std::max(mk, static_cast<double>(std::fabs(got.seqs[u].k[static_cast<size_t>(l)].a[i] -
                                                                    ref_cache.seqs[u].k[static_cast<size_t>(l)].a[i])));
                    mk = std::max(mk, static_cast<double>(std::fabs(got.seqs[u].v[static_cast<size_t>(l)].a[i] -
                                                                    ref_cache.seqs[u].v[static_cast<size_t>(l)].a[i])));
                }
            for (size_t i = 0; i < h_dev[u].a.size(); i++)
                mh = std::max(mh, static_cast<double>(std::fabs(h_dev[u].a[i] - h_ref[u].a[i])));
        }
        Mat e_dev = sc.candidate_inputs(items, pos);
        double me = 0, mx = 0;
        for (size_t i = 0; i < e_dev.a.size(); i++) me = std::max(me, static_cast<double>(std::fabs(e_dev.a[i] - e_ref.a[i])));
        Mat x_dev = sc.cross_forward(dc, plan, e_ref);
        for (size_t i = 0; i < x_dev.a.size(); i++) mx = std::max(mx, static_cast<double>(std::fabs(x_dev.a[i] - x_ref.a[i])));
        std::printf("sub-API fp32: K/V max abs %.3e, h_user %.3e, candidate_inputs %.3e, cross rows %.3e\n", mk, mh, me, mx);
        EXPECT(mk <= 1e-5 && mh <= 1e-4 && me <= 1e-6 && mx <= 1e-4, "sub-API vs context_forward / cross_forward");
        // the free functions with the reference signatures (bf16, cached model)
        b200::DeviceKVCache fc = b200::context_forward(p, table, uniques, false);
        Mat xb = b200::cross_forward(p, fc, plan, b200::candidate_inputs(p, table, items, pos));
        double mb = 0;
        for (size_t i = 0; i < xb.a.size(); i++) mb = std::max(mb, static_cast<double>(std::fabs(xb.a[i] - x_ref.a[i])));
        std::printf("sub-API free functions bf16: cross rows max abs %.3e\n", mb);
        EXPECT(mb <= 2e-2, "free-function sub-API");
        for (int window : {1, 5, 16}) {
            FixedKVCache rf = context_forward_fixed(p, table, uniques, window, 2);
            std::vector<int> kpos;
            for (int i = 0; i < plan.b; i++) kpos.push_back(rf.seqs[static_cast<size_t>(plan.rep[static_cast<size_t>(i)])].kept);
            Mat ef = candidate_inputs(p, table, items, kpos);
            Mat xr = cross_forward_fixed(p, rf, plan, ef);
            b200::DeviceKVCache df = sc.context_forward_fixed(uniques, window, 2);
            Mat xd = sc.cross_forward_fixed(df, plan, ef);
            double m = 0;
            for (size_t i = 0; i < xd.a.size(); i++) m = std::max(m, static_cast<double>(std::fabs(xd.a[i] - xr.a[i])));
            std::printf("sub-API fixed window %d: cross rows max abs %.3e\n", window, m);
            EXPECT(m <= 1e-4, "cross_forward_fixed via the device cache");
        }
        bool threw = false;
        try {
            DedupPlan bad = plan;
            bad.b_u += 1;
            sc.cross_forward(dc, bad, e_ref);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("uniques, plan") != std::string::npos;
        }
        EXPECT(threw, "cross_forward plan / cache mismatch must throw");
    }

    // 3e. one Scorer shared by several threads (calls are serialised per handle) and the free
    // function's weight fingerprint (in-place weight edits are picked up without invalidate())
    {
        ModelConfig c;
        c.d_model = 32;
        c.n_layers = 1;
        c.n_heads = 2;
        c.d_emb = 32;
        c.max_len = 20;
        TransformerParams p;
        p.init(c, 71, 0.3f);
        HashedEmbeddingTable table(4, 64, 8, 9);
        RankingHeadParams rp;
        FinetuneConfig cfg;
        cfg.max_events = 16;
        rp.init(32, 32, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, 1, 13);
        Rng r6(23);
        auto batch = make_batch(6, 5, 16, 0, r6, false);
        b200::Scorer sc(p, table, rp);
        auto one = sc.rank_forward_batch(batch, cfg);
        std::vector<std::thread> th;
        std::vector<int> ok(8, 0);
        for (int t = 0; t < 8; t++)
            th.emplace_back([&, t] {
                bool same = true;
                for (int it = 0; it < 5; it++) {
                    auto got = sc.rank_forward_batch(batch, cfg);
                    for (size_t i = 0; i < got.size(); i++)
                        for (int k = 0; k < kRankHeadCount; k++) same = same && got[i].logit[k] == one[i].logit[k];
                }
                ok[static_cast<size_t>(t)] = same;
            });
        for (auto& x : th) x.join();
        int all = 0;
        for (int v : ok) all += v;
        std::printf("8 threads x 5 calls on one Scorer: %d / 8 bit-identical\n", all);
        EXPECT(all == 8, "shared Scorer under concurrency");
        auto before = b200::rank_forward_batch(p, table, rp, batch, cfg);
        for (auto& x : p.layers[0].wq.v.a) x *= 3.0f;  // in place: same object addresses
        auto after = b200::rank_forward_batch(p, table, rp, batch, cfg);
        auto ref = rank_forward_batch(p, table, rp, batch, cfg);
        double m = 0, moved = 0;
        for (size_t i = 0; i < ref.size(); i++)
            for (int k = 0; k < kRankHeadCount; k++) {
                m = std::max(m, std::fabs(after[i].logit[k] - ref[i].logit[k]));
                moved = std::max(moved, std::fabs(after[i].logit[k] - before[i].logit[k]));
            }
        std::printf("weights edited in place: new scores follow the reference (max abs %.3e, moved %.3e)\n", m, moved);
        EXPECT(m <= 3e-2 && moved > 1e-6, "fingerprinted weight cache");
    }

    // 3a'. the shim packs one span per distinct sequence: rows whose sequences agree on the events
    // its grouping key samples (first / middle / last) but differ elsewhere must stay apart
    {
        TransformerParams p;
        p.init(tiny, 71, 0.3f);
        HashedEmbeddingTable table(4, 64, tiny.d_emb / 4, 72);
        FinetuneConfig cfg;
        cfg.max_events = 6;
        cfg.crossing_hidden = 8;
        RankingHeadParams rp;
        rp.init(tiny.d_model, tiny.d_emb, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, cfg.sel_per_example(), 73);
        Rng r4(31);
        Segment a = random_segment(1, 6, 8, r4);
        std::vector<Segment> variants{a, a, a};
        variants[1].events[1].item_id ^= 12345;  // indices 1 and 4 are not sampled by the key (0, 3, 5)
        variants[2].events[4].action = static_cast<Action>((static_cast<int>(a.events[4].action) + 1) % kActionCount);
        std::vector<RankingExample> batch;
        for (int i = 0; i < 30; i++) {
            RankingExample ex;
            ex.seq = variants[static_cast<size_t>(i % 3)];
            ex.candidate = r4.next_u64() % 100000;
            ex.age_seconds = r4.uniform(0.0, 30 * 86400.0);
            batch.push_back(ex);
        }
        auto ref = seqfm::rank_forward_batch(p, table, rp, batch, cfg);
        b200::Scorer sc(p, table, rp);
        sc.set_fp32(true);
        auto got = sc.rank_forward_batch(batch, cfg);
        double scale = 0, err = 0;
        for (auto& r : ref)
            for (int h = 0; h < 3; h++) scale = std::max(scale, std::fabs(r.logit[h]));
        for (size_t i = 0; i < ref.size(); i++)
            for (int h = 0; h < 3; h++) err = std::max(err, rel(got[i].logit[h], ref[i].logit[h], scale));
        std::printf("span sharing with grouping-key collisions: max rel err %.3e\n", err);
        EXPECT(err <= 1e-4, "span sharing must keep differing sequences apart");
        std::vector<Segment> segs;
        for (auto& ex : batch) segs.push_back(ex.seq);
        DedupPlan pr = seqfm::dedup_segments(segs, nullptr), pb = sc.dedup_segments(segs, nullptr);
        EXPECT(pr.b_u == 3 && pb.b_u == 3 && pr.rep == pb.rep, "dedup of colliding keys");
    }

    // 3b. MultiScorer: the multi-GPU drop-in for score_groups (finetune.cpp:766-786) vs the
    // reference's single-process rank_forward_batch, on 1 GPU and on 2 when the box has them
    {
        ModelConfig mc;
        mc.d_model = 64;
        mc.n_layers = 2;
        mc.n_heads = 4;
        mc.max_len = 34;
        mc.d_emb = 64;
        TransformerParams p;
        p.init(mc, 61, 0.3f);
        HashedEmbeddingTable table(4, 256, mc.d_emb / 4, 62);
        FinetuneConfig cfg;
        cfg.max_events = 32;
        cfg.crossing_hidden = 8;
        cfg.validate(mc);
        RankingHeadParams rp;
        rp.init(mc.d_model, mc.d_emb, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, cfg.sel_per_example(), 63);
        Rng rng(17);
        auto batch = make_batch(24, 7, 32, 0, rng, false);
        auto ref = seqfm::rank_forward_batch(p, table, rp, batch, cfg);
        double scale = 0;
        for (auto& r : ref)
            for (int h = 0; h < 3; h++) scale = std::max(scale, std::fabs(r.logit[h]));
        const char* lim = std::getenv("TEST_SHIM_MULTI_MAX");  // bisection aid: max devices tried (0: none)
        const int max_dev = lim ? std::atoi(lim) : 2;
        for (int ndev : {1, 2}) {
            if (ndev > max_dev) break;
            std::vector<int> devs;
            for (int i = 0; i < ndev; i++) devs.push_back(i);
            std::unique_ptr<b200::MultiScorer> ms;
            try {
                ms = std::make_unique<b200::MultiScorer>(p, table, rp, devs);
            } catch (const std::runtime_error& e) {
                if (ndev > 1) {  // fewer GPUs on this box
                    std::printf("MultiScorer x%d: skipped (%s)\n", ndev, e.what());
                    continue;
                }
                EXPECT(false, "MultiScorer x1: %s", e.what());
                continue;
            }
            for (int fp32 = 1; fp32 >= 0; fp32--) {
                ms->set_fp32(fp32 != 0);
                auto got = ms->rank_forward_batch(batch, cfg);
                double err = 0;
                for (size_t i = 0; i < ref.size(); i++)
                    for (int h = 0; h < 3; h++) err = std::max(err, rel(got[i].logit[h], ref[i].logit[h], scale));
                const double tol = fp32 ? 1e-4 : 3e-2;
                std::printf("MultiScorer x%d %s: max rel err logits %.3e (tol %.0e)\n", ndev, fp32 ? "fp32" : "bf16",
                            err, tol);
                EXPECT(err <= tol, "MultiScorer x%d parity", ndev);
            }
            // user-disjoint: every example of one user sequence on one device
            auto owner = ms->shard(batch);
            bool disjoint = true;
            for (size_t i = 0; i < batch.size(); i++)
                for (size_t j = 0; j < i; j++)
                    if (batch[i].seq.events == batch[j].seq.events && batch[i].seq.valid == batch[j].seq.valid &&
                        owner[i] != owner[j])
                        disjoint = false;
            EXPECT(disjoint, "MultiScorer x%d shards are not user-disjoint", ndev);
        }
    }

    // 4. errors surface as std::runtime_error (SEQFM_CHECK)
    {
        TransformerParams p;
        p.init(tiny, 1);
        HashedEmbeddingTable table(4, 64, 2, 2);
        RankingHeadParams rp;
        FinetuneConfig cfg;
        cfg.max_events = 4;
        cfg.crossing_hidden = 8;
        rp.init(16, 8, cfg.d_aux, cfg.n_ctx(), 8, 1, 3);
        Rng r3(9);
        auto batch = make_batch(2, 2, 4, 0, r3, false);
        batch[1].seq.events[0].action = static_cast<Action>(9);
        bool threw = false;
        try {
            b200::rank_forward_batch(p, table, rp, batch, cfg);
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()).find("unknown action") != std::string::npos;
            if (!threw) std::printf("unexpected error message: %s\n", e.what());
        }
        EXPECT(threw, "unknown action must throw std::runtime_error");
    }
    std::printf(failures ? "FAILED (%d)\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
