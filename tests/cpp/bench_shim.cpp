// bench_shim.cpp — end-to-end throughput of the drop-in C++ API on the BASELINE workload:
// std::vector<RankingExample> in (every example owns its Segment, as the reference's batches do),
// std::vector<RankingOutputs> out, through seqfm::b200::Scorer::rank_forward_batch. The timed
// region is the whole call: packing into pinned staging, H2D, the device pass, D2H and the
// RankingOutputs (double prob). Weights are the reference's own seeded init; events follow the
// run_bench recipe (dcat.cpp:493-521). Prints one JSON line. Run by bench.py on the GPU box.
//
//   bench_shim <users> <cands> <L> <layers> <d_model> <heads> <steps> <warmup>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "seqfm/dcat.hpp"
#include "seqfm/finetune.hpp"
#include "../../paper_2507_12704_b200/shim/seqfm_b200.hpp"

using namespace seqfm;

int main(int argc, char** argv) {
    const int U = argc > 1 ? std::atoi(argv[1]) : 1000, C = argc > 2 ? std::atoi(argv[2]) : 128,
              L = argc > 3 ? std::atoi(argv[3]) : 256, layers = argc > 4 ? std::atoi(argv[4]) : 4,
              d = argc > 5 ? std::atoi(argv[5]) : 256, heads = argc > 6 ? std::atoi(argv[6]) : 8,
              steps = argc > 7 ? std::atoi(argv[7]) : 5, warmup = argc > 8 ? std::atoi(argv[8]) : 2;
    ModelConfig mc;
    mc.d_model = d;
    mc.n_layers = layers;
    mc.n_heads = heads;
    mc.max_len = L + 2;
    mc.d_emb = d;
    TransformerParams p;
    p.init(mc, 42);
    HashedEmbeddingTable table(8, 4096, d / 8, 7);
    FinetuneConfig cfg;
    cfg.max_events = L;
    RankingHeadParams rp;
    rp.init(d, d, cfg.d_aux, cfg.n_ctx(), cfg.crossing_hidden, cfg.sel_per_example(), 11);
    // run_bench's events (dcat.cpp:493-521): one Segment per unique user, every example a copy
    Rng rng(mix64(1 ^ 0x62656e6368ULL));
    std::vector<Segment> uniq(static_cast<size_t>(U));
    for (int u = 0; u < U; u++) {
        Segment& s = uniq[static_cast<size_t>(u)];
        s.user_id = static_cast<u64>(u);
        s.valid = L;
        s.events.resize(static_cast<size_t>(L));
        for (int i = 0; i < L; i++) {
            Event& e = s.events[static_cast<size_t>(i)];
            e.timestamp = 1700000000ULL + static_cast<u64>(u) * 100000ULL + static_cast<u64>(i);
            e.action = static_cast<Action>(rng.uniform_u64(kActionCount));
            e.surface = static_cast<Surface>(rng.uniform_u64(kSurfaceCount));
            e.item_id = rng.uniform_u64(1000000);
        }
    }
    std::vector<RankingExample> batch(static_cast<size_t>(U) * C);
    for (size_t b = 0; b < batch.size(); b++) {
        RankingExample& ex = batch[b];
        ex.seq = uniq[b % static_cast<size_t>(U)];  // interleaved rows, like run_bench
        ex.candidate = rng.uniform_u64(1000000);
        ex.age_seconds = rng.uniform(0.0, 60 * 86400.0);
    }
    b200::Scorer sc(p, table, rp);
    for (int i = 0; i < warmup; i++) sc.rank_forward_batch(batch, cfg);
    std::vector<double> ms;
    double checksum = 0;
    for (int i = 0; i < steps; i++) {
        auto t0 = std::chrono::steady_clock::now();
        auto out = sc.rank_forward_batch(batch, cfg);
        auto t1 = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        checksum += out[0].prob[0];
    }
    std::sort(ms.begin(), ms.end());
    const double med = ms[ms.size() / 2];
    size_t events = 0;
    for (const auto& ex : batch) events += static_cast<size_t>(ex.seq.valid);
    // the shim stages one span per distinct sequence (U of them here) plus the per-row fields
    const size_t staged_events = static_cast<size_t>(U) * static_cast<size_t>(L);
    std::printf(
        "{\"value\": %.1f, \"unit\": \"candidates/s\", \"ms_per_step\": %.3f, \"ms_min\": %.3f, \"steps\": %d, "
        "\"rows\": %zu, \"events\": %zu, \"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, "
        "\"api\": \"seqfm::b200::Scorer::rank_forward_batch(std::vector<RankingExample>) -> "
        "std::vector<RankingOutputs>, a private Segment per example; the shim groups equal sequences "
        "(verified event by event) and stages one span per distinct sequence; host wall clock incl. "
        "packing\", "
        "\"checksum\": %.6f}\n",
        static_cast<double>(batch.size()) / (med / 1e3), med, ms[0], steps, batch.size(), events,
        staged_events * 18 + batch.size() * (8 + 4 + 8 + 8), batch.size() * 2 * 3 * 4, checksum);
    return 0;
}
