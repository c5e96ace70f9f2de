// test_pool.cpp — the host thread pool (paper_2507_12704_b200/csrc/host_pool.hpp) under load:
// every index of every job runs exactly once, jobs submitted from several threads at once are
// serialised, back-to-back jobs of different sizes do not leak items into each other, and an empty
// pool runs jobs on the caller. Exit code 0 = pass. Built and run by tests/test_host_pool_cpu.py.
#include <atomic>
#include <cstdio>
#include <thread>
#include <vector>

#include "../../paper_2507_12704_b200/csrc/host_pool.hpp"

static int failures = 0;
#define EXPECT(c, ...)                                       \
    do {                                                     \
        if (!(c)) {                                          \
            failures++;                                      \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                        \
            std::printf("\n");                               \
        }                                                    \
    } while (0)

int main() {
    for (unsigned workers : {0u, 1u, 3u, 15u}) {
        dcat::ThreadPool pool(workers);
        // back-to-back jobs of varying size: each index exactly once
        for (unsigned n : {1u, 2u, 7u, 64u, 1000u, 3u, 0u, 5000u}) {
            std::vector<std::atomic<int>> hit(n);
            for (auto& h : hit) h.store(0);
            pool.run(n, [&](unsigned i) { hit[i].fetch_add(1); });
            for (unsigned i = 0; i < n; i++) EXPECT(hit[i].load() == 1, "workers %u n %u index %u ran %d times", workers, n, i, hit[i].load());
        }
        // several submitting threads at once (jobs are serialised, none lost)
        std::atomic<long> total{0};
        std::vector<std::thread> subs;
        for (int t = 0; t < 4; t++)
            subs.emplace_back([&] {
                for (int r = 0; r < 200; r++) pool.run(37, [&](unsigned i) { total.fetch_add(i + 1); });
            });
        for (auto& s : subs) s.join();
        const long want = 4L * 200L * (37L * 38L / 2L);
        EXPECT(total.load() == want, "workers %u concurrent submitters: %ld vs %ld", workers, total.load(), want);
    }
    std::printf(failures ? "FAILED (%d)\n" : "ALL OK\n", failures);
    return failures ? 1 : 0;
}
