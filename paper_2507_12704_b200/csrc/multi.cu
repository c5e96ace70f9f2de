// multi.cu — rank_forward_batch over several GPUs of one box from one host process (C++):
// the multi-device host path of the reference's batch scorer (finetune.cpp:414-493, called by
// score_groups finetune.cpp:766-786).
//
// The scoring path shards by unique user: a user's context pass, K/V cache and
// its candidates' crossing pass touch no other user. So
//   1. rows are keyed by a 64-bit content hash of their event span (equal sequences, equal key),
//      hashed once per distinct (offset, valid) span by host threads;
//   2. uniques are assigned whole to devices, longest-processing-time first on a config-aware
//      cost (context GEMMs linear in n_u, causal softmax quadratic, crossing per candidate), so
//      each device's own dedup equals the global one and the devices finish together;
//   3. every device scores its rows in its own host thread (its own dcat_model, streams, CUDA
//      graphs; no collective inside the scoring pass);
//   4. the per-row scores are gathered to the first device with one NCCL group of sends / receives
//      over NVLink, copied to the host once and put back in the caller's row order.
// NCCL is loaded at run time (libnccl.so.2: the system's or the one a host framework already
// loaded); a multi-device call fails loudly when it is missing.
#include <dlfcn.h>

#include <algorithm>
#include <mutex>
#include <condition_variable>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dcat_b200.h"
#include "launch.h"
#include "host_pool.hpp"

namespace {

thread_local std::string g_merr;
int merr(int code, const std::string& m) {
    g_merr = m;
    return code;
}

// ---- NCCL through dlopen (the subset this file uses; nccl.h 2.x ABI)
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
constexpr int kNcclFloat32 = 7;  // ncclFloat32 / ncclFloat
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        commInitAll = reinterpret_cast<decltype(commInitAll)>(dlsym(h, "ncclCommInitAll"));
        commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(h, "ncclCommDestroy"));
        send = reinterpret_cast<decltype(send)>(dlsym(h, "ncclSend"));
        recv = reinterpret_cast<decltype(recv)>(dlsym(h, "ncclRecv"));
        groupStart = reinterpret_cast<decltype(groupStart)>(dlsym(h, "ncclGroupStart"));
        groupEnd = reinterpret_cast<decltype(groupEnd)>(dlsym(h, "ncclGroupEnd"));
        errorString = reinterpret_cast<decltype(errorString)>(dlsym(h, "ncclGetErrorString"));
        return commInitAll && commDestroy && send && recv && groupStart && groupEnd && errorString;
    }
};
Nccl& nccl() {
    static Nccl n;
    return n;
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != 0) throw dcat::CudaError(std::string(what) + ": " + nccl().errorString(r));
}

uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// content key of one event span (the dedup key's fields, dcat.cpp:45-56): equal spans, equal key
uint64_t span_hash(const dcat_batch& b, int64_t off, int32_t n) {
    uint64_t acc = 0;
    for (int32_t i = 0; i < n; i++) {
        const uint64_t pos = static_cast<uint64_t>(i);
        uint64_t t = mix64(b.ev_ts[off + i] ^ mix64(pos));
        t = mix64(t ^ b.ev_item[off + i]);
        t = mix64(t ^ (static_cast<uint64_t>(b.ev_action[off + i]) | static_cast<uint64_t>(b.ev_surface[off + i]) << 8));
        acc ^= mix64(t + pos);
    }
    return mix64(static_cast<uint64_t>(n) ^ acc);
}

// open-addressing map from a non-zero 64-bit key to an int32 (per-thread scratch: no locking)
struct FlatMap {
    std::vector<uint64_t> key;
    std::vector<int32_t> val;
    size_t mask = 0;
    explicit FlatMap(size_t n) {
        size_t cap = 16;
        while (cap < 2 * n) cap <<= 1;
        key.assign(cap, 0);
        val.assign(cap, -1);
        mask = cap - 1;
    }
    int32_t& slot(uint64_t k, bool* fresh) {
        size_t i = mix64(k) & mask;
        while (key[i] != 0 && key[i] != k) i = (i + 1) & mask;
        *fresh = key[i] == 0;
        key[i] = k;
        return val[i];
    }
};
// a row's event span as one non-zero key (offsets < 2^43, valid < 2^20)
inline uint64_t span_key(int64_t off, int32_t valid) {
    return (static_cast<uint64_t>(off) << 20 | static_cast<uint64_t>(valid)) + 1;
}
unsigned host_threads() { return std::max(1u, std::min(16u, std::thread::hardware_concurrency())); }


struct DevState {
    dcat_model* m = nullptr;
    int device = 0;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    float* out = nullptr;  // [rows x 6]: logits | module logits (device)
    size_t out_cap = 0;
    float* gather = nullptr;  // root only: [B x 6] in shard order
    size_t gather_cap = 0;
    void* arena = nullptr;  // page-locked staging of this device's rows
    size_t arena_bytes = 0;
};

}  // namespace

struct dcat_multi {
    dcat_model_config cfg{};
    std::vector<DevState> dev;
    std::unique_ptr<dcat::ThreadPool> pool{new dcat::ThreadPool(host_threads() - 1)};
    std::vector<int32_t> last_owner;
    std::vector<float> host_scores;
    ~dcat_multi() {
        dcat::DeviceScopeNoThrow ds(-1);  // restores the caller's current device, clears errors
        for (auto& d : dev) {
            // a device whose model was never created (e.g. an invalid ordinal) holds nothing
            if (!d.m && !d.stream && !d.comm && !d.out && !d.gather && !d.arena) continue;
            cudaSetDevice(d.device);
            cudaDeviceSynchronize();
            if (d.comm) nccl().commDestroy(d.comm);
            if (d.out) cudaFree(d.out);
            if (d.gather) cudaFree(d.gather);
            if (d.stream) cudaStreamDestroy(d.stream);
            if (d.m) dcat_model_destroy(d.m);
            if (d.arena) dcat_host_free(d.arena);
        }
    }
};

namespace {

// Seconds of device work of a unique (SURVEY §8(e) cost model; throughputs of one B200 at
// PinFM-base): context GEMMs 24 d^2 flops per token-layer + the causal softmax's
// H n (n + 1) / 2 exponentials per layer; per candidate its GEMMs and H (n + 1) exponentials per layer.
double unique_cost(const dcat_model_config& c, double n, double cands) {
    const double G = 6.0e14, X = 2.5e12, d = c.d_model, de = c.d_emb, l = c.n_layers, H = c.n_heads;
    const double tok = 2 * (de * d + d * d) + (l - 1) * 24 * d * d + 4 * d * d;
    const double ctx = n * tok / G + (l - 1) * H * n * (n + 1) / 2 / X;
    const double cand = 2 * (de * d + d * d) + l * 24 * d * d + 4 * d * d;
    return ctx + cands * (cand / G + l * H * (n + 1) / X);
}

// What shard() decides: the device of every row, and the distinct event spans (offset, valid) of
// the batch with the device that owns each (rows sharing a span are one user: one device).
struct ShardPlan {
    std::vector<int32_t> owner;  // [B] device of each row
    std::vector<int32_t> row_g;  // [B] distinct span of each row
    std::vector<int64_t> g_off;  // [S] distinct spans
    std::vector<int32_t> g_valid, g_owner;
};

// owner device of every row: content-keyed uniques, LPT on unique_cost. Host threads take
// contiguous row ranges and collect the distinct event spans (offset, valid) of their range; the
// spans are merged, each distinct span is content-hashed exactly once (in parallel), spans with
// equal content become one unique, uniques are assigned longest-processing-time first, and rows
// are mapped back to devices in parallel.
void shard(const dcat_multi* mh, const dcat_batch& b, ShardPlan& plan) {
    const int64_t B = b.n_rows;
    const int nd = static_cast<int>(mh->dev.size());
    std::vector<int32_t>& owner = plan.owner;
    owner.assign(static_cast<size_t>(B), 0);
    plan.row_g.assign(static_cast<size_t>(B), 0);
    plan.g_off.clear();
    plan.g_valid.clear();
    plan.g_owner.clear();
    if (nd == 1 || B == 0) return;
    struct Local {
        std::vector<int64_t> off;   // distinct spans of the range
        std::vector<int32_t> valid, rows;
        std::vector<int32_t> row_s;  // local span of each row of the range
        std::vector<int32_t> to_global;
    };
    const unsigned T = static_cast<unsigned>(std::min<int64_t>(host_threads(), std::max<int64_t>(1, B / 4096)));
    std::vector<Local> loc(T);
    std::vector<int64_t> r0s(T + 1);
    for (unsigned t = 0; t <= T; t++) r0s[t] = B * t / T;
    auto parallel = [&](unsigned n, const std::function<void(unsigned)>& f) { mh->pool->run(n, f); };
    // 1. distinct spans per row range
    parallel(T, [&](unsigned t) {
        Local& L = loc[t];
        const int64_t r0 = r0s[t], r1 = r0s[t + 1];
        FlatMap spans(static_cast<size_t>(r1 - r0));
        L.row_s.resize(static_cast<size_t>(r1 - r0));
        for (int64_t r = r0; r < r1; r++) {
            bool fresh;
            int32_t& si = spans.slot(span_key(b.row_offset[r], b.row_valid[r]), &fresh);
            if (fresh) {
                si = static_cast<int32_t>(L.off.size());
                L.off.push_back(b.row_offset[r]);
                L.valid.push_back(b.row_valid[r]);
                L.rows.push_back(0);
            }
            L.rows[static_cast<size_t>(si)]++;
            L.row_s[static_cast<size_t>(r - r0)] = si;
        }
    });
    // 2. merge into global distinct spans
    size_t total = 0;
    for (auto& L : loc) total += L.off.size();
    FlatMap gmap(total);
    std::vector<int64_t>& g_off = plan.g_off;
    std::vector<int32_t>& g_valid = plan.g_valid;
    std::vector<double> g_rows;
    for (auto& L : loc) {
        L.to_global.resize(L.off.size());
        for (size_t i = 0; i < L.off.size(); i++) {
            bool fresh;
            int32_t& g = gmap.slot(span_key(L.off[i], L.valid[i]), &fresh);
            if (fresh) {
                g = static_cast<int32_t>(g_off.size());
                g_off.push_back(L.off[i]);
                g_valid.push_back(L.valid[i]);
                g_rows.push_back(0);
            }
            g_rows[static_cast<size_t>(g)] += L.rows[i];
            L.to_global[i] = g;
        }
    }
    // 3. one content hash per distinct span
    const size_t S = g_off.size();
    std::vector<uint64_t> g_hash(S);
    const unsigned TH = static_cast<unsigned>(std::min<size_t>(host_threads(), std::max<size_t>(1, S / 64)));
    parallel(TH, [&](unsigned t) {
        for (size_t k = S * t / TH; k < S * (t + 1) / TH; k++)
            g_hash[k] = span_hash(b, g_off[k], g_valid[k]) | 1;  // non-zero map key
    });
    // 4. spans of equal content -> one unique (its tokens, its rows)
    FlatMap umap(S);
    std::vector<int32_t> span_u(S);
    std::vector<uint64_t> ukey;
    std::vector<double> un, uc;
    for (size_t k = 0; k < S; k++) {
        bool fresh;
        int32_t& u = umap.slot(g_hash[k], &fresh);
        if (fresh) {
            u = static_cast<int32_t>(ukey.size());
            ukey.push_back(g_hash[k]);
            un.push_back(g_valid[k]);
            uc.push_back(0);
        }
        uc[static_cast<size_t>(u)] += g_rows[k];
        span_u[k] = u;
    }
    // 5. LPT on the config-aware cost
    const size_t U = ukey.size();
    std::vector<int32_t> order(U);
    std::vector<double> cost(U);
    for (size_t u = 0; u < U; u++) {
        order[u] = static_cast<int32_t>(u);
        cost[u] = unique_cost(mh->cfg, un[u], uc[u]);
    }
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        return cost[x] != cost[y] ? cost[x] > cost[y] : ukey[x] < ukey[y];
    });
    using Load = std::pair<double, int>;
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int d = 0; d < nd; d++) heap.push({0.0, d});
    std::vector<int32_t> u_owner(U);
    for (int32_t u : order) {
        Load top = heap.top();
        heap.pop();
        u_owner[static_cast<size_t>(u)] = top.second;
        heap.push({top.first + cost[static_cast<size_t>(u)], top.second});
    }
    // 6. spans and rows -> devices
    plan.g_owner.resize(S);
    for (size_t k = 0; k < S; k++) plan.g_owner[k] = u_owner[static_cast<size_t>(span_u[k])];
    parallel(T, [&](unsigned t) {
        const Local& L = loc[t];
        for (int64_t r = r0s[t]; r < r0s[t + 1]; r++) {
            const int32_t g = L.to_global[static_cast<size_t>(L.row_s[static_cast<size_t>(r - r0s[t])])];
            plan.row_g[static_cast<size_t>(r)] = g;
            owner[static_cast<size_t>(r)] = plan.g_owner[static_cast<size_t>(g)];
        }
    });
}

// one device's rows as a compact host batch (each used span copied once)
// one device's rows as a compact batch (each used span copied once) in the device's page-locked
// staging arena, so its H2D copies are asynchronous DMA
struct LocalBatch {
    std::vector<int64_t> rows;
    dcat_batch c{};
    // P host threads copy the device's distinct spans (each once) and fill its rows
    void build(const dcat_batch& b, const ShardPlan& plan, int d, void*& arena, size_t& arena_bytes, unsigned P,
               dcat::ThreadPool& pool) {
        rows.clear();
        for (int64_t r = 0; r < b.n_rows; r++)
            if (plan.owner[static_cast<size_t>(r)] == d) rows.push_back(r);
        const size_t n = rows.size(), S = plan.g_off.size();
        // the device's distinct spans and their offsets in its compact event pool
        std::vector<int64_t> span_off(S, -1);
        std::vector<int32_t> mine;
        size_t E = 0;
        for (size_t k = 0; k < S; k++)
            if (plan.g_owner[k] == d) {
                span_off[k] = static_cast<int64_t>(E);
                E += static_cast<size_t>(plan.g_valid[k]);
                mine.push_back(static_cast<int32_t>(k));
            }
        const int da = b.aux ? b.d_aux : 0;
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        const size_t o_off = 0, o_valid = al(8 * n), o_cand = al(o_valid + 4 * n), o_age = al(o_cand + 8 * n),
                     o_aux = al(o_age + 8 * n), o_ts = al(o_aux + 4 * n * static_cast<size_t>(da)), o_item = al(o_ts + 8 * E),
                     o_act = al(o_item + 8 * E), o_surf = al(o_act + E), total = al(o_surf + E) + 16;
        if (total > arena_bytes) {
            if (arena) dcat_host_free(arena);
            arena = nullptr;
            arena_bytes = 0;
            const size_t want = total + total / 4;
            if (dcat_host_alloc(want, &arena) != DCAT_OK) throw dcat::CudaError("pinned staging allocation failed");
            arena_bytes = want;
        }
        uint8_t* base = static_cast<uint8_t*>(arena);
        int64_t* off = reinterpret_cast<int64_t*>(base + o_off);
        int32_t* valid = reinterpret_cast<int32_t*>(base + o_valid);
        uint64_t* cand = reinterpret_cast<uint64_t*>(base + o_cand);
        double* age = reinterpret_cast<double*>(base + o_age);
        float* aux = reinterpret_cast<float*>(base + o_aux);
        uint64_t* ts = reinterpret_cast<uint64_t*>(base + o_ts);
        uint64_t* item = reinterpret_cast<uint64_t*>(base + o_item);
        uint8_t* act = base + o_act;
        uint8_t* surf = base + o_surf;
        const unsigned nt = std::max(1u, std::min<unsigned>(P, static_cast<unsigned>((n + E / 64) / 8192 + 1)));
        auto part = [&](unsigned t) {
            for (size_t q = mine.size() * t / nt; q < mine.size() * (t + 1) / nt; q++) {  // the span events
                const size_t k = static_cast<size_t>(mine[q]);
                const int64_t o = plan.g_off[k], e0 = span_off[k];
                const size_t v = static_cast<size_t>(plan.g_valid[k]);
                std::memcpy(ts + e0, b.ev_ts + o, 8 * v);
                std::memcpy(item + e0, b.ev_item + o, 8 * v);
                std::memcpy(act + e0, b.ev_action + o, v);
                std::memcpy(surf + e0, b.ev_surface + o, v);
            }
            for (size_t i = n * t / nt; i < n * (t + 1) / nt; i++) {  // the rows
                const int64_t r = rows[i];
                off[i] = span_off[static_cast<size_t>(plan.row_g[static_cast<size_t>(r)])];
                valid[i] = b.row_valid[r];
                cand[i] = b.candidate[r];
                age[i] = b.age_seconds[r];
                if (da) std::memcpy(aux + i * da, b.aux + r * da, sizeof(float) * static_cast<size_t>(da));
            }
        };
        pool.run(nt, part);
        c = dcat_batch{};
        c.n_rows = static_cast<int64_t>(n);
        c.row_offset = off;
        c.row_valid = valid;
        c.n_events = static_cast<int64_t>(E);
        c.ev_ts = ts;
        c.ev_action = act;
        c.ev_surface = surf;
        c.ev_item = item;
        c.candidate = cand;
        c.age_seconds = age;
        c.aux = da ? aux : nullptr;
        c.d_aux = da;
    }
};

}  // namespace

extern "C" {

const char* dcat_multi_last_error(void) { return g_merr.c_str(); }

int dcat_multi_create(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                      const dcat_head* head, const int32_t* devices, int32_t n_devices, dcat_multi** out) {
    if (!cfg || !params || !table || !head || !devices || !out || n_devices < 1)
        return merr(DCAT_EINVAL, "null argument");
    *out = nullptr;
    std::unique_ptr<dcat_multi> mh(new dcat_multi());
    mh->cfg = *cfg;
    for (int i = 0; i < n_devices; i++)
        for (int j = 0; j < i; j++)
            if (devices[i] == devices[j]) return merr(DCAT_EINVAL, "dcat_multi_create: devices must be distinct");
    try {
        dcat::DeviceGuard dg(-1);
        mh->dev.resize(static_cast<size_t>(n_devices));
        for (int i = 0; i < n_devices; i++) {
            DevState& d = mh->dev[static_cast<size_t>(i)];
            d.device = devices[i];
            int rc = dcat_model_create(cfg, params, table, head, devices[i], &d.m);
            if (rc) return merr(rc, dcat_last_error());
            DCAT_CUDA_CHECK(cudaSetDevice(devices[i]));
            DCAT_CUDA_CHECK(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
        }
        if (n_devices > 1) {
            if (!nccl().load()) return merr(DCAT_EUNSUPPORTED, "dcat_multi_create: libnccl.so.2 not loadable");
            std::vector<ncclComm_t> comms(static_cast<size_t>(n_devices));
            nccl_check(nccl().commInitAll(comms.data(), n_devices, devices), "ncclCommInitAll");
            for (int i = 0; i < n_devices; i++) mh->dev[static_cast<size_t>(i)].comm = comms[static_cast<size_t>(i)];
        }
    } catch (const dcat::CudaError& e) {
        return merr(DCAT_ECUDA, e.msg);
    }
    *out = mh.release();
    return DCAT_OK;
}

int dcat_multi_destroy(dcat_multi* mh) {
    delete mh;
    return DCAT_OK;
}

int dcat_multi_shard(dcat_multi* mh, const dcat_batch* batch, int32_t* owner) {
    if (!mh || !batch || !owner) return merr(DCAT_EINVAL, "null argument");
    ShardPlan plan;
    shard(mh, *batch, plan);
    std::memcpy(owner, plan.owner.data(), sizeof(int32_t) * plan.owner.size());
    return DCAT_OK;
}

int dcat_multi_rank_forward_batch(dcat_multi* mh, const dcat_batch* batch, const dcat_finetune_config* ft,
                                  float* logits, float* module_logits, int32_t flags) {
    if (!mh || !batch || !ft || !logits || !module_logits) return merr(DCAT_EINVAL, "null argument");
    if (flags & (DCAT_INPUT_DEVICE | DCAT_OUTPUT_DEVICE))
        return merr(DCAT_EINVAL, "dcat_multi_rank_forward_batch takes host buffers");
    try {
        dcat::NvtxRange nr("dcat_multi_rank_forward_batch");
        dcat::DeviceGuard dg(-1);  // the calling thread's current device is restored on return
        const int nd = static_cast<int>(mh->dev.size());
        const int64_t B = batch->n_rows;
        if (B == 0) return DCAT_OK;
        if (nd == 1) {  // one device: the single-device call on the caller's buffers
            mh->last_owner.assign(static_cast<size_t>(B), 0);
            int rc = dcat_rank_forward_batch(mh->dev[0].m, batch, ft, logits, module_logits, nullptr,
                                             flags & DCAT_PRECISION_FP32, mh->dev[0].stream);
            return rc ? merr(rc, dcat_last_error()) : DCAT_OK;
        }
        // DCAT_MULTI_TIMING=1: host wall time of each phase on stderr (investigation aid)
        static const bool timing = getenv("DCAT_MULTI_TIMING") != nullptr;
        using clk = std::chrono::steady_clock;
        const auto t_start = clk::now();
        std::vector<double> t_build(static_cast<size_t>(nd)), t_score(static_cast<size_t>(nd));
        ShardPlan plan;
        shard(mh, *batch, plan);
        mh->last_owner = plan.owner;
        const auto t_shard = clk::now();
        std::vector<LocalBatch> lb(static_cast<size_t>(nd));  // built by each device's own thread
        // 3. every device scores its rows (device outputs, no host round trip), one host thread each
        std::vector<int> rc(static_cast<size_t>(nd), 0);
        std::vector<std::string> msg(static_cast<size_t>(nd));
        auto work = [&](int d) {
            DevState& s = mh->dev[static_cast<size_t>(d)];
            const auto b0 = clk::now();
            lb[static_cast<size_t>(d)].build(*batch, plan, d, s.arena, s.arena_bytes, mh->pool->size(), *mh->pool);
            const auto b1 = clk::now();
            t_build[static_cast<size_t>(d)] = std::chrono::duration<double, std::milli>(b1 - b0).count();
            const size_t n = lb[static_cast<size_t>(d)].rows.size();
            try {
                DCAT_CUDA_CHECK(cudaSetDevice(s.device));
                if (n * 6 > s.out_cap) {
                    if (s.out) DCAT_CUDA_CHECK(cudaFree(s.out));
                    s.out_cap = n * 6 + n * 6 / 4 + 64;
                    DCAT_CUDA_CHECK(cudaMalloc(&s.out, s.out_cap * sizeof(float)));
                }
                if (n == 0) return;
                rc[static_cast<size_t>(d)] =
                    dcat_rank_forward_batch(s.m, &lb[static_cast<size_t>(d)].c, ft, s.out, s.out + n * 3, nullptr,
                                            (flags & DCAT_PRECISION_FP32) | DCAT_OUTPUT_DEVICE, s.stream);
                if (rc[static_cast<size_t>(d)]) msg[static_cast<size_t>(d)] = dcat_last_error();
                if (timing) {
                    DCAT_CUDA_CHECK(cudaStreamSynchronize(s.stream));
                    t_score[static_cast<size_t>(d)] = std::chrono::duration<double, std::milli>(clk::now() - b1).count();
                }
            } catch (const dcat::CudaError& e) {
                rc[static_cast<size_t>(d)] = DCAT_ECUDA;
                msg[static_cast<size_t>(d)] = e.msg;
            }
        };
        std::vector<std::thread> th;
        for (int d = 1; d < nd; d++) th.emplace_back(work, d);
        work(0);
        for (auto& x : th) x.join();
        const auto t_scored = clk::now();
        for (int d = 0; d < nd; d++)
            if (rc[static_cast<size_t>(d)]) return merr(rc[static_cast<size_t>(d)], msg[static_cast<size_t>(d)]);
        // 4. gather to the first device: one NCCL group of sends / receives over NVLink
        DevState& root = mh->dev[0];
        DCAT_CUDA_CHECK(cudaSetDevice(root.device));
        if (static_cast<size_t>(B) * 6 > root.gather_cap) {
            if (root.gather) DCAT_CUDA_CHECK(cudaFree(root.gather));
            root.gather_cap = static_cast<size_t>(B) * 6;
            DCAT_CUDA_CHECK(cudaMalloc(&root.gather, root.gather_cap * sizeof(float)));
        }
        std::vector<size_t> at(static_cast<size_t>(nd) + 1, 0);
        for (int d = 0; d < nd; d++) at[d + 1] = at[d] + lb[static_cast<size_t>(d)].rows.size() * 6;
        const size_t n0 = lb[0].rows.size();
        if (n0) DCAT_CUDA_CHECK(cudaMemcpyAsync(root.gather, root.out, n0 * 6 * sizeof(float), cudaMemcpyDeviceToDevice,
                                                root.stream));
        if (nd > 1) {
            nccl_check(nccl().groupStart(), "ncclGroupStart");
            for (int d = 1; d < nd; d++) {
                const size_t cnt = at[d + 1] - at[d];
                if (!cnt) continue;
                DevState& s = mh->dev[static_cast<size_t>(d)];
                nccl_check(nccl().send(s.out, cnt, kNcclFloat32, 0, s.comm, s.stream), "ncclSend");
                nccl_check(nccl().recv(root.gather + at[d], cnt, kNcclFloat32, d, root.comm, root.stream), "ncclRecv");
            }
            nccl_check(nccl().groupEnd(), "ncclGroupEnd");
        }
        mh->host_scores.resize(static_cast<size_t>(B) * 6);
        DCAT_CUDA_CHECK(cudaMemcpyAsync(mh->host_scores.data(), root.gather, sizeof(float) * B * 6,
                                        cudaMemcpyDeviceToHost, root.stream));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(root.stream));
        for (int d = 1; d < nd; d++) {
            DCAT_CUDA_CHECK(cudaSetDevice(mh->dev[static_cast<size_t>(d)].device));
            DCAT_CUDA_CHECK(cudaStreamSynchronize(mh->dev[static_cast<size_t>(d)].stream));
        }
        // back to the caller's row order: device d's block holds its n_d rows as [logits | module logits]
        // every device's block in slices across the pool
        const unsigned per = std::max(1u, mh->pool->size() / static_cast<unsigned>(nd));
        mh->pool->run(static_cast<unsigned>(nd) * per, [&](unsigned k) {
            const int d = static_cast<int>(k / per), part = static_cast<int>(k % per);
            const auto& rows = lb[static_cast<size_t>(d)].rows;
            const float* blk = mh->host_scores.data() + at[d];
            const size_t n = rows.size();
            for (size_t i = n * part / per; i < n * (part + 1) / per; i++) {
                std::memcpy(logits + rows[i] * 3, blk + i * 3, 3 * sizeof(float));
                std::memcpy(module_logits + rows[i] * 3, blk + n * 3 + i * 3, 3 * sizeof(float));
            }
        });
        if (timing) {
            auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "dcat_multi: shard %.3f ms | build", ms(t_start, t_shard));
            for (double v : t_build) std::fprintf(stderr, " %.3f", v);
            std::fprintf(stderr, " | score");
            for (double v : t_score) std::fprintf(stderr, " %.3f", v);
            std::fprintf(stderr, " | threads joined %.3f | gather+d2h+scatter %.3f | total %.3f ms\n",
                         ms(t_start, t_scored), ms(t_scored, clk::now()), ms(t_start, clk::now()));
        }
        return DCAT_OK;
    } catch (const dcat::CudaError& e) {
        return merr(DCAT_ECUDA, e.msg);
    } catch (const std::bad_alloc&) {
        return merr(DCAT_ENOMEM, "host out of memory");
    }
}

}  // extern "C"
