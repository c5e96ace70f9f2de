// dcat_api.cu — the C ABI (include/dcat_b200.h) and the host runtime that
// orchestrates the DCAT scoring forward on one B200.
//
// rank_forward_batch (/root/reference/proj/src/finetune.cpp:414-493):
//   dedup (K1)  ->  context pass: gather (K2), phi_in, layers 0..L-2
//   (QKV / causal attention K5 / O+LN / FFN), last layer K,V only
//   (dcat.cpp:137-178)  ->  crossing pass: candidate gather, phi_in, L layers
//   (QKV / crossing attention K6 / O+LN / FFN), phi_out + module head
//   (dcat.cpp:199-271)  ->  ranking head (finetune.cpp:301-324)  ->  scatter.
// Inputs are validated on the device in the dedup pass (the reference's
// SEQFM_CHECKs) and reported through dcat_last_error().
#include <cuda_bf16.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/dcat_b200.h"
#include "launch.h"

using namespace dcat;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

uint64_t host_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// bumped whenever a work buffer is (re)allocated: a cached graph of the scoring pass is only
// replayed while every buffer it captured still exists
std::atomic<uint64_t> g_alloc_epoch{0};

constexpr int kDebugCounters = 8;

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    ~Buf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* get(size_t n) {
        size_t bytes = std::max<size_t>(n * sizeof(T), 256);
        if (bytes > cap) {
            if (p) DCAT_CUDA_CHECK(cudaFree(p));
            p = nullptr;
            size_t c = bytes + bytes / 4;
            c = (c + 4095) & ~size_t(4095);
            DCAT_CUDA_CHECK(cudaMalloc(&p, c));
            cap = c;
            g_alloc_epoch++;
        }
        return static_cast<T*>(p);
    }
};

// One linear layer, stored for both paths.
struct Lin {
    bf16* wt = nullptr;   // [out x in] bf16 (tensor-core path, K-major)
    float* w32 = nullptr; // [in x out] fp32 (parity path, reference layout)
    float* bias = nullptr;
    int in = 0, out = 0;
    int in32 = 0;  // fp32 path K (in, before bf16 zero padding)
};

struct LayerW {
    float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
    Lin qkv, o, f1, f2;  // qkv = [Wq | Wk | Wv] along the output dim
};

struct DevAlloc {
    std::vector<void*> ptrs;
    ~DevAlloc() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* upload(const T* h, size_t n) {
        void* p = nullptr;
        DCAT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
        ptrs.push_back(p);
        if (n) DCAT_CUDA_CHECK(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
        return static_cast<T*>(p);
    }
};

}  // namespace

struct dcat_model {
    int device = 0;
    dcat_model_config cfg{};
    DevAlloc mem;
    // embeddings (fp32)
    float* table = nullptr;
    uint8_t* qtable = nullptr;  // QuantizedTable payload (bits 4 / 8), dequantized in the gathers
    int qbits = 0, qrow_bytes = 0, qcode_bytes = 0;
    uint64_t* seed_mix = nullptr;
    int J = 0, R = 0, d_sub = 0;
    float *action_emb = nullptr, *surface_emb = nullptr, *pos_emb = nullptr;
    int t_dedup_end = 0;   // profiling mark after the plan read-back
    float* cmb = nullptr;  // (action + surface) + pos rows for the bf16 context gather, or null
    Lin phi_in1, phi_in2, phi_out1, phi_out2;
    std::vector<LayerW> layers;
    // ranking head
    int d_module = 0, head_demb = 0, n_ctx = 0, hidden = 0, d_aux = 0, kh = 0, d_feat = 0;
    Lin head1;  // [feat -> hidden], wt zero-padded to kh columns
    float *hw2 = nullptr, *hb2 = nullptr, *mod_w = nullptr, *mod_b = nullptr, *aux_proj = nullptr, *lt = nullptr;
    // status
    Status* st_dev = nullptr;
    Status* st_host = nullptr;
    unsigned* dbg = nullptr;  // DCAT_DEBUG_COUNTERS at create: device counters (dcat_debug_counters)
    // workspace
    Buf b_in[8];
    Buf b_dd[24];
    Buf b_act[28];
    Buf b_kv;
    Buf b_aux;
    Buf b_out[3];
    Buf b_x[6];  // dcat_context_forward / dcat_candidate_inputs / dcat_cross_forward staging
    // last-call bookkeeping
    int64_t last_bu = 0, last_T = 0, last_Tp = 0;
    int last_precision_f32 = 0;
    int tile_ctx = 64, tile_cross = 128;  // attention query tiles of the current call
    bool vt = false;                      // current call keeps the V cache transposed (tcgen05 attention)
    bool last_vt = false;
    void* last_kv = nullptr;
    std::vector<int64_t> last_tok_off;
    const int64_t* last_tok_off_dev = nullptr;  // the last call's context token offsets (read lazily)
    dcat_call_stats stats{};
    std::vector<std::pair<const char*, float>> stage_ms;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<const char*, std::pair<int, int>>> ev_marks;
    bool profiling = false;
    int ev_next = 0;
    // host batches: the candidate-side arrays (candidate, age, aux) are copied on a side stream
    // after the dedup inputs, overlapping the dedup and context kernels (they are first read by
    // the candidate gather, which waits on cand_ready)
    cudaStream_t side = nullptr;
    cudaEvent_t side_start = nullptr, cand_ready = nullptr;
    // two-stream scoring pass: the crossing pass runs on xs beside the context pass; crossing
    // layer l waits only for kv_ev[l] (context layer l's K / V cache written), and xs joins back
    // before the head (small batches; see run_dcat).
    cudaStream_t xs = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    std::vector<cudaEvent_t> kv_ev;
    // the dedup / plan launch sequence as a CUDA graph, re-captured when its arguments change
    struct DedupKey {
        DedupIn in;
        DedupOut o;
        uint64_t mask;
        int tile_ctx, tile_cross;
    };
    DedupKey dd_key;
    cudaGraphExec_t dd_exec = nullptr;
    cudaStream_t cap = nullptr;
    // the scoring pass after the plan read-back (run_dcat) as a CUDA graph: a call whose sizes,
    // pointers and settings equal the previous call's is captured, and replayed while they repeat
    std::vector<uint64_t> run_seen, run_key;
    cudaGraphExec_t run_exec = nullptr;
    dcat_call_stats run_stats{};
    void* run_last_kv = nullptr;  // host bookkeeping run_dcat sets, restored on replay
    int64_t run_last_Tp = 0;

    ~dcat_model() {
        if (st_host) cudaFreeHost(st_host);
        for (auto e : ev_pool) cudaEventDestroy(e);
        if (side_start) cudaEventDestroy(side_start);
        if (cand_ready) cudaEventDestroy(cand_ready);
        if (side) cudaStreamDestroy(side);
        if (xs) cudaStreamDestroy(xs);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (join_ev) cudaEventDestroy(join_ev);
        for (auto e : kv_ev) cudaEventDestroy(e);
        if (dd_exec) cudaGraphExecDestroy(dd_exec);
        if (run_exec) cudaGraphExecDestroy(run_exec);
        if (cap) cudaStreamDestroy(cap);
    }
};

// context_forward's KVCache / FixedKVCache on the device (dcat_context_forward)
struct dcat_kv {
    dcat_model* m = nullptr;
    int device = 0;
    bool f32 = false, vt = false;
    int n_layers = 0, d = 0, window = 0;
    int64_t Tp = 0, T_ctx = 0;
    void* buf = nullptr;           // [layer][K|V][Tp][d] (V^T [d][Tp] when vt), the model's layout
    std::vector<int32_t> rep;      // caller row -> plan unique (equal sequences share one)
    std::vector<int64_t> tok_off;  // plan unique -> first token, b_u + 1 entries
    ~dcat_kv() {
        if (buf) cudaFree(buf);
    }
};

namespace {

// ---------------------------------------------------------------- profiling
bool host_timing() {  // DCAT_HOST_TIMING=1: host-side phase times of each call on stderr (tools)
    static const bool on = getenv("DCAT_HOST_TIMING") != nullptr;
    return on;
}

int mark(dcat_model* m, cudaStream_t s) {
    if (!m->profiling) return -1;
    if (m->ev_next >= static_cast<int>(m->ev_pool.size())) {
        cudaEvent_t e;
        DCAT_CUDA_CHECK(cudaEventCreate(&e));
        m->ev_pool.push_back(e);
    }
    int i = m->ev_next++;
    DCAT_CUDA_CHECK(cudaEventRecord(m->ev_pool[i], s));
    return i;
}
void span(dcat_model* m, const char* name, int a, int b) {
    if (a >= 0 && b >= 0) m->ev_marks.push_back({name, {a, b}});
}

// ---------------------------------------------------------------- upload
Lin make_lin(DevAlloc& mem, const float* w, const float* b, int in, int out, int k_pad = 0) {
    Lin L;
    L.in = in;
    L.in32 = in;
    L.out = out;
    int kp = std::max(in, k_pad);
    std::vector<bf16> wt(static_cast<size_t>(out) * kp, __float2bfloat16(0.0f));
    for (int i = 0; i < in; i++)
        for (int o = 0; o < out; o++)
            wt[static_cast<size_t>(o) * kp + i] = __float2bfloat16_rn(w[static_cast<size_t>(i) * out + o]);
    L.wt = mem.upload(wt.data(), wt.size());
    L.w32 = mem.upload(w, static_cast<size_t>(in) * out);
    std::vector<float> bz(static_cast<size_t>(out), 0.0f);
    L.bias = mem.upload(b ? b : bz.data(), static_cast<size_t>(out));
    return L;
}

// [Wq | Wk | Wv] concatenated along the output dimension
Lin make_qkv(DevAlloc& mem, const float* wq, const float* bq, const float* wk, const float* bk, const float* wv,
             const float* bv, int d) {
    std::vector<float> w(static_cast<size_t>(d) * 3 * d), b(static_cast<size_t>(3) * d);
    const float* ws[3] = {wq, wk, wv};
    const float* bs[3] = {bq, bk, bv};
    for (int s = 0; s < 3; s++) {
        for (int i = 0; i < d; i++)
            for (int o = 0; o < d; o++) w[static_cast<size_t>(i) * 3 * d + s * d + o] = ws[s][static_cast<size_t>(i) * d + o];
        for (int o = 0; o < d; o++) b[s * d + o] = bs[s][o];
    }
    return make_lin(mem, w.data(), b.data(), d, 3 * d);
}

// ---------------------------------------------------------------- error text
std::string status_message(const dcat_model* m, const Status& st, int* code) {
    *code = DCAT_EINVAL;
    char buf[256];
    int b = st.err_bits;
    if (b & ERR_RANGE) snprintf(buf, sizeof buf, "row %d: events out of range (valid %d)", st.err_row, st.err_val);
    else if (b & ERR_ACTION) snprintf(buf, sizeof buf, "unknown action value %d (row %d)", st.err_val, st.err_row);
    else if (b & ERR_SURFACE) snprintf(buf, sizeof buf, "unknown surface value %d (row %d)", st.err_val, st.err_row);
    else if (b & ERR_POS_CTX)
        snprintf(buf, sizeof buf, "position %d exceeds max_len %d (row %d)", st.err_val, m->cfg.max_len, st.err_row);
    else if (b & ERR_POS_CAND)
        snprintf(buf, sizeof buf, "candidate_inputs: position %d out of range (max_len %d)", st.err_val,
                 m->cfg.max_len);
    else if (b & ERR_AGE) snprintf(buf, sizeof buf, "candidate age must be non-negative (row %d)", st.err_row);
    else if (st.nonfinite_layer > 0) {
        *code = DCAT_ENONFINITE;
        snprintf(buf, sizeof buf, "non-finite activation in layer %d", st.nonfinite_layer - 1);
    } else
        return "";
    return buf;
}

// ---------------------------------------------------------------- staging
struct Staged {
    DedupIn in;
    const uint64_t* candidate;
    const double* age;
    const float* aux;
    cudaEvent_t cand_ready = nullptr;  // side-stream copy of candidate / age / aux, or null
};
// the stream waits for the side-stream candidate copies (before the first candidate gather)
void wait_cand(const Staged& sb, cudaStream_t s) {
    if (sb.cand_ready) DCAT_CUDA_CHECK(cudaStreamWaitEvent(s, sb.cand_ready, 0));
}

template <typename T>
const T* stage(Buf& b, const T* src, size_t n, bool device, cudaStream_t s, int64_t* h2d) {
    if (device || src == nullptr) return src;
    T* d = b.get<T>(n);
    if (n) DCAT_CUDA_CHECK(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    *h2d += static_cast<int64_t>(n * sizeof(T));
    return d;
}

Staged stage_batch(dcat_model* m, const dcat_batch* b, bool device, bool aux_needed, cudaStream_t s,
                   bool side_cand = false) {
    Staged st;
    std::memset(&st.in, 0, sizeof st.in);  // padding too: the dedup graph cache compares it bytewise
    int64_t h2d = 0;
    int64_t B = b->n_rows, E = b->n_events;
    st.in.B = B;
    st.in.row_offset = stage(m->b_in[0], b->row_offset, B, device, s, &h2d);
    st.in.row_valid = stage(m->b_in[1], b->row_valid, B, device, s, &h2d);
    st.in.n_events = E;
    // one pooled copy for the four event arrays
    if (device) {
        st.in.ts = b->ev_ts;
        st.in.action = b->ev_action;
        st.in.surface = b->ev_surface;
        st.in.item = b->ev_item;
    } else {
        st.in.ts = stage(m->b_in[2], b->ev_ts, E, false, s, &h2d);
        st.in.item = stage(m->b_in[3], b->ev_item, E, false, s, &h2d);
        st.in.action = stage(m->b_in[4], b->ev_action, E, false, s, &h2d);
        st.in.surface = stage(m->b_in[5], b->ev_surface, E, false, s, &h2d);
    }
    st.in.n_actions = m->cfg.n_actions;
    st.in.n_surfaces = m->cfg.n_surfaces;
    st.in.max_len = m->cfg.max_len;
    st.in.pos_learned = m->cfg.pos_learned;
    st.in.window = 0;
    st.in.lt_token = 0;
    cudaStream_t cs = s;
    if (side_cand && !device) {  // queued behind the dedup inputs, on the side stream
        if (!m->side) {
            DCAT_CUDA_CHECK(cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking));
            DCAT_CUDA_CHECK(cudaEventCreateWithFlags(&m->side_start, cudaEventDisableTiming));
            DCAT_CUDA_CHECK(cudaEventCreateWithFlags(&m->cand_ready, cudaEventDisableTiming));
        }
        DCAT_CUDA_CHECK(cudaEventRecord(m->side_start, s));
        DCAT_CUDA_CHECK(cudaStreamWaitEvent(m->side, m->side_start, 0));
        cs = m->side;
    }
    st.candidate = stage(m->b_in[6], b->candidate, B, device, cs, &h2d);
    st.age = stage(m->b_in[7], b->age_seconds, B, device, cs, &h2d);
    st.aux = nullptr;
    if (aux_needed && b->aux) {
        st.aux = stage(m->b_aux, b->aux, static_cast<size_t>(B) * b->d_aux, device, cs, &h2d);
    }
    if (cs != s) {
        DCAT_CUDA_CHECK(cudaEventRecord(m->cand_ready, cs));
        st.cand_ready = m->cand_ready;
    }
    return st;
}

DedupOut dedup_buffers(dcat_model* m, int64_t B) {
    DedupOut o;
    std::memset(&o, 0, sizeof o);  // padding too: the dedup graph cache compares it bytewise
    int64_t cap = 1024;
    while (cap < 2 * B) cap <<= 1;
    size_t n1 = static_cast<size_t>(B) + 1;
    o.hash = m->b_dd[0].get<uint64_t>(B);
    o.tab_key = m->b_dd[1].get<uint64_t>(cap);
    o.tab_val = m->b_dd[2].get<int32_t>(cap);
    o.tab_cap = cap;
    o.slot = m->b_dd[3].get<int32_t>(B);
    o.head = m->b_dd[4].get<int32_t>(B);
    o.collided = m->b_dd[5].get<int32_t>(B);
    o.list = m->b_dd[6].get<int32_t>(B);
    o.list_n = m->b_dd[7].get<int32_t>(1);
    o.scan_tmp = m->b_dd[8].get<int64_t>(n1);
    o.scan_blk = m->b_dd[9].get<int64_t>(4 * 4097);  // four arrays' block sums
    o.uid = m->b_dd[10].get<int64_t>(n1);
    o.rep = m->b_dd[11].get<int32_t>(B);
    o.first = m->b_dd[12].get<int32_t>(B);
    o.cnt = m->b_dd[13].get<int32_t>(B);
    o.cursor = m->b_dd[14].get<int32_t>(B);
    o.goff = m->b_dd[15].get<int64_t>(n1);
    o.perm = m->b_dd[16].get<int32_t>(B);
    o.tok_off = m->b_dd[17].get<int64_t>(n1);
    o.ctx_toff = m->b_dd[18].get<int64_t>(n1);
    o.cross_toff = m->b_dd[19].get<int64_t>(n1);
    o.st = m->st_dev;
    return o;
}

uint64_t debug_hash_mask() {
    const char* e = getenv("DCAT_DEBUG_HASH_BITS");  // test knob: force 64-bit hash collisions
    if (!e) return ~0ull;
    int bits = atoi(e);
    if (bits <= 0 || bits >= 64) return ~0ull;
    return (1ull << bits) - 1;
}

// Attention kernels (bf16 path): attn_fa.cu (tcgen05 + TMA, S / P / O in TMEM) for head dims
// 16 / 32 / 64; it reads the V cache transposed (keys contiguous), so the K/V projection stores it
// that way and both passes use 128-query tiles. DCAT_ATTN_FLASH=1 selects the round-1 mma.sync
// kernel (attention.cu, row-major V) for comparisons.
bool use_tc_attention(const dcat_model* m, bool f32) {
    const int dh = m->cfg.d_model / m->cfg.n_heads;
    if (f32) return false;
    if (getenv("DCAT_ATTN_FLASH") != nullptr) return false;
    return attention_fa_supported(dh);
}

// dedup + validation; leaves the plan on the device and the counts in m->st_host
void run_dedup(dcat_model* m, const Staged& sb, const DedupOut& o, cudaStream_t s) {
    uint64_t mask = debug_hash_mask();
    const int kTileCtx = m->tile_ctx, kTileCross = m->tile_cross;
    const int t0 = mark(m, s);
    static const bool no_graph = getenv("DCAT_NO_DEDUP_GRAPH") != nullptr;
    if (no_graph) {
        dedup_plan(sb.in, o, mask, kTileCtx, kTileCross, s);
    } else {  // ~27 small launches replayed as one graph (captured on a private stream)
        dcat_model::DedupKey k;
        std::memset(&k, 0, sizeof k);
        k.in = sb.in;
        k.o = o;
        k.mask = mask;
        k.tile_ctx = kTileCtx;
        k.tile_cross = kTileCross;
        if (!m->dd_exec || std::memcmp(&k, &m->dd_key, sizeof k) != 0) {
            if (!m->cap) DCAT_CUDA_CHECK(cudaStreamCreateWithFlags(&m->cap, cudaStreamNonBlocking));
            if (m->dd_exec) {
                DCAT_CUDA_CHECK(cudaGraphExecDestroy(m->dd_exec));
                m->dd_exec = nullptr;
            }
            cudaGraph_t g = nullptr;
            DCAT_CUDA_CHECK(cudaStreamBeginCapture(m->cap, cudaStreamCaptureModeThreadLocal));
            dedup_plan(sb.in, o, mask, kTileCtx, kTileCross, m->cap);
            DCAT_CUDA_CHECK(cudaStreamEndCapture(m->cap, &g));
            DCAT_CUDA_CHECK(cudaGraphInstantiate(&m->dd_exec, g, 0));
            DCAT_CUDA_CHECK(cudaGraphDestroy(g));
            m->dd_key = k;
        }
        DCAT_CUDA_CHECK(cudaGraphLaunch(m->dd_exec, s));
    }
    m->stats.kernel_launches += 18;
    const int t1 = mark(m, s);
    DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
    DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
    span(m, "dedup.kernels", t0, t1);
    if (m->st_host->collisions > 0 && m->st_host->err_bits == 0) {
        dedup_repair(sb.in, o, m->st_host->collisions, kTileCtx, kTileCross, mask, s);
        m->stats.kernel_launches += 5 * 5 + 11;
        DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
    }
}

// ---------------------------------------------------------------- the pipeline
template <typename T>
struct Acts {
    T *E, *h1, *a, *q, *ctx, *f1, *kself, *vself, *feat;
    float *x, *hc, *logits_p, *mlog_p, *tmp;
    T* kv;  // [2 L] x Tp x d
    int64_t Tp, Bp;
};

template <typename T>
void gemm(dcat_model* m, const char* tag, const T* A, int lda, const Lin& L, int w_off, int N, int M, const Epi& e,
          float* tmp, cudaStream_t s) {
    if (M <= 0) return;
    NvtxRange nr(tag);
    int t0 = mark(m, s);
    if constexpr (std::is_same<T, bf16>::value) {
        gemm_tc(A, lda, L.wt + static_cast<size_t>(w_off) * L.in, L.in, M, N, L.in, e, s);
        m->stats.kernel_launches += 1;
    } else {
        gemm_f32(A, lda, L.w32 + w_off, L.out, M, N, L.in32, e, tmp, s);
        m->stats.kernel_launches += 2;
    }
    m->stats.gemm_launches += 1;
    m->stats.gemm_flops += 2.0 * M * N * L.in32;
    span(m, tag, t0, mark(m, s));
    static const bool debug_sync = getenv("DCAT_DEBUG_SYNC") != nullptr;  // debug: name the faulting GEMM
    if (debug_sync) {
        cudaError_t err = cudaStreamSynchronize(s);
        if (err != cudaSuccess)
            throw CudaError(std::string(tag) + " M=" + std::to_string(M) + " N=" + std::to_string(N) + " K=" +
                            std::to_string(L.in) + ": " + cudaGetErrorString(err));
    }
}

Epi base_epi(dcat_model* m, int mode, int layer_idx = -1) {
    Epi e;
    std::memset(&e, 0, sizeof e);
    e.mode = mode;
    e.st = m->st_dev;
    e.layer_idx = layer_idx;
    return e;
}

// FFN of a layer (model.cpp:386-397 / dcat.cpp:80-86): fused tcgen05 kernel when the
// shape allows (the d_ff-wide intermediate never leaves the SM), else FFN1 + FFN2 GEMMs.
// `fin` carries the residual / LN fields of the FFN2 epilogue.
template <typename T>
void ffn(dcat_model* m, const char* pass, const T* a, const LayerW& L, int M, Epi fin, T* f1, float* tmp,
         cudaStream_t s) {
    const int d = m->cfg.d_model, F = d * m->cfg.mlp_ratio;
    static const bool no_fuse = getenv("DCAT_NO_FUSED_FFN") != nullptr;
    if constexpr (std::is_same<T, bf16>::value) {
        if (!no_fuse && ffn_tc_supported(d, F)) {
            if (M <= 0) return;
            int t0 = mark(m, s);
            fin.bias = L.f1.bias;
            fin.b2 = L.f2.bias;
            ffn_tc(a, d, L.f1.wt, L.f2.wt, M, d, F, fin, s);
            m->stats.kernel_launches += 1;
            m->stats.gemm_launches += 1;
            m->stats.gemm_flops += 4.0 * M * F * d;
            span(m, pass[0] == 'c' && pass[1] == 't' ? "gemm.ctx.ffn" : "gemm.cross.ffn", t0, mark(m, s));
            return;
        }
    }
    Epi e = base_epi(m, EPI_BIAS);
    e.act = 1;
    e.bias = L.f1.bias;
    e.out[0] = f1;
    e.out_ld[0] = F;
    e.seg_cols = F;
    const bool ctx = pass[0] == 'c' && pass[1] == 't';
    gemm<T>(m, ctx ? "gemm.ctx.ffn1" : "gemm.cross.ffn1", a, d, L.f1, 0, F, M, e, tmp, s);
    fin.bias = L.f2.bias;
    gemm<T>(m, ctx ? "gemm.ctx.ffn2" : "gemm.cross.ffn2", f1, F, L.f2, 0, d, M, fin, tmp, s);
}

// The rest of a layer after attention (layer_forward model.cpp:378-397, cross_forward's tail
// dcat.cpp:80-86): x += attn_out . Wo + bo; x += FFN(LN2(x)); a = next LN1(x) (or a copy of x).
// bf16: one fused tcgen05 kernel (layer_tail_tc; DCAT_NO_TAIL_FUSION=1 selects the two-kernel
// path); otherwise the o-projection GEMM (writes x and LN2(x)) followed by ffn().
template <typename T>
void layer_tail(dcat_model* m, const char* pass, const T* attn_out, const LayerW& L, int l, int M, float* x, T* a,
                const float* next_g, const float* next_b, T* f1, float* tmp, cudaStream_t s) {
    const int d = m->cfg.d_model, F = d * m->cfg.mlp_ratio;
    const bool ctx = pass[0] == 'c' && pass[1] == 't';
    if constexpr (std::is_same<T, bf16>::value) {
        // read per call (a handful per pass) so tests can compare both paths in one process
        const bool two_kernels = getenv("DCAT_NO_TAIL_FUSION") != nullptr || getenv("DCAT_NO_FUSED_FFN") != nullptr;
        if (!two_kernels && layer_tail_tc_supported(d, F)) {
            if (M <= 0) return;
            NvtxRange nr(ctx ? "gemm.ctx.tail" : "gemm.cross.tail");
            int t0 = mark(m, s);
            Epi e = base_epi(m, EPI_RESID_LN, l);
            e.bias = L.f1.bias;
            e.b2 = L.f2.bias;
            e.o_bias = L.o.bias;
            e.ln2_g = L.ln2_g;
            e.ln2_b = L.ln2_b;
            e.resid = x;
            e.x_out = x;
            e.ld_x = d;
            e.ln_g = next_g;
            e.ln_b = next_b;
            e.ln_out = a;
            e.ln_ld = d;
            layer_tail_tc(attn_out, d, L.o.wt, L.f1.wt, L.f2.wt, M, d, F, e, s);
            m->stats.kernel_launches += 1;
            m->stats.gemm_launches += 1;
            m->stats.gemm_flops += 2.0 * M * d * d + 4.0 * M * F * d;
            span(m, ctx ? "gemm.ctx.tail" : "gemm.cross.tail", t0, mark(m, s));
            return;
        }
    }
    Epi e = base_epi(m, EPI_RESID_LN, l);
    e.bias = L.o.bias;
    e.resid = x;
    e.x_out = x;
    e.ld_x = d;
    e.ln_g = L.ln2_g;
    e.ln_b = L.ln2_b;
    e.ln_out = a;
    e.ln_ld = d;
    gemm<T>(m, ctx ? "gemm.ctx.o" : "gemm.cross.o", attn_out, d, L.o, 0, d, M, e, tmp, s);
    e = base_epi(m, EPI_RESID_LN, l);  // cross_tail's finite check (dcat.cpp:85-86)
    e.resid = x;
    e.x_out = x;
    e.ld_x = d;
    e.ln_g = next_g;
    e.ln_b = next_b;
    e.ln_out = a;
    e.ln_ld = d;
    ffn<T>(m, pass, a, L, M, e, f1, tmp, s);
}

template <typename T>
void attn(dcat_model* m, const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    NvtxRange nr(a.causal ? "attn.ctx" : "attn.cross");
    int t0 = mark(m, s);
    if constexpr (std::is_same<T, bf16>::value) {
        if (a.ldvt > 0) {
            attention_fa(a, q_rows, kv_rows, s);
        } else {
            attention_bf16(a, s);
        }
    } else {
        attention_f32(a, s);
    }
    m->stats.kernel_launches += 1;
    span(m, a.causal ? "attn.ctx" : "attn.cross", t0, mark(m, s));
}

// rank_forward_batch with the sequence module, every fusion variant (finetune.cpp:414-492):
//   Base / Aux: context pass (last layer K/V only), candidates cross the cached K/V;
//   LiteMean / LiteLast: full context pass + phi_out, selector = mean / last token row per unique
//     (the reference's model_forward per unique, :439-456), no crossing pass;
//   AuxLt: the learnable token is appended to every unique's context (its K/V enter the cache,
//     its final row through phi_out is the first selector) and candidates cross at position n + 1;
//     the reference computes the same per example (:428-431), here once per unique.
constexpr int64_t kDualStreamMaxRows = 65536;  // context / candidate rows (padded) below which run_dcat forks

// context_forward on its own (dcat_context_forward): the context pass only, its K/V left in the
// model's cache buffer; emit_hidden runs the last layer in full and, with h_user, writes
// phi_out of every context token (fp32, token order) to h_user (device)
struct CtxOnly {
    bool on = false;
    bool emit_hidden = false;
    float* h_user = nullptr;
};

// The crossing pass's transformer layers (cross_forward dcat.cpp:199-271 after phi_in): per layer
// QKV of the candidate rows (q, own k / v), attention over the unique's cached K / V plus itself,
// then the fused layer tail. kv = the cache base ([layer][K|V][Tp][d]), T_ctx = context tokens
// written, ldvt = V^T leading dimension (0: row-major V). Leaves the final rows in A.a (copy).
template <typename T>
void cross_layers(dcat_model* m, Acts<T>& A, int M, const Tile* cross_tiles, int n_tiles, bool sparse_tiles,
                  T* kv, int64_t Tp, int64_t T_ctx, int ldvt, const std::vector<char>* kv_done, cudaStream_t s) {
    const dcat_model_config& c = m->cfg;
    const int d = c.d_model, H = c.n_heads, dh = d / H, nl = c.n_layers;
    const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
    for (int l = 0; l < nl; l++) {
        const LayerW& L = m->layers[l];
        Epi e = base_epi(m, EPI_BIAS);
        e.bias = L.qkv.bias;
        e.out[0] = A.q;
        e.out[1] = A.kself;
        e.out[2] = A.vself;
        e.out_ld[0] = e.out_ld[1] = e.out_ld[2] = d;
        e.seg_cols = d;
        gemm<T>(m, "gemm.cross.qkv", A.a, d, L.qkv, 0, 3 * d, M, e, A.tmp, s);
        if (kv_done && (*kv_done)[l]) DCAT_CUDA_CHECK(cudaStreamWaitEvent(s, m->kv_ev[l], 0));
        T* K = kv + static_cast<size_t>(2 * l) * Tp * d;
        T* V = kv + static_cast<size_t>(2 * l + 1) * Tp * d;
        AttnArgs aa{A.q, d,  K,     V, d, ldvt, A.kself, A.vself, d, A.ctx, d, cross_tiles, n_tiles,
                    H,   dh, scale, 0, c.max_len + 1};
        aa.sparse_tiles = sparse_tiles;
        aa.dbg = m->dbg;
        attn<T>(m, aa, std::max(A.Tp, A.Bp), T_ctx, s);
        layer_tail<T>(m, "cross", A.ctx, L, l, M, A.x, A.a, l + 1 < nl ? m->layers[l + 1].ln1_g : nullptr,
                      l + 1 < nl ? m->layers[l + 1].ln1_b : nullptr, A.f1, A.tmp, s);  // last: copy for phi_out
    }
}

template <typename T>
void run_dcat(dcat_model* m, const Staged& sb, const DedupOut& o, const dcat_finetune_config& ft, float* logits,
              float* mlogits, float* h_cand, cudaStream_t s, const CtxOnly& co = CtxOnly()) {
    const dcat_model_config& c = m->cfg;
    const int d = c.d_model, de = c.d_emb, F = c.d_model * c.mlp_ratio, H = c.n_heads, dh = d / H, nl = c.n_layers;
    const Status& st = *m->st_host;
    const int b_u = st.b_u;
    const int64_t T_ctx = st.ctx_tokens, B = sb.in.B;
    const int64_t Tp = (T_ctx + 127) / 128 * 128, Bp = (B + 127) / 128 * 128, Rr = std::max(Tp, Bp);
    const bool f32 = std::is_same<T, float>::value;
    const int kh = f32 ? m->d_feat : m->kh;
    const bool lite = ft.variant == DCAT_VARIANT_LITE_MEAN || ft.variant == DCAT_VARIANT_LITE_LAST;
    const bool auxlt = ft.variant == DCAT_VARIANT_AUXLT;
    const bool full_last = lite || auxlt || co.emit_hidden;  // the context pass must emit the final hidden rows

    int t_stage0 = mark(m, s);
    span(m, "host.after_sync", m->t_dedup_end, t_stage0);
    // tiles + token map
    Tile* ctx_tiles = m->b_dd[20].get<Tile>(std::max(st.ctx_tiles, 1));
    Tile* cross_tiles = m->b_dd[21].get<Tile>(std::max(st.cross_tiles, 1));
    int32_t* tok_unique = m->b_dd[22].get<int32_t>(std::max<int64_t>(T_ctx, 1));
    build_tiles(sb.in, o, b_u, m->tile_ctx, m->tile_cross, ctx_tiles, cross_tiles, tok_unique, s);
    m->stats.kernel_launches += 2;
    // Two streams pay where the pass is launch-bound (small batches: tiny config 0.236 -> 0.204 ms).
    // At full-machine tile counts the persistent kernels already hold all SMs and the streams only
    // interleave (PinFM-base +0.4 %, high-fanout -2.3 %, low-dedup -1 %), so the default is by size;
    // DCAT_DUAL_STREAM=0 / 1 forces it.
    static const char* dual_env = getenv("DCAT_DUAL_STREAM");
    const bool dual_fit = dual_env ? dual_env[0] == '1' : Rr <= kDualStreamMaxRows;
    const bool dual = dual_fit && !co.on && !(ft.variant == DCAT_VARIANT_LITE_MEAN || ft.variant == DCAT_VARIANT_LITE_LAST);
    std::vector<char> kv_done(nl, 0);  // kv_ev[l] recorded in this call
    if (dual) {
        if (!m->xs) {
            DCAT_CUDA_CHECK(cudaStreamCreateWithFlags(&m->xs, cudaStreamNonBlocking));
            DCAT_CUDA_CHECK(cudaEventCreateWithFlags(&m->fork_ev, cudaEventDisableTiming));
            DCAT_CUDA_CHECK(cudaEventCreateWithFlags(&m->join_ev, cudaEventDisableTiming));
        }
        while (static_cast<int>(m->kv_ev.size()) < nl) {
            cudaEvent_t e;
            DCAT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            m->kv_ev.push_back(e);
        }
        DCAT_CUDA_CHECK(cudaEventRecord(m->fork_ev, s));  // plan + tiles are ready
    }
    auto kv_written = [&](int l) {
        if (!dual) return;
        DCAT_CUDA_CHECK(cudaEventRecord(m->kv_ev[l], s));
        kv_done[l] = 1;
    };
    // V cache layout: V^T [d][Tp] (keys contiguous) for the tcgen05 attention, else rows [Tp][d]
    const bool vt = m->vt;
    const int ldvt = vt ? static_cast<int>(Tp) : 0;

    Acts<T> A;
    A.Tp = Tp;
    A.Bp = Bp;
    A.E = m->b_act[0].get<T>(Rr * de);
    A.h1 = m->b_act[1].get<T>(Rr * d);
    A.a = m->b_act[2].get<T>(Rr * d);
    A.q = m->b_act[3].get<T>(Rr * d);
    A.ctx = m->b_act[4].get<T>(Rr * d);
    A.f1 = m->b_act[5].get<T>(Rr * F);
    A.kself = m->b_act[6].get<T>(Bp * d);
    A.vself = m->b_act[7].get<T>(Bp * d);
    A.feat = m->b_act[8].get<T>(Bp * kh);
    A.x = m->b_act[9].get<float>(Rr * d);
    A.hc = m->b_act[10].get<float>(Bp * d);
    A.logits_p = m->b_act[11].get<float>(Bp * 3);
    A.mlog_p = m->b_act[12].get<float>(Bp * 3);
    A.tmp = f32 ? m->b_act[13].get<float>(Rr * std::max(3 * d, std::max(F, m->hidden))) : nullptr;
    A.kv = m->b_kv.get<T>(std::max<int64_t>(2 * nl * Tp * d, 1));
    m->last_kv = A.kv;
    m->last_Tp = Tp;

    EmbParams ep{m->table, m->qtable,     m->qbits,       m->qrow_bytes, m->qcode_bytes, m->seed_mix, m->J,
                 m->R,     m->d_sub,      m->action_emb,  m->surface_emb, m->pos_emb,    de,          m->lt,
                 f32 ? nullptr : m->cmb, m->cfg.n_surfaces, m->cfg.max_len};
    const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
    auto K_l = [&](int l) { return A.kv + static_cast<size_t>(2 * l) * Tp * d; };
    auto V_l = [&](int l) { return A.kv + static_cast<size_t>(2 * l + 1) * Tp * d; };

    // ============ context pass (context_forward, emit_hidden = false) ============
    int t_ctx0 = mark(m, s);
    if (T_ctx > 0) {
        const int M = static_cast<int>(T_ctx);
        gather_context<T>(sb.in, o, ep, tok_unique, T_ctx, A.E, de, s);
        m->stats.kernel_launches += 1;
        // phi_in (model.cpp:144-161) -> x, then LN1 of layer 0
        Epi e = base_epi(m, EPI_BIAS);
        e.act = 1;
        e.bias = m->phi_in1.bias;
        e.out[0] = A.h1;
        e.out_ld[0] = d;
        e.seg_cols = d;
        gemm<T>(m, "gemm.ctx.phi_in1", A.E, de, m->phi_in1, 0, d, M, e, A.tmp, s);
        e = base_epi(m, EPI_L2NORM);
        e.bias = m->phi_in2.bias;
        e.x_out = A.x;
        e.ld_x = d;
        e.ln_g = m->layers[0].ln1_g;
        e.ln_b = m->layers[0].ln1_b;
        e.ln_out = A.a;
        e.ln_ld = d;
        gemm<T>(m, "gemm.ctx.phi_in2", A.h1, d, m->phi_in2, 0, d, M, e, A.tmp, s);
        for (int l = 0; l < nl; l++) {
            const LayerW& L = m->layers[l];
            if (l == nl - 1 && !full_last) {  // kv_only (dcat.cpp:60-65): K, V of the final layer
                e = base_epi(m, EPI_BIAS);
                e.bias = L.qkv.bias + d;
                e.out[0] = K_l(l);
                e.out[1] = V_l(l);
                e.out_ld[0] = d;
                e.out_ld[1] = vt ? static_cast<int>(Tp) : d;
                e.out_trans[1] = vt;
                e.seg_cols = d;
                gemm<T>(m, "gemm.ctx.kv", A.a, d, L.qkv, d, 2 * d, M, e, A.tmp, s);
                kv_written(l);
                break;
            }
            // layer_forward (model.cpp:336-398); K, V go straight to the cache
            e = base_epi(m, EPI_BIAS);
            e.bias = L.qkv.bias;
            e.out[0] = A.q;
            e.out[1] = K_l(l);
            e.out[2] = V_l(l);
            e.out_ld[0] = e.out_ld[1] = d;
            e.out_ld[2] = vt ? static_cast<int>(Tp) : d;
            e.out_trans[2] = vt;
            e.seg_cols = d;
            gemm<T>(m, "gemm.ctx.qkv", A.a, d, L.qkv, 0, 3 * d, M, e, A.tmp, s);
            kv_written(l);
            AttnArgs aa{A.q,     d,  K_l(l), V_l(l), d, ldvt, nullptr, nullptr, 0, A.ctx, d, ctx_tiles, st.ctx_tiles,
                        H,       dh, scale,  1,      c.max_len + 1};
            aa.dbg = m->dbg;
            attn<T>(m, aa, Rr, T_ctx, s);
            layer_tail<T>(m, "ctx", A.ctx, L, l, M, A.x, A.a, l + 1 < nl ? m->layers[l + 1].ln1_g : nullptr,
                          l + 1 < nl ? m->layers[l + 1].ln1_b : nullptr, A.f1, A.tmp, s);  // emitted rows: copy
        }
    }
    if (co.on) {  // context_forward alone: K/V stay in the cache; h_user = phi_out of every token
        if (co.emit_hidden && co.h_user && T_ctx > 0) {
            Epi e = base_epi(m, EPI_BIAS);
            e.act = 1;
            e.bias = m->phi_out1.bias;
            e.out[0] = A.h1;
            e.out_ld[0] = d;
            e.seg_cols = d;
            gemm<T>(m, "gemm.ctx.phi_out1", A.a, d, m->phi_out1, 0, d, static_cast<int>(T_ctx), e, A.tmp, s);
            e = base_epi(m, EPI_L2NORM);
            e.bias = m->phi_out2.bias;
            e.x_out = co.h_user;
            e.ld_x = d;
            gemm<T>(m, "gemm.ctx.phi_out2", A.h1, d, m->phi_out2, 0, d, static_cast<int>(T_ctx), e, A.tmp, s);
        }
        span(m, "context", t_ctx0, mark(m, s));
        return;
    }
    // per-unique selector rows (fp32 b_u x d): Lite pools phi_out(H) over a unique's tokens,
    // AuxLt takes phi_out of its learnable token (the unique's last context row)
    float* sel = nullptr;
    if (full_last) {
        sel = m->b_act[14].get<float>(static_cast<size_t>(std::max(b_u, 1)) * d);
        const T* src = A.a;
        int rows = static_cast<int>(T_ctx);
        if (auxlt) {
            T* lt_rows = m->b_act[15].get<T>(static_cast<size_t>(std::max(b_u, 1)) * d);
            gather_last_rows<T>(o.tok_off, b_u, A.a, d, lt_rows, s);
            m->stats.kernel_launches += 1;
            src = lt_rows;
            rows = b_u;
        }
        Epi e = base_epi(m, EPI_BIAS);
        e.act = 1;
        e.bias = m->phi_out1.bias;
        e.out[0] = A.h1;
        e.out_ld[0] = d;
        e.seg_cols = d;
        gemm<T>(m, "gemm.ctx.phi_out1", src, d, m->phi_out1, 0, d, rows, e, A.tmp, s);
        e = base_epi(m, EPI_L2NORM);
        e.bias = m->phi_out2.bias;
        e.x_out = lite ? A.x : sel;
        e.ld_x = d;
        gemm<T>(m, "gemm.ctx.phi_out2", A.h1, d, m->phi_out2, 0, d, rows, e, A.tmp, s);
        if (lite) {
            pool_selectors(o.tok_off, b_u, A.x, d, ft.variant == DCAT_VARIANT_LITE_LAST, sel, s);
            m->stats.kernel_launches += 1;
        }
    }
    int t_ctx1 = mark(m, s);
    if (lite) {  // candidate-independent selector: no crossing pass (finetune.cpp:439-456)
        CandParams cp{sb.candidate, sb.age, sb.aux, m->aux_proj, m->d_aux, 0, ft.max_events, ft.fresh_days,
                      ft.mid_days, m->d_module, kh, 0};
        wait_cand(sb, s);
        gather_candidates<T>(sb.in, o, ep, cp, B, A.E, de, A.feat, s);
        broadcast_selectors<T>(o.perm, o.rep, B, sel, d, A.feat, kh, 0, h_cand ? A.hc : nullptr, s);
        module_logits(o.perm, o.rep, B, sel, nullptr, d, m->mod_w, m->mod_b, A.mlog_p, s);
        m->stats.kernel_launches += 3;
        int t_cross1 = mark(m, s);
        Epi e = base_epi(m, EPI_HEAD);
        e.bias = m->head1.bias;
        e.w2 = m->hw2;
        e.b2 = m->hb2;
        e.logits = A.logits_p;
        gemm<T>(m, "gemm.head", A.feat, kh, m->head1, 0, m->hidden, static_cast<int>(B), e, A.tmp, s);
        scatter_outputs(o.perm, B, A.logits_p, A.mlog_p, h_cand ? A.hc : nullptr, d, logits, mlogits, h_cand, s);
        m->stats.kernel_launches += 1;
        int t_end = mark(m, s);
        span(m, "plan", t_stage0, t_ctx0);
        span(m, "context", t_ctx0, t_ctx1);
        span(m, "head", t_cross1, t_end);
        return;
    }

    // ============ crossing pass (candidate_inputs + cross_forward) ============
    const int M = static_cast<int>(B);
    const cudaStream_t s_main = s;
    if (dual) {  // own activation buffers (Rr rows: the attention's TMA maps span Rr), own stream, forked at the plan
        DCAT_CUDA_CHECK(cudaStreamWaitEvent(m->xs, m->fork_ev, 0));
        s = m->xs;
        A.E = m->b_act[20].get<T>(Rr * de);
        A.h1 = m->b_act[21].get<T>(Rr * d);
        A.a = m->b_act[22].get<T>(Rr * d);
        A.q = m->b_act[23].get<T>(Rr * d);
        A.ctx = m->b_act[24].get<T>(Rr * d);
        A.f1 = m->b_act[25].get<T>(Rr * F);
        A.x = m->b_act[26].get<float>(Rr * d);
        A.tmp = f32 ? m->b_act[27].get<float>(Rr * std::max(3 * d, std::max(F, m->hidden))) : nullptr;
    }
    CandParams cp{sb.candidate, sb.age, sb.aux, m->aux_proj, m->d_aux,
                  ft.variant == DCAT_VARIANT_AUX || ft.variant == DCAT_VARIANT_AUXLT,
                  ft.max_events, ft.fresh_days, ft.mid_days, m->d_module, kh, auxlt ? 1 : 0};
    wait_cand(sb, s);
    gather_candidates<T>(sb.in, o, ep, cp, B, A.E, de, A.feat, s);
    m->stats.kernel_launches += 1;
    Epi e = base_epi(m, EPI_BIAS);
    e.act = 1;
    e.bias = m->phi_in1.bias;
    e.out[0] = A.h1;
    e.out_ld[0] = d;
    e.seg_cols = d;
    gemm<T>(m, "gemm.cross.phi_in1", A.E, de, m->phi_in1, 0, d, M, e, A.tmp, s);
    e = base_epi(m, EPI_L2NORM);
    e.bias = m->phi_in2.bias;
    e.x_out = A.x;
    e.ld_x = d;
    e.ln_g = m->layers[0].ln1_g;
    e.ln_b = m->layers[0].ln1_b;
    e.ln_out = A.a;
    e.ln_ld = d;
    gemm<T>(m, "gemm.cross.phi_in2", A.h1, d, m->phi_in2, 0, d, M, e, A.tmp, s);
    cross_layers<T>(m, A, M, cross_tiles, st.cross_tiles, B < static_cast<int64_t>(st.cross_tiles) * (m->tile_cross / 2),
                    A.kv, Tp, T_ctx, ldvt, dual ? &kv_done : nullptr, s);
    if (dual) {  // join: the rest reads the context pass's selectors and goes out on the caller's stream
        DCAT_CUDA_CHECK(cudaEventRecord(m->join_ev, s));
        DCAT_CUDA_CHECK(cudaStreamWaitEvent(s_main, m->join_ev, 0));
        s = s_main;
    }
    // phi_out (dcat.cpp:266) + module head (finetune.cpp:317-323)
    e = base_epi(m, EPI_BIAS);
    e.act = 1;
    e.bias = m->phi_out1.bias;
    e.out[0] = A.h1;
    e.out_ld[0] = d;
    e.seg_cols = d;
    gemm<T>(m, "gemm.cross.phi_out1", A.a, d, m->phi_out1, 0, d, M, e, A.tmp, s);
    e = base_epi(m, EPI_L2NORM);
    e.bias = m->phi_out2.bias;
    e.x_out = h_cand || auxlt ? A.hc : nullptr;
    e.ld_x = d;
    e.out2 = auxlt ? A.feat + d : A.feat;  // H_cand: feat columns [0, d) (AuxLt: [d, 2d), after H_lt)
    e.out2_ld = kh;
    e.mod_w = auxlt ? nullptr : m->mod_w;
    e.mod_b = m->mod_b;
    e.mlogits = A.mlog_p;
    gemm<T>(m, "gemm.cross.phi_out2", A.h1, d, m->phi_out2, 0, d, M, e, A.tmp, s);
    if (auxlt) {  // selectors [H_lt | H_cand] (gather_selectors, finetune.cpp:251-256)
        broadcast_selectors<T>(o.perm, o.rep, B, sel, d, A.feat, kh, 0, nullptr, s);
        module_logits(o.perm, o.rep, B, sel, A.hc, d, m->mod_w, m->mod_b, A.mlog_p, s);
        m->stats.kernel_launches += 2;
    }
    int t_cross1 = mark(m, s);
    // ranking head: crossing MLP on [H_cand | cand_emb | ctx] (finetune.cpp:301-316)
    e = base_epi(m, EPI_HEAD);
    e.bias = m->head1.bias;
    e.w2 = m->hw2;
    e.b2 = m->hb2;
    e.logits = A.logits_p;
    gemm<T>(m, "gemm.head", A.feat, kh, m->head1, 0, m->hidden, M, e, A.tmp, s);
    scatter_outputs(o.perm, B, A.logits_p, A.mlog_p, h_cand ? A.hc : nullptr, d, logits, mlogits, h_cand, s);
    m->stats.kernel_launches += 1;
    int t_end = mark(m, s);
    span(m, "plan", t_stage0, t_ctx0);
    span(m, "context", t_ctx0, t_ctx1);
    span(m, "cross", t_ctx1, t_cross1);
    span(m, "head", t_cross1, t_end);
}

// use_seq_module = false: crossing MLP on [cand_emb | ctx] only (finetune.cpp:342-347)
template <typename T>
void run_head_only(dcat_model* m, const Staged& sb, const DedupOut& o, const dcat_finetune_config& ft,
                   float* logits, float* mlogits, cudaStream_t s) {
    const int64_t B = sb.in.B, Bp = (B + 127) / 128 * 128;
    const bool f32 = std::is_same<T, float>::value;
    const int kh = f32 ? m->d_feat : m->kh;
    T* feat = m->b_act[8].get<T>(Bp * kh);
    T* E = m->b_act[0].get<T>(Bp * m->cfg.d_emb);
    float* logits_p = m->b_act[11].get<float>(Bp * 3);
    float* mlog_p = m->b_act[12].get<float>(Bp * 3);
    float* tmp = f32 ? m->b_act[13].get<float>(Bp * m->hidden) : nullptr;
    EmbParams ep{m->table, m->qtable, m->qbits, m->qrow_bytes, m->qcode_bytes, m->seed_mix, m->J, m->R, m->d_sub,
                 m->action_emb, m->surface_emb, m->pos_emb,
                 m->cfg.d_emb, m->lt, nullptr, m->cfg.n_surfaces, m->cfg.max_len};
    CandParams cp{sb.candidate, sb.age, nullptr, m->aux_proj, 0, 0, ft.max_events, ft.fresh_days, ft.mid_days,
                  0, kh, 0};
    wait_cand(sb, s);
    gather_candidates<T>(sb.in, o, ep, cp, B, E, m->cfg.d_emb, feat, s);
    m->stats.kernel_launches += 1;
    Epi e = base_epi(m, EPI_HEAD);
    e.bias = m->head1.bias;
    e.w2 = m->hw2;
    e.b2 = m->hb2;
    e.logits = logits_p;
    gemm<T>(m, "gemm.head", feat, kh, m->head1, 0, m->hidden, static_cast<int>(B), e, tmp, s);
    std::vector<float> mb(static_cast<size_t>(Bp) * 3);
    float hb[3];
    DCAT_CUDA_CHECK(cudaMemcpy(hb, m->mod_b, sizeof hb, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < Bp; i++)
        for (int j = 0; j < 3; j++) mb[i * 3 + j] = hb[j];
    DCAT_CUDA_CHECK(cudaMemcpyAsync(mlog_p, mb.data(), mb.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
    scatter_outputs(o.perm, B, logits_p, mlog_p, nullptr, 0, logits, mlogits, nullptr, s);
    m->stats.kernel_launches += 1;
}

int validate_ft(const dcat_model* m, const dcat_finetune_config* ft, const dcat_batch* b) {
    // FinetuneConfig::validate (finetune.cpp:54-72) + ColdStartConfig::validate (:41-47)
    if (ft->variant < DCAT_VARIANT_BASE || ft->variant > DCAT_VARIANT_LITE_LAST)
        return set_err(DCAT_EINVAL, "unknown fusion variant");
    if (!(ft->fresh_days > 0.0 && ft->fresh_days < ft->mid_days))
        return set_err(DCAT_EINVAL, "age bands must satisfy 0 < fresh_days < mid_days");
    if (ft->max_events < 0) return set_err(DCAT_EINVAL, "max_events must be >= 0");
    // context_forward_fixed (dcat.cpp:285): window >= 1 when the fixed-window variant is on
    if (ft->window < 0) return set_err(DCAT_EINVAL, "context_forward_fixed: window must be >= 1, got " +
                                                         std::to_string(ft->window));
    if (m->cfg.max_len < ft->max_events + 2)
        return set_err(DCAT_EINVAL, "model.max_len " + std::to_string(m->cfg.max_len) + " too small for max_events " +
                                        std::to_string(ft->max_events) + " plus candidate tokens");
    if (!ft->use_seq_module && ft->variant != DCAT_VARIANT_BASE)
        return set_err(DCAT_EINVAL, "disabling the sequence module requires the base variant");
    // selector rows per variant (gather_selectors, finetune.cpp:243-274): AuxLt two, else one
    const int sel_rows = ft->variant == DCAT_VARIANT_AUXLT ? 2 : 1;
    if (ft->use_seq_module && m->d_module != sel_rows * m->cfg.d_model)
        return set_err(DCAT_EINVAL, "ranking head d_module does not match the sequence module width");
    if (ft->use_seq_module && ft->variant == DCAT_VARIANT_AUXLT && ft->window > 0)
        return set_err(DCAT_EINVAL, "the fixed-window module has no learnable token (AuxLt)");
    if (!ft->use_seq_module && m->d_module != 0)
        return set_err(DCAT_EINVAL, "ranking head expects module outputs but use_seq_module is off");
    if (ft->use_seq_module && (ft->variant == DCAT_VARIANT_AUX || ft->variant == DCAT_VARIANT_AUXLT)) {
        if (!b->aux || b->d_aux <= 0) return set_err(DCAT_EINVAL, "variant 'aux' requires an auxiliary embedding");
        if (b->d_aux != m->d_aux) return set_err(DCAT_EINVAL, "aux dim mismatch in batch");
    }
    if (ft->use_seq_module && m->cfg.n_layers < 1)
        return set_err(DCAT_EINVAL, "context_forward: needs at least one layer");
    return DCAT_OK;
}

template <typename F>
int guarded(dcat_model* m, F&& f) {
    try {
        g_err.clear();
        DeviceGuard dg(m ? m->device : -1);
        return f();
    } catch (const CudaError& e) {
        return set_err(DCAT_ECUDA, e.msg);
    } catch (const InvalidArg& e) {
        return set_err(DCAT_EINVAL, e.msg);
    } catch (const std::bad_alloc&) {
        return set_err(DCAT_ENOMEM, "host out of memory");
    }
}

// K and V rows [a, b) of one layer from a cache buffer (layout of run_dcat's A.kv) -> fp32 host
void read_kv_rows(const void* buf, bool vt, bool f32, int64_t Tp, int d, int layer, int64_t a, int64_t b, float* k,
                  float* v) {
    const size_t cnt = static_cast<size_t>(b - a) * d;
    for (int which = 0; which < 2; which++) {
        float* dst = which ? v : k;
        if (!dst) continue;
        const size_t base = (static_cast<size_t>(2 * layer + which) * Tp + a) * d;
        if (which == 1 && vt) {  // V^T [d][Tp]: gather the unique's key columns
            const size_t vbase = static_cast<size_t>(2 * layer + 1) * Tp * d;
            std::vector<bf16> tmp(static_cast<size_t>(d) * Tp);
            DCAT_CUDA_CHECK(cudaMemcpy(tmp.data(), static_cast<const bf16*>(buf) + vbase, tmp.size() * 2,
                                       cudaMemcpyDeviceToHost));
            for (int64_t t = 0; t < b - a; t++)
                for (int i = 0; i < d; i++) dst[t * d + i] = __bfloat162float(tmp[static_cast<size_t>(i) * Tp + a + t]);
            continue;
        }
        if (f32) {
            DCAT_CUDA_CHECK(cudaMemcpy(dst, static_cast<const float*>(buf) + base, cnt * 4, cudaMemcpyDeviceToHost));
        } else {
            std::vector<bf16> tmp(cnt);
            DCAT_CUDA_CHECK(cudaMemcpy(tmp.data(), static_cast<const bf16*>(buf) + base, cnt * 2, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < cnt; i++) dst[i] = __bfloat162float(tmp[i]);
        }
    }
}

EmbParams emb_params(const dcat_model* m, bool f32) {
    return EmbParams{m->table, m->qtable,     m->qbits,       m->qrow_bytes,  m->qcode_bytes, m->seed_mix, m->J,
                     m->R,     m->d_sub,      m->action_emb,  m->surface_emb, m->pos_emb,     m->cfg.d_emb, m->lt,
                     f32 ? nullptr : m->cmb, m->cfg.n_surfaces, m->cfg.max_len};
}

// cross_forward on a device cache (dcat_cross_forward): the candidate rows grouped by unique
// (perm / tiles built on the host from rep), phi_in, the crossing layers, phi_out -> h (device,
// caller row order)
template <typename T>
void run_cross_external(dcat_model* m, const dcat_kv* kv, const std::vector<int32_t>& du, const float* e_dev,
                        float* h_dev, cudaStream_t s) {
    const dcat_model_config& c = m->cfg;
    const int d = c.d_model, de = c.d_emb, F = d * c.mlp_ratio;
    const int64_t B = static_cast<int64_t>(du.size()), Bp = (B + 127) / 128 * 128;
    const int64_t Rr = std::max(kv->Tp, Bp);
    const int b_u = static_cast<int>(kv->tok_off.size()) - 1;
    // counting sort of the rows by unique (stable), 128-row crossing tiles per unique
    std::vector<int32_t> cnt(static_cast<size_t>(b_u) + 1, 0), perm(static_cast<size_t>(B));
    for (int32_t u : du) cnt[static_cast<size_t>(u)]++;
    std::vector<int64_t> goff(static_cast<size_t>(b_u) + 1, 0);
    for (int u = 0; u < b_u; u++) goff[u + 1] = goff[u] + cnt[u];
    std::vector<int64_t> cur(goff.begin(), goff.end() - 1);
    for (int64_t b = 0; b < B; b++) perm[static_cast<size_t>(cur[du[b]]++)] = static_cast<int32_t>(b);
    std::vector<Tile> tiles;
    for (int u = 0; u < b_u; u++)
        for (int64_t j = 0; j * 128 < cnt[u]; j++) {
            Tile t{};
            t.q0 = static_cast<int>(goff[u] + j * 128);
            t.nq = static_cast<int>(std::min<int64_t>(128, cnt[u] - j * 128));
            t.kv0 = static_cast<int>(kv->tok_off[u]);
            t.nkv = static_cast<int>(kv->tok_off[u + 1] - kv->tok_off[u]);
            t.u = u;
            tiles.push_back(t);
        }
    int32_t* perm_d = m->b_x[1].get<int32_t>(B);
    Tile* tiles_d = m->b_x[2].get<Tile>(std::max<size_t>(tiles.size(), 1));
    DCAT_CUDA_CHECK(cudaMemcpyAsync(perm_d, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, s));
    DCAT_CUDA_CHECK(cudaMemcpyAsync(tiles_d, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice, s));
    const bool f32 = std::is_same<T, float>::value;
    Acts<T> A;
    A.Tp = kv->Tp;
    A.Bp = Bp;
    A.E = m->b_act[0].get<T>(Rr * de);
    A.h1 = m->b_act[1].get<T>(Rr * d);
    A.a = m->b_act[2].get<T>(Rr * d);
    A.q = m->b_act[3].get<T>(Rr * d);
    A.ctx = m->b_act[4].get<T>(Rr * d);
    A.f1 = m->b_act[5].get<T>(Rr * F);
    A.kself = m->b_act[6].get<T>(Bp * d);
    A.vself = m->b_act[7].get<T>(Bp * d);
    A.x = m->b_act[9].get<float>(Rr * d);
    A.hc = m->b_act[10].get<float>(Bp * d);
    A.tmp = f32 ? m->b_act[13].get<float>(Rr * std::max(3 * d, std::max(F, m->hidden))) : nullptr;
    gather_rows<T>(e_dev, perm_d, B, de, A.E, s);
    m->stats.kernel_launches += 1;
    const int M = static_cast<int>(B);
    Epi e = base_epi(m, EPI_BIAS);
    e.act = 1;
    e.bias = m->phi_in1.bias;
    e.out[0] = A.h1;
    e.out_ld[0] = d;
    e.seg_cols = d;
    gemm<T>(m, "gemm.cross.phi_in1", A.E, de, m->phi_in1, 0, d, M, e, A.tmp, s);
    e = base_epi(m, EPI_L2NORM);
    e.bias = m->phi_in2.bias;
    e.x_out = A.x;
    e.ld_x = d;
    e.ln_g = m->layers[0].ln1_g;
    e.ln_b = m->layers[0].ln1_b;
    e.ln_out = A.a;
    e.ln_ld = d;
    gemm<T>(m, "gemm.cross.phi_in2", A.h1, d, m->phi_in2, 0, d, M, e, A.tmp, s);
    cross_layers<T>(m, A, M, tiles_d, static_cast<int>(tiles.size()), B < static_cast<int64_t>(tiles.size()) * 64,
                    static_cast<T*>(kv->buf), kv->Tp, kv->T_ctx, kv->vt ? static_cast<int>(kv->Tp) : 0, nullptr, s);
    e = base_epi(m, EPI_BIAS);
    e.act = 1;
    e.bias = m->phi_out1.bias;
    e.out[0] = A.h1;
    e.out_ld[0] = d;
    e.seg_cols = d;
    gemm<T>(m, "gemm.cross.phi_out1", A.a, d, m->phi_out1, 0, d, M, e, A.tmp, s);
    e = base_epi(m, EPI_L2NORM);
    e.bias = m->phi_out2.bias;
    e.x_out = A.hc;
    e.ld_x = d;
    gemm<T>(m, "gemm.cross.phi_out2", A.h1, d, m->phi_out2, 0, d, M, e, A.tmp, s);
    scatter_rows(A.hc, perm_d, B, d, h_dev, s);
    m->stats.kernel_launches += 1;
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

const char* dcat_last_error(void) { return g_err.c_str(); }
const char* dcat_version(void) { return "dcat_b200 0.1 (sm_100a)"; }

int dcat_model_create(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                      const dcat_head* head, int32_t device, dcat_model** out) {
    if (!cfg || !params || !table || !head || !out) return set_err(DCAT_EINVAL, "null argument");
    *out = nullptr;
    std::unique_ptr<dcat_model> m(new dcat_model());
    return guarded(nullptr, [&]() -> int {
        const dcat_model_config& c = *cfg;
        // ModelConfig::validate (model.cpp:175-183)
        if (!(c.d_model >= 1 && c.n_heads >= 1 && c.d_model % c.n_heads == 0))
            return set_err(DCAT_EINVAL, "d_model must be divisible by n_heads");
        if (c.n_layers < 0 || c.mlp_ratio < 1 || c.max_len < 1 || c.d_emb < 1)
            return set_err(DCAT_EINVAL, "invalid model config");
        int expect = 3 + (c.pos_learned ? 1 : 0) + 12 + 16 * c.n_layers;
        if (params->n_tensors != expect)
            return set_err(DCAT_EINVAL, "params: expected " + std::to_string(expect) + " tensors, got " +
                                            std::to_string(params->n_tensors));
        if (table->num_subtables * table->d_sub != c.d_emb)
            return set_err(DCAT_EINVAL, "segment_inputs: id source dim mismatch");
        int dh = c.d_model / c.n_heads;
        if (!(dh < 16 || dh == 16 || dh == 32 || dh == 64))
            return set_err(DCAT_EUNSUPPORTED, "head dim " + std::to_string(dh) + " not supported (<16, 16, 32, 64)");
        if (c.d_model % 16 || c.d_emb % 8)
            return set_err(DCAT_EUNSUPPORTED, "d_model must be a multiple of 16 and d_emb of 8");
        m->device = device;
        DeviceGuard dg(device);
        m->cfg = c;
        const float* const* t = params->tensors;
        int k = 1;
        m->action_emb = m->mem.upload(t[k++], static_cast<size_t>(c.n_actions) * c.d_emb);
        m->surface_emb = m->mem.upload(t[k++], static_cast<size_t>(c.n_surfaces) * c.d_emb);
        m->pos_emb = c.pos_learned ? m->mem.upload(t[k++], static_cast<size_t>(c.max_len) * c.d_emb) : nullptr;
        const size_t n_cmb = static_cast<size_t>(c.n_actions) * c.n_surfaces * c.max_len * c.d_emb;
        if (m->pos_emb && c.d_emb % 4 == 0 && n_cmb * 4 <= (64u << 20)) {  // <= 64 MB (7.4 MB at PinFM-base)
            DCAT_CUDA_CHECK(cudaMalloc(&m->cmb, n_cmb * 4));
            m->mem.ptrs.push_back(m->cmb);
            build_combined_emb(m->action_emb, m->surface_emb, m->pos_emb, c.n_actions, c.n_surfaces, c.max_len,
                               c.d_emb, m->cmb, nullptr);
            DCAT_CUDA_CHECK(cudaDeviceSynchronize());
        }
        int d = c.d_model, F = d * c.mlp_ratio;
        m->phi_in1 = make_lin(m->mem, t[k], t[k + 1], c.d_emb, d);
        m->phi_in2 = make_lin(m->mem, t[k + 2], t[k + 3], d, d);
        m->phi_out1 = make_lin(m->mem, t[k + 4], t[k + 5], d, d);
        m->phi_out2 = make_lin(m->mem, t[k + 6], t[k + 7], d, d);
        k += 12;  // psi is not on the scoring path
        for (int l = 0; l < c.n_layers; l++) {
            const float* const* L = t + k + 16 * l;
            LayerW w;
            w.ln1_g = m->mem.upload(L[0], d);
            w.ln1_b = m->mem.upload(L[1], d);
            w.qkv = make_qkv(m->mem, L[2], L[3], L[4], L[5], L[6], L[7], d);
            w.o = make_lin(m->mem, L[8], L[9], d, d);
            w.ln2_g = m->mem.upload(L[10], d);
            w.ln2_b = m->mem.upload(L[11], d);
            w.f1 = make_lin(m->mem, L[12], L[13], d, F);
            w.f2 = make_lin(m->mem, L[14], L[15], F, d);
            m->layers.push_back(w);
        }
        // hashed id table (embed.cpp:16-43)
        m->J = table->num_subtables;
        m->R = table->rows;
        m->d_sub = table->d_sub;
        if (table->bits != 0) {  // QuantizedTable (embed.hpp:80-125)
            if (table->bits != 4 && table->bits != 8)
                return set_err(DCAT_EINVAL, "quantized table: unsupported bit width " + std::to_string(table->bits));
            if (!table->packed) return set_err(DCAT_EINVAL, "quantized table: packed rows missing");
            m->qbits = table->bits;
            m->qcode_bytes = (m->d_sub * m->qbits + 7) / 8;
            m->qrow_bytes = m->qcode_bytes + 4;  // + fp16 scale + fp16 bias
            m->qtable = m->mem.upload(table->packed, static_cast<size_t>(m->J) * m->R * m->qrow_bytes);
        } else {
            std::vector<float> tab(static_cast<size_t>(m->J) * m->R * m->d_sub);
            for (int j = 0; j < m->J; j++)
                std::memcpy(tab.data() + static_cast<size_t>(j) * m->R * m->d_sub, table->subtables[j],
                            sizeof(float) * m->R * m->d_sub);
            m->table = m->mem.upload(tab.data(), tab.size());
        }
        std::vector<uint64_t> sm(m->J);
        for (int j = 0; j < m->J; j++) sm[j] = host_mix64(table->seeds[j]);
        m->seed_mix = m->mem.upload(sm.data(), sm.size());
        // ranking head (finetune.hpp:70-85)
        m->d_module = head->d_module;
        m->head_demb = head->d_emb;
        m->n_ctx = head->n_ctx;
        m->hidden = head->hidden;
        m->d_aux = head->d_aux;
        if (head->d_emb != c.d_emb || head->n_ctx != 8)
            return set_err(DCAT_EINVAL, "ranking head shape does not match the model (d_emb, n_ctx = 8)");
        if (m->d_module != 0 && m->d_module != d && m->d_module != 2 * d)
            return set_err(DCAT_EINVAL, "ranking head d_module must be 0, d_model or 2 d_model (AuxLt)");
        if (m->hidden < 1 || m->hidden > 256) return set_err(DCAT_EUNSUPPORTED, "crossing hidden must be in [1, 256]");
        m->d_feat = m->d_module + head->d_emb + head->n_ctx;
        m->kh = (m->d_feat + 63) / 64 * 64;
        m->head1 = make_lin(m->mem, head->w1, head->b1, m->d_feat, m->hidden, m->kh);
        m->head1.in = m->kh;  // bf16 operand is zero-padded to kh columns
        m->hw2 = m->mem.upload(head->w2, static_cast<size_t>(m->hidden) * 3);
        m->hb2 = m->mem.upload(head->b2, 3);
        std::vector<float> zero3(3 * std::max(1, m->d_module), 0.0f);
        m->mod_w = m->d_module ? m->mem.upload(head->mod_w, static_cast<size_t>(m->d_module) * 3) : nullptr;
        m->mod_b = m->mem.upload(head->mod_b ? head->mod_b : zero3.data(), 3);
        std::vector<float> za(static_cast<size_t>(std::max(1, m->d_aux)) * c.d_emb, 0.0f);
        m->aux_proj = m->mem.upload(head->aux_proj && m->d_aux ? head->aux_proj : za.data(), za.size());
        std::vector<float> zl(static_cast<size_t>(c.d_emb), 0.0f);
        m->lt = m->mem.upload(head->lt ? head->lt : zl.data(), zl.size());  // AuxLt learnable token
        DCAT_CUDA_CHECK(cudaMalloc(&m->st_dev, sizeof(Status)));
        m->mem.ptrs.push_back(m->st_dev);
        DCAT_CUDA_CHECK(cudaMallocHost(&m->st_host, sizeof(Status)));
        if (getenv("DCAT_DEBUG_COUNTERS") != nullptr) {
            DCAT_CUDA_CHECK(cudaMalloc(&m->dbg, kDebugCounters * sizeof(unsigned)));
            m->mem.ptrs.push_back(m->dbg);
            DCAT_CUDA_CHECK(cudaMemset(m->dbg, 0, kDebugCounters * sizeof(unsigned)));
        }
        *out = m.release();
        return DCAT_OK;
    });
}

int dcat_model_destroy(dcat_model* m) {
    if (!m) return DCAT_OK;
    DeviceScopeNoThrow ds(m->device);
    cudaDeviceSynchronize();
    delete m;
    return DCAT_OK;
}

int dcat_dedup(dcat_model* m, const dcat_batch* batch, int32_t* rep, int32_t* first, int32_t* b_u, int32_t flags,
               void* stream) {
    if (!m || !batch || !rep || !b_u) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        NvtxRange nr("dcat_dedup");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        bool device = flags & DCAT_INPUT_DEVICE;
        int64_t B = batch->n_rows;
        *b_u = 0;
        if (B == 0) return DCAT_OK;
        Staged sb = stage_batch(m, batch, device, false, s);
        DedupOut o = dedup_buffers(m, B);
        run_dedup(m, sb, o, s);
        const Status& st = *m->st_host;
        if (st.err_bits & ERR_RANGE) {
            int code;
            std::string msg = status_message(m, st, &code);
            return set_err(code, msg);
        }
        *b_u = st.b_u;
        cudaMemcpyKind k = device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        DCAT_CUDA_CHECK(cudaMemcpyAsync(rep, o.rep, sizeof(int32_t) * B, k, s));
        if (first) DCAT_CUDA_CHECK(cudaMemcpyAsync(first, o.first, sizeof(int32_t) * st.b_u, k, s));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        return DCAT_OK;
    });
}

namespace {
// everything run_dcat's launches depend on: sizes, every pointer, settings, the buffer epoch
std::vector<uint64_t> run_key(const dcat_model* m, const Staged& sb, const DedupOut& o,
                              const dcat_finetune_config& ft, const Status& st, const float* dl, const float* dm,
                              const float* dh, bool f32) {
    std::vector<uint64_t> k;
    auto add_bytes = [&](const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        for (size_t i = 0; i < n; i += 8) {
            uint64_t v = 0;
            std::memcpy(&v, b + i, std::min<size_t>(8, n - i));
            k.push_back(v);
        }
    };
    add_bytes(&sb.in, sizeof sb.in);  // zero-padded (stage_batch)
    add_bytes(&o, sizeof o);          // zero-padded (dedup_buffers)
    k.push_back(reinterpret_cast<uintptr_t>(sb.candidate));
    k.push_back(reinterpret_cast<uintptr_t>(sb.age));
    k.push_back(reinterpret_cast<uintptr_t>(sb.aux));
    k.push_back(static_cast<uint64_t>(st.b_u));
    k.push_back(static_cast<uint64_t>(st.ctx_tokens));
    k.push_back(static_cast<uint64_t>(st.ctx_tiles));
    k.push_back(static_cast<uint64_t>(st.cross_tiles));
    k.push_back(reinterpret_cast<uintptr_t>(dl));
    k.push_back(reinterpret_cast<uintptr_t>(dm));
    k.push_back(reinterpret_cast<uintptr_t>(dh));
    k.push_back(static_cast<uint64_t>(ft.variant) | static_cast<uint64_t>(ft.use_seq_module) << 8 |
                static_cast<uint64_t>(static_cast<uint32_t>(ft.window)) << 16 | static_cast<uint64_t>(f32) << 48 |
                static_cast<uint64_t>(m->vt) << 49);
    k.push_back(static_cast<uint64_t>(static_cast<uint32_t>(ft.max_events)) |
                static_cast<uint64_t>(static_cast<uint32_t>(ft.d_aux)) << 32);
    add_bytes(&ft.fresh_days, sizeof ft.fresh_days);
    add_bytes(&ft.mid_days, sizeof ft.mid_days);
    k.push_back(static_cast<uint64_t>(m->tile_ctx) | static_cast<uint64_t>(m->tile_cross) << 32);
    k.push_back(g_alloc_epoch.load());
    return k;
}
}  // namespace

int dcat_rank_forward_batch(dcat_model* m, const dcat_batch* batch, const dcat_finetune_config* ft, float* logits,
                            float* module_logits, float* h_cand, int32_t flags, void* stream) {
    if (!m || !batch || !ft || !logits || !module_logits) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        NvtxRange nr("dcat_rank_forward_batch");
        const auto h_entry = std::chrono::steady_clock::now();
        int rc = validate_ft(m, ft, batch);
        if (rc) return rc;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        bool device = flags & DCAT_INPUT_DEVICE;
        bool f32 = flags & DCAT_PRECISION_FP32;
        m->profiling = flags & DCAT_PROFILE;
        m->ev_next = 0;
        m->ev_marks.clear();
        m->stage_ms.clear();
        std::memset(&m->stats, 0, sizeof m->stats);
        int64_t B = batch->n_rows;
        if (B == 0) return DCAT_OK;
        m->vt = use_tc_attention(m, f32);
        m->tile_ctx = m->vt ? 128 : kCtxTile;
        m->tile_cross = m->vt ? 128 : kCrossTile;
        int t0 = mark(m, s);
        Staged sb = stage_batch(m, batch, device,
                                ft->variant == DCAT_VARIANT_AUX || ft->variant == DCAT_VARIANT_AUXLT, s, true);
        // every exit (errors included) leaves no copy of the borrowed host arrays in flight
        struct SideDone {
            cudaEvent_t e;
            ~SideDone() {
                if (e) cudaEventSynchronize(e);
            }
        } side_done{sb.cand_ready};
        sb.in.window = ft->use_seq_module ? ft->window : 0;  // fixed-window sequence module
        sb.in.lt_token = ft->use_seq_module && ft->variant == DCAT_VARIANT_AUXLT;
        DedupOut o = dedup_buffers(m, B);
        int t1 = mark(m, s);
        const double h_pre = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h_entry).count();
        run_dedup(m, sb, o, s);
        int t2 = mark(m, s);
        m->t_dedup_end = t2;
        Status st = *m->st_host;
        if (!ft->use_seq_module) st.err_bits &= ~(ERR_ACTION | ERR_SURFACE | ERR_POS_CTX | ERR_POS_CAND);
        if (st.err_bits) {
            int code;
            std::string msg = status_message(m, st, &code);
            return set_err(code, msg);
        }
        m->stats.b_u = st.b_u;
        m->stats.ctx_tokens = st.ctx_tokens;
        m->last_bu = st.b_u;
        m->last_T = st.ctx_tokens;
        m->last_precision_f32 = f32;
        m->last_vt = m->vt;
        float *dl = logits, *dm = module_logits, *dh = h_cand;
        const bool out_device = device || (flags & DCAT_OUTPUT_DEVICE);
        if (!out_device) {
            dl = m->b_out[0].get<float>(B * 3);
            dm = m->b_out[1].get<float>(B * 3);
            dh = h_cand ? m->b_out[2].get<float>(B * m->cfg.d_model) : nullptr;
        }
        if (ft->use_seq_module) {
            auto run = [&](const Staged& b, cudaStream_t rs) {
                if (f32) run_dcat<float>(m, b, o, *ft, dl, dm, dh, rs);
                else run_dcat<bf16>(m, b, o, *ft, dl, dm, dh, rs);
            };
            static const bool no_graph = getenv("DCAT_NO_RUN_GRAPH") != nullptr;
            if (no_graph || m->profiling) {
                run(sb, s);
            } else {
                wait_cand(sb, s);  // outside any capture: the graph has no external dependency
                Staged gb = sb;
                gb.cand_ready = nullptr;
                std::vector<uint64_t> key = run_key(m, gb, o, *ft, st, dl, dm, dh, f32);
                if (m->run_exec && key == m->run_key) {  // replay
                    DCAT_CUDA_CHECK(cudaGraphLaunch(m->run_exec, s));
                    const dcat_call_stats keep = m->stats;
                    m->stats = m->run_stats;
                    m->stats.b_u = keep.b_u;
                    m->stats.ctx_tokens = keep.ctx_tokens;
                    m->stats.kernel_launches += keep.kernel_launches;
                    m->last_kv = m->run_last_kv;
                    m->last_Tp = m->run_last_Tp;
                } else if (key == m->run_seen) {  // second call with this shape: capture it
                    if (!m->cap) DCAT_CUDA_CHECK(cudaStreamCreateWithFlags(&m->cap, cudaStreamNonBlocking));
                    if (m->run_exec) {
                        DCAT_CUDA_CHECK(cudaGraphExecDestroy(m->run_exec));
                        m->run_exec = nullptr;
                    }
                    const dcat_call_stats before = m->stats;
                    cudaGraph_t g = nullptr;
                    DCAT_CUDA_CHECK(cudaStreamBeginCapture(m->cap, cudaStreamCaptureModeRelaxed));
                    run(gb, m->cap);
                    DCAT_CUDA_CHECK(cudaStreamEndCapture(m->cap, &g));
                    DCAT_CUDA_CHECK(cudaGraphInstantiate(&m->run_exec, g, 0));
                    DCAT_CUDA_CHECK(cudaGraphDestroy(g));
                    DCAT_CUDA_CHECK(cudaGraphLaunch(m->run_exec, s));
                    m->run_key = run_key(m, gb, o, *ft, st, dl, dm, dh, f32);
                    m->run_stats = m->stats;  // the pass's own counters, replayed with the graph
                    m->run_stats.kernel_launches -= before.kernel_launches;
                    m->run_last_kv = m->last_kv;
                    m->run_last_Tp = m->last_Tp;
                } else {
                    run(gb, s);
                    m->run_seen = run_key(m, gb, o, *ft, st, dl, dm, dh, f32);
                }
            }
        } else {
            if (f32) run_head_only<float>(m, sb, o, *ft, dl, dm, s);
            else run_head_only<bf16>(m, sb, o, *ft, dl, dm, s);
        }
        int t3 = mark(m, s);
        if (!out_device) {
            DCAT_CUDA_CHECK(cudaMemcpyAsync(logits, dl, sizeof(float) * B * 3, cudaMemcpyDeviceToHost, s));
            DCAT_CUDA_CHECK(cudaMemcpyAsync(module_logits, dm, sizeof(float) * B * 3, cudaMemcpyDeviceToHost, s));
            if (h_cand)
                DCAT_CUDA_CHECK(cudaMemcpyAsync(h_cand, dh, sizeof(float) * B * m->cfg.d_model, cudaMemcpyDeviceToHost,
                                                s));
        }
        DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
        int t4 = mark(m, s);
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        const auto h_sync = std::chrono::steady_clock::now();
        if (m->profiling) {
            span(m, "h2d", t0, t1);
            span(m, "dedup", t1, t2);
            span(m, "device_total", t1, t3);
            span(m, "d2h", t3, t4);
            for (auto& mk : m->ev_marks) {
                float ms = 0.f;
                DCAT_CUDA_CHECK(cudaEventElapsedTime(&ms, m->ev_pool[mk.second.first], m->ev_pool[mk.second.second]));
                m->stage_ms.push_back({mk.first, ms});
            }
        }
        Status fin = *m->st_host;
        if (fin.err_bits & ERR_AGE) return set_err(DCAT_EINVAL, "candidate age must be non-negative");
        if (fin.nonfinite_layer > 0)
            return set_err(DCAT_ENONFINITE, "non-finite activation in layer " + std::to_string(fin.nonfinite_layer - 1));
        // the context token offsets stay on the device until the next call; dcat_debug_kv reads them
        m->last_tok_off.clear();
        m->last_tok_off_dev = ft->use_seq_module ? o.tok_off : nullptr;
        if (host_timing()) {
            const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h_entry).count();
            std::fprintf(stderr, "[dcat host] entry->dedup launch %.1f us, final sync->return (incl.) %.1f us, total %.1f us\n",
                         h_pre, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h_sync).count(), us);
        }
        return DCAT_OK;
    });
}

int dcat_debug_kv(dcat_model* m, int32_t layer, int32_t unique, float* k, float* v, int32_t* n) {
    if (!m || !n) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        if (m->last_tok_off.empty() && m->last_tok_off_dev && m->last_bu >= 0) {
            m->last_tok_off.resize(static_cast<size_t>(m->last_bu) + 1);
            DCAT_CUDA_CHECK(cudaMemcpy(m->last_tok_off.data(), m->last_tok_off_dev,
                                       sizeof(int64_t) * (static_cast<size_t>(m->last_bu) + 1), cudaMemcpyDeviceToHost));
        }
        if (unique < 0 || unique >= m->last_bu || layer < 0 || layer >= m->cfg.n_layers ||
            m->last_tok_off.size() < static_cast<size_t>(unique) + 2)
            return set_err(DCAT_EINVAL, "no such unique / layer in the last call");
        int64_t a = m->last_tok_off[unique], b = m->last_tok_off[unique + 1];
        *n = static_cast<int32_t>(b - a);
        read_kv_rows(m->last_kv, m->last_vt, m->last_precision_f32, m->last_Tp, m->cfg.d_model, layer, a, b, k, v);
        return DCAT_OK;
    });
}

int dcat_context_forward(dcat_model* m, const dcat_batch* uniques, int32_t window, int32_t emit_hidden,
                         float* h_user, int32_t flags, void* stream, dcat_kv** out) {
    if (!m || !uniques || !out) return set_err(DCAT_EINVAL, "null argument");
    *out = nullptr;
    return guarded(m, [&]() -> int {
        NvtxRange nr("dcat_context_forward");
        // context_forward / context_forward_fixed argument checks (dcat.cpp:141-142, 285-288)
        const char* fn = window > 0 ? "context_forward_fixed" : "context_forward";
        if (window < 0) return set_err(DCAT_EINVAL, "context_forward_fixed: window must be >= 1, got " +
                                                        std::to_string(window));
        if (m->cfg.n_layers < 1) return set_err(DCAT_EINVAL, std::string(fn) + ": needs at least one layer");
        if (h_user && !emit_hidden) return set_err(DCAT_EINVAL, std::string(fn) + ": h_user requires emit_hidden");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const bool device = flags & DCAT_INPUT_DEVICE, f32 = flags & DCAT_PRECISION_FP32;
        m->profiling = false;
        m->ev_next = 0;
        m->ev_marks.clear();
        std::memset(&m->stats, 0, sizeof m->stats);
        std::unique_ptr<dcat_kv> kv(new dcat_kv());
        kv->m = m;
        kv->device = m->device;
        kv->f32 = f32;
        kv->n_layers = m->cfg.n_layers;
        kv->d = m->cfg.d_model;
        kv->window = window;
        const int64_t B = uniques->n_rows;
        if (B == 0) {
            kv->tok_off.assign(1, 0);
            *out = kv.release();
            return DCAT_OK;
        }
        m->vt = use_tc_attention(m, f32);
        m->tile_ctx = m->vt ? 128 : kCtxTile;
        m->tile_cross = m->vt ? 128 : kCrossTile;
        Staged sb = stage_batch(m, uniques, device, false, s, false);
        sb.in.window = window;
        sb.in.lt_token = 0;
        DedupOut o = dedup_buffers(m, B);
        run_dedup(m, sb, o, s);
        Status st = *m->st_host;
        st.err_bits &= ~(ERR_POS_CAND | ERR_AGE);  // no candidate tokens here
        if (st.err_bits) {
            int code;
            std::string msg = status_message(m, st, &code);
            return set_err(code, msg);
        }
        dcat_finetune_config ft{};
        ft.variant = DCAT_VARIANT_BASE;
        ft.use_seq_module = 1;
        ft.window = window;
        ft.fresh_days = 1.0;
        ft.mid_days = 2.0;
        const int64_t T_ctx = st.ctx_tokens, d = m->cfg.d_model;
        float* hdev = emit_hidden && h_user ? m->b_x[0].get<float>(std::max<int64_t>(T_ctx, 1) * d) : nullptr;
        CtxOnly co;
        co.on = true;
        co.emit_hidden = emit_hidden != 0;
        co.h_user = hdev;
        if (f32) run_dcat<float>(m, sb, o, ft, nullptr, nullptr, nullptr, s, co);
        else run_dcat<bf16>(m, sb, o, ft, nullptr, nullptr, nullptr, s, co);
        kv->vt = m->vt;
        kv->Tp = m->last_Tp;
        kv->T_ctx = T_ctx;
        const size_t bytes = static_cast<size_t>(2 * kv->n_layers) * kv->Tp * d * (f32 ? 4 : 2);
        DCAT_CUDA_CHECK(cudaMalloc(&kv->buf, std::max<size_t>(bytes, 16)));
        if (bytes) DCAT_CUDA_CHECK(cudaMemcpyAsync(kv->buf, m->last_kv, bytes, cudaMemcpyDeviceToDevice, s));
        kv->rep.resize(static_cast<size_t>(B));
        kv->tok_off.resize(static_cast<size_t>(st.b_u) + 1);
        DCAT_CUDA_CHECK(cudaMemcpyAsync(kv->rep.data(), o.rep, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaMemcpyAsync(kv->tok_off.data(), o.tok_off, sizeof(int64_t) * (st.b_u + 1),
                                        cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        if (m->st_host->nonfinite_layer > 0)
            return set_err(DCAT_ENONFINITE,
                           "non-finite activation in layer " + std::to_string(m->st_host->nonfinite_layer - 1));
        if (hdev) {  // per caller row, its unique's tokens (duplicates repeat them)
            int64_t at = 0;
            const cudaMemcpyKind kind = device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
            for (int64_t r = 0; r < B; r++) {
                const int32_t u = kv->rep[static_cast<size_t>(r)];
                const int64_t a = kv->tok_off[u], n = kv->tok_off[u + 1] - a;
                if (n) DCAT_CUDA_CHECK(cudaMemcpyAsync(h_user + at * d, hdev + a * d, sizeof(float) * n * d, kind, s));
                at += n;
            }
            DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        }
        *out = kv.release();
        return DCAT_OK;
    });
}

int dcat_host_alloc(uint64_t bytes, void** out) {
    if (!out) return set_err(DCAT_EINVAL, "null argument");
    *out = nullptr;
    return guarded(nullptr, [&]() -> int {
        DCAT_CUDA_CHECK(cudaHostAlloc(out, std::max<uint64_t>(bytes, 16), cudaHostAllocPortable));
        return DCAT_OK;
    });
}

int dcat_host_free(void* p) {
    if (p) cudaFreeHost(p);
    return DCAT_OK;
}

int dcat_kv_destroy(dcat_kv* kv) {
    if (!kv) return DCAT_OK;
    DeviceScopeNoThrow ds(kv->device);
    cudaDeviceSynchronize();
    delete kv;
    return DCAT_OK;
}

int dcat_kv_info(const dcat_kv* kv, int32_t* n_uniques, int32_t* n_layers, int32_t* d_model, int32_t* n) {
    if (!kv) return set_err(DCAT_EINVAL, "null argument");
    if (n_uniques) *n_uniques = static_cast<int32_t>(kv->rep.size());
    if (n_layers) *n_layers = kv->n_layers;
    if (d_model) *d_model = kv->d;
    if (n)
        for (size_t r = 0; r < kv->rep.size(); r++) {
            const int32_t u = kv->rep[r];
            n[r] = static_cast<int32_t>(kv->tok_off[u + 1] - kv->tok_off[u]);
        }
    return DCAT_OK;
}

int dcat_kv_read(const dcat_kv* kv, int32_t layer, int32_t unique, float* k, float* v) {
    if (!kv) return set_err(DCAT_EINVAL, "null argument");
    return guarded(kv->m, [&]() -> int {
        if (unique < 0 || unique >= static_cast<int32_t>(kv->rep.size()) || layer < 0 || layer >= kv->n_layers)
            return set_err(DCAT_EINVAL, "dcat_kv_read: no such unique / layer");
        const int32_t u = kv->rep[static_cast<size_t>(unique)];
        read_kv_rows(kv->buf, kv->vt, kv->f32, kv->Tp, kv->d, layer, kv->tok_off[u], kv->tok_off[u + 1], k, v);
        return DCAT_OK;
    });
}

int dcat_candidate_inputs(dcat_model* m, const uint64_t* items, const int32_t* pos, int64_t n, float* e_cand,
                          int32_t flags, void* stream) {
    if (!m || (n > 0 && (!items || !pos || !e_cand))) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        NvtxRange nr("dcat_candidate_inputs");
        if (n <= 0) return DCAT_OK;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const bool device = flags & DCAT_INPUT_DEVICE;
        const int de = m->cfg.d_emb;
        const uint64_t* it = items;
        const int32_t* ps = pos;
        float* e = e_cand;
        if (!device) {
            uint64_t* it_d = m->b_x[3].get<uint64_t>(n);
            int32_t* ps_d = m->b_x[4].get<int32_t>(n);
            DCAT_CUDA_CHECK(cudaMemcpyAsync(it_d, items, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
            DCAT_CUDA_CHECK(cudaMemcpyAsync(ps_d, pos, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
            it = it_d;
            ps = ps_d;
            e = m->b_x[5].get<float>(n * de);
        }
        DCAT_CUDA_CHECK(cudaMemsetAsync(m->st_dev, 0, sizeof(Status), s));
        candidate_inputs(emb_params(m, true), it, ps, n, e, m->st_dev, s);
        if (!device) DCAT_CUDA_CHECK(cudaMemcpyAsync(e_cand, e, sizeof(float) * n * de, cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        if (m->st_host->err_bits & ERR_POS_CAND)
            return set_err(DCAT_EINVAL, "candidate_inputs: position " + std::to_string(m->st_host->err_val) +
                                            " out of range (max_len " + std::to_string(m->cfg.max_len) + ")");
        return DCAT_OK;
    });
}

int dcat_cross_forward(dcat_model* m, const dcat_kv* kv, const int32_t* rep, const float* e_cand, int64_t n,
                       float* h, int32_t flags, void* stream) {
    if (!m || !kv || (n > 0 && (!rep || !e_cand || !h))) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        NvtxRange nr("dcat_cross_forward");
        const char* fn = kv->window > 0 ? "cross_forward_fixed" : "cross_forward";
        if (kv->m != m) return set_err(DCAT_EINVAL, std::string(fn) + ": cache/model config mismatch");
        const bool device = flags & DCAT_INPUT_DEVICE, f32 = flags & DCAT_PRECISION_FP32;
        if (f32 != kv->f32)
            return set_err(DCAT_EINVAL, std::string(fn) + ": precision differs from the cache's (DCAT_PRECISION_FP32)");
        if (n <= 0) return DCAT_OK;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int d = m->cfg.d_model, de = m->cfg.d_emb;
        std::vector<int32_t> hrep(static_cast<size_t>(n));
        if (device) DCAT_CUDA_CHECK(cudaMemcpy(hrep.data(), rep, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
        else std::memcpy(hrep.data(), rep, sizeof(int32_t) * n);
        std::vector<int32_t> du(static_cast<size_t>(n));
        const int32_t n_uniques = static_cast<int32_t>(kv->rep.size());
        for (int64_t b = 0; b < n; b++) {
            const int32_t r = hrep[static_cast<size_t>(b)];
            if (r < 0 || r >= n_uniques)
                return set_err(DCAT_EINVAL, std::string(fn) + ": plan rep " + std::to_string(r) + " of row " +
                                                std::to_string(b) + " outside the cache's " +
                                                std::to_string(n_uniques) + " uniques");
            du[static_cast<size_t>(b)] = kv->rep[static_cast<size_t>(r)];
        }
        const float* e_dev = e_cand;
        if (!device) {
            float* tmp = m->b_x[5].get<float>(n * de);
            DCAT_CUDA_CHECK(cudaMemcpyAsync(tmp, e_cand, sizeof(float) * n * de, cudaMemcpyHostToDevice, s));
            e_dev = tmp;
        }
        float* h_dev = device ? h : m->b_x[0].get<float>(n * d);
        m->profiling = false;
        m->ev_next = 0;
        m->ev_marks.clear();
        std::memset(&m->stats, 0, sizeof m->stats);
        m->vt = kv->vt;
        m->tile_cross = 128;
        DCAT_CUDA_CHECK(cudaMemsetAsync(m->st_dev, 0, sizeof(Status), s));
        if (f32) run_cross_external<float>(m, kv, du, e_dev, h_dev, s);
        else run_cross_external<bf16>(m, kv, du, e_dev, h_dev, s);
        if (!device) DCAT_CUDA_CHECK(cudaMemcpyAsync(h, h_dev, sizeof(float) * n * d, cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaMemcpyAsync(m->st_host, m->st_dev, sizeof(Status), cudaMemcpyDeviceToHost, s));
        DCAT_CUDA_CHECK(cudaStreamSynchronize(s));
        if (m->st_host->nonfinite_layer > 0)
            return set_err(DCAT_ENONFINITE,
                           "non-finite activation in layer " + std::to_string(m->st_host->nonfinite_layer - 1));
        return DCAT_OK;
    });
}

int dcat_stage_times(dcat_model* m, const char** names, float* ms, int32_t cap) {
    if (!m) return 0;
    int n = 0;
    for (auto& p : m->stage_ms) {
        if (n >= cap) break;
        if (names) names[n] = p.first;
        if (ms) ms[n] = p.second;
        n++;
    }
    return n;
}

int dcat_debug_counters(dcat_model* m, uint64_t* out, int32_t cap) {
    if (!m || !out) return set_err(DCAT_EINVAL, "null argument");
    return guarded(m, [&]() -> int {
        unsigned h[kDebugCounters] = {};
        if (m->dbg) {
            DCAT_CUDA_CHECK(cudaDeviceSynchronize());
            DCAT_CUDA_CHECK(cudaMemcpy(h, m->dbg, sizeof h, cudaMemcpyDeviceToHost));
            DCAT_CUDA_CHECK(cudaMemset(m->dbg, 0, sizeof h));
        }
        const int n = std::min<int>(cap, kDebugCounters);
        for (int i = 0; i < n; i++) out[i] = h[i];
        return m->dbg ? n : 0;
    });
}

int dcat_last_stats(dcat_model* m, dcat_call_stats* out) {
    if (!m || !out) return set_err(DCAT_EINVAL, "null argument");
    *out = m->stats;
    return DCAT_OK;
}

}  // extern "C"
