/*
 * dcat_oracle.c — plain-C restatement of the reference DCAT scoring path.
 *
 * TEST INFRASTRUCTURE (the checker, never the product). See dcat_oracle.h.
 * Each function names the reference file:line it restates; loop order and
 * float operation order follow the reference so that, compiled without
 * -ffast-math / FMA contraction, results are bit-identical to the reference
 * (checked against oracle/_ref fixtures in tests/test_oracle_golden.py).
 */
#include "dcat_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* error handling + scratch arena (freed at every API exit)                  */

static _Thread_local char g_err[512];
static _Thread_local jmp_buf* g_jmp;
typedef struct blk { struct blk* next; } blk;
static _Thread_local blk* g_arena;

const char* oracle_last_error(void) { return g_err; }

static void fail(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    longjmp(*g_jmp, 1);
}
#define CHECK(c, ...) do { if (!(c)) fail(__VA_ARGS__); } while (0)

static void* amalloc(size_t n) {
    blk* b = (blk*)calloc(1, sizeof(blk) + (n ? n : 1) + 64);
    if (!b) fail("oracle: out of memory");
    b->next = g_arena;
    g_arena = b;
    return (void*)((char*)b + 64);
}
static void arena_free(void) {
    while (g_arena) { blk* n = g_arena->next; free(g_arena); g_arena = n; }
}
#define API_BEGIN                                   \
    jmp_buf jb__; jmp_buf* prev__ = g_jmp;          \
    g_err[0] = 0;                                   \
    if (setjmp(jb__)) { g_jmp = prev__; arena_free(); return -1; } \
    g_jmp = &jb__;
#define API_END g_jmp = prev__; arena_free(); return 0;

/* ------------------------------------------------------------------------ */
/* L0 primitives: mat.hpp, rng.hpp                                          */

typedef struct { int rows, cols; float* a; } Mat;

static Mat mat(int r, int c) { Mat m = {r, c, (float*)amalloc(sizeof(float) * (size_t)r * c)}; return m; }
static float* row(const Mat* m, int r) { return m->a + (size_t)r * m->cols; }

/* mix64 (rng.hpp:13-18) */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* Rng (rng.hpp:21-73) */
typedef struct { uint64_t state; double cached; int has_cached; } Rng;
static Rng rng_make(uint64_t seed) { Rng r = {seed, 0.0, 0}; return r; }
static uint64_t rng_next(Rng* r) {
    r->state += 0x9e3779b97f4a7c15ULL;
    uint64_t x = r->state;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static double rng_uniform(Rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_normal(Rng* r) {
    if (r->has_cached) { r->has_cached = 0; return r->cached; }
    double u1 = rng_uniform(r);
    double u2 = rng_uniform(r);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    double rr = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    r->cached = rr * sin(a);
    r->has_cached = 1;
    return rr * cos(a);
}
static void init_gaussian(float* v, size_t n, Rng* r, float stddev) {
    for (size_t i = 0; i < n; i++) v[i] = (float)(rng_normal(r) * stddev);
}

/* dot / axpy / l2_norm (mat.hpp:43-59) */
static float dot(const float* x, const float* y, int n) {
    float s = 0.0f;
    for (int i = 0; i < n; i++) s += x[i] * y[i];
    return s;
}
static void axpy(float alpha, const float* x, float* y, int n) {
    for (int i = 0; i < n; i++) y[i] += alpha * x[i];
}
static float l2_norm(const float* x, int n) {
    float s = 0.0f;
    for (int i = 0; i < n; i++) s += x[i] * x[i];
    return sqrtf(s);
}

/* matmul, ikj with zero skip (mat.hpp:61-76). B is k x n row-major. */
static Mat matmul(const Mat* A, const float* B, int bcols) {
    Mat C = mat(A->rows, bcols);
    for (int i = 0; i < A->rows; i++) {
        const float* ar = row(A, i);
        float* cr = row(&C, i);
        for (int k = 0; k < A->cols; k++) {
            float av = ar[k];
            if (av == 0.0f) continue;
            const float* br = B + (size_t)k * bcols;
            for (int j = 0; j < bcols; j++) cr[j] += av * br[j];
        }
    }
    return C;
}

/* gelu, tanh form (model.hpp:14-18) */
static float gelu(float x) {
    const float c = 0.7978845608028654f;
    float x3 = x * x * x;
    return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x3)));
}

/* ------------------------------------------------------------------------ */
/* L3 model math: model.cpp                                                  */

typedef struct { const float *w1, *b1, *w2, *b2; int d_in, d_hidden, d_out; } Mlp;
typedef struct {
    const float *ln1_g, *ln1_b, *wq, *bq, *wk, *bk, *wv, *bv, *wo, *bo, *ln2_g, *ln2_b, *fw1, *fb1,
        *fw2, *fb2;
} Layer;
typedef struct {
    dcat_model_config cfg;
    const float *action_emb, *surface_emb, *pos_emb;
    Mlp phi_in, phi_out;
    Layer* layers;
} Model;

static int n_tensors(const dcat_model_config* c) { return 3 + (c->pos_learned ? 1 : 0) + 12 + 16 * c->n_layers; }

static void model_config_validate(const dcat_model_config* c) {
    /* ModelConfig::validate (model.cpp:175-183) */
    CHECK(c->d_model >= 1 && c->n_heads >= 1 && c->d_model % c->n_heads == 0,
          "d_model %d must be divisible by n_heads %d", c->d_model, c->n_heads);
    CHECK(c->n_layers >= 0, "n_layers must be >= 0");
    CHECK(c->mlp_ratio >= 1, "mlp_ratio must be >= 1");
    CHECK(c->max_len >= 1, "max_len must be >= 1");
    CHECK(c->d_emb >= 1, "d_emb must be >= 1");
}

static Model bind_model(const dcat_model_config* cfg, const dcat_params* p) {
    model_config_validate(cfg);
    CHECK(p->n_tensors == n_tensors(cfg), "params: expected %d tensors, got %d", n_tensors(cfg), p->n_tensors);
    Model m;
    memset(&m, 0, sizeof m);
    m.cfg = *cfg;
    int t = 1; /* skip log_tau */
    m.action_emb = p->tensors[t++];
    m.surface_emb = p->tensors[t++];
    m.pos_emb = cfg->pos_learned ? p->tensors[t++] : NULL;
    int d = cfg->d_model;
    Mlp* mlps[2] = {&m.phi_in, &m.phi_out};
    int dins[2] = {cfg->d_emb, d};
    for (int i = 0; i < 2; i++) {
        mlps[i]->w1 = p->tensors[t++]; mlps[i]->b1 = p->tensors[t++];
        mlps[i]->w2 = p->tensors[t++]; mlps[i]->b2 = p->tensors[t++];
        mlps[i]->d_in = dins[i]; mlps[i]->d_hidden = d; mlps[i]->d_out = d;
    }
    t += 4; /* psi: not on the scoring path */
    m.layers = (Layer*)amalloc(sizeof(Layer) * (size_t)(cfg->n_layers > 0 ? cfg->n_layers : 1));
    for (int l = 0; l < cfg->n_layers; l++) {
        Layer* L = &m.layers[l];
        const float** f[16] = {&L->ln1_g, &L->ln1_b, &L->wq, &L->bq, &L->wk, &L->bk, &L->wv, &L->bv,
                               &L->wo, &L->bo, &L->ln2_g, &L->ln2_b, &L->fw1, &L->fb1, &L->fw2, &L->fb2};
        for (int i = 0; i < 16; i++) *f[i] = p->tensors[t++];
    }
    return m;
}

/* linear_forward (model.cpp:43-46) */
static Mat linear(const Mat* x, const float* w, const float* b, int out) {
    Mat y = matmul(x, w, out);
    for (int i = 0; i < y.rows; i++) axpy(1.0f, b, row(&y, i), y.cols);
    return y;
}

/* layernorm_forward, eps 1e-5 (model.cpp:14, 54-81) */
static Mat layernorm(const Mat* x, const float* g, const float* b) {
    int n = x->rows, d = x->cols;
    Mat y = mat(n, d);
    for (int i = 0; i < n; i++) {
        const float* xi = row(x, i);
        float mu = 0.0f;
        for (int j = 0; j < d; j++) mu += xi[j];
        mu /= (float)d;
        float var = 0.0f;
        for (int j = 0; j < d; j++) { float c = xi[j] - mu; var += c * c; }
        var /= (float)d;
        float rs = 1.0f / sqrtf(var + 1e-5f);
        float* yi = row(&y, i);
        for (int j = 0; j < d; j++) { float h = (xi[j] - mu) * rs; yi[j] = g[j] * h + b[j]; }
    }
    return y;
}

/* l2norm_rows, eps 1e-12 (model.cpp:15, 107-117) */
static Mat l2norm_rows(const Mat* y) {
    Mat o = mat(y->rows, y->cols);
    for (int i = 0; i < y->rows; i++) {
        float nrm = l2_norm(row(y, i), y->cols);
        float inv = 1.0f / (nrm < 1e-12f ? 1e-12f : nrm);
        for (int j = 0; j < y->cols; j++) row(&o, i)[j] = row(y, i)[j] * inv;
    }
    return o;
}

/* mlp_forward (model.cpp:144-161) */
static Mat mlp_forward(const Mlp* p, const Mat* x) {
    CHECK(x->cols == p->d_in, "mlp_forward: input dim %d expected %d", x->cols, p->d_in);
    Mat z1 = linear(x, p->w1, p->b1, p->d_hidden);
    Mat a1 = mat(z1.rows, z1.cols);
    for (size_t i = 0; i < (size_t)z1.rows * z1.cols; i++) a1.a[i] = gelu(z1.a[i]);
    Mat y = linear(&a1, p->w2, p->b2, p->d_out);
    return l2norm_rows(&y);
}

static void check_finite(const Mat* x, int layer) {
    for (size_t i = 0; i < (size_t)x->rows * x->cols; i++)
        CHECK(isfinite(x->a[i]), "non-finite activation in layer %d", layer);
}

/* layer_forward without dropout / prob recording (model.cpp:336-398).
 * k_out / v_out (may be NULL) receive the layer's K and V (LayerCache k, v). */
static Mat layer_forward(const Layer* L, const dcat_model_config* cfg, const Mat* x_in, Mat* k_out,
                         Mat* v_out, int layer_idx) {
    int n = x_in->rows, d = cfg->d_model, heads = cfg->n_heads, dh = d / heads;
    float scale = 1.0f / sqrtf((float)dh);
    Mat a = layernorm(x_in, L->ln1_g, L->ln1_b);
    Mat q = linear(&a, L->wq, L->bq, d);
    Mat k = linear(&a, L->wk, L->bk, d);
    Mat v = linear(&a, L->wv, L->bv, d);
    Mat ctx = mat(n, d);
    float* logits = (float*)amalloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (int h = 0; h < heads; h++) {
        int off = h * dh;
        for (int i = 0; i < n; i++) {
            const float* qi = row(&q, i) + off;
            float mx = -INFINITY;
            for (int j = 0; j <= i; j++) {
                logits[j] = dot(qi, row(&k, j) + off, dh) * scale;
                mx = mx < logits[j] ? logits[j] : mx;
            }
            float denom = 0.0f;
            for (int j = 0; j <= i; j++) { logits[j] = expf(logits[j] - mx); denom += logits[j]; }
            float inv = 1.0f / denom;
            float* crow = row(&ctx, i) + off;
            for (int j = 0; j <= i; j++) { float pj = logits[j] * inv; axpy(pj, row(&v, j) + off, crow, dh); }
        }
    }
    Mat o = linear(&ctx, L->wo, L->bo, d);
    Mat x2 = mat(n, d);
    memcpy(x2.a, x_in->a, sizeof(float) * (size_t)n * d);
    for (size_t i = 0; i < (size_t)n * d; i++) x2.a[i] += o.a[i];
    Mat m = layernorm(&x2, L->ln2_g, L->ln2_b);
    int dff = d * cfg->mlp_ratio;
    Mat f1 = linear(&m, L->fw1, L->fb1, dff);
    for (size_t i = 0; i < (size_t)n * dff; i++) f1.a[i] = gelu(f1.a[i]);
    Mat f2 = linear(&f1, L->fw2, L->fb2, d);
    Mat x_out = x2;
    for (size_t i = 0; i < (size_t)n * d; i++) x_out.a[i] += f2.a[i];
    check_finite(&x_out, layer_idx);
    if (k_out) *k_out = k;
    if (v_out) *v_out = v;
    return x_out;
}

/* forward_rows without caches (model.cpp:478-502) */
static Mat forward_rows(const Model* M, const Mat* E) {
    CHECK(E->cols == M->cfg.d_emb, "forward_rows: input dim %d expected %d", E->cols, M->cfg.d_emb);
    Mat x = mlp_forward(&M->phi_in, E);
    for (int l = 0; l < M->cfg.n_layers; l++) x = layer_forward(&M->layers[l], &M->cfg, &x, NULL, NULL, l);
    return mlp_forward(&M->phi_out, &x);
}

/* ------------------------------------------------------------------------ */
/* L2 embeddings: embed.cpp                                                  */

/* hash_id (embed.cpp:11-14) */
static uint32_t hash_id(uint64_t id, uint64_t seed, uint32_t rows) {
    CHECK(rows > 0, "hash_id: rows must be positive");
    return (uint32_t)(mix64(id ^ mix64(seed)) % rows);
}

/* HashedEmbeddingTable::lookup (embed.cpp:38-43) */
/* IEEE binary16 conversions (fp16.hpp): round-to-nearest-even to half, exact back.
 * _Float16 casts are IEEE conversions, identical to the reference's bit routines
 * for every finite value (quantize rejects non-finite rows, embed.cpp:138-140). */
static uint16_t f32_to_f16(float f) {
    _Float16 h = (_Float16)f;
    uint16_t u;
    memcpy(&u, &h, 2);
    return u;
}
static float f16_to_f32(uint16_t u) {
    _Float16 h;
    memcpy(&h, &u, 2);
    return (float)h;
}

static int q_code_bytes(const dcat_table* t) { return (t->d_sub * t->bits + 7) / 8; }
static int q_row_bytes(const dcat_table* t) { return q_code_bytes(t) + 4; }

/* QuantizedTable::dequantize_row (embed.cpp:92-103): codes (int4: element e in byte
 * e / 2, low nibble first), fp16 scale, fp16 bias; v = (float)code * scale + bias */
static void dequantize_row(const dcat_table* t, int j, uint32_t r, float* out) {
    const uint8_t* row = t->packed + ((size_t)j * t->rows + r) * (size_t)q_row_bytes(t);
    const int cb = q_code_bytes(t);
    const float s = f16_to_f32((uint16_t)(row[cb] | (row[cb + 1] << 8)));
    const float b = f16_to_f32((uint16_t)(row[cb + 2] | (row[cb + 3] << 8)));
    for (int e = 0; e < t->d_sub; e++) {
        uint32_t code = t->bits == 8 ? row[e] : (uint32_t)((row[e / 2] >> ((e % 2) * 4)) & 15);
        float cs = (float)code * s;
        out[e] = cs + b;
    }
}

/* HashedEmbeddingTable::lookup (embed.cpp:38-43) / QuantizedTable::qlookup (:111-113) */
static void lookup(const dcat_table* t, uint64_t id, float* out) {
    for (int j = 0; j < t->num_subtables; j++) {
        uint32_t r = hash_id(id, t->seeds[j], (uint32_t)t->rows);
        if (t->bits)
            dequantize_row(t, j, r, out + (size_t)j * t->d_sub);
        else
            memcpy(out + (size_t)j * t->d_sub, t->subtables[j] + (size_t)r * t->d_sub, sizeof(float) * t->d_sub);
    }
}

/* segment_inputs (model.cpp:517-540); events of one row from the pool */
static Mat segment_inputs(const Model* M, const dcat_table* t, const dcat_batch* b, int64_t off, int n,
                          int pos_offset) {
    const dcat_model_config* cfg = &M->cfg;
    CHECK(t->num_subtables * t->d_sub == cfg->d_emb, "segment_inputs: id source dim mismatch");
    Mat E = mat(n, cfg->d_emb);
    for (int i = 0; i < n; i++) {
        int a = b->ev_action[off + i];
        int s = b->ev_surface[off + i];
        CHECK(a >= 0 && a < cfg->n_actions, "unknown action value %d at token %d", a, i);
        CHECK(s >= 0 && s < cfg->n_surfaces, "unknown surface value %d at token %d", s, i);
        float* r = row(&E, i);
        lookup(t, b->ev_item[off + i], r);
        axpy(1.0f, M->action_emb + (size_t)a * cfg->d_emb, r, cfg->d_emb);
        axpy(1.0f, M->surface_emb + (size_t)s * cfg->d_emb, r, cfg->d_emb);
        if (cfg->pos_learned) {
            int pos = pos_offset + i;
            CHECK(pos < cfg->max_len, "position %d exceeds max_len %d", pos, cfg->max_len);
            axpy(1.0f, M->pos_emb + (size_t)pos * cfg->d_emb, r, cfg->d_emb);
        }
    }
    return E;
}

/* ------------------------------------------------------------------------ */
/* L4 DCAT: dcat.cpp                                                         */

/* segment_key equality (dcat.cpp:45-56): 18 bytes per valid event */
static int same_key(const dcat_batch* b, int64_t i, int64_t j) {
    int n = b->row_valid[i];
    if (n != b->row_valid[j]) return 0;
    int64_t oi = b->row_offset[i], oj = b->row_offset[j];
    if (oi == oj) return 1;
    for (int e = 0; e < n; e++) {
        if (b->ev_ts[oi + e] != b->ev_ts[oj + e] || b->ev_action[oi + e] != b->ev_action[oj + e] ||
            b->ev_surface[oi + e] != b->ev_surface[oj + e] || b->ev_item[oi + e] != b->ev_item[oj + e])
            return 0;
    }
    return 1;
}
static uint64_t key_hash(const dcat_batch* b, int64_t i) {
    /* FNV-1a over the 18-byte-per-event key; any hash works, equality decides */
    uint64_t h = 1469598103934665603ULL;
    int64_t o = b->row_offset[i];
    for (int e = 0; e < b->row_valid[i]; e++) {
        uint64_t w[3] = {b->ev_ts[o + e], (uint64_t)b->ev_action[o + e] | ((uint64_t)b->ev_surface[o + e] << 8),
                         b->ev_item[o + e]};
        for (int k = 0; k < 3; k++) { h ^= w[k]; h *= 1099511628211ULL; }
    }
    h ^= (uint64_t)b->row_valid[i];
    return mix64(h);
}

/* dedup_segments (dcat.cpp:91-108): unordered_map first-seen, uniques in
 * first-appearance order. */
static int dedup(const dcat_batch* b, int32_t* rep, int32_t* first) {
    int64_t n = b->n_rows;
    size_t cap = 16;
    while (cap < (size_t)n * 2) cap <<= 1;
    int32_t* slot_row = (int32_t*)amalloc(sizeof(int32_t) * cap);
    int32_t* slot_uid = (int32_t*)amalloc(sizeof(int32_t) * cap);
    for (size_t s = 0; s < cap; s++) slot_row[s] = -1;
    int b_u = 0;
    for (int64_t i = 0; i < n; i++) {
        CHECK(b->row_valid[i] >= 0, "row %lld: negative valid", (long long)i);
        size_t s = key_hash(b, i) & (cap - 1);
        for (;;) {
            if (slot_row[s] < 0) {
                slot_row[s] = (int32_t)i;
                slot_uid[s] = b_u;
                if (first) first[b_u] = (int32_t)i;
                rep[i] = b_u++;
                break;
            }
            if (same_key(b, slot_row[s], i)) { rep[i] = slot_uid[s]; break; }
            s = (s + 1) & (cap - 1);
        }
    }
    return b_u;
}

/* kv_only (dcat.cpp:60-65) */
static void kv_only(const Layer* L, const dcat_model_config* cfg, const Mat* x, Mat* k, Mat* v) {
    Mat a = layernorm(x, L->ln1_g, L->ln1_b);
    *k = linear(&a, L->wk, L->bk, cfg->d_model);
    *v = linear(&a, L->wv, L->bv, cfg->d_model);
}

typedef struct { int n; Mat* k; Mat* v; } SeqKV;

/* context_forward with emit_hidden = false (dcat.cpp:137-178). Uniques are
 * batch rows `urow[u]`. */
static SeqKV* context_forward(const Model* M, const dcat_table* t, const dcat_batch* b, const int32_t* urow,
                              int b_u) {
    const dcat_model_config* cfg = &M->cfg;
    CHECK(cfg->n_layers >= 1, "context_forward: needs at least one layer");
    SeqKV* kv = (SeqKV*)amalloc(sizeof(SeqKV) * (size_t)(b_u > 0 ? b_u : 1));
    for (int u = 0; u < b_u; u++) {
        int64_t r = urow[u];
        kv[u].n = b->row_valid[r];
        kv[u].k = (Mat*)amalloc(sizeof(Mat) * cfg->n_layers);
        kv[u].v = (Mat*)amalloc(sizeof(Mat) * cfg->n_layers);
        Mat e = segment_inputs(M, t, b, b->row_offset[r], b->row_valid[r], 0);
        Mat x = mlp_forward(&M->phi_in, &e);
        for (int l = 0; l < cfg->n_layers; l++) {
            if (l == cfg->n_layers - 1) { kv_only(&M->layers[l], cfg, &x, &kv[u].k[l], &kv[u].v[l]); break; }
            x = layer_forward(&M->layers[l], cfg, &x, &kv[u].k[l], &kv[u].v[l], l);
        }
    }
    return kv;
}

/* candidate_inputs (dcat.cpp:180-197) */
static Mat candidate_inputs(const Model* M, const dcat_table* t, const uint64_t* items, const int* pos, int64_t n) {
    const dcat_model_config* cfg = &M->cfg;
    CHECK(t->num_subtables * t->d_sub == cfg->d_emb, "candidate_inputs: embedding dim mismatch");
    Mat e = mat((int)n, cfg->d_emb);
    for (int64_t i = 0; i < n; i++) {
        float* r = row(&e, (int)i);
        lookup(t, items[i], r);
        if (cfg->pos_learned) {
            CHECK(pos[i] >= 0 && pos[i] < cfg->max_len, "candidate_inputs: position %d out of range (max_len %d)",
                  pos[i], cfg->max_len);
            axpy(1.0f, M->pos_emb + (size_t)pos[i] * cfg->d_emb, r, cfg->d_emb);
        }
    }
    return e;
}

/* cross_tail (dcat.cpp:77-87) on a 1-row state */
static void cross_tail(const Layer* L, const dcat_model_config* cfg, Mat* x, const Mat* ctx, int layer_idx) {
    int d = cfg->d_model, dff = d * cfg->mlp_ratio;
    Mat o = linear(ctx, L->wo, L->bo, d);
    for (int i = 0; i < d; i++) x->a[i] += o.a[i];
    Mat m = layernorm(x, L->ln2_g, L->ln2_b);
    Mat f1 = linear(&m, L->fw1, L->fb1, dff);
    for (int i = 0; i < dff; i++) f1.a[i] = gelu(f1.a[i]);
    Mat f2 = linear(&f1, L->fw2, L->fb2, d);
    for (int i = 0; i < d; i++) x->a[i] += f2.a[i];
    for (int i = 0; i < d; i++) CHECK(isfinite(x->a[i]), "non-finite activation in layer %d", layer_idx);
}

/* cross_forward (dcat.cpp:199-271): per candidate, attention over the
 * materialized [K_u; k] / [V_u; v] (dcat.cpp:231-243). */
static Mat cross_forward(const Model* M, const SeqKV* cache, int b_u, const int32_t* rep, int64_t B, const Mat* e_cand) {
    const dcat_model_config* cfg = &M->cfg;
    CHECK(e_cand->rows == B, "cross_forward: %d candidate rows for %lld batch rows", e_cand->rows, (long long)B);
    CHECK(e_cand->cols == cfg->d_emb, "cross_forward: candidate dim mismatch");
    int d = cfg->d_model, heads = cfg->n_heads, dh = d / heads;
    float scale = 1.0f / sqrtf((float)dh);
    Mat out = mat((int)B, d);
    for (int64_t bi = 0; bi < B; bi++) {
        CHECK(rep[bi] >= 0 && rep[bi] < b_u, "cross_forward: bad rep");
        const SeqKV* kv = &cache[rep[bi]];
        int n = kv->n;
        Mat e_row = {1, cfg->d_emb, row(e_cand, (int)bi)};
        Mat x = mlp_forward(&M->phi_in, &e_row);
        float* logits = (float*)amalloc(sizeof(float) * (size_t)(n + 1));
        for (int l = 0; l < cfg->n_layers; l++) {
            const Layer* L = &M->layers[l];
            Mat a = layernorm(&x, L->ln1_g, L->ln1_b);
            Mat q = linear(&a, L->wq, L->bq, d);
            Mat kc = linear(&a, L->wk, L->bk, d);
            Mat vc = linear(&a, L->wv, L->bv, d);
            Mat ctx = mat(1, d);
            for (int h = 0; h < heads; h++) {
                int off = h * dh;
                const float* qi = q.a + off;
                float mx = -INFINITY;
                for (int j = 0; j <= n; j++) {
                    const float* kr = j < n ? row(&kv->k[l], j) : kc.a;
                    logits[j] = dot(qi, kr + off, dh) * scale;
                    mx = mx < logits[j] ? logits[j] : mx;
                }
                float denom = 0.0f;
                for (int j = 0; j <= n; j++) { logits[j] = expf(logits[j] - mx); denom += logits[j]; }
                float inv = 1.0f / denom;
                float* crow = ctx.a + off;
                for (int j = 0; j <= n; j++) {
                    const float* vr = j < n ? row(&kv->v[l], j) : vc.a;
                    axpy(logits[j] * inv, vr + off, crow, dh);
                }
            }
            cross_tail(L, cfg, &x, &ctx, l);
        }
        Mat h = mlp_forward(&M->phi_out, &x);
        memcpy(row(&out, (int)bi), h.a, sizeof(float) * d);
    }
    return out;
}

/* ------------------------------------------------------------------------ */
/* L5 ranking: finetune.cpp                                                  */

/* ctx_features (finetune.cpp:212-226) */
static void ctx_features(const dcat_batch* b, int64_t i, const dcat_finetune_config* ft, float* out) {
    double days = b->age_seconds[i] / 86400.0;
    CHECK(b->age_seconds[i] >= 0.0, "candidate age must be non-negative");
    for (int k = 0; k < 8; k++) out[k] = 0.0f;
    out[days < ft->fresh_days ? 0 : days < ft->mid_days ? 1 : 2] = 1.0f;
    float r = (float)b->row_valid[i] / (float)ft->max_events;
    out[3] = ft->max_events > 0 ? (r < 1.0f ? r : 1.0f) : 0.0f;
    if (b->row_valid[i] > 0) {
        int s = b->ev_surface[b->row_offset[i] + b->row_valid[i] - 1];
        out[4 + s] = 1.0f;
    }
}

/* crossing_forward + outputs_from (finetune.cpp:301-324, 350-359) */
static void crossing_forward(const dcat_head* hp, const dcat_finetune_config* ft, const float* sel,
                             const float* cand_emb, const dcat_batch* b, int64_t i, double* logit, double* mlogit,
                             double* prob) {
    int d_feat = hp->d_module + hp->d_emb + hp->n_ctx;
    Mat feat = mat(1, d_feat);
    if (hp->d_module > 0) memcpy(feat.a, sel, sizeof(float) * hp->d_module);
    memcpy(feat.a + hp->d_module, cand_emb, sizeof(float) * hp->d_emb);
    ctx_features(b, i, ft, feat.a + hp->d_module + hp->d_emb);
    Mat z1 = matmul(&feat, hp->w1, hp->hidden);
    for (int j = 0; j < hp->hidden; j++) z1.a[j] += hp->b1[j];
    Mat a1 = mat(1, hp->hidden);
    for (int j = 0; j < hp->hidden; j++) a1.a[j] = gelu(z1.a[j]);
    Mat lg = matmul(&a1, hp->w2, 3);
    for (int j = 0; j < 3; j++) lg.a[j] += hp->b2[j];
    Mat ml = mat(1, 3);
    if (hp->d_module > 0) {
        Mat selflat = {1, hp->d_module, (float*)sel};
        ml = matmul(&selflat, hp->mod_w, 3);
    }
    for (int j = 0; j < 3; j++) ml.a[j] += hp->mod_b[j];
    for (int j = 0; j < 3; j++) {
        double l = lg.a[j];
        logit[j] = l;
        prob[j] = 1.0 / (1.0 + exp(-l));
        mlogit[j] = ml.a[j];
    }
}

/* gather_selectors for the lite variants (finetune.cpp:258-274): the mean of H's rows
 * (axpy in row order, then one division per element) or its last row; zeros when empty. */
static void lite_selector(const Mat* H, int variant, float* sel, int d) {
    memset(sel, 0, sizeof(float) * d);
    if (H->rows <= 0) return;
    if (variant == DCAT_VARIANT_LITE_LAST) {
        memcpy(sel, row(H, H->rows - 1), sizeof(float) * d);
        return;
    }
    for (int r = 0; r < H->rows; r++) axpy(1.0f, row(H, r), sel, d);
    for (int j = 0; j < d; j++) sel[j] /= (float)H->rows;
}

/* build_input + forward_one (finetune.cpp:160-205, 326-348): the per-example path
 * rank_forward (finetune.cpp:403-409) for every fusion variant:
 *   Base / Aux: [seq; cand] -> selector H[cand];
 *   AuxLt: [seq; lt + pos[n]; cand] -> selectors [H[lt]; H[cand]] (d_module = 2 d);
 *   LiteMean / LiteLast: [seq] -> mean / last row of H (zeros for an empty sequence). */
static void rank_forward_one(const Model* M, const dcat_table* t, const dcat_head* hp, const dcat_finetune_config* ft,
                             const dcat_batch* b, int64_t i, double* logit, double* mlogit, double* prob) {
    const dcat_model_config* cfg = &M->cfg;
    CHECK(b->age_seconds[i] >= 0.0, "candidate age must be non-negative");
    float* cand_emb = (float*)amalloc(sizeof(float) * cfg->d_emb);
    lookup(t, b->candidate[i], cand_emb);
    if (!ft->use_seq_module) { crossing_forward(hp, ft, NULL, cand_emb, b, i, logit, mlogit, prob); return; }
    const int lite = ft->variant == DCAT_VARIANT_LITE_MEAN || ft->variant == DCAT_VARIANT_LITE_LAST;
    const int with_lt = ft->variant == DCAT_VARIANT_AUXLT;
    const int with_aux = ft->variant == DCAT_VARIANT_AUX || ft->variant == DCAT_VARIANT_AUXLT;
    int n_seq = b->row_valid[i];
    int n = lite ? n_seq : n_seq + (with_lt ? 2 : 1);
    CHECK(n <= cfg->max_len, "input of %d tokens exceeds max_len %d", n, cfg->max_len);
    Mat e = mat(n, cfg->d_emb);
    if (n_seq > 0) {
        Mat s = segment_inputs(M, t, b, b->row_offset[i], n_seq, 0);
        memcpy(e.a, s.a, sizeof(float) * (size_t)n_seq * cfg->d_emb);
    }
    if (!lite) {
        if (with_lt) { /* learnable token between context and candidate (finetune.cpp:186-191) */
            float* lrow = row(&e, n_seq);
            memcpy(lrow, hp->lt, sizeof(float) * cfg->d_emb);
            if (cfg->pos_learned) axpy(1.0f, M->pos_emb + (size_t)n_seq * cfg->d_emb, lrow, cfg->d_emb);
        }
        float* crow = row(&e, n - 1);
        memcpy(crow, cand_emb, sizeof(float) * cfg->d_emb);
        if (with_aux) {
            CHECK(b->aux != NULL && b->d_aux > 0, "variant requires an auxiliary embedding");
            CHECK(b->d_aux == hp->d_aux, "aux dim %d != projector rows %d", b->d_aux, hp->d_aux);
            for (int r = 0; r < hp->d_aux; r++)
                axpy(b->aux[(size_t)i * b->d_aux + r], hp->aux_proj + (size_t)r * hp->d_emb, crow, cfg->d_emb);
        }
        if (cfg->pos_learned) axpy(1.0f, M->pos_emb + (size_t)(n - 1) * cfg->d_emb, crow, cfg->d_emb);
    }
    Mat H = n > 0 ? forward_rows(M, &e) : mat(0, cfg->d_model);
    int d = cfg->d_model;
    float* sel = (float*)amalloc(sizeof(float) * 2 * d);
    if (lite) {
        lite_selector(&H, ft->variant, sel, d);
    } else if (with_lt) {
        memcpy(sel, row(&H, n - 2), sizeof(float) * d);
        memcpy(sel + d, row(&H, n - 1), sizeof(float) * d);
    } else {
        memcpy(sel, row(&H, n - 1), sizeof(float) * d);
    }
    crossing_forward(hp, ft, sel, cand_emb, b, i, logit, mlogit, prob);
}

static void validate_batch(const dcat_batch* b) {
    CHECK(b->n_rows >= 0, "negative row count");
    for (int64_t i = 0; i < b->n_rows; i++) {
        CHECK(b->row_valid[i] >= 0, "row %lld: negative valid", (long long)i);
        CHECK(b->row_offset[i] >= 0 && b->row_offset[i] + b->row_valid[i] <= b->n_events,
              "row %lld: events out of range", (long long)i);
    }
}

/* Fixed-window view of a batch for the sequence module (context_forward_fixed,
 * dcat.cpp:300-313): row i keeps its newest kept = min(valid, window - 1) events,
 * positions restarting at 0. The reference stores them in a ring of `window`
 * slots with the candidate in the free slot; the scores are rotation invariant
 * (test_dcat.cpp:341-361) and equal the truncate-then-forward DCAT result
 * (test_dcat.cpp:300-339), which is what this view feeds to the plain path. */
static dcat_batch window_view(const dcat_batch* b, int window) {
    dcat_batch v = *b;
    int64_t B = b->n_rows;
    int64_t* off = (int64_t*)amalloc(sizeof(int64_t) * (B ? B : 1));
    int32_t* val = (int32_t*)amalloc(sizeof(int32_t) * (B ? B : 1));
    for (int64_t i = 0; i < B; i++) {
        int kept = b->row_valid[i] < window - 1 ? b->row_valid[i] : window - 1;
        off[i] = b->row_offset[i] + (b->row_valid[i] - kept);
        val[i] = kept;
    }
    v.row_offset = off;
    v.row_valid = val;
    return v;
}

static int run_rank_batch(const Model* M, const dcat_table* t, const dcat_head* hp, const dcat_finetune_config* ft,
                          const dcat_batch* b, double* logits, double* mlogits, double* probs, float* h_cand) {
    const dcat_model_config* cfg = &M->cfg;
    int64_t B = b->n_rows;
    if (B == 0) return 0;
    CHECK(ft->variant >= DCAT_VARIANT_BASE && ft->variant <= DCAT_VARIANT_LITE_LAST, "unknown fusion variant %d",
          ft->variant);
    const int lite = ft->variant == DCAT_VARIANT_LITE_MEAN || ft->variant == DCAT_VARIANT_LITE_LAST;
    /* FinetuneConfig::validate essentials (finetune.cpp:54-72) */
    CHECK(cfg->max_len >= ft->max_events + 2, "model.max_len %d too small for max_events %d plus candidate tokens",
          cfg->max_len, ft->max_events);
    CHECK(ft->use_seq_module || ft->variant == DCAT_VARIANT_BASE,
          "disabling the sequence module requires the base variant");
    CHECK(ft->window >= 0, "context_forward_fixed: window must be >= 1, got %d", ft->window);
    const int fixed = ft->use_seq_module && ft->window > 0;
    int empty_seq = 0;
    for (int64_t i = 0; i < B; i++) empty_seq |= b->row_valid[i] == 0;
    /* finetune.cpp:428-431: no sequence module, AuxLt, or an empty sequence run one example at
     * a time (the fixed-window path has no such fallback: cross_forward_fixed handles an
     * empty ring, dcat.cpp:360-390) */
    if (!ft->use_seq_module || ft->variant == DCAT_VARIANT_AUXLT || (empty_seq && !fixed)) {
        for (int64_t i = 0; i < B; i++)
            rank_forward_one(M, t, hp, ft, b, i, logits + 3 * i, mlogits + 3 * i, probs + 3 * i);
        return 0;
    }
    int32_t* rep = (int32_t*)amalloc(sizeof(int32_t) * B);
    int32_t* first = (int32_t*)amalloc(sizeof(int32_t) * B);
    int b_u = dedup(b, rep, first); /* dedup keys on the full prefix in both variants */
    if (lite) { /* finetune.cpp:439-456: the candidate-independent selector once per unique */
        const int d = cfg->d_model;
        float* sel_u = (float*)amalloc(sizeof(float) * (size_t)(b_u ? b_u : 1) * d);
        for (int u = 0; u < b_u; u++) {
            const int64_t r0 = first[u];
            Mat e = segment_inputs(M, t, b, b->row_offset[r0], b->row_valid[r0], 0);
            Mat H = forward_rows(M, &e);
            lite_selector(&H, ft->variant, sel_u + (size_t)u * d, d);
        }
        float* cand_emb = (float*)amalloc(sizeof(float) * cfg->d_emb);
        for (int64_t i = 0; i < B; i++) {
            CHECK(b->age_seconds[i] >= 0.0, "candidate age must be non-negative");
            lookup(t, b->candidate[i], cand_emb);
            crossing_forward(hp, ft, sel_u + (size_t)rep[i] * d, cand_emb, b, i, logits + 3 * i, mlogits + 3 * i,
                             probs + 3 * i);
        }
        return 0;
    }
    dcat_batch sb = fixed ? window_view(b, ft->window) : *b;
    SeqKV* cache = context_forward(M, t, &sb, first, b_u);
    uint64_t* items = (uint64_t*)amalloc(sizeof(uint64_t) * B);
    int* pos = (int*)amalloc(sizeof(int) * B);
    for (int64_t i = 0; i < B; i++) { items[i] = b->candidate[i]; pos[i] = sb.row_valid[first[rep[i]]]; }
    Mat e_cand = candidate_inputs(M, t, items, pos, B);
    if (ft->variant == DCAT_VARIANT_AUX) { /* finetune.cpp:469-479 */
        CHECK(b->aux != NULL && b->d_aux > 0, "variant 'aux' requires an auxiliary embedding");
        CHECK(b->d_aux == hp->d_aux, "aux dim mismatch in batch");
        for (int64_t i = 0; i < B; i++)
            for (int r = 0; r < hp->d_aux; r++)
                axpy(b->aux[(size_t)i * b->d_aux + r], hp->aux_proj + (size_t)r * hp->d_emb, row(&e_cand, (int)i),
                     cfg->d_emb);
    }
    Mat H = cross_forward(M, cache, b_u, rep, B, &e_cand);
    float* cand_emb = (float*)amalloc(sizeof(float) * cfg->d_emb);
    for (int64_t i = 0; i < B; i++) {
        CHECK(b->age_seconds[i] >= 0.0, "candidate age must be non-negative");
        lookup(t, b->candidate[i], cand_emb);
        crossing_forward(hp, ft, row(&H, (int)i), cand_emb, b, i, logits + 3 * i, mlogits + 3 * i, probs + 3 * i);
    }
    if (h_cand) memcpy(h_cand, H.a, sizeof(float) * (size_t)B * cfg->d_model);
    return 1;
}

/* ------------------------------------------------------------------------ */
/* API                                                                       */

int oracle_param_count(const dcat_model_config* cfg) { return n_tensors(cfg); }

int oracle_param_shapes(const dcat_model_config* c, int32_t* rows, int32_t* cols) {
    int t = 0, d = c->d_model, dff = d * c->mlp_ratio;
#define SH(r_, c_) do { rows[t] = (r_); cols[t] = (c_); t++; } while (0)
    SH(1, 1);
    SH(c->n_actions, c->d_emb);
    SH(c->n_surfaces, c->d_emb);
    if (c->pos_learned) SH(c->max_len, c->d_emb);
    int dins[3] = {c->d_emb, d, c->d_emb};
    for (int i = 0; i < 3; i++) { SH(dins[i], d); SH(1, d); SH(d, d); SH(1, d); }
    for (int l = 0; l < c->n_layers; l++) {
        SH(1, d); SH(1, d);
        for (int k = 0; k < 4; k++) { SH(d, d); SH(1, d); }
        SH(1, d); SH(1, d);
        SH(d, dff); SH(1, dff); SH(dff, d); SH(1, d);
    }
#undef SH
    return t;
}

static void mlp_init(float* w1, float* b1, float* w2, float* b2, int d_in, int d_hidden, int d_out, Rng* r) {
    /* MlpP::init (model.cpp:128-142) */
    init_gaussian(w1, (size_t)d_in * d_hidden, r, sqrtf(2.0f / (float)d_in));
    init_gaussian(w2, (size_t)d_hidden * d_out, r, sqrtf(2.0f / (float)d_hidden));
    init_gaussian(b1, (size_t)d_hidden, r, 0.002f);
    init_gaussian(b2, (size_t)d_out, r, 0.002f);
}

int oracle_init_transformer(const dcat_model_config* c, uint64_t seed, float tau_init, float* const* out) {
    API_BEGIN
    model_config_validate(c);
    CHECK(tau_init > 0.0f, "tau_init must be positive");
    int nt = n_tensors(c);
    int32_t* rows = (int32_t*)amalloc(sizeof(int32_t) * nt);
    int32_t* cols = (int32_t*)amalloc(sizeof(int32_t) * nt);
    oracle_param_shapes(c, rows, cols);
    for (int i = 0; i < nt; i++) memset(out[i], 0, sizeof(float) * (size_t)rows[i] * cols[i]);
    Rng r = rng_make(mix64(seed ^ 0x6d6f64656cULL));
    int d = c->d_model, dff = d * c->mlp_ratio;
    int base = 3 + (c->pos_learned ? 1 : 0) + 12;
    /* layers first (model.cpp:228-250) */
    for (int l = 0; l < c->n_layers; l++) {
        float* const* L = out + base + 16 * l;
        for (int k = 0; k < d; k++) { L[0][k] = 1.0f; L[10][k] = 1.0f; } /* ln1_g, ln2_g */
        init_gaussian(L[2], (size_t)d * d, &r, 0.02f);   /* wq */
        init_gaussian(L[4], (size_t)d * d, &r, 0.02f);   /* wk */
        init_gaussian(L[6], (size_t)d * d, &r, 0.02f);   /* wv */
        init_gaussian(L[8], (size_t)d * d, &r, 0.02f);   /* wo */
        init_gaussian(L[12], (size_t)d * dff, &r, 0.02f); /* fw1 */
        init_gaussian(L[14], (size_t)dff * d, &r, 0.02f); /* fw2 */
    }
    int t = 3 + (c->pos_learned ? 1 : 0);
    mlp_init(out[t], out[t + 1], out[t + 2], out[t + 3], c->d_emb, d, d, &r); /* phi_in */
    mlp_init(out[t + 4], out[t + 5], out[t + 6], out[t + 7], d, d, d, &r);    /* phi_out */
    mlp_init(out[t + 8], out[t + 9], out[t + 10], out[t + 11], c->d_emb, d, d, &r); /* psi */
    init_gaussian(out[1], (size_t)c->n_actions * c->d_emb, &r, 0.02f);
    init_gaussian(out[2], (size_t)c->n_surfaces * c->d_emb, &r, 0.02f);
    if (c->pos_learned) init_gaussian(out[3], (size_t)c->max_len * c->d_emb, &r, 0.02f);
    out[0][0] = logf(tau_init);
    API_END
}

int oracle_init_table(int32_t J, int32_t R, int32_t d_sub, uint64_t seed, float stddev, uint64_t* seeds, float* data) {
    API_BEGIN
    CHECK(J >= 1 && R >= 1 && d_sub >= 1, "HashedEmbeddingTable: bad shape");
    Rng r = rng_make(mix64(seed ^ 0x656d62ULL));
    for (int j = 0; j < J; j++) seeds[j] = mix64(seed ^ (0x5eedULL + (uint64_t)j));
    init_gaussian(data, (size_t)J * R * d_sub, &r, stddev);
    API_END
}

int oracle_init_head(int32_t d_model, int32_t d_emb, int32_t d_aux, int32_t n_ctx, int32_t hidden, int32_t sel,
                     uint64_t seed, float* w1, float* b1, float* w2, float* b2, float* mod_w, float* mod_b,
                     float* aux_proj, float* lt) {
    API_BEGIN
    int d_module = sel * d_model;
    int d_feat = d_module + d_emb + n_ctx;
    Rng r = rng_make(mix64(seed ^ 0x72616e6bULL));
    memset(b1, 0, sizeof(float) * hidden);
    memset(b2, 0, sizeof(float) * 3);
    memset(mod_b, 0, sizeof(float) * 3);
    memset(aux_proj, 0, sizeof(float) * (size_t)d_aux * d_emb);
    init_gaussian(w1, (size_t)d_feat * hidden, &r, sqrtf(2.0f / (float)d_feat));
    init_gaussian(w2, (size_t)hidden * 3, &r, 0.02f);
    init_gaussian(mod_w, (size_t)d_module * 3, &r, 0.02f);
    init_gaussian(lt, (size_t)d_emb, &r, 0.02f);
    API_END
}

int oracle_dedup(const dcat_batch* batch, int32_t* rep, int32_t* first, int32_t* b_u) {
    API_BEGIN
    validate_batch(batch);
    *b_u = dedup(batch, rep, first);
    API_END
}

int oracle_rank_forward_batch(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                              const dcat_head* head, const dcat_finetune_config* ft, const dcat_batch* batch,
                              double* logits, double* module_logits, double* probs, float* h_cand,
                              int32_t* used_dcat) {
    API_BEGIN
    Model M = bind_model(cfg, params);
    validate_batch(batch);
    int used = run_rank_batch(&M, table, head, ft, batch, logits, module_logits, probs, h_cand);
    if (used_dcat) *used_dcat = used;
    API_END
}

int oracle_context_kv(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                      const dcat_batch* uniques, int32_t layer, int32_t unique, float* k, float* v) {
    API_BEGIN
    Model M = bind_model(cfg, params);
    validate_batch(uniques);
    CHECK(unique >= 0 && unique < uniques->n_rows, "unique out of range");
    CHECK(layer >= 0 && layer < cfg->n_layers, "layer out of range");
    int32_t one = unique;
    SeqKV* kv = context_forward(&M, table, uniques, &one, 1);
    size_t n = (size_t)kv[0].n * cfg->d_model;
    memcpy(k, kv[0].k[layer].a, sizeof(float) * n);
    memcpy(v, kv[0].v[layer].a, sizeof(float) * n);
    API_END
}

int oracle_naive_candidate_outputs(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                                   const dcat_batch* b, float* out) {
    API_BEGIN
    Model M = bind_model(cfg, params);
    validate_batch(b);
    int d = cfg->d_model;
    for (int64_t i = 0; i < b->n_rows; i++) { /* dcat.cpp:423-433 */
        int n = b->row_valid[i];
        Mat e = segment_inputs(&M, table, b, b->row_offset[i], n, 0);
        int pos = n;
        Mat ec = candidate_inputs(&M, table, &b->candidate[i], &pos, 1);
        Mat e2 = mat(n + 1, cfg->d_emb);
        if (n > 0) memcpy(e2.a, e.a, sizeof(float) * (size_t)n * cfg->d_emb);
        memcpy(row(&e2, n), ec.a, sizeof(float) * cfg->d_emb);
        Mat h = forward_rows(&M, &e2);
        memcpy(out + (size_t)i * d, row(&h, n), sizeof(float) * d);
    }
    API_END
}

/* quantize (embed.cpp:124-171): per-row min-max; bias = half(min), scale =
 * half((max - min) / (2^b - 1)); codes = round-half-even((x - bias) / scale)
 * clamped to [0, 2^b - 1]; a non-positive scale stores 0 and zero codes. */
int oracle_quantize_table(const dcat_table* t, int32_t bits, uint8_t* packed) {
    API_BEGIN
    CHECK(bits == 4 || bits == 8, "quantize: bits must be 4 or 8, got %d", bits);
    dcat_table q = *t;
    q.bits = bits;
    const int cb = q_code_bytes(&q), rb = q_row_bytes(&q);
    const uint32_t max_code = (1u << bits) - 1;
    memset(packed, 0, (size_t)t->num_subtables * t->rows * rb);
    for (int j = 0; j < t->num_subtables; j++)
        for (int r = 0; r < t->rows; r++) {
            const float* src = t->subtables[j] + (size_t)r * t->d_sub;
            float lo = src[0], hi = src[0];
            for (int e = 0; e < t->d_sub; e++) {
                CHECK(isfinite(src[e]), "quantize: non-finite value at subtable %d row %d elem %d", j, r, e);
                lo = src[e] < lo ? src[e] : lo;
                hi = src[e] > hi ? src[e] : hi;
            }
            float bias = f16_to_f32(f32_to_f16(lo));
            float scale = f16_to_f32(f32_to_f16((hi - lo) / (float)max_code));
            uint8_t* dst = packed + ((size_t)j * t->rows + r) * rb;
            if (scale > 0.0f) {
                for (int e = 0; e < t->d_sub; e++) {
                    long c = lrintf((src[e] - bias) / scale);
                    c = c < 0 ? 0 : (c > (long)max_code ? (long)max_code : c);
                    if (bits == 8) dst[e] = (uint8_t)c;
                    else dst[e / 2] |= (uint8_t)(c << ((e % 2) * 4));
                }
            } else {
                scale = 0.0f;
            }
            uint16_t sb = f32_to_f16(scale), bb = f32_to_f16(bias);
            dst[cb] = (uint8_t)(sb & 255); dst[cb + 1] = (uint8_t)(sb >> 8);
            dst[cb + 2] = (uint8_t)(bb & 255); dst[cb + 3] = (uint8_t)(bb >> 8);
        }
    API_END
}

int oracle_dcat_outputs_fixed(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                              const dcat_batch* b, int32_t window, float* h_cand) {
    API_BEGIN
    Model M = bind_model(cfg, params);
    validate_batch(b);
    CHECK(window >= 1, "context_forward_fixed: window must be >= 1, got %d", window);
    int64_t B = b->n_rows;
    int32_t* rep = (int32_t*)amalloc(sizeof(int32_t) * (B ? B : 1));
    int32_t* first = (int32_t*)amalloc(sizeof(int32_t) * (B ? B : 1));
    int b_u = dedup(b, rep, first);
    dcat_batch sb = window_view(b, window);
    SeqKV* cache = context_forward(&M, table, &sb, first, b_u);
    int* pos = (int*)amalloc(sizeof(int) * (B ? B : 1));
    for (int64_t i = 0; i < B; i++) pos[i] = sb.row_valid[first[rep[i]]];
    Mat e_cand = candidate_inputs(&M, table, b->candidate, pos, B);
    Mat H = cross_forward(&M, cache, b_u, rep, B, &e_cand);
    memcpy(h_cand, H.a, sizeof(float) * (size_t)B * cfg->d_model);
    API_END
}

int oracle_dcat_outputs(const dcat_model_config* cfg, const dcat_params* params, const dcat_table* table,
                        const dcat_batch* b, float* h_cand) {
    API_BEGIN
    Model M = bind_model(cfg, params);
    validate_batch(b);
    int64_t B = b->n_rows;
    int32_t* rep = (int32_t*)amalloc(sizeof(int32_t) * (B ? B : 1));
    int32_t* first = (int32_t*)amalloc(sizeof(int32_t) * (B ? B : 1));
    int b_u = dedup(b, rep, first);
    SeqKV* cache = context_forward(&M, table, b, first, b_u);
    int* pos = (int*)amalloc(sizeof(int) * (B ? B : 1));
    for (int64_t i = 0; i < B; i++) pos[i] = b->row_valid[first[rep[i]]];
    Mat e_cand = candidate_inputs(&M, table, b->candidate, pos, B);
    Mat H = cross_forward(&M, cache, b_u, rep, B, &e_cand);
    memcpy(h_cand, H.a, sizeof(float) * (size_t)B * cfg->d_model);
    API_END
}
