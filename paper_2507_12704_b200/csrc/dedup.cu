// dedup.cu — K1: bit-exact request-batch deduplication on the device.
//
// Replaces dedup_segments (/root/reference/proj/src/dcat.cpp:91-108), whose
// key is segment_key (dcat.cpp:45-56): the 18 bytes (ts u64, action u8,
// surface u8, item u64) of each event of the valid prefix. Uniques are
// numbered in first-appearance order and rep[i] names row i's unique.
//
// Device recipe (no sort, no CPU fallback):
//   1. one warp per row hashes its key into 64 bits (and validates enums /
//      positions like segment_inputs, model.cpp:524-535);
//   2. rows insert (hash -> min row) into an open-addressing table with
//      atomicCAS + atomicMin: the slot's min row is the first appearance of
//      that hash;
//   3. every row byte-compares its key with that first row; a mismatch is a
//      genuine 64-bit collision and the row is re-keyed with a fresh seed in
//      a repair round (rows of one content class always collide together, so
//      classes never straddle rounds); after a few rounds an exact pairwise
//      pass settles the rest;
//   4. uid = exclusive scan of (head == row) in row order gives the reference's
//      first-appearance numbering; rep = uid[head].
// Then the rows are grouped by unique (counting sort), and the per-unique
// context-token and attention-tile offsets are scanned.
#include "launch.h"

namespace dcat {

namespace {

constexpr uint64_t kEmpty = ~0ull;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ void record_error(Status* st, int bit, int row, int val) {
    atomicOr(&st->err_bits, bit);
    int prev = atomicMin(&st->err_row, row);
    if (row < prev) atomicExch(&st->err_val, val);
}

// content hash of row r (one warp) + validation of its events (round 0)
__device__ void hash_row(const DedupIn& in, int r, uint64_t seed, uint64_t mask, uint64_t* hash, Status* st,
                         int validate, int lane) {
    int valid = in.row_valid[r];
    int64_t off = in.row_offset[r];
    if (validate) {
        if (valid < 0 || off < 0 || off + valid > in.n_events) {
            if (lane == 0) record_error(st, ERR_RANGE, r, valid);
            return;
        }
        if (in.pos_learned && lane == 0) {
            const int pv = seq_tokens(in, valid);  // positions used: context 0..pv-1, candidate pv
            if (pv > in.max_len) record_error(st, ERR_POS_CTX, r, pv - 1 >= in.max_len ? in.max_len : pv);
            else if (pv >= in.max_len) record_error(st, ERR_POS_CAND, r, pv);
        }
    }
    uint64_t sa = mix64(seed ^ 0x7473ull), sb = mix64(seed ^ 0x6974656dull);
    uint64_t acc = 0;
    for (int e = lane; e < valid; e += 32) {
        uint64_t t = in.ts[off + e];
        uint32_t a = in.action[off + e];
        uint32_t s = in.surface[off + e];
        uint64_t it = in.item[off + e];
        if (validate) {
            if (a >= static_cast<uint32_t>(in.n_actions)) record_error(st, ERR_ACTION, r, static_cast<int>(a));
            if (s >= static_cast<uint32_t>(in.n_surfaces)) record_error(st, ERR_SURFACE, r, static_cast<int>(s));
        }
        uint64_t tag = static_cast<uint64_t>(a) | (static_cast<uint64_t>(s) << 8) |
                       (static_cast<uint64_t>(e) << 16);
        acc += mix64(mix64(mix64(t ^ sa) ^ it ^ sb) ^ tag);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        uint64_t h = mix64(acc ^ mix64(static_cast<uint64_t>(valid) + seed)) & mask;
        if (h == kEmpty) h = kEmpty - 1;
        hash[r] = h;
    }
}

__global__ void k_hash(DedupIn in, const int32_t* rows, const int32_t* n_rows_dev, int64_t n_rows, uint64_t seed,
                       uint64_t mask, uint64_t* hash, Status* st, int validate) {
    const int64_t n = n_rows_dev ? *n_rows_dev : n_rows;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n; w += nw) {
        const int r = rows ? rows[w] : static_cast<int>(w);
        hash_row(in, r, seed, mask, hash, st, validate, lane);
    }
}

// span fast path (round 0): rows with the same (row_offset, row_valid) are the same key
// (dcat.cpp:45-56 compares contents; a shared span trivially compares equal), so only one
// row per distinct span is content-hashed. k_span also performs the per-row range checks.
constexpr uint64_t kSpanOffLimit = 1ull << 42;
__global__ void k_span(DedupIn in, uint64_t* tkey, int32_t* tval, int64_t cap, int32_t* span_slot, Status* st) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= in.B) return;
    const int r = static_cast<int>(i);
    const int valid = in.row_valid[r];
    const int64_t off = in.row_offset[r];
    span_slot[r] = -1;
    if (valid < 0 || off < 0 || off + valid > in.n_events) {
        record_error(st, ERR_RANGE, r, valid);
        return;
    }
    if (in.pos_learned) {
        const int pv = seq_tokens(in, valid);  // positions used: context 0..pv-1, candidate pv
        if (pv > in.max_len) record_error(st, ERR_POS_CTX, r, pv - 1 >= in.max_len ? in.max_len : pv);
        else if (pv >= in.max_len) record_error(st, ERR_POS_CAND, r, pv);
    }
    if (static_cast<uint64_t>(off) >= kSpanOffLimit || valid >= (1 << 21)) return;  // hashed on its own
    const uint64_t key = (static_cast<uint64_t>(off) << 21) | static_cast<uint64_t>(valid);
    const uint64_t m = static_cast<uint64_t>(cap - 1);
    for (uint64_t s = mix64(key) & m;; s = (s + 1) & m) {
        const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkey + s), kEmpty, key);
        if (prev == kEmpty || prev == key) {
            atomicMin(tval + s, r);
            span_slot[r] = static_cast<int32_t>(s);
            return;
        }
    }
}
// rows to content-hash: the first row of every span, and rows outside the span path
__global__ void k_span_reps(int64_t B, const int32_t* span_slot, const int32_t* tval, const Status* st,
                            int32_t* list, int32_t* list_n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const int s = span_slot[i];
    if (s >= 0 ? tval[s] == static_cast<int32_t>(i) : true) list[atomicAdd(list_n, 1)] = static_cast<int32_t>(i);
}
__global__ void k_span_copy(int64_t B, const int32_t* span_slot, const int32_t* tval, uint64_t* hash) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const int s = span_slot[i];
    if (s >= 0) {
        const int h = tval[s];
        if (h != static_cast<int32_t>(i)) hash[i] = hash[h];
    }
}

__global__ void k_insert(const int32_t* rows, const int32_t* n_rows_dev, int64_t n_rows, const uint64_t* hash,
                         uint64_t* tkey, int32_t* tval, int64_t cap, int32_t* slot) {
    int64_t n = n_rows_dev ? *n_rows_dev : n_rows;
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int r = rows ? rows[i] : static_cast<int>(i);
    uint64_t h = hash[r];
    uint64_t mask = static_cast<uint64_t>(cap - 1);
    uint64_t s = mix64(h) & mask;
    for (;;) {
        unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkey + s), kEmpty, h);
        if (prev == kEmpty || prev == h) {
            atomicMin(tval + s, r);
            slot[r] = static_cast<int32_t>(s);
            return;
        }
        s = (s + 1) & mask;
    }
}

// warp-cooperative key equality of rows a and b (dcat.cpp:45-56 semantics)
__device__ bool same_key(const DedupIn& in, int a, int b, int lane) {
    int va = in.row_valid[a];
    if (va != in.row_valid[b]) return false;
    int64_t oa = in.row_offset[a], ob = in.row_offset[b];
    if (oa == ob) return true;
    bool diff = false;
    for (int e = lane; e < va; e += 32) {
        diff |= in.ts[oa + e] != in.ts[ob + e];
        diff |= in.action[oa + e] != in.action[ob + e];
        diff |= in.surface[oa + e] != in.surface[ob + e];
        diff |= in.item[oa + e] != in.item[ob + e];
    }
    return __ballot_sync(0xffffffffu, diff) == 0;
}

__global__ void k_head_verify(DedupIn in, const int32_t* rows, const int32_t* n_rows_dev, int64_t n_rows,
                              const int32_t* slot, const int32_t* tval, int32_t* head, int32_t* collided,
                              Status* st) {
    const int64_t n = n_rows_dev ? *n_rows_dev : n_rows;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n; w += nw) {
        const int r = rows ? rows[w] : static_cast<int>(w);
        const int h = tval[slot[r]];
        const bool ok = (h == r) || same_key(in, r, h, lane);
        if (lane == 0) {
            head[r] = ok ? h : r;
            collided[r] = ok ? 0 : 1;
            if (!ok) atomicAdd(&st->collisions, 1);
        }
    }
}

// round 0, one thread per row: rows whose table head is themselves or shares their event span
// are settled here; the rest go to a list for the warp-cooperative content comparison
__global__ void k_verify_fast(DedupIn in, const int32_t* slot, const int32_t* tval, int32_t* head,
                              int32_t* collided, int32_t* list, int32_t* list_n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= in.B) return;
    const int r = static_cast<int>(i);
    const int h = tval[slot[r]];
    if (h == r || (in.row_valid[r] == in.row_valid[h] && in.row_offset[r] == in.row_offset[h])) {
        head[r] = h;
        collided[r] = 0;
    } else {
        list[atomicAdd(list_n, 1)] = r;
    }
}

__global__ void k_compact(int64_t B, const int32_t* collided, int32_t* list, int32_t* list_n) {
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B || !collided[i]) return;
    list[atomicAdd(list_n, 1)] = static_cast<int32_t>(i);
}

// exact pairwise settlement of the rows still colliding after the re-keyed rounds
__global__ void k_exact(DedupIn in, const int32_t* list, const int32_t* list_n, int32_t* head, int32_t* collided) {
    int n = *list_n;
    int lane = threadIdx.x & 31;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
        int r = list[w];
        int best = r;
        for (int j = 0; j < n; j++) {
            int c = list[j];
            if (c < best && same_key(in, r, c, lane)) best = c;
        }
        if (lane == 0) {
            head[r] = best;
            collided[r] = 0;
        }
    }
}

__global__ void k_first_flags(int64_t B, const int32_t* head, int64_t* flags) {
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < B) flags[i] = head[i] == i ? 1 : 0;
}

__global__ void k_rep(int64_t B, const int32_t* head, const int64_t* uid, int32_t* rep, int32_t* first, int32_t* cnt,
                      Status* st) {
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i == 0) st->b_u = static_cast<int>(uid[B]);
    if (i >= B) return;
    int h = head[i];
    int u = static_cast<int>(uid[h]);
    rep[i] = u;
    if (h == i) first[u] = static_cast<int32_t>(i);
    atomicAdd(cnt + u, 1);
}

// per-unique scan inputs: candidate count, context tokens, tile counts
__global__ void k_unique_sizes(int64_t B, DedupIn in, const int32_t* first, const int32_t* cnt, const Status* st,
                               int tile_ctx, int tile_cross, int64_t* a_cnt, int64_t* a_tok, int64_t* a_ctx_t,
                               int64_t* a_cross_t) {
    int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (u >= B) return;
    int b_u = st->b_u;
    if (u < b_u) {
        int n = seq_tokens(in, in.row_valid[first[u]]);
        int c = cnt[u];
        a_cnt[u] = c;
        a_tok[u] = n;
        a_ctx_t[u] = (n + tile_ctx - 1) / tile_ctx;
        a_cross_t[u] = (c + tile_cross - 1) / tile_cross;
    } else {
        a_cnt[u] = a_tok[u] = a_ctx_t[u] = a_cross_t[u] = 0;
    }
}

__global__ void k_totals(int64_t B, const int64_t* tok_off, const int64_t* ctx_toff, const int64_t* cross_toff,
                         const int32_t* cnt, Status* st) {
    st->ctx_tokens = tok_off[B];
    st->ctx_tiles = static_cast<int>(ctx_toff[B]);
    st->cross_tiles = static_cast<int>(cross_toff[B]);
}

__global__ void k_perm(int64_t B, const int32_t* rep, const int64_t* goff, int32_t* cursor, int32_t* perm) {
    int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B) return;
    int u = rep[i];
    perm[goff[u] + atomicAdd(cursor + u, 1)] = static_cast<int32_t>(i);
}

// ---- exclusive scan (3 kernels: block sums, scan of sums, block rescans) ----

__device__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
    __shared__ int64_t warp_tot[32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        int64_t t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) warp_tot[lane] = t;
    }
    __syncthreads();
    int64_t base = wid > 0 ? warp_tot[wid - 1] : 0;
    if (total) *total = warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
    return base + x - v;
}

// Up to 4 independent exclusive scans of n items in one launch sequence: blockIdx.y picks the
// array, each with its own block-sum row in blk (stride kScanTile + 1).
struct ScanSet {
    const int64_t* in[4];
    int64_t* out[4];
};

__global__ void k_scan_sums(ScanSet x, int64_t n, int64_t* blk) {
    const int64_t* in = x.in[blockIdx.y];
    blk += blockIdx.y * (kScanTile + 1);
    int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++)
        if (base + k < n) s += in[base + k];
    int64_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void k_scan_top(int64_t* blk, int64_t nb) {
    // one block per array; nb <= kScanTile
    blk += blockIdx.x * (kScanTile + 1);
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = threadIdx.x * kScanItems + k;
        v[k] = idx < nb ? blk[idx] : 0;
        s += v[k];
    }
    int64_t tot;
    int64_t pre = block_exclusive_scan(s, &tot);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = threadIdx.x * kScanItems + k;
        if (idx < nb) blk[idx] = pre;
        pre += v[k];
    }
    if (threadIdx.x == 0) blk[nb] = tot;
}

__global__ void k_scan_apply(ScanSet x, int64_t n, const int64_t* blk, int64_t nb) {
    const int64_t* in = x.in[blockIdx.y];
    int64_t* out = x.out[blockIdx.y];
    blk += blockIdx.y * (kScanTile + 1);
    int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    int64_t pre = block_exclusive_scan(s, nullptr) + blk[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) out[base + k] = pre;
        pre += v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = blk[nb];
}

__global__ void k_tok_unique(const int64_t* tok_off, const Status* st, int32_t* tok_unique) {
    int b_u = st->b_u;
    for (int u = blockIdx.x; u < b_u; u += gridDim.x) {
        int64_t a = tok_off[u], b = tok_off[u + 1];
        for (int64_t t = a + threadIdx.x; t < b; t += blockDim.x) tok_unique[t] = u;
    }
}

__global__ void k_tiles(DedupIn in, const int32_t* first, const int32_t* cnt, const int64_t* tok_off,
                        const int64_t* goff, const int64_t* ctx_toff, const int64_t* cross_toff, const Status* st,
                        int tile_ctx, int tile_cross, Tile* ctx_tiles, Tile* cross_tiles) {
    int b_u = st->b_u;
    int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (u >= b_u) return;
    int n = seq_tokens(in, in.row_valid[first[u]]);
    int c = cnt[u];
    int64_t t0 = ctx_toff[u];
    for (int j = 0; j * tile_ctx < n; j++) {
        Tile t;
        t.q0 = static_cast<int>(tok_off[u]) + j * tile_ctx;
        t.nq = min(tile_ctx, n - j * tile_ctx);
        t.kv0 = static_cast<int>(tok_off[u]);
        t.nkv = min(n, (j + 1) * tile_ctx);
        t.qloc = j * tile_ctx;
        t.u = static_cast<int>(u);
        t.pad0 = t.pad1 = 0;
        ctx_tiles[t0 + j] = t;
    }
    int64_t c0 = cross_toff[u];
    for (int j = 0; j * tile_cross < c; j++) {
        Tile t;
        t.q0 = static_cast<int>(goff[u]) + j * tile_cross;
        t.nq = min(tile_cross, c - j * tile_cross);
        t.kv0 = static_cast<int>(tok_off[u]);
        t.nkv = n;
        t.qloc = 0;
        t.u = static_cast<int>(u);
        t.pad0 = t.pad1 = 0;
        cross_tiles[c0 + j] = t;
    }
}

inline unsigned grid_for(int64_t n, int per_block) { return static_cast<unsigned>((n + per_block - 1) / per_block); }
// grid for the grid-stride warp-per-row kernels (256 threads): <= 8 resident blocks per SM
inline unsigned warp_grid(int64_t rows) {
    const int64_t g = (rows * 32 + 255) / 256;
    return static_cast<unsigned>(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

}  // namespace

// exclusive scans (out[n] = total) of `count` arrays of n items; in place when in == out (each
// thread of k_scan_apply reads only the items it writes). blk: count * (kScanTile + 1) items.
static void scan_multi(const ScanSet& x, int count, int64_t n, int64_t* blk, cudaStream_t s) {
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 0) nb = 1;
    if (nb > kScanTile) throw InvalidArg("scan: batch too large (max 16M rows)");
    const dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>(count));
    k_scan_sums<<<grid, kScanThreads, 0, s>>>(x, n, blk);
    k_scan_top<<<count, kScanThreads, 0, s>>>(blk, nb);
    k_scan_apply<<<grid, kScanThreads, 0, s>>>(x, n, blk, nb);
    DCAT_LAUNCH_CHECK();
}

void scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* blk, cudaStream_t s) {
    ScanSet x{};
    x.in[0] = in;
    x.out[0] = out;
    scan_multi(x, 1, n, blk, s);
}

// uid / rep / groups / offsets from head[]. Scans run in place (each thread
// of k_scan_apply reads only the items it writes).
static void finish_plan(const DedupIn& in, const DedupOut& o, int tile_ctx, int tile_cross, cudaStream_t s) {
    int64_t B = in.B;
    k_first_flags<<<grid_for(B, 256), 256, 0, s>>>(B, o.head, o.scan_tmp);
    scan_i64(o.scan_tmp, o.uid, B, o.scan_blk, s);
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.cnt, 0, sizeof(int32_t) * B, s));
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.cursor, 0, sizeof(int32_t) * B, s));
    k_rep<<<grid_for(B, 256), 256, 0, s>>>(B, o.head, o.uid, o.rep, o.first, o.cnt, o.st);
    k_unique_sizes<<<grid_for(B, 256), 256, 0, s>>>(B, in, o.first, o.cnt, o.st, tile_ctx, tile_cross, o.goff,
                                                    o.tok_off, o.ctx_toff, o.cross_toff);
    ScanSet x{{o.goff, o.tok_off, o.ctx_toff, o.cross_toff}, {o.goff, o.tok_off, o.ctx_toff, o.cross_toff}};
    scan_multi(x, 4, B, o.scan_blk, s);  // the four per-unique offset arrays, one launch sequence
    k_totals<<<1, 1, 0, s>>>(B, o.tok_off, o.ctx_toff, o.cross_toff, o.cnt, o.st);
    k_perm<<<grid_for(B, 256), 256, 0, s>>>(B, o.rep, o.goff, o.cursor, o.perm);
    DCAT_LAUNCH_CHECK();
}

void dedup_plan(const DedupIn& in, const DedupOut& o, uint64_t hash_mask, int tile_ctx, int tile_cross,
                cudaStream_t s) {
    int64_t B = in.B;
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.st, 0, sizeof(Status), s));
    DCAT_CUDA_CHECK(cudaMemsetAsync(&o.st->err_row, 0x7f, sizeof(int), s));
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_key, 0xff, sizeof(uint64_t) * o.tab_cap, s));
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_val, 0x7f, sizeof(int32_t) * o.tab_cap, s));
    // span fast path: content-hash one row per distinct (offset, valid) span, copy to the rest
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.list_n, 0, sizeof(int32_t), s));
    k_span<<<grid_for(B, 256), 256, 0, s>>>(in, o.tab_key, o.tab_val, o.tab_cap, o.cursor, o.st);
    k_span_reps<<<grid_for(B, 256), 256, 0, s>>>(B, o.cursor, o.tab_val, o.st, o.list, o.list_n);
    k_hash<<<warp_grid(B), 256, 0, s>>>(in, o.list, o.list_n, 0, 0, hash_mask, o.hash, o.st, 1);
    k_span_copy<<<grid_for(B, 256), 256, 0, s>>>(B, o.cursor, o.tab_val, o.hash);
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_key, 0xff, sizeof(uint64_t) * o.tab_cap, s));
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_val, 0x7f, sizeof(int32_t) * o.tab_cap, s));
    // content-hash table: head = first row with the same key, verified by comparing contents
    k_insert<<<grid_for(B, 256), 256, 0, s>>>(nullptr, nullptr, B, o.hash, o.tab_key, o.tab_val, o.tab_cap, o.slot);
    DCAT_CUDA_CHECK(cudaMemsetAsync(o.list_n, 0, sizeof(int32_t), s));
    k_verify_fast<<<grid_for(B, 256), 256, 0, s>>>(in, o.slot, o.tab_val, o.head, o.collided, o.list, o.list_n);
    k_head_verify<<<warp_grid(B), 256, 0, s>>>(in, o.list, o.list_n, 0, o.slot, o.tab_val, o.head, o.collided, o.st);
    DCAT_LAUNCH_CHECK();
    finish_plan(in, o, tile_ctx, tile_cross, s);
}

void dedup_repair(const DedupIn& in, const DedupOut& o, int n_collided, int tile_ctx, int tile_cross,
                  uint64_t hash_mask, cudaStream_t s) {
    int64_t B = in.B;
    const int kRounds = 4;
    for (int round = 1; round <= kRounds + 1; round++) {
        DCAT_CUDA_CHECK(cudaMemsetAsync(o.list_n, 0, sizeof(int32_t), s));
        k_compact<<<grid_for(B, 256), 256, 0, s>>>(B, o.collided, o.list, o.list_n);
        if (round <= kRounds) {
            DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_key, 0xff, sizeof(uint64_t) * o.tab_cap, s));
            DCAT_CUDA_CHECK(cudaMemsetAsync(o.tab_val, 0x7f, sizeof(int32_t) * o.tab_cap, s));
            unsigned g32 = warp_grid(n_collided);
            k_hash<<<g32, 256, 0, s>>>(in, o.list, o.list_n, 0, 0x9e3779b97f4a7c15ull * round, hash_mask, o.hash,
                                       o.st, 0);
            k_insert<<<grid_for(n_collided, 256), 256, 0, s>>>(o.list, o.list_n, 0, o.hash, o.tab_key, o.tab_val,
                                                                o.tab_cap, o.slot);
            k_head_verify<<<g32, 256, 0, s>>>(in, o.list, o.list_n, 0, o.slot, o.tab_val, o.head, o.collided,
                                              o.st);
        } else {
            k_exact<<<148, 256, 0, s>>>(in, o.list, o.list_n, o.head, o.collided);
        }
        DCAT_LAUNCH_CHECK();
    }
    finish_plan(in, o, tile_ctx, tile_cross, s);
}

void build_tiles(const DedupIn& in, const DedupOut& o, int b_u, int tile_ctx, int tile_cross, Tile* ctx_tiles,
                 Tile* cross_tiles, int32_t* tok_unique, cudaStream_t s) {
    if (b_u <= 0) return;
    k_tiles<<<grid_for(b_u, 128), 128, 0, s>>>(in, o.first, o.cnt, o.tok_off, o.goff, o.ctx_toff, o.cross_toff, o.st,
                                               tile_ctx, tile_cross, ctx_tiles, cross_tiles);
    k_tok_unique<<<static_cast<unsigned>(b_u < 4096 ? b_u : 4096), 256, 0, s>>>(o.tok_off, o.st, tok_unique);
    DCAT_LAUNCH_CHECK();
}

}  // namespace dcat
