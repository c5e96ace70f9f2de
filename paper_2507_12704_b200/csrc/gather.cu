// gather.cu — K2: embedding gathers for the context and crossing passes.
//
// Context token rows (segment_inputs, model.cpp:517-540):
//   E[t] = concat_j sub_j[hash_id(item, seed_j, R)] + action_emb[a]
//          + surface_emb[s] + pos_emb[i]
// with hash_id = mix64(id ^ mix64(seed)) % R (embed.cpp:11-14, lookup
// embed.cpp:38-43). Candidate rows (candidate_inputs, dcat.cpp:180-197, plus
// the Aux term of finetune.cpp:469-479):
//   E[b] = lookup(item_b) + pos_emb[n_u] (+ sum_r aux[r] * aux_proj[r])
// and the ranking-head feature block [cand_emb | ctx_features]
// (crossing_forward finetune.cpp:303-308, ctx_features :212-226).
// One warp per row, 128-bit loads of the fp32 table rows (4 MB at PinFM-base,
// L2-resident), additions in the reference's order, output bf16 (or fp32 in
// the parity path). The bf16 context gather reads one precombined
// (action + surface) + pos row (EmbParams::cmb, 7.4 MB at PinFM-base) instead of
// three: the sum is associated differently from the reference's
// ((lookup + action) + surface) + pos, a last-bit fp32 difference before the
// bf16 rounding; the fp32 parity path keeps the reference's order.
#include <cuda_fp16.h>

#include <type_traits>

#include "launch.h"

namespace dcat {

namespace {

template <typename T>
__device__ __forceinline__ void store4(T* dst, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* dst, float4 v) {
    *reinterpret_cast<float4*>(dst) = v;
}
template <>
__device__ __forceinline__ void store4<bf16>(bf16* dst, float4 v) {
    uint2 p;
    p.x = pack_bf16(v.x, v.y);
    p.y = pack_bf16(v.z, v.w);
    *reinterpret_cast<uint2*>(dst) = p;
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// hash_id(item, seed_j, R) = mix64(item ^ mix64(seed_j)) % R (embed.cpp:11-14)
__device__ __forceinline__ uint32_t table_row(const EmbParams& ep, uint64_t item, int j) {
    const uint64_t h = mix64(item ^ ep.seed_mix[j]);
    const uint64_t R = static_cast<uint64_t>(ep.R);
    return static_cast<uint32_t>((R & (R - 1)) == 0 ? (h & (R - 1)) : h % R);
}
// The J sub-table rows of one item are hashed once per warp: lane j (< J <= 32) holds row j
// and lanes fetch it by shuffle. Every lane must call this (all 32 take part in the shuffle).
__device__ __forceinline__ uint32_t warp_rows(const EmbParams& ep, uint64_t item, int lane) {
    return lane < ep.J ? table_row(ep, item, lane) : 0u;
}
// QuantizedTable row element (dequantize_row, embed.cpp:92-103): codes, then fp16 scale and
// fp16 bias (read bytewise: rows are not 2-byte aligned for odd code byte counts);
// value = (float)code * scale + bias with the reference's separate rounding of * and +.
__device__ __forceinline__ float deq1(const EmbParams& ep, int j, uint32_t r, int e) {
    const uint8_t* row = ep.q + (static_cast<size_t>(j) * ep.R + r) * ep.row_bytes;
    const int cb = ep.code_bytes;
    const float sc = __half2float(__ushort_as_half(static_cast<unsigned short>(row[cb] | (row[cb + 1] << 8))));
    const float bi = __half2float(__ushort_as_half(static_cast<unsigned short>(row[cb + 2] | (row[cb + 3] << 8))));
    const uint32_t code = ep.bits == 8 ? row[e] : ((row[e >> 1] >> ((e & 1) * 4)) & 15u);
    return __fadd_rn(__fmul_rn(static_cast<float>(code), sc), bi);
}
// elements cc .. cc + 3 of sub-table j row r (fp32 or quantized table)
__device__ __forceinline__ float4 sub4(const EmbParams& ep, int j, uint32_t r, int cc) {
    if (ep.q == nullptr)
        return __ldg(reinterpret_cast<const float4*>(ep.table + (static_cast<size_t>(j) * ep.R + r) * ep.d_sub + cc));
    return make_float4(deq1(ep, j, r, cc), deq1(ep, j, r, cc + 1), deq1(ep, j, r, cc + 2), deq1(ep, j, r, cc + 3));
}
__device__ __forceinline__ float sub1(const EmbParams& ep, int j, uint32_t r, int cc) {
    if (ep.q == nullptr) return __ldg(ep.table + (static_cast<size_t>(j) * ep.R + r) * ep.d_sub + cc);
    return deq1(ep, j, r, cc);
}
// row of sub-table j holding column c: lane j's hash (shuffled) or, past 32 sub-tables, recomputed
__device__ __forceinline__ uint32_t col_row(const EmbParams& ep, uint64_t item, uint32_t rows, int j) {
    const uint32_t r = ep.J <= 32 ? __shfl_sync(0xffffffffu, rows, j & 31) : 0u;
    return ep.J > 32 ? table_row(ep, item, j) : r;
}
__device__ __forceinline__ float4 lookup4(const EmbParams& ep, uint64_t item, uint32_t rows, int c) {
    const int cl = c < ep.d_emb ? c : ep.d_emb - 1;  // inactive lanes shuffle a valid source lane
    const int j = cl / ep.d_sub;
    const uint32_t r = col_row(ep, item, rows, j);
    return c < ep.d_emb ? sub4(ep, j, r, cl - j * ep.d_sub) : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ float lookup1(const EmbParams& ep, uint64_t item, uint32_t rows, int c) {
    const int cl = c < ep.d_emb ? c : ep.d_emb - 1;
    const int j = cl / ep.d_sub;
    const uint32_t r = col_row(ep, item, rows, j);
    return c < ep.d_emb ? sub1(ep, j, r, cl - j * ep.d_sub) : 0.f;
}

// this lane's 4-column groups of a d_emb row (c = 128 k + 4 lane): sub-table j and offset
// in it, computed once per kernel instead of once per token
constexpr int kMaxSteps = 8;  // d_emb <= 1024 on the vectorised path
struct LaneCols {
    int j[kMaxSteps], cc[kMaxSteps];
};
__device__ __forceinline__ LaneCols lane_cols(const EmbParams& ep, int lane) {
    LaneCols L;
#pragma unroll
    for (int k = 0; k < kMaxSteps; k++) {
        int c = 128 * k + 4 * lane;
        c = c < ep.d_emb ? c : ep.d_emb - 4;
        L.j[k] = c / ep.d_sub;
        L.cc[k] = c - L.j[k] * ep.d_sub;
    }
    return L;
}
// vectorised token row: all lanes shuffle (uniform trip count), inactive lanes skip the I/O
template <typename T>
__device__ __forceinline__ void gather_ctx_token_vec(const EmbParams& ep, const LaneCols& L, int64_t t, int i,
                                                     uint64_t item, int a, int s, T* __restrict__ E, int ldE,
                                                     int lane) {
    const float* pe = ep.pos_emb ? ep.pos_emb + static_cast<size_t>(i) * ep.d_emb : nullptr;
    T* out = E + t * ldE;
    if (a < 0) {  // AuxLt learnable token: lt + pos_emb[i] (finetune.cpp:188-190); warp-uniform
        for (int c = 4 * lane; c < ep.d_emb; c += 128) {
            float4 v = __ldg(reinterpret_cast<const float4*>(ep.lt + c));
            if (pe) v = add4(v, __ldg(reinterpret_cast<const float4*>(pe + c)));
            store4<T>(out + c, v);
        }
        return;
    }
    const uint32_t rows = warp_rows(ep, item, lane);
    if (ep.cmb != nullptr) {  // bf16 path: lookup + ((action + surface) + pos), one row read instead of three
        const float* ce = ep.cmb + (static_cast<size_t>(a * ep.n_surf + s) * ep.max_len + i) * ep.d_emb;
#pragma unroll
        for (int k = 0; k < kMaxSteps; k++) {
            if (128 * k >= ep.d_emb) break;
            const int c = 128 * k + 4 * lane;
            const uint32_t r = __shfl_sync(0xffffffffu, rows, L.j[k] & 31);
            if (c < ep.d_emb)
                store4<T>(out + c, add4(sub4(ep, L.j[k], r, L.cc[k]), __ldg(reinterpret_cast<const float4*>(ce + c))));
        }
        return;
    }
    const float* ae = ep.action_emb + static_cast<size_t>(a) * ep.d_emb;
    const float* se = ep.surface_emb + static_cast<size_t>(s) * ep.d_emb;
#pragma unroll
    for (int k = 0; k < kMaxSteps; k++) {
        if (128 * k >= ep.d_emb) break;
        const int c = 128 * k + 4 * lane;
        const uint32_t r = __shfl_sync(0xffffffffu, rows, L.j[k] & 31);
        if (c < ep.d_emb) {
            float4 v = sub4(ep, L.j[k], r, L.cc[k]);
            v = add4(v, __ldg(reinterpret_cast<const float4*>(ae + c)));
            v = add4(v, __ldg(reinterpret_cast<const float4*>(se + c)));
            if (pe) v = add4(v, __ldg(reinterpret_cast<const float4*>(pe + c)));
            store4<T>(out + c, v);
        }
    }
}

// one context token row (one warp): E[t] = ((lookup + action) + surface) + pos, model.cpp:517-540
template <typename T, bool VEC>
__device__ __forceinline__ void gather_ctx_token(const EmbParams& ep, int64_t t, int i, uint64_t item, int a, int s,
                                                 T* __restrict__ E, int ldE, int lane) {
    if (a < 0) {  // AuxLt learnable token: lt + pos_emb[i] (finetune.cpp:188-190); warp-uniform
        T* out = E + t * ldE;
        for (int c = lane; c < ep.d_emb; c += 32) {
            float v = ep.lt[c];
            if (ep.pos_emb) v = v + ep.pos_emb[static_cast<size_t>(i) * ep.d_emb + c];
            ActIO<T>::store(out + c, v);
        }
        return;
    }
    {
        const uint32_t rows = warp_rows(ep, item, lane);
        const float* ae = ep.action_emb + static_cast<size_t>(a) * ep.d_emb;
        const float* se = ep.surface_emb + static_cast<size_t>(s) * ep.d_emb;
        const float* pe = ep.pos_emb ? ep.pos_emb + static_cast<size_t>(i) * ep.d_emb : nullptr;
        T* out = E + t * ldE;
        if constexpr (VEC) {
            for (int c0 = 0; c0 < ep.d_emb; c0 += 128) {
                const int c = c0 + lane * 4;
                float4 v = lookup4(ep, item, rows, c);
                if (c < ep.d_emb) {
                    v = add4(v, __ldg(reinterpret_cast<const float4*>(ae + c)));
                    v = add4(v, __ldg(reinterpret_cast<const float4*>(se + c)));
                    if (pe) v = add4(v, __ldg(reinterpret_cast<const float4*>(pe + c)));
                    store4<T>(out + c, v);
                }
            }
        } else {
            for (int c0 = 0; c0 < ep.d_emb; c0 += 32) {
                const int c = c0 + lane;
                float v = lookup1(ep, item, rows, c);
                if (c < ep.d_emb) {
                    v = v + ae[c];
                    v = v + se[c];
                    if (pe) v = v + pe[c];
                    ActIO<T>::store(out + c, v);
                }
            }
        }
    }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256, 4) k_gather_ctx(DedupIn in, const int32_t* __restrict__ first, const int64_t* __restrict__ tok_off,
                             EmbParams ep, const int32_t* __restrict__ tok_unique, int64_t T_ctx, T* __restrict__ E,
                             int ldE) {
    constexpr int TOK = 8;  // tokens per warp step: lanes 0..7 resolve their metadata in parallel
    const int lane = threadIdx.x & 31;
    const LaneCols L = lane_cols(ep, lane);
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t tb = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * TOK; tb < T_ctx;
         tb += nw * TOK) {
        int mi = 0, ma = 0, ms = 0;
        uint64_t mitem = 0;
        if (lane < TOK && tb + lane < T_ctx) {
            const int64_t t = tb + lane;
            const int u = tok_unique[t];
            mi = static_cast<int>(t - tok_off[u]);
            const int fr = first[u], rv = in.row_valid[fr], kept = seq_kept(in, rv);
            if (mi < kept) {
                const int64_t ev = in.row_offset[fr] + (rv - kept) + mi;  // fixed window: newest events
                mitem = in.item[ev];
                ma = in.action[ev];
                ms = in.surface[ev];
            } else {
                ma = -1;  // AuxLt's learnable token after the events (finetune.cpp:186-191)
            }
        }
        const int nt = T_ctx - tb < TOK ? static_cast<int>(T_ctx - tb) : TOK;
        for (int k = 0; k < nt; k++) {
            const int ti = __shfl_sync(0xffffffffu, mi, k), ta = __shfl_sync(0xffffffffu, ma, k);
            const int ts = __shfl_sync(0xffffffffu, ms, k);
            const uint64_t titem = __shfl_sync(0xffffffffu, mitem, k);
            if constexpr (VEC) gather_ctx_token_vec<T>(ep, L, tb + k, ti, titem, ta, ts, E, ldE, lane);
            else gather_ctx_token<T, VEC>(ep, tb + k, ti, titem, ta, ts, E, ldE, lane);
        }
    }
}

// bf16 context gather, 4 tokens per warp: lane group g (8 lanes) owns token tb + g. Each lane
// resolves its group's token metadata (same addresses within a group: broadcast loads), lane
// j < J of a group hashes sub-table row j once, and the group writes the row as 8 x 16-byte
// chunks per 128 columns: lookup + cmb, cmb = (action + surface) + pos (EmbParams::cmb).
// Needs J <= 8, d_sub % 4 == 0, d_emb % 32 == 0, the fp32 table and cmb.
__global__ void __launch_bounds__(256) k_gather_ctx_g8(DedupIn in, const int32_t* __restrict__ first,
                                                      const int64_t* __restrict__ tok_off, EmbParams ep,
                                                      const int32_t* __restrict__ tok_unique, int64_t T_ctx,
                                                      bf16* __restrict__ E, int ldE) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, l8 = lane & 7;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t tb = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 4; tb < T_ctx;
         tb += nw * 4) {
        const int64_t t = tb + grp;
        const bool live = t < T_ctx;
        int i = 0, a = 0, sf = 0;
        uint64_t item = 0;
        if (live) {
            const int u = tok_unique[t];
            i = static_cast<int>(t - tok_off[u]);
            const int fr = first[u], rv = in.row_valid[fr], kept = seq_kept(in, rv);
            if (i < kept) {
                const int64_t ev = in.row_offset[fr] + (rv - kept) + i;  // fixed window: newest events
                item = in.item[ev];
                a = in.action[ev];
                sf = in.surface[ev];
            } else {
                a = -1;  // AuxLt's learnable token after the events (finetune.cpp:186-191)
            }
        }
        const uint32_t row_j = (live && a >= 0 && l8 < ep.J) ? table_row(ep, item, l8) : 0u;
        if (!live) continue;  // groups are independent from here (8-lane shuffles only)
        bf16* out = E + t * ldE;
        if (a < 0) {  // lt + pos_emb[i] (finetune.cpp:188-190)
            for (int c = 4 * l8; c < ep.d_emb; c += 32) {
                float4 v = __ldg(reinterpret_cast<const float4*>(ep.lt + c));
                if (ep.pos_emb) v = add4(v, __ldg(reinterpret_cast<const float4*>(ep.pos_emb + static_cast<size_t>(i) * ep.d_emb + c)));
                store4<bf16>(out + c, v);
            }
            continue;
        }
        const float* ce = ep.cmb + (static_cast<size_t>(a * ep.n_surf + sf) * ep.max_len + i) * ep.d_emb;
        const unsigned gmask = 0xffu << (grp * 8);
        for (int c = 4 * l8; c < ep.d_emb; c += 32) {
            const int j = c / ep.d_sub;  // the 8 lanes share one sub-table row when d_sub >= 32
            const uint32_t r = __shfl_sync(gmask, row_j, j, 8);
            const float4 v = __ldg(reinterpret_cast<const float4*>(ep.table + (static_cast<size_t>(j) * ep.R + r) * ep.d_sub +
                                                                   (c - j * ep.d_sub)));
            store4<bf16>(out + c, add4(v, __ldg(reinterpret_cast<const float4*>(ce + c))));
        }
    }
}

// ctx_features (finetune.cpp:212-226)
__device__ float ctx_feature(int k, double age, int valid, int last_surface, int max_events, double fresh,
                             double mid) {
    double days = age / 86400.0;
    int band = days < fresh ? 0 : days < mid ? 1 : 2;
    if (k < 3) return k == band ? 1.0f : 0.0f;
    if (k == 3) {
        if (max_events <= 0) return 0.0f;
        float r = static_cast<float>(valid) / static_cast<float>(max_events);
        return r < 1.0f ? r : 1.0f;
    }
    return (valid > 0 && k - 4 == last_surface) ? 1.0f : 0.0f;
}

// per-row metadata of a candidate, resolved by one lane (8 rows per warp step in parallel)
struct CandMeta {
    int i, n, valid, last_s;
    uint64_t item;
    double age;
};
__device__ __forceinline__ CandMeta cand_meta(const DedupIn& in, const int32_t* __restrict__ perm,
                                              const int32_t* __restrict__ rep, const int32_t* __restrict__ first,
                                              const CandParams& cp, bool want_feat, int64_t p) {
    CandMeta m;
    m.i = perm[p];
    m.n = seq_tokens(in, in.row_valid[first[rep[m.i]]]);  // candidate position (after the context / lt token)
    m.item = cp.candidate[m.i];
    m.valid = 0;
    m.last_s = -1;
    m.age = 0.0;
    if (want_feat) {
        m.age = cp.age[m.i];
        m.valid = in.row_valid[m.i];
        m.last_s = m.valid > 0 ? in.surface[in.row_offset[m.i] + m.valid - 1] : -1;
    }
    return m;
}
__device__ __forceinline__ CandMeta shfl_meta(const CandMeta& m, int k) {
    CandMeta r;
    r.i = __shfl_sync(0xffffffffu, m.i, k);
    r.n = __shfl_sync(0xffffffffu, m.n, k);
    r.valid = __shfl_sync(0xffffffffu, m.valid, k);
    r.last_s = __shfl_sync(0xffffffffu, m.last_s, k);
    r.item = __shfl_sync(0xffffffffu, m.item, k);
    r.age = __shfl_sync(0xffffffffu, m.age, k);
    return r;
}

template <typename T>
__device__ void gather_cand_row(const EmbParams& ep, const CandParams& cp, const CandMeta& m, int64_t p,
                                T* __restrict__ E, int ldE, T* __restrict__ feat, Status* st, int lane) {
    const int i = m.i, n = m.n;
    const uint64_t item = m.item;
    const uint32_t rows = warp_rows(ep, item, lane);
    const float* pe = ep.pos_emb ? ep.pos_emb + static_cast<size_t>(n) * ep.d_emb : nullptr;
    const float* aux = cp.variant_aux ? cp.aux + static_cast<size_t>(i) * cp.d_aux : nullptr;
    T* out = E + p * ldE;
    T* fo = feat ? feat + p * cp.feat_ld : nullptr;
    bool vec = (ep.d_sub % 4) == 0 && (ep.d_emb % 4) == 0;
    if (vec) {
        for (int c0 = 0; c0 < ep.d_emb; c0 += 128) {
            const int c = c0 + lane * 4;
            float4 raw = lookup4(ep, item, rows, c);
            if (c >= ep.d_emb) continue;
            if (fo) store4<T>(fo + cp.d_model + c, raw);
            float4 v = raw;
            if (pe && !cp.aux_first) v = add4(v, __ldg(reinterpret_cast<const float4*>(pe + c)));
            if (aux) {
                for (int r = 0; r < cp.d_aux; r++) {
                    float al = aux[r];
                    float4 pr = __ldg(reinterpret_cast<const float4*>(cp.aux_proj + static_cast<size_t>(r) * ep.d_emb + c));
                    v.x = __fadd_rn(v.x, __fmul_rn(al, pr.x));
                    v.y = __fadd_rn(v.y, __fmul_rn(al, pr.y));
                    v.z = __fadd_rn(v.z, __fmul_rn(al, pr.z));
                    v.w = __fadd_rn(v.w, __fmul_rn(al, pr.w));
                }
            }
            if (pe && cp.aux_first) v = add4(v, __ldg(reinterpret_cast<const float4*>(pe + c)));
            store4<T>(out + c, v);
        }
    } else {
        for (int c0 = 0; c0 < ep.d_emb; c0 += 32) {
            const int c = c0 + lane;
            float raw = lookup1(ep, item, rows, c);
            if (c >= ep.d_emb) continue;
            if (fo) ActIO<T>::store(fo + cp.d_model + c, raw);
            float v = raw;
            if (pe && !cp.aux_first) v = v + pe[c];
            if (aux)
                for (int r = 0; r < cp.d_aux; r++)
                    v = __fadd_rn(v, __fmul_rn(aux[r], cp.aux_proj[static_cast<size_t>(r) * ep.d_emb + c]));
            if (pe && cp.aux_first) v = v + pe[c];
            ActIO<T>::store(out + c, v);
        }
    }
    if (fo) {
        const double age = m.age;
        if (lane == 0 && age < 0.0) {
            atomicOr(&st->err_bits, ERR_AGE);
            atomicMin(&st->err_row, i);
        }
        const int valid = m.valid, last_s = m.last_s;
        int c0 = cp.d_model + ep.d_emb;
        for (int c = c0 + lane; c < cp.feat_ld; c += 32) {
            int k = c - c0;
            float f = k < 8 ? ctx_feature(k, age, valid, last_s, cp.max_events, cp.fresh_days, cp.mid_days) : 0.0f;
            ActIO<T>::store(fo + c, f);
        }
    }
}

template <typename T>
__global__ void k_gather_cand(DedupIn in, const int32_t* __restrict__ perm, const int32_t* __restrict__ rep,
                              const int32_t* __restrict__ first, EmbParams ep, CandParams cp, int64_t B,
                              T* __restrict__ E, int ldE, T* __restrict__ feat, Status* st) {
    constexpr int TOK = 8;  // rows per warp step: lanes 0..7 resolve their metadata chains in parallel
    const int lane = threadIdx.x & 31;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t pb = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * TOK; pb < B;
         pb += nw * TOK) {
        CandMeta mine{};
        if (lane < TOK && pb + lane < B) mine = cand_meta(in, perm, rep, first, cp, feat != nullptr, pb + lane);
        const int nt = B - pb < TOK ? static_cast<int>(B - pb) : TOK;
        for (int k = 0; k < nt; k++)
            gather_cand_row(ep, cp, shfl_meta(mine, k), pb + k, E, ldE, feat, st, lane);
    }
}

// grid for the grid-stride warp-per-row kernels (256 threads): <= 8 resident blocks per SM
inline unsigned warp_grid(int64_t rows) {
    const int64_t g = (rows * 32 + 255) / 256;
    return static_cast<unsigned>(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

__global__ void k_build_cmb(const float* __restrict__ ae, const float* __restrict__ se, const float* __restrict__ pe,
                            int n_surf, int max_len, int d_emb, int64_t n, float* __restrict__ cmb) {
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < n;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(x % d_emb);
        const int64_t row = x / d_emb;
        const int i = static_cast<int>(row % max_len);
        const int as = static_cast<int>(row / max_len);
        const int a = as / n_surf, s = as % n_surf;
        cmb[x] = (ae[static_cast<size_t>(a) * d_emb + c] + se[static_cast<size_t>(s) * d_emb + c]) +
                 pe[static_cast<size_t>(i) * d_emb + c];
    }
}

}  // namespace

void build_combined_emb(const float* action_emb, const float* surface_emb, const float* pos_emb, int n_act,
                        int n_surf, int max_len, int d_emb, float* cmb, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(n_act) * n_surf * max_len * d_emb;
    if (n <= 0) return;
    k_build_cmb<<<1184, 256, 0, s>>>(action_emb, surface_emb, pos_emb, n_surf, max_len, d_emb, n, cmb);
    DCAT_LAUNCH_CHECK();
}

// candidate_inputs (dcat.cpp:180-197) as its own entry point: e[i] = lookup(items[i]) +
// pos_emb[pos[i]] (learned positions), fp32, one warp per row; a position outside [0, max_len)
// is reported like the reference's check (dcat.cpp:190-192)
__global__ void __launch_bounds__(256) k_cand_inputs(EmbParams ep, const uint64_t* __restrict__ items,
                                                     const int32_t* __restrict__ pos, int64_t n, float* __restrict__ e,
                                                     Status* st) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= n) return;
    const uint64_t item = items[row];
    const uint32_t rows = warp_rows(ep, item, lane);
    const int ps = pos[row];
    const bool pos_ok = ps >= 0 && ps < ep.max_len;
    if (ep.pos_emb && !pos_ok) {
        if (lane == 0) {
            atomicOr(&st->err_bits, ERR_POS_CAND);
            atomicMin(&st->err_row, static_cast<int>(row));
            st->err_val = ps;
        }
        return;
    }
    const float* pe = ep.pos_emb ? ep.pos_emb + static_cast<size_t>(ps) * ep.d_emb : nullptr;
    float* out = e + row * ep.d_emb;
    for (int c0 = 0; c0 < ep.d_emb; c0 += 32) {
        const int c = c0 + lane;
        const float v = lookup1(ep, item, rows, c);  // every lane takes part in the shuffle
        if (c < ep.d_emb) out[c] = pe ? v + pe[c] : v;
    }
}

void candidate_inputs(const EmbParams& ep, const uint64_t* items, const int32_t* pos, int64_t n, float* e, Status* st,
                      cudaStream_t s) {
    if (n <= 0) return;
    k_cand_inputs<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, s>>>(ep, items, pos, n, e, st);
    DCAT_LAUNCH_CHECK();
}

template <typename T>
void gather_context(const DedupIn& in, const DedupOut& o, const EmbParams& ep, const int32_t* tok_unique,
                    int64_t T_ctx, T* E, int ldE, cudaStream_t s) {
    if (T_ctx <= 0) return;
    const unsigned g = warp_grid(T_ctx);
    if constexpr (std::is_same<T, bf16>::value) {
        if (ep.cmb && ep.q == nullptr && ep.J <= 8 && ep.d_sub % 4 == 0 && ep.d_emb % 32 == 0 && ldE % 4 == 0) {
            k_gather_ctx_g8<<<warp_grid((T_ctx + 3) / 4), 256, 0, s>>>(in, o.first, o.tok_off, ep, tok_unique, T_ctx, E,
                                                                        ldE);
            DCAT_LAUNCH_CHECK();
            return;
        }
    }
    if ((ep.d_sub % 4) == 0 && (ep.d_emb % 4) == 0 && (ldE % 4) == 0 && ep.d_emb <= 128 * 8 && ep.J <= 32)
        k_gather_ctx<T, true><<<g, 256, 0, s>>>(in, o.first, o.tok_off, ep, tok_unique, T_ctx, E, ldE);
    else
        k_gather_ctx<T, false><<<g, 256, 0, s>>>(in, o.first, o.tok_off, ep, tok_unique, T_ctx, E, ldE);
    DCAT_LAUNCH_CHECK();
}

template <typename T>
void gather_candidates(const DedupIn& in, const DedupOut& o, const EmbParams& ep, const CandParams& cp, int64_t B,
                       T* E, int ldE, T* feat, cudaStream_t s) {
    if (B <= 0) return;
    const unsigned g = warp_grid(B);
    k_gather_cand<T><<<g, 256, 0, s>>>(in, o.perm, o.rep, o.first, ep, cp, B, E, ldE, feat, o.st);
    DCAT_LAUNCH_CHECK();
}

template void gather_context<float>(const DedupIn&, const DedupOut&, const EmbParams&, const int32_t*, int64_t,
                                    float*, int, cudaStream_t);
template void gather_context<bf16>(const DedupIn&, const DedupOut&, const EmbParams&, const int32_t*, int64_t, bf16*,
                                   int, cudaStream_t);
template void gather_candidates<float>(const DedupIn&, const DedupOut&, const EmbParams&, const CandParams&, int64_t,
                                       float*, int, float*, cudaStream_t);
template void gather_candidates<bf16>(const DedupIn&, const DedupOut&, const EmbParams&, const CandParams&, int64_t,
                                      bf16*, int, bf16*, cudaStream_t);

}  // namespace dcat
