// attn_pipe.cu — K5/K6 attention on the 5th-gen tensor cores, persistent and pipelined
// (head dim 32; sm_100a).
//
// Same math as attention.cu / attn_tc.cu (context: layer_forward's causal softmax
// attention, model.cpp:353-376; crossing: cross_forward's attention over [K_u; k] / [V_u; v],
// dcat.cpp:231-263). Work item = (query tile of <= 128 rows of one unique, head), items
// in head-fastest order so the heads of a tile share its K/V lines in L2. An item's keys
// are walked in chunks of 128.
//
// One CTA per SM runs TWO independent pipelines (g = 0, 1) on alternate items, each with
//   * a TMA producer thread: Q (+ the candidates' own k / v rows) into a double-buffered
//     q slot, each 128-key K / V^T chunk into a 4-deep kv ring;
//   * an MMA thread and two 128-column TMEM buffers: S_c = Q K_c^T (M = 128, N = 128,
//     K = 32) goes to buffer c & 1 while the softmax works on the other one; O_c = P_c V_c
//     reads P from TMEM (A-from-TMEM MMA) and V^T (keys contiguous) from smem;
//   * 4 softmax warps, one thread per query row: S leaves TMEM with tcgen05.ld, masks on
//     partial chunks only, max, exp2, row sum; P (bf16) goes back into TMEM over the
//     consumed S columns with tcgen05.st (no shared-memory P). A chunk's O is read one
//     chunk later (while the next S is already in flight), so the softmax warps rarely wait.
// The SFU exp2 rate (16 / clk / SM, tools/kbench/mufu_bw.cu) is this kernel's floor.
// Online-softmax state (m, l, O) lives in the row's registers across chunks; the crossing
// pass starts it at the candidate's own key/value (m = q.k_self, l = 1, O = v_self), so
// the reference's materialized [K_u; k] (dcat.cpp:239-243) never exists.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace dcat {

namespace {

constexpr int P_DH = 32;             // head dim
constexpr int P_KC = 128;            // keys per chunk (S columns of one buffer)
constexpr int P_ROWB = P_DH * 2;     // bytes per Q / K row (SW64)
constexpr int P_Q = 128 * P_ROWB;    // one [128 x DH] tile
constexpr int P_K = P_KC * P_ROWB;   // [KC x DH]
constexpr int P_VTB = P_DH * 128;    // V^T block [DH x 64 keys], SW128
constexpr int P_VT = (P_KC / 64) * P_VTB;
constexpr int P_KV = P_K + P_VT;     // one kv ring slot
constexpr int P_KVS = 4;             // kv ring depth per pipeline
constexpr int P_WARPS = 12;          // 0-3 control, 4-7 softmax g0, 8-11 softmax g1
constexpr int P_O = 64;              // O column offset inside a buffer (P uses [0, 64))

template <bool CAUSAL>
struct PipeCfg {
    static constexpr int QSLOT = CAUSAL ? P_Q : 3 * P_Q;  // Q | k_self | v_self
    static constexpr int GROUP = 2 * QSLOT + P_KVS * P_KV;
    static constexpr int SMEM = 2 * GROUP + 1024 + 512;
};

struct GroupBars {
    uint64_t q_full[2], q_empty[2], kv_full[P_KVS], kv_empty[P_KVS];
    uint64_t s_full[2], p_full[2], o_full[2], s_free[2];
};

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint64_t layout, uint64_t sbo) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((sbo >> 4) << 32) | (1ull << 46) |
           (layout << 61);
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// D[tmem] (+)= A[tmem] . B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    DCAT_TMEM_LD32(taddr, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}
// this thread's row of a [128 x 32] bf16 SW64 tile -> fp32
__device__ __forceinline__ void row_sw64(uint32_t tile, int r, float* v) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t x0, x1, x2, x3;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                     : "r"(tile + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)));
        const uint32_t w[4] = {x0, x1, x2, x3};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
            v[8 * j + 2 * k] = f.x;
            v[8 * j + 2 * k + 1] = f.y;
        }
    }
}

// 16-byte chunk jc (8 bf16 values, dims 8 jc .. 8 jc + 7) of this thread's row of a SW64 tile
__device__ __forceinline__ void row_sw64_chunk(uint32_t tile, int r, int jc, float* v) {
    uint32_t x0, x1, x2, x3;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                 : "r"(tile + r * 64 + ((jc ^ ((r >> 1) & 3)) << 4)));
    const uint32_t w[4] = {x0, x1, x2, x3};
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    DCAT_TMEM_LD16(taddr, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void sts1(uint32_t a, float x) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
}
__device__ __forceinline__ float lds1(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct ItemInfo {
    Tile t;
    int h, a0, nchunks;
};
__device__ __forceinline__ ItemInfo item_info(const AttnArgs& p, int w) {
    ItemInfo it;
    it.t = p.tiles[w / p.n_heads];
    it.h = w % p.n_heads;
    // chunks start at kv0 rounded down to 8 tokens (16-byte TMA inner coordinate of V^T);
    // the <= 7 leading keys of the previous unique are masked
    it.a0 = it.t.kv0 & ~7;
    it.nchunks = it.t.nkv > 0 ? (it.t.kv0 + it.t.nkv - it.a0 + P_KC - 1) / P_KC : 0;
    return it;
}

#ifndef DCAT_ATTN_TRACE
#define DCAT_ATTN_TRACE 0  // debug builds only: clock64 timeline of CTA 0, printed at kernel end
#endif
#if DCAT_ATTN_TRACE
__device__ unsigned long long g_atrace[4096];
__device__ unsigned int g_atrace_n;
#define ATR(code_, val_)                                                                                  \
    do {                                                                                                  \
        if (blockIdx.x == 0) {                                                                            \
            unsigned k_ = atomicAdd(&g_atrace_n, 1u);                                                     \
            if (k_ < 4096)                                                                                \
                g_atrace[k_] = (static_cast<unsigned long long>(clock64()) << 16) | ((code_) << 8) | ((val_) & 255); \
        }                                                                                                 \
    } while (0)
#else
#define ATR(code_, val_) \
    do {                 \
    } while (0)
#endif

template <bool CAUSAL>
__global__ void __launch_bounds__(P_WARPS * 32, 1)
    k_attn_pipe(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmVt, const __grid_constant__ CUtensorMap tmKs,
                const __grid_constant__ CUtensorMap tmVs, const AttnArgs p) {
    using C = PipeCfg<CAUSAL>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    GroupBars* gb = reinterpret_cast<GroupBars*>(smem + 2 * C::GROUP);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(gb + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = p.n_tiles * p.n_heads;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmQ);
        ptx::tma_prefetch(&tmK);
        ptx::tma_prefetch(&tmVt);
        for (int g = 0; g < 2; g++) {
            GroupBars& b = gb[g];
            for (int s = 0; s < 2; s++) {
                ptx::mbar_init(&b.q_full[s], 1);
                ptx::mbar_init(&b.q_empty[s], 1 + 4);  // MMA commit (Q consumed) + 4 softmax warps (self rows)
                ptx::mbar_init(&b.s_full[s], 1);
                ptx::mbar_init(&b.p_full[s], 4);
                ptx::mbar_init(&b.o_full[s], 1);
                ptx::mbar_init(&b.s_free[s], 4);
            }
            for (int s = 0; s < P_KVS; s++) {
                ptx::mbar_init(&b.kv_full[s], 1);
                ptx::mbar_init(&b.kv_empty[s], 1);
            }
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc(tslot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp < 4) {
        const int g = warp >> 1;
        GroupBars& b = gb[g];
        uint8_t* gs = smem + g * C::GROUP;  // q slots | kv ring
        if (lane == 0 && (warp & 1) == 0) {
            // ---- producer of pipeline g
            uint32_t j = 0, kc = 0;
            for (int w = blockIdx.x + g * gridDim.x; w < n_items; w += 2 * gridDim.x, j++) {
                const ItemInfo it = item_info(p, w);
                const int hc = it.h * P_DH;
                const int qs = j & 1;
                uint8_t* qb = gs + qs * C::QSLOT;
                ptx::mbar_wait(&b.q_empty[qs], ((j >> 1) & 1) ^ 1);
                ATR(1 + 16 * g, j);
                ptx::mbar_expect_tx(&b.q_full[qs], C::QSLOT);
                ptx::tma_load_2d(qb, &tmQ, &b.q_full[qs], hc, it.t.q0);
                if constexpr (!CAUSAL) {
                    ptx::tma_load_2d(qb + P_Q, &tmKs, &b.q_full[qs], hc, it.t.q0);
                    ptx::tma_load_2d(qb + 2 * P_Q, &tmVs, &b.q_full[qs], hc, it.t.q0);
                }
                for (int c = 0; c < it.nchunks; c++, kc++) {
                    const int ks = kc % P_KVS;
                    uint8_t* kb = gs + 2 * C::QSLOT + ks * P_KV;
                    const int k0 = it.a0 + c * P_KC;
                    ptx::mbar_wait(&b.kv_empty[ks], ((kc / P_KVS) & 1) ^ 1);
                    ptx::mbar_expect_tx(&b.kv_full[ks], P_KV);
                    ptx::tma_load_2d(kb, &tmK, &b.kv_full[ks], hc, k0);
#pragma unroll
                    for (int vb = 0; vb < P_KC / 64; vb++)
                        ptx::tma_load_2d(kb + P_K + vb * P_VTB, &tmVt, &b.kv_full[ks], k0 + vb * 64, hc);
                }
            }
        } else if (lane == 0) {
            // ---- MMA issuer of pipeline g: S(c) into buffer c & 1, then PV(c - 1)
            constexpr uint32_t idesc_s = ptx::idesc_bf16(128, P_KC);
            constexpr uint32_t idesc_o = ptx::idesc_bf16(128, P_DH);
            const uint32_t TG = tmem + 256 * g;
            uint32_t j = 0, sc = 0;
            bool pend = false;  // a PV (chunk sc - 1 of the current item) is owed
            uint32_t pend_ks = 0;
            auto issue_pv = [&](uint32_t c, uint32_t ks) {
                const uint32_t T = TG + 128 * (c & 1);
                const uint32_t ka = ptx::smem_u32(gs + 2 * C::QSLOT + ks * P_KV);
                ptx::mbar_wait(&b.p_full[c & 1], (c >> 1) & 1);  // P in TMEM
                ATR(3 + 16 * g, c);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < P_KC / 16; kk++)
                    mma_ts(T + P_O, T + 8 * kk, desc(ka + P_K + (kk >> 2) * P_VTB + (kk & 3) * 32, 2, 1024), idesc_o,
                           kk > 0);
                ptx::mma_commit(&b.o_full[c & 1]);
                ptx::mma_commit(&b.kv_empty[ks]);
            };
            for (int w = blockIdx.x + g * gridDim.x; w < n_items; w += 2 * gridDim.x, j++) {
                const ItemInfo it = item_info(p, w);
                const int qs = j & 1;
                const uint32_t qa = ptx::smem_u32(gs + qs * C::QSLOT);
                ptx::mbar_wait(&b.q_full[qs], (j >> 1) & 1);
                for (int c = 0; c < it.nchunks; c++, sc++) {
                    const uint32_t ks = sc % P_KVS, bb = sc & 1;
                    const uint32_t T = TG + 128 * bb;
                    const uint32_t ka = ptx::smem_u32(gs + 2 * C::QSLOT + ks * P_KV);
                    ptx::mbar_wait(&b.kv_full[ks], (sc / P_KVS) & 1);
                    ptx::mbar_wait(&b.s_free[bb], ((sc >> 1) & 1) ^ 1);  // chunk sc - 2's O read back
                    ATR(2 + 16 * g, sc);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int k = 0; k < P_DH / 16; k++)
                        ptx::mma_bf16(T, desc(qa + k * 32, 4, 8 * P_ROWB), desc(ka + k * 32, 4, 8 * P_ROWB), idesc_s,
                                      k > 0);
                    ptx::mma_commit(&b.s_full[bb]);
                    if (c + 1 == it.nchunks) ptx::mma_commit(&b.q_empty[qs]);  // Q consumed by the item's S MMAs
                    if (pend) issue_pv(sc - 1, pend_ks);  // PV of the previous chunk of this item
                    pend = c + 1 < it.nchunks;            // the item's last PV is not deferred:
                    pend_ks = ks;                         // its O finishes the item's output
                    if (!pend) issue_pv(sc, ks);
                }
                if (it.nchunks == 0) ptx::mma_commit(&b.q_empty[qs]);
            }
        }
    } else {
        // ---- softmax warps of pipeline g: one thread per query row
        const int g = (warp - 4) >> 2, q = warp & 3;
        GroupBars& b = gb[g];
        uint8_t* gs = smem + g * C::GROUP;
        const int r = q * 32 + lane;
        const uint32_t TG = tmem + 256 * g + (static_cast<uint32_t>(q * 32) << 16);
        const float sl2 = p.scale * 1.4426950408889634f;
        uint32_t j = 0, sc = 0;
        for (int w = blockIdx.x + g * gridDim.x; w < n_items; w += 2 * gridDim.x, j++) {
            const ItemInfo it = item_info(p, w);
            const int hc = it.h * P_DH;
            const int qs = j & 1;
            const bool live = r < it.t.nq;
            float o[P_DH];
            float m = -INFINITY, l = 0.f;
            ptx::mbar_wait(&b.q_full[qs], (j >> 1) & 1);
            if constexpr (!CAUSAL) {
                // self term (the candidate's own key / value, dcat.cpp:242-243): initial state
                const uint32_t qa = ptx::smem_u32(gs + qs * C::QSLOT);
                float qv[P_DH], kv[P_DH];
                row_sw64(qa, r, qv);
                row_sw64(qa + P_Q, r, kv);
                row_sw64(qa + 2 * P_Q, r, o);
                float s = 0.f;
#pragma unroll
                for (int i = 0; i < P_DH; i++) s += qv[i] * kv[i];
                m = s;
                l = 1.f;
            } else {
#pragma unroll
                for (int i = 0; i < P_DH; i++) o[i] = 0.f;
            }
            __syncwarp();
            if (lane == 0) arrive(&b.q_empty[qs]);
            for (int c = 0; c < it.nchunks; c++, sc++) {
                const uint32_t bb = sc & 1;
                const uint32_t T = TG + 128 * bb;
                const int cb = it.a0 + c * P_KC;                   // token row of S column 0
                const int lo = max(0, it.t.kv0 - cb);              // valid S columns [lo, lim)
                int lim = min(P_KC, it.t.kv0 + it.t.nkv - cb);
                if (CAUSAL) lim = min(lim, it.t.kv0 + it.t.qloc + r + 1 - cb);
                const bool full = lo == 0 && lim == P_KC;
                // warp-uniform class of each 32-column group: all-valid / all-masked / partial
                const int lim_min = __reduce_min_sync(0xffffffffu, lim), lim_max = __reduce_max_sync(0xffffffffu, lim);
                auto grp_full = [&](int k) { return 32 * k >= lo && 32 * k + 32 <= lim_min; };
                auto grp_none = [&](int k) { return 32 * k >= lim_max || 32 * k + 32 <= lo; };
                ptx::mbar_wait(&b.s_full[bb], (sc >> 1) & 1);
                if (lane == 0 && q == 0) ATR(4 + 16 * g, sc);
                ptx::tc_fence_after();
                float v[32];
                // pass 1: row max; TMEM loads double-buffered (load k + 1 while reducing k)
                uint32_t ra[32], rb[32];
                float mx = -INFINITY;
                DCAT_TMEM_LD32(T, ra);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < P_KC / 32; k++) {
                    uint32_t* cur = (k & 1) ? rb : ra;
                    uint32_t* nxt = (k & 1) ? ra : rb;
                    if (k + 1 < P_KC / 32) DCAT_TMEM_LD32(T + (k + 1) * 32, nxt);
                    float t[16];
                    if (grp_none(k)) {
#pragma unroll
                        for (int i = 0; i < 16; i++) t[i] = -INFINITY;
                    } else if (full || grp_full(k)) {
#pragma unroll
                        for (int i = 0; i < 16; i++) t[i] = fmaxf(__uint_as_float(cur[2 * i]), __uint_as_float(cur[2 * i + 1]));
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; i++) {
                            const int c0 = k * 32 + 2 * i;
                            const float x0 = (c0 >= lo && c0 < lim) ? __uint_as_float(cur[2 * i]) : -INFINITY;
                            const float x1 = (c0 + 1 >= lo && c0 + 1 < lim) ? __uint_as_float(cur[2 * i + 1]) : -INFINITY;
                            t[i] = fmaxf(x0, x1);
                        }
                    }
#pragma unroll
                    for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
                        for (int i = 0; i < w2; i++) t[i] = fmaxf(t[i], t[i + w2]);
                    mx = fmaxf(mx, t[0]);
                    if (k + 1 < P_KC / 32) ptx::tmem_wait_ld();
                }
                const float mn = fmaxf(m, mx);
                const float u = mn == -INFINITY ? 0.f : -mn * sl2;
                const float alpha = ex2a(fmaf(m, sl2, u));  // m = -inf -> 0
                m = mn;
                // pass 2: P = exp2(s * scale * log2e - m'), row sum; P (bf16) back into TMEM
                float sum = 0.f;
                DCAT_TMEM_LD32(T, ra);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < P_KC / 32; k++) {
                    uint32_t* cur = (k & 1) ? rb : ra;
                    uint32_t* nxt = (k & 1) ? ra : rb;
                    if (k + 1 < P_KC / 32) DCAT_TMEM_LD32(T + (k + 1) * 32, nxt);
                    uint32_t pk[16];
                    float s2[4] = {0.f, 0.f, 0.f, 0.f};
                    if (grp_none(k)) {
#pragma unroll
                        for (int i = 0; i < 16; i++) pk[i] = 0u;
                    } else if (full || grp_full(k)) {
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float e0 = ex2a(fmaf(__uint_as_float(cur[i]), sl2, u));
                            const float e1 = ex2a(fmaf(__uint_as_float(cur[i + 1]), sl2, u));
                            s2[(i >> 1) & 3] += e0 + e1;
                            pk[i >> 1] = pack_bf16(e0, e1);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            float e0 = ex2a(fmaf(__uint_as_float(cur[i]), sl2, u));
                            float e1 = ex2a(fmaf(__uint_as_float(cur[i + 1]), sl2, u));
                            e0 = (k * 32 + i >= lo && k * 32 + i < lim) ? e0 : 0.f;
                            e1 = (k * 32 + i + 1 >= lo && k * 32 + i + 1 < lim) ? e1 : 0.f;
                            s2[(i >> 1) & 3] += e0 + e1;
                            pk[i >> 1] = pack_bf16(e0, e1);
                        }
                    }
                    sum += (s2[0] + s2[1]) + (s2[2] + s2[3]);
                    st16(T + k * 16, pk);  // P over S columns already consumed
                    if (k + 1 < P_KC / 32) ptx::tmem_wait_ld();
                }
                ptx::tmem_wait_st();
                l = l * alpha + sum;
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive(&b.p_full[bb]);
                if (lane == 0 && q == 0) ATR(6 + 16 * g, sc);
                // O of the previous chunk of this item (its PV ran while this chunk was in softmax):
                // o = (o + O_{c-1}) * alpha_c; for c = 0 just o *= alpha_0
                if (c > 0) {
                    const uint32_t pb = bb ^ 1;
                    ptx::mbar_wait(&b.o_full[pb], ((sc - 1) >> 1) & 1);
                    ptx::tc_fence_after();
                    ld32(TG + 128 * pb + P_O, v);
#pragma unroll
                    for (int i = 0; i < P_DH; i++) o[i] += v[i];
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive(&b.s_free[pb]);
                }
#pragma unroll
                for (int i = 0; i < P_DH; i++) o[i] *= alpha;
                if (c == it.nchunks - 1) {  // last chunk of the item: its own O now
                    ptx::mbar_wait(&b.o_full[bb], (sc >> 1) & 1);
                    if (lane == 0 && q == 0) ATR(7 + 16 * g, sc);
                    ptx::tc_fence_after();
                    ld32(T + P_O, v);
#pragma unroll
                    for (int i = 0; i < P_DH; i++) o[i] += v[i];
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive(&b.s_free[bb]);
                }
            }
            if (lane == 0 && q == 0) ATR(8 + 16 * g, j);
            if (live) {
                const float inv = 1.f / l;
                bf16* op = static_cast<bf16*>(p.out) + static_cast<size_t>(it.t.q0 + r) * p.ldo + hc;
#pragma unroll
                for (int i = 0; i < P_DH; i += 8) {
                    uint4 wv;
                    wv.x = pack_bf16(o[i] * inv, o[i + 1] * inv);
                    wv.y = pack_bf16(o[i + 2] * inv, o[i + 3] * inv);
                    wv.z = pack_bf16(o[i + 4] * inv, o[i + 5] * inv);
                    wv.w = pack_bf16(o[i + 6] * inv, o[i + 7] * inv);
                    *reinterpret_cast<uint4*>(op + i) = wv;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
#if DCAT_ATTN_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned n = g_atrace_n < 4096 ? g_atrace_n : 4096;
        for (unsigned k = 0; k < n && k < 400; k++)
            printf("ATR %llu %llu %llu\n", g_atrace[k] >> 16, (g_atrace[k] >> 8) & 255, g_atrace[k] & 255);
        g_atrace_n = 0;
    }
#endif
}

typedef CUresult (*EncodeFnP)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFnP encoder_p() {
    static EncodeFnP fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFnP>(f);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap map_p(const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems, uint32_t box_c, uint32_t box_r,
                  CUtensorMapSwizzle sw) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    if (!base) return m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * 2) & 15))
        throw CudaError("attention tensor map: 16-byte alignment");
    CUresult r = encoder_p()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
    return m;
}

int sm_count() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    });
    return n;
}

template <bool CAUSAL>
void launch_pipe(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    using C = PipeCfg<CAUSAL>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    static std::once_flag once;
    std::call_once(once, [] {
        DCAT_CUDA_CHECK(cudaFuncSetAttribute(k_attn_pipe<CAUSAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    });
    const int d = a.n_heads * P_DH;
    const CUtensorMap tq = map_p(a.q, d, q_rows, a.ldq, P_DH, 128, CU_TENSOR_MAP_SWIZZLE_64B);
    const CUtensorMap tk = map_p(a.k, d, kv_rows, a.ldkv, P_DH, P_KC, CU_TENSOR_MAP_SWIZZLE_64B);
    const CUtensorMap tv = map_p(a.v, a.ldvt, d, a.ldvt, 64, P_DH, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tks, tvs;
    std::memset(&tks, 0, sizeof tks);
    std::memset(&tvs, 0, sizeof tvs);
    if (!CAUSAL) {
        tks = map_p(a.kself, d, q_rows, a.ldself, P_DH, 128, CU_TENSOR_MAP_SWIZZLE_64B);
        tvs = map_p(a.vself, d, q_rows, a.ldself, P_DH, 128, CU_TENSOR_MAP_SWIZZLE_64B);
    }
    const int64_t items = static_cast<int64_t>(a.n_tiles) * a.n_heads;
    const int grid = static_cast<int>(items < 2 * sm_count() ? (items + 1) / 2 : sm_count());
    k_attn_pipe<CAUSAL><<<grid, P_WARPS * 32, C::SMEM, s>>>(tq, tk, tv, tks, tvs, a);
    DCAT_LAUNCH_CHECK();
}

}  // namespace

bool attention_pipe_supported(int dh) { return dh == P_DH; }

void attention_pipe(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    if (a.n_tiles <= 0) return;
    if (a.dh != P_DH) throw InvalidArg("attention_pipe: head dim " + std::to_string(a.dh));
    if (a.ldvt <= 0) throw InvalidArg("attention_pipe needs the transposed V cache");
    if (a.causal) launch_pipe<true>(a, q_rows, kv_rows, s);
    else launch_pipe<false>(a, q_rows, kv_rows, s);
}

}  // namespace dcat
