// attn_fa.cu — K5 / K6 attention on the 5th-gen tensor cores (sm_100a): TMA-staged Q / K / V^T,
// S = Q K^T and O += P V on tcgen05 with S, P and O in TMEM, online softmax on CUDA cores.
//
// Same math as the reference:
//   K5 context pass: layer_forward's causal multi-head attention (model.cpp:353-376), scale
//      1/sqrt(dh), max-subtracted softmax;
//   K6 crossing pass: cross_forward's attention of each candidate over its unique's cached
//      K_u / V_u plus its own key / value (dcat.cpp:231-263). The reference copies [K_u; k] /
//      [V_u; v] per candidate (dcat.cpp:239-243); here the candidates of one unique are the
//      M = 128 rows of a query tile over the cached K / V, and the candidate's own key / value is
//      the initial online-softmax state (m = q.k_self, l = 1, O = v_self).
//
// Work item = (query tile of <= 128 rows of one unique, head). One persistent CTA per SM runs
// two independent pipelines g = 0, 1 (FA4-style ping-pong: while one pipeline's softmax works,
// the tensor core serves the other). Pipeline g of CTA b takes items 2 (b + k grid) + g, so the
// two pipelines of a CTA work on adjacent heads of one tile (their K / V rows share L2 lines).
// Per pipeline:
//   * a TMA producer thread: Q per item into a 2-slot ring; per 128-key chunk, K [128 x dh] and
//     V^T [dh x 128] (keys contiguous) into an NST-slot ring;
//   * an MMA thread: S(c) = Q K_c^T (M = 128, N = 128, K = dh) into the pipeline's S columns once
//     the softmax has released S(c - 1) (p_full), right after O += P(c-1) V_{c-1} (A = P from
//     TMEM, B = V^T from smem, N = dh). MMAs of one thread complete in order, so s_full(c) also
//     says PV(c - 1) is done: the softmax reads / rescales O without another barrier;
//   * 4 softmax warps, one thread per query row (TMEM lane = row), no cross-thread reduction.
// Softmax per chunk, one pass over S in the common case: p = exp2(s * scale * log2e + u) with
// u = -m * scale * log2e for the running max m, P (bf16) into the pipeline's P columns, row sum l
// in registers, chunk row max with 3-input FMNMX. Lazy rescale: m only moves when the chunk max
// exceeds it by more than LAZY (log2 units); then O (TMEM) and l are scaled by alpha and the
// chunk's P is recomputed from S (still intact); otherwise p <= 2^LAZY against the stale max and
// O / l is unchanged up to rounding. Causal items compute the first chunk's max in a separate pass.
// The candidate's q, k_self, v_self rows (self term) are read from global memory by its thread.
// POLY > 0: every POLY-th pair of exponentials runs as an FMA-pipe polynomial beside MUFU.EX2.
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace dcat {

namespace {

template <int DH>
struct FaCfg {
    static constexpr int ROWB = DH * 2;                                  // bytes per Q / K row
    static constexpr uint64_t LAYOUT = DH == 16 ? 6 : (DH == 32 ? 4 : 2);  // SW32 / SW64 / SW128
    static constexpr int SBO = 8 * ROWB;                                 // 8-row swizzle atom
    static constexpr int TQ = 128 * ROWB;                                // one [128 x dh] tile
    static constexpr int KC = 128;                                       // keys per chunk
    static constexpr int TK = KC * ROWB;                                 // K chunk [128 x dh]
    static constexpr int VTB = DH * 128;                                 // V^T block [dh x 64 keys], SW128
    static constexpr int SLOT = TK + (KC / 64) * VTB;                    // one kv ring slot (all TMA bytes)
    static constexpr int NST = DH == 64 ? 2 : 3;                         // kv ring depth per pipeline
    // TMEM columns of pipeline g (base 256 g): S [0, 128) | P [128, 192) (bf16 pairs) | O [192, 192 + dh)
    static constexpr int T_S = 0, T_P = 128, T_O = 192;
    static_assert(T_O + DH <= 256, "TMEM columns");
};

template <int DH, bool CAUSAL>
struct FaSmem {
    using C = FaCfg<DH>;
    // per pipeline: NQS item slots (Q, plus the crossing candidates' k_self / v_self tiles) | kv ring
    static constexpr int QTILES = CAUSAL ? 1 : 3;
    static constexpr int NQS = (DH == 64 && !CAUSAL) ? 1 : 2;
    static constexpr int QSLOT = QTILES * C::TQ;
    static constexpr int GROUP = NQS * QSLOT + C::NST * C::SLOT;
    static constexpr int BAR = 2 * GROUP;
    static constexpr int TOTAL = BAR + 512 + 1024;              // + barriers + alignment slack
};

struct FaBars {  // one set per pipeline
    uint64_t q_full[2], q_empty[2], s_full, p_full, o_final;
    uint64_t kv_full[3], kv_empty[3];
};

__device__ __forceinline__ uint64_t fdesc(uint32_t saddr, uint64_t layout, uint32_t sbo) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(sbo >> 4) << 32) |
           (1ull << 46) | (layout << 61);
}
__device__ __forceinline__ void arrive1(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x on the FMA pipe: round-to-nearest split x = j + f, |f| <= 1/2, cubic fit of 2^f (relative
// error 1.4e-4, below the bf16 rounding of P), j added to the exponent field.
__device__ __forceinline__ float ex2p(float x) {
    x = fmaxf(x, -127.f);
    const float t = x + 12582912.f;  // 1.5 * 2^23: round(x) lands in the low mantissa bits
    const float f = x - (t - 12582912.f);
    const float p = fmaf(fmaf(fmaf(0.05502927f, f, 0.24225698f), f, 0.69325305f), f, 0.99995134f);
    return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void st1(uint32_t taddr, uint32_t r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(r) : "memory");
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ uint32_t ld1(uint32_t taddr) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
    return r;
}
// O columns [c0, c0 + n) of this thread's TMEM row <-> registers, n in {8, 16, 32}
template <int N>
__device__ __forceinline__ void o_load(uint32_t taddr, float* v) {
    uint32_t r[N];
#pragma unroll
    for (int i = 0; i < N; i += 8) ld8(taddr + i, r + i);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < N; i++) v[i] = __uint_as_float(r[i]);
}
template <int N>
__device__ __forceinline__ void o_store(uint32_t taddr, const float* v) {
#pragma unroll
    for (int i = 0; i < N; i += 8) {
        uint32_t r[8];
#pragma unroll
        for (int k = 0; k < 8; k++) r[k] = __float_as_uint(v[i + k]);
        st8(taddr + i, r);
    }
}
// 16-byte chunk jc (8 bf16, packed) of row r of a [128 x DH] swizzled tile (TMA SWIZZLE_{32,64,128}B)
template <int DH>
__device__ __forceinline__ void row_chunk_w(uint32_t tile, int r, int jc, uint32_t* w) {
    constexpr int ROWB = DH * 2;
    constexpr int SWM = (DH == 16 ? 2 : (DH == 32 ? 4 : 8)) - 1;
    const uint32_t a = tile + r * ROWB + ((jc ^ ((r * ROWB >> 7) & SWM)) << 4);
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
}

struct FaItem {
    Tile t;
    int h, a0, nchunks;
};
__device__ __forceinline__ FaItem fa_item(const AttnArgs& p, int w) {
    FaItem it;
    it.t = p.tiles[w / p.n_heads];
    it.h = w % p.n_heads;
    // chunks start at kv0 rounded down to 8 tokens (16-byte inner coordinate of the V^T box); the
    // <= 7 leading keys of the previous unique are masked
    it.a0 = it.t.kv0 & ~7;
    it.nchunks = it.t.nkv > 0 ? (it.t.kv0 + it.t.nkv - it.a0 + 127) / 128 : 0;
    return it;
}

#ifdef DCAT_FA_WATCHDOG  // bring-up builds: trap with the role / barrier after ~2^28 polls
__device__ __forceinline__ void fa_wait(uint64_t* bar, uint32_t parity, int code) {
    const uint32_t a = ptx::smem_u32(bar);
    for (uint64_t n = 0; !ptx::mbar_try_wait(a, parity); n++) {
        if (n == (1ull << 28)) {
            printf("fa watchdog: block %d thread %d code %d parity %u\n", blockIdx.x, threadIdx.x, code, parity);
            __trap();
        }
    }
}
#define FA_WAIT(bar, par, code) fa_wait(bar, par, code)
#else
// try_wait with a suspend-time hint: the waiting thread sleeps until the phase completes (or the
// hint expires) instead of spinning, so the producer / MMA threads and idle softmax warps do not
// take issue slots from the softmax warps sharing their SM sub-partition
__device__ __forceinline__ void fa_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = ptx::smem_u32(bar);
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
}
#define FA_WAIT(bar, par, code) fa_wait(bar, par)
#endif

#ifndef DCAT_FA_LAZY
#define DCAT_FA_LAZY 12.0f
#endif

// One softmax pass over the S chunk at TS (TMEM address with the warp's lane base): P = exp2(s *
// sl2 + u) into the P columns at TP (bf16 pairs, key c at column c / 2), masked columns (outside
// [lo, lim)) -> p = 0. Returns the row sum of p. No row max: the caller detects a stale running
// max from the sum (see the kernel). lo is uniform over the CTA's rows; lim_min / lim_max are the
// warp's extremes of lim.
template <int POLY>
__device__ __forceinline__ float p_pass(uint32_t TS, uint32_t TP, float sl2, float u, int lo, int lim, int lim_min,
                                        int lim_max) {
    float s0 = 0.f, s1 = 0.f;
    uint32_t ra[32], rb[32];
    DCAT_TMEM_LD32(TS, ra);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint32_t* cur = (k & 1) ? rb : ra;
        uint32_t* nxt = (k & 1) ? ra : rb;
        if (k + 1 < 4) DCAT_TMEM_LD32(TS + (k + 1) * 32, nxt);
        const int c0 = 32 * k;
        uint32_t pk[16];
        const bool none = c0 >= lim_max || c0 + 32 <= lo;
        const bool full = c0 >= lo && c0 + 32 <= lim_min;
        if (none) {
#pragma unroll
            for (int i = 0; i < 16; i++) pk[i] = 0u;
        } else if (full) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float x0 = fmaf(__uint_as_float(cur[i]), sl2, u);
                const float x1 = fmaf(__uint_as_float(cur[i + 1]), sl2, u);
                constexpr int PP = POLY > 0 ? POLY : 1;
                const bool poly = POLY > 0 && ((i >> 1) % PP) == PP - 1;
                const float e0 = poly ? ex2p(x0) : ex2a(x0);
                const float e1 = poly ? ex2p(x1) : ex2a(x1);
                pk[i >> 1] = pack_bf16(e0, e1);
                // l sums the bf16 values the PV MMA multiplies: O / l is then an exactly normalised
                // weighting (a dominant key gets weight 1 whatever the rounding of its p)
                s0 += __uint_as_float(pk[i >> 1] << 16);
                s1 += __uint_as_float(pk[i >> 1] & 0xFFFF0000u);
            }
        } else {
            const uint32_t span = static_cast<uint32_t>(max(lim - lo, 0));  // valid: (c - lo) < span, unsigned
            // (lim < lo: a causal row whose visible keys all lie before this chunk)
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float x0 = static_cast<uint32_t>(c0 + i - lo) < span ? fmaf(__uint_as_float(cur[i]), sl2, u)
                                                                           : -INFINITY;
                const float x1 = static_cast<uint32_t>(c0 + i + 1 - lo) < span
                                     ? fmaf(__uint_as_float(cur[i + 1]), sl2, u)
                                     : -INFINITY;
                const float e0 = ex2a(x0), e1 = ex2a(x1);  // exp2(-inf) = 0
                pk[i >> 1] = pack_bf16(e0, e1);
                s0 += __uint_as_float(pk[i >> 1] << 16);
                s1 += __uint_as_float(pk[i >> 1] & 0xFFFF0000u);
            }
        }
        st16(TP + (c0 >> 1), pk);
        if (k + 1 < 4) ptx::tmem_wait_ld();
    }
    return s0 + s1;
}
// row max only (causal first chunk: no running max yet)
__device__ __forceinline__ float max_pass(uint32_t TS, int lo, int lim) {
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint32_t r[32];
        DCAT_TMEM_LD32(TS + 32 * k, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const float a0 = (32 * k + i >= lo && 32 * k + i < lim) ? __uint_as_float(r[i]) : -INFINITY;
            const float a1 = (32 * k + i + 1 >= lo && 32 * k + i + 1 < lim) ? __uint_as_float(r[i + 1]) : -INFINITY;
            mx = fmax3(mx, a0, a1);
        }
    }
    return mx;
}
// DH bf16 of one global row -> packed registers (DH / 2 words)
template <int DH>
__device__ __forceinline__ void load_row(const bf16* src, uint32_t* w) {
#pragma unroll
    for (int i = 0; i < DH / 8; i++) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + i);
        w[4 * i] = v.x;
        w[4 * i + 1] = v.y;
        w[4 * i + 2] = v.z;
        w[4 * i + 3] = v.w;
    }
}
__device__ __forceinline__ float2 unpack2(uint32_t w) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
}

template <int DH, bool CAUSAL, int POLY>
__global__ void __launch_bounds__(384, 1)
    k_attn_fa(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmVt, const __grid_constant__ CUtensorMap tmKs,
              const __grid_constant__ CUtensorMap tmVs, const AttnArgs p) {
    using C = FaCfg<DH>;
    using S = FaSmem<DH, CAUSAL>;
    constexpr int NQS = S::NQS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    FaBars* bars = reinterpret_cast<FaBars*>(smem + S::BAR);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = p.n_tiles * p.n_heads;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmQ);
        ptx::tma_prefetch(&tmK);
        ptx::tma_prefetch(&tmVt);
        for (int g = 0; g < 2; g++) {
            FaBars& b = bars[g];
            for (int s = 0; s < 2; s++) {
                ptx::mbar_init(&b.q_full[s], 1);
                ptx::mbar_init(&b.q_empty[s], CAUSAL ? 1 : 1 + 4);  // MMA commit (+ softmax: self rows read)
            }
            ptx::mbar_init(&b.s_full, 1);
            ptx::mbar_init(&b.p_full, 4);
            ptx::mbar_init(&b.o_final, 1);
            for (int s = 0; s < C::NST; s++) {
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
    // item of pipeline g, k-th turn: adjacent heads of one tile on the two pipelines of a CTA
    auto item_of = [&](int g, int k) { return 2 * (static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x)) + g; };

    if (warp < 4) {
        const int g = warp >> 1;
        FaBars& b = bars[g];
        uint8_t* gs = smem + g * S::GROUP;  // NQS item slots | kv ring
        uint8_t* kv0 = gs + NQS * S::QSLOT;
        if (lane == 0 && (warp & 1) == 0) {
            // ---------------- TMA producer of pipeline g
            uint32_t j = 0, kc = 0;
            for (int k = 0;; k++, j++) {
                const int w = item_of(g, k);
                if (w >= n_items) break;
                const FaItem it = fa_item(p, w);
                const int hc = it.h * DH;
                const int qs = j % NQS;
                FA_WAIT(&b.q_empty[qs], ((j / NQS) & 1) ^ 1, 1);
                ptx::mbar_expect_tx(&b.q_full[qs], S::QSLOT);
                ptx::tma_load_2d(gs + qs * S::QSLOT, &tmQ, &b.q_full[qs], hc, it.t.q0);
                if constexpr (!CAUSAL) {
                    ptx::tma_load_2d(gs + qs * S::QSLOT + C::TQ, &tmKs, &b.q_full[qs], hc, it.t.q0);
                    ptx::tma_load_2d(gs + qs * S::QSLOT + 2 * C::TQ, &tmVs, &b.q_full[qs], hc, it.t.q0);
                }
                for (int c = 0; c < it.nchunks; c++, kc++) {
                    const int ks = kc % C::NST;
                    uint8_t* kb = kv0 + ks * C::SLOT;
                    const int k0 = it.a0 + c * C::KC;
                    FA_WAIT(&b.kv_empty[ks], ((kc / C::NST) & 1) ^ 1, 2);
                    ptx::mbar_expect_tx(&b.kv_full[ks], C::SLOT);
                    ptx::tma_load_2d(kb, &tmK, &b.kv_full[ks], hc, k0);
#pragma unroll
                    for (int vb = 0; vb < C::KC / 64; vb++)
                        ptx::tma_load_2d(kb + C::TK + vb * C::VTB, &tmVt, &b.kv_full[ks], k0 + vb * 64, hc);
                }
            }
        } else if (lane == 0) {
            // ---------------- MMA issuer of pipeline g
            constexpr uint32_t idesc_s = ptx::idesc_bf16(128, C::KC);
            constexpr uint32_t idesc_o = ptx::idesc_bf16(128, DH);
            const uint32_t TG = tmem + 256 * g;
            uint32_t j = 0, sc = 0, pks = 0;
            bool pend = false;
            auto issue_pv = [&](uint32_t x, uint32_t ks) {  // O += P(x) V_x, then release the kv slot
                const uint32_t va = ptx::smem_u32(kv0 + ks * C::SLOT + C::TK);
                FA_WAIT(&b.p_full, x & 1, 3);  // P(x) in TMEM, S(x) read, O initialised / rescaled
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < C::KC / 16; kk++)
                    mma_ts(TG + C::T_O, TG + C::T_P + 8 * kk, fdesc(va + (kk >> 2) * C::VTB + (kk & 3) * 32, 2, 1024),
                           idesc_o, 1);
                ptx::mma_commit(&b.kv_empty[ks]);
            };
            for (int k = 0;; k++, j++) {
                const int w = item_of(g, k);
                if (w >= n_items) break;
                const FaItem it = fa_item(p, w);
                const int qs = j % NQS;
                const uint32_t qa = ptx::smem_u32(gs + qs * S::QSLOT);
                FA_WAIT(&b.q_full[qs], (j / NQS) & 1, 4);
                for (int c = 0; c < it.nchunks; c++, sc++) {
                    const uint32_t ks = sc % C::NST;
                    const uint32_t ka = ptx::smem_u32(kv0 + ks * C::SLOT);
                    FA_WAIT(&b.kv_full[ks], (sc / C::NST) & 1, 5);
                    if (pend) issue_pv(sc - 1, pks);  // also: S(sc - 1) fully read -> S may be overwritten
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kq = 0; kq < DH / 16; kq++)
                        ptx::mma_bf16(TG + C::T_S, fdesc(qa + kq * 32, C::LAYOUT, C::SBO),
                                      fdesc(ka + kq * 32, C::LAYOUT, C::SBO), idesc_s, kq > 0);
                    ptx::mma_commit(&b.s_full);  // completes after S(sc) and every earlier PV
                    if (c + 1 == it.nchunks) ptx::mma_commit(&b.q_empty[qs]);
                    pend = true;
                    pks = ks;
                }
                if (it.nchunks == 0) ptx::mma_commit(&b.q_empty[qs]);
            }
            if (pend) issue_pv(sc - 1, pks);
            ptx::mma_commit(&b.o_final);
        }
    } else {
        // ---------------- softmax of pipeline g: one thread per query row
        const int g = (warp - 4) >> 2, q = warp & 3;
        FaBars& b = bars[g];
        const int r = q * 32 + lane;
        const uint32_t TG = tmem + 256 * g + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t TS = TG + C::T_S, TP = TG + C::T_P, TO = TG + C::T_O;
        const float sl2 = p.scale * 1.4426950408889634f;
        const float lazy_hi = exp2f(DCAT_FA_LAZY), lazy_lo = exp2f(-DCAT_FA_LAZY);
        bf16* const out = static_cast<bf16*>(p.out);
        uint32_t sc = 0;
        bool pend_out = false;  // the previous item's O waits in TMEM until its last PV is known done
        int pend_row = 0, pend_hc = 0;
        float pend_l = 1.f;
        auto store_row = [&](int row, int hc, const float* o, float inv) {
            bf16* op = out + static_cast<size_t>(row) * p.ldo + hc;
#pragma unroll
            for (int i = 0; i < DH; i += 8) {
                uint4 wv;
                wv.x = pack_bf16(o[i] * inv, o[i + 1] * inv);
                wv.y = pack_bf16(o[i + 2] * inv, o[i + 3] * inv);
                wv.z = pack_bf16(o[i + 4] * inv, o[i + 5] * inv);
                wv.w = pack_bf16(o[i + 6] * inv, o[i + 7] * inv);
                *reinterpret_cast<uint4*>(op + i) = wv;
            }
        };
        auto flush = [&]() {  // O final of the pending item (its last PV has completed)
            float o[DH];
            o_load<DH>(TO, o);
            if (pend_row >= 0) store_row(pend_row, pend_hc, o, 1.f / pend_l);
            pend_out = false;
        };
        for (int k = 0;; k++) {
            const int w = item_of(g, k);
            if (w >= n_items) break;
            const FaItem it = fa_item(p, w);
            const int hc = it.h * DH;
            const bool live = r < it.t.nq;
            float m = -INFINITY, l = 0.f;
            const int qs = k % NQS;  // crossing: the item's Q | k_self | v_self slot
            const uint32_t qa = ptx::smem_u32(smem + g * S::GROUP + qs * S::QSLOT);
            if constexpr (!CAUSAL) {
                // self term (the candidate's own key / value, dcat.cpp:242-243): m = q . k_self, l = 1;
                // v_self becomes the O initial state (read at the first chunk, then the slot is released)
                FA_WAIT(&b.q_full[qs], (k / NQS) & 1, 14);
                float d0 = 0.f, d1 = 0.f;
#pragma unroll
                for (int jc = 0; jc < DH / 8; jc++) {
                    uint32_t qw[4], kw[4];
                    row_chunk_w<DH>(qa, r, jc, qw);
                    row_chunk_w<DH>(qa + C::TQ, r, jc, kw);
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const float2 a = unpack2(qw[i]), c = unpack2(kw[i]);
                        d0 = fmaf(a.x, c.x, d0);
                        d1 = fmaf(a.y, c.y, d1);
                    }
                }
                m = d0 + d1;
                l = 1.f;
            }
            // v_self chunk jc (8 columns) of this row, fp32
            auto vself8 = [&](int jc, float* v) {
                uint32_t w4[4];
                row_chunk_w<DH>(qa + 2 * C::TQ, r, jc, w4);
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const float2 f = unpack2(w4[i]);
                    v[2 * i] = f.x;
                    v[2 * i + 1] = f.y;
                }
            };
            if (it.nchunks == 0) {  // no context keys: softmax over the self term alone -> v_self
                if constexpr (!CAUSAL) {
                    if (live) {
                        float o[DH];
#pragma unroll
                        for (int jc = 0; jc < DH / 8; jc++) vself8(jc, o + 8 * jc);
                        store_row(it.t.q0 + r, hc, o, 1.f);
                    }
                    __syncwarp();
                    if (lane == 0) arrive1(&b.q_empty[qs]);
                }
                continue;
            }
            for (int c = 0; c < it.nchunks; c++, sc++) {
                const int cb = it.a0 + c * C::KC;       // token row of S column 0
                const int lo = max(0, it.t.kv0 - cb);   // valid S columns [lo, lim)
                int lim = min(C::KC, it.t.kv0 + it.t.nkv - cb);
                if (CAUSAL) lim = min(lim, it.t.kv0 + it.t.qloc + r + 1 - cb);
                const int lim_min = __reduce_min_sync(0xffffffffu, lim), lim_max = __reduce_max_sync(0xffffffffu, lim);
                FA_WAIT(&b.s_full, sc & 1, 7);  // S(sc) ready, and every earlier PV of this pipeline done
                ptx::tc_fence_after();
                // a warp whose 32 rows all lie past the tile's queries (sparse crossing tiles: a unique
                // with few candidates; the last tile of a unique's causal pass) keeps the pipeline's
                // barrier protocol but does no softmax: its P / O lanes feed rows nobody reads
                const bool idle = 32 * q >= it.t.nq;  // warp-uniform
                if (c == 0) {  // O: flush the previous item's, then this item's initial state
                    if (pend_out) flush();
#pragma unroll
                    for (int jc = 0; jc < DH / 8; jc++) {
                        if (idle) break;
                        float o[8];
                        if constexpr (CAUSAL) {
#pragma unroll
                            for (int i = 0; i < 8; i++) o[i] = 0.f;
                        } else {
                            vself8(jc, o);
                        }
                        o_store<8>(TO + 8 * jc, o);
                    }
                    if constexpr (!CAUSAL) {
                        __syncwarp();
                        if (lane == 0) arrive1(&b.q_empty[qs]);  // slot read (q, k_self, v_self)
                    }
                    pend_out = !idle;
                    pend_row = live ? it.t.q0 + r : -1;
                    pend_hc = hc;
                }
                if (idle) {
                    __syncwarp();
                    if (lane == 0) arrive1(&b.p_full);
                    continue;
                }
                // Running max by exception: P is computed against the current m (the self logit for the
                // crossing pass; 0 for a causal item's first chunk, which has no prior). Every p <= the
                // chunk's row sum, so a sum <= 2^LAZY bounds every p; a larger sum (or, on a causal
                // first chunk, a sum below 2^-LAZY) sends the row through an exact max pass and a
                // recompute. Rows below the bound keep m: p <= 2^LAZY and o / l is unchanged up to
                // rounding.
#ifdef DCAT_FA_CAUSAL_MAXPASS
                if (CAUSAL && c == 0) m = max_pass(TS, lo, lim);
#else
                if (CAUSAL && c == 0) m = 0.f;
#endif
                float u = -m * sl2;
                float csum = p_pass<POLY>(TS, TP, sl2, u, lo, lim, lim_min, lim_max);
                const bool redo = !(csum <= lazy_hi) || (CAUSAL && c == 0 && csum < lazy_lo);  // NaN / inf too
                // warp-uniform branch (tcgen05.ld / st are .sync.aligned): rows that need no redo keep
                // their max (alpha = 1) and recompute the same P
                if (__any_sync(0xffffffffu, redo)) {
                    ptx::tmem_wait_st();
                    const float cm = max_pass(TS, lo, lim);
                    float alpha = 1.f;
                    if (redo && cm != -INFINITY) {
                        const float mn = (CAUSAL && c == 0) ? cm : fmaxf(m, cm);
                        alpha = ex2a((m - mn) * sl2);  // O, l are still 0 on a causal first chunk
                        m = mn;
                    }
                    u = -m * sl2;
#pragma unroll
                    for (int jc = 0; jc < DH / 8; jc++) {
                        float o[8];
                        o_load<8>(TO + 8 * jc, o);
#pragma unroll
                        for (int i = 0; i < 8; i++) o[i] *= alpha;
                        o_store<8>(TO + 8 * jc, o);
                    }
                    l *= alpha;
                    csum = p_pass<POLY>(TS, TP, sl2, u, lo, lim, lim_min, lim_max);
                    if (p.dbg != nullptr && redo) atomicAdd(p.dbg + (CAUSAL ? 0 : 1), 1u);
                }
                l += csum;
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive1(&b.p_full);
            }
            pend_l = l;
        }
        if (pend_out) {  // the last item's final PV
            FA_WAIT(&b.o_final, 0, 6);
            ptx::tc_fence_after();
            flush();
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

typedef CUresult (*EncodeFnF)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFnF encoder_f() {
    static EncodeFnF fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFnF>(f);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D bf16 map: `cols` x `rows` (cols contiguous, ld_elems apart), box box_c x box_r
CUtensorMap map_f(const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems, uint32_t box_c, uint32_t box_r,
                  CUtensorMapSwizzle sw) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    if (!base) return m;
    cuuint64_t dims[2] = {cols, rows > 0 ? rows : 1};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * 2) & 15))
        throw CudaError("attention tensor map: 16-byte alignment");
    CUresult r = encoder_f()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
    return m;
}

int sm_count_f() {
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

// POLY: every POLY-th pair of exponentials on the FMA pipe (ex2p) beside MUFU.EX2. Measured
// (profiles/r02_attention.md): the crossing kernel gains at POLY = 4 (PinFM-base 0.631 -> 0.607 ms,
// high-fanout 8.96 -> 8.61 ms per step), the causal kernel loses (0.597 -> 0.681 ms), so only the
// crossing kernel uses it.
#ifndef DCAT_FA_POLY
#define DCAT_FA_POLY 0
#endif
#ifndef DCAT_FA_POLY_CROSS
#define DCAT_FA_POLY_CROSS 4
#endif

template <int DH, bool CAUSAL>
void launch_fa(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    using Sm = FaSmem<DH, CAUSAL>;
    static_assert(Sm::TOTAL <= 227 * 1024, "shared memory budget");
    auto kern = k_attn_fa<DH, CAUSAL, CAUSAL ? DCAT_FA_POLY : DCAT_FA_POLY_CROSS>;
    set_smem_attr(reinterpret_cast<const void*>(kern), Sm::TOTAL);
    const int d = a.n_heads * DH;
    const CUtensorMapSwizzle swq =
        DH == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : (DH == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
    // K / V^T extents are the real key count (kv_rows): keys past it read as zeros, never as
    // uninitialised padding (0 * NaN would poison the PV accumulation)
    const CUtensorMap tq = map_f(a.q, d, q_rows, a.ldq, DH, 128, swq);
    const CUtensorMap tk = map_f(a.k, d, kv_rows, a.ldkv, DH, 128, swq);
    const CUtensorMap tv = map_f(a.v, kv_rows, d, a.ldvt, 64, DH, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tks, tvs;
    std::memset(&tks, 0, sizeof tks);
    std::memset(&tvs, 0, sizeof tvs);
    if (!CAUSAL) {
        tks = map_f(a.kself, d, q_rows, a.ldself, DH, 128, swq);
        tvs = map_f(a.vself, d, q_rows, a.ldself, DH, 128, swq);
    }
    const int64_t items = static_cast<int64_t>(a.n_tiles) * a.n_heads;
    const int64_t pairs = (items + 1) / 2;
    const int grid = static_cast<int>(pairs < sm_count_f() ? pairs : sm_count_f());
    kern<<<grid, 384, Sm::TOTAL, s>>>(tq, tk, tv, tks, tvs, a);
    DCAT_LAUNCH_CHECK();
}

}  // namespace

bool attention_fa_supported(int dh) { return dh == 16 || dh == 32 || dh == 64; }

void attention_fa(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    if (a.n_tiles <= 0) return;
    if (a.ldvt <= 0) throw InvalidArg("attention_fa needs the transposed V cache");
    switch (a.dh) {
        case 16: a.causal ? launch_fa<16, true>(a, q_rows, kv_rows, s) : launch_fa<16, false>(a, q_rows, kv_rows, s); break;
        case 32: a.causal ? launch_fa<32, true>(a, q_rows, kv_rows, s) : launch_fa<32, false>(a, q_rows, kv_rows, s); break;
        case 64: a.causal ? launch_fa<64, true>(a, q_rows, kv_rows, s) : launch_fa<64, false>(a, q_rows, kv_rows, s); break;
        default: throw InvalidArg("attention_fa: head dim " + std::to_string(a.dh) + " not supported");
    }
}

}  // namespace dcat
