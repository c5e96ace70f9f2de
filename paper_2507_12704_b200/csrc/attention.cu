// attention.cu — K5 context attention and K6 crossing attention.
//
// K5 (context pass): causal multi-head softmax attention of each unique's
//    tokens over its own tokens, as in layer_forward (model.cpp:353-376).
// K6 (crossing pass): each candidate query attends to its unique's cached
//    context K/V plus its own key/value, as in cross_forward (dcat.cpp:231-263).
//    The reference materializes [K_u; k] per candidate (dcat.cpp:239-243);
//    here the candidates of one unique are packed as the M dimension of a
//    query tile (Tile in launch.h), the unique's K/V blocks are staged once per
//    tile in shared memory and the self key/value enters the online softmax as
//    a per-row initial state (m = q.k_self, l = 1, o = v_self).
//
// bf16 path: flash-style kernel, WARPS x 16 query rows per CTA, 64-key blocks
// through an NST-stage cp.async ring, QK^T and PV on mma.sync m16n8k16 (bf16 in,
// fp32 accumulate). With head dim 32 the kernel is bound by the softmax, not
// the tensor pipe, so the per-score work is cut to one FFMA + one MUFU.EX2:
// masks only on partial blocks, row max on raw scores, and the row sums are
// accumulated by the tensor core (P times a ones column) in the same rescaled
// accumulators as O.
// fp32 path (parity) and tiny head dims: one warp per (query, head) restating
// the reference's exact loop order: logits, max, exp-sum, axpy over keys.
#include <math.h>

#include <mutex>

#include "launch.h"

namespace dcat {

namespace {

constexpr int BKV = 64;  // keys per block (cp.async stage)

__device__ __forceinline__ void cp_async16(uint32_t s, const void* gmem, bool pred) {
    int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, uint32_t s) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, uint32_t s) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s));
}
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
    uint32_t y;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int DH, bool CAUSAL, int WARPS, int RT>
struct FlashCfg {
    static constexpr int BQ = WARPS * 16 * RT;
    static constexpr int LD = DH + 8;  // padded smem row (bf16): conflict-free ldmatrix
    static constexpr int Q_ELEMS = BQ * LD;
    static constexpr int KV_ELEMS = BKV * LD;
    // K/V blocks in flight (cp.async ring). More stages than 2 cost L1 (the carve-out grows)
    // and measured slower for the crossing kernel; the context kernel keeps 3.
#ifndef DCAT_XNST
#define DCAT_XNST 2
#endif
    static constexpr int NST = DH <= 32 ? (CAUSAL && RT == 1 ? 3 : DCAT_XNST) : 2;
    static constexpr int SMEM = (Q_ELEMS + 2 * NST * KV_ELEMS) * 2;
};

// RT: 16-row m-tiles per warp. With RT = 2 (crossing) a warp holds two independent online-
// softmax states: every K / V fragment read by ldmatrix feeds both, and the two dependency
// chains (mma -> max -> exp -> mma) interleave.
#ifndef DCAT_XSUB
#define DCAT_XSUB 32
#endif
#ifndef DCAT_XRT
#define DCAT_XRT 2
#endif
#ifndef DCAT_FLASH_ABLATE  // kernel experiments only (tools/build_variant.sh): 1 no exp, 2 no PV, 4 no QK, 8 no K/V loads
#define DCAT_FLASH_ABLATE 0
#endif
#ifndef DCAT_CRT
#define DCAT_CRT 2
#endif
// resident CTAs per SM: crossing 4 (128 queries); context 6 (4 warps x 1 m-tile, 80 registers)
// or 8 (2 warps x 2 m-tiles, 128 registers)
template <int DH, bool CAUSAL, int WARPS, int RT>
constexpr int flash_min_blocks() {
#ifdef DCAT_FLASH_THREADS_PER_SM  // experiments: resident threads per SM the register budget targets
    return DH <= 32 ? (RT == 2 ? DCAT_FLASH_THREADS_PER_SM / (WARPS * 32) : (CAUSAL ? 6 : 4)) : (CAUSAL ? 4 : 2);
#else
    return DH <= 32 ? (RT == 2 ? 512 / (WARPS * 32) : (CAUSAL ? 6 : 4)) : (CAUSAL ? 4 : 2);
#endif
}
// SKIP: warps whose rows all lie past the tile's queries only stage K/V. Instantiated for sparse
// crossing tiles (a unique with few candidates fills a fraction of the 128 rows: low-dedup has 4
// per tile, attention 10.0 -> 7.2 ms); full tiles run the variant without the branch, which
// measured 1-2 % faster on them.
template <int DH, bool CAUSAL, int WARPS, int RT, bool SKIP>
__global__ void __launch_bounds__(WARPS * 32, flash_min_blocks<DH, CAUSAL, WARPS, RT>()) k_flash(AttnArgs p) {
    // keys per online-softmax step: the context kernel keeps whole 64-key blocks (6 CTAs/SM at
    // 80 registers), the crossing kernel halves them (register footprint)
    constexpr int SUB = CAUSAL && RT == 1 ? 64 : DCAT_XSUB;
    using C = FlashCfg<DH, CAUSAL, WARPS, RT>;
    constexpr int LD = C::LD;
    constexpr int NST = C::NST;
    constexpr int CHUNKS = DH / 8;  // 16-byte chunks per row
    constexpr int NT = DH / 8;      // n-tiles of the output
    constexpr int NTHR = WARPS * 32;
    extern __shared__ __align__(16) bf16 smem_attn[];
    const uint32_t sQ = static_cast<uint32_t>(__cvta_generic_to_shared(smem_attn));
    const uint32_t sK0 = sQ + C::Q_ELEMS * 2;
    const uint32_t sV0 = sK0 + NST * C::KV_ELEMS * 2;

    // linear grid, head fastest: the heads of one tile run together and share its K/V lines in L2
    const Tile tile = p.tiles[blockIdx.x / p.n_heads];
    const int h = blockIdx.x % p.n_heads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const bf16* Q = static_cast<const bf16*>(p.q);
    const bf16* K = static_cast<const bf16*>(p.k);
    const bf16* V = static_cast<const bf16*>(p.v);
    const int hc = h * DH;

    for (int i = threadIdx.x; i < C::BQ * CHUNKS; i += NTHR) {
        int r = i / CHUNKS, c = i % CHUNKS;
        bool ok = r < tile.nq;
        const bf16* src = Q + static_cast<size_t>(tile.q0 + (ok ? r : 0)) * p.ldq + hc + c * 8;
        cp_async16(sQ + 2 * (r * LD + c * 8), src, ok);
    }
    const int nblk = (tile.nkv + BKV - 1) / BKV;
    auto load_kv = [&](int blk, int buf) {
        for (int i = threadIdx.x; i < BKV * CHUNKS; i += NTHR) {
            int r = i / CHUNKS, c = i % CHUNKS;
            int key = blk * BKV + r;
            bool ok = key < tile.nkv;
            size_t off = static_cast<size_t>(tile.kv0 + (ok ? key : 0)) * p.ldkv + hc + c * 8;
            uint32_t so = 2 * (buf * C::KV_ELEMS + r * LD + c * 8);
            if (DCAT_FLASH_ABLATE & 8) continue;
            cp_async16(sK0 + so, K + off, ok);
            cp_async16(sV0 + so, V + off, ok);
        }
    };
    cp_async_commit();  // group Q
#pragma unroll
    for (int b = 0; b < NST - 1; b++) {  // groups of blocks 0 .. NST-2 (empty past the end)
        if (b < nblk) load_kv(b, b);
        cp_async_commit();
    }

    const float sl2 = p.scale * 1.4426950408889634f;  // scale * log2(e)
    const uint32_t ONES = 0x3F803F80u;                  // bf16x2 (1, 1)
    // m-tile t of this warp: tile-local rows rw[t] + g and rw[t] + g + 8
    int rw[RT];
#pragma unroll
    for (int t = 0; t < RT; t++) rw[t] = (warp * RT + t) * 16;
    float o[RT][NT][4];
    float lacc[RT][4];  // row sums (every column equal), rescaled with o
    float mx[RT][2];    // running row max of the RAW scores (rows g, g + 8)
#pragma unroll
    for (int t = 0; t < RT; t++) {
#pragma unroll
        for (int j = 0; j < NT; j++) o[t][j][0] = o[t][j][1] = o[t][j][2] = o[t][j][3] = 0.f;
        lacc[t][0] = lacc[t][1] = lacc[t][2] = lacc[t][3] = 0.f;
        mx[t][0] = mx[t][1] = -INFINITY;
    }

    if constexpr (!CAUSAL) {
        // self term: initial state m = q . k_self, l = 1, o = v_self. The self rows are loaded
        // while the K/V blocks are in flight; q comes from smem once group Q has landed.
        const bf16* KS = static_cast<const bf16*>(p.kself);
        const bf16* VS = static_cast<const bf16*>(p.vself);
        const bf16* sq = smem_attn;
        __nv_bfloat162 ks[RT][NT][2];
#pragma unroll
        for (int t = 0; t < RT; t++) {
            const int r0 = rw[t] + g, r1 = r0 + 8;
            const int q0r = tile.q0 + (r0 < tile.nq ? r0 : 0), q1r = tile.q0 + (r1 < tile.nq ? r1 : 0);
#pragma unroll
            for (int j = 0; j < NT; j++) {
                int c = j * 8 + 2 * t4;
                ks[t][j][0] = *reinterpret_cast<const __nv_bfloat162*>(KS + static_cast<size_t>(q0r) * p.ldself + hc + c);
                ks[t][j][1] = *reinterpret_cast<const __nv_bfloat162*>(KS + static_cast<size_t>(q1r) * p.ldself + hc + c);
                float2 va = __bfloat1622float2(
                    *reinterpret_cast<const __nv_bfloat162*>(VS + static_cast<size_t>(q0r) * p.ldself + hc + c));
                float2 vb = __bfloat1622float2(
                    *reinterpret_cast<const __nv_bfloat162*>(VS + static_cast<size_t>(q1r) * p.ldself + hc + c));
                o[t][j][0] = va.x;
                o[t][j][1] = va.y;
                o[t][j][2] = vb.x;
                o[t][j][3] = vb.y;
            }
        }
        cp_async_wait<NST - 1>();  // group Q
        __syncthreads();
#pragma unroll
        for (int t = 0; t < RT; t++) {
            const int r0 = rw[t] + g, r1 = r0 + 8;
            float d0 = 0.f, d1 = 0.f;
#pragma unroll
            for (int j = 0; j < NT; j++) {
                int c = j * 8 + 2 * t4;
                float2 qa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + r0 * LD + c));
                float2 qb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + r1 * LD + c));
                float2 ka = __bfloat1622float2(ks[t][j][0]), kb = __bfloat1622float2(ks[t][j][1]);
                d0 += qa.x * ka.x + qa.y * ka.y;
                d1 += qb.x * kb.x + qb.y * kb.y;
            }
            d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
            d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
            d1 += __shfl_xor_sync(0xffffffffu, d1, 1);
            d1 += __shfl_xor_sync(0xffffffffu, d1, 2);
            mx[t][0] = d0;
            mx[t][1] = d1;
            lacc[t][0] = lacc[t][1] = lacc[t][2] = lacc[t][3] = 1.f;
        }
    } else {
        cp_async_wait<NST - 1>();  // group Q
        __syncthreads();
    }

    // Q fragments (A operand), kept in registers for all key blocks
    uint32_t qf[RT][DH / 16][4];
#pragma unroll
    for (int t = 0; t < RT; t++)
#pragma unroll
        for (int kk = 0; kk < DH / 16; kk++) {
            int row = rw[t] + (lane & 7) + 8 * ((lane >> 3) & 1);
            int col = kk * 16 + 8 * (lane >> 4);
            ldsm_x4(qf[t][kk], sQ + 2 * (row * LD + col));
        }

    const bool warp_idle = rw[0] >= tile.nq;  // warp-uniform
    for (int blk = 0; blk < nblk; blk++) {
        const int buf = blk % NST;
        cp_async_wait<NST - 2>();  // block blk has landed (the NST - 2 newer groups may be in flight)
        __syncthreads();           // ... for every thread, and block blk - 1's buffer is free
        if (blk + NST - 1 < nblk) load_kv(blk + NST - 1, (blk + NST - 1) % NST);
        cp_async_commit();

#pragma unroll
        for (int sub = 0; sub < BKV / SUB; sub++) {  // SUB-key online-softmax steps (register footprint)
            constexpr int NJ = SUB / 8;                // n-tiles of S
            const int kbase = blk * BKV + sub * SUB;
            if (kbase >= tile.nkv) break;  // uniform across the CTA
            if (SKIP && warp_idle) continue;  // idle warp: K/V staging only
            // causal: keys past this warp's last query row are masked for all its rows (warp-uniform)
            if (CAUSAL && kbase > tile.qloc + rw[RT - 1] + 15) continue;
            float s[RT][NJ][4];
#pragma unroll
            for (int t = 0; t < RT; t++)
#pragma unroll
                for (int j = 0; j < NJ; j++) s[t][j][0] = s[t][j][1] = s[t][j][2] = s[t][j][3] = 0.f;
            const uint32_t kb = sK0 + 2 * (buf * C::KV_ELEMS + sub * SUB * LD);
#pragma unroll
            for (int kk = 0; kk < DH / 16; kk++) {
#pragma unroll
                for (int j = 0; j < NJ; j += 2) {
                    uint32_t b[4];
                    int key = 8 * (j + (lane >> 4)) + (lane & 7);
                    int col = kk * 16 + 8 * ((lane >> 3) & 1);
                    ldsm_x4(b, kb + 2 * (key * LD + col));
                    if (DCAT_FLASH_ABLATE & 4) { s[0][j][0] += __uint_as_float(b[0]); continue; }
#pragma unroll
                    for (int t = 0; t < RT; t++) {
                        mma16816(s[t][j], qf[t][kk], b[0], b[1]);
                        mma16816(s[t][j + 1], qf[t][kk], b[2], b[3]);
                    }
                }
            }
            uint32_t pf[RT][NJ / 2][4];
#pragma unroll
            for (int t = 0; t < RT; t++) {
                const int r0 = rw[t] + g, r1 = r0 + 8;
                const bool full = (kbase + SUB <= tile.nkv) && (!CAUSAL || kbase + SUB - 1 <= tile.qloc + rw[t]);
                if (!full) {
#pragma unroll
                    for (int j = 0; j < NJ; j++) {
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            int key = kbase + 8 * j + 2 * t4 + (e & 1);
                            int row = (e < 2) ? r0 : r1;
                            bool ok = key < tile.nkv;
                            if (CAUSAL) ok = ok && key <= tile.qloc + row;
                            if (!ok) s[t][j][e] = -INFINITY;
                        }
                    }
                }
                float bm0 = s[t][0][0], bm1 = s[t][0][2];
#pragma unroll
                for (int j = 0; j < NJ; j++) {
                    bm0 = fmaxf(bm0, fmaxf(s[t][j][0], s[t][j][1]));
                    bm1 = fmaxf(bm1, fmaxf(s[t][j][2], s[t][j][3]));
                }
                bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 1));
                bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
                bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 1));
                bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
                // Lazy rescale: the running max only moves (and O, l are rescaled) when some row of
                // the warp sees a block max more than LAZY (log2 units) above it; otherwise the
                // stale max stays and p <= 2^LAZY. o / l is unchanged up to rounding, and the
                // per-step rescale (2 MUFU + 20 FMUL per thread) is skipped on most steps.
                constexpr float LAZY = 8.f;
                float& m0 = mx[t][0];
                float& m1 = mx[t][1];
                const bool grow = (bm0 - m0) * sl2 > LAZY || (bm1 - m1) * sl2 > LAZY;  // -inf - -inf: NaN
                if (__any_sync(0xffffffffu, grow)) {
                    if (p.dbg != nullptr && lane == 0) atomicAdd(p.dbg + (CAUSAL ? 0 : 1), 1u);
                    const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
                    const float a0 = nm0 == -INFINITY ? 1.f : ex2((m0 - nm0) * sl2);  // m = -inf -> 0
                    const float a1 = nm1 == -INFINITY ? 1.f : ex2((m1 - nm1) * sl2);
                    m0 = nm0;
                    m1 = nm1;
#pragma unroll
                    for (int j = 0; j < NT; j++) {
                        o[t][j][0] *= a0;
                        o[t][j][1] *= a0;
                        o[t][j][2] *= a1;
                        o[t][j][3] *= a1;
                    }
                    lacc[t][0] *= a0;
                    lacc[t][1] *= a0;
                    lacc[t][2] *= a1;
                    lacc[t][3] *= a1;
                }
                const float u0 = m0 == -INFINITY ? 0.f : -m0 * sl2;  // exponent offset (scaled)
                const float u1 = m1 == -INFINITY ? 0.f : -m1 * sl2;
#pragma unroll
                for (int j = 0; j < NJ; j++) {
                    float p0, p1, p2, p3;
                    if (DCAT_FLASH_ABLATE & 1) {
                        p0 = fmaf(s[t][j][0], sl2, u0), p1 = fmaf(s[t][j][1], sl2, u0);
                        p2 = fmaf(s[t][j][2], sl2, u1), p3 = fmaf(s[t][j][3], sl2, u1);
                    } else {
                        p0 = ex2(fmaf(s[t][j][0], sl2, u0)), p1 = ex2(fmaf(s[t][j][1], sl2, u0));
                        p2 = ex2(fmaf(s[t][j][2], sl2, u1)), p3 = ex2(fmaf(s[t][j][3], sl2, u1));
                    }
                    pf[t][j >> 1][(j & 1) * 2 + 0] = pack_bf16(p0, p1);
                    pf[t][j >> 1][(j & 1) * 2 + 1] = pack_bf16(p2, p3);
                }
            }
            // O += P V, l += P 1
            const uint32_t vb = sV0 + 2 * (buf * C::KV_ELEMS + sub * SUB * LD);
#pragma unroll
            for (int kk = 0; kk < NJ / 2; kk++) {
                int key = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
                for (int j = 0; j < NT; j += 2) {
                    uint32_t b[4];
                    ldsm_x4_t(b, vb + 2 * (key * LD + 8 * (j + (lane >> 4))));
                    if (DCAT_FLASH_ABLATE & 2) { o[0][j][0] += __uint_as_float(b[0] ^ pf[0][kk][0]); continue; }
#pragma unroll
                    for (int t = 0; t < RT; t++) {
                        mma16816(o[t][j], pf[t][kk], b[0], b[1]);
                        mma16816(o[t][j + 1], pf[t][kk], b[2], b[3]);
                    }
                }
#pragma unroll
                for (int t = 0; t < RT; t++) mma16816(lacc[t], pf[t][kk], ONES, ONES);
            }
        }
    }

    bf16* O = static_cast<bf16*>(p.out);
#pragma unroll
    for (int t = 0; t < RT; t++) {
        const int r0 = rw[t] + g, r1 = r0 + 8;
        const float i0 = 1.f / lacc[t][0], i1 = 1.f / lacc[t][2];
#pragma unroll
        for (int j = 0; j < NT; j++) {
            int c = hc + j * 8 + 2 * t4;
            if (r0 < tile.nq)
                *reinterpret_cast<uint32_t*>(O + static_cast<size_t>(tile.q0 + r0) * p.ldo + c) =
                    DCAT_FLASH_ABLATE ? 0u : pack_bf16(o[t][j][0] * i0, o[t][j][1] * i0);
            if (r1 < tile.nq)
                *reinterpret_cast<uint32_t*>(O + static_cast<size_t>(tile.q0 + r1) * p.ldo + c) =
                    DCAT_FLASH_ABLATE ? 0u : pack_bf16(o[t][j][2] * i1, o[t][j][3] * i1);
        }
    }
}

// ---- SIMT kernel: one warp per (query row, head), the reference's exact loop
// order (logits, max, exp-sum, axpy over keys in order). fp32 parity path for
// every head dim, and the bf16 path for head dims below the mma k-step (< 16).
template <typename T>
__global__ void k_attn_simt(AttnArgs p, int max_keys) {
    extern __shared__ float logits_all[];
    // linear grid, head fastest: the heads of one tile run together and share its K/V lines in L2
    const Tile tile = p.tiles[blockIdx.x / p.n_heads];
    const int h = blockIdx.x % p.n_heads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    float* logits = logits_all + warp * (max_keys + 1);
    const T* Q = static_cast<const T*>(p.q);
    const T* K = static_cast<const T*>(p.k);
    const T* V = static_cast<const T*>(p.v);
    const int dh = p.dh, hc = h * dh;
    for (int r = warp; r < tile.nq; r += nw) {
        const T* q = Q + static_cast<size_t>(tile.q0 + r) * p.ldq + hc;
        int nkeys = p.causal ? tile.qloc + r + 1 : tile.nkv + 1;  // crossing: context + self (last)
        float mx = -INFINITY;
        for (int j = 0; j < nkeys; j++) {
            const T* kr;
            if (!p.causal && j == tile.nkv)
                kr = static_cast<const T*>(p.kself) + static_cast<size_t>(tile.q0 + r) * p.ldself + hc;
            else
                kr = K + static_cast<size_t>(tile.kv0 + j) * p.ldkv + hc;
            float part = 0.f;
            for (int d = lane; d < dh; d += 32) part += ActIO<T>::load(q + d) * ActIO<T>::load(kr + d);
            float sdot = warp_sum(part) * p.scale;
            if (lane == 0) logits[j] = sdot;
            mx = fmaxf(mx, sdot);
        }
        __syncwarp();
        float denom = 0.f;
        for (int j = 0; j < nkeys; j++) denom += expf(logits[j] - mx);
        float inv = 1.0f / denom;
        for (int d = lane; d < dh; d += 32) {
            float acc = 0.f;
            for (int j = 0; j < nkeys; j++) {
                const T* vr;
                if (!p.causal && j == tile.nkv)
                    vr = static_cast<const T*>(p.vself) + static_cast<size_t>(tile.q0 + r) * p.ldself + hc;
                else
                    vr = V + static_cast<size_t>(tile.kv0 + j) * p.ldkv + hc;
                acc += (expf(logits[j] - mx) * inv) * ActIO<T>::load(vr + d);
            }
            ActIO<T>::store(static_cast<T*>(p.out) + static_cast<size_t>(tile.q0 + r) * p.ldo + hc + d, acc);
        }
        __syncwarp();
    }
}

template <typename T>
void launch_simt(const AttnArgs& a, cudaStream_t s) {
    const int warps = 4;
    size_t smem = static_cast<size_t>(warps) * (a.max_keys + 2) * sizeof(float);
    const dim3 grid(static_cast<unsigned>(a.n_tiles) * static_cast<unsigned>(a.n_heads));
    if (smem > 48 * 1024)
        DCAT_CUDA_CHECK(cudaFuncSetAttribute(k_attn_simt<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem)));
    k_attn_simt<T><<<grid, warps * 32, smem, s>>>(a, a.max_keys + 1);
    DCAT_LAUNCH_CHECK();
}

template <int DH, bool CAUSAL, int WARPS, int RT, bool SKIP = false>
void launch_flash_t(const AttnArgs& a, cudaStream_t s) {
    using C = FlashCfg<DH, CAUSAL, WARPS, RT>;
    set_smem_attr(reinterpret_cast<const void*>(k_flash<DH, CAUSAL, WARPS, RT, SKIP>), C::SMEM);
    const dim3 grid(static_cast<unsigned>(a.n_tiles) * static_cast<unsigned>(a.n_heads));
    k_flash<DH, CAUSAL, WARPS, RT, SKIP><<<grid, WARPS * 32, C::SMEM, s>>>(a);
    DCAT_LAUNCH_CHECK();
}

// context tiles hold 64 queries (DCAT_CRT m-tiles per warp), crossing tiles 128 (DCAT_XRT)
template <int DH>
void launch_flash(const AttnArgs& a, cudaStream_t s) {
    constexpr int RT = DH <= 32 ? DCAT_XRT : 1;
    constexpr int CRT = DH <= 32 ? DCAT_CRT : 1;
    if (a.causal) launch_flash_t<DH, true, kCtxTile / (16 * CRT), CRT>(a, s);
    else if (a.sparse_tiles) launch_flash_t<DH, false, (DH <= 32 ? kCrossTile : 128) / (16 * RT), RT, true>(a, s);
    else launch_flash_t<DH, false, (DH <= 32 ? kCrossTile : 128) / (16 * RT), RT, false>(a, s);
}

}  // namespace

void attention_bf16(const AttnArgs& a, cudaStream_t s) {
    if (a.n_tiles <= 0) return;
    switch (a.dh) {
        case 16: launch_flash<16>(a, s); break;
        case 32: launch_flash<32>(a, s); break;
        case 64: launch_flash<64>(a, s); break;
        default:
            if (a.dh % 16 == 0) throw InvalidArg("attention: head dim " + std::to_string(a.dh) + " not supported");
            launch_simt<bf16>(a, s);  // tiny head dims (< one mma k-step)
    }
}

void attention_f32(const AttnArgs& a, cudaStream_t s) {
    if (a.n_tiles <= 0) return;
    launch_simt<float>(a, s);
}

}  // namespace dcat
