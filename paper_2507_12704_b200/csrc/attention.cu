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
// double-buffered with cp.async, QK^T and PV on mma.sync m16n8k16 (bf16 in,
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
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int DH, int WARPS>
struct FlashCfg {
    static constexpr int BQ = WARPS * 16;
    static constexpr int LD = DH + 8;  // padded smem row (bf16): conflict-free ldmatrix
    static constexpr int Q_ELEMS = BQ * LD;
    static constexpr int KV_ELEMS = BKV * LD;
    static constexpr int SMEM = (Q_ELEMS + 4 * KV_ELEMS) * 2;
};

template <int DH, bool CAUSAL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, CAUSAL ? 6 : 4) k_flash(AttnArgs p) {
    // keys per online-softmax step: the context kernel keeps whole 64-key blocks (6 CTAs/SM at
    // 80 registers), the crossing kernel halves them to fit 4 CTAs of 8 warps (measured best)
    constexpr int SUB = CAUSAL ? 64 : 32;
    using C = FlashCfg<DH, WARPS>;
    constexpr int LD = C::LD;
    constexpr int CHUNKS = DH / 8;  // 16-byte chunks per row
    constexpr int NT = DH / 8;      // n-tiles of the output
    constexpr int NTHR = WARPS * 32;
    extern __shared__ __align__(16) bf16 smem_attn[];
    const uint32_t sQ = static_cast<uint32_t>(__cvta_generic_to_shared(smem_attn));
    const uint32_t sK0 = sQ + C::Q_ELEMS * 2;
    const uint32_t sV0 = sK0 + 2 * C::KV_ELEMS * 2;

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
            cp_async16(sK0 + so, K + off, ok);
            cp_async16(sV0 + so, V + off, ok);
        }
    };
    if (nblk > 0) load_kv(0, 0);
    cp_async_commit();

    const float sl2 = p.scale * 1.4426950408889634f;  // scale * log2(e)
    const int r0 = warp * 16 + g, r1 = r0 + 8;          // tile-local rows of this thread
    const uint32_t ONES = 0x3F803F80u;                  // bf16x2 (1, 1)
    float o[NT][4];
    float lacc[4];  // row sums (every column equal), rescaled with o
    float m0, m1;   // running row max of the RAW scores
#pragma unroll
    for (int j = 0; j < NT; j++) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    lacc[0] = lacc[1] = lacc[2] = lacc[3] = 0.f;
    m0 = m1 = -INFINITY;

    cp_async_wait<0>();
    __syncthreads();

    if constexpr (!CAUSAL) {
        // self term: initial state m = q . k_self, l = 1, o = v_self
        const bf16* KS = static_cast<const bf16*>(p.kself);
        const bf16* VS = static_cast<const bf16*>(p.vself);
        const bf16* sq = smem_attn;
        int q0r = tile.q0 + (r0 < tile.nq ? r0 : 0), q1r = tile.q0 + (r1 < tile.nq ? r1 : 0);
        float d0 = 0.f, d1 = 0.f;
#pragma unroll
        for (int j = 0; j < NT; j++) {
            int c = j * 8 + 2 * t4;
            float2 qa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + r0 * LD + c));
            float2 qb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + r1 * LD + c));
            float2 ka = __bfloat1622float2(
                *reinterpret_cast<const __nv_bfloat162*>(KS + static_cast<size_t>(q0r) * p.ldself + hc + c));
            float2 kb = __bfloat1622float2(
                *reinterpret_cast<const __nv_bfloat162*>(KS + static_cast<size_t>(q1r) * p.ldself + hc + c));
            d0 += qa.x * ka.x + qa.y * ka.y;
            d1 += qb.x * kb.x + qb.y * kb.y;
            float2 va = __bfloat1622float2(
                *reinterpret_cast<const __nv_bfloat162*>(VS + static_cast<size_t>(q0r) * p.ldself + hc + c));
            float2 vb = __bfloat1622float2(
                *reinterpret_cast<const __nv_bfloat162*>(VS + static_cast<size_t>(q1r) * p.ldself + hc + c));
            o[j][0] = va.x;
            o[j][1] = va.y;
            o[j][2] = vb.x;
            o[j][3] = vb.y;
        }
        d0 += __shfl_xor_sync(0xffffffffu, d0, 1);
        d0 += __shfl_xor_sync(0xffffffffu, d0, 2);
        d1 += __shfl_xor_sync(0xffffffffu, d1, 1);
        d1 += __shfl_xor_sync(0xffffffffu, d1, 2);
        m0 = d0;
        m1 = d1;
        lacc[0] = lacc[1] = lacc[2] = lacc[3] = 1.f;
    }

    // Q fragments (A operand), kept in registers for all key blocks
    uint32_t qf[DH / 16][4];
#pragma unroll
    for (int kk = 0; kk < DH / 16; kk++) {
        int row = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
        int col = kk * 16 + 8 * (lane >> 4);
        ldsm_x4(qf[kk], sQ + 2 * (row * LD + col));
    }

    for (int blk = 0; blk < nblk; blk++) {
        const int buf = blk & 1;
        if (blk + 1 < nblk) load_kv(blk + 1, buf ^ 1);
        cp_async_commit();

#pragma unroll
        for (int sub = 0; sub < BKV / SUB; sub++) {  // SUB-key online-softmax steps (register footprint)
            constexpr int NJ = SUB / 8;                // n-tiles of S
            float s[NJ][4];
#pragma unroll
            for (int j = 0; j < NJ; j++) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
            const uint32_t kb = sK0 + 2 * (buf * C::KV_ELEMS + sub * SUB * LD);
#pragma unroll
            for (int kk = 0; kk < DH / 16; kk++) {
#pragma unroll
                for (int j = 0; j < NJ; j += 2) {
                    uint32_t b[4];
                    int key = 8 * (j + (lane >> 4)) + (lane & 7);
                    int col = kk * 16 + 8 * ((lane >> 3) & 1);
                    ldsm_x4(b, kb + 2 * (key * LD + col));
                    mma16816(s[j], qf[kk], b[0], b[1]);
                    mma16816(s[j + 1], qf[kk], b[2], b[3]);
                }
            }
            const int kbase = blk * BKV + sub * SUB;
            if (kbase >= tile.nkv) break;  // uniform across the CTA
            const bool full = (kbase + SUB <= tile.nkv) && (!CAUSAL || kbase + SUB - 1 <= tile.qloc + warp * 16);
            if (!full) {
#pragma unroll
                for (int j = 0; j < NJ; j++) {
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        int key = kbase + 8 * j + 2 * t4 + (e & 1);
                        int row = (e < 2) ? r0 : r1;
                        bool ok = key < tile.nkv;
                        if (CAUSAL) ok = ok && key <= tile.qloc + row;
                        if (!ok) s[j][e] = -INFINITY;
                    }
                }
            }
            float bm0 = s[0][0], bm1 = s[0][2];
#pragma unroll
            for (int j = 0; j < NJ; j++) {
                bm0 = fmaxf(bm0, fmaxf(s[j][0], s[j][1]));
                bm1 = fmaxf(bm1, fmaxf(s[j][2], s[j][3]));
            }
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 1));
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, 2));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 1));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, 2));
            const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
            const float u0 = nm0 == -INFINITY ? 0.f : -nm0 * sl2;  // exponent offset (scaled)
            const float u1 = nm1 == -INFINITY ? 0.f : -nm1 * sl2;
            const float a0 = ex2(fmaf(m0, sl2, u0)), a1 = ex2(fmaf(m1, sl2, u1));  // m = -inf -> 0
            m0 = nm0;
            m1 = nm1;
#pragma unroll
            for (int j = 0; j < NT; j++) {
                o[j][0] *= a0;
                o[j][1] *= a0;
                o[j][2] *= a1;
                o[j][3] *= a1;
            }
            lacc[0] *= a0;
            lacc[1] *= a0;
            lacc[2] *= a1;
            lacc[3] *= a1;
            uint32_t pf[NJ / 2][4];
#pragma unroll
            for (int j = 0; j < NJ; j++) {
                float p0 = ex2(fmaf(s[j][0], sl2, u0)), p1 = ex2(fmaf(s[j][1], sl2, u0));
                float p2 = ex2(fmaf(s[j][2], sl2, u1)), p3 = ex2(fmaf(s[j][3], sl2, u1));
                pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p0, p1);
                pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p2, p3);
            }
            // O += P V, l += P 1
            const uint32_t vb = sV0 + 2 * (buf * C::KV_ELEMS + sub * SUB * LD);
#pragma unroll
            for (int kk = 0; kk < NJ / 2; kk++) {
                const uint32_t* a = pf[kk];
                int key = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
                for (int j = 0; j < NT; j += 2) {
                    uint32_t b[4];
                    ldsm_x4_t(b, vb + 2 * (key * LD + 8 * (j + (lane >> 4))));
                    mma16816(o[j], a, b[0], b[1]);
                    mma16816(o[j + 1], a, b[2], b[3]);
                }
                mma16816(lacc, a, ONES, ONES);
            }
        }
        cp_async_wait<0>();
        __syncthreads();
    }

    const float i0 = 1.f / lacc[0], i1 = 1.f / lacc[2];
    bf16* O = static_cast<bf16*>(p.out);
#pragma unroll
    for (int j = 0; j < NT; j++) {
        int c = hc + j * 8 + 2 * t4;
        if (r0 < tile.nq)
            *reinterpret_cast<uint32_t*>(O + static_cast<size_t>(tile.q0 + r0) * p.ldo + c) =
                pack_bf16(o[j][0] * i0, o[j][1] * i0);
        if (r1 < tile.nq)
            *reinterpret_cast<uint32_t*>(O + static_cast<size_t>(tile.q0 + r1) * p.ldo + c) =
                pack_bf16(o[j][2] * i1, o[j][3] * i1);
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

template <int DH, bool CAUSAL, int WARPS>
void launch_flash_t(const AttnArgs& a, cudaStream_t s) {
    using C = FlashCfg<DH, WARPS>;
    static std::once_flag once;
    std::call_once(once, [] {
        DCAT_CUDA_CHECK(cudaFuncSetAttribute(k_flash<DH, CAUSAL, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM));
    });
    const dim3 grid(static_cast<unsigned>(a.n_tiles) * static_cast<unsigned>(a.n_heads));
    k_flash<DH, CAUSAL, WARPS><<<grid, WARPS * 32, C::SMEM, s>>>(a);
    DCAT_LAUNCH_CHECK();
}

// context tiles hold 64 queries (causal, 4 warps); crossing tiles 128 (8 warps)
template <int DH>
void launch_flash(const AttnArgs& a, cudaStream_t s) {
    if (a.causal) launch_flash_t<DH, true, 4>(a, s);
    else launch_flash_t<DH, false, 8>(a, s);
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
