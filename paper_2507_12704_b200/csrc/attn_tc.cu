// attn_tc.cu — K5/K6 attention on the 5th-gen tensor cores (sm_100a).
//
// Same math as attention.cu (context: layer_forward's causal softmax attention,
// model.cpp:353-376; crossing: cross_forward's attention over [K_u; k] / [V_u; v],
// dcat.cpp:231-263), restructured for tcgen05:
//   * one CTA per (query tile of <= 128 rows of one unique, head);
//   * S = Q K^T for a chunk of KC keys by one elected thread (tcgen05.mma,
//     M = 128, N = KC, K = head dim) into TMEM;
//   * 4 softmax warps, ONE THREAD PER QUERY ROW: the row's scores come out of
//     TMEM with tcgen05.ld (no shuffles, no per-block barriers), masked (causal /
//     chunk end), max, exp2, row sum, and P (bf16) is written to shared memory in
//     the 128-byte-swizzled K-major layout the next MMA reads;
//   * O_chunk = P V by tcgen05.mma with V^T (keys contiguous) as the K-major B
//     operand — the context pass stores the V cache transposed for this;
//   * online-softmax state (m, l, O) lives in the row's registers across key
//     chunks; the crossing pass starts it at the candidate's own key/value
//     (m = q.k_self, l = 1, O = v_self), so the reference's materialized
//     [K_u; k] copy (dcat.cpp:239-243) never exists.
// Operands arrive by TMA (Q, K chunk, V^T chunk) with mbarrier completion.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace dcat {

namespace {

template <int DH>
struct AttnCfg {
    static constexpr int QROWS = 128;
    static constexpr int KC = DH >= 64 ? 128 : 256;  // keys per chunk (TMEM columns of S)
    static constexpr int ROWB = DH * 2;               // bytes per Q/K row (K-major, K = head dim)
    static constexpr int P_BYTES = QROWS * KC * 2;    // P: KC/64 blocks of [128 x 64] bf16, SW128
    static constexpr int VT_BLOCK = DH * 128;         // V^T block: [DH x 64 keys] bf16, SW128
    static constexpr int VT_BYTES = (KC / 64) * VT_BLOCK;
    static constexpr int K_BYTES = KC * ROWB;
    static constexpr int Q_BYTES = QROWS * ROWB;
    static constexpr int SMEM = P_BYTES + VT_BYTES + K_BYTES + Q_BYTES + 1024 + 128;
    static constexpr uint32_t TMEM_COLS = KC;
    // UMMA layout type / stride of the Q and K tiles (rows of ROWB bytes)
    static constexpr uint64_t LAYOUT = ROWB == 128 ? 2 : ROWB == 64 ? 4 : 6;  // SW128 / SW64 / SW32
    static constexpr uint64_t SBO = 8 * ROWB;
};

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint64_t layout, uint64_t sbo) {
    return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((sbo >> 4) << 32) | (1ull << 46) |
           (layout << 61);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    DCAT_TMEM_LD32(taddr, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(256, 2)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmVt, const AttnArgs p) {
    using C = AttnCfg<DH>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sP = smem;
    uint8_t* sVt = sP + C::P_BYTES;
    uint8_t* sK = sVt + C::VT_BYTES;
    uint8_t* sQ = sK + C::K_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sQ + C::Q_BYTES);
    uint64_t* bar_q = bars + 0;      // Q landed
    uint64_t* bar_kv = bars + 1;     // K + V^T chunk landed
    uint64_t* bar_s = bars + 2;      // S in TMEM (tcgen05.commit)
    uint64_t* bar_p = bars + 3;      // P in smem (4 softmax warps)
    uint64_t* bar_o = bars + 4;      // O_chunk in TMEM, K/V/P smem free (tcgen05.commit)
    uint64_t* bar_oread = bars + 5;  // O_chunk read back (4 softmax warps)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);

    // linear grid, head fastest: the heads of one tile run together and share its K/V lines in L2
    const Tile tile = p.tiles[blockIdx.x / p.n_heads];
    const int h = blockIdx.x % p.n_heads, hc = h * DH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Key chunks start at kv0 rounded down to 8 tokens: the V^T box's inner (token)
    // coordinate must be 16-byte aligned for TMA. S column j of chunk c is key
    // a0 + c*KC + j; the <= 7 leading keys of other users are masked.
    const int a0 = tile.kv0 & ~7;
    const int nchunks = tile.nkv > 0 ? (tile.kv0 + tile.nkv - a0 + C::KC - 1) / C::KC : 0;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmQ);
        ptx::tma_prefetch(&tmK);
        ptx::tma_prefetch(&tmVt);
        ptx::mbar_init(bar_q, 1);
        ptx::mbar_init(bar_kv, 1);
        ptx::mbar_init(bar_s, 1);
        ptx::mbar_init(bar_p, 4);
        ptx::mbar_init(bar_o, 1);
        ptx::mbar_init(bar_oread, 4);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tslot, C::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0 && nchunks > 0) {
            ptx::mbar_expect_tx(bar_q, C::Q_BYTES);
            ptx::tma_load_2d(sQ, &tmQ, bar_q, hc, tile.q0);
            for (int c = 0; c < nchunks; c++) {
                if (c > 0) ptx::mbar_wait(bar_o, (c - 1) & 1);  // previous chunk's K / V^T consumed
                const int k0 = a0 + c * C::KC;
                ptx::mbar_expect_tx(bar_kv, C::K_BYTES + C::VT_BYTES);
                ptx::tma_load_2d(sK, &tmK, bar_kv, hc, k0);
#pragma unroll
                for (int kb = 0; kb < C::KC / 64; kb++)
                    ptx::tma_load_2d(sVt + kb * C::VT_BLOCK, &tmVt, bar_kv, k0 + kb * 64, hc);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && nchunks > 0) {
            constexpr uint32_t idesc_s = ptx::idesc_bf16(128, C::KC);
            constexpr uint32_t idesc_o = ptx::idesc_bf16(128, DH);
            ptx::mbar_wait(bar_q, 0);
            for (int c = 0; c < nchunks; c++) {
                ptx::mbar_wait(bar_kv, c & 1);
                if (c > 0) ptx::mbar_wait(bar_oread, (c - 1) & 1);  // O_chunk (TMEM cols 0..DH) read back
                ptx::tc_fence_after();
                const uint32_t qa = ptx::smem_u32(sQ), ka = ptx::smem_u32(sK);
#pragma unroll
                for (int k = 0; k < DH / 16; k++)
                    ptx::mma_bf16(tmem, sdesc(qa + k * 32, C::LAYOUT, C::SBO), sdesc(ka + k * 32, C::LAYOUT, C::SBO),
                                  idesc_s, k > 0);
                ptx::mma_commit(bar_s);
                ptx::mbar_wait(bar_p, c & 1);  // softmax wrote P (and finished reading S)
                ptx::tc_fence_after();
                const uint32_t pa = ptx::smem_u32(sP), va = ptx::smem_u32(sVt);
#pragma unroll
                for (int kb = 0; kb < C::KC / 64; kb++)
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        ptx::mma_bf16(tmem, sdesc(pa + kb * 16384 + k * 32, 2, 1024),
                                      sdesc(va + kb * C::VT_BLOCK + k * 32, 2, 1024), idesc_o, (kb | k) != 0);
                ptx::mma_commit(bar_o);
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const int r = q * 32 + lane;  // query row of this thread (tile-local)
        const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const float sl2 = p.scale * 1.4426950408889634f;
        const bool live = r < tile.nq;
        const int qrow = tile.q0 + (live ? r : 0);
        float o[DH];
        float m = -INFINITY, l = 0.f;
#pragma unroll
        for (int i = 0; i < DH; i++) o[i] = 0.f;
        if constexpr (!CAUSAL) {
            // self term (the candidate's own key / value, dcat.cpp:242-243)
            const bf16* qp = static_cast<const bf16*>(p.q) + static_cast<size_t>(qrow) * p.ldq + hc;
            const bf16* kp = static_cast<const bf16*>(p.kself) + static_cast<size_t>(qrow) * p.ldself + hc;
            const bf16* vp = static_cast<const bf16*>(p.vself) + static_cast<size_t>(qrow) * p.ldself + hc;
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < DH; i += 8) {
                uint4 a = *reinterpret_cast<const uint4*>(qp + i);
                uint4 b = *reinterpret_cast<const uint4*>(kp + i);
                uint4 v = *reinterpret_cast<const uint4*>(vp + i);
                const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
                const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    float2 x = __bfloat1622float2(a2[j]), y = __bfloat1622float2(b2[j]), z = __bfloat1622float2(v2[j]);
                    s += x.x * y.x + x.y * y.y;
                    o[i + 2 * j] = z.x;
                    o[i + 2 * j + 1] = z.y;
                }
            }
            m = s;
            l = 1.f;
        }
        for (int c = 0; c < nchunks; c++) {
            const int cb = a0 + c * C::KC;                     // first key (token row) of the chunk
            const int lo = max(0, tile.kv0 - cb);               // valid S columns: [lo, lim)
            int lim = min(C::KC, tile.kv0 + tile.nkv - cb);
            if (CAUSAL) lim = min(lim, tile.kv0 + tile.qloc + r + 1 - cb);
            ptx::mbar_wait(bar_s, c & 1);
            ptx::tc_fence_after();
            float v[32];
            float mx = -INFINITY;
#pragma unroll 1
            for (int sc = 0; sc < C::KC / 32; sc++) {
                tmem_ld32(trow + sc * 32, v);
#pragma unroll
                for (int i = 0; i < 32; i++)
                    if (sc * 32 + i >= lo && sc * 32 + i < lim) mx = fmaxf(mx, v[i]);
            }
            const float mn = fmaxf(m, mx);
            const float u = mn == -INFINITY ? 0.f : -mn * sl2;
            const float alpha = ex2f(fmaf(m, sl2, u));  // m = -inf -> 0
            m = mn;
            float sum = 0.f;
#pragma unroll 1
            for (int sc = 0; sc < C::KC / 32; sc++) {
                tmem_ld32(trow + sc * 32, v);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    float e = ex2f(fmaf(v[i], sl2, u));
                    v[i] = (sc * 32 + i >= lo && sc * 32 + i < lim) ? e : 0.f;
                    sum += v[i];
                }
                // P row r, keys [sc*32, sc*32+32): block kb = sc/2, 16-byte chunks (sc&1)*4 .. +3, 128B swizzle
                const uint32_t rowb = ptx::smem_u32(sP) + (sc >> 1) * 16384 + r * 128;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint32_t ch = ((sc & 1) * 4 + j) ^ (r & 7);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowb + ch * 16),
                                 "r"(pack_bf16(v[8 * j], v[8 * j + 1])), "r"(pack_bf16(v[8 * j + 2], v[8 * j + 3])),
                                 "r"(pack_bf16(v[8 * j + 4], v[8 * j + 5])), "r"(pack_bf16(v[8 * j + 6], v[8 * j + 7]))
                                 : "memory");
                }
            }
            l = l * alpha + sum;
#pragma unroll
            for (int i = 0; i < DH; i++) o[i] *= alpha;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic stores) -> MMA (async proxy)
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_p);
            ptx::mbar_wait(bar_o, c & 1);
            ptx::tc_fence_after();
            if constexpr (DH >= 32) {
#pragma unroll
                for (int c32 = 0; c32 < DH / 32; c32++) {
                    tmem_ld32(trow + c32 * 32, v);
#pragma unroll
                    for (int i = 0; i < 32; i++) o[c32 * 32 + i] += v[i];
                }
            } else {
                tmem_ld16(trow, v);
#pragma unroll
                for (int i = 0; i < 16; i++) o[i] += v[i];
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_oread);
        }
        if (live) {
            const float inv = 1.f / l;
            bf16* op = static_cast<bf16*>(p.out) + static_cast<size_t>(qrow) * p.ldo + hc;
#pragma unroll
            for (int i = 0; i < DH; i += 8) {
                uint4 w;
                w.x = pack_bf16(o[i] * inv, o[i + 1] * inv);
                w.y = pack_bf16(o[i + 2] * inv, o[i + 3] * inv);
                w.z = pack_bf16(o[i + 4] * inv, o[i + 5] * inv);
                w.w = pack_bf16(o[i + 6] * inv, o[i + 7] * inv);
                *reinterpret_cast<uint4*>(op + i) = w;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap map2d(const void* base, uint64_t cols, uint64_t rows, uint64_t ld_elems, uint32_t box_c, uint32_t box_r,
                  CUtensorMapSwizzle sw) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld_elems * 2) & 15))
        throw CudaError("attention tensor map: 16-byte alignment");
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
    return m;
}

template <int DH, bool CAUSAL>
void launch_tc(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    using C = AttnCfg<DH>;
    static std::once_flag once;
    std::call_once(once, [] {
        DCAT_CUDA_CHECK(
            cudaFuncSetAttribute(k_attn_tc<DH, CAUSAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    });
    const CUtensorMapSwizzle sw = C::ROWB == 128   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : C::ROWB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                  : CU_TENSOR_MAP_SWIZZLE_32B;
    const int d = a.n_heads * DH;
    CUtensorMap tq = map2d(a.q, static_cast<uint64_t>(d), static_cast<uint64_t>(q_rows), a.ldq, DH, 128, sw);
    CUtensorMap tk = map2d(a.k, static_cast<uint64_t>(d), static_cast<uint64_t>(kv_rows), a.ldkv, DH, C::KC, sw);
    CUtensorMap tv = map2d(a.v, static_cast<uint64_t>(a.ldvt), static_cast<uint64_t>(d), a.ldvt, 64, DH,
                           CU_TENSOR_MAP_SWIZZLE_128B);
    const dim3 grid(static_cast<unsigned>(a.n_tiles) * static_cast<unsigned>(a.n_heads));
    k_attn_tc<DH, CAUSAL><<<grid, 256, C::SMEM, s>>>(tq, tk, tv, a);
    DCAT_LAUNCH_CHECK();
}

}  // namespace

// Attention on tcgen05 (bf16, V cache stored transposed). q_rows / kv_rows: rows of the
// Q and K tensors (tensor-map extents).
void attention_tc(const AttnArgs& a, int64_t q_rows, int64_t kv_rows, cudaStream_t s) {
    if (a.n_tiles <= 0) return;
    if (a.ldvt <= 0) throw InvalidArg("attention_tc needs the transposed V cache");
    switch (a.dh) {
        case 16: a.causal ? launch_tc<16, true>(a, q_rows, kv_rows, s) : launch_tc<16, false>(a, q_rows, kv_rows, s); break;
        case 32: a.causal ? launch_tc<32, true>(a, q_rows, kv_rows, s) : launch_tc<32, false>(a, q_rows, kv_rows, s); break;
        case 64: a.causal ? launch_tc<64, true>(a, q_rows, kv_rows, s) : launch_tc<64, false>(a, q_rows, kv_rows, s); break;
        default: throw InvalidArg("attention_tc: head dim " + std::to_string(a.dh));
    }
}

}  // namespace dcat
