// gemm_tc.cu — K3: bf16 tcgen05 GEMM with fused DCAT epilogues (sm_100a).
//
// C[M x N] = A[M x K] . W^T with A = activations (bf16, K contiguous) and
// W = weights stored [N x K] (bf16, K contiguous; the reference's in x out
// matrices transposed once at upload). Replaces every linear_forward ->
// matmul on the scoring path (model.cpp:43-46, mat.hpp:61-76): phi_in /
// phi_out (model.cpp:144-161), Q/K/V/O/FFN of layer_forward (model.cpp:344-396),
// kv_only (dcat.cpp:60-65), cross_forward's projections and cross_tail
// (dcat.cpp:226-229, 77-87), and the ranking head's crossing MLP
// (finetune.cpp:310-315).
//
// One CTA computes one 128 x BN tile:
//   warp 0     TMA producer (A 128x64 and B BNx64 boxes, 128B swizzle)
//   warp 1     single-thread tcgen05.mma issuer, fp32 accumulator in TMEM
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> registers, one row per thread
// STAGES-deep smem ring with full/empty mbarriers; 2 CTAs per SM (BN <= 256)
// so one CTA's epilogue overlaps the other's main loop.
//
// Epilogues (launch.h EpiMode), all row-local so one thread owns a row:
//   EPI_BIAS     act(acc + b) -> bf16, split into up to 3 column segments
//                (QKV -> q, K cache, V cache; FFN1 with GELU)
//   EPI_RESID_LN x = acc + b + resid -> fp32 residual stream, then LayerNorm
//                (eps 1e-5, model.cpp:54-81) of x -> bf16 for the next GEMM
//   EPI_L2NORM   y = (acc + b) / max(||acc + b||, 1e-12) (model.cpp:107-117)
//                -> fp32, optional LN, optional bf16 copy, optional module
//                logits y . mod_w + mod_b (finetune.cpp:317-323)
//   EPI_HEAD     z = gelu(acc + b1); logits = z . w2 + b2 (finetune.cpp:310-315)
#include <cuda.h>

#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace dcat {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;

template <int BN>
struct Cfg {
    static constexpr int STAGES = BN == 64 ? 4 : BN == 128 ? 3 : 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int MMA_N = BN > 256 ? 256 : BN;
    static constexpr int N_HALVES = BN > 256 ? 2 : 1;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 + 256;
    static constexpr int MIN_BLOCKS = BN <= 256 ? 2 : 1;
};

__device__ __forceinline__ void tmem_load32(uint32_t taddr, float* v) {
    uint32_t r[32];
    DCAT_TMEM_LD32(taddr, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_store32(uint32_t taddr, const float* v) {
    uint32_t r[32];
#pragma unroll
    for (int i = 0; i < 32; i++) r[i] = __float_as_uint(v[i]);
    DCAT_TMEM_ST32(taddr, r);
    ptx::tmem_wait_st();
}

// store 32 values (columns c0..c0+31 of a segment-local row) as bf16
__device__ __forceinline__ void store_bf16_32(bf16* dst, const float* v, int ncols) {
    if (ncols >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            uint4 p;
            p.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            p.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            p.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            p.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            reinterpret_cast<uint4*>(dst)[j] = p;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++)
            if (i < ncols) dst[i] = __float2bfloat16_rn(v[i]);
    }
}

__device__ __forceinline__ void load_f32_32(const float* src, float* v, int ncols) {
    if (ncols >= 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            float4 f = __ldg(reinterpret_cast<const float4*>(src) + j);
            v[4 * j] = f.x;
            v[4 * j + 1] = f.y;
            v[4 * j + 2] = f.z;
            v[4 * j + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++) v[i] = i < ncols ? __ldg(src + i) : 0.0f;
    }
}

__device__ __forceinline__ void store_f32_32(float* dst, const float* v, int ncols) {
    if (ncols >= 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 8; j++)
            reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++)
            if (i < ncols) dst[i] = v[i];
    }
}

template <int BN, int MODE>
__device__ __forceinline__ void epilogue(const Epi& e, uint32_t tbase, int row, bool live, int n0, int nvalid) {
    constexpr int CH = (BN + 31) / 32;
    float v[32];
    if constexpr (MODE == EPI_BIAS) {
#pragma unroll 1
        for (int ch = 0; ch < CH; ch++) {
            int c0 = ch * 32;
            if (c0 >= nvalid) break;
            tmem_load32(tbase + c0, v);
            int nc = min(32, nvalid - c0);
            float b[32];
            load_f32_32(e.bias + n0 + c0, b, nc);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                float x = v[i] + b[i];
                v[i] = e.act ? gelu_tanh(x) : x;
            }
            if (!live) continue;
            int g0 = n0 + c0;
            int seg = g0 / e.seg_cols;
            int lc = g0 - seg * e.seg_cols;
            if (lc + nc <= e.seg_cols) {
                bf16* dst = static_cast<bf16*>(e.out[seg]) + static_cast<size_t>(row) * e.out_ld[seg] + lc;
                store_bf16_32(dst, v, nc);
            } else {
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    if (i >= nc) continue;
                    int g = g0 + i, sg = g / e.seg_cols;
                    static_cast<bf16*>(e.out[sg])[static_cast<size_t>(row) * e.out_ld[sg] + (g - sg * e.seg_cols)] =
                        __float2bfloat16_rn(v[i]);
                }
            }
        }
    } else if constexpr (MODE == EPI_HEAD) {
        float lg0 = 0.f, lg1 = 0.f, lg2 = 0.f;
#pragma unroll 1
        for (int ch = 0; ch < CH; ch++) {
            int c0 = ch * 32;
            if (c0 >= nvalid) break;
            tmem_load32(tbase + c0, v);
            int nc = min(32, nvalid - c0);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                if (i >= nc) continue;
                float z = gelu_tanh(v[i] + __ldg(e.bias + c0 + i));
                const float* w = e.w2 + (c0 + i) * 3;
                lg0 += z * __ldg(w);
                lg1 += z * __ldg(w + 1);
                lg2 += z * __ldg(w + 2);
            }
        }
        if (live) {
            e.logits[static_cast<size_t>(row) * 3 + 0] = lg0 + e.b2[0];
            e.logits[static_cast<size_t>(row) * 3 + 1] = lg1 + e.b2[1];
            e.logits[static_cast<size_t>(row) * 3 + 2] = lg2 + e.b2[2];
        }
    } else {
        // full-row modes: nvalid == N == d, n0 == 0
        const float d = static_cast<float>(nvalid);
        float s1 = 0.f;
        bool bad = false;
        if constexpr (MODE == EPI_RESID_LN) {
#pragma unroll 1
            for (int ch = 0; ch < CH; ch++) {
                int c0 = ch * 32;
                if (c0 >= nvalid) break;
                int nc = min(32, nvalid - c0);
                tmem_load32(tbase + c0, v);
                float b[32], r[32];
                load_f32_32(e.bias + c0, b, nc);
                if (live) {
                    load_f32_32(e.resid + static_cast<size_t>(row) * e.ld_x + c0, r, nc);
                } else {
                    for (int i = 0; i < 32; i++) r[i] = 0.f;
                }
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] = v[i] + b[i] + r[i];
                    if (i < nc) {
                        bad |= !isfinite(v[i]);
                        s1 += v[i];
                    }
                }
                if (live) store_f32_32(e.x_out + static_cast<size_t>(row) * e.ld_x + c0, v, nc);
                tmem_store32(tbase + c0, v);
            }
            if (live && bad && e.layer_idx >= 0) atomicMax(&e.st->nonfinite_layer, e.layer_idx + 1);
        } else {  // EPI_L2NORM
            float ss = 0.f;
#pragma unroll 1
            for (int ch = 0; ch < CH; ch++) {
                int c0 = ch * 32;
                if (c0 >= nvalid) break;
                int nc = min(32, nvalid - c0);
                tmem_load32(tbase + c0, v);
                float b[32];
                load_f32_32(e.bias + c0, b, nc);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] += b[i];
                    if (i < nc) ss += v[i] * v[i];
                }
                tmem_store32(tbase + c0, v);
            }
            float nrm = sqrtf(ss);
            float inv = 1.0f / (nrm < 1e-12f ? 1e-12f : nrm);
            float ml0 = 0.f, ml1 = 0.f, ml2 = 0.f;
#pragma unroll 1
            for (int ch = 0; ch < CH; ch++) {
                int c0 = ch * 32;
                if (c0 >= nvalid) break;
                int nc = min(32, nvalid - c0);
                tmem_load32(tbase + c0, v);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] *= inv;
                    if (i < nc) s1 += v[i];
                }
                if (e.mod_w) {
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        if (i >= nc) continue;
                        const float* w = e.mod_w + (c0 + i) * 3;
                        ml0 += v[i] * __ldg(w);
                        ml1 += v[i] * __ldg(w + 1);
                        ml2 += v[i] * __ldg(w + 2);
                    }
                }
                if (live) {
                    if (e.x_out) store_f32_32(e.x_out + static_cast<size_t>(row) * e.ld_x + c0, v, nc);
                    if (e.out2)
                        store_bf16_32(static_cast<bf16*>(e.out2) + static_cast<size_t>(row) * e.out2_ld + c0, v, nc);
                }
                tmem_store32(tbase + c0, v);
            }
            if (live && e.mod_w) {
                e.mlogits[static_cast<size_t>(row) * 3 + 0] = ml0 + e.mod_b[0];
                e.mlogits[static_cast<size_t>(row) * 3 + 1] = ml1 + e.mod_b[1];
                e.mlogits[static_cast<size_t>(row) * 3 + 2] = ml2 + e.mod_b[2];
            }
        }
        if (e.ln_out == nullptr) return;
        float mu = s1 / d;
        float var = 0.f;
        if (e.ln_g) {
#pragma unroll 1
            for (int ch = 0; ch < CH; ch++) {
                int c0 = ch * 32;
                if (c0 >= nvalid) break;
                int nc = min(32, nvalid - c0);
                tmem_load32(tbase + c0, v);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    float c = v[i] - mu;
                    if (i < nc) var += c * c;
                }
            }
        }
        float rs = 1.0f / sqrtf(var / d + 1e-5f);
#pragma unroll 1
        for (int ch = 0; ch < CH; ch++) {
            int c0 = ch * 32;
            if (c0 >= nvalid) break;
            int nc = min(32, nvalid - c0);
            tmem_load32(tbase + c0, v);
            if (e.ln_g) {
                float g[32], bb[32];
                load_f32_32(e.ln_g + c0, g, nc);
                load_f32_32(e.ln_b + c0, bb, nc);
#pragma unroll
                for (int i = 0; i < 32; i++) v[i] = g[i] * ((v[i] - mu) * rs) + bb[i];
            }
            if (live) store_bf16_32(static_cast<bf16*>(e.ln_out) + static_cast<size_t>(row) * e.ln_ld + c0, v, nc);
        }
    }
}

template <int BN, int MODE>
__global__ void __launch_bounds__(256, Cfg<BN>::MIN_BLOCKS)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
              const __grid_constant__ Epi e) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const int nk = (K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < C::STAGES; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tslot, C::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; kb++) {
                int s = kb % C::STAGES;
                if (kb >= C::STAGES) ptx::mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
                ptx::mbar_expect_tx(&full[s], A_BYTES + C::B_BYTES);
                ptx::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
#pragma unroll
                for (int h = 0; h < C::N_HALVES; h++)
                    ptx::tma_load_2d(sB + s * C::B_BYTES + h * C::MMA_N * 128, &tmB, &full[s], kb * BK,
                                     n0 + h * C::MMA_N);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(BM, C::MMA_N);
            for (int kb = 0; kb < nk; kb++) {
                int s = kb % C::STAGES;
                ptx::mbar_wait(&full[s], (kb / C::STAGES) & 1);
                ptx::tc_fence_after();
                uint32_t a_base = ptx::smem_u32(sA + s * A_BYTES);
                uint32_t b_base = ptx::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; k++) {
                    uint64_t ad = ptx::sdesc_sw128(a_base + k * 32);
#pragma unroll
                    for (int h = 0; h < C::N_HALVES; h++) {
                        uint64_t bd = ptx::sdesc_sw128(b_base + h * C::MMA_N * 128 + k * 32);
                        ptx::mma_bf16(tmem + h * C::MMA_N, ad, bd, idesc, (kb | k) != 0);
                    }
                }
                ptx::mma_commit(&empty[s]);
            }
            ptx::mma_commit(tfull);
        }
    } else if (warp >= 4) {
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        const int q = warp & 3;
        const int row = m0 + q * 32 + lane;
        const int nvalid = min(BN, N - n0);
        epilogue<BN, MODE>(e, tmem + (static_cast<uint32_t>(q * 32) << 16), row, row < M, n0, nvalid);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap tmap_bf16(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_outer};
    cuuint32_t es[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_bytes & 15))
        throw CudaError("tensor map: base / row stride must be 16-byte aligned");
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

template <int BN, int MODE>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e, cudaStream_t s) {
    using C = Cfg<BN>;
    static std::once_flag once;
    std::call_once(once, [] {
        DCAT_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_tc<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM));
    });
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
    k_gemm_tc<BN, MODE><<<grid, 256, C::SMEM, s>>>(ta, tb, M, N, K, e);
    DCAT_LAUNCH_CHECK();
}

template <int MODE>
void launch_mode(int BN, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e,
                 cudaStream_t s) {
    switch (BN) {
        case 64: launch<64, MODE>(ta, tb, M, N, K, e, s); break;
        case 128: launch<128, MODE>(ta, tb, M, N, K, e, s); break;
        case 256: launch<256, MODE>(ta, tb, M, N, K, e, s); break;
        case 512:
            if constexpr (MODE == EPI_RESID_LN || MODE == EPI_L2NORM) {
                launch<512, MODE>(ta, tb, M, N, K, e, s);
                break;
            }
            [[fallthrough]];
        default: throw InvalidArg("gemm_tc: unsupported tile width " + std::to_string(BN));
    }
}

}  // namespace

void gemm_tc(const bf16* A, int lda, const bf16* W, int ldw, int M, int N, int K, const Epi& e, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    bool full_row = e.mode == EPI_RESID_LN || e.mode == EPI_L2NORM || e.mode == EPI_HEAD;
    int BN;
    if (full_row) {
        BN = N <= 64 ? 64 : N <= 128 ? 128 : N <= 256 ? 256 : 512;
        if (N > 512 || (e.mode == EPI_HEAD && N > 256)) throw InvalidArg("gemm_tc: full-row epilogue needs N <= 512");
    } else {
        BN = N >= 256 ? 256 : N > 128 ? 256 : N > 64 ? 128 : 64;
    }
    int box_b = BN > 256 ? 256 : BN;
    CUtensorMap ta = tmap_bf16(A, static_cast<uint64_t>(K), static_cast<uint64_t>(M), static_cast<uint64_t>(lda) * 2,
                               BM);
    CUtensorMap tb = tmap_bf16(W, static_cast<uint64_t>(K), static_cast<uint64_t>(N), static_cast<uint64_t>(ldw) * 2,
                               static_cast<uint32_t>(box_b));
    switch (e.mode) {
        case EPI_BIAS: launch_mode<EPI_BIAS>(BN, ta, tb, M, N, K, e, s); break;
        case EPI_RESID_LN: launch_mode<EPI_RESID_LN>(BN, ta, tb, M, N, K, e, s); break;
        case EPI_L2NORM: launch_mode<EPI_L2NORM>(BN, ta, tb, M, N, K, e, s); break;
        case EPI_HEAD: launch_mode<EPI_HEAD>(BN, ta, tb, M, N, K, e, s); break;
        default: throw InvalidArg("gemm_tc: bad epilogue mode");
    }
}

}  // namespace dcat
