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
// Persistent, warp-specialized, one CTA per SM:
//   warp 0        TMA producer: A 128x64 and B BNx64 boxes (128B swizzle) into
//                 a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1        single-thread tcgen05.mma issuer (M=128, N<=256 per MMA,
//                 K=16), fp32 accumulators in TMEM, double-buffered across
//                 tiles (tmem_full/tmem_empty mbarriers) so tile i+1's main
//                 loop overlaps tile i's epilogue
//   warp 2        TMEM allocator
//   warps 4..     epilogue: CG warps per TMEM lane quadrant, each owning
//                 BN/CG columns of 32 rows; tcgen05.ld 32x32b, math in
//                 registers (one row per thread), global I/O transposed through
//                 per-warp smem so every load/store is row-contiguous
// Epilogues (launch.h EpiMode):
//   EPI_BIAS     act(acc + b) -> bf16, split into up to 3 column segments
//                (QKV -> q, K cache, V cache; FFN1 with GELU)
//   EPI_RESID_LN x = acc + b + resid -> fp32 residual stream; LayerNorm
//                (eps 1e-5, model.cpp:54-81) of x -> bf16 operand of the next GEMM
//   EPI_L2NORM   y = (acc + b) / max(||acc + b||, 1e-12) (model.cpp:107-117)
//                -> fp32, optional LN, optional bf16 copy, optional module
//                logits y . mod_w + mod_b (finetune.cpp:317-323)
//   EPI_HEAD     z = gelu(acc + b1); logits = z . w2 + b2 (finetune.cpp:310-315)
// Row statistics (LN mean/var, l2 norm, head dots) are reduced across the CG
// warps of a quadrant through smem with a per-quadrant named barrier, in a
// fixed order (deterministic).
#include <cuda.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "launch.h"
#include "ptx.cuh"

#ifndef DCAT_FFN_ABLATE
#define DCAT_FFN_ABLATE 0  // product build: nothing ablated
#endif
#ifndef DCAT_FFN_TRACE
#define DCAT_FFN_TRACE 0  // kernel micro-bench only: clock64 event trace of CTA 0 of k_ffn_tc
#endif

namespace dcat {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;
// Epilogue tiles are 32 rows x 32 columns per warp-chunk, moved by TMA:
//   fp32 blocks (residual in, x out): 32 x 128 B rows, 128-byte swizzle (1 KB atoms)
//   bf16 blocks (activations out):    32 x  64 B rows,  64-byte swizzle
// One row per lane; the swizzles make every lane's 16-byte shared access
// bank-conflict free within a quarter warp.
constexpr int F_BYTES = 32 * 32 * 4;
constexpr int H_BYTES = 32 * 32 * 2;

struct EpiMaps {
    CUtensorMap resid, xout, ln, o[3], out2;
};

// RB (resident B): EPI_BIAS with BN = 256 and K <= 256 only. The CTA keeps its 256-column weight
// slice in shared memory for the whole launch (the grid is a multiple of the N-slice count, so
// every tile of a CTA has the same n0) and streams only A: per 128 x 256 tile the TMA moves
// 64 KB instead of 192 KB (a per-SM TMA ingress of ~27 B/clk is the bound of these small-K
// GEMMs; profiles/r01_ffn.md).
// SPL = 2: a full-row epilogue over d = 2 BN columns split across a CTA pair (thread-block cluster
// of 2): each CTA owns BN columns with double-buffered accumulators, and the per-row statistics
// (LayerNorm mean / variance, l2 norm) are summed over the pair through distributed shared memory.
// LK (with SPL = 2, long K): one epilogue warp per lane quadrant, which frees the shared memory for
// a third 48 KB operand stage. The operand stream of a long-K GEMM (d = 512 FFN2: 32 k-blocks per
// tile) needs the depth; a short-K one (o-projection, K = 512) needs the epilogue warps instead.
#ifndef DCAT_BIAS_STAGES4
#define DCAT_BIAS_STAGES4 1
#endif
template <int BN, int MODE, bool RB = false, int SPL = 1, bool LK = false>
struct Cfg {
    static_assert(!RB || (MODE == EPI_BIAS && BN == 256), "resident B: EPI_BIAS, BN = 256");
    static_assert(SPL == 1 || ((MODE == EPI_RESID_LN || MODE == EPI_L2NORM) && BN == 256), "split: full-row, BN 256");
    static constexpr bool FULL = MODE == EPI_RESID_LN || MODE == EPI_L2NORM;
    static constexpr bool SPL1 = SPL == 2 && LK;
    // BIAS4: EPI_BIAS at BN = 256 without resident B (K > 256: the d = 512 QKV and FFN1 GEMMs) trades
    // two epilogue warps per quadrant and the second staging buffer for a fourth 48 KB operand
    // stage: long-seq ctx ffn1 4.17 -> 3.77 ms, qkv 3.00 -> 2.55 ms (the operand stream's depth is
    // what these GEMMs lack, as for the long-K full-row epilogues below)
    static constexpr bool BIAS4 = DCAT_BIAS_STAGES4 && MODE == EPI_BIAS && BN == 256 && !RB;
    static constexpr int CG = BN == 64 ? 2 : (FULL ? ((BN == 512 || SPL1) ? 1 : 2) : (BIAS4 ? 2 : 4));  // epilogue warps per lane quadrant
    static constexpr int EPI_WARPS = 4 * CG;
    static constexpr int EPI_THREADS = 32 * EPI_WARPS;
    static constexpr int THREADS = 128 + EPI_THREADS;
    static constexpr int CPW = BN / CG;  // columns per epilogue warp
    static constexpr int CHUNKS = CPW / 32;
    static constexpr int MMA_N = BN > 256 ? 256 : BN;
    static constexpr int N_HALVES = BN / MMA_N;
    static constexpr int ACC_BUFS = BN <= 256 ? 2 : 1;
    static constexpr int TMEM_COLS = BN * ACC_BUFS < 32 ? 32 : BN * ACC_BUFS;
    static constexpr int STAGES =
        RB ? 4 : BN == 64 ? (FULL ? 4 : 6) : BN == 128 ? (FULL ? 3 : 4) : BN == 256 ? (FULL ? (SPL1 ? 3 : 2) : (BIAS4 ? 4 : 3)) : 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int KB_RES = 4;  // resident B: k-blocks (K <= 256)
    static constexpr int RING = RB ? STAGES * A_BYTES + KB_RES * B_BYTES : STAGES * (A_BYTES + B_BYTES);
    static constexpr int HBUF = (RB || BIAS4) ? 1 : 2;  // bf16 staging buffers per epilogue warp
    static constexpr int EW = FULL ? 2 * F_BYTES + 2 * H_BYTES : (MODE == EPI_BIAS ? HBUF * H_BYTES : 0);  // per warp
    static constexpr int EPI_SMEM = EW * EPI_WARPS;
    static constexpr int RED = MODE == EPI_BIAS ? 0 : 4 * 3 * CG * 32 * 4;  // [quadrant][value][cg][lane]
    // smem params: EPI_BIAS keeps the whole bias (N <= 4096, every N tile of a persistent CTA);
    // full-row / head modes: bias | ln_g | ln_b | mod_w/w2 | mod_b/b2 of one row (d <= 512)
    static constexpr int PARAM_FLOATS = RB ? BN : MODE == EPI_BIAS ? 4096 : (BN == 512 || SPL == 2) ? 3088 : 1600;
    static constexpr int XCH = SPL == 2 ? 2 * 4 * 3 * 32 * 4 + 8 * 8 : 0;  // pair exchange: [set][quadrant][value][lane] + 8 mbarriers
    static constexpr int SMEM = RING + EPI_SMEM + RED + PARAM_FLOATS * 4 + 512 + XCH + 1024;
    static_assert((2 * STAGES + 4 + 2 * EPI_WARPS + 1) * 8 + 4 <= 512, "barrier block");
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sts4(uint32_t a, float x, float y, float z, float w) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ void sts4u(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts1(uint32_t a, float x) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
}
// read-only parameter vector through L1 (16-byte aligned device arrays)
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float lds1(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
// ---- TMA store / bulk groups (per issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(src), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_s(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    while (!ptx::mbar_try_wait(bar, parity)) {
    }
}

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// tanh-form GELU (model.hpp:14-18) with the MUFU tanh: its ~2^-11 relative
// error is below the bf16 rounding of every consumer of this value.
__device__ __forceinline__ float gelu_fast(float x) {
    const float u = x * fmaf(x * x, 0.7978845608028654f * 0.044715f, 0.7978845608028654f);
    const float h = 0.5f * x;
    return fmaf(h, tanh_fast(u), h);
}

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

// 32 consecutive params starting at smem float index p (broadcast reads)
__device__ __forceinline__ void lds32(uint32_t sp, int p, float* out) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        float4 t = lds4(sp + 4u * (p + i));
        out[i] = t.x;
        out[i + 1] = t.y;
        out[i + 2] = t.z;
        out[i + 3] = t.w;
    }
}

// this lane's row of a swizzled fp32 block <-> registers
__device__ __forceinline__ void read_f32_row(uint32_t buf, int lane, float* v) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
        float4 t = lds4(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
        v[4 * j] = t.x;
        v[4 * j + 1] = t.y;
        v[4 * j + 2] = t.z;
        v[4 * j + 3] = t.w;
    }
}
__device__ __forceinline__ void write_f32_row(uint32_t buf, int lane, const float* v) {
#pragma unroll
    for (int j = 0; j < 8; j++)
        sts4(buf + lane * 128 + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
__device__ __forceinline__ void write_bf16_row(uint32_t buf, int lane, const float* v) {
#pragma unroll
    for (int j = 0; j < 4; j++)
        sts4u(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
              pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
              pack_bf16(v[8 * j + 6], v[8 * j + 7]));
}

// transposed: value i of this lane's row -> element (i, lane) of a [32][32] bf16 SW64 block
__device__ __forceinline__ void write_bf16_col(uint32_t buf, int lane, const float* v) {
#pragma unroll
    for (int i = 0; i < 32; i++) {
        const uint32_t a = buf + i * 64 + ((((lane >> 3) ^ ((i >> 1) & 3)) << 4) | ((lane & 7) << 1));
        const __nv_bfloat16 h = __float2bfloat16_rn(v[i]);
        asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(*reinterpret_cast<const unsigned short*>(&h))
                     : "memory");
    }
}

// publish this warp's staged block to the async proxy and TMA-store it (lane 0)
__device__ __forceinline__ void store_block(const CUtensorMap* m, uint32_t buf, int col, int row, int lane) {
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
        tma_store_2d(m, buf, col, row);
        bulk_commit();
    }
}
// before re-filling a staging buffer: wait until at most N of this lane-0's stores still read smem
template <int N>
__device__ __forceinline__ void staging_free(int lane) {
    if (lane == 0) bulk_wait_read<N>();
    __syncwarp();
}

// sum of NV per-row partials over the CG warps of one lane quadrant (fixed order)
template <int CG, int NV, int NVS = 3>  // NVS: values per quadrant the buffer is laid out for
__device__ __forceinline__ void quad_reduce(uint32_t red, float* vals, int cg, int lane, int q) {
    static_assert(NV <= NVS, "reduction buffer layout");
    if constexpr (CG == 1) return;
    const uint32_t r = red + 4u * (q * NVS * CG * 32);
#pragma unroll
    for (int k = 0; k < NV; k++) sts1(r + 4u * ((k * CG + cg) * 32 + lane), vals[k]);
    named_bar(1 + q, CG * 32);
#pragma unroll
    for (int k = 0; k < NV; k++) {
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < CG; c++) s += lds1(r + 4u * ((k * CG + c) * 32 + lane));
        vals[k] = s;
    }
    named_bar(1 + q, CG * 32);
}

// Split full-row epilogue (SPL = 2): the per-row partials of this CTA's columns plus the
// partner CTA's, summed in rank order (both CTAs get bit-identical totals). The cg == 0 warp of
// each quadrant writes its NV partials into the partner's exchange slot over DSMEM and arrives
// (release.cluster) on the partner's mbarrier; every warp of the quadrant then waits for the
// partner's partials in its own slot. Slots and barriers alternate by round (set r & 1, phase
// r >> 1). The quad_reduce barrier that precedes every exchange keeps the partner from reaching
// round r + 2 before every warp here has read round r: its round r + 1 write follows its own
// quadrant's barrier, which follows its reads of round r.
struct PairX {
    uint32_t slots;   // smem: float [2][4][3][32]
    uint32_t bars;    // smem: uint64 [2][4]
    uint32_t round;   // exchanges so far (same count in every epilogue warp of both CTAs)
    uint32_t rank;    // cluster rank of this CTA (0 / 1)
};
template <int NV>
__device__ __forceinline__ void pair_sum(PairX& X, float* vals, int cg, int lane, int q) {
    static_assert(NV <= 3, "exchange slot");
    const uint32_t set = X.round & 1;
    const uint32_t slot = X.slots + 4u * (((set * 4 + q) * 3) * 32 + lane);
    const uint32_t bar = X.bars + 8u * (set * 4 + q);
    if (cg == 0) {
        const uint32_t rs = ptx::mapa(slot, X.rank ^ 1u);
#pragma unroll
        for (int k = 0; k < NV; k++)
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(rs + 128u * k), "f"(vals[k]) : "memory");
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cl(ptx::mapa(bar, X.rank ^ 1u));
    }
    while (!ptx::mbar_try_wait_cl(bar, (X.round >> 1) & 1)) {
    }
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const float other = lds1(slot + 128u * k);
        vals[k] = X.rank == 0 ? vals[k] + other : other + vals[k];
    }
    X.round++;
}

// smem parameter layout (floats): [0, N) bias; then per mode
//   RESID_LN / L2NORM: [P_G, +N) ln_g, [P_B, +N) ln_b; L2NORM: [P_W, +3N) mod_w, [P_W + 3N, +3) mod_b
//   HEAD: [P_W, +3N) w2, [P_W + 3N, +3) b2
struct ParamLayout {
    int npad, P_G, P_B, P_W;
};
__device__ __forceinline__ ParamLayout param_layout(int N) {
    ParamLayout L;
    L.npad = (N + 31) & ~31;
    L.P_G = L.npad;
    L.P_B = 2 * L.npad;
    L.P_W = 3 * L.npad;
    return L;
}

template <int MODE>
__device__ void load_params(const Epi& e, uint32_t sp, int N, int tid, int nthreads) {
    const ParamLayout L = param_layout(N);
    for (int i = tid; i < L.npad; i += nthreads) sts1(sp + 4u * i, i < N ? e.bias[i] : 0.f);
    if constexpr (MODE == EPI_RESID_LN || MODE == EPI_L2NORM) {
        for (int i = tid; i < L.npad; i += nthreads) {
            sts1(sp + 4u * (L.P_G + i), (e.ln_g && i < N) ? e.ln_g[i] : 0.f);
            sts1(sp + 4u * (L.P_B + i), (e.ln_b && i < N) ? e.ln_b[i] : 0.f);
        }
    }
    if constexpr (MODE == EPI_L2NORM || MODE == EPI_HEAD) {
        const float* w = MODE == EPI_HEAD ? e.w2 : e.mod_w;
        const float* b = MODE == EPI_HEAD ? e.b2 : e.mod_b;
        for (int i = tid; i < 3 * L.npad + 3; i += nthreads) {
            float x = 0.f;
            if (w && i < 3 * N) x = w[i];
            if (b && i >= 3 * L.npad) x = b[i - 3 * L.npad];
            sts1(sp + 4u * (L.P_W + i), x);
        }
    }
}

// Per-warp epilogue state kept across tiles (prefetch pipeline of residual blocks).
struct EpiWarp {
    uint32_t ew;       // staging region of this warp
    uint32_t rbar;     // 2 mbarriers for residual blocks
    uint32_t rph;      // phase bits of the two residual barriers
    uint32_t gc;       // residual blocks consumed so far (slot = gc & 1)
    uint32_t hb;       // next bf16 staging buffer (alternates on every bf16 store)
};

template <int BN, int MODE, bool RB, int SPL = 1, bool LK = false>
__device__ __forceinline__ void epilogue_tile(const Epi& e, const EpiMaps& mp, uint32_t tacc, EpiWarp& W,
                                              uint32_t red, uint32_t sp, int q, int cg, int lane, int m0, int n0,
                                              int M, int N, int nvalid, int t, int tiles, int step, PairX& X) {
    using C = Cfg<BN, MODE, RB, SPL, LK>;
    const ParamLayout PL = param_layout(N);
    const int row_base = m0 + q * 32;
    const int row = row_base + lane;
    const bool live = row < M;
    const int col_lo = cg * C::CPW;
    float v[32], p[32];
    if constexpr (MODE == EPI_BIAS) {
        const bool tma_ok = (e.seg_cols % 32) == 0;
#pragma unroll 1
        for (int ch = 0; ch < C::CHUNKS; ch++) {
            const int c = col_lo + ch * 32;
            if (c >= nvalid) break;
            const int nc = min(32, nvalid - c);
            tmem_load32(tacc + c, v);
            lds32(sp, (RB ? 0 : n0) + c, p);  // resident B: the smem bias holds this CTA's slice
            if (e.act) {
#pragma unroll
                for (int i = 0; i < 32; i++) v[i] = gelu_fast(v[i] + p[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; i++) v[i] += p[i];
            }
            const int g0 = n0 + c;
            const int seg = g0 / e.seg_cols;
            if (tma_ok) {
                const uint32_t buf = W.ew + W.hb * H_BYTES;
                if constexpr (C::HBUF == 2) W.hb ^= 1;
                staging_free<C::HBUF - 1>(lane);
                if (e.out_trans[seg]) {  // V^T: this lane's row becomes column `lane` of a [dims][rows] block
                    write_bf16_col(buf, lane, v);
                    store_block(&mp.o[seg], buf, row_base, g0 - seg * e.seg_cols, lane);
                } else {
                    write_bf16_row(buf, lane, v);
                    store_block(&mp.o[seg], buf, g0 - seg * e.seg_cols, row_base, lane);
                }
            } else if (live) {
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    if (i >= nc) continue;
                    int g = g0 + i, sg = g / e.seg_cols;
                    size_t off = e.out_trans[sg] ? static_cast<size_t>(g - sg * e.seg_cols) * e.out_ld[sg] + row
                                                 : static_cast<size_t>(row) * e.out_ld[sg] + (g - sg * e.seg_cols);
                    static_cast<bf16*>(e.out[sg])[off] = __float2bfloat16_rn(v[i]);
                }
            }
        }
    } else if constexpr (MODE == EPI_HEAD) {
        float lg[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
        for (int ch = 0; ch < C::CHUNKS; ch++) {
            const int c = col_lo + ch * 32;
            if (c >= nvalid) break;
            tmem_load32(tacc + c, v);
            lds32(sp, c, p);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                float z = gelu_fast(v[i] + p[i]);  // padded columns: acc 0, bias 0 -> z = 0
                const uint32_t w = sp + 4u * (PL.P_W + (c + i) * 3);
                lg[0] += z * lds1(w);
                lg[1] += z * lds1(w + 4);
                lg[2] += z * lds1(w + 8);
            }
        }
        quad_reduce<C::CG, 3>(red, lg, cg, lane, q);
        if (live && cg == 0) {
            const uint32_t b = sp + 4u * (PL.P_W + 3 * PL.npad);
            float* o = e.logits + static_cast<size_t>(row) * 3;
            o[0] = lg[0] + lds1(b);
            o[1] = lg[1] + lds1(b + 4);
            o[2] = lg[2] + lds1(b + 8);
        }
    } else {
        // full-row modes: n0 == 0, nvalid == N == d (SPL = 2: this CTA's columns [n0, n0 + nvalid) of
        // d = N, row statistics summed over the pair). Columns past d carry zeros (TMA zero fill of
        // W and of the residual, zero params) and are masked out of the centred variance.
        const uint32_t F0 = W.ew, H0 = W.ew + 2 * F_BYTES;
        const float dn = static_cast<float>(SPL == 2 ? N : nvalid);
        const int pc = SPL == 2 ? n0 : 0;  // global column of local column 0 (params, stores)
        int nchunks = 0;
#pragma unroll 1
        for (int ch = 0; ch < C::CHUNKS; ch++)
            if (col_lo + ch * 32 < nvalid) nchunks++;
        float s1[1] = {0.f};
        if constexpr (MODE == EPI_RESID_LN) {
            bool bad = false;
#pragma unroll 1
            for (int ch = 0; ch < nchunks; ch++) {
                const int c = col_lo + ch * 32;
                const int b = W.gc & 1;
                const uint32_t F = F0 + b * F_BYTES;
                mbar_wait_s(W.rbar + 8 * b, (W.rph >> b) & 1);  // residual block (prefetched)
                W.rph ^= 1u << b;
                read_f32_row(F, lane, p);
                tmem_load32(tacc + c, v);
#pragma unroll
                for (int i = 0; i < 32; i++) p[i] += v[i];
                lds32(sp, pc + c, v);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] = p[i] + v[i];  // (acc + resid) + bias
                    bad |= !isfinite(v[i]);
                    s1[0] += v[i];
                }
                __syncwarp();
                write_f32_row(F, lane, v);  // the residual slot becomes the x_out slot
                store_block(&mp.xout, F, pc + c, row_base, lane);
                if (e.ln_g == nullptr && e.ln_out) {
                    const uint32_t H = H0 + W.hb * H_BYTES;
                    W.hb ^= 1;
                    staging_free<1>(lane);
                    write_bf16_row(H, lane, v);
                    store_block(&mp.ln, H, pc + c, row_base, lane);
                }
                tmem_store32(tacc + c, v);
                // refill this slot with the residual block two chunks ahead (maybe in a later tile;
                // full-row GEMMs have one N tile, so tile index -> m0 = tile * BM)
                const int ahead = (ch + 2) / nchunks;
                const int ta = t + ahead * step;
                if (lane == 0 && ta < tiles) {
                    bulk_wait_read<0>();  // the x_out store must have read the slot
                    mbar_expect_tx_s(W.rbar + 8 * b, F_BYTES);
                    tma_load_s(F, &mp.resid, W.rbar + 8 * b, pc + col_lo + ((ch + 2) % nchunks) * 32, ta * BM + q * 32);
                }
                W.gc++;
                __syncwarp();
            }
            if (live && bad && e.layer_idx >= 0) atomicMax(&e.st->nonfinite_layer, e.layer_idx + 1);
        } else {  // EPI_L2NORM
            float ss[1] = {0.f};
#pragma unroll 1
            for (int ch = 0; ch < nchunks; ch++) {
                const int c = col_lo + ch * 32;
                tmem_load32(tacc + c, v);
                lds32(sp, pc + c, p);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] += p[i];
                    ss[0] += v[i] * v[i];
                }
                tmem_store32(tacc + c, v);
            }
            quad_reduce<C::CG, 1>(red, ss, cg, lane, q);
            if constexpr (SPL == 2) pair_sum<1>(X, ss, cg, lane, q);
            const float nrm = sqrtf(ss[0]);
            const float inv = 1.0f / (nrm < 1e-12f ? 1e-12f : nrm);
            float ml[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
            for (int ch = 0; ch < nchunks; ch++) {
                const int c = col_lo + ch * 32;
                tmem_load32(tacc + c, v);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    v[i] *= inv;
                    s1[0] += v[i];
                }
                if (e.mod_w) {
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const uint32_t w = sp + 4u * (PL.P_W + (pc + c + i) * 3);
                        ml[0] += v[i] * lds1(w);
                        ml[1] += v[i] * lds1(w + 4);
                        ml[2] += v[i] * lds1(w + 8);
                    }
                }
                if (e.x_out) {
                    const uint32_t F = F0;
                    staging_free<0>(lane);
                    write_f32_row(F, lane, v);
                    store_block(&mp.xout, F, pc + c, row_base, lane);
                }
                if (e.out2) {
                    const uint32_t H = H0;
                    staging_free<0>(lane);
                    write_bf16_row(H, lane, v);
                    store_block(&mp.out2, H, pc + c, row_base, lane);
                }
                if (e.ln_g == nullptr && e.ln_out) {
                    const uint32_t H = H0 + H_BYTES;
                    staging_free<0>(lane);
                    write_bf16_row(H, lane, v);
                    store_block(&mp.ln, H, pc + c, row_base, lane);
                }
                tmem_store32(tacc + c, v);
            }
            if (e.mod_w) {
                quad_reduce<C::CG, 3>(red, ml, cg, lane, q);
                if constexpr (SPL == 2) pair_sum<3>(X, ml, cg, lane, q);
                if (live && cg == 0 && (SPL == 1 || X.rank == 0)) {
                    const uint32_t b = sp + 4u * (PL.P_W + 3 * PL.npad);
                    float* o = e.mlogits + static_cast<size_t>(row) * 3;
                    o[0] = ml[0] + lds1(b);
                    o[1] = ml[1] + lds1(b + 4);
                    o[2] = ml[2] + lds1(b + 8);
                }
            }
        }
        if (e.ln_out == nullptr || e.ln_g == nullptr) return;
        quad_reduce<C::CG, 1>(red, s1, cg, lane, q);
        if constexpr (SPL == 2) pair_sum<1>(X, s1, cg, lane, q);
        const float mu = s1[0] / dn;
        float var[1] = {0.f};
#pragma unroll 1
        for (int ch = 0; ch < nchunks; ch++) {
            const int c = col_lo + ch * 32;
            const int nc = min(32, nvalid - c);
            tmem_load32(tacc + c, v);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                float t = v[i] - mu;
                var[0] += (i < nc) ? t * t : 0.f;
            }
        }
        quad_reduce<C::CG, 1>(red, var, cg, lane, q);
        if constexpr (SPL == 2) pair_sum<1>(X, var, cg, lane, q);
        const float rs = 1.0f / sqrtf(var[0] / dn + 1e-5f);
#pragma unroll 1
        for (int ch = 0; ch < nchunks; ch++) {
            const int c = col_lo + ch * 32;
            tmem_load32(tacc + c, v);
            lds32(sp, PL.P_G + pc + c, p);
#pragma unroll
            for (int i = 0; i < 32; i++) v[i] = p[i] * ((v[i] - mu) * rs);
            lds32(sp, PL.P_B + pc + c, p);
#pragma unroll
            for (int i = 0; i < 32; i++) v[i] += p[i];
            const uint32_t H = H0 + W.hb * H_BYTES;
            W.hb ^= 1;
            staging_free<1>(lane);
            write_bf16_row(H, lane, v);
            store_block(&mp.ln, H, pc + c, row_base, lane);
        }
    }
}

template <int BN, int MODE, bool RB, int SPL = 1, bool LK = false>
__global__ void __launch_bounds__(Cfg<BN, MODE, RB, SPL, LK>::THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
              const __grid_constant__ Epi e, const __grid_constant__ EpiMaps mp) {
    using C = Cfg<BN, MODE, RB, SPL, LK>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * A_BYTES;
    const uint32_t s_epi = ptx::smem_u32(smem + C::RING);  // 1 KB aligned (RING is a multiple of 1 KB)
    const uint32_t s_red = s_epi + C::EPI_SMEM;
    const uint32_t s_par = s_red + C::RED;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::RING + C::EPI_SMEM + C::RED + C::PARAM_FLOATS * 4);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* rbars = tempty + 2;  // 2 per epilogue warp
    uint64_t* b_full = rbars + 2 * C::EPI_WARPS;  // resident B loaded
    uint32_t* tslot = reinterpret_cast<uint32_t*>(b_full + 1);
    // pair exchange (SPL = 2): slots and mbarriers after the 512-byte barrier block
    const uint32_t s_xch = ptx::smem_u32(full) + 512;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (K + BK - 1) / BK;
    // SPL = 2: a cluster of 2 walks the row tiles, CTA rank r owns columns [r BN, (r + 1) BN)
    const int rank = SPL == 2 ? static_cast<int>(ptx::cluster_rank()) : 0;
    const int cta0 = SPL == 2 ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int step = SPL == 2 ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
    const int num_n = SPL == 2 ? 1 : (N + BN - 1) / BN;
    const int tiles = ((M + BM - 1) / BM) * num_n;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < C::STAGES; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], C::EPI_WARPS);
        }
        for (int b = 0; b < 2 * C::EPI_WARPS; b++) ptx::mbar_init(&rbars[b], 1);
        ptx::mbar_init(b_full, 1);
        if constexpr (SPL == 2)
            for (int b = 0; b < 8; b++)
                ptx::mbar_init(reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(full) + 512 + 3072 + 8 * b), 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tslot, C::TMEM_COLS);
    // resident B: every tile of this CTA has n0 = n_res (grid is a multiple of num_n)
    const int n_res = static_cast<int>(blockIdx.x % num_n) * BN;
    if (warp >= 4) {
        if constexpr (RB) {
            for (int i = threadIdx.x - 128; i < BN; i += C::EPI_THREADS)
                sts1(s_par + 4u * i, n_res + i < N ? e.bias[n_res + i] : 0.f);
        } else {
            load_params<MODE>(e, s_par, N, threadIdx.x - 128, C::EPI_THREADS);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (SPL == 2) ptx::cluster_sync();  // the partner's exchange barriers are initialised
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t it = 0;
            if constexpr (RB) {  // the CTA's weight slice, once
                ptx::mbar_expect_tx(b_full, nk * C::B_BYTES);
                for (int kb = 0; kb < nk; kb++)
#pragma unroll
                    for (int h = 0; h < C::N_HALVES; h++)
                        ptx::tma_load_2d(sB + kb * C::B_BYTES + h * C::MMA_N * 128, &tmB, b_full, kb * BK,
                                         n_res + h * C::MMA_N);
            }
            for (int t = cta0; t < tiles; t += step) {
                const int m0 = (t / num_n) * BM, n0 = SPL == 2 ? rank * BN : (t % num_n) * BN;
                for (int kb = 0; kb < nk; kb++, it++) {
                    const int s = it % C::STAGES;
                    ptx::mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
                    ptx::mbar_expect_tx(&full[s], RB ? A_BYTES : A_BYTES + C::B_BYTES);
                    ptx::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
                    if constexpr (!RB)
#pragma unroll
                        for (int h = 0; h < C::N_HALVES; h++)
                            ptx::tma_load_2d(sB + s * C::B_BYTES + h * C::MMA_N * 128, &tmB, &full[s], kb * BK,
                                             n0 + h * C::MMA_N);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(BM, C::MMA_N);
            uint32_t it = 0, i = 0;
            if constexpr (RB) ptx::mbar_wait(b_full, 0);
            for (int t = cta0; t < tiles; t += step, i++) {
                const int buf = i % C::ACC_BUFS;
                ptx::mbar_wait(&tempty[buf], ((i / C::ACC_BUFS) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t tacc = tmem + buf * BN;
                for (int kb = 0; kb < nk; kb++, it++) {
                    const int s = it % C::STAGES;
                    ptx::mbar_wait(&full[s], (it / C::STAGES) & 1);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(sA + s * A_BYTES);
                    const uint32_t b_base = ptx::smem_u32(sB + (RB ? kb : s) * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; k++) {
                        const uint64_t ad = ptx::sdesc_sw128(a_base + k * 32);
#pragma unroll
                        for (int h = 0; h < C::N_HALVES; h++) {
                            const uint64_t bd = ptx::sdesc_sw128(b_base + h * C::MMA_N * 128 + k * 32);
                            ptx::mma_bf16(tacc + h * C::MMA_N, ad, bd, idesc, (kb | k) != 0);
                        }
                    }
                    ptx::mma_commit(&empty[s]);
                }
                ptx::mma_commit(&tfull[buf]);
            }
        }
    } else if (warp >= 4) {
        const int ew = warp - 4;
        const int q = warp & 3, cg = ew >> 2;
        EpiWarp W;
        PairX X;
        X.slots = s_xch;
        X.bars = s_xch + 3072;
        X.round = 0;
        X.rank = static_cast<uint32_t>(rank);
        W.ew = s_epi + ew * C::EW;
        W.rbar = ptx::smem_u32(&rbars[2 * ew]);
        W.rph = 0;
        W.gc = 0;
        W.hb = 0;
        if constexpr (MODE == EPI_RESID_LN) {
            // prime the residual pipeline: global blocks 0 and 1 of this warp
            int nck = 0;
            for (int ch = 0; ch < C::CHUNKS; ch++)
                if (cg * C::CPW + ch * 32 < (SPL == 2 ? min(BN, N - rank * BN) : N)) nck++;
            if (lane == 0 && nck > 0) {
                for (int g = 0; g < 2; g++) {
                    const int ta = cta0 + (g / nck) * step;
                    if (ta < tiles) {
                        mbar_expect_tx_s(W.rbar + 8 * g, F_BYTES);
                        tma_load_s(W.ew + g * F_BYTES, &mp.resid, W.rbar + 8 * g,
                                   (SPL == 2 ? rank * BN : 0) + cg * C::CPW + (g % nck) * 32, ta * BM + q * 32);
                    }
                }
            }
            __syncwarp();
        }
        uint32_t i = 0;
        for (int t = cta0; t < tiles; t += step, i++) {
            const int buf = i % C::ACC_BUFS;
            const int m0 = (t / num_n) * BM, n0 = SPL == 2 ? rank * BN : (t % num_n) * BN;
            ptx::mbar_wait(&tfull[buf], (i / C::ACC_BUFS) & 1);
            ptx::tc_fence_after();
            const uint32_t tacc = tmem + buf * BN + (static_cast<uint32_t>(q * 32) << 16);
            epilogue_tile<BN, MODE, RB, SPL, LK>(e, mp, tacc, W, s_red, s_par, q, cg, lane, m0, n0, M, N,
                                             min(BN, N - n0), t, tiles, step, X);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
        if (lane == 0) bulk_wait_all();  // smem must stay valid until every store has been read
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (SPL == 2) ptx::cluster_sync();  // no CTA leaves while its partner may still write to it
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------- fused FFN
// The FFN half of layer_forward / cross_tail (model.cpp:386-397, dcat.cpp:80-86):
//   x_out = x + gelu(a . W1 + b1) . W2 + b2 ;  ln_out = LN(x_out) (next LN1) or a plain copy
// as ONE persistent kernel per 128-row tile: the d_ff-wide intermediate stays on the
// SM (TMEM -> GELU -> bf16 smem -> next MMA) instead of a 2 x d_ff x 2 B round trip
// through HBM per row. The A tile (128 x D) is resident in smem for the tile; the
// hidden dimension is walked in 128-column chunks: FFN1 chunk j goes to one of two
// TMEM accumulators (double-buffered), one group of 8 epilogue warps per buffer applies
// bias + GELU and writes the chunk as the next MMA's K-major A operand, FFN2 accumulates all chunks into a
// D-column TMEM accumulator; the residual / LayerNorm epilogue then runs on it.
// TAIL: the layer tail (layer_forward model.cpp:378-397, cross_tail dcat.cpp:80-86) in the same
// kernel: acc2 <- x rows (tcgen05.cp), acc2 += A_o . Wo^T (the attention output projection),
// then x_mid = acc2 + bo stays in acc2 as the FFN residual and LN2(x_mid) is written by the
// epilogue warps straight into the A tile as the FFN1 operand. x_mid and LN2(x_mid) never
// reach HBM: 384 KB less traffic per 128-row tile than the o-projection GEMM + FFN pair.
#ifndef DCAT_FFN_PAIR_N
#define DCAT_FFN_PAIR_N 1
#endif
#ifndef DCAT_FFN_PRODUCERS
#define DCAT_FFN_PRODUCERS 2
#endif
template <int D, int CL, bool TAIL = false>
struct FfnCfg {
    static_assert(!TAIL || (CL == 1 && D >= 128), "fused layer tail: single CTA, D = 128 or 256");
    static constexpr int CH = 128;                        // hidden columns per chunk
    static constexpr int KB1 = D / 64;                    // k-blocks of the A tile
    // Weight blocks this CTA loads: CL = 1 the whole block, CL = 2 its half of the N rows
    // (the pair MMA reads B rows [0, N/2) from the leader and [N/2, N) from the peer).
    static constexpr int NW2 = CL == 1 && D > 128 ? 128 : D;  // N of one FFN2 MMA (single CTA: <= 128)
    static constexpr int W1_ROWS = CH / CL;               // W1 rows (hidden units) per block
    static constexpr int W2_ROWS = CL == 2 ? D / 2 : NW2;  // W2 rows (output dims) per block
    static constexpr int W1_BLK = W1_ROWS * 128;          // one 64-wide k-block, SW128
    static constexpr int W2_BLK = W2_ROWS * 128;
    static constexpr int SLOT = 16384;                    // ring slot
    static constexpr int W1_PER_SLOT = SLOT / W1_BLK;     // k-blocks per slot
    static constexpr int W2_PER_SLOT = SLOT / W2_BLK;
    static constexpr int S1 = KB1 / W1_PER_SLOT;          // slots per FFN1 chunk
    static constexpr int S2 = 2 / W2_PER_SLOT;            // slots per FFN2 chunk (2 k-blocks of 64)
    // single CTA, D = 256: the two 128-row N halves of a W2 / Wo k-block are consecutive ring slots
    // and, with an even ring, always adjacent in smem (every phase pushes an even number of
    // slots), so one N = 256 MMA reads both: the A operand (H / A_o) is read from smem once per
    // 256 output columns instead of twice
    static constexpr bool PAIR_N = CL == 1 && D == 256 && DCAT_FFN_PAIR_N;
#ifndef DCAT_FFN_STAGES256
#define DCAT_FFN_STAGES256 (DCAT_FFN_PAIR_N ? 6 : 5)
#endif
    static constexpr int STAGES = D == 256 ? DCAT_FFN_STAGES256 : 7;  // weight blocks in flight (L2 latency)
    static_assert(!PAIR_N || STAGES % 2 == 0, "paired N halves need an even ring");
    static_assert(!PAIR_N || CH * 64 * 2 == SLOT, "paired FFN1: one [CH x 64] W1 block per slot");
    static constexpr int A_TILE = KB1 * 16384;
    static constexpr int H_BUF = 2 * 16384;  // [128 x CH] bf16 = 2 SW128 k-blocks
    // warp 0: TMA producer + TMEM allocator, warp 1: MMA issuer (leader CTA), warps 2..17:
    // epilogue. Epilogue warp w reads TMEM lane quadrant w % 4; the 4 warps of a quadrant
    // split the columns (GELU: 32 of each 128-column chunk; final: FCOLS of the D outputs).
    static constexpr int EPI_WARPS = 16;
    // NPROD TMA producer warps: warp 0 and NPROD - 1 more after the epilogue warps; producer p
    // issues the ring slots it = p (mod NPROD). One issuing thread's TMA stream caps near 27 B/clk
    // (tools/kbench/l2_stream.cu), below what the weight stream needs (profiles/r02_tail.md)
    static constexpr int NPROD = CL == 1 ? DCAT_FFN_PRODUCERS : 1;
    static constexpr int THREADS = 64 + 32 * EPI_WARPS + 32 * (NPROD - 1);
    // GELU warps per chunk: the epilogue warps form two groups that take alternate chunks
    // (acc1 buffer 0 / 1), 64 columns per warp, so one group's barrier / TMEM-load latency
    // overlaps the other group's math (388 -> 377 us in tools/kbench against all 16 warps on
    // every chunk).
    static constexpr int GELU_WARPS = EPI_WARPS / 2;
    static constexpr int CGF = D >= 128 ? 4 : 2;  // final-epilogue warps per quadrant
    static constexpr int FCOLS = D / CGF;         // final-epilogue columns per warp
    static constexpr int STG = 4096;              // final-epilogue staging per warp (in the H buffers)
    // The epilogue parameters (b1 | b2 | ln_g | ln_b [| bo | ln2_g | ln2_b]) are read through L1
    // (__ldg, every lane of a warp the same address), not staged in shared memory: the 10 KB go
    // to the weight ring instead. Row statistics: one value per row, [quadrant][cg][lane].
    static constexpr int RED = 4 * 1 * CGF * 32 * 4;
    // no alignment slack: the dynamic shared window starts 1 KB-aligned (checked in the kernel)
    static constexpr int SMEM = A_TILE + 2 * H_BUF + STAGES * SLOT + RED + 512;
    static_assert(EPI_WARPS * STG <= 2 * H_BUF, "final-epilogue staging lives in the H buffers");
    static_assert(FCOLS == 32 || FCOLS == 64, "final epilogue works on one or two 32-column blocks");
    static_assert(CL == 1 || D >= 128, "CTA-pair FFN needs D >= 128");
    static_assert(W1_PER_SLOT * W1_BLK == SLOT && W2_PER_SLOT * W2_BLK == SLOT && S1 >= 1 && S2 >= 1,
                  "slot holds whole weight blocks");
};

#if DCAT_FFN_TRACE
// clock64 timeline of CTAs 0 and 1, first 4 tiles: one recording thread per role (producer,
// MMA issuer, epilogue warps 0 and 15), each with its own array and a register-free shared
// cursor, so an event costs a shared increment and a fire-and-forget global store.
constexpr int FFN_TR_ROLES = 8, FFN_TR_CAP = 1024;
__device__ unsigned long long g_ffn_trace[FFN_TR_ROLES * FFN_TR_CAP];
__device__ unsigned int g_ffn_trace_n[FFN_TR_ROLES];
#define FFN_EV(code, j)                                                                                   \
    do {                                                                                                  \
        if (blockIdx.x < 2 && i < 4) {                                                                    \
            const int r_ = static_cast<int>(blockIdx.x) * 4 + (warp < 2 ? warp : (warp == 2 ? 2 : 3));    \
            const unsigned k_ = s_tr_n[r_ & 3]++;                                                         \
            if (k_ < FFN_TR_CAP) {                                                                        \
                g_ffn_trace[r_ * FFN_TR_CAP + k_] = (static_cast<unsigned long long>(clock64()) << 16) | \
                                                    (static_cast<unsigned>(code) << 8) |                  \
                                                    static_cast<unsigned>(j);                             \
                g_ffn_trace_n[r_] = k_ + 1;                                                               \
            }                                                                                             \
        }                                                                                                 \
    } while (0)
#else
#define FFN_EV(code, j) \
    do {                \
    } while (0)
#endif

// CL = 1: one CTA per 128-row tile. CL = 2: a CTA pair (cluster of 2 on one TPC) per
// 256-row tile; the leader issues M = 256 tcgen05.mma.cta_group::2 reading each CTA's
// own A / H rows and its half of every weight block, so each SM streams half the
// weight bytes per row. Every barrier the MMA issuer waits on lives in the leader
// (peer producers / epilogue warps arrive remotely); MMA completions are multicast to
// the same barrier in both CTAs.
template <int D, int CL, bool TAIL>
__global__ void __launch_bounds__(FfnCfg<D, CL, TAIL>::THREADS, 1)
    k_ffn_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW1,
             const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmWo, int M, int F,
             const __grid_constant__ Epi e, const __grid_constant__ EpiMaps mp) {
    using C = FfnCfg<D, CL, TAIL>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (ptx::smem_u32(smem_raw) & 1023) __trap();  // SW128 operands need a 1 KB-aligned window
    uint8_t* smem = smem_raw;
    uint8_t* sA = smem;
    uint8_t* sH = sA + C::A_TILE;
    uint8_t* ring = sH + 2 * C::H_BUF;
    const uint32_t s_red = ptx::smem_u32(ring + C::STAGES * C::SLOT);
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + C::STAGES * C::SLOT + C::RED);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 1;
    uint64_t* full = bars + 2;
    uint64_t* empty = full + C::STAGES;
    uint64_t* acc1_full = empty + C::STAGES;
    uint64_t* acc1_empty = acc1_full + 2;
    uint64_t* h_full = acc1_empty + 2;
    uint64_t* h_empty = h_full + 2;
    uint64_t* acc2_full = h_empty + 2;
    uint64_t* acc2_empty = acc2_full + 1;
    uint64_t* rbar = acc2_empty + 1;  // residual block loads, one per epilogue warp
    uint64_t* o_full = rbar + C::EPI_WARPS;  // TAIL: residual + A_o . Wo^T complete in acc2
    uint64_t* a2_full = o_full + 1;          // TAIL: LN2 rows in the A tile, x_mid in acc2
    uint32_t* tslot = reinterpret_cast<uint32_t*>(a2_full + 1);

#if DCAT_FFN_TRACE
    // trace cursors in the spare tail of the 512-byte barrier block (no static shared memory: the
    // kernel's dynamic budget is within 512 bytes of the limit)
    unsigned* s_tr_n = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(bars) + 512 - 16);
    if (threadIdx.x < 4) s_tr_n[threadIdx.x] = 0;
#endif
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CL == 2 ? ptx::cluster_rank() : 0;
    const int units = ((M + 127) / 128 + CL - 1) / CL;  // row tiles of 128 * CL rows
    const int unit0 = blockIdx.x / CL, ustride = gridDim.x / CL;
    const int nch = F / C::CH;
    // MMA issue order F1_0 .. F1_{LA-1}, then F1_j, F2_{j-LA}: FFN1 runs LA chunks ahead, so a
    // chunk's GELU overlaps ~2 LA chunk-MMAs and F1_j only needs GELU_{j-2}'s TMEM read.
    constexpr int LA = 2;
    // Hidden chunks in ascending order for every tile: a row's FP32 accumulation order never
    // depends on which CTA processes it (bit-exact under batch permutation).
    auto chunk = [](int j) { return j; };

    // barrier plumbing: arrivals that the MMA issuer waits on go to the leader CTA
    auto lead = [&](uint64_t* b) -> uint32_t {
        if constexpr (CL == 2) return ptx::mapa(ptx::smem_u32(b), 0);
        else return ptx::smem_u32(b);
    };
    auto arrive_lead = [&](uint64_t* b) {
        if constexpr (CL == 2) ptx::mbar_arrive_cl(lead(b));
        else mbar_arrive(b);
    };
    auto commit = [&](uint64_t* b) {
        if constexpr (CL == 2) ptx::mma_commit_pair(b);
        else ptx::mma_commit(b);
    };
    auto wait_lead = [&](uint64_t* b, uint32_t parity) {  // leader-side wait on remote arrivals
        if constexpr (CL == 2) ptx::mbar_wait_cl(b, parity);
        else ptx::mbar_wait(b, parity);
    };

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmW1);
        ptx::tma_prefetch(&tmW2);
        ptx::mbar_init(a_full, CL);  // one expect_tx arrival per CTA
        ptx::mbar_init(a_empty, 1);
        for (int s = 0; s < C::STAGES; s++) {
            ptx::mbar_init(&full[s], CL);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            ptx::mbar_init(&acc1_full[b], 1);
            ptx::mbar_init(&acc1_empty[b], CL * C::GELU_WARPS);
            ptx::mbar_init(&h_full[b], CL * C::GELU_WARPS);
            ptx::mbar_init(&h_empty[b], 1);
        }
        ptx::mbar_init(acc2_full, 1);
        ptx::mbar_init(acc2_empty, CL * 4 * C::CGF);
        ptx::mbar_init(o_full, 1);
        ptx::mbar_init(a2_full, 4 * C::CGF);
        for (int w = 0; w < C::EPI_WARPS; w++) ptx::mbar_init(&rbar[w], 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) {
        if constexpr (CL == 2) ptx::tmem_alloc_pair(tslot, 512);
        else ptx::tmem_alloc(tslot, 512);
    }
    ptx::tc_fence_before();
    if constexpr (CL == 2) ptx::cluster_sync();  // peer barriers initialised before any remote arrival
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t T_ACC2 = tmem, T_ACC1 = tmem + 256;

    const int prod_warp0 = 2 + C::EPI_WARPS;  // producers 1 .. NPROD - 1, after the epilogue warps
    if (warp == 0 || warp >= prod_warp0) {
        if (lane == 0) {
            // every producer walks the same slot sequence; producer `me` issues the slots
            // it = me (mod NPROD), warp 0 also the A tiles
            const uint32_t me = warp == 0 ? 0u : static_cast<uint32_t>(warp - prod_warp0 + 1);
            uint32_t it = 0, i = 0;
            // one ring slot: `n` weight blocks of `blk` bytes at k offsets k0 + 64 w, rows r0
            auto push = [&](const CUtensorMap* map, int k0, int r0, int n, int blk) {
                if (C::NPROD > 1 && it % C::NPROD != me) {
                    it++;
                    return;
                }
                const int s = it % C::STAGES;
                ptx::mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
                FFN_EV(11, it & 255);
                const uint32_t dst = ptx::smem_u32(ring + s * C::SLOT);
#if DCAT_FFN_ABLATE & 4  // kernel micro-bench only: weights loaded once, ring recycled without TMA
                if (it >= static_cast<uint32_t>(C::STAGES)) {
                    if constexpr (CL == 2) ptx::mbar_arrive_cl(lead(&full[s]));
                    else mbar_arrive(&full[s]);
                    it++;
                    return;
                }
#endif
                if constexpr (CL == 2) {
                    ptx::mbar_expect_tx_cl(lead(&full[s]), C::SLOT);
                    for (int w = 0; w < n; w++) ptx::tma_load_2d_pair(dst + w * blk, map, lead(&full[s]), k0 + 64 * w, r0);
                } else {
                    ptx::mbar_expect_tx(&full[s], C::SLOT);
                    for (int w = 0; w < n; w++) ptx::tma_load_2d(ring + s * C::SLOT + w * blk, map, &full[s], k0 + 64 * w, r0);
                }
                it++;
            };
            for (int u = unit0; u < units; u += ustride, i++) {
                const int t = u * CL + static_cast<int>(rank);  // this CTA's 128-row tile
                if (me == 0) {
                ptx::mbar_wait(a_empty, (i & 1) ^ 1);
                FFN_EV(10, 0);
                if constexpr (CL == 2) {
                    ptx::mbar_expect_tx_cl(lead(a_full), C::A_TILE);
                    for (int kb = 0; kb < C::KB1; kb++)
                        ptx::tma_load_2d_pair(ptx::smem_u32(sA + kb * 16384), &tmA, lead(a_full), kb * 64, t * 128);
                } else {
                    ptx::mbar_expect_tx(a_full, C::A_TILE);
                    for (int kb = 0; kb < C::KB1; kb++) ptx::tma_load_2d(sA + kb * 16384, &tmA, a_full, kb * 64, t * 128);
                }
                }
                // No L2 prefetch of the next tile's rows: issued a tile (~36 us, ~230 MB of DRAM
                // traffic) ahead, it is evicted from the 126 MB L2 before use (ncu: +190-250 MB of
                // DRAM reads per context launch, and 368 vs 378 us in tools/kbench without it).
                if constexpr (TAIL) {  // x rows (acc2's initial value), then Wo^T [NW2 x 64] blocks
                    for (int cc = 0; cc < D; cc += 32) push(&mp.resid, cc, t * 128, 1, C::SLOT);
                    for (int kb = 0; kb < C::KB1; kb++)
                        for (int nh = 0; nh < D / C::NW2; nh++) push(&tmWo, kb * 64, nh * C::NW2, 1, C::SLOT);
                }
                for (int j = 0; j < nch + LA; j++) {  // same order as the MMA issuer
                    if (C::PAIR_N && j < nch && (j & 1) == 0) {  // W1 blocks of chunks j, j + 1 per k-block
                        for (int kb = 0; kb < C::KB1; kb++) {
                            push(&tmW1, kb * 64, chunk(j) * C::CH, 1, C::SLOT);
                            push(&tmW1, kb * 64, chunk(j + 1) * C::CH, 1, C::SLOT);
                        }
                    } else if (!C::PAIR_N && j < nch)
                        for (int p = 0; p < C::S1; p++)
                            push(&tmW1, p * C::W1_PER_SLOT * 64, chunk(j) * C::CH + static_cast<int>(rank) * C::W1_ROWS,
                                 C::W1_PER_SLOT, C::W1_BLK);
                    if (j >= LA) {
                        const int jj = j - LA;
                        if (!TAIL && jj == 0)  // residual [128 x 32] fp32 blocks: the initial value of acc2
                            for (int cc = 0; cc < D; cc += 32) push(&mp.resid, cc, t * 128, 1, C::SLOT);
                        if constexpr (CL == 1 && C::NW2 < D) {  // single CTA, D = 256: N halves per slot
                            for (int kb2 = 0; kb2 < 2; kb2++)
                                for (int nh = 0; nh < D / C::NW2; nh++)
                                    push(&tmW2, chunk(jj) * C::CH + kb2 * 64, nh * C::NW2, 1, C::SLOT);
                        } else {
                            for (int p = 0; p < C::S2; p++)
                                push(&tmW2, chunk(jj) * C::CH + p * C::W2_PER_SLOT * 64,
                                     static_cast<int>(rank) * C::W2_ROWS, C::W2_PER_SLOT, C::W2_BLK);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc1 = ptx::idesc_bf16(128 * CL, C::CH);
            constexpr uint32_t idesc2 = ptx::idesc_bf16(128 * CL, C::NW2);
            constexpr uint32_t idesc_n2 = ptx::idesc_bf16(128, D);  // PAIR_N: N = 256 over two slots
            constexpr uint32_t idesc_f1p = ptx::idesc_bf16(128, 2 * C::CH);  // PAIR_N: two FFN1 chunks
            uint32_t it = 0, c1 = 0, c2 = 0, i = 0;
            const uint32_t a_base = ptx::smem_u32(sA), h_base = ptx::smem_u32(sH), r_base = ptx::smem_u32(ring);
            auto mma = [&](uint32_t d, uint32_t a, uint32_t b, uint32_t idesc, uint32_t acc) {
#if DCAT_FFN_ABLATE & 8  // kernel micro-bench only: no MMAs issued
                return;
#endif
                if constexpr (CL == 2) ptx::mma_bf16_pair(d, ptx::sdesc_sw128(a), ptx::sdesc_sw128(b), idesc, acc);
                else ptx::mma_bf16(d, ptx::sdesc_sw128(a), ptx::sdesc_sw128(b), idesc, acc);
            };
            auto next_slot = [&]() -> uint32_t {
                const int s = it % C::STAGES;
                wait_lead(&full[s], (it / C::STAGES) & 1);
                FFN_EV(12, it & 255);
                ptx::tc_fence_after();
                return static_cast<uint32_t>(s);
            };
            // acc2 <- residual rows: [128 x 32] fp32 ring slots copied into TMEM (tcgen05.cp is ordered
            // before the MMAs that accumulate onto it)
            // TAIL: x rows + A_o . Wo^T accumulate in the acc1 columns (free once the previous
            // tile's last two GELU chunks are read), so this phase overlaps the previous tile's
            // final epilogue on acc2; the LN2 epilogue then moves x_mid into acc2.
            auto resid_to = [&](uint32_t t_dst) {
                if constexpr (!TAIL) wait_lead(acc2_empty, (i & 1) ^ 1);
                ptx::tc_fence_after();
                for (int cc = 0; cc < D; cc += 32, it++) {
                    const uint32_t s = next_slot();
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint64_t sd = ptx::sdesc_sw128(r_base + s * C::SLOT + k * 32);
                        if constexpr (CL == 2) ptx::tmem_cp_128x256b_pair(t_dst + cc + 8 * k, sd);
                        else ptx::tmem_cp_128x256b(t_dst + cc + 8 * k, sd);
                    }
                    commit(&empty[s]);
                }
            };
            auto resid_to_acc2 = [&]() { resid_to(T_ACC2); };
            for (int u = unit0; u < units; u += ustride, i++) {
                wait_lead(a_full, i & 1);
                ptx::tc_fence_after();
                if constexpr (TAIL) {  // acc1 cols = x + A_o . Wo^T, then the epilogue's x_mid / LN2 hand-off
                    // both acc1 buffers free: the waits the next two FFN1 chunks would do
                    wait_lead(&acc1_empty[c1 & 1], ((c1 >> 1) & 1) ^ 1);
                    wait_lead(&acc1_empty[(c1 + 1) & 1], (((c1 + 1) >> 1) & 1) ^ 1);
                    resid_to(T_ACC1);
                    ptx::tc_fence_after();
                    for (int kb = 0; kb < C::KB1; kb++) {
                        if constexpr (C::PAIR_N) {  // both N halves (adjacent slots) in one N = 256 MMA
                            const uint32_t s0 = next_slot();
                            it++;
                            const uint32_t s1 = next_slot();
                            it++;
#pragma unroll
                            for (int k = 0; k < 4; k++)
                                mma(T_ACC1, a_base + kb * 16384 + k * 32, r_base + s0 * C::SLOT + k * 32, idesc_n2, 1u);
                            commit(&empty[s0]);
                            commit(&empty[s1]);
                        } else {
                            for (int nh = 0; nh < D / C::NW2; nh++, it++) {
                                const uint32_t s = next_slot();
#pragma unroll
                                for (int k = 0; k < 4; k++)
                                    mma(T_ACC1 + nh * C::NW2, a_base + kb * 16384 + k * 32,
                                        r_base + s * C::SLOT + k * 32, idesc2, 1u);
                                commit(&empty[s]);
                            }
                        }
                    }
                    commit(o_full);
                    FFN_EV(13, 0);
                    ptx::mbar_wait(a2_full, i & 1);  // x_mid in acc2, LN2 rows in the A tile, acc1 free
                    FFN_EV(14, 0);
                    ptx::tc_fence_after();
                }
                for (int j = 0; j < nch + LA; j++) {
                    if (C::PAIR_N && j < nch && (j & 1) == 0) {
                        // FFN1 of chunks j, j + 1 as N = 256 MMAs into both acc1 buffers: per k-block
                        // the two chunks' W1 blocks sit in adjacent slots (A read once per 256 columns)
                        if (!TAIL || j >= 2) {
                            wait_lead(&acc1_empty[c1 & 1], ((c1 >> 1) & 1) ^ 1);
                            wait_lead(&acc1_empty[(c1 + 1) & 1], (((c1 + 1) >> 1) & 1) ^ 1);
                        }
                        FFN_EV(1, j);
                        ptx::tc_fence_after();
                        for (int kb = 0; kb < C::KB1; kb++) {
                            const uint32_t s0 = next_slot();
                            it++;
                            const uint32_t s1 = next_slot();
                            it++;
#pragma unroll
                            for (int k = 0; k < 4; k++)
                                mma(T_ACC1, a_base + kb * 16384 + k * 32, r_base + s0 * C::SLOT + k * 32, idesc_f1p,
                                    (kb | k) != 0);
                            commit(&empty[s0]);
                            commit(&empty[s1]);
                        }
                        commit(&acc1_full[c1 & 1]);
                        commit(&acc1_full[(c1 + 1) & 1]);
                        c1 += 2;
                        if (j + 1 == nch - 1) commit(a_empty);  // the A tiles are free once these complete
                    } else if (!C::PAIR_N && j < nch) {  // FFN1 chunk j -> acc1[b]
                        const int b = c1 & 1;
                        if (!TAIL || j >= 2) wait_lead(&acc1_empty[b], ((c1 >> 1) & 1) ^ 1);
                        FFN_EV(1, j);
                        ptx::tc_fence_after();
                        for (int p = 0; p < C::S1; p++, it++) {
                            const uint32_t s = next_slot();
                            for (int w = 0; w < C::W1_PER_SLOT; w++) {
                                const int kb = p * C::W1_PER_SLOT + w;
#pragma unroll
                                for (int k = 0; k < 4; k++)
                                    mma(T_ACC1 + b * C::CH, a_base + kb * 16384 + k * 32,
                                        r_base + s * C::SLOT + w * C::W1_BLK + k * 32, idesc1, (kb | k) != 0);
                            }
                            commit(&empty[s]);
                        }
                        commit(&acc1_full[b]);
                        c1++;
                        if (j == nch - 1) commit(a_empty);  // the A tiles are free once these complete
                    }
                    if (j >= LA) {  // FFN2 of chunk jj = j - LA: acc2 += H . W2_chunk
                        const int jj = j - LA;
                        const int hb = c2 & 1;
                        wait_lead(&h_full[hb], (c2 >> 1) & 1);
                        FFN_EV(2, jj);
                        if (!TAIL && jj == 0) resid_to_acc2();
                        ptx::tc_fence_after();
                        if constexpr (C::PAIR_N) {
                            for (int kb2 = 0; kb2 < 2; kb2++) {
                                const uint32_t s0 = next_slot();
                                it++;
                                const uint32_t s1 = next_slot();
                                it++;
#pragma unroll
                                for (int k = 0; k < 4; k++)
                                    mma(T_ACC2, h_base + hb * C::H_BUF + kb2 * 16384 + k * 32,
                                        r_base + s0 * C::SLOT + k * 32, idesc_n2, 1u);
                                commit(&empty[s0]);
                                commit(&empty[s1]);
                            }
                        } else if constexpr (CL == 1 && C::NW2 < D) {
                            for (int kb2 = 0; kb2 < 2; kb2++)
                                for (int nh = 0; nh < D / C::NW2; nh++, it++) {
                                    const uint32_t s = next_slot();
#pragma unroll
                                    for (int k = 0; k < 4; k++)
                                        mma(T_ACC2 + nh * C::NW2, h_base + hb * C::H_BUF + kb2 * 16384 + k * 32,
                                            r_base + s * C::SLOT + k * 32, idesc2, 1u);
                                    commit(&empty[s]);
                                }
                        } else {
                            for (int p = 0; p < C::S2; p++, it++) {
                                const uint32_t s = next_slot();
                                for (int w = 0; w < C::W2_PER_SLOT; w++) {
                                    const int kb2 = p * C::W2_PER_SLOT + w;
#pragma unroll
                                    for (int k = 0; k < 4; k++)
                                        mma(T_ACC2, h_base + hb * C::H_BUF + kb2 * 16384 + k * 32,
                                            r_base + s * C::SLOT + w * C::W2_BLK + k * 32, idesc2, 1u);
                                }
                                commit(&empty[s]);
                            }
                        }
                        commit(&h_empty[hb]);
                        c2++;
                    }
                }
                commit(acc2_full);
            }
        }
    } else {
        const int ew = warp - 2, q = warp & 3, cg = ew >> 2;
        const int r = q * 32 + lane;  // tile row of this thread
        const uint32_t h_base = ptx::smem_u32(sH);
        const uint32_t S0 = h_base + ew * C::STG;  // final-epilogue staging (in the H buffers)
        const bool fin = cg < C::CGF;              // this warp takes part in the final epilogue
        const int c0 = cg * C::FCOLS;
        uint32_t c1 = 0, i = 0;
        for (int u = unit0; u < units; u += ustride, i++) {
            const int t = u * CL + static_cast<int>(rank);
            const int m0 = t * 128, row_base = m0 + q * 32, row = row_base + lane;
            if constexpr (TAIL) {
                // ---- x_mid = acc2 + bo (acc2 = x + A_o . Wo^T) back into acc2 as the FFN residual;
                // LN2(x_mid) (model.cpp:386) -> row r of the A tile, bf16, SW128 K-major
                const bool live = row < M;
                const uint32_t tacc = T_ACC2 + (static_cast<uint32_t>(q * 32) << 16) + c0;
                const uint32_t tsrc = T_ACC1 + (static_cast<uint32_t>(q * 32) << 16) + c0;  // x + A_o . Wo^T
                const uint32_t a_row = ptx::smem_u32(sA) + r * 128;
                float v[32];
                float s1[1] = {0.f};
                bool bad = false;
                ptx::mbar_wait(o_full, i & 1);
                ptx::tc_fence_after();
                if (lane == 0 && ew == 0) FFN_EV(8, 0);
#pragma unroll 1
                for (int h = 0; h < C::FCOLS; h += 32) {
                    tmem_load32(tsrc + h, v);
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const float4 bb = ldg4(e.o_bias + c0 + h + 4 * j);
                        float* w = v + 4 * j;
                        w[0] += bb.x;
                        w[1] += bb.y;
                        w[2] += bb.z;
                        w[3] += bb.w;
                    }
#pragma unroll
                    for (int k = 0; k < 32; k++) {
                        bad |= !isfinite(v[k]);
                        s1[0] += v[k];
                    }
                    tmem_store32(tacc + h, v);
                }
                if (bad && live && e.layer_idx >= 0) atomicMax(&e.st->nonfinite_layer, e.layer_idx + 1);
                quad_reduce<C::CGF, 1, 1>(s_red, s1, cg, lane, q);
                const float dn = static_cast<float>(D);
                const float mu = s1[0] / dn;
                float var[1] = {0.f};
#pragma unroll 1
                for (int h = 0; h < C::FCOLS; h += 32) {
                    tmem_load32(tacc + h, v);
#pragma unroll
                    for (int k = 0; k < 32; k++) {
                        const float d0 = v[k] - mu;
                        var[0] += d0 * d0;
                    }
                }
                quad_reduce<C::CGF, 1, 1>(s_red, var, cg, lane, q);
                const float rs = 1.0f / sqrtf(var[0] / dn + 1e-5f);
#pragma unroll 1
                for (int h = 0; h < C::FCOLS; h += 32) {
                    tmem_load32(tacc + h, v);
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const float4 gg = ldg4(e.ln2_g + c0 + h + 4 * j);
                        const float4 bb = ldg4(e.ln2_b + c0 + h + 4 * j);
                        float* w = v + 4 * j;
                        w[0] = gg.x * ((w[0] - mu) * rs) + bb.x;
                        w[1] = gg.y * ((w[1] - mu) * rs) + bb.y;
                        w[2] = gg.z * ((w[2] - mu) * rs) + bb.z;
                        w[3] = gg.w * ((w[3] - mu) * rs) + bb.w;
                    }
                    // columns col .. col + 31: k-block col / 64, 16-byte chunks (col % 64) / 8 + k
                    const int col = c0 + h;
                    const uint32_t rowa = a_row + (col >> 6) * 16384;
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        sts4u(rowa + (((((col & 63) >> 3) + k) ^ (r & 7)) << 4), pack_bf16(v[8 * k], v[8 * k + 1]),
                              pack_bf16(v[8 * k + 2], v[8 * k + 3]), pack_bf16(v[8 * k + 4], v[8 * k + 5]),
                              pack_bf16(v[8 * k + 6], v[8 * k + 7]));
                }
                fence_async_smem();  // the A tile is read by the FFN1 MMAs (async proxy)
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(a2_full);
                if (lane == 0 && ew == 0) FFN_EV(14, 0);
            }
            // ---- GELU chunks: group cg >> 1 takes the chunks in acc1 buffer cg >> 1; this warp
            // owns columns [64 (cg & 1), +64) of them = H k-block cg & 1, all eight 16-byte chunks
            const int grp = cg >> 1, sub = cg & 1;
            for (int j = 0; j < nch; j++, c1++) {
                const int b = c1 & 1;
                if (b != grp) continue;
                ptx::mbar_wait(&acc1_full[b], (c1 >> 1) & 1);
                if (lane == 0 && ew == 0) FFN_EV(3, j);
                ptx::tc_fence_after();
                uint32_t hp[32];  // row r's 64 columns as bf16 pairs
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    float g[32];
                    tmem_load32(T_ACC1 + b * C::CH + sub * 64 + h * 32 + (static_cast<uint32_t>(q * 32) << 16), g);
                    if (h == 1) {  // both halves are in registers: the accumulator is free
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) arrive_lead(&acc1_empty[b]);
                    }
                    const int pc = chunk(j) * C::CH + sub * 64 + h * 32;
#if DCAT_FFN_ABLATE & 1  // kernel micro-bench only (tools/kbench): skip the GELU math
                    if (pc < 0)
#endif
#pragma unroll
                    for (int k = 0; k < 32; k += 4) {
                        const float4 bb = ldg4(e.bias + pc + k);
                        g[k] = gelu_fast(g[k] + bb.x);
                        g[k + 1] = gelu_fast(g[k + 1] + bb.y);
                        g[k + 2] = gelu_fast(g[k + 2] + bb.z);
                        g[k + 3] = gelu_fast(g[k + 3] + bb.w);
                    }
#pragma unroll
                    for (int k = 0; k < 16; k++) hp[16 * h + k] = pack_bf16(g[2 * k], g[2 * k + 1]);
                }
                ptx::mbar_wait(&h_empty[b], ((c1 >> 1) & 1) ^ 1);
                // row r of k-block `sub` of H buffer b, 128 B swizzle
                const uint32_t rowa = h_base + b * C::H_BUF + sub * 16384 + r * 128;
#pragma unroll
                for (int k = 0; k < 8; k++)
                    sts4u(rowa + ((k ^ (r & 7)) << 4), hp[4 * k], hp[4 * k + 1], hp[4 * k + 2], hp[4 * k + 3]);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) arrive_lead(&h_full[b]);
                if (lane == 0 && ew == 0) FFN_EV(4, j);
                if (lane == 0 && ew == 15) FFN_EV(7, j);
            }
            // ---- residual + LayerNorm
            if (fin) {
                // acc2 started as the residual rows (tcgen05.cp): x = acc2 + b2 -> x_out, written
                // back into acc2 for the LayerNorm passes.
                const bool live = row < M;
                const uint32_t tacc = T_ACC2 + (static_cast<uint32_t>(q * 32) << 16) + c0;
                float v[32];
                float s1[1] = {0.f};
                bool bad = false;
                ptx::mbar_wait(acc2_full, i & 1);
                ptx::tc_fence_after();
                if (lane == 0 && ew == 0) FFN_EV(5, 0);
#pragma unroll 1
                for (int h = 0; h < C::FCOLS; h += 32) {
                    if (h) staging_free<0>(lane);
                    tmem_load32(tacc + h, v);
#pragma unroll
                    for (int j = 0; j < 8; j++) {  // (resid + acc) + b2
                        const float4 bb = ldg4(e.b2 + c0 + h + 4 * j);
                        float* w = v + 4 * j;
                        w[0] += bb.x;
                        w[1] += bb.y;
                        w[2] += bb.z;
                        w[3] += bb.w;
                    }
#pragma unroll
                    for (int k = 0; k < 32; k++) {
                        bad |= !isfinite(v[k]);
                        s1[0] += v[k];
                    }
                    __syncwarp();
#if DCAT_FFN_ABLATE & 2  // kernel micro-bench only (tools/kbench): skip the output stores / LayerNorm
                    if (m0 < 0)
#endif
                    {
                        write_f32_row(S0, lane, v);
                        store_block(&mp.xout, S0, c0 + h, row_base, lane);
                    }
                    tmem_store32(tacc + h, v);
                }
                if (bad && live && e.layer_idx >= 0) atomicMax(&e.st->nonfinite_layer, e.layer_idx + 1);
#if DCAT_FFN_ABLATE & 2
                if (m0 < 0)
#endif
                if (e.ln_out) {
                    float mu = 0.f, rs = 1.f;
                    if (e.ln_g) {
                        quad_reduce<C::CGF, 1, 1>(s_red, s1, cg, lane, q);
                        const float dn = static_cast<float>(D);
                        mu = s1[0] / dn;
                        float var[1] = {0.f};
#pragma unroll 1
                        for (int h = 0; h < C::FCOLS; h += 32) {
                            tmem_load32(tacc + h, v);
#pragma unroll
                            for (int k = 0; k < 32; k++) {
                                const float d0 = v[k] - mu;
                                var[0] += d0 * d0;
                            }
                        }
                        quad_reduce<C::CGF, 1, 1>(s_red, var, cg, lane, q);
                        rs = 1.0f / sqrtf(var[0] / dn + 1e-5f);
                    }
                    staging_free<0>(lane);
#pragma unroll 1
                    for (int h = 0; h < C::FCOLS; h += 32) {
                        tmem_load32(tacc + h, v);
                        if (e.ln_g) {
#pragma unroll
                            for (int j = 0; j < 8; j++) {
                                const float4 gg = ldg4(e.ln_g + c0 + h + 4 * j);
                                const float4 bb = ldg4(e.ln_b + c0 + h + 4 * j);
                                float* w = v + 4 * j;
                                w[0] = gg.x * ((w[0] - mu) * rs) + bb.x;
                                w[1] = gg.y * ((w[1] - mu) * rs) + bb.y;
                                w[2] = gg.z * ((w[2] - mu) * rs) + bb.z;
                                w[3] = gg.w * ((w[3] - mu) * rs) + bb.w;
                            }
                        }
                        write_bf16_row(S0 + h * 64, lane, v);
                        store_block(&mp.ln, S0 + h * 64, c0 + h, row_base, lane);
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_lead(acc2_empty);
                if (lane == 0 && ew == 0) FFN_EV(6, 0);
            }
            // the next tile's GELU writes reuse this staging: all epilogue warps drain first
            staging_free<0>(lane);
            named_bar(5, 32 * C::EPI_WARPS);
            if (lane == 0 && ew == 0) FFN_EV(9, 0);
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    ptx::tc_fence_before();
    if constexpr (CL == 2) ptx::cluster_sync();  // the leader's MMAs / commits reach the peer until here
    else __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        if constexpr (CL == 2) ptx::tmem_dealloc_pair(tmem, 512);
        else ptx::tmem_dealloc(tmem, 512);
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

// epilogue I/O map: rows x cols matrix (ld elements), 32 x 32 boxes; fp32 -> 128B swizzle, bf16 -> 64B
CUtensorMap tmap_epi(const void* base, bool f32, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows = 32) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    if (!base) return m;
    const uint64_t es = f32 ? 4 : 2;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * es};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t el[2] = {1, 1};
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * es) & 15))
        throw CudaError("epilogue tensor map: base / row stride must be 16-byte aligned");
    CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(base), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (epilogue) failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

EpiMaps make_maps(const Epi& e, int M, int N) {
    EpiMaps mp;
    std::memset(&mp, 0, sizeof mp);
    const uint64_t rows = static_cast<uint64_t>(M);
    if (e.mode == EPI_BIAS) {
        if (e.seg_cols % 32 == 0)
            for (int s = 0; s < 3 && s * e.seg_cols < N; s++)
                mp.o[s] = e.out_trans[s]
                              ? tmap_epi(e.out[s], false, static_cast<uint64_t>(e.out_ld[s]),
                                         static_cast<uint64_t>(e.seg_cols), e.out_ld[s])  // [seg_cols][ld] (V^T)
                              : tmap_epi(e.out[s], false, static_cast<uint64_t>(e.seg_cols), rows, e.out_ld[s]);
    } else if (e.mode == EPI_RESID_LN || e.mode == EPI_L2NORM) {
        mp.resid = tmap_epi(e.resid, true, static_cast<uint64_t>(N), rows, e.ld_x);
        mp.xout = tmap_epi(e.x_out, true, static_cast<uint64_t>(N), rows, e.ld_x);
        mp.ln = tmap_epi(e.ln_out, false, static_cast<uint64_t>(N), rows, e.ln_ld);
        mp.out2 = tmap_epi(e.out2, false, static_cast<uint64_t>(N), rows, e.out2_ld);
    }
    return mp;
}

int num_sms() {
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

template <int BN, int MODE, bool RB = false>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e, cudaStream_t s);

// full-row epilogue over d = 512 on a CTA pair (SPL = 2): BN = 256 columns per CTA
template <int MODE, bool LK>
void launch_split(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e, cudaStream_t s) {
    using C = Cfg<256, MODE, false, 2, LK>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    auto kern = k_gemm_tc<256, MODE, false, 2, LK>;
    set_smem_attr(reinterpret_cast<const void*>(kern), C::SMEM);
    {
        const int npad = (N + 31) & ~31;
        if (6 * npad + 3 > C::PARAM_FLOATS)
            throw InvalidArg("gemm_tc: epilogue parameters of N=" + std::to_string(N) + " exceed the smem staging");
    }
    const EpiMaps mp = make_maps(e, M, N);
    const int m_tiles = (M + BM - 1) / BM;
    const int pairs = m_tiles < num_sms() / 2 ? m_tiles : num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DCAT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, e, mp));
}

template <int BN, int MODE, bool RB>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e, cudaStream_t s) {
    using C = Cfg<BN, MODE, RB>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    set_smem_attr(reinterpret_cast<const void*>(k_gemm_tc<BN, MODE, RB>), C::SMEM);
    {
        const int npad = (N + 31) & ~31;
        const int need = RB ? BN : MODE == EPI_BIAS ? npad : MODE == EPI_HEAD ? 4 * npad + 3 : 6 * npad + 3;
        if (need > C::PARAM_FLOATS)
            throw InvalidArg("gemm_tc: epilogue parameters of N=" + std::to_string(N) + " exceed the smem staging");
    }
    const EpiMaps mp = make_maps(e, M, N);
    const int num_n = (N + BN - 1) / BN;
    int tiles = ((M + BM - 1) / BM) * num_n;
    int grid = tiles < num_sms() ? tiles : num_sms();
    if constexpr (RB) grid = grid / num_n * num_n;  // a fixed N slice per CTA (tiles >= num_sms here)
    k_gemm_tc<BN, MODE, RB><<<grid, C::THREADS, C::SMEM, s>>>(ta, tb, M, N, K, e, mp);
    DCAT_LAUNCH_CHECK();
}

bool resident_b_disabled() {  // A/B switch for measurements: DCAT_NO_RESIDENT_B=1
    static const bool off = getenv("DCAT_NO_RESIDENT_B") != nullptr;
    return off;
}

template <int MODE>
void launch_mode(int BN, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e,
                 cudaStream_t s) {
    switch (BN) {
        case 64: launch<64, MODE>(ta, tb, M, N, K, e, s); break;
        case 128: launch<128, MODE>(ta, tb, M, N, K, e, s); break;
        case 256:
            // resident weight slice: large M (every CTA gets many tiles of its slice), K <= 256
            if constexpr (MODE == EPI_BIAS)
                if (K <= 64 * Cfg<256, EPI_BIAS, true>::KB_RES && !resident_b_disabled() &&
                    static_cast<long>((M + BM - 1) / BM) * ((N + 255) / 256) >= 4L * num_sms()) {
                    launch<256, MODE, true>(ta, tb, M, N, K, e, s);
                    break;
                }
            launch<256, MODE>(ta, tb, M, N, K, e, s);
            break;
        case 512:
            if constexpr (MODE == EPI_RESID_LN || MODE == EPI_L2NORM) {
                // d = 512: the row split over a CTA pair (double-buffered accumulators, 8 epilogue
                // warps per CTA) unless DCAT_NO_PAIR_EPILOGUE selects the one-CTA BN = 512 tile
                static const bool one_cta = getenv("DCAT_NO_PAIR_EPILOGUE") != nullptr;
                if (one_cta) launch<512, MODE>(ta, tb, M, N, K, e, s);
                // long K (FFN2: d_ff = 2048): 3 operand stages, 4 epilogue warps (LK); short K: 2, 8
                else if (K >= 1024) launch_split<MODE, true>(ta, tb, M, N, K, e, s);
                else launch_split<MODE, false>(ta, tb, M, N, K, e, s);
                break;
            }
            [[fallthrough]];
        default: throw InvalidArg("gemm_tc: unsupported tile width " + std::to_string(BN));
    }
}

}  // namespace

namespace {
template <int D, int CL, bool TAIL = false>
void launch_ffn(const bf16* A, int lda, const bf16* W1t, const bf16* W2t, int M, int F, const Epi& e,
                const EpiMaps& mp, cudaStream_t s, const bf16* Wot = nullptr) {
    using C = FfnCfg<D, CL, TAIL>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    // the epilogues read their parameter vectors as float4 through L1
    auto vec = [](const float* p, bool need, const char* what) {
        if ((need && p == nullptr) || (reinterpret_cast<uintptr_t>(p) & 15))
            throw InvalidArg(std::string("ffn_tc: parameter vector '") + what + "' missing or not 16-byte aligned");
    };
    vec(e.bias, true, "b1");
    vec(e.b2, true, "b2");
    vec(e.ln_g, false, "ln_g");
    vec(e.ln_b, e.ln_g != nullptr, "ln_b");
    if constexpr (TAIL) {
        vec(e.o_bias, true, "bo");
        vec(e.ln2_g, true, "ln2_g");
        vec(e.ln2_b, true, "ln2_b");
    }
    set_smem_attr(reinterpret_cast<const void*>(k_ffn_tc<D, CL, TAIL>), C::SMEM);
    const CUtensorMap ta = tmap_bf16(A, static_cast<uint64_t>(D), static_cast<uint64_t>(M),
                                     static_cast<uint64_t>(lda) * 2, 128);
    const CUtensorMap t1 = tmap_bf16(W1t, static_cast<uint64_t>(D), static_cast<uint64_t>(F),
                                     static_cast<uint64_t>(D) * 2, static_cast<uint32_t>(C::W1_ROWS));
    const CUtensorMap t2 = tmap_bf16(W2t, static_cast<uint64_t>(F), static_cast<uint64_t>(D),
                                     static_cast<uint64_t>(F) * 2, static_cast<uint32_t>(C::W2_ROWS));
    // TAIL: Wo^T [D x D] (K-major) in [NW2 x 64] ring-slot blocks
    const CUtensorMap to = TAIL ? tmap_bf16(Wot, static_cast<uint64_t>(D), static_cast<uint64_t>(D),
                                            static_cast<uint64_t>(D) * 2, static_cast<uint32_t>(C::NW2))
                                : t2;
    EpiMaps mpf = mp;  // residual in [128 x 32] fp32 blocks: one ring slot each, copied into acc2
    mpf.resid = tmap_epi(e.resid, true, static_cast<uint64_t>(D), static_cast<uint64_t>(M), e.ld_x, 128);
    const int units = ((M + 127) / 128 + CL - 1) / CL;
    const int per = num_sms() / CL;
    const int grid = CL * (units < per ? units : per);
    if constexpr (CL == 1) {
        k_ffn_tc<D, 1, TAIL><<<grid, C::THREADS, C::SMEM, s>>>(ta, t1, t2, to, M, F, e, mpf);
        DCAT_LAUNCH_CHECK();
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DCAT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_ffn_tc<D, CL, TAIL>, ta, t1, t2, to, M, F, e, mpf));
    }
}
}  // namespace

#if DCAT_FFN_TRACE
void ffn_trace_reset() {
    unsigned z[FFN_TR_ROLES] = {};
    DCAT_CUDA_CHECK(cudaMemcpyToSymbol(g_ffn_trace_n, z, sizeof(z)));
}
// all roles' events, concatenated (the viewer sorts by time)
int ffn_trace_read(unsigned long long* out, int cap) {
    unsigned n[FFN_TR_ROLES];
    DCAT_CUDA_CHECK(cudaMemcpyFromSymbol(n, g_ffn_trace_n, sizeof(n)));
    std::vector<unsigned long long> all(FFN_TR_ROLES * FFN_TR_CAP);
    DCAT_CUDA_CHECK(cudaMemcpyFromSymbol(all.data(), g_ffn_trace, all.size() * sizeof(unsigned long long)));
    int m = 0;
    for (int r = 0; r < FFN_TR_ROLES; r++)
        for (unsigned k = 0; k < n[r] && m < cap; k++)
            out[m++] = all[r * FFN_TR_CAP + k] + (static_cast<unsigned long long>(16 * r) << 8);  // code += 16 role
    return m;
}
extern "C" void dcat_ffn_trace_reset() { ffn_trace_reset(); }
extern "C" int dcat_ffn_trace_read(unsigned long long* out, int cap) { return ffn_trace_read(out, cap); }
#endif

// D = 256 runs FFN1 of two hidden chunks as one N = 256 MMA (PAIR_N): the chunk count F / 128 must
// be even there, or the kernel would read the W1 blocks of a chunk that does not exist
bool ffn_tc_supported(int D, int F) {
    return (D == 64 || D == 128 || D == 256) && F % 128 == 0 && F <= 1024 && (D != 256 || (F / 128) % 2 == 0);
}

void ffn_tc(const bf16* A, int lda, const bf16* W1t, const bf16* W2t, int M, int D, int F, const Epi& e,
            cudaStream_t s) {
    if (M <= 0) return;
    if (!ffn_tc_supported(D, F)) throw InvalidArg("ffn_tc: unsupported shape");
    Epi em = e;
    em.mode = EPI_RESID_LN;
    const EpiMaps mp = make_maps(em, M, D);
    // One CTA per 128-row tile. DCAT_FFN_PAIR=1 selects the CTA-pair kernel (M = 256 per pair,
    // half the weight bytes per SM); it measured slower on the PinFM-base step (profiles/r01_ffn.md).
    static const bool single = getenv("DCAT_FFN_PAIR") == nullptr;
    switch (D) {
        case 64: launch_ffn<64, 1>(A, lda, W1t, W2t, M, F, e, mp, s); break;
        case 128:
            if (single) launch_ffn<128, 1>(A, lda, W1t, W2t, M, F, e, mp, s);
            else launch_ffn<128, 2>(A, lda, W1t, W2t, M, F, e, mp, s);
            break;
        default:
            if (single) launch_ffn<256, 1>(A, lda, W1t, W2t, M, F, e, mp, s);
            else launch_ffn<256, 2>(A, lda, W1t, W2t, M, F, e, mp, s);
            break;
    }
}

bool layer_tail_tc_supported(int D, int F) {
    return (D == 128 || D == 256) && F % 128 == 0 && F <= 1024 && (D != 256 || (F / 128) % 2 == 0);
}

void layer_tail_tc(const bf16* A_o, int lda, const bf16* Wot, const bf16* W1t, const bf16* W2t, int M, int D, int F,
                   const Epi& e, cudaStream_t s) {
    if (M <= 0) return;
    if (!layer_tail_tc_supported(D, F)) throw InvalidArg("layer_tail_tc: unsupported shape");
    if (!e.o_bias || !e.ln2_g || !e.ln2_b) throw InvalidArg("layer_tail_tc: o_bias / ln2_g / ln2_b required");
    Epi em = e;
    em.mode = EPI_RESID_LN;
    const EpiMaps mp = make_maps(em, M, D);
    if (D == 128) launch_ffn<128, 1, true>(A_o, lda, W1t, W2t, M, F, e, mp, s, Wot);
    else launch_ffn<256, 1, true>(A_o, lda, W1t, W2t, M, F, e, mp, s, Wot);
}

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
