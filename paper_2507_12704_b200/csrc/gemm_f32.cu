// gemm_f32.cu — fp32 parity path of K3: SIMT GEMM + row epilogue.
//
// Same contract as gemm_tc (launch.h) but fp32 storage and fp32 CUDA-core math,
// W in the reference's own in x out layout (linear_forward, model.cpp:43-46).
// Used with DCAT_PRECISION_FP32 to separate algorithm errors from bf16
// rounding: this path must match the CPU oracle to the reference's own 1e-4
// (test_dcat.cpp:227). Each thread accumulates its outputs over k in
// ascending order like matmul (mat.hpp:66-75).
#include "launch.h"

namespace dcat {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) k_sgemm(const float* __restrict__ A, int lda, const float* __restrict__ W,
                                               int ldw, int M, int N, int K, float* __restrict__ C, int ldc) {
    __shared__ float sA[TK][TM + 4];
    __shared__ float sW[TK][TN + 4];
    int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += 256) {
            int r = i / TK, c = i % TK;
            int gm = m0 + r, gk = k0 + c;
            sA[c][r] = (gm < M && gk < K) ? A[static_cast<size_t>(gm) * lda + gk] : 0.f;
        }
        for (int i = threadIdx.x; i < TK * TN; i += 256) {
            int r = i / TN, c = i % TN;
            int gk = k0 + r, gn = n0 + c;
            sW[r][c] = (gk < K && gn < N) ? W[static_cast<size_t>(gk) * ldw + gn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TK; k++) {
            float a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = sA[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; j++) w[j] = sW[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] += a[i] * w[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int gn = n0 + tx * 4 + j;
            if (gn < N) C[static_cast<size_t>(gm) * ldc + gn] = acc[i][j];
        }
    }
}

constexpr int MAXV = 32;  // columns per lane: N <= 1024

// one warp per row; lanes own columns c = lane + 32 k
template <int MODE>
__global__ void k_row_epi(const float* __restrict__ acc, int ldacc, int M, int N, Epi e) {
    int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= M) return;
    const float* a = acc + static_cast<size_t>(row) * ldacc;
    float v[MAXV];
    int nv = (N + 31) / 32;
    if constexpr (MODE == EPI_BIAS) {
        for (int k = 0; k < nv; k++) {
            int c = lane + 32 * k;
            if (c >= N) break;
            float x = a[c] + e.bias[c];
            if (e.act) x = gelu_tanh(x);
            int sg = c / e.seg_cols;
            static_cast<float*>(e.out[sg])[static_cast<size_t>(row) * e.out_ld[sg] + (c - sg * e.seg_cols)] = x;
        }
    } else if constexpr (MODE == EPI_HEAD) {
        float l0 = 0.f, l1 = 0.f, l2 = 0.f;
        for (int k = 0; k < nv; k++) {
            int c = lane + 32 * k;
            if (c >= N) break;
            float z = gelu_tanh(a[c] + e.bias[c]);
            l0 += z * e.w2[c * 3];
            l1 += z * e.w2[c * 3 + 1];
            l2 += z * e.w2[c * 3 + 2];
        }
        l0 = warp_sum(l0);
        l1 = warp_sum(l1);
        l2 = warp_sum(l2);
        if (lane == 0) {
            e.logits[static_cast<size_t>(row) * 3] = l0 + e.b2[0];
            e.logits[static_cast<size_t>(row) * 3 + 1] = l1 + e.b2[1];
            e.logits[static_cast<size_t>(row) * 3 + 2] = l2 + e.b2[2];
        }
    } else {
        float s1 = 0.f;
        if constexpr (MODE == EPI_RESID_LN) {
            bool bad = false;
            for (int k = 0; k < nv; k++) {
                int c = lane + 32 * k;
                v[k] = 0.f;
                if (c >= N) continue;
                v[k] = a[c] + e.bias[c] + e.resid[static_cast<size_t>(row) * e.ld_x + c];
                bad |= !isfinite(v[k]);
                s1 += v[k];
                e.x_out[static_cast<size_t>(row) * e.ld_x + c] = v[k];
            }
            if (__any_sync(0xffffffffu, bad) && lane == 0 && e.layer_idx >= 0)
                atomicMax(&e.st->nonfinite_layer, e.layer_idx + 1);
        } else {  // EPI_L2NORM
            float ss = 0.f;
            for (int k = 0; k < nv; k++) {
                int c = lane + 32 * k;
                v[k] = 0.f;
                if (c >= N) continue;
                v[k] = a[c] + e.bias[c];
                ss += v[k] * v[k];
            }
            ss = warp_sum(ss);
            float nrm = sqrtf(ss);
            float inv = 1.0f / (nrm < 1e-12f ? 1e-12f : nrm);
            float m0 = 0.f, m1 = 0.f, m2 = 0.f;
            for (int k = 0; k < nv; k++) {
                int c = lane + 32 * k;
                if (c >= N) continue;
                v[k] *= inv;
                s1 += v[k];
                if (e.x_out) e.x_out[static_cast<size_t>(row) * e.ld_x + c] = v[k];
                if (e.out2) static_cast<float*>(e.out2)[static_cast<size_t>(row) * e.out2_ld + c] = v[k];
                if (e.mod_w) {
                    m0 += v[k] * e.mod_w[c * 3];
                    m1 += v[k] * e.mod_w[c * 3 + 1];
                    m2 += v[k] * e.mod_w[c * 3 + 2];
                }
            }
            if (e.mod_w) {
                m0 = warp_sum(m0);
                m1 = warp_sum(m1);
                m2 = warp_sum(m2);
                if (lane == 0) {
                    e.mlogits[static_cast<size_t>(row) * 3] = m0 + e.mod_b[0];
                    e.mlogits[static_cast<size_t>(row) * 3 + 1] = m1 + e.mod_b[1];
                    e.mlogits[static_cast<size_t>(row) * 3 + 2] = m2 + e.mod_b[2];
                }
            }
        }
        if (e.ln_out == nullptr) return;
        float* lo = static_cast<float*>(e.ln_out) + static_cast<size_t>(row) * e.ln_ld;
        if (e.ln_g == nullptr) {
            for (int k = 0; k < nv; k++) {
                int c = lane + 32 * k;
                if (c < N) lo[c] = v[k];
            }
            return;
        }
        float mu = warp_sum(s1) / static_cast<float>(N);
        float var = 0.f;
        for (int k = 0; k < nv; k++) {
            int c = lane + 32 * k;
            if (c < N) {
                float d = v[k] - mu;
                var += d * d;
            }
        }
        var = warp_sum(var) / static_cast<float>(N);
        float rs = 1.0f / sqrtf(var + 1e-5f);
        for (int k = 0; k < nv; k++) {
            int c = lane + 32 * k;
            if (c < N) lo[c] = e.ln_g[c] * ((v[k] - mu) * rs) + e.ln_b[c];
        }
    }
}

}  // namespace

void gemm_f32(const float* A, int lda, const float* W, int ldw, int M, int N, int K, const Epi& e, float* tmp,
              cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    if (N > 32 * MAXV && e.mode != EPI_BIAS)  // only the row-statistics modes keep the row in registers
        throw InvalidArg("gemm_f32: N too large for the row epilogue");
    dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
    k_sgemm<<<grid, 256, 0, s>>>(A, lda, W, ldw, M, N, K, tmp, N);
    unsigned g = static_cast<unsigned>((static_cast<int64_t>(M) * 32 + 255) / 256);
    switch (e.mode) {
        case EPI_BIAS: k_row_epi<EPI_BIAS><<<g, 256, 0, s>>>(tmp, N, M, N, e); break;
        case EPI_RESID_LN: k_row_epi<EPI_RESID_LN><<<g, 256, 0, s>>>(tmp, N, M, N, e); break;
        case EPI_L2NORM: k_row_epi<EPI_L2NORM><<<g, 256, 0, s>>>(tmp, N, M, N, e); break;
        case EPI_HEAD: k_row_epi<EPI_HEAD><<<g, 256, 0, s>>>(tmp, N, M, N, e); break;
        default: throw InvalidArg("gemm_f32: bad epilogue mode");
    }
    DCAT_LAUNCH_CHECK();
}

}  // namespace dcat
