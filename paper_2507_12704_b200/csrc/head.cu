// head.cu — K7 tail: scatter per-candidate results from unique-grouped order
// back to the caller's row order (rank_forward_batch fills out[i] per input
// row, finetune.cpp:481-491).
#include "launch.h"

namespace dcat {

namespace {

__global__ void k_scatter(const int32_t* __restrict__ perm, int64_t B, const float* __restrict__ logits_p,
                          const float* __restrict__ mlog_p, const float* __restrict__ h_p, int d,
                          float* __restrict__ logits, float* __restrict__ mlogits, float* __restrict__ h_cand) {
    int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (p >= B) return;
    int64_t i = perm[p];
    if (lane < 3) {
        logits[i * 3 + lane] = logits_p[p * 3 + lane];
        mlogits[i * 3 + lane] = mlog_p[p * 3 + lane];
    }
    // (mlog_p holds mod_b broadcast when the sequence module is off: d_module = 0,
    //  crossing_forward finetune.cpp:317-323)
    if (h_cand && h_p)
        for (int c = lane; c < d; c += 32) h_cand[i * d + c] = h_p[p * d + c];
}

__global__ void k_pool(const int64_t* __restrict__ tok_off, int b_u, const float* __restrict__ H, int d, int last,
                       float* __restrict__ sel) {
    const int u = blockIdx.x;
    if (u >= b_u) return;
    const int64_t t0 = tok_off[u], n = tok_off[u + 1] - t0;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float v = 0.f;
        if (n > 0) {
            if (last) {
                v = H[(t0 + n - 1) * d + c];
            } else {
                for (int64_t i = 0; i < n; i++) v = __fadd_rn(v, H[(t0 + i) * d + c]);  // axpy in row order
                v = __fdiv_rn(v, static_cast<float>(n));
            }
        }
        sel[static_cast<size_t>(u) * d + c] = v;
    }
}

template <typename T>
__global__ void k_last_rows(const int64_t* __restrict__ tok_off, int b_u, const T* __restrict__ src, int d,
                            T* __restrict__ dst) {
    const int u = blockIdx.x;
    if (u >= b_u) return;
    const int64_t r = tok_off[u + 1] - 1;
    for (int c = threadIdx.x; c < d; c += blockDim.x) dst[static_cast<size_t>(u) * d + c] = src[r * d + c];
}

template <typename T>
__global__ void k_bcast(const int32_t* __restrict__ perm, const int32_t* __restrict__ rep, int64_t B,
                        const float* __restrict__ sel, int d, T* __restrict__ feat, int ld, int col0,
                        float* __restrict__ hc) {
    const int64_t p = blockIdx.x;
    if (p >= B) return;
    const float* s = sel + static_cast<size_t>(rep[perm[p]]) * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        ActIO<T>::store(feat + p * ld + col0 + c, s[c]);
        if (hc) hc[p * d + c] = s[c];
    }
}

__global__ void k_mlogits(const int32_t* __restrict__ perm, const int32_t* __restrict__ rep, int64_t B,
                          const float* __restrict__ sel_u, const float* __restrict__ hc, int d,
                          const float* __restrict__ mod_w, const float* __restrict__ mod_b, float* __restrict__ mlog) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= B) return;
    float acc[3] = {0.f, 0.f, 0.f};
    int k = 0;
    if (sel_u) {  // matmul(selflat, mod_w): one row, k ascending (mat.hpp:61-76)
        const float* s = sel_u + static_cast<size_t>(rep[perm[p]]) * d;
        for (int c = 0; c < d; c++, k++)
            for (int j = 0; j < 3; j++) acc[j] = __fadd_rn(acc[j], __fmul_rn(s[c], mod_w[k * 3 + j]));
    }
    if (hc) {
        const float* h = hc + p * d;
        for (int c = 0; c < d; c++, k++)
            for (int j = 0; j < 3; j++) acc[j] = __fadd_rn(acc[j], __fmul_rn(h[c], mod_w[k * 3 + j]));
    }
    for (int j = 0; j < 3; j++) mlog[p * 3 + j] = __fadd_rn(acc[j], mod_b[j]);
}

}  // namespace

// dst[p] = src[perm[p]] (fp32 source rows -> activation type), and the inverse scatter of fp32 rows
template <typename T>
__global__ void k_gather_rows(const float* __restrict__ src, const int32_t* __restrict__ perm, int64_t B, int d,
                              T* __restrict__ dst) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B * d) return;
    const int64_t p = i / d;
    const int c = static_cast<int>(i - p * d);
    ActIO<T>::store(dst + i, src[static_cast<int64_t>(perm[p]) * d + c]);
}
__global__ void k_scatter_rows(const float* __restrict__ src, const int32_t* __restrict__ perm, int64_t B, int d,
                               float* __restrict__ dst) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B * d) return;
    const int64_t p = i / d;
    const int c = static_cast<int>(i - p * d);
    dst[static_cast<int64_t>(perm[p]) * d + c] = src[i];
}
template <typename T>
void gather_rows(const float* src, const int32_t* perm, int64_t B, int d, T* dst, cudaStream_t s) {
    if (B <= 0) return;
    k_gather_rows<T><<<static_cast<unsigned>((B * d + 255) / 256), 256, 0, s>>>(src, perm, B, d, dst);
    DCAT_LAUNCH_CHECK();
}
void scatter_rows(const float* src, const int32_t* perm, int64_t B, int d, float* dst, cudaStream_t s) {
    if (B <= 0) return;
    k_scatter_rows<<<static_cast<unsigned>((B * d + 255) / 256), 256, 0, s>>>(src, perm, B, d, dst);
    DCAT_LAUNCH_CHECK();
}
template void gather_rows<float>(const float*, const int32_t*, int64_t, int, float*, cudaStream_t);
template void gather_rows<bf16>(const float*, const int32_t*, int64_t, int, bf16*, cudaStream_t);

void pool_selectors(const int64_t* tok_off, int b_u, const float* H, int d, int last, float* sel, cudaStream_t s) {
    if (b_u <= 0) return;
    k_pool<<<b_u, 128, 0, s>>>(tok_off, b_u, H, d, last, sel);
    DCAT_LAUNCH_CHECK();
}
template <typename T>
void gather_last_rows(const int64_t* tok_off, int b_u, const T* src, int d, T* dst, cudaStream_t s) {
    if (b_u <= 0) return;
    k_last_rows<T><<<b_u, 128, 0, s>>>(tok_off, b_u, src, d, dst);
    DCAT_LAUNCH_CHECK();
}
template <typename T>
void broadcast_selectors(const int32_t* perm, const int32_t* rep, int64_t B, const float* sel, int d, T* feat,
                         int ld, int col0, float* hc, cudaStream_t s) {
    if (B <= 0) return;
    k_bcast<T><<<static_cast<unsigned>(B), 128, 0, s>>>(perm, rep, B, sel, d, feat, ld, col0, hc);
    DCAT_LAUNCH_CHECK();
}
void module_logits(const int32_t* perm, const int32_t* rep, int64_t B, const float* sel_u, const float* hc, int d,
                   const float* mod_w, const float* mod_b, float* mlog, cudaStream_t s) {
    if (B <= 0) return;
    k_mlogits<<<static_cast<unsigned>((B + 127) / 128), 128, 0, s>>>(perm, rep, B, sel_u, hc, d, mod_w, mod_b, mlog);
    DCAT_LAUNCH_CHECK();
}
template void gather_last_rows<float>(const int64_t*, int, const float*, int, float*, cudaStream_t);
template void gather_last_rows<bf16>(const int64_t*, int, const bf16*, int, bf16*, cudaStream_t);
template void broadcast_selectors<float>(const int32_t*, const int32_t*, int64_t, const float*, int, float*, int,
                                         int, float*, cudaStream_t);
template void broadcast_selectors<bf16>(const int32_t*, const int32_t*, int64_t, const float*, int, bf16*, int, int,
                                        float*, cudaStream_t);

void scatter_outputs(const int32_t* perm, int64_t B, const float* logits_p, const float* mlog_p, const float* h_p,
                     int d, float* logits, float* mlogits, float* h_cand, cudaStream_t s) {
    if (B <= 0) return;
    k_scatter<<<static_cast<unsigned>((B * 32 + 255) / 256), 256, 0, s>>>(perm, B, logits_p, mlog_p, h_p, d, logits,
                                                                         mlogits, h_cand);
    DCAT_LAUNCH_CHECK();
}

}  // namespace dcat
