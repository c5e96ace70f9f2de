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

}  // namespace

void scatter_outputs(const int32_t* perm, int64_t B, const float* logits_p, const float* mlog_p, const float* h_p,
                     int d, float* logits, float* mlogits, float* h_cand, cudaStream_t s) {
    if (B <= 0) return;
    k_scatter<<<static_cast<unsigned>((B * 32 + 255) / 256), 256, 0, s>>>(perm, B, logits_p, mlog_p, h_p, d, logits,
                                                                         mlogits, h_cand);
    DCAT_LAUNCH_CHECK();
}

}  // namespace dcat
