// kbench.cu — kernel micro-bench for the GEMM-class kernels (not part of the product).
//
// Times dcat::ffn_tc (fused FFN) against the unfused FFN1 + FFN2 gemm_tc pair and
// plain gemm_tc shapes at a large M, with CUDA events over repeated launches.
// Built several times with -DDCAT_FFN_ABLATE=0..3 (see Makefile) to measure how much
// of the fused kernel's time the GELU / final epilogue stages cost.
//   usage: kbench [M] [D] [F] [iters]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2507_12704_b200/csrc/launch.h"

using namespace dcat;

#if DCAT_FFN_TRACE
namespace dcat {
void ffn_trace_reset();
int ffn_trace_read(unsigned long long* out, int cap);
}  // namespace dcat
#endif

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

template <typename T>
T* dalloc(size_t n) {
    T* p;
    CK(cudaMalloc(&p, n * sizeof(T)));
    CK(cudaMemset(p, 0, n * sizeof(T)));
    return p;
}

__global__ void k_fill(bf16* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t h = static_cast<uint32_t>(i) * 2654435761u ^ seed;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        p[i] = __float2bfloat16((static_cast<int>(h & 1023) - 512) * (1.0f / 4096.0f));
    }
}

template <typename F>
float time_it(F&& f, int iters) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; i++) f();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int i = 0; i < iters; i++) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1000.f / iters;  // us
}

int main(int argc, char** argv) {
    const int M = argc > 1 ? std::atoi(argv[1]) : 262144;
    const int D = argc > 2 ? std::atoi(argv[2]) : 256;
    const int F = argc > 3 ? std::atoi(argv[3]) : 1024;
    const int iters = argc > 4 ? std::atoi(argv[4]) : 20;
    bf16* A = dalloc<bf16>(static_cast<size_t>(M) * D);
    bf16* W1t = dalloc<bf16>(static_cast<size_t>(F) * D);
    bf16* W2t = dalloc<bf16>(static_cast<size_t>(D) * F);
    bf16* H = dalloc<bf16>(static_cast<size_t>(M) * F);
    bf16* ln = dalloc<bf16>(static_cast<size_t>(M) * D);
    float* resid = dalloc<float>(static_cast<size_t>(M) * D);
    float* xout = dalloc<float>(static_cast<size_t>(M) * D);
    float* b1 = dalloc<float>(F);
    float* b2 = dalloc<float>(D);
    float* g = dalloc<float>(D);
    float* bb = dalloc<float>(D);
    Status* st = dalloc<Status>(1);
    k_fill<<<1024, 256>>>(A, static_cast<size_t>(M) * D, 1);
    k_fill<<<1024, 256>>>(W1t, static_cast<size_t>(F) * D, 2);
    k_fill<<<1024, 256>>>(W2t, static_cast<size_t>(D) * F, 3);
    CK(cudaDeviceSynchronize());

    Epi fin{};
    fin.mode = EPI_RESID_LN;
    fin.bias = b1;
    fin.b2 = b2;
    fin.resid = resid;
    fin.x_out = xout;
    fin.ld_x = D;
    fin.ln_g = g;
    fin.ln_b = bb;
    fin.ln_out = ln;
    fin.ln_ld = D;
    fin.st = st;
    fin.layer_idx = -1;

    Epi e1{};
    e1.mode = EPI_BIAS;
    e1.act = 1;
    e1.bias = b1;
    e1.out[0] = H;
    e1.out_ld[0] = F;
    e1.seg_cols = F;
    e1.st = st;
    e1.layer_idx = -1;
    Epi e2 = fin;
    e2.bias = b2;

    const double flops = 4.0 * M * D * F;
    const double io = static_cast<double>(M) * D * (2 + 4 + 4 + 2);  // A, resid, xout, ln
    float t_fused = time_it([&] { ffn_tc(A, D, W1t, W2t, M, D, F, fin, 0); }, iters);
    CK(cudaGetLastError());
    float t1 = time_it([&] { gemm_tc(A, D, W1t, D, M, F, D, e1, 0); }, iters);
    float t2 = time_it([&] { gemm_tc(H, F, W2t, F, M, D, F, e2, 0); }, iters);
    CK(cudaDeviceSynchronize());
    std::printf("{\"ablate\": %d, \"M\": %d, \"D\": %d, \"F\": %d, \"fused_us\": %.1f, \"fused_tflops\": %.1f, "
                "\"fused_io_gbs\": %.0f, \"ffn1_us\": %.1f, \"ffn2_us\": %.1f, \"unfused_tflops\": %.1f}\n",
                DCAT_FFN_ABLATE, M, D, F, t_fused, flops / t_fused * 1e-6, io / t_fused * 1e-3, t1, t2,
                flops / (t1 + t2) * 1e-6);
#if DCAT_FFN_TRACE
    ffn_trace_reset();
    ffn_tc(A, D, W1t, W2t, M, D, F, fin, 0);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> tr(8192);
    const int n = ffn_trace_read(tr.data(), 8192);
    std::printf("TRACE");
    for (int k = 0; k < n; k++)
        std::printf(" %llu:%llu:%llu", tr[k] >> 16, (tr[k] >> 8) & 255, tr[k] & 255);
    std::printf("\n");
#endif
    return 0;
}
