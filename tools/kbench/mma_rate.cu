// mma_rate.cu — issue-rate probe of tcgen05.mma kind::f16 on one B200 (not part of the product).
// One persistent CTA per SM; one thread issues `iters` x 4 MMAs (a 64-deep K block) from
// operands that sit in shared memory (SS) or with A in TMEM (TS), no loads, commit + wait at
// the end. Reports chip TF/s per shape, i.e. the ceiling of the layer-tail's MMA phases when
// nothing else limits them.
//   variant 0: SS M128 N256    1: SS M128 N128    2: SS M128 N64
//   variant 3: TS M128 N256    4: TS M128 N128
//   variant 5: SS cta_group::2 M256 N256 (CTA pair, leader issues)
//   variant 6: SS M128 N256, A and B re-read from two alternating stages (ring-like addresses)
#include <cstdio>
#include <cstdlib>

#include "../../paper_2507_12704_b200/csrc/ptx.cuh"

using namespace dcat;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

template <int V>
__global__ void k_rate(int iters, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t done;
    __shared__ uint32_t slot;
    constexpr bool PAIR = V == 5;
    constexpr int N = (V == 1 || V == 4) ? 128 : V == 2 ? 64 : 256;
    constexpr int M = PAIR ? 256 : 128;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = PAIR ? ptx::cluster_rank() : 0;
    // zero the operand tiles (finite inputs)
    for (int i = threadIdx.x; i < 2 * (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) {
        if (PAIR) ptx::tmem_alloc_pair(&slot, 512);
        else ptx::tmem_alloc(&slot, 512);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    if (PAIR) ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t a0 = ptx::smem_u32(sm), b0 = a0 + 2 * 16384;
        const uint32_t idesc = ptx::idesc_bf16(M, N);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            const int st = V == 6 ? (it & 1) : 0;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const uint64_t ad = ptx::sdesc_sw128(a0 + st * 16384 + k * 32);
                const uint64_t bd = ptx::sdesc_sw128(b0 + st * 32768 + k * 32);
                if constexpr (V == 3 || V == 4)
                    mma_ts(tmem, tmem + 256 + k * 8, bd, idesc, 1);
                else if constexpr (PAIR)
                    ptx::mma_bf16_pair(tmem, ad, bd, idesc, 1);
                else
                    ptx::mma_bf16(tmem, ad, bd, idesc, 1);
            }
        }
        if (PAIR) ptx::mma_commit_pair(&done);
        else ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
        const unsigned long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    if (PAIR && threadIdx.x == 0 && rank == 1) ptx::mbar_wait(&done, 0);
    ptx::tc_fence_before();
    __syncthreads();
    if (PAIR) ptx::cluster_sync();
    if (warp == 0) {
        ptx::tc_fence_after();
        if (PAIR) ptx::tmem_dealloc_pair(tmem, 512);
        else ptx::tmem_dealloc(tmem, 512);
    }
}

template <int V>
void run(int sms, int iters) {
    constexpr int N = (V == 1 || V == 4) ? 128 : V == 2 ? 64 : 256;
    constexpr int M = V == 5 ? 256 : 128;
    const int smem = 2 * (16384 + 32768) + 1024;
    CK(cudaFuncSetAttribute(k_rate<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, sms * sizeof(unsigned long long)));
    CK(cudaMemset(d, 0, sms * sizeof(unsigned long long)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = V == 5 ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; rep++) CK(cudaLaunchKernelEx(&cfg, k_rate<V>, iters, d));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k_rate<V>, iters, d));
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long h[256] = {0};
    CK(cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
    const double issuers = V == 5 ? sms / 2 : sms;
    const double flops = issuers * static_cast<double>(iters) * 4 * 2.0 * M * N * 16;
    const double per_mma_clk = static_cast<double>(mx) / (iters * 4.0);
    std::printf("{\"variant\": %d, \"M\": %d, \"N\": %d, \"ts\": %d, \"ctas\": %d, \"ms\": %.3f, \"tflops\": %.1f, "
                "\"clk_per_mma\": %.1f, \"flop_per_clk_per_sm\": %.0f}\n",
                V, M, N, (V == 3 || V == 4) ? 1 : 0, sms, ms, flops / (ms * 1e-3) / 1e12, per_mma_clk,
                2.0 * M * N * 16 / per_mma_clk / (V == 5 ? 2 : 1));
    CK(cudaFree(d));
}

int main(int argc, char** argv) {
    const int iters = argc > 1 ? std::atoi(argv[1]) : 20000;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    run<0>(sms, iters);
    run<1>(sms, iters);
    run<2>(sms, iters);
    run<3>(sms, iters);
    run<4>(sms, iters);
    run<5>(sms, iters);
    run<6>(sms, iters);
    return 0;
}
