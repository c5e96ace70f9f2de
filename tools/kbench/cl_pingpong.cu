// cl_pingpong.cu — latency of one cross-CTA mbarrier hop inside a CTA pair (not part of the
// product): CTA 0 arrives remotely on CTA 1's barrier, CTA 1 answers on CTA 0's, N round trips.
// Variants: release.cluster arrive + acquire.cluster try_wait (what the pair kernels use),
// and the same with a relaxed arrive.
#include <cstdio>

#include "../../paper_2507_12704_b200/csrc/ptx.cuh"

using namespace dcat;

__device__ __forceinline__ void arrive_relaxed_cl(uint32_t cl_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}

template <int RELAXED>
__global__ void __cluster_dims__(2, 1, 1) k_pingpong(int n, unsigned long long* out) {
    __shared__ uint64_t bar;
    const uint32_t rank = ptx::cluster_rank();
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    ptx::cluster_sync();
    if (threadIdx.x == 0) {
        const uint32_t peer_bar = ptx::mapa(ptx::smem_u32(&bar), rank ^ 1);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < n; i++) {
            if (rank == 0) {
                if (RELAXED) arrive_relaxed_cl(peer_bar);
                else ptx::mbar_arrive_cl(peer_bar);
                ptx::mbar_wait_cl(&bar, i & 1);
            } else {
                ptx::mbar_wait_cl(&bar, i & 1);
                if (RELAXED) arrive_relaxed_cl(peer_bar);
                else ptx::mbar_arrive_cl(peer_bar);
            }
        }
        if (blockIdx.x == 0) out[RELAXED] = (clock64() - t0) / n;
    }
    __syncwarp();
    ptx::cluster_sync();
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    k_pingpong<0><<<2, 32>>>(1000, d);
    k_pingpong<1><<<2, 32>>>(1000, d);
    cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    std::printf("{\"round_trip_clk_release\": %llu, \"round_trip_clk_relaxed\": %llu, \"err\": \"%s\"}\n", h[0], h[1],
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
