// tmem_bw.cu — TMEM -> register load bandwidth probe (tcgen05.ld.32x32b.x32), not part of the product.
// Each CTA allocates 512 TMEM columns; W warps (w % 4 = lane quadrant) each load 32 columns per
// instruction, sweeping the columns REPS times. Prints bytes/cycle per SM for W = 4, 8, 16.
#include <cstdio>

#include "../../paper_2507_12704_b200/csrc/ptx.cuh"

using namespace dcat;

template <int W>
__global__ void __launch_bounds__(W * 32, 1) k_tmem_bw(unsigned long long* cycles, float* sink, int reps) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const int cpw = 512 / (W / 4);  // columns owned by this warp
    const int col0 = (warp >> 2) * cpw;
    float acc = 0.f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        for (int c = 0; c < cpw; c += 32) {
            uint32_t v[32];
            DCAT_TMEM_LD32(base + col0 + c, v);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++) acc += __uint_as_float(v[i]);
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int W>
void run(unsigned long long* d_cyc, float* sink) {
    const int reps = 64;
    k_tmem_bw<W><<<148, W * 32>>>(d_cyc, sink, reps);
    k_tmem_bw<W><<<148, W * 32>>>(d_cyc, sink, reps);
    cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, d_cyc, sizeof(c), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; i++) avg += c[i];
    avg /= 148;
    const double bytes = 128.0 * 512 * 4 * reps;  // whole TMEM, reps times
    std::printf("{\"warps\": %d, \"cycles\": %.0f, \"bytes_per_cycle_per_sm\": %.1f, \"err\": \"%s\"}\n", W, avg,
                bytes / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d_cyc;
    float* sink;
    cudaMalloc(&d_cyc, 148 * sizeof(unsigned long long));
    cudaMalloc(&sink, 148 * 512 * sizeof(float));
    run<4>(d_cyc, sink);
    run<8>(d_cyc, sink);
    run<16>(d_cyc, sink);
    return 0;
}
