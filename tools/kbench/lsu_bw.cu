// lsu_bw.cu — per-SM LSU bandwidth against L2-resident data (not part of the product).
// One CTA of 512 threads per SM: 16-byte ld.global (all CTAs read the same 1 MB, L2-resident)
// or 16-byte st.global (each CTA writes its own 256 KB region); bytes/clk per SM, for comparison
// with the ~27 B/clk of the TMA engine (l2_stream.cu).
#include <cstdio>

__global__ void __launch_bounds__(512, 1) k_ld(const uint4* __restrict__ src, int n16, int reps, unsigned long long* out,
                                               uint4* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = threadIdx.x; i < n16; i += blockDim.x) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(src + i));
            acc.x ^= v.x;
            acc.y ^= v.y;
            acc.z ^= v.z;
            acc.w ^= v.w;
        }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (acc.x == 0x12345678u) sink[threadIdx.x] = acc;
}
__global__ void __launch_bounds__(512, 1) k_st(uint4* dst, int n16, int reps, unsigned long long* out) {
    uint4* d = dst + static_cast<size_t>(blockIdx.x) * n16;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = threadIdx.x; i < n16; i += blockDim.x) d[i] = make_uint4(r, i, 1, 2);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    const int n_ld = (1 << 20) / 16, n_st = (256 << 10) / 16, reps = 64;
    uint4 *src, *dst, *sink;
    unsigned long long* d_out;
    cudaMalloc(&src, 1 << 20);
    cudaMemset(src, 1, 1 << 20);
    cudaMalloc(&dst, 148ull * (256 << 10));
    cudaMalloc(&sink, 512 * 16);
    cudaMalloc(&d_out, 148 * 8);
    unsigned long long h[148];
    for (int grid : {148, 8}) {
        k_ld<<<grid, 512>>>(src, n_ld, 2, d_out, sink);
        k_ld<<<grid, 512>>>(src, n_ld, reps, d_out, sink);
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        double c = 0;
        for (int i = 0; i < grid; i++) c += h[i];
        c /= grid;
        std::printf("{\"op\": \"ld.global.cg\", \"grid\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", grid,
                    static_cast<double>(reps) * (1 << 20) / c);
        k_st<<<grid, 512>>>(dst, n_st, 2, d_out);
        k_st<<<grid, 512>>>(dst, n_st, reps, d_out);
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        c = 0;
        for (int i = 0; i < grid; i++) c += h[i];
        c /= grid;
        std::printf("{\"op\": \"st.global\", \"grid\": %d, \"bytes_per_clk_per_sm\": %.1f, \"err\": \"%s\"}\n", grid,
                    static_cast<double>(reps) * (256 << 10) / c, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
