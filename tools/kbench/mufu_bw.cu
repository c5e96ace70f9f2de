// mufu_bw.cu — throughput probe: ex2.approx (MUFU) vs a degree-3 polynomial exp2 on the FMA pipe,
// and tanh.approx. Not part of the product. Prints ops/clk/SM.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float tanhx(float x) {
    float y;
    asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2h2(float x) {  // two exp2 in one f16x2 op (result: sum as float)
    uint32_t h, r;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x), "f"(x - 0.25f));
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
    __half2 v = *reinterpret_cast<__half2*>(&r);
    return __low2float(v) + __high2float(v);
}
__device__ __forceinline__ float ex2bf2(float x) {
    uint32_t h, r;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x), "f"(x - 0.25f));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(h));
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&r);
    return __low2float(v) + __high2float(v);
}
// 2^x for x <= 0: Cody-Waite split, minimax cubic on [0, 1), exponent add
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -127.f);
    const float fl = floorf(x);
    const float f = x - fl;
    float p = fmaf(f, 0.0790199f, 0.2243545f);
    p = fmaf(p, f, 0.6963492f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (static_cast<int>(fl) << 23));
}

template <int MODE>
__global__ void k(float* out, int iters, unsigned long long* cyc) {
    float a0 = -threadIdx.x * 1e-3f, a1 = a0 - 0.1f, a2 = a0 - 0.2f, a3 = a0 - 0.3f;
    float a4 = a0 - 0.4f, a5 = a0 - 0.5f, a6 = a0 - 0.6f, a7 = a0 - 0.7f;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (MODE == 0) {
            a0 = ex2(a0) - 1.5f; a1 = ex2(a1) - 1.5f; a2 = ex2(a2) - 1.5f; a3 = ex2(a3) - 1.5f;
            a4 = ex2(a4) - 1.5f; a5 = ex2(a5) - 1.5f; a6 = ex2(a6) - 1.5f; a7 = ex2(a7) - 1.5f;
        } else if (MODE == 1) {
            a0 = ex2_poly(a0) - 1.5f; a1 = ex2_poly(a1) - 1.5f; a2 = ex2_poly(a2) - 1.5f; a3 = ex2_poly(a3) - 1.5f;
            a4 = ex2_poly(a4) - 1.5f; a5 = ex2_poly(a5) - 1.5f; a6 = ex2_poly(a6) - 1.5f; a7 = ex2_poly(a7) - 1.5f;
        } else if (MODE == 3) {
            a0 = ex2h2(a0) - 1.5f; a1 = ex2h2(a1) - 1.5f; a2 = ex2h2(a2) - 1.5f; a3 = ex2h2(a3) - 1.5f;
            a4 = ex2h2(a4) - 1.5f; a5 = ex2h2(a5) - 1.5f; a6 = ex2h2(a6) - 1.5f; a7 = ex2h2(a7) - 1.5f;
        } else if (MODE == 4) {
            a0 = ex2bf2(a0) - 1.5f; a1 = ex2bf2(a1) - 1.5f; a2 = ex2bf2(a2) - 1.5f; a3 = ex2bf2(a3) - 1.5f;
            a4 = ex2bf2(a4) - 1.5f; a5 = ex2bf2(a5) - 1.5f; a6 = ex2bf2(a6) - 1.5f; a7 = ex2bf2(a7) - 1.5f;
        } else {
            a0 = tanhx(a0) - 0.5f; a1 = tanhx(a1) - 0.5f; a2 = tanhx(a2) - 0.5f; a3 = tanhx(a3) - 0.5f;
            a4 = tanhx(a4) - 0.5f; a5 = tanhx(a5) - 0.5f; a6 = tanhx(a6) - 0.5f; a7 = tanhx(a7) - 0.5f;
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int MODE>
void run(const char* name, float* out, unsigned long long* cyc) {
    const int iters = 4096, threads = 1024;
    k<MODE><<<148, threads>>>(out, iters, cyc);
    k<MODE><<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; i++) avg += c[i];
    avg /= 148;
    std::printf("{\"op\": \"%s\", \"ops_per_clk_per_sm\": %.2f}\n", name, 8.0 * iters * threads / avg);
}

int main() {
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
    run<0>("ex2.approx.ftz.f32", out, cyc);
    run<1>("ex2 cubic poly (FMA pipe)", out, cyc);
    run<2>("tanh.approx.f32", out, cyc);
    run<3>("ex2.approx.f16x2 (x2 results per op: ops counted as pairs)", out, cyc);
    run<4>("ex2.approx.ftz.bf16x2 (pairs)", out, cyc);
    return 0;
}
