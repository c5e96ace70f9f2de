// common.cuh — shared device helpers for the DCAT B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <mutex>
#include <set>
#include <string>
#include <utility>

namespace dcat {

// NVTX range around a host-side stage (API calls, GEMM / attention / tail launches): named spans
// in nsys / `ncu --nvtx` timelines; a no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

using bf16 = __nv_bfloat16;

// Error kinds raised on the device and turned into reference-style messages
// on the host (the reference's SEQFM_CHECKs, common.hpp:9-16).
enum ErrBits : int {
    ERR_ACTION = 1,      // segment_inputs: unknown action value   (model.cpp:525)
    ERR_SURFACE = 2,     // segment_inputs: unknown surface value  (model.cpp:526)
    ERR_POS_CTX = 4,     // segment_inputs: position exceeds max_len (model.cpp:534)
    ERR_POS_CAND = 8,    // candidate_inputs: position out of range (dcat.cpp:190)
    ERR_AGE = 16,        // ctx_features: negative age (finetune.cpp:214)
    ERR_RANGE = 32,      // row events outside the event pool
    ERR_NONFINITE = 64,  // non-finite activation (model.cpp:25-28, dcat.cpp:85-86)
};

// Device status block, read back once per call (after dedup) and once at the end.
struct Status {
    int err_bits;
    int err_row;          // first offending row (atomicMin)
    int err_val;          // offending value of err_row
    int nonfinite_layer;  // layer index + 1 of a non-finite activation (max)
    int collisions;       // rows whose 64-bit content hash collided
    int b_u;
    long long ctx_tokens;
    int ctx_tiles;
    int cross_tiles;
    int max_cnt;
    int pad[5];
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    // splitmix64 finalizer (rng.hpp:13-18)
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__device__ __forceinline__ float gelu_tanh(float x) {
    // tanh-form GELU (model.hpp:14-18)
    const float c = 0.7978845608028654f;
    float x3 = x * x * x;
    return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x3)));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

template <typename T>
struct ActIO;
template <>
struct ActIO<float> {
    static __device__ __forceinline__ float load(const float* p) { return *p; }
    static __device__ __forceinline__ void store(float* p, float v) { *p = v; }
};
template <>
struct ActIO<bf16> {
    static __device__ __forceinline__ float load(const bf16* p) { return __bfloat162float(*p); }
    static __device__ __forceinline__ void store(bf16* p, float v) { *p = __float2bfloat16_rn(v); }
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace dcat

// A failed runtime call also leaves its code as the thread's "last error" (non-sticky errors such as
// an invalid device ordinal): it is consumed here, so a later launch check does not report it again.
#define DCAT_CUDA_CHECK(expr)                                                               \
    do {                                                                                    \
        cudaError_t e__ = (expr);                                                           \
        if (e__ != cudaSuccess) {                                                           \
            (void)cudaGetLastError();                                                       \
            throw ::dcat::CudaError(std::string(#expr) + " (" + __FILE__ + ":" + std::to_string(__LINE__) + "): " + \
                                    cudaGetErrorString(e__));                                  \
        }                                                                                   \
    } while (0)

#define DCAT_LAUNCH_CHECK() DCAT_CUDA_CHECK(cudaGetLastError())


namespace dcat {
struct CudaError {
    std::string msg;
    explicit CudaError(std::string m) : msg(std::move(m)) {}
};
struct InvalidArg {
    std::string msg;
    int code;
    explicit InvalidArg(std::string m, int c = -1) : msg(std::move(m)), code(c) {}
};
// true when the calling thread has a current CUDA context (cuCtxGetCurrent through the runtime's
// driver entry point; the library does not link libcuda directly)
inline bool thread_has_context() {
    typedef int (*GetCur)(void**);
    static GetCur fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            (void)cudaGetLastError();
            return static_cast<GetCur>(nullptr);
        }
        return reinterpret_cast<GetCur>(p);
    }();
    if (!fn) return true;  // unknown: restore as if there were one
    void* ctx = nullptr;
    return fn(&ctx) == 0 && ctx != nullptr;
}
// Makes `dev` the current device for a scope and restores the caller's current device after it
// (the C ABI never leaves the calling thread on another GPU). dev < 0: no switch. A thread that
// had no current context is left without a restore (restoring its default device 0 would create a
// context on GPU 0 in a process that only drives another GPU).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (!thread_has_context() || cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            (void)cudaGetLastError();
        }
        if (dev >= 0 && dev != prev) DCAT_CUDA_CHECK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};
// Teardown form (destroy entry points, possibly run from static destructors at process exit when
// the runtime may already be unloading): never throws, ignores and clears errors.
struct DeviceScopeNoThrow {
    int prev = -1;
    explicit DeviceScopeNoThrow(int dev) {
        if (!thread_has_context() || cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
        (void)cudaGetLastError();
    }
    ~DeviceScopeNoThrow() {
        if (prev >= 0) cudaSetDevice(prev);
        (void)cudaGetLastError();
    }
    DeviceScopeNoThrow(const DeviceScopeNoThrow&) = delete;
    DeviceScopeNoThrow& operator=(const DeviceScopeNoThrow&) = delete;
};
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// belongs to the device context, so a process driving several GPUs (csrc/multi.cu) sets it on every
// device it launches on
inline void set_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    DCAT_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({func, dev}).second)
        DCAT_CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace dcat
