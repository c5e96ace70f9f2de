// l2_stream.cu — TMA streaming probe (not part of the product): CTAs pull 16 KB boxes through
// an S-stage mbarrier ring, the access pattern of the FFN weight stream.
//   mode 0: every CTA reads the same 1 MB in the same order (the FFN's W1/W2 stream)
//   mode 1: same 1 MB, each CTA starting at a different 16 KB block (staggered)
//   mode 2: each CTA reads its own 1 MB region (no sharing)
//   mode 3: as mode 0 with 1-D bulk copies (no tensor map), each box as `pieces` copies
//   mode 4: CTA pairs as in the pair FFN: each CTA loads its own box with the .cta_group::2 TMA,
//           completion on the leader CTA's mbarrier (expect_tx from both); the leader frees the
//           slot for both (remote arrive on the peer's empty barrier)
//   mode 5: CTA pairs, each CTA loads its own box with plain TMA onto its own mbarrier; the peer
//           forwards "my half landed" to the leader with one remote arrive per slot
//   mode 6: as mode 4 with relaxed remote arrivals (expect_tx and the empty-slot arrivals)
//   mode 7: clusters of 2, but each CTA streams independently (plain TMA, own barriers)
//   mode 8: CTA pairs, plain TMA per CTA onto its own barrier; a forwarder warp in the peer
//           relays each completed slot to a second leader barrier (relaxed remote arrive); the
//           leader consumes when both are complete and frees the slot in both CTAs (relaxed)
//   mode 9: as mode 0 with C > 1 (multicast) but relaxed cross-CTA slot release
//   mode 10: CTA pairs, .cta_group::2 TMA of both CTAs onto the leader's barrier, ONLY the leader
//           arrives (expect_tx of both boxes, local); the peer issues its copy with no arrival
//           (the CUTLASS 2-SM pattern); the leader frees the slot in both CTAs (relaxed)
//   C > 1: clusters of C CTAs; each CTA loads 1/C of every box multicast to the whole cluster
// Prints per-CTA bytes/clk landed in shared memory and the mean TMA issue -> full latency.
#include <cuda.h>

#include <cstdio>
#include <cstring>

#include "../../paper_2507_12704_b200/csrc/ptx.cuh"

using namespace dcat;

constexpr int BOX_ROWS = 128, BOX_BYTES = BOX_ROWS * 128;  // [128 x 64] bf16, SW128

template <int S, int C>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap map, int mode, int iters,
                                                 int blocks_per_region, unsigned long long* out,
                                                 const uint8_t* gsrc, int pieces) {
    extern __shared__ uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[S], empty[S], fwd[S];
    const uint32_t rank = C > 1 ? ptx::cluster_rank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            ptx::mbar_init(&full[s], mode == 4 || mode == 6 || (mode == 5 && rank == 0) ? 2 : 1);
            ptx::mbar_init(&empty[s], (mode >= 4 && mode <= 8) || mode == 10 ? 1 : C);
            ptx::mbar_init(&fwd[s], 1);
        }
        ptx::fence_barrier_init();
    }
    if (C > 1) ptx::cluster_sync();
    if (C == 2 && mode == 8 && rank == 1 && threadIdx.x == 32) {
        for (int it = 0; it < iters; it++) {
            ptx::mbar_wait(&full[it % S], (it / S) & 1);
            ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&fwd[it % S]), 0));
        }
    }
    if (threadIdx.x == 0) {
    const int cid = blockIdx.x / C;
    const int region = mode == 2 ? cid : 0;
    const int start = mode == 1 ? (cid * 7) % blocks_per_region : 0;
    unsigned long long lat = 0, t_issue[S];
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters + S; it++) {
        const int s = it % S;
        if (C == 2 && mode == 8 && it >= S) {
            if (rank == 0) {
                ptx::mbar_wait(&full[s], ((it - S) / S) & 1);
                ptx::mbar_wait(&fwd[s], ((it - S) / S) & 1);
                lat += clock64() - t_issue[s];
                ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&empty[s]), 0));
                ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&empty[s]), 1));
            }
            ptx::mbar_wait_cl(&empty[s], ((it - S) / S) & 1);
        } else if (C == 2 && mode == 5 && it >= S) {
            if (rank == 0) {
                ptx::mbar_wait(&full[s], ((it - S) / S) & 1);  // own bytes + the peer's forward
                lat += clock64() - t_issue[s];
                ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&empty[s]), 0));
                ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&empty[s]), 1));
            } else {
                ptx::mbar_wait(&full[s], ((it - S) / S) & 1);
                ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&full[s]), 0));
            }
            ptx::mbar_wait_cl(&empty[s], ((it - S) / S) & 1);
        } else if (C == 2 && (mode == 4 || mode == 6 || mode == 10) && it >= S) {  // pair: the leader consumes both halves and frees the slot in both CTAs
            if (rank == 0) {
                ptx::mbar_wait(&full[s], ((it - S) / S) & 1);
                lat += clock64() - t_issue[s];
                if (mode == 6 || mode == 10) {
                    ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&empty[s]), 0));
                    ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&empty[s]), 1));
                } else {
                    ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&empty[s]), 0));
                    ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&empty[s]), 1));
                }
            }
            ptx::mbar_wait_cl(&empty[s], ((it - S) / S) & 1);
        } else if (it >= S) {  // consume the box issued S iterations ago, then free the slot cluster-wide
            ptx::mbar_wait(&full[s], ((it - S) / S) & 1);
            lat += clock64() - t_issue[s];
            if (C > 1 && mode != 7) {
                for (int r = 0; r < C; r++) {
                    if (mode == 9) ptx::mbar_arrive_cl_relaxed(ptx::mapa(ptx::smem_u32(&empty[s]), r));
                    else ptx::mbar_arrive_cl(ptx::mapa(ptx::smem_u32(&empty[s]), r));
                }
                ptx::mbar_wait_cl(&empty[s], ((it - S) / S) & 1);
            }
        }
        if (it < iters) {
            // pair modes: the peer streams the other half of the region, as the pair FFN's halves
            const int half = (((mode >= 4 && mode <= 8) || mode == 10) && rank == 1) ? blocks_per_region / 2 : 0;
            const int blk = (start + it + half) % blocks_per_region;
            const int row0 = (region * blocks_per_region + blk) * BOX_ROWS;
            if (C == 2 && mode == 10) {
                const uint32_t lead_full = ptx::mapa(ptx::smem_u32(&full[s]), 0);
                if (rank == 0) ptx::mbar_expect_tx(&full[s], 2 * BOX_BYTES);
                t_issue[s] = clock64();
                ptx::tma_load_2d_pair(ptx::smem_u32(ring + s * BOX_BYTES), &map, lead_full, 0, row0);
                continue;
            }
            if (C == 2 && (mode == 4 || mode == 6)) {
                const uint32_t lead_full = ptx::mapa(ptx::smem_u32(&full[s]), 0);
                if (mode == 6) ptx::mbar_expect_tx_cl_relaxed(lead_full, BOX_BYTES);
                else ptx::mbar_expect_tx_cl(lead_full, BOX_BYTES);
                t_issue[s] = clock64();
                ptx::tma_load_2d_pair(ptx::smem_u32(ring + s * BOX_BYTES), &map, lead_full, 0, row0);
                continue;
            }
            ptx::mbar_expect_tx(&full[s], BOX_BYTES);
            t_issue[s] = clock64();
            if ((C == 2 && (mode == 5 || mode == 8)) || mode == 7)
                ptx::tma_load_2d(ring + s * BOX_BYTES, &map, &full[s], 0, row0);
            else if (mode == 3)
                for (int p = 0; p < pieces; p++)
                    ptx::bulk_load(ring + s * BOX_BYTES + p * (BOX_BYTES / pieces),
                                   gsrc + static_cast<size_t>(row0) * 128 + p * (BOX_BYTES / pieces), BOX_BYTES / pieces,
                                   &full[s]);
            else if (C == 1)
                ptx::tma_load_2d(ring + s * BOX_BYTES, &map, &full[s], 0, row0);
            else
                ptx::tma_load_2d_mc(ring + s * BOX_BYTES + rank * (BOX_BYTES / C), &map, &full[s], 0,
                                    row0 + rank * (BOX_ROWS / C), static_cast<uint16_t>((1u << C) - 1));
        }
    }
    const unsigned long long t1 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = lat / iters;
    }
    __syncwarp();
    if (C > 1) ptx::cluster_sync();  // .aligned: the whole warp, converged
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int C>
void run(EncodeFn enc, void* buf, int mode, int grid, unsigned long long* d_out, int pieces = 1) {
    const int blocks_per_region = (1 << 20) / BOX_BYTES;  // 1 MB regions
    const int regions = mode == 2 ? grid / C : 1;
    CUtensorMap m;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(regions) * blocks_per_region * BOX_ROWS};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>((mode >= 4 && mode <= 8) || mode == 10 ? BOX_ROWS : BOX_ROWS / C)};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4096, smem = S * BOX_BYTES + 1024;
    cudaFuncSetAttribute(k_stream<S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; rep++) {
        if (rep == 1) cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k_stream<S, C>, m, mode, iters, blocks_per_region, d_out,
                           static_cast<const uint8_t*>(buf), pieces);
    }
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    // whole-kernel rate: every CTA's bytes over the wall time (co-resident CTAs add up per SM)
    const double tot_gbs = static_cast<double>(grid) * iters * BOX_BYTES / (ms * 1e-3) / 1e9;
    unsigned long long h[1024];
    cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
    double cyc = 0, lat = 0;
    int nm = 0;
    for (int i = 0; i < grid; i++) {
        if (((mode >= 4 && mode <= 8 && mode != 7) || mode == 10) && (i & 1)) continue;  // latency is measured by the leader
        cyc += h[2 * i];
        lat += h[2 * i + 1];
        nm++;
    }
    cyc /= nm;
    lat /= nm;
    std::printf(
        "{\"mode\": %d, \"pieces\": %d, \"cluster\": %d, \"grid\": %d, \"stages\": %d, \"bytes_per_clk_per_cta\": %.1f, "
        "\"latency_clk\": %.0f, \"kernel_GBps\": %.0f, \"per_SM_GBps\": %.1f, \"err\": \"%s\"}\n",
        mode, pieces, C, grid, S, static_cast<double>(iters) * BOX_BYTES / cyc, lat, tot_gbs, tot_gbs / 148,
        cudaGetErrorString(cudaGetLastError()));
    std::fflush(stdout);
}


// P producer warps in ONE CTA, each with its own S-stage ring and mbarriers, all streaming the
// same 1 MB: is the ~27 B/clk per CTA a per-CTA or a per-issuing-thread limit?
template <int S, int P>
__global__ void __launch_bounds__(32 * P, 1) k_stream_multi(const __grid_constant__ CUtensorMap map, int iters,
                                                          int blocks_per_region) {
    extern __shared__ uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[P][S];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < S; s++) ptx::mbar_init(&full[w][s], 1);
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if ((threadIdx.x & 31) != 0) return;
    uint8_t* my = ring + static_cast<size_t>(w) * S * BOX_BYTES;
    const int n = iters / P;
    for (int it = 0; it < n + S; it++) {
        const int s = it % S;
        if (it >= S) ptx::mbar_wait(&full[w][s], ((it - S) / S) & 1);
        if (it < n) {
            const int blk = (it * P + w) % blocks_per_region;
            ptx::mbar_expect_tx(&full[w][s], BOX_BYTES);
            ptx::tma_load_2d(my + s * BOX_BYTES, &map, &full[w][s], 0, blk * BOX_ROWS);
        }
    }
}

template <int S, int P>
void run_multi(EncodeFn enc, void* buf, int grid) {
    const int blocks_per_region = (1 << 20) / BOX_BYTES;
    CUtensorMap m;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(blocks_per_region) * BOX_ROWS};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BOX_ROWS)};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4096, smem = P * S * BOX_BYTES + 1024;
    cudaFuncSetAttribute(k_stream_multi<S, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_stream_multi<S, P><<<grid, 32 * P, smem>>>(m, iters, blocks_per_region);
    cudaEventRecord(e0);
    k_stream_multi<S, P><<<grid, 32 * P, smem>>>(m, iters, blocks_per_region);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = static_cast<double>(grid) * iters * BOX_BYTES / (ms * 1e-3) / 1e9;
    std::printf("{\"multi_producer\": %d, \"stages_each\": %d, \"grid\": %d, \"kernel_GBps\": %.0f, \"per_SM_GBps\": %.1f, \"err\": \"%s\"}\n",
                P, S, grid, gbs, gbs / 148, cudaGetErrorString(cudaGetLastError()));
    std::fflush(stdout);
}

// One producer WARP, S-slot ring of 16 KB slots, each slot loaded as NL boxes of 128 / NL rows
// issued by NL different lanes: does splitting a slot across issuing threads raise the rate at a
// fixed number of bytes in flight (the layer tail's ring is capped at 4 x 16 KB by shared memory)?
template <int S, int NL>
__global__ void __launch_bounds__(32, 1) k_stream_lanes(const __grid_constant__ CUtensorMap map, int iters,
                                                       int blocks_per_region) {
    extern __shared__ uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[S];
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        for (int s = 0; s < S; s++) ptx::mbar_init(&full[s], 1);
        ptx::fence_barrier_init();
    }
    __syncwarp();
    for (int it = 0; it < iters + S; it++) {
        const int s = it % S;
        if (it >= S) ptx::mbar_wait(&full[s], ((it - S) / S) & 1);
        __syncwarp();
        if (it < iters) {
            const int blk = it % blocks_per_region;
            if (lane == 0) ptx::mbar_expect_tx(&full[s], BOX_BYTES);
            __syncwarp();
            if (lane < NL)
                ptx::tma_load_2d(ring + s * BOX_BYTES + lane * (BOX_BYTES / NL), &map, &full[s], 0,
                                 blk * BOX_ROWS + lane * (BOX_ROWS / NL));
        }
    }
}

template <int S, int NL>
void run_lanes(EncodeFn enc, void* buf, int grid) {
    const int blocks_per_region = (1 << 20) / BOX_BYTES;
    CUtensorMap m;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(blocks_per_region) * BOX_ROWS};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BOX_ROWS / NL)};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4096, smem = S * BOX_BYTES + 1024;
    cudaFuncSetAttribute(k_stream_lanes<S, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_stream_lanes<S, NL><<<grid, 32, smem>>>(m, iters, blocks_per_region);
    cudaEventRecord(e0);
    k_stream_lanes<S, NL><<<grid, 32, smem>>>(m, iters, blocks_per_region);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = static_cast<double>(grid) * iters * BOX_BYTES / (ms * 1e-3) / 1e9;
    std::printf("{\"lanes_per_slot\": %d, \"stages\": %d, \"grid\": %d, \"kernel_GBps\": %.0f, \"per_SM_GBps\": %.1f, \"err\": \"%s\"}\n",
                NL, S, grid, gbs, gbs / 148, cudaGetErrorString(cudaGetLastError()));
    std::fflush(stdout);
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    void* buf;
    cudaMalloc(&buf, 448ull << 20);
    cudaMemset(buf, 0, 448ull << 20);
    unsigned long long* d_out;
    cudaMalloc(&d_out, 1024 * sizeof(unsigned long long));
    run<4, 1>(enc, buf, 0, 148, d_out);
    run<6, 1>(enc, buf, 0, 148, d_out);
    // two CTAs per SM (296 CTAs, 6 x 16 KB each): is ~27 B/clk a per-SM or a per-issuer limit?
    run<6, 1>(enc, buf, 0, 296, d_out);
    run<4, 1>(enc, buf, 0, 444, d_out);
    run<6, 1>(enc, buf, 2, 296, d_out);
    run_multi<8, 1>(enc, buf, 148);
    run_multi<4, 2>(enc, buf, 148);
    run_multi<6, 2>(enc, buf, 148);
    run_multi<3, 4>(enc, buf, 148);
    run_multi<2, 4>(enc, buf, 148);
    run_lanes<4, 1>(enc, buf, 148);
    run_lanes<4, 2>(enc, buf, 148);
    run_lanes<4, 4>(enc, buf, 148);
    run_lanes<4, 8>(enc, buf, 148);
    run_lanes<6, 1>(enc, buf, 148);
    run_lanes<6, 4>(enc, buf, 148);
    return 0;
}
