// Microbenchmark: does TMA multicast raise the operand bandwidth an SM receives above the L2 (LTS)
// throughput cap?  Every CTA streams 32 KB stages (four 64 x 64 bf16 SW128 boxes, the K2 operand
// box shape) from an L2-resident 16 MB buffer through a 4-stage full/empty mbarrier ring:
//   U  (unicast)   each CTA loads its own four boxes;
//   M2 (multicast) clusters of 2: CTA r loads boxes 2r, 2r+1 to both CTAs (same bytes per CTA);
//   M4 (multicast) clusters of 4: CTA r loads box r to all four.
// 4- or 6-stage rings (128 / 192 KB in flight per SM).
// The consumer releases a stage with a plain (CTA-scope) mbarrier arrive on every CTA of the cluster; a
// .release.cluster arrive costs ~1000 cycles per stage and caps any mode at ~30 B/cycle per SM.
// Prints received bytes per SM per cycle and the aggregate (B/cycle) per mode.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mc_bench mc_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr int kStageBytes = 32768;     // 32 KB
constexpr int kRows = 131072;            // 16 MB of 64-column bf16 rows

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t a, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(a), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint32_t a, uint32_t ph) { while (!try_wait(a, ph)) {} }

template <int CS, int kStages, int BR = 64, int NP = 1, int F = 0, int NT = 99, int W = 0>
__global__ void __launch_bounds__(256, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* gbuf, int T,
                                                        unsigned long long* cyc) {
    constexpr int kBox = BR * 128, NB = kStageBytes / kBox;
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const uint32_t rank = CS > 1 ? cta_rank() : 0;
    const int cluster = blockIdx.x / CS;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1 + 32 * W));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(CS));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (CS > 1) cluster_sync(); else __syncthreads();
    // tiles of a CTA (unicast) or of a cluster (multicast): distinct per CTA / cluster, wrapping in the buffer
    const int owner = CS > 1 ? cluster : blockIdx.x;
    long long t0 = clock64();
    if (threadIdx.x % 32 == 0 && threadIdx.x / 32 < NP) {
        for (int t = threadIdx.x / 32; t < T; t += NP) {
            const int s = t % kStages;
            wait(su32(&empty[s]), ((t / kStages) & 1) ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                         "r"(min(NT, NB) * kBox) : "memory");
            const int row0 = (int)(((long long)owner * 977 + (long long)t * 4 * 64) % (kRows - 256));
            for (int b = 0; b < min(NT, NB); ++b) {
                if (F == 2) {  // 1-D bulk copy of the same bytes (contiguous rows)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        ::"r"(su32(smem + s * kStageBytes + b * kBox)), "l"(gbuf + (size_t)(row0 + BR * b) * 128),
                        "r"(kBox), "r"(su32(&full[s])) : "memory");
                } else if (CS == 1) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(smem + s * kStageBytes + b * kBox)),
                        "l"(&tm), "r"(su32(&full[s])), "r"(0), "r"(row0 + BR * b) : "memory");
                } else if (b / (NB / CS) == (int)rank) {
                    const uint16_t mask = (uint16_t)((1u << CS) - 1);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(smem + s * kStageBytes + b * kBox)),
                        "l"(&tm), "r"(su32(&full[s])), "r"(0), "r"(row0 + BR * b), "h"(mask) : "memory");
                }
            }
        }
    } else if (W > 0 && threadIdx.x >= 32 * NP && threadIdx.x < 32 * (NP + W)) {
        // cp.async (LDGSTS) 16-byte chunks of boxes NT.. into the SW128 layout the TMA would produce
        const int ct = threadIdx.x - 32 * NP;
        constexpr int kChunks = (NB - (NT < NB ? NT : NB)) * kBox / 16;
        for (int t = 0; t < T; ++t) {
            const int s = t % kStages;
            wait(su32(&empty[s]), ((t / kStages) & 1) ^ 1);
            const int row0 = (int)(((long long)owner * 977 + (long long)t * 4 * 64) % (kRows - 256));
            const uint32_t base = su32(smem + s * kStageBytes + (NT < NB ? NT : NB) * kBox);
            const uint8_t* src = gbuf + (size_t)(row0 + BR * (NT < NB ? NT : NB)) * 128;
            for (int c = ct; c < kChunks; c += 32 * W) {
                const int row = c >> 3, ch = c & 7;
                const uint32_t dst = base + row * 128 + ((ch ^ (row & 7)) << 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + (size_t)c * 16) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
        }
    } else if (threadIdx.x == 32 * (NP + W)) {
        for (int t = 0; t < T; ++t) {
            const int s = t % kStages;
            wait(su32(&full[s]), (t / kStages) & 1);
            if (CS == 1) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            } else {
                for (int r = 0; r < CS; ++r)
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(
                                     mapa(su32(&empty[s]), r)) : "memory");
            }
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (CS > 1) cluster_sync();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int CS, int kStages, int BR = 64, int NP = 1, int F = 0, int NT = 99, int W = 0>
int run(const CUtensorMap& tm, int grid, int T, const char* name, const uint8_t* gbuf = nullptr) {
    const int smem = kStages * kStageBytes + 1024;
    CK(cudaFuncSetAttribute(stream_kernel<CS, kStages, BR, NP, F, NT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, grid * sizeof(unsigned long long)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * (NP + W + 1));
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {  // first run warms L2
        cudaEventRecord(a);
        CK(cudaLaunchKernelEx(&cfg, stream_kernel<CS, kStages, BR, NP, F, NT, W>, tm, gbuf, T, d));
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(grid);
    cudaMemcpy(h.data(), d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (auto v : h) {
        mx = v > mx ? v : mx;
        sum += v;
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double bytes_sm = (double)T * kStageBytes;
    printf("%-3s TMA boxes %d copy warps %d flavor %d producers %d box %3d stages %d grid %3d  per-SM %.1f B/cyc (mean cycles)  aggregate received %.0f B/cyc  L2-read %.0f B/cyc  (%.3f ms)\n",
           name, NT < 4 ? NT : 4, W, F, NP, BR, kStages, grid, bytes_sm / (sum / grid), bytes_sm * grid / mx, bytes_sm * grid / CS / mx, ms);
    cudaFree(d);
    return 0;
}

int main() {
    void* buf;
    CK(cudaMalloc(&buf, (size_t)kRows * 64 * 2));
    CK(cudaMemset(buf, 0, (size_t)kRows * 64 * 2));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm, tm128;
    cuuint64_t dims[2] = {64, (cuuint64_t)kRows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, 64}, box128[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    r = r != CUDA_SUCCESS ? r : ((EncodeFn)fn)(&tm128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box128, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    CUtensorMap tmn;
    r = ((EncodeFn)fn)(&tmn, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1;
    const uint8_t* g = (const uint8_t*)buf;
    const int T = 4000;
    if (run<1, 4>(tm, 148, T, "U", g)) return 1;
    if (run<1, 6>(tm, 148, T, "U", g)) return 1;
    if (run<1, 4>(tm, 37, T, "U", g)) return 1;
    if (run<1, 3>(tm, 296, T, "U", g)) return 1;
    if (run<2, 4>(tm, 148, T, "M2", g)) return 1;
    if (run<2, 6>(tm, 148, T, "M2", g)) return 1;
    if (run<4, 6>(tm, 144, T, "M4", g)) return 1;
    return 0;
}
