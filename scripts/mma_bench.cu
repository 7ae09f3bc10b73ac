// Microbenchmark: cycles per tcgen05.mma (kind::f16, SS operands from smem, no loads) for
// 1-CTA / 2-CTA and N = 128 / 256, issue loop with 64-bit descriptor adds vs precomputed
// 32-bit low halves.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2605_08523_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ffg;

template <int CG, int N, int STYLE>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        if (CG == 2) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = umma_idesc_f16(0, 128 * CG, N);
    long long t0 = 0, t1 = 0;
    if (warp == 0 && rank == 0) {
        const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
        const uint32_t lo0 = (uint32_t)d0, hi0 = (uint32_t)(d0 >> 32);
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (STYLE == 0) {
                    if (elect_one_sync()) {
                        const uint64_t da = d0 + (kk * 32 >> 4);
                        const uint64_t db = d0 + ((16384 + kk * 32) >> 4);
                        if (CG == 2) umma_f16_pair(tmem, da, db, idesc, 1u);
                        else umma_f16(tmem, da, db, idesc, 1u);
                    }
                    __syncwarp();
                } else {
                    const uint32_t la = lo0 + (kk * 32 >> 4), lb = lo0 + ((16384 + kk * 32) >> 4);
                    if (elect_one_sync()) {
                        if (CG == 2)
                            asm volatile(
                                "{\n .reg .b64 a, b;\n mov.b64 a, {%1, %3};\n mov.b64 b, {%2, %3};\n"
                                " tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %4, 1;\n}" ::"r"(tmem),
                                "r"(la), "r"(lb), "r"(hi0), "r"(idesc) : "memory");
                        else
                            asm volatile(
                                "{\n .reg .b64 a, b;\n mov.b64 a, {%1, %3};\n mov.b64 b, {%2, %3};\n"
                                " tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %4, 1;\n}" ::"r"(tmem),
                                "r"(la), "r"(lb), "r"(hi0), "r"(idesc) : "memory");
                    }
                    __syncwarp();
                }
            }
        }
        if (elect_one_sync()) {
            if (CG == 2) umma_commit_pair(&bar); else umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    } else if (CG == 2 && rank == 1 && warp == 0) {
        mbar_wait(&bar, 0);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
    }
}

template <int CG, int N, int STYLE>
void run(const char* name) {
    auto k = mma_bench<CG, N, STYLE>;
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    cudaMallocManaged(&out, 148 * 8);
    const int iters = 4096;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
        cudaLaunchKernelEx(&cfg, k, iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    }
    double cyc = 0;
    int cnt = 0;
    for (int b = 0; b < 148; b += CG) { cyc += out[b]; ++cnt; }
    cyc /= cnt;
    const double per = cyc / (iters * 4.0);
    // per-SM MACs per instruction: 128 x N x 16 (each CTA of a pair computes 128 rows)
    const double nominal = 128.0 * N * 16 / 4096.0;  // cycles at 4096 MAC/clk/SM
    printf("%-28s %8.1f cyc/MMA  nominal %5.1f  -> %.0f%% of nominal\n", name, per, nominal, 100.0 * nominal / per);
    cudaFree(out);
}


// Pipeline variant: a producer warp and the MMA warp hand stages back and forth through
// full/empty mbarriers (no data movement), MMAs committed per stage like the real kernel.
template <int CG, int N, int STAGES, int MMAS_PER_STAGE>
__global__ void __launch_bounds__(128, 1) mma_pipe(int stages_total, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES], done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], CG); mbar_init(&empty[i], 1); }
        mbar_init(&done, 1);
        fence_barrier_init();
    }
    if (warp == 1) { if (CG == 2) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512); }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = umma_idesc_f16(0, 128 * CG, N);
    if (warp == 0 && lane == 0) {
        for (int it = 0; it < stages_total; ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            mbar_arrive_cluster(mapa_shared(smem_u32(&full[s]), 0));
        }
    } else if (warp == 1 && rank == 0) {
        const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
        const long long t0 = clock64();
        for (int it = 0; it < stages_total; ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            tc_fence_after();
            if (elect_one_sync()) {
#pragma unroll
                for (int kk = 0; kk < MMAS_PER_STAGE; ++kk) {
                    const uint64_t da = d0 + ((s * 8192 + (kk & 3) * 32) >> 4);
                    const uint64_t db = d0 + ((s * 8192 + 4096 + (kk & 3) * 32) >> 4);
                    if (CG == 2) umma_f16_pair(tmem, da, db, idesc, 1u); else umma_f16(tmem, da, db, idesc, 1u);
                }
                if (CG == 2) umma_commit_pair(&empty[s]); else umma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one_sync()) { if (CG == 2) umma_commit_pair(&done); else umma_commit(&done); }
        __syncwarp();
        mbar_wait(&done, 0);
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    } else if (CG == 2 && rank == 1 && warp == 1) {
        mbar_wait(&done, 0);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 1) { tc_fence_after(); if (CG == 2) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512); }
}

template <int CG, int N, int STAGES, int MPS>
void runp(const char* name) {
    auto k = mma_pipe<CG, N, STAGES, MPS>;
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    cudaMallocManaged(&out, 148 * 8);
    const int st = 4096;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
        cudaLaunchKernelEx(&cfg, k, st, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    }
    double cyc = 0; int cnt = 0;
    for (int b = 0; b < 148; b += CG) { cyc += out[b]; ++cnt; }
    cyc /= cnt;
    const double per = cyc / (st * (double)MPS);
    const double nominal = 128.0 * N * 16 / 4096.0;
    printf("%-34s %8.1f cyc/MMA  nominal %5.1f  -> %.0f%%\n", name, per, nominal, 100.0 * nominal / per);
    cudaFree(out);
}

int main() {
    run<1, 128, 0>("1cta N=128 desc64");
    run<1, 128, 1>("1cta N=128 desc32");
    run<1, 256, 0>("1cta N=256 desc64");
    run<1, 256, 1>("1cta N=256 desc32");
    run<2, 128, 0>("2cta N=128 desc64");
    run<2, 128, 1>("2cta N=128 desc32");
    run<2, 256, 0>("2cta N=256 desc64");
    run<2, 256, 1>("2cta N=256 desc32");
    runp<2, 128, 6, 4>("pipe 2cta N=128 S=6 x4 (bf16)");
    runp<2, 128, 3, 12>("pipe 2cta N=128 S=3 x12 (f32e)");
    runp<2, 128, 4, 4>("pipe 2cta N=128 S=4 x4");
    runp<1, 128, 6, 4>("pipe 1cta N=128 S=6 x4");
    runp<2, 256, 4, 4>("pipe 2cta N=256 S=4 x4");
    return 0;
}
