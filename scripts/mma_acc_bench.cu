// Microbenchmark: tcgen05 pair MMA (cta_group::2, M=256, N=128, K=16, kind::f16) issue patterns of the
// K2 pair kernel's K-block, no loads (operands stay in shared memory), cycles per MMA:
//   P0  one accumulator, the same A and B every MMA
//   P1  normal-layer K-block: 4 x (A_hi.B_lo, A_lo.B_hi) then 4 x A_hi.B_hi, all into ONE accumulator
//   P2  the same 12 MMAs with A_hi.B_hi into a second accumulator
//   P3  exact-layer K-block: 4 x (A_hi.B_lo, A_lo.B_hi, A_lo.B_lo -> acc X; A_hi.B_hi -> acc H)
//   P4  one accumulator, per K16 step A_hi.B_lo, A_lo.B_hi, A_hi.B_hi
//   P5  one accumulator, 12 MMAs A_hi.B_hi only (descriptors change with the K16 step)
//   P6  P1 + the kernel's commits: multicast commit to an empty barrier per K-block, a slot commit
//       every two K-blocks
//   P7  P6 + the K-block's operands rotating over three 48 KB stages
//   P8  P7 + the issuer waits on a (completed) full barrier and fences per K-block, like the kernel
// and P1 / P3 / P8 again with pseudo-random operand values (hi in [-1, 1], lo ~2^-11 of it) instead of zeros;
// P8 with 16 more warps per CTA waiting on an mbarrier (spinning / suspend-hint try_wait), like the kernel's workers;
// P10 / P11: the normal layers' chunks (a fresh accumulator every two K-blocks, rotating over four slots / one slot).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2605_08523_b200/csrc mma_acc_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "ptx.cuh"
using namespace ffg;

constexpr uint32_t kAhi = 0, kAlo = 16384, kBhi = 32768, kBlo = 40960;

template <int P, int FILL = 0, int SPIN = 0>
__global__ void __launch_bounds__(640, 1) acc_bench(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, ebar[3], sbar[4], fbar[3], never;
    __shared__ uint32_t slot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 3; ++i) { mbar_init(&ebar[i], 1); mbar_init(&fbar[i], 1); }
        for (int i = 0; i < 4; ++i) mbar_init(&sbar[i], 1);
        mbar_init(&never, 1);
        stop = 0;
        fence_barrier_init();
    }
    if (FILL) {  // operands: pseudo-random binary16 values in [-1, 1] (hi) and ~2^-11 of that (lo)
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        for (int i = threadIdx.x; i < 3 * 49152 / 4; i += blockDim.x) {
            uint32_t h = (uint32_t)i * 2654435761u + 12345u * (blockIdx.x + 1);
            h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
            const float a = ((h & 0xffff) / 32768.0f) - 1.0f, b = ((h >> 16) / 32768.0f) - 1.0f;
            const bool lo = ((i * 4) % 49152) >= 16384 && ((i * 4) % 49152) < 32768;
            const __half2 v = __floats2half2_rn(lo ? a * 4.8828125e-4f : a, lo ? b * 4.8828125e-4f : b);
            w[i] = *reinterpret_cast<const uint32_t*>(&v);
        }
        __syncthreads();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) tmem_alloc_pair(&slot, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t t0a = slot, t1a = slot + 128;
    constexpr uint32_t idesc = umma_idesc_f16(0, 256, 128);
    if (warp == 0 && rank == 0) {
        const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
        auto D = [&](uint32_t off, int kk) { return d0 + ((off + kk * 32) >> 4); };
        const long long c0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (P == 8) {
                if (i == 0 && elect_one_sync()) {
                    for (int f = 0; f < 3; ++f) mbar_arrive(&fbar[f]);
                }
                __syncwarp();
                mbar_wait(&fbar[i % 3], 0);  // completed once: every later wait returns at once
                tc_fence_after();
            }
            if (elect_one_sync()) {
                if (P == 0) {
#pragma unroll
                    for (int j = 0; j < 12; ++j) umma_f16_pair(t0a, D(kAhi, 0), D(kBhi, 0), idesc, 1u);
                } else if (P == 1 || P == 2) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_pair(t0a, D(kAhi, kk), D(kBlo, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(kAlo, kk), D(kBhi, kk), idesc, 1u);
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_f16_pair(P == 1 ? t0a : t1a, D(kAhi, kk), D(kBhi, kk), idesc, 1u);
                } else if (P == 3) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_pair(t0a, D(kAhi, kk), D(kBlo, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(kAlo, kk), D(kBhi, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(kAlo, kk), D(kBlo, kk), idesc, 1u);
                        umma_f16_pair(t1a, D(kAhi, kk), D(kBhi, kk), idesc, 1u);
                    }
                } else if (P == 4) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_pair(t0a, D(kAhi, kk), D(kBlo, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(kAlo, kk), D(kBhi, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(kAhi, kk), D(kBhi, kk), idesc, 1u);
                    }
                } else if (P == 10 || P == 11) {
                    // chunked: a new accumulator slot (of four) every two K-blocks, overwritten by its
                    // first MMA, committed to a slot barrier at the chunk's end (P11: one slot, same commits)
                    const uint32_t st = (uint32_t)(i % 3) * 49152u;
                    const uint32_t ta = P == 10 ? slot + ((i >> 1) & 3) * 128 : t0a;
                    const bool first = (i & 1) == 0;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_pair(ta, D(st + kAhi, kk), D(st + kBlo, kk), idesc, (first && kk == 0) ? 0u : 1u);
                        umma_f16_pair(ta, D(st + kAlo, kk), D(st + kBhi, kk), idesc, 1u);
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_f16_pair(ta, D(st + kAhi, kk), D(st + kBhi, kk), idesc, 1u);
                    if (i & 1) umma_commit_pair(&sbar[(i >> 1) & 3]);
                    umma_commit_pair(&ebar[i % 3]);
                } else if (P >= 6) {
                    const uint32_t st = P >= 7 ? (uint32_t)(i % 3) * 49152u : 0u;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_pair(t0a, D(st + kAhi, kk), D(st + kBlo, kk), idesc, 1u);
                        umma_f16_pair(t0a, D(st + kAlo, kk), D(st + kBhi, kk), idesc, 1u);
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_f16_pair(t0a, D(st + kAhi, kk), D(st + kBhi, kk), idesc, 1u);
                    if (i & 1) umma_commit_pair(&sbar[(i >> 1) & 3]);
                    umma_commit_pair(&ebar[i % 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 3; ++j)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) umma_f16_pair(t0a, D(kAhi, kk), D(kBhi, kk), idesc, 1u);
                }
            }
            __syncwarp();
        }
        if (elect_one_sync()) umma_commit_pair(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) {
            out[blockIdx.x] = (unsigned long long)(clock64() - c0);
            stop = 1;
        }
    } else if (rank == 1 && warp == 0) {
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) stop = 1;
    } else if (warp >= 4) {
        // the kernel's 16 worker warps waiting on a barrier (spin or suspend-hint try_wait) meanwhile
        const uint32_t a = smem_u32(&never);
        if (SPIN == 1) {
            while (!stop) mbar_try_wait(a, 0);
        } else if (SPIN == 2) {
            while (!stop) mbar_try_wait_sleep(a, 0);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(slot, 512);
    }
}

template <int P, int FILL = 0, int SPIN = 0>
void run(const char* name, int grid) {
    auto k = acc_bench<P, FILL, SPIN>;
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    cudaMallocManaged(&out, 148 * 8);
    const int iters = 2048;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(SPIN ? 640 : 128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
        cudaLaunchKernelEx(&cfg, k, iters, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(e));
            return;
        }
    }
    double cyc = 0;
    int cnt = 0;
    for (int b = 0; b < grid; b += 2) {
        cyc += out[b];
        ++cnt;
    }
    cyc /= cnt;
    const double per = cyc / (iters * 12.0 * (P == 3 ? 16.0 / 12.0 : 1.0));
    printf("%-64s grid %3d %6.1f cyc/MMA -> %3.0f%% of 64\n", name, grid, per, 100.0 * 64.0 / per);
    cudaFree(out);
}

int main() {
    for (int grid : {2, 148}) {
        run<0>("P0 one accumulator, same A/B", grid);
        run<1>("P1 normal K-block (cross x8, hh x4), one accumulator", grid);
        run<2>("P2 normal K-block, hh into a second accumulator", grid);
        run<3>("P3 exact K-block (x, x, lolo -> X; hh -> H) per K16", grid);
        run<4>("P4 one accumulator, per K16 (hi.lo, lo.hi, hi.hi)", grid);
        run<5>("P5 one accumulator, hi.hi only, K16 descriptors", grid);
        run<6>("P6 P1 + per-K-block multicast commit + slot commit", grid);
        run<7>("P7 P6 + three rotating 48 KB stages", grid);
        run<8>("P8 P7 + full-barrier wait + fence per K-block", grid);
        run<1, 1>("P1 with random operand data", grid);
        run<3, 1>("P3 with random operand data", grid);
        run<8, 1>("P8 with random operand data", grid);
        run<8, 1, 1>("P8 + 16 warps spinning on try_wait", grid);
        run<8, 1, 2>("P8 + 16 warps on suspend-hint try_wait", grid);
        run<10, 1>("P10 chunks: new accumulator slot every 2 K-blocks", grid);
        run<11, 1>("P11 chunks: one slot, overwrite every 2 K-blocks", grid);
    }
    return 0;
}
