// Microbenchmark: tcgen05.ld throughput (bytes/cycle/SM) vs shape, warps and loads in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2605_08523_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace ffg;

__device__ __forceinline__ void ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32"
        " {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
}

// WARPS warps; each warp reads its lane quarter (warp & 3), COLS columns per round starting at
// column (warp >> 2) * COLS, SHAPE 32 or 64 columns per instruction.
template <int WARPS, int COLS, int SHAPE>
__global__ void tmem_bench(int rounds, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * COLS;
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < rounds; ++i) {
        if constexpr (SHAPE == 32) {
#pragma unroll
            for (int c = 0; c < COLS; c += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem + c, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; e += 4) { acc0 ^= v[e]; acc1 ^= v[e + 1]; acc2 ^= v[e + 2]; acc3 ^= v[e + 3]; }
            }
        } else {
#pragma unroll
            for (int c = 0; c < COLS; c += 64) {
                uint32_t v[64];
                ld_x64(tmem + c, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 64; e += 4) { acc0 ^= v[e]; acc1 ^= v[e + 1]; acc2 ^= v[e + 2]; acc3 ^= v[e + 3]; }
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(acc0 ^ acc1 ^ acc2 ^ acc3);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(slot, 512);
    }
}

template <int WARPS, int COLS, int SHAPE>
void run() {
    unsigned long long* out;
    float* sink;
    cudaMallocManaged(&out, 148 * 8);
    cudaMalloc(&sink, 148 * WARPS * 32 * 4);
    const int rounds = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        tmem_bench<WARPS, COLS, SHAPE><<<148, WARPS * 32>>>(rounds, out, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    }
    double cyc = 0;
    for (int b = 0; b < 148; ++b) cyc += out[b];
    cyc /= 148;
    const double bytes = (double)rounds * WARPS * 32 * COLS * 4;
    printf("warps=%2d cols/warp=%3d x%d : %7.1f B/clk/SM\n", WARPS, COLS, SHAPE, bytes / cyc);
    cudaFree(out);
    cudaFree(sink);
}

int main() {
    run<4, 128, 32>();
    run<8, 64, 32>();
    run<8, 128, 32>();
    run<16, 64, 32>();
    run<16, 128, 32>();
    run<8, 64, 64>();
    run<16, 64, 64>();
    run<16, 128, 64>();
    return 0;
}
