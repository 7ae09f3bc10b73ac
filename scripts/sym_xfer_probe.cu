// Probe: host<->device traffic of the bench step (16 x N=1024 fp64, page-locked host buffers) when only
// the upper block triangle travels (one cudaMemcpy2DAsync per 128-row block row) vs whole matrices, both
// directions concurrent on two streams; and the host cost of mirroring the lower blocks of D from the
// upper ones with T threads.
// Build: nvcc -O3 -std=c++17 -o sym_xfer_probe sym_xfer_probe.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

constexpr int N = 1024, B = 16, BS = 128, NB = N / BS;
constexpr size_t MAT = (size_t)N * N;

static void copy_upper(double* dst, const double* src, cudaMemcpyKind kind, cudaStream_t st) {
    for (int m = 0; m < B; ++m)
        for (int R = 0; R < NB; ++R) {
            const size_t off = m * MAT + (size_t)R * BS * N + (size_t)R * BS;
            cudaMemcpy2DAsync(dst + off, N * 8, src + off, N * 8, (size_t)(N - R * BS) * 8, BS, kind, st);
        }
}

// lower blocks (I > J) of every matrix <- transpose of block (J, I); blocks split over T threads
static void mirror(double* D, int T) {
    std::vector<std::thread> th;
    const int nblk = B * NB * (NB - 1) / 2;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=] {
            int k = 0;
            for (int m = 0; m < B; ++m)
                for (int I = 1; I < NB; ++I)
                    for (int J = 0; J < I; ++J, ++k) {
                        if (k % T != t) continue;
                        double* M = D + m * MAT;
                        for (int i0 = 0; i0 < BS; i0 += 16)
                            for (int j0 = 0; j0 < BS; j0 += 16)
                                for (int i = i0; i < i0 + 16; ++i)
                                    for (int j = j0; j < j0 + 16; ++j)
                                        M[(size_t)(I * BS + i) * N + J * BS + j] = M[(size_t)(J * BS + j) * N + I * BS + i];
                    }
            (void)nblk;
        });
    for (auto& x : th) x.join();
}

int main() {
    double *hH, *hD, *dH, *dD;
    cudaHostAlloc(&hH, B * MAT * 8, cudaHostAllocDefault);
    cudaHostAlloc(&hD, B * MAT * 8, cudaHostAllocDefault);
    cudaMalloc(&dH, B * MAT * 8);
    cudaMalloc(&dD, B * MAT * 8);
    memset(hH, 0, B * MAT * 8);
    memset(hD, 0, B * MAT * 8);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b1, b2;
    cudaEventCreate(&a);
    cudaEventCreate(&b1);
    cudaEventCreate(&b2);
    const int reps = 10;
    for (int mode = 0; mode < 6; ++mode) {
        // 0 full both, 1 upper both, 2 full H2D, 3 full D2H, 4 upper H2D, 5 upper D2H
        for (int w = 0; w < 2; ++w) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s1);
            cudaStreamWaitEvent(s2, a, 0);
            for (int r = 0; r < reps; ++r) {
                const bool up = mode == 1 || mode == 4 || mode == 5;
                const bool h2d = mode == 0 || mode == 1 || mode == 2 || mode == 4;
                const bool d2h = mode == 0 || mode == 1 || mode == 3 || mode == 5;
                if (h2d) {
                    if (up) copy_upper(dH, hH, cudaMemcpyHostToDevice, s1);
                    else cudaMemcpyAsync(dH, hH, B * MAT * 8, cudaMemcpyHostToDevice, s1);
                }
                if (d2h) {
                    if (up) copy_upper(hD, dD, cudaMemcpyDeviceToHost, s2);
                    else cudaMemcpyAsync(hD, dD, B * MAT * 8, cudaMemcpyDeviceToHost, s2);
                }
            }
            cudaEventRecord(b1, s1);
            cudaEventRecord(b2, s2);
            cudaDeviceSynchronize();
            float m1, m2;
            cudaEventElapsedTime(&m1, a, b1);
            cudaEventElapsedTime(&m2, a, b2);
            const float ms = (m1 > m2 ? m1 : m2) / reps;
            const char* names[] = {"full H2D+D2H", "upper H2D+D2H", "full H2D", "full D2H", "upper H2D", "upper D2H"};
            if (w) printf("%-16s %.3f ms per step (16 x 8 MiB per direction%s)\n", names[mode], ms,
                          (mode == 1 || mode >= 4) ? ", upper block rows" : "");
        }
    }
    for (int T : {1, 4, 8, 16, 32}) {
        mirror(hD, T);
        auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < 5; ++r) mirror(hD, T);
        auto t1 = std::chrono::steady_clock::now();
        printf("host mirror of the lower blocks, %2d threads: %.3f ms per step\n", T,
               std::chrono::duration<double, std::milli>(t1 - t0).count() / 5);
    }
    printf("hardware threads: %u\n", std::thread::hardware_concurrency());
    return 0;
}
