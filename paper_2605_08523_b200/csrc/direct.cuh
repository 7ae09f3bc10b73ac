// DOUBLE / SINGLE precision modes: the MLSP2 recursion evaluated in fp64 / fp32
// arithmetic throughout -- scalar_models.cpp:243-252 lifted to matrices, in the reference's order:
//
//   A = d_0 X_0;  for l:  Y = X_l X_l;  X_{l+1} = a_l Y + b_l X_l + c_l I;  A += d_{l+1} X_{l+1};
//   D = A + X_L
//
// These modes are not the north-star tensor-core path (no fp64 / true-fp32 tcgen05 kinds): the
// square is a plain library GEMM (cuBLAS {D,S}gemmStridedBatched, loaded lazily by the host side so
// the FP32E/BF16/FP16 path never loads cuBLAS), the rest is ours: a fused, tiled layer update that
// uses only the upper-triangle entries of Y and writes both triangles of X_{l+1} (X stays EXACTLY
// symmetric whatever the GEMM's summation order), and a final pass D = A + X with fixed-order per-row
// statistics for K3.  An instrumented count of n squarings per matrix.
#pragma once
#include "kernels.cuh"

namespace ffg {

constexpr int kModeF64 = 3;  // internal ids of the direct modes (after kModeF32E / F16 / BF16)
constexpr int kModeF32 = 4;

template <typename T>
struct DirectLayer {
    const T* Y;      // [B][n][n] X_l X_l (cuBLAS; only the upper triangle is read)
    T* X;            // [B][n][n] X_l in, X_{l+1} out (both triangles)
    T* A;            // [B][n][n] running sum
    double a, b, c, d_next;  // layer coefficients; d_next = d_{l+1} (0 for the last layer)
    int n;
    int* flags;      // [B][2]: [0] first non-finite X index (atomicMin)
    int layer;       // l
};

// X0 = alpha H + gamma I, A = d0 X0 (elementwise, T precision); non-finite X0 flags layer 0.
template <typename T>
__global__ void __launch_bounds__(256) direct_init_kernel(const double* __restrict__ H, const double* alpha,
                                                          const double* gamma, double d0, T* X, T* A, int n,
                                                          int* flags) {
    const int m = blockIdx.y;
    const size_t nn = (size_t)n * n;
    const double al = alpha[m], ga = gamma[m];
    bool bad = false;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
        const size_t i = e / n, j = e - i * n;
        double v = al * H[m * nn + e];
        if (i == j) v += ga;
        const T x = (T)v;
        X[m * nn + e] = x;
        A[m * nn + e] = (T)d0 * x;
        bad |= !isfinite((double)x);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(&flags[2 * m], 0);
}

// One layer's update over 32 x 32 tiles of the upper block triangle: tile (I, J), I <= J, computes
// X' = a Y + b X (+ c on the diagonal) from the upper entries (i <= j) and stores the tile and its
// transpose (through shared memory, both coalesced); A += d' X' likewise.
template <typename T>
__global__ void __launch_bounds__(256) direct_layer_kernel(const __grid_constant__ DirectLayer<T> p) {
    __shared__ T sx[32][33], sa[32][33];
    const int m = blockIdx.y;
    const int n = p.n, nt = (n + 31) / 32;
    // blockIdx.x -> (I, J), I <= J, row-major over the upper tile triangle
    int t = blockIdx.x, I = 0;
    while (t >= nt - I) {
        t -= nt - I;
        ++I;
    }
    const int J = I + t;
    const size_t base = (size_t)m * n * n;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    const T a = (T)p.a, b = (T)p.b, c = (T)p.c, dn = (T)p.d_next;
    bool bad = false;
    for (int r = ty; r < 32; r += 8) {
        const int i = 32 * I + r, j = 32 * J + tx;
        T xn = (T)0, an = (T)0;
        if (i < n && j < n) {
            // upper entry (i <= j); in a diagonal tile the lower entries take the transposed upper value
            const int ui = min(i, j), uj = max(i, j);
            const size_t e = base + (size_t)ui * n + uj;
            xn = a * p.Y[e] + b * p.X[e];
            if (ui == uj) xn += c;
            an = p.A[e] + dn * xn;
            bad |= !isfinite((double)xn);
        }
        sx[r][tx] = xn;
        sa[r][tx] = an;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = 32 * I + r, j = 32 * J + tx;
        if (i < n && j < n) {
            p.X[base + (size_t)i * n + j] = sx[r][tx];
            if (p.d_next != 0.0) p.A[base + (size_t)i * n + j] = sa[r][tx];
        }
        // the transposed tile (J, I): row 32J + r, column 32I + tx <- (32I + tx, 32J + r)
        const int i2 = 32 * J + r, j2 = 32 * I + tx;
        if (I != J && i2 < n && j2 < n) {
            p.X[base + (size_t)i2 * n + j2] = sx[tx][r];
            if (p.d_next != 0.0) p.A[base + (size_t)i2 * n + j2] = sa[tx][r];
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(&p.flags[2 * m], p.layer + 1);
}

// D = A + X (fp64 out) and per-row partials {D_ii, sum_j D_ij^2} (fixed order: a row per warp, lanes
// over columns, fixed butterfly) for K3; the instrumented squaring count.
template <typename T>
__global__ void __launch_bounds__(256) direct_final_kernel(const T* X, const T* A, double* D, int n,
                                                           double2* partials, RegionCheck region, int L,
                                                           uint32_t* products) {
    const int m = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * 8 + warp;
    const size_t nn = (size_t)n * n;
    if (blockIdx.x == 0 && threadIdx.x == 0) products[m] = matrix_in_region(region, m) ? (uint32_t)L : 0u;
    if (i >= n) return;
    double dg = 0.0, sq = 0.0;
    for (int j = lane; j < n; j += 32) {
        const size_t e = (size_t)m * nn + (size_t)i * n + j;
        const T s = A[e] + X[e];
        const double dv = (double)s;
        if (D) D[e] = dv;
        if (j == i) dg = dv;
        sq += dv * dv;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dg += __shfl_xor_sync(0xffffffffu, dg, o);  // exactly one lane holds D_ii
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    if (lane == 0) partials[(size_t)m * n + i] = make_double2(dg, sq);
}

}  // namespace ffg
