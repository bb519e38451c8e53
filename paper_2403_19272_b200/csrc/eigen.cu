// Rest-shape eigenbasis on the device (setup): the block
// kernels of a Chebyshev-filtered subspace iteration (ChFSI) over the free-vertex
// elastic matrix H, replacing the reference's shift-invert eigsh (subspace.py:49-84)
// for paper-scale meshes.  The small p x p algebra (Cholesky, triangular inverse,
// symmetric eigensolve of the Rayleigh quotient) stays on the host (eigen.py).
//
//   k_blk_spmm<NQ, MODE>  one warp per row of H (CSR); lanes span the block's columns.
//                         MODE 0: Y = H X; MODE 1: Y = (H X - c X) s1 (first filter
//                         term); MODE 2: Y = (H X - c X) s1 - s2 X_prev (three-term
//                         Chebyshev recurrence) - one pass over the block per degree
//   k_blk_gram_partial    A^T B over a row chunk, 32 x 32 output tile per block (4 row
//                         groups, 4 x 4 register tiles), partials summed in order
//   k_blk_mul             Y = X S (S p x p, staged in shared memory 32 columns at a time)
//   k_blk_resid           per-column sum of squares of H X_j - w_j X_j (Ritz residuals)
//
// Blocks are row-major n x pp doubles, pp = p rounded up to 32 (padding columns are
// kept zero), so every row is a run of whole 256-byte lane groups.
#include "common.cuh"

namespace cs {

template <int NQ, int MODE>
__global__ void __launch_bounds__(256) k_blk_spmm(int n, const int* __restrict__ indptr,
                                                  const int* __restrict__ indices, const double* __restrict__ data,
                                                  const double* __restrict__ X, const double* __restrict__ Xp, int pp,
                                                  double c, double s1, double s2, double* __restrict__ Y) {
    const int lane = threadIdx.x & 31;
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= n) return;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const int beg = indptr[row], end = indptr[row + 1];
    for (int k = beg; k < end; ++k) {
        const double v = __ldg(data + k);
        const double* xr = X + (int64_t)__ldg(indices + k) * pp + lane;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = fma(v, __ldg(xr + 32 * q), acc[q]);
    }
    const int64_t o = (int64_t)row * pp + lane;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double y = acc[q];
        if (MODE >= 1) y = (y - c * X[o + 32 * q]) * s1;
        if (MODE == 2) y = y - s2 * Xp[o + 32 * q];
        Y[o + 32 * q] = y;
    }
}

// part[chunk][a * pp + b] = sum over the chunk's rows of A[row][a] B[row][b] for the
// 32 x 32 output tile (blockIdx.y): 64-row tiles staged in shared memory, 4 row groups
// x 64 threads, each thread a 4 x 4 register tile; group partials summed in order.
__global__ void __launch_bounds__(256) k_blk_gram_partial(int n, int pp, const double* __restrict__ A,
                                                          const double* __restrict__ B, int rows_per_chunk,
                                                          double* __restrict__ part) {
    constexpr int kT = 64;
    __shared__ __align__(16) double sbuf[2][kT][32];
    const int ntile = pp / 32;
    const int ta0 = (blockIdx.y / ntile) * 32, tb0 = (blockIdx.y % ntile) * 32;
    const int beg = blockIdx.x * rows_per_chunk, end = min(n, beg + rows_per_chunk);
    const int t = threadIdx.x, grp = t >> 6;
    const int ta = ((t & 63) >> 3) * 4, tb = (t & 7) * 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int t0 = beg; t0 < end; t0 += kT) {
        const int nt = min(kT, end - t0);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kT * 32 / 256; ++u) {
            const int e = t + u * 256, k = e >> 5, cc = e & 31;
            sbuf[0][k][cc] = k < nt ? A[(int64_t)(t0 + k) * pp + ta0 + cc] : 0.0;
            sbuf[1][k][cc] = k < nt ? B[(int64_t)(t0 + k) * pp + tb0 + cc] : 0.0;
        }
        __syncthreads();
        for (int k = grp; k < nt; k += 4) {
            const double2 a01 = *reinterpret_cast<const double2*>(&sbuf[0][k][ta]);
            const double2 a23 = *reinterpret_cast<const double2*>(&sbuf[0][k][ta + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&sbuf[1][k][tb]);
            const double2 b23 = *reinterpret_cast<const double2*>(&sbuf[1][k][tb + 2]);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
    }
    __syncthreads();
    double* red = &sbuf[0][0][0];  // [grp][32 x 32]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[grp * 1024 + (ta + i) * 32 + tb + j] = acc[i][j];
    __syncthreads();
    for (int o = t; o < 1024; o += 256) {
        const int a = o >> 5, b = o & 31;
        part[(int64_t)blockIdx.x * pp * pp + (int64_t)(ta0 + a) * pp + tb0 + b] =
            ((red[o] + red[1024 + o]) + red[2048 + o]) + red[3072 + o];
    }
}

// Y[row][chunk cols] = X[row][:] S[:, chunk]: S columns staged 32 at a time; one warp
// per row, lane = output column.
__global__ void __launch_bounds__(256) k_blk_mul(int n, int pp, const double* __restrict__ X,
                                                 const double* __restrict__ S, double* __restrict__ Y) {
    extern __shared__ double sS[];  // [pp][33]
    const int c0 = blockIdx.y * 32;
    for (int e = threadIdx.x; e < pp * 32; e += blockDim.x) {
        const int k = e >> 5, cc = e & 31;
        sS[k * 33 + cc] = S[(int64_t)k * pp + c0 + cc];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int row = blockIdx.x * 8 + warp; row < n; row += gridDim.x * 8) {
        const double* xr = X + (int64_t)row * pp;
        double acc = 0.0;
        for (int k0 = 0; k0 < pp; k0 += 32) {
            const double xv = __ldg(xr + k0 + lane);
#pragma unroll 8
            for (int kk = 0; kk < 32; ++kk) acc = fma(__shfl_sync(0xffffffffu, xv, kk), sS[(k0 + kk) * 33 + lane], acc);
        }
        Y[(int64_t)row * pp + c0 + lane] = acc;
    }
}

// part[blk][j] = sum over the block's rows of (HX[row][j] - w_j X[row][j])^2, j < pp
__global__ void __launch_bounds__(256) k_blk_resid(int n, int pp, const double* __restrict__ HX,
                                                   const double* __restrict__ X, const double* __restrict__ w,
                                                   double* __restrict__ part) {
    __shared__ double red[8][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q0 = 0; q0 < pp; q0 += 256) {
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
        for (int row = blockIdx.x * 8 + warp; row < n; row += gridDim.x * 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = q0 + lane + 32 * u;
                if (j < pp) {
                    const double d = HX[(int64_t)row * pp + j] - w[j] * X[(int64_t)row * pp + j];
                    acc[u] = fma(d, d, acc[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) red[warp][lane + 32 * u] = acc[u];
        __syncthreads();
        for (int j = threadIdx.x; j < 256 && q0 + j < pp; j += blockDim.x) {
            double s = 0.0;
            for (int wq = 0; wq < 8; ++wq) s += red[wq][j];
            part[(int64_t)blockIdx.x * pp + q0 + j] = s;
        }
        __syncthreads();
    }
}

}  // namespace cs
