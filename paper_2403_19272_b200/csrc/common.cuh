// Shared device helpers for the sm_100a cloth pipeline.
//
// Every routine here reproduces the reference's numpy evaluation order so the
// fp64 results (pair sets, CCD hit sets, TOIs, partial-CCD classes) are
// bit-identical to the reference on identical inputs.  The whole library is
// compiled with -fmad=false: a multiply followed by an add is never fused
// unless an explicit fma() is written (only where OpenBLAS fuses, or in
// reductions whose reference order is BLAS-internal anyway).
//
//   dot3    = np.einsum("ij,ij->i")  over 3 terms: (a0 b0 + a2 b2) + a1 b1
//   norm3   = np.linalg.norm(axis=1) over 3 terms: sqrt((a0^2 + a1^2) + a2^2)
//   cross3  = np.cross (componentwise a1 b2 - a2 b1, ...)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define CS_VT 0
#define CS_EE 1

struct d3 {
    double x, y, z;
};

__device__ __forceinline__ d3 mk3(double a, double b, double c) { return d3{a, b, c}; }
__device__ __forceinline__ d3 operator-(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ d3 operator+(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
// scalar * vector, evaluated per component as numpy's broadcast s[:,None] * v
__device__ __forceinline__ d3 operator*(double s, d3 v) { return d3{s * v.x, s * v.y, s * v.z}; }

__device__ __forceinline__ double dot3(d3 a, d3 b) {
    double s = a.x * b.x + a.z * b.z;
    return s + a.y * b.y;
}
__device__ __forceinline__ double norm3(d3 a) {
    double s = a.x * a.x + a.y * a.y;
    return sqrt(s + a.z * a.z);
}
__device__ __forceinline__ d3 cross3(d3 a, d3 b) {
    return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// 32-byte stamp records (x, y, z, w) move as one 256-bit access (LDG/STG .256 on sm_100a)
// instead of two 128-bit halves of the same sector; the pointers are 32-byte aligned
// (pool allocations, double4 indexing)
__device__ __forceinline__ double4 ldg256(const double4* p) {
    double4 v;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void stg256(double4* p, double x, double y, double z, double w) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w) : "memory");
}
__device__ __forceinline__ d3 ld3(const double* __restrict__ p, int64_t i) {
    return d3{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
}
__device__ __forceinline__ void st3(double* __restrict__ p, int64_t i, d3 v) {
    p[3 * i] = v.x;
    p[3 * i + 1] = v.y;
    p[3 * i + 2] = v.z;
}
// np.clip(v, 0, 1) (NaN propagates like numpy's minimum/maximum)
__device__ __forceinline__ double clip01(double v) {
    if (v != v) return v;
    return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
}
// numpy np.minimum / np.maximum propagate NaN
__device__ __forceinline__ double np_min(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return a < b ? a : b;
}
__device__ __forceinline__ double np_max(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return a > b ? a : b;
}
__device__ __forceinline__ double np_sign(double v) {
    if (v != v) return v;
    return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0);
}

#define CS_TINY 1e-14  // reference geometry.py:7

// fp64 box stored as 6 contiguous doubles lo.xyz, hi.xyz (16-byte aligned rows)
__device__ __forceinline__ void load_box(const double* __restrict__ box, int p, double lo[3], double hi[3]) {
    const double2* b = reinterpret_cast<const double2*>(box + 6 * (int64_t)p);
    const double2 a0 = b[0], a1 = b[1], a2 = b[2];
    lo[0] = a0.x;
    lo[1] = a0.y;
    lo[2] = a1.x;
    hi[0] = a1.y;
    hi[1] = a2.x;
    hi[2] = a2.y;
}


// Count `flag` over the whole block with one global atomic per block (warp ballots
// -> shared partials).  Every thread of the block must call it (integer count, so
// the result is order independent).
__device__ __forceinline__ void block_count(bool flag, int* __restrict__ count) {
    __shared__ int sh_cnt[32];
    __syncthreads();  // a previous block_count in the same kernel may still be reading sh_cnt
    const unsigned ballot = __ballot_sync(0xffffffffu, flag);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh_cnt[w] = __popc(ballot);
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int k = 0; k < (int)((blockDim.x + 31) >> 5); ++k) c += sh_cnt[k];
        if (c) atomicAdd(count, c);
    }
}

// Closest point on triangle (a,b,c) to p: reference geometry.py:10-79.
// Returns distance; u, v = barycentric weights of b and c; q = closest point.
__device__ __forceinline__ double pt_tri_closest(d3 p, d3 a, d3 b, d3 c, double& u, double& v, d3& q) {
    d3 ab = b - a, ac = c - a;
    d3 ap = p - a, bp = p - b, cp = p - c;
    double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
    double d3_ = dot3(ab, bp), d4 = dot3(ac, bp);
    double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
    u = 0.0;
    v = 0.0;
    bool done = (d1 <= 0.0) && (d2 <= 0.0);
    if (!done && d3_ >= 0.0 && d4 <= d3_) {
        u = 1.0;
        done = true;
    }
    if (!done && d6 >= 0.0 && d5 <= d6) {
        v = 1.0;
        done = true;
    }
    double vc = d1 * d4 - d3_ * d2;
    if (!done && vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) {
        double den = d1 - d3_;
        u = fabs(den) > CS_TINY ? d1 / den : 0.0;
        done = true;
    }
    double vb = d5 * d2 - d1 * d6;
    if (!done && vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        double den = d2 - d6;
        v = fabs(den) > CS_TINY ? d2 / den : 0.0;
        done = true;
    }
    double va = d3_ * d6 - d5 * d4;
    double g1 = d4 - d3_, g2 = d5 - d6;
    if (!done && va <= 0.0 && g1 >= 0.0 && g2 >= 0.0) {
        double den = g1 + g2;
        double w = fabs(den) > CS_TINY ? g1 / den : 0.0;
        u = 1.0 - w;
        v = w;
        done = true;
    }
    if (!done) {
        double den = (va + vb) + vc;
        double inv = fabs(den) > CS_TINY ? 1.0 / den : 0.0;
        u = vb * inv;
        v = vc * inv;
    }
    q = (a + u * ab) + v * ac;
    return norm3(p - q);
}

// Segment-segment closest points: reference geometry.py:82-112.
__device__ __forceinline__ double seg_seg_closest(d3 a0, d3 a1, d3 b0, d3 b1, double& s, double& t, d3& pa, d3& pb) {
    d3 da = a1 - a0, db = b1 - b0, r = a0 - b0;
    double aa = dot3(da, da), ee = dot3(db, db);
    double f = dot3(db, r), c = dot3(da, r), bb = dot3(da, db);
    double den = aa * ee - bb * bb;
    double ae = aa * ee;
    s = den > CS_TINY * (ae > 1.0 || ae != ae ? ae : 1.0) ? (bb * f - c * ee) / den : 0.0;
    s = clip01(s);
    double traw = ee > CS_TINY ? (bb * s + f) / ee : 0.0;
    t = clip01(traw);
    if (traw != t) {
        double sn = aa > CS_TINY ? (bb * t - c) / aa : 0.0;
        s = clip01(sn);
    }
    pa = a0 + s * da;
    pb = b0 + t * db;
    return norm3(pa - pb);
}

// Witness distance of a pair from its 4 gathered corners (reference ccd.py:207-218).
__device__ __forceinline__ double pair_distance(int kind, d3 p0, d3 p1, d3 p2, d3 p3) {
    if (kind == CS_VT) {
        double u, v;
        d3 q;
        return pt_tri_closest(p0, p1, p2, p3, u, v, q);
    }
    double s, t;
    d3 pa, pb;
    return seg_seg_closest(p0, p1, p2, p3, s, t, pa, pb);
}

__host__ __device__ __forceinline__ int cs_div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

#define CS_CHECK_LAUNCH()                                  \
    do {                                                   \
        cudaError_t e_ = cudaGetLastError();               \
        if (e_ != cudaSuccess) return (int)e_ + 1000;      \
    } while (0)
