// Device triangle-triangle intersection check: the penetration-free invariant.
//
// Restates the reference's validation oracle oracle_intersect
// (pkg/src/clothsim/oracles.py:83-131) + tri_tri_intersect (:33-48): every pair of
// world triangles that share no vertex, whose closed bounding boxes overlap, and
// that the 17-axis separating-axis test cannot separate (touching counts as
// intersecting; axes shorter than 1e-14 scale^2 are unusable).  Projections are
// np.einsum-ordered ((a0 b0 + a2 b2) + a1 b1, as dot3), cross products naive.
//
// Candidates come from the broad phase's hash grid over the triangles' static
// boxes (margin 0): one warp per bucket, pairs reported in the cell holding their
// box intersection's min corner (exactly once), oversize triangles brute-forced.
// Output: the count (order independent) and up to `cap` index pairs (atomic
// append; callers sort).
#include "common.cuh"

namespace cs {

// reference tri_tri_intersect for one pair (oracles.py:33-48)
__device__ bool tri_tri_intersect_dev(const d3 p[3], const d3 q[3]) {
    const d3 ep[3] = {p[1] - p[0], p[2] - p[1], p[0] - p[2]};
    const d3 eq[3] = {q[1] - q[0], q[2] - q[1], q[0] - q[2]};
    const d3 npn = cross3(ep[0], ep[1]);
    const d3 nqn = cross3(eq[0], eq[1]);
    double scale = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        scale = fmax(scale, fmax(fmax(fabs(p[k].x), fabs(p[k].y)), fabs(p[k].z)));
        scale = fmax(scale, fmax(fmax(fabs(q[k].x), fabs(q[k].y)), fabs(q[k].z)));
    }
    scale = scale + 1.0;
    const double thresh = 1e-14 * (scale * scale);
    for (int a = 0; a < 17; ++a) {
        d3 ax;
        if (a == 0) ax = npn;
        else if (a == 1) ax = nqn;
        else if (a < 11) ax = cross3(ep[(a - 2) / 3], eq[(a - 2) % 3]);
        else if (a < 14) ax = cross3(npn, ep[a - 11]);
        else ax = cross3(nqn, eq[a - 14]);
        if (!(norm3(ax) > thresh)) continue;
        double pmin = dot3(ax, p[0]), pmax = pmin, qmin = dot3(ax, q[0]), qmax = qmin;
#pragma unroll
        for (int k = 1; k < 3; ++k) {
            const double dp = dot3(ax, p[k]), dq = dot3(ax, q[k]);
            pmin = fmin(pmin, dp);
            pmax = fmax(pmax, dp);
            qmin = fmin(qmin, dq);
            qmax = fmax(qmax, dq);
        }
        if (pmax < qmin || qmax < pmin) return false;
    }
    return true;
}

__device__ __forceinline__ void report_hit(int a, int b, int* __restrict__ count, int* __restrict__ out, int cap) {
    const int k = atomicAdd(count, 1);
    if (k < cap) {
        out[2 * k] = a < b ? a : b;
        out[2 * k + 1] = a < b ? b : a;
    }
}

__device__ __forceinline__ bool tris_disjoint(const int* __restrict__ T, int a, int b) {
    const int a0 = T[3 * a], a1 = T[3 * a + 1], a2 = T[3 * a + 2];
    const int b0 = T[3 * b], b1 = T[3 * b + 1], b2 = T[3 * b + 2];
    return a0 != b0 && a0 != b1 && a0 != b2 && a1 != b0 && a1 != b1 && a1 != b2 && a2 != b0 && a2 != b1 &&
           a2 != b2;
}

__device__ __forceinline__ bool tri_pair_hits(const int* __restrict__ T, const double* __restrict__ x, int a, int b) {
    d3 p[3], q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        p[k] = ld3(x, T[3 * a + k]);
        q[k] = ld3(x, T[3 * b + k]);
    }
    return tri_tri_intersect_dev(p, q);
}

// one warp per triangle-table bucket run; candidate pairs as in k_pairs_ee
__global__ void __launch_bounds__(128) k_tri_intersect(EntryTable E, const double* __restrict__ tbox,
                                                       const int* __restrict__ tris, const double* __restrict__ x,
                                                       int* __restrict__ count, int* __restrict__ out, int cap) {
    const int lane = threadIdx.x & 31;
    const int nr = E.n_run[0];
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr; r += (gridDim.x * blockDim.x) >> 5) {
        const int eb = E.run[r], ee = r + 1 < nr ? E.run[r + 1] : E.m;
        for (int i = eb; i + 1 < ee; ++i) {
            const int a = E.prim[i];
            const unsigned long long ca = E.code[i];
            double qlo[3], qhi[3];
            load_box(tbox, a, qlo, qhi);
            for (int j0 = i + 1; j0 < ee; j0 += 32) {
                const int j = j0 + lane;
                if (j < ee && E.code[j] == ca && ((E.zb[i] | E.zb[j]) & 7) == 7) {
                    const int b = E.prim[j];
                    double lo[3], hi[3];
                    load_box(tbox, b, lo, hi);
                    if (overlap6(qlo, qhi, lo, hi) && tris_disjoint(tris, a, b) && tri_pair_hits(tris, x, a, b))
                        report_hit(a, b, count, out, cap);
                }
            }
        }
    }
}

// oversize triangle over[t] against every other triangle (entered ones always,
// oversize ones only with a larger id)
__global__ void k_tri_intersect_over(const int* __restrict__ over, int n_over, const uint8_t* __restrict__ is_over,
                                     const double* __restrict__ tbox, int ntris, const int* __restrict__ tris,
                                     const double* __restrict__ x, int* __restrict__ count, int* __restrict__ out,
                                     int cap) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_over) return;
    const int a = over[t];
    double qlo[3], qhi[3];
    load_box(tbox, a, qlo, qhi);
    for (int b = 0; b < ntris; ++b) {
        if (b == a || (is_over[b] && b < a)) continue;
        double lo[3], hi[3];
        load_box(tbox, b, lo, hi);
        if (overlap6(qlo, qhi, lo, hi) && tris_disjoint(tris, a, b) && tri_pair_hits(tris, x, a, b))
            report_hit(a, b, count, out, cap);
    }
}

}  // namespace cs
