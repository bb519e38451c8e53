// Narrow phase: per-pair fp64 kernels, bit-identical to the reference.
//
//   k_full_ccd       reference ccd.py:138-196   (cubic coplanarity TOI + flat fallback)
//   k_distance_toi   reference ccd.py:221-266   (conservative-advancement line-search filter)
//   k_witness        reference stepper.py:194-216 + geometry.py:115-148
//   k_partial_ndb    reference partial.py:149-204 fused with the NDB life-span update
//                    (stepper.py:517-523, _pair_gaps :218-236, pairs.py:65-70)
//   k_engage_init    stepper.py:483-487 / 564-565 (engaged set + weights after a CCD site)
//
// One thread per pair; all positions are fp64 world arrays (n_w, 3).  These
// kernels are FP64-ALU / latency bound: the pair stream is
// ~25-64 B/pair while a full-CCD pair costs 300-2000 flops.
#include "common.cuh"

namespace cs {

// inv(vander([0, 1/3, 2/3, 1], increasing)) exactly as numpy/LAPACK produce it
// (reference ccd.py:21-22); hex literals pinned by tests/test_oracle_golden.py.
__constant__ double kFit[4][4] = {
    {0x1.0p+0, 0x0.0p+0, 0x0.0p+0, 0x0.0p+0},
    {-0x1.6000000000001p+2, 0x1.2p+3, -0x1.1fffffffffffcp+2, 0x1.0p+0},
    {0x1.2000000000001p+3, -0x1.68p+4, 0x1.1ffffffffffffp+4, -0x1.2p+2},
    {-0x1.2000000000001p+2, 0x1.bp+3, -0x1.bp+3, 0x1.2p+2},
};

__device__ __forceinline__ double horner(const double c[4], double t) {
    return c[0] + t * (c[1] + t * (c[2] + t * c[3]));
}

// correctly rounded x^3 (numpy `** 3` goes through libm pow, not x*x*x)
__device__ __forceinline__ double cube_rn(double x) {
    double h = x * x;
    double l = fma(x, x, -h);
    double hh = h * x;
    double e1 = fma(h, x, -hh);
    return hh + (e1 + l * x);
}

struct Corners {
    d3 p[4];
};

__device__ __forceinline__ Corners gather4(const double* __restrict__ x, int4 id) {
    Corners c;
    c.p[0] = ld3(x, id.x);
    c.p[1] = ld3(x, id.y);
    c.p[2] = ld3(x, id.z);
    c.p[3] = ld3(x, id.w);
    return c;
}

__device__ __forceinline__ d3 lerp_node(d3 a, d3 b, double t) {
    double s = 1.0 - t;  // (1.0 - t) * x_start + t * x_end, reference ccd.py:40
    return (s * a) + (t * b);
}

__device__ __forceinline__ double triple(int kind, const d3 p[4]) {
    d3 u, v, w;
    if (kind == CS_VT) {
        u = p[2] - p[1];
        v = p[3] - p[1];
        w = p[0] - p[1];
    } else {
        u = p[1] - p[0];
        v = p[3] - p[2];
        w = p[2] - p[0];
    }
    return dot3(cross3(u, v), w);
}

// inflated inside test at time t (reference ccd.py:111-135)
__device__ bool confirm_hit(int kind, const Corners& a, const Corners& b, double t, double tol) {
    d3 q[4];
    double s = 1.0 - t;
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = (s * a.p[k]) + (t * b.p[k]);
    if (kind == CS_VT) {
        double u, v;
        d3 cl;
        double d = pt_tri_closest(q[0], q[1], q[2], q[3], u, v, cl);
        double size = norm3(q[2] - q[1]) + norm3(q[3] - q[1]);
        bool inside = (u >= -1e-8) && (v >= -1e-8) && (u + v <= 1.0 + 1e-8);
        return inside && (d <= tol * np_max(size, 1.0));
    }
    double s2, t2;
    d3 pa, pb;
    double d = seg_seg_closest(q[0], q[1], q[2], q[3], s2, t2, pa, pb);
    double size = norm3(q[1] - q[0]) + norm3(q[3] - q[2]);
    return d <= tol * np_max(size, 1.0);
}

__device__ __forceinline__ double pair_extent(const Corners& a, const Corners& b) {
    d3 lo = a.p[0], hi = a.p[0];
    // min/max are exact, so evaluation order is irrelevant
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const d3 q0 = a.p[k], q1 = b.p[k];
        lo.x = np_min(lo.x, np_min(q0.x, q1.x));
        lo.y = np_min(lo.y, np_min(q0.y, q1.y));
        lo.z = np_min(lo.z, np_min(q0.z, q1.z));
        hi.x = np_max(hi.x, np_max(q0.x, q1.x));
        hi.y = np_max(hi.y, np_max(q0.y, q1.y));
        hi.z = np_max(hi.z, np_max(q0.z, q1.z));
    }
    return norm3(hi - lo);
}

// Exact early-out for full_ccd: every TOI full_ccd can report needs a witness
// distance <= tol * max(scale, 1) at that time (validated roots, ccd.py:111-135)
// or <= 1e-9 * max(extent, 1) (flat fallback, ccd.py:171-195), with scale <= 2 x
// the pair extent.  Positions at any t lie in the box of each side's start/end
// corners (up to lerp rounding), so a box gap on some axis above that bound
// proves the reference result is NaN.  The margin absorbs rounding by 1e-9
// relative to the coordinates - far above the fp64 error of any of the terms.
__device__ __forceinline__ bool separated_sides(int kd, const Corners& a, const Corners& b, double tol) {
    const int na = kd == CS_VT ? 1 : 2;
    double alo[3], ahi[3], blo[3], bhi[3], mag = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        alo[c] = blo[c] = INFINITY;
        ahi[c] = bhi[c] = -INFINITY;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double q0[3] = {a.p[k].x, a.p[k].y, a.p[k].z}, q1[3] = {b.p[k].x, b.p[k].y, b.p[k].z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double lo = fmin(q0[c], q1[c]), hi = fmax(q0[c], q1[c]);
            mag = fmax(mag, fmax(fabs(lo), fabs(hi)));
            if (k < na) {
                alo[c] = fmin(alo[c], lo);
                ahi[c] = fmax(ahi[c], hi);
            } else {
                blo[c] = fmin(blo[c], lo);
                bhi[c] = fmax(bhi[c], hi);
            }
        }
    }
    double gap = 0.0, e2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        gap = fmax(gap, fmax(blo[c] - ahi[c], alo[c] - bhi[c]));
        const double span = fmax(ahi[c], bhi[c]) - fmin(alo[c], blo[c]);
        e2 += span * span;
    }
    if (!(gap > 0.0)) return false;  // NaN-safe: non-finite input takes the full path
    const double ext = sqrt(e2);
    const double bound = fmax(tol * fmax(2.0 * ext, 1.0), 1e-9 * fmax(ext, 1.0));
    return gap > bound * (1.0 + 1e-6) + 1e-9 * mag;
}

// coplanarity samples at t = 0, 1/3, 2/3, 1 and the monomial fit (coplanarity_coefficients,
// ccd.py:36-44), lowest order first
__device__ __forceinline__ void coplanarity_fit(int kd, const Corners& a, const Corners& b, int single, double c[4]) {
    const double nodes[4] = {0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0};
    double f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        d3 q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q[k] = lerp_node(a.p[k], b.p[k], nodes[j]);
        f[j] = triple(kd, q);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (!single) {  // OpenBLAS dgemm k=4 kernel: forward FMA chain
            double acc = f[0] * kFit[j][0];
            acc = fma(f[1], kFit[j][1], acc);
            acc = fma(f[2], kFit[j][2], acc);
            c[j] = fma(f[3], kFit[j][3], acc);
        } else {        // m == 1 takes OpenBLAS's gemv-like path
            double even = f[0] * kFit[j][0] + f[2] * kFit[j][2];
            double odd = f[1] * kFit[j][1] + f[3] * kFit[j][3];
            c[j] = even + odd;
        }
    }
}

// full_ccd for one pair (ccd.py:138-196); NaN = miss
__device__ double full_ccd_pair(int kd, const Corners& a, const Corners& b, int single, double tol) {
    const double NaN = __longlong_as_double(0x7ff8000000000000ULL);
    if (separated_sides(kd, a, b, tol)) return NaN;
    double c[4];
    coplanarity_fit(kd, a, b, single, c);
    const double csum = ((fabs(c[0]) + fabs(c[1])) + fabs(c[2])) + fabs(c[3]);
    const double ext = pair_extent(a, b);
    const bool flat = csum <= 1e-12 * np_max(cube_rn(fabs(ext)), 1e-30);

    double toi = NaN;
    if (!flat) {
        // ---- _candidate_roots (ccd.py:53-108)
        double qa = 3.0 * c[3], qb = 2.0 * c[2], ql = c[1];
        bool quad = fabs(qa) > 0.0;
        double disc = qb * qb - (4.0 * qa) * ql;
        bool real = quad && disc >= 0.0;
        double sq = sqrt(real ? disc : 0.0);
        double r1 = real ? (-qb - sq) / (2.0 * qa) : NaN;
        double r2 = real ? (-qb + sq) / (2.0 * qa) : NaN;
        double rl = (!quad && fabs(qb) > 0.0) ? -ql / qb : NaN;
        double br0 = quad ? np_min(r1, r2) : rl;
        double br1 = quad ? np_max(r1, r2) : NaN;
        if (!(br0 > 0.0 && br0 < 1.0)) br0 = NaN;
        if (!(br1 > 0.0 && br1 < 1.0)) br1 = NaN;
        if (br0 != br0 && br1 == br1) {  // np.sort puts nan last
            br0 = br1;
            br1 = NaN;
        } else if (br0 == br0 && br1 == br1 && br1 < br0) {
            double tmp = br0;
            br0 = br1;
            br1 = tmp;
        }
        double k1 = (br0 != br0) ? 1.0 : br0;
        double k2 = (br1 != br1) ? k1 : np_max(br1, k1);
        double lo[3] = {0.0, k1, k2}, hi[3] = {k1, k2, 1.0};
        double roots[5];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            double flo = horner(c, lo[s]), fhi = horner(c, hi[s]);
            bool bracket = (hi[s] > lo[s]) && (flo * fhi < 0.0);
            bool at_end = (hi[s] > lo[s]) && (fhi == 0.0);
            double r = NaN;
            if (bracket) {
                double al = lo[s], ah = hi[s];
                for (int it = 0; it < 80; ++it) {
                    double mid = 0.5 * (al + ah);
                    double fm = horner(c, mid);
                    if (np_sign(fm) == np_sign(flo)) {
                        al = mid;
                        flo = fm;
                    } else {
                        ah = mid;
                    }
                }
                r = 0.5 * (al + ah);
            } else if (at_end) {
                r = hi[s];
            }
            roots[s] = r;
        }
        const double mag = csum + 1e-300;
        const double brk[2] = {br0, br1};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            double tb = brk[j];
            double fv = fabs(horner(c, tb != tb ? 0.0 : tb));
            roots[3 + j] = (tb == tb && fv <= 1e-9 * mag) ? tb : NaN;
        }
#pragma unroll
        for (int s = 0; s < 5; ++s)
            if (!(roots[s] > 0.0 && roots[s] <= 1.0)) roots[s] = NaN;
        // validate in ascending order; first confirmed root is the TOI
        for (int pass = 0; pass < 5; ++pass) {
            int best = -1;
            for (int s = 0; s < 5; ++s)
                if (roots[s] == roots[s] && (best < 0 || roots[s] < roots[best])) best = s;
            if (best < 0) break;
            double t = roots[best];
            roots[best] = NaN;
            if (confirm_hit(kd, a, b, t, tol)) {
                toi = t;
                break;
            }
        }
    } else {
        // ---- dense distance sampling for identically coplanar motion (ccd.py:171-195)
        double d0 = pair_distance(kd, a.p[0], a.p[1], a.p[2], a.p[3]);
        double mv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) mv[k] = norm3(b.p[k] - a.p[k]);
        double ra, rb;
        if (kd == CS_VT) {
            ra = np_max(np_max(np_max(mv[0], 0.0), 0.0), 0.0);
            rb = np_max(np_max(np_max(0.0, mv[1]), mv[2]), mv[3]);
        } else {
            ra = np_max(np_max(np_max(mv[0], mv[1]), 0.0), 0.0);
            rb = np_max(np_max(np_max(0.0, 0.0), mv[2]), mv[3]);
        }
        double reach = ra + rb;
        double e1 = np_max(ext, 1.0);
        if (d0 <= reach + 1e-9 * e1) {
            d3 dp[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) dp[k] = b.p[k] - a.p[k];
            for (int s = 1; s <= 64; ++s) {
                double t = (double)s * (1.0 / 64.0);
                d3 q[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) q[k] = a.p[k] + t * dp[k];
                double d = pair_distance(kd, q[0], q[1], q[2], q[3]);
                if (d <= 1e-9 * e1) {
                    toi = t;
                    break;
                }
            }
        }
    }
    return toi;
}

__global__ void k_full_ccd(const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                           const double* __restrict__ x0, const double* __restrict__ x1, int64_t P,
                           int single, double tol, double* __restrict__ toi_out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    const int4 id = idx[i];
    toi_out[i] = full_ccd_pair(kind[i], gather4(x0, id), gather4(x1, id), single, tol);
}

// gap between the boxes of the two sides at the start positions, minus a
// rounding allowance of 1e-9 x the coordinate magnitude (lower bound on the
// witness distance; <= 0 when undecided)
__device__ __forceinline__ double start_gap(int kd, const Corners& a) {
    const int na = kd == CS_VT ? 1 : 2;
    double alo[3], ahi[3], blo[3], bhi[3], mag = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        alo[c] = blo[c] = INFINITY;
        ahi[c] = bhi[c] = -INFINITY;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double q[3] = {a.p[k].x, a.p[k].y, a.p[k].z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            mag = fmax(mag, fabs(q[c]));
            if (k < na) {
                alo[c] = fmin(alo[c], q[c]);
                ahi[c] = fmax(ahi[c], q[c]);
            } else {
                blo[c] = fmin(blo[c], q[c]);
                bhi[c] = fmax(bhi[c], q[c]);
            }
        }
    }
    double gap = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) gap = fmax(gap, fmax(blo[c] - ahi[c], alo[c] - bhi[c]));
    return gap - 1e-9 * mag;
}

// distance_toi for one pair (ccd.py:221-266)
// Exact shortcut for the conservative-advancement march (ccd.py:251-266): the
// witness distance moves by at most the sides' displacements RELATIVE to a common
// translation c (distances are translation invariant), here c = corner 0's
// displacement, so over t in [0, 1]
//     d(t) >= dmin = d0 - (max_A |dp - c| + max_B |dp - c|)
// (minus a 1e-12 x |coordinate| rounding allowance).  If dmin stays above the hit
// threshold goal (1 + 1e-9), no iteration can hit, and every advance
// (d_k - goal) / L is at least (dmin - goal) / L; if 60 such advances already pass
// t = 1, the march exits through t > 1 (NaN) well before max_iter.  Co-moving
// cloth (rigid rotation with the body) otherwise costs ~L / (0.8 d0) distance
// evaluations per pair for the same NaN.
__device__ __forceinline__ bool march_never_reaches(int kd, const Corners& a, const Corners& b, const d3 dp[4],
                                                    double d0, double goal, double L, int max_iter) {
    if (max_iter < 60) return false;
    const int na = kd == CS_VT ? 1 : 2;
    double ra = 0.0, rb = 0.0, mag = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double r = norm3(dp[k] - dp[0]);
        if (k < na) ra = fmax(ra, r);
        else rb = fmax(rb, r);
        mag = fmax(mag, fmax(fmax(fabs(a.p[k].x), fabs(a.p[k].y)), fabs(a.p[k].z)));
        mag = fmax(mag, fmax(fmax(fabs(b.p[k].x), fabs(b.p[k].y)), fabs(b.p[k].z)));
    }
    const double dmin = d0 * (1.0 - 1e-12) - (ra + rb) * (1.0 + 1e-12) - 1e-12 * mag;
    if (!(dmin > goal * (1.0 + 2e-9))) return false;
    const double step = (dmin - goal) / L;
    return step * 60.0 > 1.0 + 1e-9;
}

// ---- fp32 closest-point directions for the march's relative-motion shortcut.
// Only the DIRECTION of the witness is taken from fp32; the bounds below are
// evaluated in fp64 and are valid for any unit direction n:
//     dist(A, B) >= min_{a in A, b in B} (a - b) . n = min over vertex pairs,
// and dist(A, B) <= |pA - pB| for any pair of points taken on A and B.
struct f3 {
    float x, y, z;
};
__device__ __forceinline__ f3 fsub(f3 a, f3 b) { return f3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ float fdot(f3 a, f3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ float fclip(float v) { return fminf(fmaxf(v, 0.0f), 1.0f); }

// barycentric weights (u of b, v of c) of the closest point of triangle abc to p
__device__ __forceinline__ void pt_tri_weights_f(f3 p, f3 a, f3 b, f3 c, float& u, float& v) {
    const f3 ab = fsub(b, a), ac = fsub(c, a), ap = fsub(p, a), bp = fsub(p, b), cp = fsub(p, c);
    const float d1 = fdot(ab, ap), d2 = fdot(ac, ap), d3v = fdot(ab, bp), d4 = fdot(ac, bp);
    const float d5 = fdot(ab, cp), d6 = fdot(ac, cp);
    u = 0.0f;
    v = 0.0f;
    if (d1 <= 0.0f && d2 <= 0.0f) return;
    if (d3v >= 0.0f && d4 <= d3v) { u = 1.0f; return; }
    if (d6 >= 0.0f && d5 <= d6) { v = 1.0f; return; }
    const float vc = d1 * d4 - d3v * d2;
    if (vc <= 0.0f && d1 >= 0.0f && d3v <= 0.0f) { u = fclip(d1 / (d1 - d3v)); return; }
    const float vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0f && d2 >= 0.0f && d6 <= 0.0f) { v = fclip(d2 / (d2 - d6)); return; }
    const float va = d3v * d6 - d5 * d4;
    const float g1 = d4 - d3v, g2 = d5 - d6;
    if (va <= 0.0f && g1 >= 0.0f && g2 >= 0.0f) {
        const float w = fclip(g1 / (g1 + g2));
        u = 1.0f - w;
        v = w;
        return;
    }
    const float inv = 1.0f / (va + vb + vc);
    u = fclip(vb * inv);
    v = fclip(vc * inv);
    if (u + v > 1.0f) {
        const float sum = u + v;
        u /= sum;
        v /= sum;
    }
}

__device__ __forceinline__ void seg_seg_params_f(f3 a0, f3 a1, f3 b0, f3 b1, float& s, float& t) {
    const f3 da = fsub(a1, a0), db = fsub(b1, b0), r = fsub(a0, b0);
    const float aa = fdot(da, da), ee = fdot(db, db), f = fdot(db, r), c = fdot(da, r), bb = fdot(da, db);
    const float den = aa * ee - bb * bb;
    s = den > 1e-20f ? fclip((bb * f - c * ee) / den) : 0.0f;
    const float traw = ee > 1e-20f ? (bb * s + f) / ee : 0.0f;
    t = fclip(traw);
    if (traw != t) s = aa > 1e-20f ? fclip((bb * t - c) / aa) : 0.0f;
}

// The march's NaN proven without the fp64 witness distance: as march_never_reaches,
// with d0 bracketed by [lower, upper] from an fp32-chosen direction (see above).
// Lower bound on the pair's witness distance over t in [0, 1] (distances are
// translation invariant: d(t) >= d(0) - relative motion), d(0) bracketed from an
// fp32-chosen witness direction; returns -inf when undecided.  d_hi = upper bound on
// d(0); L = upper bound on the reference's march Lipschitz constant.
__device__ __forceinline__ double rel_motion_dmin(int kd, const Corners& a, const Corners& b, double& d_hi,
                                                  double& L) {
    d3 r[4], dp[4];
    double mag = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        r[k] = a.p[k] - a.p[0];  // relative start positions (fp64)
        dp[k] = b.p[k] - a.p[k];
        mag = fmax(mag, fmax(fmax(fabs(a.p[k].x), fabs(a.p[k].y)), fabs(a.p[k].z)));
        mag = fmax(mag, fmax(fmax(fabs(b.p[k].x), fabs(b.p[k].y)), fabs(b.p[k].z)));
    }
    f3 rf[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rf[k] = f3{(float)r[k].x, (float)r[k].y, (float)r[k].z};
    d3 pa, pb;  // fp64 points on side A and side B (valid convex combinations)
    if (kd == CS_VT) {
        float u, v;
        pt_tri_weights_f(rf[0], rf[1], rf[2], rf[3], u, v);
        double ud = u, vd = v;
        const double sum = ud + vd;
        if (sum > 1.0) {  // keep the point inside the triangle (fp32 rounding)
            ud /= sum;
            vd /= sum;
            if (ud + vd > 1.0) vd = 1.0 - ud;
        }
        pa = r[0];
        pb = r[1] + ud * (r[2] - r[1]) + vd * (r[3] - r[1]);
    } else {
        float sp, tp;
        seg_seg_params_f(rf[0], rf[1], rf[2], rf[3], sp, tp);
        pa = r[0] + (double)sp * (r[1] - r[0]);
        pb = r[2] + (double)tp * (r[3] - r[2]);
    }
    const d3 nv = pa - pb;
    const double len = norm3(nv);
    d_hi = INFINITY;
    L = 0.0;
    if (!(len > 0.0)) return -INFINITY;
    const d3 n = (1.0 / len) * nv;
    const int na = kd == CS_VT ? 1 : 2;
    double lb = INFINITY;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (i < na && j >= na) lb = fmin(lb, dot3(r[i] - r[j], n));
    const double slack = 1e-12 * mag;
    const double d_lo = lb * (1.0 - 1e-12) - slack;
    d_hi = len * (1.0 + 1e-12) + slack;
    double ra = 0.0, rb = 0.0, la = 0.0, lbm = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double rel = norm3(dp[k] - dp[0]), mvk = norm3(dp[k]);
        if (k < na) {
            ra = fmax(ra, rel);
            la = fmax(la, mvk);
        } else {
            rb = fmax(rb, rel);
            lbm = fmax(lbm, mvk);
        }
    }
    L = (la + lbm) * (1.0 + 1e-12);  // >= the reference's L
    return d_lo - (ra + rb) * (1.0 + 1e-12) - slack;
}

__device__ __forceinline__ bool march_never_reaches_f32(int kd, const Corners& a, const Corners& b, double floor_frac,
                                                        int max_iter) {
    if (max_iter < 60 || !(floor_frac < 1.0) || !(floor_frac >= 0.0)) return false;
    double d_hi, L;
    const double dmin = rel_motion_dmin(kd, a, b, d_hi, L);
    if (!(L > 0.0)) return false;
    const double goal_hi = floor_frac * d_hi;
    if (!(dmin > goal_hi * (1.0 + 2e-9))) return false;
    return ((dmin - goal_hi) / L) * 60.0 > 1.0 + 1e-9;
}

// full_ccd is NaN when the witness distance provably stays above every validation
// threshold over t in [0, 1] (see separated_sides for the thresholds)
__device__ __forceinline__ bool ccd_never_hits_f32(int kd, const Corners& a, const Corners& b, double tol) {
    double d_hi, L;
    const double dmin = rel_motion_dmin(kd, a, b, d_hi, L);
    if (!(dmin > 0.0)) return false;
    const double ext = pair_extent(a, b);
    const double bound = fmax(tol * fmax(2.0 * ext, 1.0), 1e-9 * fmax(ext, 1.0));
    return dmin > bound * (1.0 + 1e-6) + 1e-12 * (ext + 1.0);
}

__device__ double distance_toi_pair(int kd, const Corners& a, const Corners& b, double floor_frac, int max_iter) {
    d3 dp[4];
    double mv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        dp[k] = b.p[k] - a.p[k];
        mv[k] = norm3(dp[k]);
    }
    // L = max(side-1 displacement) + max(side-2 displacement)  (ccd.py:241-245)
    double la, lb;
    if (kd == CS_VT) {
        la = np_max(np_max(np_max(mv[0], 0.0), 0.0), 0.0);
        lb = np_max(np_max(np_max(0.0, mv[1]), mv[2]), mv[3]);
    } else {
        la = np_max(np_max(np_max(mv[0], mv[1]), 0.0), 0.0);
        lb = np_max(np_max(np_max(0.0, 0.0), mv[2]), mv[3]);
    }
    const double L = la + lb;
    const double NaN = __longlong_as_double(0x7ff8000000000000ULL);
    // exact early-out: the first advance (d - goal) / L already leaves [0, 1]
    // whenever the start-box gap bounds d from below well enough (ccd.py:251-255)
    if (L > 0.0 && floor_frac < 1.0) {
        const double g = start_gap(kd, a);
        if (g > 0.0 && g * (1.0 - floor_frac) * (1.0 - 1e-9) > L * (1.0 + 1e-9)) return NaN;
    }
    double d = pair_distance(kd, a.p[0], a.p[1], a.p[2], a.p[3]);
    const double goal = floor_frac * d;
    if (d > 0.0 && L > 0.0 && march_never_reaches(kd, a, b, dp, d, goal, L, max_iter)) return NaN;
    double toi = NaN;
    if (d <= 0.0) toi = 0.0;
    if (d > 0.0 && L > 0.0) {
        double t = 0.0;
        bool alive = true;
        for (int it = 0; it < max_iter; ++it) {
            t += (d - goal) / L;
            if (!(t <= 1.0)) {
                alive = false;  // left the interval: never reaches the goal
                break;
            }
            d3 q[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = a.p[k] + t * dp[k];
            d = pair_distance(kd, q[0], q[1], q[2], q[3]);
            if (d <= goal * 0x1.000000044b830p+0) {  // goal * (1.0 + 1e-9), ccd.py:261
                toi = t;
                alive = false;
                break;
            }
        }
        if (alive) toi = t;  // unresolved: safe time reached so far
    }
    return toi;
}

__global__ void k_distance_toi(const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                               const double* __restrict__ x0, const double* __restrict__ x1, int64_t P,
                               double floor_frac, int max_iter, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    const int4 id = idx[i];
    out[i] = distance_toi_pair(kind[i], gather4(x0, id), gather4(x1, id), floor_frac, max_iter);
}

// One CCD site's narrow phase (stepper.py:436-441) as filter + worklists.
// k_site_filter settles every pair whose results are provably NaN (the full_ccd
// bound of separated_sides; the distance march's first advance leaving [0, 1],
// or L == 0 where the reference returns 0 only for d <= 0); the rest go to two
// worklists (warp-aggregated appends; results are written by pair index, so
// worklist order is irrelevant).  The heavy kernels then run only over the
// worklists, grid-striding over the device-side counts.
__device__ __forceinline__ void wl_append(bool want, int64_t i, int* __restrict__ wl, int* __restrict__ n) {
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (want) wl[base + __popc(m & ((1u << lane) - 1u))] = (int)i;
}

// Settling works from the broad phase's primitive data of the same site (no
// per-pair corner gathers): margin-inflated swept boxes (vertex / triangle / edge,
// fp32 copies rounded outward - they contain the fp64 boxes, so every gap below
// only shrinks) and per-primitive max displacement norms.  Removing the margin from both boxes
// widens their gap by 2 x margin; the 1e-9 x |coordinate| slack covers the
// rounding of the inflation, so g below is a lower bound on the true gap between
// the two sides' swept (and hence start) positions.
struct SiteBoxes {
    // 64-byte records per vertex / triangle / edge: {lo.xyz, hi.x} {hi.yz, disp, 0}
    // {c.xyz, dev} {p0.xyz, 0} (broad.cu k_vertex_boxes / k_prim_boxes / k_prim_motion)
    const float4* __restrict__ vbox;
    const float4* __restrict__ tbox;
    const float4* __restrict__ ebox;
    double margin;
};

// conservative box (fp32, rounded outward) + max displacement (rounded up)
__device__ __forceinline__ void load_frec(const float4* __restrict__ rec, int p, double lo[3], double hi[3],
                                          double& disp) {
    const float4 a = rec[4 * (int64_t)p], b = rec[4 * (int64_t)p + 1];
    lo[0] = a.x;
    lo[1] = a.y;
    lo[2] = a.z;
    hi[0] = a.w;
    hi[1] = b.x;
    hi[2] = b.y;
    disp = b.z;
}

__global__ void __launch_bounds__(256) k_site_filter(const unsigned long long* __restrict__ keys, int64_t P,
                                                     SiteBoxes B, double tol, double floor_frac, int max_iter,
                                                     double* __restrict__ toi_out, double* __restrict__ filt_out,
                                                     int* __restrict__ wl_full, int* __restrict__ wl_dist,
                                                     int* __restrict__ counts) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool need_full = false, need_dist = false;
    if (i < P) {
        const double NaN = __longlong_as_double(0x7ff8000000000000ULL);
        const unsigned long long k = keys[i];
        const int p = (int)((k >> 32) & 0x7fffffffu), q = (int)(k & 0xffffffffu);
        double alo[3], ahi[3], blo[3], bhi[3], LA, LB;
        if (k >> 63) {
            load_frec(B.ebox, p, alo, ahi, LA);
            load_frec(B.ebox, q, blo, bhi, LB);
        } else {
            load_frec(B.vbox, p, alo, ahi, LA);
            load_frec(B.tbox, q, blo, bhi, LB);
        }
        double gm = -INFINITY, e2 = 0.0, mag = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            gm = fmax(gm, fmax(blo[c] - ahi[c], alo[c] - bhi[c]));
            const double lo = fmin(alo[c], blo[c]), hi = fmax(ahi[c], bhi[c]);
            e2 += (hi - lo) * (hi - lo);
            mag = fmax(mag, fmax(fabs(lo), fabs(hi)));
        }
        const double g = (gm + 2.0 * B.margin) - 1e-9 * mag;
        const double ext = sqrt(e2);
        const double bound = fmax(tol * fmax(2.0 * ext, 1.0), 1e-9 * fmax(ext, 1.0));
        need_full = !(g > bound * (1.0 + 1e-6));
        if (!need_full) toi_out[i] = NaN;
        const double L = (LA + LB) * (1.0 + 1e-12);  // >= the reference's L (records round up)
        bool settled = false;
        if (g > 0.0) {
            if (!(L > 0.0)) settled = L == 0.0;  // d > 0 and L == 0: never alive
            else if (floor_frac < 1.0) settled = g * (1.0 - floor_frac) * (1.0 - 1e-9) > L * (1.0 + 1e-9);
        }
        if (!settled && g > 0.0 && L > 0.0 && floor_frac < 1.0 && floor_frac >= 0.0 && max_iter >= 60) {
            // relative motion (march_never_reaches with record bounds): c = first-vertex
            // displacement, dev = spread around it, p0 = first-vertex start position;
            // d0 <= |pA - pB| (both are points of the pair), every d_k >= g - Lrel
            const float4* RA = (k >> 63) ? B.ebox : B.vbox;
            const float4* RB = (k >> 63) ? B.ebox : B.tbox;
            const float4 ca = RA[4 * (int64_t)p + 2], pa = RA[4 * (int64_t)p + 3];
            const float4 cb = RB[4 * (int64_t)q + 2], pb = RB[4 * (int64_t)q + 3];
            const d3 dc{(double)ca.x - (double)cb.x, (double)ca.y - (double)cb.y, (double)ca.z - (double)cb.z};
            const double cmag = fabs((double)ca.x) + fabs((double)ca.y) + fabs((double)ca.z) + fabs((double)cb.x) +
                                fabs((double)cb.y) + fabs((double)cb.z);
            const double lrel = ((double)ca.w + (double)cb.w + norm3(dc)) * (1.0 + 1e-9) + 1e-6 * cmag;
            const d3 dpp{(double)pa.x - (double)pb.x, (double)pa.y - (double)pb.y, (double)pa.z - (double)pb.z};
            const double d_hi = norm3(dpp) * (1.0 + 1e-9) + 1e-6 * mag;
            const double dmin = g - lrel;
            const double goal_hi = floor_frac * d_hi;
            settled = dmin > goal_hi * (1.0 + 2e-9) && ((dmin - goal_hi) / L) * 60.0 > 1.0 + 1e-9;
        }
        need_dist = !settled;
        if (settled) filt_out[i] = NaN;
    }
    wl_append(need_full, i, wl_full, counts);
    wl_append(need_dist, i, wl_dist, counts + 1);
}

__global__ void __launch_bounds__(128, 4) k_full_ccd_wl(const int* __restrict__ wl, const int* __restrict__ count,
                                                     const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                                                     const double* __restrict__ x0, const double* __restrict__ x1,
                                                     int single, double tol, double* __restrict__ toi_out) {
    const int n = count[0];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = wl[k];
        const int4 id = idx[i];
        const int kd = kind[i];
        const Corners a = gather4(x0, id), b = gather4(x1, id);
        toi_out[i] = ccd_never_hits_f32(kd, a, b, tol) ? __longlong_as_double(0x7ff8000000000000ULL)
                                                       : full_ccd_pair(kd, a, b, single, tol);
    }
}

// distance march over its worklist + the minimum folded with one atomicMin on the
// (non-negative) fp64 bit pattern per block - exact and order independent.
// min_slot must hold +inf before the launch.
__global__ void __launch_bounds__(128, 4) k_distance_toi_wl(const int* __restrict__ wl, const int* __restrict__ count,
                                                         const int8_t* __restrict__ kind,
                                                         const int4* __restrict__ idx, const double* __restrict__ x0,
                                                         const double* __restrict__ x1, double floor_frac,
                                                         int max_iter, double* __restrict__ out,
                                                         unsigned long long* __restrict__ min_slot) {
    const int n = count[0];
    double m = __longlong_as_double(0x7ff0000000000000ULL);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = wl[k];
        const int4 id = idx[i];
        const int kd = kind[i];
        const Corners a = gather4(x0, id), b = gather4(x1, id);
        const double f = march_never_reaches_f32(kd, a, b, floor_frac, max_iter)
                             ? __longlong_as_double(0x7ff8000000000000ULL)
                             : distance_toi_pair(kd, a, b, floor_frac, max_iter);
        out[i] = f;
        if (f == f) m = fmin(m, f);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_down_sync(0xffffffffu, m, o));
    __shared__ double sm[4];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, sm[w]);
        if (m < __longlong_as_double(0x7ff0000000000000ULL))
            atomicMin(min_slot, (unsigned long long)__double_as_longlong(m));
    }
}

// clamp factor from the folded minimum (stepper.py:445-452)
__global__ void k_clamp_from_min(const unsigned long long* __restrict__ min_slot, double alpha,
                                 double* __restrict__ out) {
    const double t = __longlong_as_double((long long)min_slot[0]);
    const bool none = isinf(t);
    out[0] = t;
    out[1] = none ? 1.0 : alpha * t;
    out[2] = (!none && t <= 0.0) ? 1.0 : 0.0;
}

// Witness refresh: bary/params, distance and separating normal (stepper.py:194-216).
// NDB engagement of a fresh pair set fused into its witness pass (stepper.py:483-487,
// 564-565): engaged = full-CCD hit or witness distance < 2 d_hat, weight from the life
// span (k_engage_init's arithmetic); engaged == null: witness only.
struct EngageOut {
    const double* __restrict__ toi;
    const int* __restrict__ life;
    double d_hat, k_ndb, base;
    uint8_t* __restrict__ engaged;
    double* __restrict__ weight;
    int* __restrict__ count;
    // near / far split (the far-pair classification below k_far_gate, from the same toi and distance):
    // near pairs fill split[0, n_near) from the front, far pairs split[n_near, P) from
    // the back, block-aggregated (each block's pairs stay in pair order); null: no split
    int* __restrict__ split;
    int* __restrict__ n_near;
    int* __restrict__ n_far;
    double near_thresh;
};

// block-aggregated two-sided append (one atomic per block and side)
__device__ __forceinline__ void block_split_append(bool valid, bool near, int64_t i, int64_t P,
                                                   int* __restrict__ split, int* __restrict__ n_near,
                                                   int* __restrict__ n_far) {
    __shared__ int sh_pre[2][32];
    __shared__ int sh_base[2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    const unsigned mn = __ballot_sync(0xffffffffu, valid && near);
    const unsigned mf = __ballot_sync(0xffffffffu, valid && !near);
    __syncthreads();
    if (lane == 0) {
        sh_pre[0][w] = __popc(mn);
        sh_pre[1][w] = __popc(mf);
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        int tot = 0;
        for (int k = 0; k < nw; ++k) {
            const int c = sh_pre[threadIdx.x][k];
            sh_pre[threadIdx.x][k] = tot;
            tot += c;
        }
        sh_base[threadIdx.x] = tot ? atomicAdd(threadIdx.x == 0 ? n_near : n_far, tot) : 0;
    }
    __syncthreads();
    if (valid) {
        const int side = near ? 0 : 1;
        const int pos = sh_base[side] + sh_pre[side][w] + __popc((near ? mn : mf) & ((1u << lane) - 1u));
        if (near) split[pos] = (int)i;
        else split[P - 1 - pos] = (int)i;
    }
}
__device__ __forceinline__ double ndb_weight(int life, double k, double base);

__global__ void __launch_bounds__(128, 10) k_witness(const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                          const double* __restrict__ x, int64_t P, double* __restrict__ bary,
                          double* __restrict__ dist, double* __restrict__ normal, double* __restrict__ p1_out,
                          double* __restrict__ p2_out, EngageOut eo) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool eng = false, near = false;
    if (i < P) {
    const int kd = kind[i];
    Corners a = gather4(x, idx[i]);
    d3 p1, p2;
    double l1, l2, d;
    if (kd == CS_VT) {
        d = pt_tri_closest(a.p[0], a.p[1], a.p[2], a.p[3], l1, l2, p2);
        p1 = a.p[0];
    } else {
        d = seg_seg_closest(a.p[0], a.p[1], a.p[2], a.p[3], l1, l2, p1, p2);
    }
    d3 n = p1 - p2;
    double nn = norm3(n);
    if (nn > 1e-12) {
        n = d3{n.x / nn, n.y / nn, n.z / nn};
    } else {
        d3 alt = kd == CS_VT ? cross3(a.p[2] - a.p[1], a.p[3] - a.p[1]) : cross3(a.p[1] - a.p[0], a.p[3] - a.p[2]);
        double an = norm3(alt);
        if (an > 0.0) alt = d3{alt.x / an, alt.y / an, alt.z / an};
        if (an == 0.0) alt = d3{1.0, 0.0, 0.0};
        n = alt;
    }
    bary[2 * i] = l1;
    bary[2 * i + 1] = l2;
    dist[i] = d;
    if (normal) st3(normal, i, n);
    if (p1_out) st3(p1_out, i, p1);
    if (p2_out) st3(p2_out, i, p2);
    if (eo.engaged != nullptr) {
        const double t = eo.toi[i];
        eng = (t == t) || (d < 2.0 * eo.d_hat);
        eo.engaged[i] = eng;
        eo.weight[i] = eng ? ndb_weight(eo.life[i], eo.k_ndb, eo.base) : 0.0;
        near = (t == t) || !(d > eo.near_thresh);
    }
    }
    if (eo.count != nullptr) block_count(eng, eo.count);
    if (eo.split != nullptr) block_split_append(i < P, near, i, P, eo.split, eo.n_near, eo.n_far);
}

__device__ __forceinline__ double ndb_weight(int life, double k, double base) {
    int span = life < 64 ? life : 64;
    double p = (base == 2.0) ? ldexp(1.0, span) : pow(base, (double)span);
    return k * p;
}

// frozen-witness points on both sides at positions x (stepper.py:226-236, 254-263)
__device__ __forceinline__ void witness_sides(int kd, const Corners& q, double l1, double l2, d3& s1, d3& s2) {
    if (kd == CS_VT) {
        s1 = q.p[0];
        s2 = (q.p[1] + l1 * (q.p[2] - q.p[1])) + l2 * (q.p[3] - q.p[1]);
    } else {
        s1 = q.p[0] + l1 * (q.p[1] - q.p[0]);
        s2 = q.p[2] + l2 * (q.p[3] - q.p[2]);
    }
}

// The 4 positional targets of a pair (stepper.py:238-285) from the frozen witness
// (l1, l2, nrm), the gap along nrm at positions q, and the pair weight wp: target
// tg[k], weight w[k] = wp * clip(gamma_k); mov[k] = endpoint k is a free cloth vertex.
__device__ __forceinline__ void pair_stamps(int kd, const Corners& q, int4 id, double l1, double l2, d3 nrm,
                                            double gap, double wp, double d_hat, int n_cloth,
                                            const int* __restrict__ free_index, d3 tg[4], double w[4],
                                            bool mov[4], double g[4]) {
    double deficit = d_hat - gap;
    deficit = (deficit != deficit) ? deficit : (deficit > 0.0 ? deficit : 0.0);
    double gam[4];
    if (kd == CS_VT) {
        gam[0] = 1.0;
        gam[1] = (1.0 - l1) - l2;
        gam[2] = l1;
        gam[3] = l2;
    } else {
        gam[0] = 1.0 - l1;
        gam[1] = l1;
        gam[2] = 1.0 - l2;
        gam[3] = l2;
    }
    const int ids[4] = {id.x, id.y, id.z, id.w};
    bool m1 = false, m2 = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int v = ids[k];
        mov[k] = (v < n_cloth) && (free_index[v < n_cloth ? v : n_cloth - 1] >= 0);
        bool first = (kd == CS_VT) ? (k == 0) : (k < 2);
        if (first) m1 = m1 || mov[k];
        else m2 = m2 || mov[k];
    }
    const bool both = m1 && m2;
    const double sh1 = (both ? 0.5 : (m1 ? 1.0 : 0.0)) * deficit;
    const double sh2 = (both ? 0.5 : (m2 ? 1.0 : 0.0)) * deficit;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        bool first = (kd == CS_VT) ? (k == 0) : (k < 2);
        double mvs = first ? sh1 : -sh2;
        tg[k] = q.p[k] + mvs * nrm;
        g[k] = clip01(gam[k]);
        w[k] = wp * g[k];
    }
}

// a stamp at its cached plan position: dst >= 0 main list, dst <= -2 side list
// (-2 - position), -1 not a plan entry
__device__ __forceinline__ void plan_store(int dst, d3 tg, double w, double4* __restrict__ main_out,
                                           double4* __restrict__ side_out) {
    if (dst >= 0) stg256(main_out + dst, tg.x, tg.y, tg.z, w);
    else if (dst <= -2) stg256(side_out + (-2 - dst), tg.x, tg.y, tg.z, w);
}

// The driver's cached stamp plan as seen by k_partial_ndb (all null: no plan).
struct PlanView {
    const int* pair_u;   // pair -> position in the plan's pair list, -1 outside the plan
    int* n_new;          // count of engaged pairs outside the plan (appended to new_list)
    int* new_list;
    int new_cap;
    const int* dst;      // plan position of entry 4u + k (plan_store encoding)
    double4* main_out;   // fused stamps (null: counting only)
    double4* side_out;
    int n_cloth;
    const int* free_index;
};

struct SamplePattern {
    double vt[6][2];
    double ee[6][2];
    int width;  // max(kv, ke); shorter pattern already padded by repetition
};

// Partial CCD classifier + NDB update of pair i (partial.py:149-204, stepper.py:511-523).
struct NdbArgs {
    const int8_t* __restrict__ kind;
    const int4* __restrict__ idx;
    const double* __restrict__ xa;
    const double* __restrict__ xc;
    SamplePattern pat;
    const double* __restrict__ bary;
    const double* __restrict__ normal;
    double d_hat, k_ndb, base;
    int* __restrict__ life;
    double* __restrict__ weight;
    uint8_t* __restrict__ engaged;
    int write_active;
    uint8_t* __restrict__ active_out;
    int proj_is_witness;
    int* __restrict__ live_count;  // nullable: pairs left with a nonzero life span (the carry's table size)
};

__device__ __forceinline__ void ndb_pair(const NdbArgs& A, const PlanView& plan, int64_t i, bool& eng, bool& fresh,
                                         bool& alive) {
    const int8_t* __restrict__ kind = A.kind;
    const int4* __restrict__ idx = A.idx;
    const double* __restrict__ xa = A.xa;
    const double* __restrict__ xc = A.xc;
    const SamplePattern& pat = A.pat;
    const double* __restrict__ bary = A.bary;
    const double* __restrict__ normal = A.normal;
    const double d_hat = A.d_hat, k_ndb = A.k_ndb, base = A.base;
    int* __restrict__ life = A.life;
    double* __restrict__ weight = A.weight;
    uint8_t* __restrict__ engaged = A.engaged;
    const int write_active = A.write_active, proj_is_witness = A.proj_is_witness;
    uint8_t* __restrict__ active_out = A.active_out;
    const int kd = kind[i];
    const int4 id = idx[i];
    Corners s = gather4(xa, id), e = gather4(xc, id);
    const double w1 = bary[2 * i], w2 = bary[2 * i + 1];
    // projection sample: closest point at the interval start (partial.py:170-178).  In the
    // step the interval starts at the anchor, where the frozen witness (bary) was computed
    // by the same closest-point routines on the same coordinates (stepper.py:483-487,
    // 564-565 -> 511-516): proj_is_witness reuses it bit for bit.
    double pl1, pl2;
    if (proj_is_witness) {
        pl1 = w1;
        pl2 = w2;
    } else {
        d3 tmp1, tmp2;
        if (kd == CS_VT)
            pt_tri_closest(s.p[0], s.p[1], s.p[2], s.p[3], pl1, pl2, tmp1);
        else
            seg_seg_closest(s.p[0], s.p[1], s.p[2], s.p[3], pl1, pl2, tmp1, tmp2);
    }
    d3 be[3], bs[3];
    if (kd == CS_VT) {
        be[0] = e.p[1] - e.p[0]; be[1] = e.p[2] - e.p[1]; be[2] = e.p[3] - e.p[1];
        bs[0] = s.p[1] - s.p[0]; bs[1] = s.p[2] - s.p[1]; bs[2] = s.p[3] - s.p[1];
    } else {
        be[0] = e.p[2] - e.p[0]; be[1] = e.p[0] - e.p[1]; be[2] = e.p[3] - e.p[2];
        bs[0] = s.p[2] - s.p[0]; bs[1] = s.p[0] - s.p[1]; bs[2] = s.p[3] - s.p[2];
    }
    double g[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) g[a][b] = dot3(be[a], bs[b]);
    const double c1 = g[0][1] + g[1][0], c2 = g[0][2] + g[2][0], c12 = g[1][2] + g[2][1];
    bool act = false;
    for (int k = 0; k <= pat.width; ++k) {
        double l1, l2;
        if (k < pat.width) {
            l1 = kd == CS_VT ? pat.vt[k][0] : pat.ee[k][0];
            l2 = kd == CS_VT ? pat.vt[k][1] : pat.ee[k][1];
        } else {
            l1 = pl1;
            l2 = pl2;
        }
        double q = g[0][0] + c1 * l1;
        q = q + c2 * l2;
        q = q + g[1][1] * (l1 * l1);
        q = q + c12 * (l1 * l2);
        q = q + g[2][2] * (l2 * l2);
        act = act || (q <= 0.0);
    }
    // gap along the frozen witness direction at the candidate (stepper.py:218-236)
    d3 s1, s2;
    witness_sides(kd, e, w1, w2, s1, s2);
    const double gap = dot3(s1 - s2, ld3(normal, i));
    act = act || (gap < d_hat);
    int lf = act ? min(life[i] + 1, 64) : 0;
    alive = lf > 0;
    eng = act || (gap < 2.0 * d_hat);
    life[i] = lf;
    engaged[i] = eng;
    const double wnew = eng ? ndb_weight(lf, k_ndb, base) : 0.0;
    weight[i] = wnew;
    if (write_active) active_out[i] = act;
    if (plan.pair_u != nullptr) {
        const int u = plan.pair_u[i];
        fresh = eng && u < 0;
        if (u >= 0 && plan.main_out != nullptr) {
            // fused collision terms of the next LG iteration: same candidate positions,
            // the weight just computed, the driver's cached plan positions
            d3 tg[4];
            double w[4], gg[4];
            bool mov[4];
            pair_stamps(kd, e, id, w1, w2, ld3(normal, i), gap, wnew, d_hat, plan.n_cloth, plan.free_index, tg, w,
                        mov, gg);
            const int4 d = reinterpret_cast<const int4*>(plan.dst)[u];
            plan_store(d.x, tg[0], w[0], plan.main_out, plan.side_out);
            plan_store(d.y, tg[1], w[1], plan.main_out, plan.side_out);
            plan_store(d.z, tg[2], w[2], plan.main_out, plan.side_out);
            plan_store(d.w, tg[3], w[3], plan.main_out, plan.side_out);
        }
    }
}

__device__ __forceinline__ void ndb_counts(const PlanView& plan, int* __restrict__ eng_count,
                                           int* __restrict__ live_count, int64_t i, bool eng, bool fresh, bool alive) {
    if (eng_count != nullptr) block_count(eng, eng_count);
    if (live_count != nullptr) block_count(alive, live_count);
    // engaged pairs outside the driver's stamp plan, appended (any order: the driver
    // sorts their entries by merge key) for the plan merge
    if (plan.n_new != nullptr) {
        const unsigned m = __ballot_sync(0xffffffffu, fresh);
        if (m) {
            const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
            int bpos = 0;
            if (lane == leader) bpos = atomicAdd(plan.n_new, __popc(m));
            bpos = __shfl_sync(0xffffffffu, bpos, leader);
            const int pos = bpos + __popc(m & ((1u << lane) - 1u));
            if (fresh && pos < plan.new_cap) plan.new_list[pos] = (int)i;
        }
    }
}

// One pass per inner LG iteration over all P pairs (wl == null) or over the n pair
// indices of a worklist (the near list of the step's near / far split).
__global__ void __launch_bounds__(128, 6) k_partial_ndb(NdbArgs A, int64_t n, int* __restrict__ eng_count,
                                                        const PlanView plan, const int* __restrict__ wl) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = k < n;
    const int64_t i = !valid ? 0 : (wl != nullptr ? (int64_t)wl[k] : k);
    bool eng = false, fresh = false, alive = false;
    if (valid) ndb_pair(A, plan, i, eng, fresh, alive);
    ndb_counts(plan, eng_count, A.live_count, i, eng, fresh, alive);
}

// The far list of the split (EngageOut.split): a far pair whose witness distance d exceeds
// (2 d_hat + D1 + D2)(1 + 1e-6) + 1e-12, with D1, D2 the largest anchor -> candidate
// displacements of its two sides' vertices (vdisp), is provably inactive and disengaged
// (the split's argument, below): life 0, engaged 0, weight 0 without the classifier.  Two light
// passes (one kernel with the classifier inlined ran the bound check at the
// classifier's register budget and occupancy: 0.62 vs 0.36 ms on the skirt):
// k_far_gate: the displacement bound alone (no classifier inlined, full occupancy for
// a streaming pass); pairs it settles are written inactive and disengaged, the rest
// (bound failed, or in the stamp plan) are appended to a worklist (any order: each
// pair's result is its own, the counts are sums) that k_partial_ndb_dyn runs through
// the full classifier, its length read on the device.
__global__ void __launch_bounds__(256) k_far_gate(NdbArgs A, int64_t n, const PlanView plan,
                                                  const int* __restrict__ wl, const double* __restrict__ dist,
                                                  const double* __restrict__ vdisp, int* __restrict__ rest,
                                                  int* __restrict__ n_rest) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool full = false;
    int i = 0;
    if (k < n) {
        i = wl[k];
        const int4 id = A.idx[i];
        const bool vt = A.kind[i] == CS_VT;
        const double v0 = vdisp[id.x], v1 = vdisp[id.y], v2 = vdisp[id.z], v3 = vdisp[id.w];
        const double D1 = vt ? v0 : fmax(v0, v1), D2 = vt ? fmax(fmax(v1, v2), v3) : fmax(v2, v3);
        const bool in_plan = plan.pair_u != nullptr && plan.pair_u[i] >= 0;
        if (!in_plan && dist[i] > (2.0 * A.d_hat + D1 + D2) * (1.0 + 1e-6) + 1e-12) {
            A.life[i] = 0;
            A.engaged[i] = 0;
            A.weight[i] = 0.0;
        } else {
            full = true;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, full);
    if (m) {
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(n_rest, __popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (full) rest[base + __popc(m & ((1u << lane) - 1u))] = i;
    }
}

__global__ void __launch_bounds__(128, 6) k_partial_ndb_dyn(NdbArgs A, const int* __restrict__ n_dev,
                                                            int* __restrict__ eng_count, const PlanView plan,
                                                            const int* __restrict__ wl) {
    const int64_t n = *n_dev;
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = b0 + threadIdx.x;
        const bool valid = k < n;
        const int64_t i = valid ? (int64_t)wl[k] : 0;
        bool eng = false, fresh = false, alive = false;
        if (valid) ndb_pair(A, plan, i, eng, fresh, alive);
        ndb_counts(plan, eng_count, A.live_count, i, eng, fresh, alive);
    }
}

// Near / far split of a step's pair set at its engagement (anchor = the interval start
// of every partial CCD on this set), classified inside k_witness (EngageOut.split).
// Far: not hit by the full CCD and witness distance d > (2 d_hat + delta)(1 + 1e-6) +
// 1e-12 (delta = kFarDelta d_hat, 0: a larger margin only moved pairs from the cheap
// gate into the classifier, measured).  With D1, D2 the largest anchor -> candidate
// displacements of the two sides' vertices, a far pair with d > 2 d_hat + D1 + D2
// keeps every sampled offset at |o_start| >= d > D1 + D2 >= |o_end - o_start| (so
// Q > 0) and its frozen-witness gap at the candidate at >= d - D1 - D2 > 2 d_hat: the
// classifier finds it inactive and disengaged (life 0, weight 0), which is what
// k_far_gate writes for it (with a relative slack on the bound); the others run the
// classifier.

// |x1 - x0| per world vertex (k_far_gate's displacement bounds)
__global__ void k_vertex_disp_norm(const double* __restrict__ x0, const double* __restrict__ x1, int n,
                                   double* __restrict__ out) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) {
        const double d = norm3(ld3(x1, v) - ld3(x0, v));
        out[v] = d == d ? d : INFINITY;  // NaN: never far
    }
}

// any pair at distance <= 0 (the motion-free exit site's march reports t = 0 exactly
// for those, ccd.py:246-249)
__global__ void k_any_nonpositive(const double* __restrict__ d, int64_t P, int* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool hit = i < P && d[i] <= 0.0;
    if (__any_sync(0xffffffffu, hit) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Engaged set and weights after a full-CCD site (stepper.py:483-487, 564-565).
__global__ void k_engage_init(const double* __restrict__ toi, const double* __restrict__ dist, const int* __restrict__ life,
                              int64_t P, double d_hat, double k_ndb, double base, uint8_t* __restrict__ engaged,
                              double* __restrict__ weight, int* __restrict__ eng_count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool eng = false;
    if (i < P) {
        double t = toi[i];
        eng = (t == t) || (dist[i] < 2.0 * d_hat);
        engaged[i] = eng;
        weight[i] = eng ? ndb_weight(life[i], k_ndb, base) : 0.0;
    }
    if (eng_count != nullptr) block_count(eng, eng_count);
}

// Per engaged pair: 4 positional targets (stepper.py:238-285).  Entries for
// immovable or zero-weight endpoints get key 0x7fffffff (sorted to the end).
// key == nullptr: payload only, for every entry of the driver's cached stamp plan, at
// its plan position plan_dst[4a + k] (pairs no longer engaged get w = 0).
__global__ void __launch_bounds__(256, 4) k_collision_terms(const int* __restrict__ sel, int64_t A, const int8_t* __restrict__ kind,
                                  const int4* __restrict__ idx, const double* __restrict__ xw,
                                  const double* __restrict__ bary, const double* __restrict__ normal,
                                  const double* __restrict__ weight, double d_hat, int n_cloth,
                                  const int* __restrict__ free_index, int cloth_only,
                                  int* __restrict__ key, double4* __restrict__ stamp_out,
                                  const int* __restrict__ plan_dst, double4* __restrict__ side_out) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= A) return;
    const int i = sel[a];
    const int kd = kind[i];
    const int4 id = idx[i];
    Corners q = gather4(xw, id);
    const double l1 = bary[2 * i], l2 = bary[2 * i + 1];
    d3 s1, s2;
    witness_sides(kd, q, l1, l2, s1, s2);
    const d3 nrm = ld3(normal, i);
    const double gap = dot3(s1 - s2, nrm);
    d3 tg[4];
    double w[4], g[4];
    bool mov[4];
    pair_stamps(kd, q, id, l1, l2, nrm, gap, weight[i], d_hat, n_cloth, free_index, tg, w, mov, g);
    const int ids[4] = {id.x, id.y, id.z, id.w};
    if (key == nullptr) {
        const int4 d = reinterpret_cast<const int4*>(plan_dst)[a];
        plan_store(d.x, tg[0], w[0], stamp_out, side_out);
        plan_store(d.y, tg[1], w[1], stamp_out, side_out);
        plan_store(d.z, tg[2], w[2], stamp_out, side_out);
        plan_store(d.w, tg[3], w[3], stamp_out, side_out);
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        bool keep = mov[k] && (w[k] > 0.0);
        if (cloth_only && ids[k] >= n_cloth) keep = false;
        int64_t o = 4 * a + k;
        key[o] = keep ? free_index[ids[k]] : 0x7fffffff;
        if (keep) stg256(stamp_out + o, tg[k].x, tg[k].y, tg[k].z, w[k]);  // others are never read
    }
}

// min over non-NaN TOIs; flag any TOI <= 0 (stepper.py:445-452).  Two passes.
__global__ void k_min_toi_partial(const double* __restrict__ toi, int64_t P, double* __restrict__ part) {
    __shared__ double sm[256];
    double m = __longlong_as_double(0x7ff0000000000000ULL);  // +inf
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        double t = toi[i];
        if (t == t && t < m) m = t;
    }
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sm[threadIdx.x] = fmin(sm[threadIdx.x], sm[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_min_toi_final(const double* __restrict__ part, int nparts, double alpha, double* __restrict__ out) {
    __shared__ double sm[256];
    double m = __longlong_as_double(0x7ff0000000000000ULL);
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) m = fmin(m, part[i]);
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sm[threadIdx.x] = fmin(sm[threadIdx.x], sm[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double t = sm[0];
        // out[0] = min toi (inf if none), out[1] = clamp factor (1 if none), out[2] = penetration flag
        out[0] = t;
        bool none = isinf(t);
        out[1] = none ? 1.0 : alpha * t;
        out[2] = (!none && t <= 0.0) ? 1.0 : 0.0;
    }
}

}  // namespace cs
