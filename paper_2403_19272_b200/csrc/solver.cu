// Global-step solver kernels (fp64, HBM/L2-bound).
//
//   k_inertia_target   reference mesh.py:174-196
//   k_assemble_rhs     reference constraints.py:212-256 (edge projection owner-computes,
//                      pinned columns, sorted collision stamps) - bitwise the reference's
//                      np.add.at order for the elastic part
//   k_jacobi_a/_b      reference smoothing.py:23-66: one rank-2 aggregated step =
//                      two SELL-32 SpMV passes; bitwise the reference's CSR order
//   k_project_partial  U^T r / V^T r tall-skinny reduction (subspace.py:179-180, 191)
//                      fused with the residual SpMV; warp lanes own basis columns
//   k_gram_partial     sum_j w_j V_j V_j^T over collided rows (subspace.py:97-106)
//   k_reduced_solve    one CTA: reduce partials, A = diag(lambda)+G, beta-scaled LU
//                      inverse with residual check and symmetric-eigen pinv fallback
//                      (subspace.py:122-140), q = beta X rhs
//   k_prolong          x += B q (subspace.py:186, 192)
//   k_energy_grad      reference stepper.py:309-380 gradient ("quad" collision form)
//
// H (free x free) is stored SELL-32: slices of 32 rows, column-major inside the
// slice, per-slice width = longest row; padding col = -1.  Columns keep CSR order
// so every row sum is evaluated in scipy's order.
#include "common.cuh"

namespace cs {

struct Sell {
    int nrows;
    int nslices;
    const int* __restrict__ slice_ptr;  // (nslices+1) element offsets
    const int* __restrict__ col;
    const double* __restrict__ val;
};

// y_row = H[row, :] @ x (3 right-hand sides), scipy csr_matvecs order.
// Padding sits only at the end of a row (col = -1), so skipping it keeps the
// sequential CSR summation order.  The (col, val) stream is read 4 slots at a time
// with all loads issued before the dependent x gathers (memory-level parallelism
// instead of a load-use chain per nonzero).
__device__ __forceinline__ d3 sell_row(const Sell& H, int row, const double* __restrict__ x) {
    const int s = row >> 5, lane = row & 31;
    const int beg = H.slice_ptr[s], width = (H.slice_ptr[s + 1] - beg) >> 5;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const int* cp = H.col + beg + lane;
    const double* vp = H.val + beg + lane;
    int k = 0;
    if (width <= 16) {
        // whole row in flight: 16 (col, val) loads, then 16 x gathers, then the ordered sum
        int c[16];
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            c[u] = u < width ? __ldg(cp + 32 * u) : -1;
            v[u] = u < width ? __ldg(vp + 32 * u) : 0.0;
        }
        double g[16][3];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int cc = c[u] < 0 ? 0 : c[u];
            if (c[u] >= 0) {
                g[u][0] = __ldg(x + 3 * cc);
                g[u][1] = __ldg(x + 3 * cc + 1);
                g[u][2] = __ldg(x + 3 * cc + 2);
            } else {
                g[u][0] = g[u][1] = g[u][2] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (c[u] >= 0) {
                a0 = a0 + v[u] * g[u][0];
                a1 = a1 + v[u] * g[u][1];
                a2 = a2 + v[u] * g[u][2];
            }
        }
        return d3{a0, a1, a2};
    }
    for (; k + 4 <= width; k += 4) {
        int c[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            c[u] = __ldg(cp + 32 * (k + u));
            v[u] = __ldg(vp + 32 * (k + u));
        }
        double g[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int cc = c[u] < 0 ? 0 : c[u];
            g[u][0] = __ldg(x + 3 * cc);
            g[u][1] = __ldg(x + 3 * cc + 1);
            g[u][2] = __ldg(x + 3 * cc + 2);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (c[u] >= 0) {
                a0 = a0 + v[u] * g[u][0];
                a1 = a1 + v[u] * g[u][1];
                a2 = a2 + v[u] * g[u][2];
            }
        }
    }
    for (; k < width; ++k) {
        const int c = __ldg(cp + 32 * k);
        if (c < 0) break;
        const double v = __ldg(vp + 32 * k);
        a0 = a0 + v * __ldg(x + 3 * c);
        a1 = a1 + v * __ldg(x + 3 * c + 1);
        a2 = a2 + v * __ldg(x + 3 * c + 2);
    }
    return d3{a0, a1, a2};
}

// ---------------------------------------------------------------- inertia target
__global__ void k_inertia_target(const double* __restrict__ x, const double* __restrict__ v,
                                 const double* __restrict__ fext, const double* __restrict__ df,
                                 const double* __restrict__ mass, int n, double h,
                                 const int* __restrict__ pin_slot, const double* __restrict__ pins,
                                 double* __restrict__ z, int* __restrict__ bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double hh = h * h, m = mass[i];
    double o[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double a = x[3 * i + c] + h * v[3 * i + c];
        o[c] = a + (hh * (fext[3 * i + c] + df[3 * i + c])) / m;
    }
    const int ps = pin_slot[i];
    if (ps >= 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c] = pins[3 * ps + c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (!isfinite(o[c])) *bad = 1;
        z[3 * i + c] = o[c];
    }
}

// ---------------------------------------------------------------- rhs
// Per free vertex i: b_i = (sum_incident +-w y_e) + M/h^2 z_i - (H_fp pins)_i,
// then collision stamps delta_i += w, b_i += w t in pair order.
// inc_ptr/inc_edge/inc_sign: vertex->edge incidence, edges where the vertex is
// endpoint 0 first (edge order) then endpoint 1 (edge order) = np.add.at order.
// the stamp plan's side list (recently joined pairs, row-sorted by merge key) and the
// main list's merge keys; seg_beg == null: no side list
struct StampSide {
    const int* __restrict__ seg_beg;
    const int* __restrict__ seg_end;
    const unsigned long long* __restrict__ key;
    const double4* __restrict__ stamp;
    const unsigned long long* __restrict__ main_key;
};

struct EdgeSet {
    const int* __restrict__ e0;
    const int* __restrict__ e1;
    const double* __restrict__ rest;
    const double* __restrict__ w;
};

__device__ __forceinline__ d3 edge_projection(const double* __restrict__ x, int a, int b, double rest) {
    const d3 xa = ld3(x, a), xb = ld3(x, b);
    const d3 d = xb - xa;
    const double len = norm3(d);
    const d3 unit = len > 0.0 ? d3{d.x / len, d.y / len, d.z / len} : d3{1.0, 0.0, 0.0};
    const d3 mid = 0.5 * (xa + xb);
    const d3 half = (0.5 * rest) * unit;
    return (mid + half) - (mid - half);
}

__global__ void k_assemble_rhs(int nf, const int* __restrict__ free_ids, const double* __restrict__ x,
                               const double* __restrict__ z, const double* __restrict__ mh2, EdgeSet E,
                               const int* __restrict__ inc_ptr, const int* __restrict__ inc_edge,
                               const int* __restrict__ fp_ptr, const int* __restrict__ fp_col,
                               const double* __restrict__ fp_val, const double* __restrict__ pins,
                               const int* __restrict__ seg_beg, const int* __restrict__ seg_end,
                               const int* __restrict__ stamp_src, const double4* __restrict__ stamp,
                               double* __restrict__ b,
                               double* __restrict__ delta, StampSide side) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int v = free_ids[i];
    d3 acc{0.0, 0.0, 0.0};
    for (int k = inc_ptr[v]; k < inc_ptr[v + 1]; ++k) {
        const int code = inc_edge[k];
        const int e = code >> 1;
        const double w = E.w[e];
        const d3 y = edge_projection(x, E.e0[e], E.e1[e], E.rest[e]);
        const double s = (code & 1) ? w : -w;  // endpoint 1 gets +w y, endpoint 0 gets (-w) y
        acc = acc + s * y;
    }
    const double m = mh2[i];
    d3 bi = acc + m * ld3(z, v);
    if (fp_ptr != nullptr) {
        double h0 = 0.0, h1 = 0.0, h2 = 0.0;
        for (int k = fp_ptr[i]; k < fp_ptr[i + 1]; ++k) {
            const double a = fp_val[k];
            const int c = fp_col[k];
            h0 = h0 + a * pins[3 * c];
            h1 = h1 + a * pins[3 * c + 1];
            h2 = h2 + a * pins[3 * c + 2];
        }
        bi = bi - d3{h0, h1, h2};
    }
    double dl = 0.0;
    if (seg_beg != nullptr) {
        int k = seg_beg[i];
        const int ke = seg_end[i];
        int q = 0, qe = 0;
        if (side.seg_beg != nullptr) {
            q = side.seg_beg[i];
            qe = side.seg_end[i];
        }
        if (q == qe) {
            // main list only, 4 stamps in flight per step (the sums stay sequential)
            for (; k + 4 <= ke; k += 4) {
                double4 st[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) st[u] = ldg256(stamp + (stamp_src != nullptr ? stamp_src[k + u] : k + u));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double w = st[u].w;
                    if (!(w > 0.0)) continue;
                    dl = dl + w;
                    bi = bi + w * d3{st[u].x, st[u].y, st[u].z};
                }
            }
        }
        while (k < ke || q < qe) {
            // entry order (gather through the row sort) or plan order (stamp_src == null:
            // streamed); a row with side-list entries interleaves both lists by merge key
            const bool from_main = q >= qe || (k < ke && side.main_key[k] < side.key[q]);
            const double4 st = ldg256(from_main ? stamp + (stamp_src != nullptr ? stamp_src[k] : k) : side.stamp + q);
            k += from_main ? 1 : 0;
            q += from_main ? 0 : 1;
            const double w = st.w;
            if (!(w > 0.0)) continue;  // plan entry of a pair that left the engaged set
            dl = dl + w;
            bi = bi + w * d3{st.x, st.y, st.z};
        }
    }
    st3(b, i, bi);
    delta[i] = dl;
}

// ---------------------------------------------------------------- A-Jacobi
// pass A: t = D^-1 (b - (H x + delta x)); optional per-block sum of r^2.
__global__ void k_jacobi_a(Sell H, const double* __restrict__ diag, const double* __restrict__ delta,
                           const double* __restrict__ b, const double* __restrict__ x, double* __restrict__ t,
                           double* __restrict__ norm_part) {
    __shared__ double red[8];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double r2 = 0.0;
    if (i < H.nrows) {
        const d3 hx = sell_row(H, i, x);
        const double dl = delta[i];
        const double inv = 1.0 / (diag[i] + dl);
        const d3 xi = ld3(x, i);
        const d3 r = ld3(b, i) - (hx + dl * xi);
        st3(t, i, inv * r);
        if (norm_part) r2 = fma(r.z, r.z, fma(r.y, r.y, r.x * r.x));
    }
    if (norm_part) {  // deterministic block tree
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
        __syncthreads();
        if (threadIdx.x < 32) {
            double s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (threadIdx.x == 0) norm_part[blockIdx.x] = s;
        }
    }
}

// pass B: x += c (2 t - c D^-1 (H t + delta t))
__global__ void k_jacobi_b(Sell H, const double* __restrict__ diag, const double* __restrict__ delta,
                           const double* __restrict__ t, double c, double* __restrict__ x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H.nrows) return;
    const d3 ht = sell_row(H, i, t);
    const double dl = delta[i];
    const double inv = 1.0 / (diag[i] + dl);
    const d3 ti = ld3(t, i);
    const d3 out = ht + dl * ti;
    const d3 upd = c * ((2.0 * ti) - c * (inv * out));
    st3(x, i, ld3(x, i) + upd);
}

// ---------------------------------------------------------------- Chebyshev (opt-in)
// Chebyshev-accelerated Jacobi for (H + delta) x = b, D = diag + delta: one fused SELL
// pass per iteration - SpMV, the Jacobi residual step, the three-term Chebyshev
// extrapolation and (when norm_part) the residual-norm block partials:
//   x_{k+1} = w_{k+1} (g D^-1 (b - (H + delta) x_k) + x_k - x_{k-1}) + x_{k-1}
// (x_{-1} = x_0, w_1 = 1).  Not the reference's smoother: opt-in only.
__global__ void k_cheb_step(Sell H, const double* __restrict__ diag, const double* __restrict__ delta,
                            const double* __restrict__ b, const double* __restrict__ xk,
                            const double* __restrict__ xkm1, double w, double g, double* __restrict__ xk1,
                            double* __restrict__ norm_part) {
    __shared__ double red[8];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double r2 = 0.0;
    if (i < H.nrows) {
        const d3 hx = sell_row(H, i, xk);
        const double dl = delta[i];
        const double inv = 1.0 / (diag[i] + dl);
        const d3 xi = ld3(xk, i), xp = ld3(xkm1, i);
        const d3 r = ld3(b, i) - (hx + dl * xi);
        st3(xk1, i, w * ((g * (inv * r) + xi) - xp) + xp);
        if (norm_part) r2 = fma(r.z, r.z, fma(r.y, r.y, r.x * r.x));
    }
    if (norm_part) {
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
        __syncthreads();
        if (threadIdx.x < 32) {
            double s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if (threadIdx.x == 0) norm_part[blockIdx.x] = s;
        }
    }
}

// Gershgorin radius of D^-1 H: max_i sum_{j != i} |h_ij| / h_ii (block maxima); the
// Chebyshev interval is [1 - rho, 1 + rho] (delta >= 0 only shrinks it)
__global__ void k_gershgorin(Sell H, const double* __restrict__ diag, double* __restrict__ part) {
    __shared__ double sm[256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double rho = 0.0;
    if (i < H.nrows) {
        const int s = i >> 5, lane = i & 31;
        const int beg = H.slice_ptr[s], width = (H.slice_ptr[s + 1] - beg) >> 5;
        double off = 0.0;
        for (int k = 0; k < width; ++k) {
            const int c = H.col[beg + 32 * k + lane];
            if (c >= 0 && c != i) off += fabs(H.val[beg + 32 * k + lane]);
        }
        rho = off / diag[i];
    }
    sm[threadIdx.x] = rho;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// out = x + c t (jacobi_step's update, smoothing.py:78)
__global__ void k_axpy_step(const double* __restrict__ x, const double* __restrict__ t, double c, int64_t n,
                            double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = x[i] + c * t[i];
}

// divergence guard between the k=0 and k=10 residual norms (smoothing.py:57-63)
__global__ void k_norm_final(const double* __restrict__ part, int nparts, double* __restrict__ slot) {
    __shared__ double sm[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *slot = sqrt(sm[0]);
}

// ---------------------------------------------------------------- basis projection
// part[blk][3 j + c] = sum over the block's rows of B[row, j] * res[row][c], where
// res = b - H x - delta x (delta may be null) or res = b (x null).
// Persistent: block b takes row tiles b, b + grid, ...  Per tile, every thread computes
// one row's residual (SELL row, scipy order) into shared memory while the tile's B rows
// are staged there by 16-byte loads (row stride rb | 1); then output (j, c) of group g
// accumulates the tile rows i = g (mod G) in order.  Block partial = groups summed in
// order; the partials are summed in order by k_reduce_partials.
__host__ __device__ constexpr int proj_rows(int rb) { return rb <= 32 ? 256 : 64; }
__host__ constexpr size_t proj_smem(int rb) {
    return sizeof(double) * ((size_t)proj_rows(rb) * (rb | 1) + 3 * (size_t)proj_rows(rb) + 2 * 3 * 128);
}
__global__ void __launch_bounds__(256) k_project_partial(Sell H, const double* __restrict__ b,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ delta,
                                                         const double* __restrict__ B, int rb,
                                                         double* __restrict__ part) {
    extern __shared__ double psm[];
    const int TR = proj_rows(rb), rbp = rb | 1, O = 3 * rb;
    double* sB = psm;                         // [TR][rbp]
    double* res = psm + (size_t)TR * rbp;     // [TR][3]
    double* red = res + 3 * TR;               // [2][3 * 128] group partials
    const int G = O <= 128 ? 2 : 1;           // row groups (rb = 30: 2 x 90 outputs)
    const int t = threadIdx.x;
    const int grp = G == 2 ? (t >= 128 ? 1 : 0) : 0;
    const int o0 = G == 2 ? (t & 127) : t;    // first output of this thread
    double acc0 = 0.0, acc1 = 0.0;            // outputs o0 and o0 + 256 (rb = 120)
    const int ntiles = (H.nrows + TR - 1) / TR;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tile0 = tile * TR;
        const int nr = min(TR, H.nrows - tile0);
        __syncthreads();
        // stage B rows (16-byte loads; tile0 * rb is even)
        const int tot = nr * rb, tot2 = tot >> 1;
        const double2* src2 = reinterpret_cast<const double2*>(B + (int64_t)tile0 * rb);
        for (int e0 = t; e0 < tot2; e0 += 4 * 256) {
            double2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e2 = e0 + u * 256;
                v[u] = e2 < tot2 ? __ldg(src2 + e2) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e2 = e0 + u * 256;
                if (e2 < tot2) {
                    const int e = 2 * e2, ra = e / rb, rb1 = (e + 1) / rb;
                    sB[ra * rbp + (e - ra * rb)] = v[u].x;
                    sB[rb1 * rbp + (e + 1 - rb1 * rb)] = v[u].y;
                }
            }
        }
        if ((tot & 1) && t == 0) {
            const int e = tot - 1, ra = e / rb;
            sB[ra * rbp + (e - ra * rb)] = __ldg(B + (int64_t)tile0 * rb + e);
        }
        // residual rows
        for (int rr = t; rr < nr; rr += 256) {
            const int i = tile0 + rr;
            d3 v;
            if (x != nullptr) {
                const d3 hx = sell_row(H, i, x);
                v = ld3(b, i) - hx;
                if (delta != nullptr) v = v - delta[i] * ld3(x, i);
            } else {
                v = ld3(b, i);
            }
            res[3 * rr] = v.x;
            res[3 * rr + 1] = v.y;
            res[3 * rr + 2] = v.z;
        }
        __syncthreads();
        if (o0 < O) {
            const int j = o0 / 3, c = o0 - 3 * j;
            for (int rr = grp; rr < nr; rr += G) acc0 = fma(sB[rr * rbp + j], res[3 * rr + c], acc0);
        }
        if (o0 + 256 < O) {
            const int o1 = o0 + 256, j = o1 / 3, c = o1 - 3 * j;
            for (int rr = 0; rr < nr; ++rr) acc1 = fma(sB[rr * rbp + j], res[3 * rr + c], acc1);
        }
    }
    __syncthreads();
    if (o0 < O) red[grp * 384 + o0] = acc0;
    if (o0 + 256 < O) red[o0 + 256] = acc1;
    __syncthreads();
    for (int o = t; o < O; o += 256)
        part[(int64_t)blockIdx.x * O + o] = G == 2 ? red[o] + red[384 + o] : red[o];
}

// G partials over the ascending list of collided rows (count read on device):
// block b owns a contiguous chunk of the list.  Rows are staged 64 at a time in
// shared memory (V_i and delta_i V_i, padded to 32 columns; the next tile's loads are
// in flight while the current one is consumed).  The 256 threads form 4 groups; each
// thread of a group owns a 4x4 register tile of the 32x32 output and accumulates the
// group's rows (every 4th row of a tile) in order, s = fma(V_ia, delta_i V_ib, s); the
// block partial is ((g0 + g1) + g2) + g3 - a fixed order, so run-to-run deterministic.
constexpr int kGramThreads = 256;
__global__ void __launch_bounds__(kGramThreads) k_gram_partial(const int* __restrict__ rows,
                                                               const int* __restrict__ nrows_ptr,
                                                               const double* __restrict__ delta,
                                                               const double* __restrict__ V, int r,
                                                               double* __restrict__ part,
                                                               const double* __restrict__ wlist = nullptr) {
    // weight of list entry j: delta[rows[j]] (the step), or wlist[j] (reduced_update's
    // explicit (active_vertices, weights), subspace.py:97-106)
    constexpr int kT = 64;
    constexpr int kPer = kT * 32 / kGramThreads;
    __shared__ __align__(16) double sbuf[2][kT][32];
    double(&sv)[kT][32] = sbuf[0];
    double(&sw)[kT][32] = sbuf[1];
    const int cnt = *nrows_ptr;
    const int per = (cnt + gridDim.x - 1) / gridDim.x;
    const int beg = min(cnt, (int)blockIdx.x * per);
    const int end = min(cnt, beg + per);
    const int t = threadIdx.x, grp = t >> 6;
    const int ta = ((t & 63) >> 3) * 4, tb = (t & 7) * 4;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    double v[kPer], d[kPer];
    auto load = [&](int t0) {
        const int nt = min(kT, end - t0);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = t + u * kGramThreads, k = e >> 5, c = e & 31;
            v[u] = 0.0;
            d[u] = 0.0;
            if (k < nt && c < r) {
                const int row = rows[t0 + k];
                v[u] = V[(int64_t)row * r + c];
                d[u] = wlist != nullptr ? wlist[t0 + k] : delta[row];
            }
        }
    };
    if (beg < end) load(beg);
    for (int t0 = beg; t0 < end; t0 += kT) {
        const int nt = min(kT, end - t0);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int e = t + u * kGramThreads, k = e >> 5, c = e & 31;
            sv[k][c] = v[u];
            sw[k][c] = d[u] * v[u];
        }
        __syncthreads();
        if (t0 + kT < end) load(t0 + kT);
        for (int k = grp; k < nt; k += 4) {
            const double2 a01 = *reinterpret_cast<const double2*>(&sv[k][ta]);
            const double2 a23 = *reinterpret_cast<const double2*>(&sv[k][ta + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&sw[k][tb]);
            const double2 b23 = *reinterpret_cast<const double2*>(&sw[k][tb + 2]);
            const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
    }
    // group partials -> shared (sv and sw hold 4 x 32 x 32 doubles), summed in group order
    __syncthreads();
    double* red = &sbuf[0][0][0];  // [grp][a * 32 + b]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[grp * 1024 + (ta + i) * 32 + tb + j] = acc[i][j];
    __syncthreads();
    for (int o = t; o < r * r; o += kGramThreads) {
        const int a = o / r, b2 = o - a * r, q = a * 32 + b2;
        part[(int64_t)blockIdx.x * r * r + o] = ((red[q] + red[1024 + q]) + red[2048 + q]) + red[3072 + q];
    }
}

// ---------------------------------------------------------------- reduced solve (one CTA)
// state layout (persisted per scene): X[r*r] scaled inverse, beta, flags
struct ReducedState {
    double* X;      // r*r, A X = I / beta
    double* beta;   // 1
    int* fallback;  // 1 (pinv used)
};

__device__ void jacobi_eig_pinv(double* A, double* Q, double* w, int r, double* out) {
    // cyclic Jacobi on symmetric A (r x r, smem); Q accumulates eigenvectors
    const int tid = threadIdx.x;
    for (int o = tid; o < r * r; o += blockDim.x) Q[o] = (o / r == o % r) ? 1.0 : 0.0;
    __syncthreads();
    __shared__ double cs_sn[2];
    __shared__ int conv;
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (tid == 0) {
            double off = 0.0, tot = 0.0;
            for (int a = 0; a < r; ++a)
                for (int c = 0; c < r; ++c) {
                    double v = A[a * r + c] * A[a * r + c];
                    tot += v;
                    if (a != c) off += v;
                }
            conv = off <= 1e-30 * tot;
        }
        __syncthreads();
        if (conv) break;
        for (int p = 0; p < r - 1; ++p)
            for (int q = p + 1; q < r; ++q) {
                if (tid == 0) {
                    double apq = A[p * r + q];
                    double c = 1.0, s = 0.0;
                    if (fabs(apq) > 0.0) {
                        double theta = (A[q * r + q] - A[p * r + p]) / (2.0 * apq);
                        double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                    cs_sn[0] = c;
                    cs_sn[1] = s;
                }
                __syncthreads();
                const double c = cs_sn[0], s = cs_sn[1];
                if (s != 0.0) {
                    // rotate rows p,q then columns p,q
                    for (int k = tid; k < r; k += blockDim.x) {
                        double ap = A[p * r + k], aq = A[q * r + k];
                        A[p * r + k] = c * ap - s * aq;
                        A[q * r + k] = s * ap + c * aq;
                    }
                    __syncthreads();
                    for (int k = tid; k < r; k += blockDim.x) {
                        double ap = A[k * r + p], aq = A[k * r + q];
                        A[k * r + p] = c * ap - s * aq;
                        A[k * r + q] = s * ap + c * aq;
                        double qp = Q[k * r + p], qq = Q[k * r + q];
                        Q[k * r + p] = c * qp - s * qq;
                        Q[k * r + q] = s * qp + c * qq;
                    }
                }
                __syncthreads();
            }
    }
    for (int k = tid; k < r; k += blockDim.x) w[k] = A[k * r + k];
    __syncthreads();
    __shared__ double wmax;
    if (tid == 0) {
        double m = 0.0;
        for (int k = 0; k < r; ++k) m = fmax(m, fabs(w[k]));
        wmax = m;
    }
    __syncthreads();
    // numpy pinv: singular values below rcond(1e-15) * max are dropped
    for (int o = tid; o < r * r; o += blockDim.x) {
        const int a = o / r, c = o % r;
        double s = 0.0;
        for (int k = 0; k < r; ++k)
            if (fabs(w[k]) > 1e-15 * wmax) s += Q[a * r + k] * (1.0 / w[k]) * Q[c * r + k];
        out[o] = s;
    }
    __syncthreads();
}

// mode 0: reuse-basis reduced correction (factor if refactor != 0)
// mode 1: warm-start (q = rhs / lambda)
__global__ void __launch_bounds__(256) k_reduced_solve(const double* __restrict__ rhs_in,
                                                       const double* __restrict__ gram_in,
                                                       const double* __restrict__ lam, int rb, int mode,
                                                       int refactor, ReducedState st, double* __restrict__ q_out,
                                                       double beta_given = -1.0) {
    // beta_given >= 0: build_reduced(sub, G, rhs_scale) - beta = rhs_scale (1 if <= 0),
    // factor only (q_out unused)
    __shared__ double rhs[3 * 128];
    __shared__ double A[32 * 32], LU[32 * 32], X[32 * 32], Q[32 * 32], wv[32];
    __shared__ int piv[32];
    __shared__ double beta_sm;
    __shared__ int singular;
    const int tid = threadIdx.x;
    for (int o = tid; o < 3 * rb; o += blockDim.x) rhs[o] = rhs_in[o];
    __syncthreads();
    if (mode == 1) {
        for (int o = tid; o < 3 * rb; o += blockDim.x) q_out[o] = rhs[o] / lam[o / 3];
        return;
    }
    const int r = rb;
    if (refactor) {
        for (int o = tid; o < r * r; o += blockDim.x) {
            const double g = gram_in != nullptr ? gram_in[o] : 0.0;
            const int a = o / r, c = o % r;
            // np.diag(lambda) + G  (symmetrised like the dense BLAS product)
            A[o] = (a == c ? lam[a] : 0.0) + g;
        }
        __syncthreads();
        if (tid == 0) {
            double bt = beta_given;
            if (bt < 0.0) {
                double s = 0.0;
                for (int o = 0; o < 3 * r; ++o) s += fabs(rhs[o]);
                bt = s / (3.0 * r);
            }
            beta_sm = bt > 0.0 ? bt : 1.0;
            singular = 0;
        }
        for (int o = tid; o < r * r; o += blockDim.x) LU[o] = A[o];
        __syncthreads();
        // LU with partial pivoting (LAPACK getrf semantics: the first row of largest |a_ik|,
        // scanning down from the diagonal with strict >; a NaN diagonal keeps row k)
        const int lane = tid & 31;
        for (int k = 0; k < r; ++k) {
            if (tid < 32) {
                const int i2 = k + lane;
                double v = (i2 < r) ? fabs(LU[i2 * r + k]) : -1.0;
                const double vk = __shfl_sync(0xffffffffu, v, 0);
                if (!(v == v)) v = -1.0;  // NaN below the diagonal never wins the strict > scan
                int p = i2;
                for (int o = 16; o > 0; o >>= 1) {
                    const double v2 = __shfl_down_sync(0xffffffffu, v, o);
                    const int p2 = __shfl_down_sync(0xffffffffu, p, o);
                    if (v2 > v || (v2 == v && p2 < p)) {
                        v = v2;
                        p = p2;
                    }
                }
                if (lane == 0) {
                    if (!(vk == vk)) p = k;
                    piv[k] = p;
                    if ((vk == vk ? v : vk) == 0.0) singular = 1;
                }
            }
            __syncthreads();
            const int p = piv[k];
            if (p != k && tid < r) {
                const double tmp = LU[k * r + tid];
                LU[k * r + tid] = LU[p * r + tid];
                LU[p * r + tid] = tmp;
            }
            __syncthreads();
            const double pv = LU[k * r + k];
            for (int i2 = k + 1 + tid; i2 < r; i2 += blockDim.x) LU[i2 * r + k] = pv != 0.0 ? LU[i2 * r + k] / pv : 0.0;
            __syncthreads();
            // rank-1 update: lane = column, warps stride the rows (r <= 32)
            {
                const int c = k + 1 + lane;
                if (c < r)
                    for (int i2 = k + 1 + (tid >> 5); i2 < r; i2 += (int)(blockDim.x >> 5))
                        LU[i2 * r + c] = LU[i2 * r + c] - LU[i2 * r + k] * LU[k * r + c];
            }
            __syncthreads();
        }
        const double bt = beta_sm;
        // X = A^-1 (I / beta): permuted identity / beta, then forward substitution
        // (unit L) and back substitution (U), right-looking and element-parallel
        for (int o = tid; o < r * r; o += blockDim.x) X[o] = 0.0;
        __syncthreads();
        if (tid < r) {
            // column tid of P (I / beta): apply the row interchanges in order
            int row = tid;
            for (int k = 0; k < r; ++k) {
                const int p = piv[k];
                if (row == k) row = p;
                else if (row == p) row = k;
            }
            X[row * r + tid] = 1.0 / bt;
        }
        __syncthreads();
        const int wstride = (int)(blockDim.x >> 5);
        for (int k = 0; k < r; ++k) {  // rows i2 > k: x_i2 -= L_i2k x_k (lane = column)
            if (lane < r)
                for (int i2 = k + 1 + (tid >> 5); i2 < r; i2 += wstride)
                    X[i2 * r + lane] = X[i2 * r + lane] - LU[i2 * r + k] * X[k * r + lane];
            __syncthreads();
        }
        // back substitution, right-looking: x_k /= U_kk, then rows i2 < k: x_i2 -= U_i2k x_k
        for (int k = r - 1; k >= 0; --k) {
            if (tid < r) X[k * r + tid] = X[k * r + tid] / LU[k * r + k];
            __syncthreads();
            if (lane < r)
                for (int i2 = tid >> 5; i2 < k; i2 += wstride)
                    X[i2 * r + lane] = X[i2 * r + lane] - LU[i2 * r + k] * X[k * r + lane];
            __syncthreads();
        }
        __syncthreads();
        // residual |A (beta X) - I|_max  (subspace.py:136-139)
        __shared__ double worst;
        if (tid == 0) worst = 0.0;
        __syncthreads();
        double wl = 0.0;
        bool nonfinite = false;
        for (int a = tid >> 5; a < r; a += (int)(blockDim.x >> 5)) {
            const int c = lane;
            if (c >= r) break;
            double s = 0.0;
            for (int k = 0; k < r; ++k) s += A[a * r + k] * (bt * X[k * r + c]);
            const double e = fabs(s - (a == c ? 1.0 : 0.0));
            if (!(e == e) || isinf(e)) nonfinite = true;
            wl = fmax(wl, e);
        }
        __shared__ int nf_flag;
        if (tid == 0) nf_flag = 0;
        __syncthreads();
        if (nonfinite) atomicExch(&nf_flag, 1);
        // max-reduce via atomics on the bit pattern (non-negative doubles order like ints)
        atomicMax((unsigned long long*)&worst, (unsigned long long)__double_as_longlong(wl));
        __syncthreads();
        const bool use_pinv = singular || nf_flag || worst > 1e-4;
        if (use_pinv) {
            for (int o = tid; o < r * r; o += blockDim.x) Q[o] = 0.0;  // scratch reuse below
            __syncthreads();
            for (int o = tid; o < r * r; o += blockDim.x) LU[o] = 0.5 * (A[o] + A[(o % r) * r + o / r]);
            __syncthreads();
            jacobi_eig_pinv(LU, Q, wv, r, X);
            for (int o = tid; o < r * r; o += blockDim.x) X[o] = X[o] / bt;
            __syncthreads();
        }
        for (int o = tid; o < r * r; o += blockDim.x) st.X[o] = X[o];
        if (tid == 0) {
            *st.beta = bt;
            *st.fallback = use_pinv ? 1 : 0;
        }
        __syncthreads();
    } else {
        for (int o = tid; o < r * r; o += blockDim.x) X[o] = st.X[o];
        if (tid == 0) beta_sm = *st.beta;
        __syncthreads();
    }
    if (beta_given >= 0.0) return;  // build only
    // q = beta * (X @ rhs)
    const double bt = beta_sm;
    for (int o = tid; o < 3 * r; o += blockDim.x) {
        const int a = o / 3, c = o % 3;
        double s = 0.0;
        for (int k = 0; k < r; ++k) s = fma(X[a * r + k], rhs[3 * k + c], s);
        q_out[o] = bt * s;
    }
}

// out[c] = sum_p part[p][c] in fixed order: block = 32 columns, 8 warps stride the parts
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ part, int nparts, int ncols,
                                                         double* __restrict__ out) {
    __shared__ double sm[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (c < ncols) {
#pragma unroll 4
        for (int p = warp; p < nparts; p += 8) s += part[(int64_t)p * ncols + c];
    }
    sm[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && c < ncols) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sm[w][lane];
        out[c] = t;
    }
}

// x_i += sum_j B[i, j] q[j]
// One thread per row: the block's rows of B (one contiguous span) are staged in
// shared memory by coalesced loads (row stride rb | 1: odd, conflict-free), then each
// thread forms its row's B_i q in column order.  prolong_rows(rb) rows per block.
__host__ __device__ constexpr int prolong_rows(int rb) { return rb <= 32 ? 128 : 32; }
__global__ void __launch_bounds__(128) k_prolong(const double* __restrict__ B, int rb, const double* __restrict__ q,
                                                 int n, double* __restrict__ x) {
    __shared__ double qs[3 * 128];
    extern __shared__ double sB[];
    for (int o = threadIdx.x; o < 3 * rb; o += blockDim.x) qs[o] = q[o];
    const int rpb = prolong_rows(rb), rbp = rb | 1;
    const int r0 = blockIdx.x * rpb;
    const int nr = min(rpb, n - r0);
    const double* src = B + (int64_t)r0 * rb;
    // 16-byte loads, 8 in flight per thread (r0 * rb is even: the span is 16-byte aligned)
    const int tot = nr * rb, tot2 = tot >> 1;
    const double2* src2 = reinterpret_cast<const double2*>(src);
    for (int e0 = threadIdx.x; e0 < tot2; e0 += 8 * blockDim.x) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e2 = e0 + u * blockDim.x;
            v[u] = e2 < tot2 ? __ldg(src2 + e2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e2 = e0 + u * blockDim.x;
            if (e2 < tot2) {
                const int e = 2 * e2, ra = e / rb, rb1 = (e + 1) / rb;
                sB[ra * rbp + (e - ra * rb)] = v[u].x;
                sB[rb1 * rbp + (e + 1 - rb1 * rb)] = v[u].y;
            }
        }
    }
    if ((tot & 1) && threadIdx.x == 0) {
        const int e = tot - 1, ra = e / rb;
        sB[ra * rbp + (e - ra * rb)] = __ldg(src + e);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nr; t += blockDim.x) {
        const double* br = sB + t * rbp;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int j = 0; j < rb; ++j) {
            const double v = br[j];
            a0 = fma(v, qs[3 * j], a0);
            a1 = fma(v, qs[3 * j + 1], a1);
            a2 = fma(v, qs[3 * j + 2], a2);
        }
        const int row = r0 + t;
        x[3 * row] += a0;
        x[3 * row + 1] += a1;
        x[3 * row + 2] += a2;
    }
}

// ---------------------------------------------------------------- reductions
// sum of squares of (a - b) over n*3 values (optionally gathered through ids)
__global__ void k_sqdiff_partial(const double* __restrict__ a, const double* __restrict__ b, int n,
                                 const int* __restrict__ ids_a, double* __restrict__ part) {
    __shared__ double sm[256];
    double s = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        // ids given: both a and b are cloth-indexed arrays compared over free rows
        const int ia = ids_a ? ids_a[i] : i;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double d = a[3 * ia + c] - (b ? b[3 * ia + c] : 0.0);
            s = fma(d, d, s);
        }
    }
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// ---------------------------------------------------------------- gather / scatter helpers
__global__ void k_gather_rows(const double* __restrict__ src, const int* __restrict__ ids, int n,
                              double* __restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = ids[i];
    dst[3 * i] = src[3 * s];
    dst[3 * i + 1] = src[3 * s + 1];
    dst[3 * i + 2] = src[3 * s + 2];
}

__global__ void k_scatter_rows(const double* __restrict__ src, const int* __restrict__ ids, int n,
                               double* __restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = ids[i];
    dst[3 * d] = src[3 * i];
    dst[3 * d + 1] = src[3 * i + 1];
    dst[3 * d + 2] = src[3 * i + 2];
}

// out = a + t (b - a)   (line-search clamp, stepper.py:477, 555, 586)
__global__ void k_set_scalar(double* __restrict__ p, double v) { *p = v; }
// *acc = min(*acc, *v) (fmin: a NaN operand is ignored)
__global__ void k_min_scalar(double* __restrict__ acc, const double* __restrict__ v) { *acc = fmin(*acc, *v); }

__global__ void k_lerp(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ tptr,
                       int64_t m, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double t = *tptr;
    out[i] = t < 1.0 ? a[i] + t * (b[i] - a[i]) : b[i];
}

// ---------------------------------------------------------------- energy gradient
// grad_v = s (x - z) + sum_{e: v=e1} g_e - sum_{e: v=e0} g_e + bend + quad stamps
struct BendSet {
    const int* __restrict__ st;  // (s,4)
    const double* __restrict__ k;  // (s,4)
    const double* __restrict__ w;  // (s,)
};

__global__ void k_energy_grad(int n, const double* __restrict__ x, const double* __restrict__ z,
                              const double* __restrict__ mass, double h, EdgeSet E,
                              const int* __restrict__ ginc_ptr, const int* __restrict__ ginc_edge,
                              BendSet Bd, const int* __restrict__ binc_ptr, const int* __restrict__ binc,
                              const int* __restrict__ free_index, const int* __restrict__ seg_beg,
                              const int* __restrict__ seg_end, const int* __restrict__ stamp_src,
                              const double4* __restrict__ stamp, double* __restrict__ grad) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int fi = free_index[v];
    if (fi < 0) {
        st3(grad, v, d3{0.0, 0.0, 0.0});
        return;
    }
    const double s = mass[v] / (h * h);
    const d3 xv = ld3(x, v);
    d3 g = s * (xv - ld3(z, v));
    // stretch: np.add.at(grad, e1, g) then np.add.at(grad, e0, -g)
    for (int k = ginc_ptr[v]; k < ginc_ptr[v + 1]; ++k) {
        const int code = ginc_edge[k];
        const int e = code >> 1;
        const d3 ev = ld3(x, E.e1[e]) - ld3(x, E.e0[e]);
        const double ln = norm3(ev);
        const d3 unit = ln > 0.0 ? d3{ev.x / ln, ev.y / ln, ev.z / ln} : d3{0.0, 0.0, 0.0};
        const d3 ge = (E.w[e] * (ln - E.rest[e])) * unit;
        g = (code & 1) ? g + ge : g + d3{-ge.x, -ge.y, -ge.z};
    }
    // bend: flat_s = sum_j k_sj x_sj ; grad += w_s k_sj flat_s
    for (int k = binc_ptr[v]; k < binc_ptr[v + 1]; ++k) {
        const int code = binc[k];
        const int si = code >> 2, j = code & 3;
        d3 flat{0.0, 0.0, 0.0};
        for (int a = 0; a < 4; ++a) {
            const double ka = Bd.k[4 * si + a];
            const d3 xa = ld3(x, Bd.st[4 * si + a]);
            flat = flat + ka * xa;
        }
        g = g + (Bd.w[si] * Bd.k[4 * si + j]) * flat;
    }
    if (seg_beg != nullptr) {
        for (int k = seg_beg[fi]; k < seg_end[fi]; ++k) {
            const double4 st = ldg256(stamp + stamp_src[k]);
            if (!(st.w > 0.0)) continue;  // plan entry outside the engaged set
            g = g + st.w * (xv - d3{st.x, st.y, st.z});
        }
    }
    st3(grad, v, g);
}

// delta_f = 2 m dx / h^2 over free rows, zero elsewhere (stepper.py:667-668)
__global__ void k_forward_force(const double* __restrict__ dx, const int* __restrict__ free_ids, int nf,
                                const double* __restrict__ mass, double h, double* __restrict__ df) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int v = free_ids[i];
    const double m2 = 2.0 * mass[v];
#pragma unroll
    for (int c = 0; c < 3; ++c) df[3 * v + c] = m2 * dx[3 * i + c] / (h * h);
}

__global__ void k_scale(double* __restrict__ a, int64_t m, const double* __restrict__ sptr) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) a[i] *= *sptr;
}

}  // namespace cs

namespace cs {
// out = (f - H dx) - delta dx  (stepper.py:663)
__global__ void k_residual(Sell H, const double* __restrict__ f, const double* __restrict__ x,
                           const double* __restrict__ delta, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H.nrows) return;
    const d3 hx = sell_row(H, i, x);
    st3(out, i, (ld3(f, i) - hx) - delta[i] * ld3(x, i));
}
}  // namespace cs
