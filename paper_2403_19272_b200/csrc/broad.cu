// Broad phase: candidate VT / EE pairs over swept, margin-inflated fp64 boxes.
//
// Produces exactly the SET reference broad_phase returns
// (pkg/src/clothsim/collision/bvh.py:207-292; derivation in oracle/broad.py):
//   VT (v, f): v not in f, box(v) overlaps box(f), not (v static and f static)
//   EE (E, F): E < F, vertex-disjoint, box(E) overlaps box(F), not both static
// with the reference's edge-edge ORIENTATION (which edge comes first in the row),
// computed from the static patch partition exactly as the reference's
// first-occurrence dedup picks it (bvh.py:264-286).  Row order is deterministic
// (VT block, then EE block; inside a block: hash-bucket order, then entry
// order) but is not the reference's order - only the rounding of the
// np.add.at collision stamps depends on it.
//
// Structure (B200-first: sort-based, no pointer chasing, warp-cooperative):
//   1. vertex boxes (fp64, exact min/max -/+ margin) -> primitive boxes
//      (triangles, edges); a fixed-order reduction of the mean box extent of
//      the moving primitives picks each grid's cell size
//   2. every box is entered once per cell it spans, as (bucket = hash(cell),
//      primitive, cell code); entries are radix-sorted by bucket (stable, so a
//      bucket lists its entries in primitive-then-cell order)
//   3. one warp per non-empty bucket tests all entry pairs of that bucket that
//      carry the same cell code: VT = bucket's vertex entries x the triangle
//      entries of the same bucket, EE = all edge-entry pairs i < j.  A pair is
//      reported only in the cell holding its intersection box's min corner,
//      so every overlapping pair is produced exactly once.  Ballot compaction
//      keeps the output order deterministic; count pass -> scan -> write pass.
//   4. primitives spanning more than kMaxCellsPerPrim cells (pathological
//      motion or giant obstacle faces) are not entered; a brute-force pass pairs
//      them with every primitive of the other set.
//
// Exactness: cell indices are floor(x * inv_cell) of the same fp64 box
// coordinates everywhere; floor of a correctly rounded product is monotone, so
// the min-corner cell lies inside both boxes' cell ranges.  Cell size and hash
// only change speed, never the set.
#include "common.cuh"

namespace cs {

constexpr long long kMaxCellsPerPrim = 1LL << 15;

// fbox (optional): the same boxes in fp32 rounded outward (lo down, hi up) as 32-byte
// records {lo.xyz, hi.xyz, max displacement (rounded up), 0} - one sector per
// primitive for the narrow-phase filter
__global__ void k_vertex_boxes(const double* __restrict__ x0, const double* __restrict__ x1, int n, double margin,
                               double* __restrict__ vlo, double* __restrict__ vhi, float* __restrict__ fbox = nullptr) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const double a = x0[i], b = x1[i];
    const double lo = np_min(a, b) - margin, hi = np_max(a, b) + margin;
    vlo[i] = lo;
    vhi[i] = hi;
    if (fbox) {
        const int v = i / 3, c = i - 3 * v;
        fbox[16 * (int64_t)v + c] = __double2float_rd(lo);
        fbox[16 * (int64_t)v + 3 + c] = __double2float_ru(hi);
    }
}

// |x_end - x_start| per vertex, as the reference's distance march computes it (ccd.py:240)
__global__ void k_vertex_disp(const double* __restrict__ x0, const double* __restrict__ x1, int n,
                              double* __restrict__ vdisp, float* __restrict__ fbox = nullptr) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const d3 p0 = ld3(x0, v), dp = ld3(x1, v) - p0;
    const double d = norm3(dp);
    vdisp[v] = d;
    if (fbox) {
        float* r = fbox + 16 * (int64_t)v;
        r[6] = __double2float_ru(d);
        r[7] = 0.0f;
        // motion part: reference displacement c (= own), deviation 0, start position
        r[8] = (float)dp.x;
        r[9] = (float)dp.y;
        r[10] = (float)dp.z;
        r[11] = 0.0f;
        r[12] = (float)p0.x;
        r[13] = (float)p0.y;
        r[14] = (float)p0.z;
        r[15] = 0.0f;
    }
}

// ------------------------------------------------------------------ boxes + cell size
// box[6p..6p+5] = lo.xyz, hi.xyz over the primitive's vertex boxes.  Block
// partial sums of the max-axis extent (moving primitives, all primitives) for the
// cell size: part[4 b + {0,1,2,3}] = {sum moving, count moving, sum all, count all}.
template <int ARITY>
__global__ void __launch_bounds__(256) k_prim_boxes(const int* __restrict__ verts, int np,
                                                    const uint8_t* __restrict__ is_static,
                                                    const double* __restrict__ vlo, const double* __restrict__ vhi,
                                                    const double* __restrict__ vdisp, double* __restrict__ box,
                                                    double* __restrict__ pdisp, double* __restrict__ part,
                                                    float* __restrict__ fbox = nullptr) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (p < np) {
        double lo[3], hi[3];
        const int a = verts[ARITY * p];
        double dmax = vdisp[a];
#pragma unroll
        for (int k = 1; k < ARITY; ++k) dmax = fmax(dmax, vdisp[verts[ARITY * p + k]]);
        pdisp[p] = dmax;
        if (fbox) {
            fbox[16 * (int64_t)p + 6] = __double2float_ru(dmax);
            fbox[16 * (int64_t)p + 7] = 0.0f;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = vlo[3 * a + c];
            hi[c] = vhi[3 * a + c];
        }
#pragma unroll
        for (int k = 1; k < ARITY; ++k) {
            const int b = verts[ARITY * p + k];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                lo[c] = np_min(lo[c], vlo[3 * b + c]);
                hi[c] = np_max(hi[c], vhi[3 * b + c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            box[6 * (int64_t)p + c] = lo[c];
            box[6 * (int64_t)p + 3 + c] = hi[c];
            if (fbox) {
                fbox[16 * (int64_t)p + c] = __double2float_rd(lo[c]);
                fbox[16 * (int64_t)p + 3 + c] = __double2float_ru(hi[c]);
            }
        }
        const double ext = fmax(fmax(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
        const bool moving = !is_static[p];
        v[0] = moving ? ext : 0.0;
        v[1] = moving ? 1.0 : 0.0;
        v[2] = ext;
        v[3] = 1.0;
    }
    // fixed-order block tree reduction (deterministic)
    __shared__ double sh[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double s = v[k];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[threadIdx.x][w];
        part[4 * blockIdx.x + threadIdx.x] = s;
    }
}

// inv_cell[0] = 1 / mean max-axis box extent of the moving primitives (all
// primitives if none move); fixed-order reduction of the block partials.
__global__ void k_cell_size(const double* __restrict__ part, int nparts, double* __restrict__ inv_cell,
                            double scale = 1.0) {
    __shared__ double sh[4][256];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] += part[4 * b + k];
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
#pragma unroll
            for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double cell = sh[1][0] > 0.0 ? sh[0][0] / sh[1][0] : (sh[3][0] > 0.0 ? sh[2][0] / sh[3][0] : 1.0);
        cell *= scale;
        if (!(cell > 1e-12)) cell = 1e-12;
        inv_cell[0] = 1.0 / cell;
    }
}

// Motion part of a primitive's filter record (floats 8..15): displacement c of its
// first vertex, max deviation of its vertices' displacements from c (rounded up),
// start position of its first vertex.  Lets the site filter bound a pair's RELATIVE
// motion (distances are translation invariant) - cloth riding a moving body.
template <int ARITY>
__global__ void k_prim_motion(const int* __restrict__ verts, int np, const double* __restrict__ x0,
                              const double* __restrict__ x1, float* __restrict__ fbox) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    const int a = verts[ARITY * p];
    const d3 p0 = ld3(x0, a), c = ld3(x1, a) - p0;
    double dev = 0.0;
#pragma unroll
    for (int k = 1; k < ARITY; ++k) {
        const int b = verts[ARITY * p + k];
        dev = fmax(dev, norm3((ld3(x1, b) - ld3(x0, b)) - c));
    }
    float* r = fbox + 16 * (int64_t)p;
    r[8] = (float)c.x;
    r[9] = (float)c.y;
    r[10] = (float)c.z;
    r[11] = __double2float_ru(dev);
    r[12] = (float)p0.x;
    r[13] = (float)p0.y;
    r[14] = (float)p0.z;
    r[15] = 0.0f;
}

// ------------------------------------------------------------------ cells
__device__ __forceinline__ long long cell_of(double x, double inv) {
    double c = floor(x * inv);
    c = fmin(fmax(c, -1.0e15), 1.0e15);  // keep the integer conversion defined
    return (long long)c;
}

// 21 bits per axis (wraps only across 2^21 cells - kilometres at cloth scales)
__device__ __forceinline__ unsigned long long cell_code(long long ix, long long iy, long long iz) {
    const unsigned long long m = (1ull << 21) - 1;
    return ((unsigned long long)ix & m) | (((unsigned long long)iy & m) << 21) | (((unsigned long long)iz & m) << 42);
}

// Bucket = low bits of the cell's Morton code: neighbouring cells get neighbouring
// buckets, so bucket-ordered runs (and the pair rows they emit) walk space
// coherently - every later per-pair gather by vertex id hits cache lines its
// neighbours just touched.  Cells 2^(bits/3) apart share a bucket; the cell-code
// comparison keeps the set exact.
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}
__device__ __forceinline__ unsigned bucket_of(unsigned long long code, unsigned mask) {
    const unsigned long long m = (1ull << 21) - 1;
    const unsigned long long h =
        spread3(code & m) | (spread3((code >> 21) & m) << 1) | (spread3((code >> 42) & m) << 2);
    return (unsigned)h & mask;
}

struct CellRange {
    long long lo[3], hi[3];
    __device__ long long count() const {
        return (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
    }
};

__device__ __forceinline__ CellRange cell_range(const double lo[3], const double hi[3], double inv) {
    CellRange r;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        r.lo[c] = cell_of(lo[c], inv);
        r.hi[c] = cell_of(hi[c], inv);
    }
    return r;
}


// Box source of a grid: primitive boxes (box != null) or vertex boxes (used vertices only).
struct BoxSrc {
    const double* __restrict__ box;
    const double* __restrict__ vlo;
    const double* __restrict__ vhi;
    const uint8_t* __restrict__ used;
    int np;
    __device__ __forceinline__ bool load(int p, double lo[3], double hi[3]) const {
        if (box) {
            load_box(box, p, lo, hi);
            return true;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = vlo[3 * (int64_t)p + c];
            hi[c] = vhi[3 * (int64_t)p + c];
        }
        return used[p] != 0;
    }
};

// per primitive: number of cells spanned (0 if oversize / unused) + oversize flag
__global__ void k_cell_count(BoxSrc S, const double* __restrict__ inv_cell, int* __restrict__ count,
                             uint8_t* __restrict__ over) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= S.np) return;
    double lo[3], hi[3];
    if (!S.load(p, lo, hi)) {
        count[p] = 0;
        over[p] = 0;
        return;
    }
    const long long nc = cell_range(lo, hi, inv_cell[0]).count();
    const bool big = nc > kMaxCellsPerPrim || nc <= 0;
    count[p] = big ? 0 : (int)nc;
    over[p] = big ? 1 : 0;
}

// Low-corner bits: cell_of is monotone, so for two boxes A, B both spanning cell c,
// cell_of(max(loA, loB)) = max(cell_of(loA), cell_of(loB)) per axis, which equals c
// iff c is A's or B's low-corner cell on that axis.  With zb = per-axis "c is my
// low-corner cell" bits, "the pair's min corner lies in c" is (zA | zB) == 7 -
// the exact integer form of min_corner_in(), evaluated before any fp64 test.
// 8 threads per primitive: thread k writes the primitive's cells k, k+8, ... in
// (z, y, x) order (x fastest), so a warp's stores land on contiguous entries.
__global__ void k_cell_fill(BoxSrc S, const double* __restrict__ inv_cell, unsigned mask,
                            const int* __restrict__ count, const int* __restrict__ offset,
                            unsigned* __restrict__ key, int* __restrict__ prim, unsigned long long* __restrict__ code,
                            uint8_t* __restrict__ zb) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int p = (int)(tid >> 3), k0 = (int)(tid & 7);
    if (p >= S.np) return;
    const int n = count[p];
    if (k0 >= n) return;
    double lo[3], hi[3];
    S.load(p, lo, hi);
    const CellRange r = cell_range(lo, hi, inv_cell[0]);
    // n <= kMaxCellsPerPrim, so the per-axis spans fit 32-bit arithmetic
    const int sx = (int)(r.hi[0] - r.lo[0] + 1), sxy = sx * (int)(r.hi[1] - r.lo[1] + 1);
    const int o = offset[p];
    for (int k = k0; k < n; k += 8) {
        const int kz = k / sxy, rem = k - kz * sxy, ky = rem / sx, kx = rem - ky * sx;
        const long long x = r.lo[0] + kx, y = r.lo[1] + ky, z = r.lo[2] + kz;
        const unsigned long long c = cell_code(x, y, z);
        key[o + k] = bucket_of(c, mask);
        prim[o + k] = p;
        code[o + k] = c;
        // which axes of this cell are the primitive's low-corner cell (see lo_corner_bits)
        zb[o + k] = (uint8_t)((x == r.lo[0]) | ((y == r.lo[1]) << 1) | ((z == r.lo[2]) << 2));
    }
}

// sorted order -> (primitive, code) arrays; run heads; dense bucket ranges
__global__ void k_entries_sorted(const int* __restrict__ perm, int m, const int* __restrict__ prim,
                                 const unsigned long long* __restrict__ code, const uint8_t* __restrict__ zb,
                                 const unsigned* __restrict__ key_s, int* __restrict__ prim_s,
                                 unsigned long long* __restrict__ code_s, uint8_t* __restrict__ zb_s,
                                 uint8_t* __restrict__ head, int* __restrict__ bstart, int* __restrict__ bend) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int k = perm[i];
    prim_s[i] = prim[k];
    code_s[i] = code[k];
    zb_s[i] = zb[k];
    const unsigned b = key_s[i];
    const bool h = i == 0 || key_s[i - 1] != b;
    head[i] = h;
    if (bstart) {
        if (h) bstart[b] = i;
        if (i == m - 1 || key_s[i + 1] != b) bend[b] = i + 1;
    }
}

// one sorted entry table (vertices, triangles or edges)
struct EntryTable {
    const unsigned* __restrict__ key;           // bucket, sorted
    const int* __restrict__ prim;
    const unsigned long long* __restrict__ code;
    const uint8_t* __restrict__ zb;             // low-corner bits
    const int* __restrict__ run;                // run heads (first entry of each bucket)
    const int* __restrict__ n_run;              // device scalar
    const int* __restrict__ bstart;             // dense bucket ranges
    const int* __restrict__ bend;
    int m;                                      // entries
};

struct WorldTopo {
    int nw;                              // world vertices
    const int* __restrict__ tris;        // (m,3)
    const int* __restrict__ edges;       // (E,2) sorted endpoints
    const uint8_t* __restrict__ tri_static;
    const uint8_t* __restrict__ vert_static;
    const uint8_t* __restrict__ vert_used;
    const uint8_t* __restrict__ edge_static;
    const int* __restrict__ edge_tris;   // (E,2) incident triangles (-1 pad)
    const int* __restrict__ edge_slot;   // (E,2) slot of the edge inside each triangle
    const int* __restrict__ patch;       // (m,) patch id (reference build_patches)
    const int* __restrict__ pslot;       // (m,) slot inside the patch
    const ulonglong2* __restrict__ flip; // (E,) packed incident-triangle records for ee_flip
};

struct PairOut {
    int* __restrict__ counts;            // pass 0
    const int* __restrict__ offsets;     // pass 1 (row offsets relative to base)
    int8_t* __restrict__ kind;
    int4* __restrict__ idx;
    unsigned long long* __restrict__ keys;
};

__device__ __forceinline__ bool overlap6(const double alo[3], const double ahi[3], const double blo[3],
                                         const double bhi[3]) {
    return (alo[0] <= bhi[0]) && (blo[0] <= ahi[0]) && (alo[1] <= bhi[1]) && (blo[1] <= ahi[1]) &&
           (alo[2] <= bhi[2]) && (blo[2] <= ahi[2]);
}

// the intersection box's min corner lies in cell `code`
__device__ __forceinline__ bool min_corner_in(const double alo[3], const double blo[3], double inv,
                                              unsigned long long code) {
    return cell_code(cell_of(fmax(alo[0], blo[0]), inv), cell_of(fmax(alo[1], blo[1]), inv),
                     cell_of(fmax(alo[2], blo[2]), inv)) == code;
}

__device__ __forceinline__ unsigned long long place_key(int pa, int sa, int pb, int sb, bool& a_first) {
    a_first = (pa < pb) || (pa == pb && sa < sb);
    const unsigned long long p1 = a_first ? pa : pb, p2 = a_first ? pb : pa;
    const unsigned long long s1 = a_first ? sa : sb, s2 = a_first ? sb : sa;
    const unsigned long long same = pa == pb;
    return ((((same << 24 | p1) << 24 | p2) << 3 | s1) << 3) | s2;
}

// Per-edge record of each incident triangle (built once per scene):
//   bit 63 valid, bit 62 static, bits 8..39 patch, bits 3..5 patch slot, bits 0..1 edge slot
__global__ void k_edge_flip_info(int n_edges, const int* __restrict__ edge_tris, const int* __restrict__ edge_slot,
                                 const uint8_t* __restrict__ tri_static, const int* __restrict__ patch,
                                 const int* __restrict__ pslot, ulonglong2* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_edges) return;
    unsigned long long rec[2];
    for (int k = 0; k < 2; ++k) {
        const int a = edge_tris[2 * e + k];
        rec[k] = a < 0 ? 0ull
                       : (1ull << 63) | ((unsigned long long)(tri_static[a] != 0) << 62) |
                             ((unsigned long long)(unsigned)patch[a] << 8) | ((unsigned long long)pslot[a] << 3) |
                             (unsigned long long)edge_slot[2 * e + k];
    }
    out[e] = make_ulonglong2(rec[0], rec[1]);
}

// reference orientation of edge pair (E, F), E < F: true when F comes first (bvh.py:264-286)
__device__ bool ee_flip(const WorldTopo& W, int E, int F) {
    const ulonglong2 re = W.flip[E], rf = W.flip[F];
    const unsigned long long ra[2] = {re.x, re.y}, rb[2] = {rf.x, rf.y};
    unsigned long long best = ~0ull;
    bool flip = false;
#pragma unroll
    for (int ka = 0; ka < 2; ++ka) {
        const unsigned long long a = ra[ka];
        if (!(a >> 63)) continue;
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
            const unsigned long long b = rb[kb];
            if (!(b >> 63)) continue;
            if (((a >> 62) & 1) && ((b >> 62) & 1)) continue;
            bool a_first;
            const unsigned long long place = place_key((int)((a >> 8) & 0xffffffffu), (int)((a >> 3) & 7),
                                                       (int)((b >> 8) & 0xffffffffu), (int)((b >> 3) & 7), a_first);
            const int sa = (int)(a & 3), sb = (int)(b & 3);
            const unsigned long long sub = a_first ? (sa * 3 + sb) : (sb * 3 + sa);
            const unsigned long long key = (place << 5) | (sub << 1) | (a_first ? 0ull : 1ull);
            if (key < best) {
                best = key;
                flip = !a_first;
            }
        }
    }
    return flip;
}

__device__ __forceinline__ void write_vt(const PairOut& O, int row, int v, int f, const WorldTopo& W) {
    O.kind[row] = CS_VT;
    O.idx[row] = make_int4(v, W.tris[3 * f], W.tris[3 * f + 1], W.tris[3 * f + 2]);
    O.keys[row] = ((unsigned long long)(unsigned)v << 32) | (unsigned)f;
}

// EE rows are written as (lower edge, higher edge); k_ee_orient applies the
// reference orientation afterwards in one dense pass (keeps the divergent
// emission path short).
__device__ __forceinline__ void write_ee(const PairOut& O, int row, int E, int F, const WorldTopo& W) {
    const int lo = E < F ? E : F, hi = E < F ? F : E;
    O.kind[row] = CS_EE;
    O.idx[row] = make_int4(W.edges[2 * lo], W.edges[2 * lo + 1], W.edges[2 * hi], W.edges[2 * hi + 1]);
    O.keys[row] = (1ull << 63) | ((unsigned long long)(unsigned)lo << 32) | (unsigned)hi;
}

__global__ void k_ee_orient(const unsigned long long* __restrict__ keys, int4* __restrict__ idx, int64_t n,
                            WorldTopo W) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    const int lo = (int)((k >> 32) & 0x7fffffffu), hi = (int)(k & 0xffffffffu);
    if (ee_flip(W, lo, hi)) {
        const int4 v = idx[i];
        idx[i] = make_int4(v.z, v.w, v.x, v.y);
    }
}

__device__ __forceinline__ bool vt_ok(const WorldTopo& W, int v, int f) {
    if (W.vert_static[v] && W.tri_static[f]) return false;
    const int a = W.tris[3 * f], b = W.tris[3 * f + 1], c = W.tris[3 * f + 2];
    return a != v && b != v && c != v;
}

__device__ __forceinline__ bool ee_ok(const WorldTopo& W, int E, int F) {
    if (W.edge_static[E] && W.edge_static[F]) return false;
    const int a0 = W.edges[2 * E], a1 = W.edges[2 * E + 1];
    const int b0 = W.edges[2 * F], b1 = W.edges[2 * F + 1];
    return a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1;
}

// Bucket-pair kernels run twice.  Pass 0 tests every candidate pair and stores
// one 32-bit ballot word per warp iteration (masks) plus the run's hit count;
// pass 1 replays the same loop structure reading the ballots (no box tests) and
// writes rows at the run's scanned offset, hits in lane order.
template <int PASS>
__device__ __forceinline__ unsigned warp_hits(bool hit, unsigned* __restrict__ masks, int64_t it) {
    if (PASS == 0) {
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if ((threadIdx.x & 31) == 0) masks[it] = m;
        return m;
    }
    return masks[it];
}
__device__ __forceinline__ int lane_rank(unsigned mask) {
    return __popc(mask & ((1u << (threadIdx.x & 31)) - 1u));
}

// Shared-memory copy of one bucket entry: box, cell code, primitive, its vertices
// (edge: a, b; triangle: a, b, c; vertex: a = id) and static flag.
struct SmEntry {
    double lo[3], hi[3];
    unsigned long long code;
    int prim, a, b, c, stat, z;
};
constexpr int kRunCap = 112;  // edge / triangle runs up to this many entries are staged in shared memory
constexpr int kRunCapV = 32;  // vertex runs
constexpr int kPairWarps = 4; // warps per block of the bucket-pair kernels

__device__ __forceinline__ bool sm_overlap(const SmEntry& a, const SmEntry& b) {
    return (a.lo[0] <= b.hi[0]) && (b.lo[0] <= a.hi[0]) && (a.lo[1] <= b.hi[1]) && (b.lo[1] <= a.hi[1]) &&
           (a.lo[2] <= b.hi[2]) && (b.lo[2] <= a.hi[2]);
}

// k in [0, m(m-1)/2) -> (i, j), i < j, row-major over i (emission order = i, then j)
__device__ __forceinline__ void tri_index(int k, int m, int& i, int& j) {
    const float b = 2.0f * m - 1.0f;
    int r = (int)((b - sqrtf(b * b - 8.0f * (float)k)) * 0.5f);
    r = max(0, min(r, m - 2));
    while (r > 0 && r * (2 * m - 1 - r) / 2 > k) --r;
    while (r + 1 <= m - 2 && (r + 1) * (2 * m - 2 - r) / 2 <= k) ++r;
    i = r;
    j = k - r * (2 * m - 1 - r) / 2 + r + 1;
}

// warp iterations a run takes (must mirror the loops below exactly)
// (runs longer than the staging caps are enumerated by k_long_ee / k_long_vt, one thread
// per row, and take no iterations here)
// A run beyond the staging caps is enumerated by one warp row by row (lanes over the
// partners) while that takes at most kLongIters warp iterations; longer runs (dense
// piles) go to k_long_ee / k_long_vt, one thread per row.
constexpr long long kLongIters = 1024;
__host__ __device__ __forceinline__ long long serial_iters_ee(int m) {
    const long long n = m - 1, q = n / 32, r = n % 32;  // sum_{L=1..n} ceil(L/32)
    return 32 * q * (q + 1) / 2 + (q + 1) * r;
}
__host__ __device__ __forceinline__ bool ee_long(int m) { return m > kRunCap && serial_iters_ee(m) > kLongIters; }
__host__ __device__ __forceinline__ bool vt_long(int mv, int mt) {
    return mt > 0 && mv > 0 && !(mv <= kRunCapV && mt <= kRunCap) && (long long)mv * ((mt + 31) / 32) > kLongIters;
}
__device__ __forceinline__ long long iters_ee(int m) {
    if (m < 2 || ee_long(m)) return 0;
    if (m <= kRunCap) return ((long long)m * (m - 1) / 2 + 31) / 32;
    return serial_iters_ee(m);
}
__device__ __forceinline__ long long iters_vt(int mv, int mt) {
    if (mt <= 0 || mv <= 0 || vt_long(mv, mt)) return 0;
    if (mv <= kRunCapV && mt <= kRunCap) return ((long long)mv * mt + 31) / 32;
    return (long long)mv * ((mt + 31) / 32);
}

// per run: warp iterations (for the ballot buffer); entries beyond n_run stay 0
// (+ *long_flag = 1 when some run goes to the row kernels)
__global__ void k_run_iters(EntryTable R, EntryTable T, int vt, long long* __restrict__ iters,
                            int* __restrict__ long_flag) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R.n_run[0]) return;
    const int b0 = R.run[r], b1 = r + 1 < R.n_run[0] ? R.run[r + 1] : R.m;
    bool lng;
    if (vt) {
        const unsigned b = R.key[b0];
        const int mt = T.bend[b] - T.bstart[b];
        iters[r] = iters_vt(b1 - b0, mt);
        lng = vt_long(b1 - b0, mt);
    } else {
        iters[r] = iters_ee(b1 - b0);
        lng = ee_long(b1 - b0);
    }
    if (lng) atomicOr(long_flag, 1);
}

// VT per-warp staging, structure of arrays; static flags ride in bit 3 of the
// low-corner bytes
struct VtStage {
    double vlo[3][kRunCapV], vhi[3][kRunCapV];
    unsigned long long vcode[kRunCapV];
    int vprim[kRunCapV];
    unsigned char vzs[kRunCapV];
    double tlo[3][kRunCap], thi[3][kRunCap];
    unsigned long long tcode[kRunCap];
    int ta[kRunCap], tb[kRunCap], tc[kRunCap];
    unsigned char tzs[kRunCap];
};

// k in [0, mv * mt) -> (i, j) = (k / mt, k % mt) via a float reciprocal (k < 2^12)
__device__ __forceinline__ void vt_index(int k, int mt, float inv_mt, int& i, int& j) {
    int q = (int)((float)k * inv_mt);
    int r = k - q * mt;
    if (r < 0) {
        --q;
        r += mt;
    } else if (r >= mt) {
        ++q;
        r -= mt;
    }
    i = q;
    j = r;
}

// VT: one warp per vertex-table bucket run x the same bucket's triangle entries.
template <int PASS>
__global__ void __launch_bounds__(32 * kPairWarps) k_pairs_vt(EntryTable V, EntryTable T,
                                                              const double* __restrict__ vlo,
                                                              const double* __restrict__ vhi,
                                                              const double* __restrict__ tbox,
                                                              const double* __restrict__ inv_cell, WorldTopo W,
                                                              const long long* __restrict__ iter_off,
                                                              unsigned* __restrict__ masks, PairOut O) {
    __shared__ VtStage smvt[PASS == 0 ? kPairWarps : 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    VtStage& S = smvt[PASS == 0 ? w : 0];
    const int nr = V.n_run[0];
    const double inv = inv_cell[0];
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr; r += (gridDim.x * blockDim.x) >> 5) {
        const int vb = V.run[r], ve = r + 1 < nr ? V.run[r + 1] : V.m;
        const unsigned b = V.key[vb];
        const int tb = T.bstart[b], te = T.bend[b];
        const int mv = ve - vb, mt = te - tb;
        int base = PASS == 1 ? O.offsets[r] : 0, cnt = 0;
        long long it = iter_off[r];
        if (mt > 0 && mv <= kRunCapV && mt <= kRunCap) {
            if (PASS == 0) {
                for (int k = lane; k < mv; k += 32) {
                    const int v = V.prim[vb + k];
                    S.vprim[k] = v;
                    S.vcode[k] = V.code[vb + k];
                    S.vzs[k] = (unsigned char)(V.zb[vb + k] | (W.vert_static[v] ? 8 : 0));
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        S.vlo[c][k] = vlo[3 * (int64_t)v + c];
                        S.vhi[c][k] = vhi[3 * (int64_t)v + c];
                    }
                }
                for (int k = lane; k < mt; k += 32) {
                    const int f = T.prim[tb + k];
                    S.tcode[k] = T.code[tb + k];
                    S.tzs[k] = (unsigned char)(T.zb[tb + k] | (W.tri_static[f] ? 8 : 0));
                    S.ta[k] = W.tris[3 * f];
                    S.tb[k] = W.tris[3 * f + 1];
                    S.tc[k] = W.tris[3 * f + 2];
                    double lo[3], hi[3];
                    load_box(tbox, f, lo, hi);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        S.tlo[c][k] = lo[c];
                        S.thi[c][k] = hi[c];
                    }
                }
                __syncwarp();
            }
            const int np = mv * mt;
            const float inv_mt = 1.0f / (float)mt;
            for (int k0 = 0; k0 < np; k0 += 32, ++it) {
                const int k = k0 + lane;
                bool hit = false;
                if (PASS == 0 && k < np) {
                    int i, j;
                    vt_index(k, mt, inv_mt, i, j);
                    const int zi = S.vzs[i], zj = S.tzs[j];
                    const int v = S.vprim[i];
                    hit = ((zi | zj) & 7) == 7 && !(zi & zj & 8) && S.vcode[i] == S.tcode[j];
                    hit = hit && ((v != S.ta[j]) & (v != S.tb[j]) & (v != S.tc[j]) & (S.vlo[0][i] <= S.thi[0][j]) &
                                  (S.tlo[0][j] <= S.vhi[0][i]) & (S.vlo[1][i] <= S.thi[1][j]) &
                                  (S.tlo[1][j] <= S.vhi[1][i]) & (S.vlo[2][i] <= S.thi[2][j]) &
                                  (S.tlo[2][j] <= S.vhi[2][i]));
                }
                const unsigned m = warp_hits<PASS>(hit, masks, it);
                if (PASS == 1 && ((m >> lane) & 1u)) {
                    int i, j;
                    vt_index(k, mt, inv_mt, i, j);
                    write_vt(O, base + lane_rank(m), V.prim[vb + i], T.prim[tb + j], W);
                }
                base += __popc(m);
                cnt += __popc(m);
            }
            if (PASS == 0) __syncwarp();
        } else if (mt > 0 && !vt_long(mv, mt)) {  // moderately long: one warp, rows in turn
            for (int i = vb; i < ve; ++i) {
                const int v = V.prim[i];
                const unsigned long long cv = V.code[i];
                double qlo[3], qhi[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    qlo[c] = vlo[3 * (int64_t)v + c];
                    qhi[c] = vhi[3 * (int64_t)v + c];
                }
                for (int j0 = tb; j0 < te; j0 += 32, ++it) {
                    const int j = j0 + lane;
                    bool hit = false;
                    if (PASS == 0 && j < te && T.code[j] == cv) {
                        const int f = T.prim[j];
                        double lo[3], hi[3];
                        load_box(tbox, f, lo, hi);
                        hit = overlap6(qlo, qhi, lo, hi) && min_corner_in(qlo, lo, inv, cv) && vt_ok(W, v, f);
                    }
                    const unsigned m = warp_hits<PASS>(hit, masks, it);
                    if (PASS == 1 && ((m >> lane) & 1u)) write_vt(O, base + lane_rank(m), v, T.prim[j], W);
                    base += __popc(m);
                    cnt += __popc(m);
                }
            }
        }  // longer runs: k_long_vt
        if (PASS == 0 && lane == 0) O.counts[r] = cnt;
    }
}

// Round-robin enumeration of the m(m-1)/2 unordered entry pairs of a run: k ->
// (offset d, i), j = (i + d) mod m; offsets 1 .. ceil(m/2)-1 take all m rows, and
// for even m the offset m/2 takes rows i < m/2 only.  Division by m via a float
// reciprocal with one correction (k < 2^13, exact).  The hit test is symmetric, so
// (i, j) orientation does not matter; pass 1 replays the same mapping.
__device__ __forceinline__ void rr_index(int k, int m, float inv_m, int& i, int& j) {
    const int half = m >> 1;
    const int full = (m & 1) ? m * half : m * (half - 1);
    int d;
    if (k < full) {
        int q = (int)((float)k * inv_m);
        int r = k - q * m;
        if (r < 0) {
            --q;
            r += m;
        } else if (r >= m) {
            ++q;
            r -= m;
        }
        d = q + 1;
        i = r;
    } else {
        d = half;
        i = k - full;
    }
    j = i + d;
    if (j >= m) j -= m;
}

// EE per-warp staging, structure of arrays (conflict-free lane access); the static
// flag rides in bit 3 of the low-corner byte
struct EeStage {
    double lo[3][kRunCap], hi[3][kRunCap];
    unsigned long long code[kRunCap];
    int a[kRunCap], b[kRunCap];
    unsigned char zs[kRunCap];
};

// EE: one warp per edge-table bucket run; all unordered entry pairs of the run.
template <int PASS>
__global__ void __launch_bounds__(32 * kPairWarps) k_pairs_ee(EntryTable E, const double* __restrict__ ebox,
                                                              const double* __restrict__ inv_cell, WorldTopo W,
                                                              const long long* __restrict__ iter_off,
                                                              unsigned* __restrict__ masks, PairOut O) {
    __shared__ EeStage sme[kPairWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    EeStage& S = sme[w];
    const int nr = E.n_run[0];
    const double inv = inv_cell[0];
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr; r += (gridDim.x * blockDim.x) >> 5) {
        const int eb = E.run[r], ee = r + 1 < nr ? E.run[r + 1] : E.m;
        const int m = ee - eb;
        int base = PASS == 1 ? O.offsets[r] : 0, cnt = 0;
        long long it = iter_off[r];
        if (m <= kRunCap) {
            if (PASS == 0) {
                for (int k = lane; k < m; k += 32) {
                    const int q = E.prim[eb + k];
                    S.code[k] = E.code[eb + k];
                    S.a[k] = W.edges[2 * q];
                    S.b[k] = W.edges[2 * q + 1];
                    S.zs[k] = (unsigned char)(E.zb[eb + k] | (W.edge_static[q] ? 8 : 0));
                    double lo[3], hi[3];
                    load_box(ebox, q, lo, hi);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        S.lo[c][k] = lo[c];
                        S.hi[c][k] = hi[c];
                    }
                }
                __syncwarp();
            }
            const int np = m * (m - 1) / 2;
            const float inv_m = 1.0f / (float)m;
            for (int k0 = 0; k0 < np; k0 += 32, ++it) {
                const int k = k0 + lane;
                bool hit = false;
                if (PASS == 0 && k < np) {
                    int i, j;
                    rr_index(k, m, inv_m, i, j);
                    const int zi = S.zs[i], zj = S.zs[j];
                    // the selective class / cell tests short-circuit; the adjacency and box
                    // tests after them are evaluated branch-free (fewer divergent branches)
                    hit = ((zi | zj) & 7) == 7 && !(zi & zj & 8) && S.code[i] == S.code[j];
                    hit = hit && ((S.a[i] != S.a[j]) & (S.a[i] != S.b[j]) & (S.b[i] != S.a[j]) & (S.b[i] != S.b[j]) &
                                  (S.lo[0][i] <= S.hi[0][j]) & (S.lo[0][j] <= S.hi[0][i]) & (S.lo[1][i] <= S.hi[1][j]) &
                                  (S.lo[1][j] <= S.hi[1][i]) & (S.lo[2][i] <= S.hi[2][j]) & (S.lo[2][j] <= S.hi[2][i]));
                }
                const unsigned msk = warp_hits<PASS>(hit, masks, it);
                if (PASS == 1 && ((msk >> lane) & 1u)) {
                    int i, j;
                    rr_index(k, m, inv_m, i, j);
                    write_ee(O, base + lane_rank(msk), E.prim[eb + i], E.prim[eb + j], W);
                }
                base += __popc(msk);
                cnt += __popc(msk);
            }
            if (PASS == 0) __syncwarp();
        } else if (!ee_long(m)) {  // moderately long: one warp, rows in turn
            for (int i = eb; i + 1 < ee; ++i) {
                const int a = E.prim[i];
                const unsigned long long ca = E.code[i];
                double qlo[3], qhi[3];
                load_box(ebox, a, qlo, qhi);
                for (int j0 = i + 1; j0 < ee; j0 += 32, ++it) {
                    const int j = j0 + lane;
                    bool hit = false;
                    if (PASS == 0 && j < ee && E.code[j] == ca) {
                        const int f = E.prim[j];
                        double lo[3], hi[3];
                        load_box(ebox, f, lo, hi);
                        hit = overlap6(qlo, qhi, lo, hi) && min_corner_in(qlo, lo, inv, ca) && ee_ok(W, a, f);
                    }
                    const unsigned msk = warp_hits<PASS>(hit, masks, it);
                    if (PASS == 1 && ((msk >> lane) & 1u)) write_ee(O, base + lane_rank(msk), a, E.prim[j], W);
                    base += __popc(msk);
                    cnt += __popc(msk);
                }
            }
        }  // longer runs: k_long_ee
        if (PASS == 0 && lane == 0) O.counts[r] = cnt;
    }
}

// Long bucket runs (dense piles: more entries than the shared-memory staging holds),
// one thread per row instead of one warp per run (a run of m entries is m rows of up to
// m tests: the serial tail of a single warp made config 3's late steps 10x slower).
// Rows are the entries of long runs in table order (LongRow); pass 0 counts a row's
// hits, pass 1 writes them at the row's scanned offset in (row, partner) order.  Same
// predicates as the staged path: same cell code, box overlap, the overlap's min corner
// in this cell (reported once), adjacency / static filters.
struct LongRow {
    const unsigned* __restrict__ key;
    const int* __restrict__ bstart;
    const int* __restrict__ bend;
    const int* __restrict__ tstart;  // VT: the triangle table's bucket ranges (null: EE)
    const int* __restrict__ tend;
    __host__ __device__ __forceinline__ bool operator()(int e) const {
        const unsigned b = key[e];
        const int m = bend[b] - bstart[b];
        if (tstart == nullptr) return ee_long(m);
        return vt_long(m, tend[b] - tstart[b]);
    }
};

template <int PASS>
__global__ void k_long_ee(EntryTable E, const double* __restrict__ ebox, const double* __restrict__ inv_cell,
                          WorldTopo W, const int* __restrict__ rows, const int* __restrict__ n_rows, PairOut O) {
    const int n = n_rows[0];
    const double inv = inv_cell[0];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = rows[k];
        const int end = E.bend[E.key[i]];
        const int a = E.prim[i];
        const unsigned long long ca = E.code[i];
        double qlo[3], qhi[3];
        load_box(ebox, a, qlo, qhi);
        int row = PASS == 1 ? O.offsets[k] : 0, cnt = 0;
        for (int j = i + 1; j < end; ++j) {
            if (E.code[j] != ca) continue;
            const int f = E.prim[j];
            double lo[3], hi[3];
            load_box(ebox, f, lo, hi);
            if (overlap6(qlo, qhi, lo, hi) && min_corner_in(qlo, lo, inv, ca) && ee_ok(W, a, f)) {
                if (PASS == 1) write_ee(O, row++, a, f, W);
                ++cnt;
            }
        }
        if (PASS == 0) O.counts[k] = cnt;
    }
}

template <int PASS>
__global__ void k_long_vt(EntryTable V, EntryTable T, const double* __restrict__ vlo, const double* __restrict__ vhi,
                          const double* __restrict__ tbox, const double* __restrict__ inv_cell, WorldTopo W,
                          const int* __restrict__ rows, const int* __restrict__ n_rows, PairOut O) {
    const int n = n_rows[0];
    const double inv = inv_cell[0];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int i = rows[k];
        const unsigned b = V.key[i];
        const int tb = T.bstart[b], te = T.bend[b];
        const int v = V.prim[i];
        const unsigned long long cv = V.code[i];
        double qlo[3], qhi[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            qlo[c] = vlo[3 * (int64_t)v + c];
            qhi[c] = vhi[3 * (int64_t)v + c];
        }
        int row = PASS == 1 ? O.offsets[k] : 0, cnt = 0;
        for (int j = tb; j < te; ++j) {
            if (T.code[j] != cv) continue;
            const int f = T.prim[j];
            double lo[3], hi[3];
            load_box(tbox, f, lo, hi);
            if (overlap6(qlo, qhi, lo, hi) && min_corner_in(qlo, lo, inv, cv) && vt_ok(W, v, f)) {
                if (PASS == 1) write_vt(O, row++, v, f, W);
                ++cnt;
            }
        }
        if (PASS == 0) O.counts[k] = cnt;
    }
}

// Brute-force side for primitives that were not entered in the grid (oversize).
// VT: thread t < n_ov handles oversize vertex over[t] against every triangle;
// thread n_ov + k handles oversize triangle overt[k] against every entered vertex.
template <int PASS>
__global__ void k_over_vt(const int* __restrict__ over_v, int n_ov, const int* __restrict__ over_t, int n_ot,
                          const uint8_t* __restrict__ v_over, const double* __restrict__ vlo,
                          const double* __restrict__ vhi, const double* __restrict__ tbox, int ntris, WorldTopo W,
                          PairOut O) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_ov + n_ot) return;
    int row = PASS == 1 ? O.offsets[t] : 0, cnt = 0;
    if (t < n_ov) {
        const int v = over_v[t];
        double qlo[3], qhi[3];
        for (int c = 0; c < 3; ++c) {
            qlo[c] = vlo[3 * (int64_t)v + c];
            qhi[c] = vhi[3 * (int64_t)v + c];
        }
        for (int f = 0; f < ntris; ++f) {
            double lo[3], hi[3];
            load_box(tbox, f, lo, hi);
            if (overlap6(qlo, qhi, lo, hi) && vt_ok(W, v, f)) {
                if (PASS == 1) write_vt(O, row++, v, f, W);
                ++cnt;
            }
        }
    } else {
        const int f = over_t[t - n_ov];
        double lo[3], hi[3];
        load_box(tbox, f, lo, hi);
        for (int v = 0; v < W.nw; ++v) {
            if (!W.vert_used[v] || v_over[v]) continue;
            double qlo[3], qhi[3];
            for (int c = 0; c < 3; ++c) {
                qlo[c] = vlo[3 * (int64_t)v + c];
                qhi[c] = vhi[3 * (int64_t)v + c];
            }
            if (overlap6(qlo, qhi, lo, hi) && vt_ok(W, v, f)) {
                if (PASS == 1) write_vt(O, row++, v, f, W);
                ++cnt;
            }
        }
    }
    if (PASS == 0) O.counts[t] = cnt;
}

// EE: oversize edge E against every other edge F (entered F always; oversize F only if F > E).
template <int PASS>
__global__ void k_over_ee(const int* __restrict__ over_e, int n_oe, const uint8_t* __restrict__ e_over,
                          const double* __restrict__ ebox, int n_edges, WorldTopo W, PairOut O) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_oe) return;
    int row = PASS == 1 ? O.offsets[t] : 0, cnt = 0;
    const int E = over_e[t];
    double qlo[3], qhi[3];
    load_box(ebox, E, qlo, qhi);
    for (int F = 0; F < n_edges; ++F) {
        if (F == E || (e_over[F] && F < E)) continue;
        double lo[3], hi[3];
        load_box(ebox, F, lo, hi);
        if (overlap6(qlo, qhi, lo, hi) && ee_ok(W, E, F)) {
            if (PASS == 1) write_ee(O, row++, E, F, W);
            ++cnt;
        }
    }
    if (PASS == 0) O.counts[t] = cnt;
}

// ------------------------------------------------------------------ motion-free sites
// A site with x_start == x_end (the exit line search: the anchor was just set to
// the clamped candidate) has static boxes x -/+ margin.  When every such vertex box
// lies inside the vertex box of the previous site (both with the same margin), every
// primitive box does too, so the new candidate set is exactly the previous set's
// pairs whose new boxes still overlap (pair conditions other than overlap are
// topological and unchanged).  flag != 0: some box escaped -> full broad phase.
__global__ void k_box_contained(const double* __restrict__ x, int n3, double margin,
                                const double* __restrict__ vlo, const double* __restrict__ vhi,
                                int* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n3) return;
    const double a = x[i];
    const double lo = np_min(a, a) - margin, hi = np_max(a, a) + margin;
    if (!(lo >= vlo[i] && hi <= vhi[i])) atomicOr(flag, 1);
}

// Violators of a base site (subset sites, see abi.cu subset_site): used vertices
// whose box at this site is not inside their base box, or that the base grid left
// out (oversize); primitives with a violating vertex or left out themselves.
__global__ void k_viol_vertices(const double* __restrict__ vlo, const double* __restrict__ vhi,
                                const double* __restrict__ blo, const double* __restrict__ bhi, int nw,
                                const uint8_t* __restrict__ used, const uint8_t* __restrict__ over,
                                uint8_t* __restrict__ viol) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nw) return;
    bool out = over[v] != 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t i = 3 * (int64_t)v + c;
        out |= !(vlo[i] >= blo[i] && vhi[i] <= bhi[i]);
    }
    viol[v] = used[v] && out ? 1 : 0;
}

template <int ARITY>
__global__ void k_viol_prims(const int* __restrict__ verts, int np, const uint8_t* __restrict__ vviol,
                             const uint8_t* __restrict__ over, uint8_t* __restrict__ viol) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    bool out = over[p] != 0;
#pragma unroll
    for (int k = 0; k < ARITY; ++k) out |= vviol[verts[ARITY * p + k]] != 0;
    viol[p] = out ? 1 : 0;
}

// Pairs of a subset site with at least one violator.  Thread t takes violator
// list entry t of [vertices | triangles | edges] and finds its partners at this
// site's boxes:
//  * non-violators through the base grid: the cells covering its box, entries with
//    that cell code, exact box overlap, reported in the cell holding the overlap's
//    min corner (a non-violator's box lies inside its base box, so it is entered in
//    that cell) - once;
//  * violators by brute force over the violator lists (vertex x triangle from the
//    vertex side, edge x edge from the lower list position).
// A violator box spanning more cells than the grid enters for one primitive scans
// every non-violator instead.  PASS 0 counts, PASS 1 writes at the scanned offset (deterministic).
constexpr long long kQueryCells = kMaxCellsPerPrim;

struct QueryArgs {
    const int* __restrict__ vlist;
    const int* __restrict__ tlist;
    const int* __restrict__ elist;
    int nv, nt, ne;
    const uint8_t* __restrict__ vviol;
    const uint8_t* __restrict__ tviol;
    const uint8_t* __restrict__ eviol;
    const double* __restrict__ vlo;
    const double* __restrict__ vhi;
    const double* __restrict__ tbox;
    const double* __restrict__ ebox;
    EntryTable V, T, E;  // base grid (V/T share cells and buckets)
    const double* __restrict__ inv_vt;
    const double* __restrict__ inv_ee;
    unsigned mask_vt, mask_ee;
    int ntris, nedges;
    unsigned long long* big;  // diagnostics (nullable): [class] big-box violators, [3] max cells
};

__device__ __forceinline__ void vbox(const QueryArgs& A, int v, double lo[3], double hi[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        lo[c] = A.vlo[3 * (int64_t)v + c];
        hi[c] = A.vhi[3 * (int64_t)v + c];
    }
}

// one warp per violator; hits are ballot-ordered, so both passes emit in the same order
template <int PASS>
__global__ void __launch_bounds__(128) k_subset_query(QueryArgs A, WorldTopo W, int* __restrict__ counts,
                                                      const int* __restrict__ offsets, PairOut O) {
    const int lane = threadIdx.x & 31;
    const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int ntot = A.nv + A.nt + A.ne;
    if (t >= ntot) return;
    const int cls = t < A.nv ? 0 : (t < A.nv + A.nt ? 1 : 2);  // 0 vertex, 1 triangle, 2 edge
    const int li = cls == 0 ? t : (cls == 1 ? t - A.nv : t - A.nv - A.nt);
    const int p = cls == 0 ? A.vlist[li] : (cls == 1 ? A.tlist[li] : A.elist[li]);
    int row = PASS == 1 ? offsets[t] : 0, cnt = 0;
    // one warp step: lanes with hit emit (a, b) in lane order
    auto step = [&](bool hit, int a, int b) {
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (PASS == 1 && hit) {
            if (cls == 2) write_ee(O, row + lane_rank(m), a, b, W);
            else write_vt(O, row + lane_rank(m), a, b, W);
        }
        row += __popc(m);
        cnt += __popc(m);
    };
    auto partner_ok = [&](int q) {
        return cls == 0 ? vt_ok(W, p, q) : (cls == 1 ? vt_ok(W, q, p) : ee_ok(W, p, q));
    };
    double lo[3], hi[3];
    if (cls == 0) vbox(A, p, lo, hi);
    else load_box(cls == 1 ? A.tbox : A.ebox, p, lo, hi);
    const double inv = cls == 2 ? A.inv_ee[0] : A.inv_vt[0];
    const CellRange r = cell_range(lo, hi, inv);
    const long long nc = r.count();
    const EntryTable& G = cls == 0 ? A.T : (cls == 1 ? A.V : A.E);
    const uint8_t* __restrict__ qviol = cls == 0 ? A.tviol : (cls == 1 ? A.vviol : A.eviol);
    const unsigned mask = cls == 2 ? A.mask_ee : A.mask_vt;
    if (PASS == 0 && A.big != nullptr && lane == 0) {
        if (!(nc > 0 && nc <= kQueryCells)) atomicAdd(&A.big[cls], 1ull);
        atomicMax(&A.big[3], (unsigned long long)nc);
    }
    if (nc > 0 && nc <= kQueryCells) {
        // lanes take cells; each walks its cell's bucket run, one entry per warp step
        const int sx = (int)(r.hi[0] - r.lo[0] + 1), sxy = sx * (int)(r.hi[1] - r.lo[1] + 1);
        for (int c0 = 0; c0 < (int)nc; c0 += 32) {
            const int c = c0 + lane;
            int beg = 0, end = 0;
            unsigned long long code = 0;
            if (c < (int)nc) {
                const int kz = c / sxy, rem = c - kz * sxy, ky = rem / sx, kx = rem - ky * sx;
                code = cell_code(r.lo[0] + kx, r.lo[1] + ky, r.lo[2] + kz);
                const unsigned b = bucket_of(code, mask);
                beg = G.bstart[b];
                end = G.bend[b];
            }
            const int len = __reduce_max_sync(0xffffffffu, end - beg);
            for (int k = 0; k < len; ++k) {
                const int j = beg + k;
                bool hit = false;
                int q = -1;
                if (j < end && G.code[j] == code) {
                    q = G.prim[j];
                    if (!qviol[q]) {
                        double qlo[3], qhi[3];
                        if (cls == 1) vbox(A, q, qlo, qhi);
                        else load_box(cls == 0 ? A.tbox : A.ebox, q, qlo, qhi);
                        hit = overlap6(lo, hi, qlo, qhi) && min_corner_in(lo, qlo, inv, code) && partner_ok(q);
                    }
                }
                if (cls == 1) step(hit, q, p);
                else step(hit, p, q);
            }
        }
    } else {
        // box too large for a cell walk: every non-violating partner
        const int nq = cls == 0 ? A.ntris : (cls == 1 ? W.nw : A.nedges);
        for (int q0 = 0; q0 < nq; q0 += 32) {
            const int q = q0 + lane;
            bool hit = false;
            if (q < nq && !qviol[q] && (cls != 1 || W.vert_used[q])) {
                double qlo[3], qhi[3];
                if (cls == 1) vbox(A, q, qlo, qhi);
                else load_box(cls == 0 ? A.tbox : A.ebox, q, qlo, qhi);
                hit = overlap6(lo, hi, qlo, qhi) && partner_ok(q);
            }
            if (cls == 1) step(hit, q, p);
            else step(hit, p, q);
        }
    }
    // violator x violator: vertex side against violating triangles, edges against later ones
    if (cls != 1) {
        const int* __restrict__ L = cls == 0 ? A.tlist : A.elist;
        const int n = cls == 0 ? A.nt : A.ne;
        for (int k0 = cls == 0 ? 0 : li + 1; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool hit = false;
            int f = -1;
            if (k < n) {
                f = L[k];
                double qlo[3], qhi[3];
                load_box(cls == 0 ? A.tbox : A.ebox, f, qlo, qhi);
                hit = overlap6(lo, hi, qlo, qhi) && partner_ok(f);
            }
            step(hit, p, f);
        }
    }
    if (PASS == 0 && lane == 0) counts[t] = cnt;
}


// Fused filter + stable compaction of a pair set (subset / motion-free sites).
// Pass 1 (k_keep_tiles): per tile of kKeepTile pairs (one block), the keep test as
// a bitmask (one ballot word per 32 pairs) and the tile's count.  Pass 2
// (k_compact_tiles), after an exclusive scan of the counts: kept rows copied in
// order.  Replaces flag array + select + index gather (one pass less over P).
constexpr int kKeepTile = 256;  // one pair per thread

struct KeepArgs {
    const unsigned long long* __restrict__ keys;
    int64_t P;
    const double* __restrict__ vlo;
    const double* __restrict__ vhi;
    const double* __restrict__ tbox;
    const double* __restrict__ ebox;
    const uint8_t* __restrict__ vviol;  // nullable: no violators
    const uint8_t* __restrict__ tviol;
    const uint8_t* __restrict__ eviol;
};

__device__ __forceinline__ bool keep_pair(const KeepArgs& A, int64_t i) {
    const unsigned long long k = A.keys[i];
    const int p = (int)((k >> 32) & 0x7fffffffu), q = (int)(k & 0xffffffffu);
    const bool ee = (k >> 63) != 0;
    if (A.vviol != nullptr && (ee ? (A.eviol[p] | A.eviol[q]) != 0 : (A.vviol[p] | A.tviol[q]) != 0))
        return false;  // re-found by k_subset_query
    double alo[3], ahi[3], blo[3], bhi[3];
    if (ee) {
        load_box(A.ebox, p, alo, ahi);
        load_box(A.ebox, q, blo, bhi);
    } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            alo[c] = A.vlo[3 * (int64_t)p + c];
            ahi[c] = A.vhi[3 * (int64_t)p + c];
        }
        load_box(A.tbox, q, blo, bhi);
    }
    return overlap6(alo, ahi, blo, bhi);
}

__global__ void __launch_bounds__(256) k_keep_tiles(KeepArgs A, unsigned* __restrict__ bits,
                                                    int* __restrict__ tile_count) {
    __shared__ int wsum[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kKeepTile;
    const int64_t i = base + threadIdx.x;
    const bool keep = i < A.P && keep_pair(A, i);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) {
        bits[(base >> 5) + w] = m;
        wsum[w] = __popc(m);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int j = 0; j < 8; ++j) t += wsum[j];
        tile_count[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_compact_tiles(const unsigned* __restrict__ bits,
                                                       const int* __restrict__ tile_off, int64_t P,
                                                       const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                                                       const unsigned long long* __restrict__ keys,
                                                       int8_t* __restrict__ kind_o, int4* __restrict__ idx_o,
                                                       unsigned long long* __restrict__ keys_o) {
    constexpr int W = kKeepTile / 32;  // ballot words per tile
    __shared__ int wpre[W];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kKeepTile;
    const unsigned* __restrict__ tb = bits + (base >> 5);
    if (w == 0) {  // exclusive prefix of the word popcounts
        const int c = lane < W ? __popc(tb[lane]) : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane < W) wpre[lane] = inc - c;
    }
    __syncthreads();
    const unsigned m = tb[w];
    const int64_t i = base + threadIdx.x;
    if (i < P && ((m >> lane) & 1u)) {
        const int pos = tile_off[blockIdx.x] + wpre[w] + __popc(m & ((1u << lane) - 1u));
        kind_o[pos] = kind[i];
        idx_o[pos] = idx[i];
        keys_o[pos] = keys[i];
    }
}


}  // namespace cs
