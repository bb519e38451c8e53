// Broad phase: candidate VT / EE pairs over swept, margin-inflated fp64 boxes.
//
// Produces exactly the SET reference broad_phase returns
// (pkg/src/clothsim/collision/bvh.py:207-292; derivation in oracle/broad.py):
//   VT (v, f): v not in f, box(v) overlaps box(f), not (v static and f static)
//   EE (E, F): E < F, vertex-disjoint, box(E) overlaps box(F), not both static
// with the reference's edge-edge ORIENTATION (which edge comes first in the row),
// computed from the static patch partition exactly as the reference's
// first-occurrence dedup picks it (bvh.py:264-286).  Row order is deterministic
// (vertex-major VT block, then edge-major EE block, traversal order inside).
//
// Structure: two static-topology binary trees over Morton-sorted rest-pose
// primitives (triangles for VT queries, edges for EE queries), built once on the
// host; per query: vertex boxes -> leaf boxes -> atomic-flag bottom-up refit ->
// count pass -> exclusive scan -> write pass.  Boxes stay fp64 so overlap tests
// are exact (an fp32 filter could reject a pair the reference keeps).
#include "common.cuh"

namespace cs {

struct Tree {
    int nleaf;                       // number of primitives
    const int* __restrict__ left;    // (nleaf-1) child codes: >=0 internal, <0 leaf ~pos
    const int* __restrict__ right;
    const int* __restrict__ parent;  // (nleaf-1) internal parent (-1 root)
    const int* __restrict__ leaf_parent;  // (nleaf)
    const int* __restrict__ prim;    // (nleaf) primitive id at sorted leaf position
    double* node_lo;                 // (nleaf-1)*3
    double* node_hi;
    double* leaf_lo;                 // (nleaf)*3 in leaf order
    double* leaf_hi;
    int* flags;                      // (nleaf-1)
};

__global__ void k_vertex_boxes(const double* __restrict__ x0, const double* __restrict__ x1, int n, double margin,
                               double* __restrict__ vlo, double* __restrict__ vhi) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const double a = x0[i], b = x1[i];
    vlo[i] = np_min(a, b) - margin;
    vhi[i] = np_max(a, b) + margin;
}

// leaf boxes (primitive = triangle (arity 3) or edge (arity 2)) then bottom-up refit
__global__ void k_refit(Tree T, const int* __restrict__ verts, int arity, const double* __restrict__ vlo,
                        const double* __restrict__ vhi) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= T.nleaf) return;
    const int pr = T.prim[p];
    double lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        lo[c] = vlo[3 * verts[arity * pr] + c];
        hi[c] = vhi[3 * verts[arity * pr] + c];
    }
    for (int k = 1; k < arity; ++k) {
        const int v = verts[arity * pr + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = np_min(lo[c], vlo[3 * v + c]);
            hi[c] = np_max(hi[c], vhi[3 * v + c]);
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        T.leaf_lo[3 * p + c] = lo[c];
        T.leaf_hi[3 * p + c] = hi[c];
    }
    if (T.nleaf == 1) return;
    int node = T.leaf_parent[p];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&T.flags[node], 1) == 0) return;  // first child to arrive stops
        __threadfence();
        const int l = T.left[node], r = T.right[node];
        const volatile double* llo = l >= 0 ? T.node_lo + 3 * l : T.leaf_lo + 3 * (~l);
        const volatile double* lhi = l >= 0 ? T.node_hi + 3 * l : T.leaf_hi + 3 * (~l);
        const volatile double* rlo = r >= 0 ? T.node_lo + 3 * r : T.leaf_lo + 3 * (~r);
        const volatile double* rhi = r >= 0 ? T.node_hi + 3 * r : T.leaf_hi + 3 * (~r);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T.node_lo[3 * node + c] = fmin(llo[c], rlo[c]);
            T.node_hi[3 * node + c] = fmax(lhi[c], rhi[c]);
        }
        node = T.parent[node];
    }
}

__device__ __forceinline__ bool overlap(const double* lo_a, const double* hi_a, const double* __restrict__ lo_b,
                                        const double* __restrict__ hi_b) {
    return (lo_a[0] <= hi_b[0]) && (lo_b[0] <= hi_a[0]) && (lo_a[1] <= hi_b[1]) && (lo_b[1] <= hi_a[1]) &&
           (lo_a[2] <= hi_b[2]) && (lo_b[2] <= hi_a[2]);
}

// Visit every leaf whose box overlaps [qlo, qhi]; f(leaf_pos) called in traversal order.
template <typename F>
__device__ __forceinline__ void traverse(const Tree& T, const double qlo[3], const double qhi[3], F&& f) {
    if (T.nleaf == 1) {
        if (overlap(qlo, qhi, T.leaf_lo, T.leaf_hi)) f(0);
        return;
    }
    int stack[64];
    int sp = 0;
    int node = 0;
    while (true) {
        const int l = T.left[node], r = T.right[node];
        bool go_l, go_r;
        if (l >= 0) go_l = overlap(qlo, qhi, T.node_lo + 3 * l, T.node_hi + 3 * l);
        else {
            go_l = false;
            if (overlap(qlo, qhi, T.leaf_lo + 3 * (~l), T.leaf_hi + 3 * (~l))) f(~l);
        }
        if (r >= 0) go_r = overlap(qlo, qhi, T.node_lo + 3 * r, T.node_hi + 3 * r);
        else {
            go_r = false;
            if (overlap(qlo, qhi, T.leaf_lo + 3 * (~r), T.leaf_hi + 3 * (~r))) f(~r);
        }
        if (go_l && go_r) {
            stack[sp++] = r;
            node = l;
        } else if (go_l) {
            node = l;
        } else if (go_r) {
            node = r;
        } else {
            if (sp == 0) break;
            node = stack[--sp];
        }
    }
}

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
};

// pass 0: counts; pass 1: write rows at offsets
template <int PASS>
__global__ void k_query_vt(Tree T, WorldTopo W, const double* __restrict__ vlo, const double* __restrict__ vhi,
                           int* __restrict__ counts, const int* __restrict__ offsets, int8_t* __restrict__ kind,
                           int4* __restrict__ idx, unsigned long long* __restrict__ keys) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= W.nw) return;
    int cnt = 0;
    if (W.vert_used[v]) {
        const double qlo[3] = {vlo[3 * v], vlo[3 * v + 1], vlo[3 * v + 2]};
        const double qhi[3] = {vhi[3 * v], vhi[3 * v + 1], vhi[3 * v + 2]};
        const bool vs = W.vert_static[v];
        int out = PASS == 1 ? offsets[v] : 0;
        traverse(T, qlo, qhi, [&](int leaf) {
            const int f = T.prim[leaf];
            const int a = W.tris[3 * f], b = W.tris[3 * f + 1], c = W.tris[3 * f + 2];
            if (a == v || b == v || c == v) return;
            if (vs && W.tri_static[f]) return;
            if (PASS == 1) {
                kind[out] = CS_VT;
                idx[out] = make_int4(v, a, b, c);
                keys[out] = ((unsigned long long)(unsigned)v << 32) | (unsigned)f;
                ++out;
            }
            ++cnt;
        });
    }
    if (PASS == 0) counts[v] = cnt;
}

__device__ __forceinline__ unsigned long long place_key(int pa, int sa, int pb, int sb, bool& a_first) {
    a_first = (pa < pb) || (pa == pb && sa < sb);
    const unsigned long long p1 = a_first ? pa : pb, p2 = a_first ? pb : pa;
    const unsigned long long s1 = a_first ? sa : sb, s2 = a_first ? sb : sa;
    const unsigned long long same = pa == pb;
    return ((((same << 24 | p1) << 24 | p2) << 3 | s1) << 3) | s2;
}

// reference orientation of edge pair (E, F), E < F: true when F comes first (bvh.py:264-286)
__device__ bool ee_flip(const WorldTopo& W, int E, int F) {
    unsigned long long best = ~0ull;
    bool flip = false;
    for (int ka = 0; ka < 2; ++ka) {
        const int a = W.edge_tris[2 * E + ka];
        if (a < 0) continue;
        for (int kb = 0; kb < 2; ++kb) {
            const int b = W.edge_tris[2 * F + kb];
            if (b < 0) continue;
            if (W.tri_static[a] && W.tri_static[b]) continue;
            bool a_first;
            const unsigned long long place = place_key(W.patch[a], W.pslot[a], W.patch[b], W.pslot[b], a_first);
            const int sa = W.edge_slot[2 * E + ka], sb = W.edge_slot[2 * F + kb];
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

template <int PASS>
__global__ void k_query_ee(Tree T, WorldTopo W, int n_edges, const double* __restrict__ vlo,
                           const double* __restrict__ vhi, int* __restrict__ counts,
                           const int* __restrict__ offsets, int8_t* __restrict__ kind, int4* __restrict__ idx,
                           unsigned long long* __restrict__ keys) {
    const int E = blockIdx.x * blockDim.x + threadIdx.x;
    if (E >= n_edges) return;
    const int a0 = W.edges[2 * E], a1 = W.edges[2 * E + 1];
    double qlo[3], qhi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        qlo[c] = np_min(vlo[3 * a0 + c], vlo[3 * a1 + c]);
        qhi[c] = np_max(vhi[3 * a0 + c], vhi[3 * a1 + c]);
    }
    const bool es = W.edge_static[E];
    int cnt = 0;
    int out = PASS == 1 ? offsets[E] : 0;
    traverse(T, qlo, qhi, [&](int leaf) {
        const int F = T.prim[leaf];
        if (F <= E) return;
        const int b0 = W.edges[2 * F], b1 = W.edges[2 * F + 1];
        if (a0 == b0 || a0 == b1 || a1 == b0 || a1 == b1) return;
        if (es && W.edge_static[F]) return;
        if (PASS == 1) {
            const bool fl = ee_flip(W, E, F);
            kind[out] = CS_EE;
            idx[out] = fl ? make_int4(b0, b1, a0, a1) : make_int4(a0, a1, b0, b1);
            keys[out] = (1ull << 63) | ((unsigned long long)(unsigned)E << 32) | (unsigned)F;
            ++out;
        }
        ++cnt;
    });
    if (PASS == 0) counts[E] = cnt;
}

}  // namespace cs
