// Pair bookkeeping between CCD sites.
//
//   k_hash_insert / k_hash_lookup   life-span carry-over by canonical pair key
//                                   (reference stepper.py:300-305, pairs.py:51-62).
//                                   Keys: VT (0, v, f), EE (1, E, F) with E < F, which
//                                   identify the same pairs as the reference's sorted
//                                   vertex-id keys.  Open addressing, 64-bit CAS; the
//                                   result is order independent, hence deterministic.
//   k_mark_segments                 per-free-vertex [beg, end) ranges over the stably
//                                   sorted collision stamps (np.add.at order per vertex)
//   k_flag_engaged                  engaged & weight > 0 flags (stepper.py:245)
#include "common.cuh"

namespace cs {

#define CS_EMPTY_KEY 0xffffffffffffffffull

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

__global__ void k_hash_insert(const unsigned long long* __restrict__ keys, const int* __restrict__ life, int64_t P,
                              unsigned long long* __restrict__ tkeys, int* __restrict__ tvals,
                              unsigned long long mask) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    if (life[i] == 0) return;  // absent keys read back as 0
    const unsigned long long k = keys[i];
    unsigned long long h = mix64(k) & mask;
    while (true) {
        const unsigned long long prev = atomicCAS(&tkeys[h], CS_EMPTY_KEY, k);
        if (prev == CS_EMPTY_KEY || prev == k) {
            tvals[h] = life[i];
            return;
        }
        h = (h + 1) & mask;
    }
}

__global__ void k_hash_lookup(const unsigned long long* __restrict__ keys, int64_t P,
                              const unsigned long long* __restrict__ tkeys, const int* __restrict__ tvals,
                              unsigned long long mask, int* __restrict__ life) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    const unsigned long long k = keys[i];
    unsigned long long h = mix64(k) & mask;
    int out = 0;
    while (true) {
        const unsigned long long t = tkeys[h];
        if (t == k) {
            out = tvals[h];
            break;
        }
        if (t == CS_EMPTY_KEY) break;
        h = (h + 1) & mask;
    }
    life[i] = out;
}

__global__ void k_flag_engaged(const uint8_t* __restrict__ engaged, const double* __restrict__ weight, int64_t P,
                               uint8_t* __restrict__ flags, int* __restrict__ count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool f = false;
    if (i < P) {
        f = engaged[i] && (weight[i] > 0.0);
        flags[i] = f;
    }
    block_count(f, count);
}

__global__ void k_count_nonzero(const int* __restrict__ v, int64_t P, int* __restrict__ count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool f = i < P && v[i] != 0;
    block_count(f, count);
}

__global__ void k_count_true(const uint8_t* __restrict__ v, int64_t P, int* __restrict__ count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool f = i < P && v[i];
    block_count(f, count);
}

// sorted keys (free row < nrows, or a sentinel >= nrows for dropped) -> seg_beg/seg_end
// per row, plus the ascending list of distinct rows (collided vertices for the reduced update)
__global__ void k_mark_segments(const int* __restrict__ skey, int m, int nrows, int* __restrict__ seg_beg,
                                int* __restrict__ seg_end, int* __restrict__ rows_out_flag) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int k = skey[j];
    if (k >= nrows) return;
    if (j == 0 || skey[j - 1] != k) {
        seg_beg[k] = j;
        if (rows_out_flag) rows_out_flag[j] = 1;
    }
    if (j == m - 1 || skey[j + 1] != k) seg_end[k] = j + 1;
}

// Stable compaction of the indices of the set u8 flags (the engaged pairs, in pair
// order): tiles of 1024 flags (256 threads x 4), tile counts, exclusive scan, writes.
constexpr int kFlagTile = 1024;
__device__ __forceinline__ uchar4 load_flags4(const uint8_t* __restrict__ f, int64_t i0, int64_t n) {
    if (i0 + 4 <= n) return *reinterpret_cast<const uchar4*>(f + i0);
    uchar4 v = make_uchar4(0, 0, 0, 0);
    if (i0 < n) v.x = f[i0];
    if (i0 + 1 < n) v.y = f[i0 + 1];
    if (i0 + 2 < n) v.z = f[i0 + 2];
    return v;
}
__global__ void __launch_bounds__(256) k_flag_tiles(const uint8_t* __restrict__ flags, int64_t n,
                                                    int* __restrict__ tile_count) {
    using Reduce = cub::BlockReduce<int, 256>;
    __shared__ typename Reduce::TempStorage tmp;
    const uchar4 v = load_flags4(flags, (int64_t)blockIdx.x * kFlagTile + 4 * threadIdx.x, n);
    const int t = Reduce(tmp).Sum((v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0));
    if (threadIdx.x == 0) tile_count[blockIdx.x] = t;
}
__global__ void __launch_bounds__(256) k_flag_compact(const uint8_t* __restrict__ flags, int64_t n,
                                                      const int* __restrict__ tile_off, int* __restrict__ out) {
    using Scan = cub::BlockScan<int, 256>;
    __shared__ typename Scan::TempStorage tmp;
    const int64_t i0 = (int64_t)blockIdx.x * kFlagTile + 4 * threadIdx.x;
    const uchar4 v = load_flags4(flags, i0, n);
    const bool f[4] = {v.x != 0, v.y != 0, v.z != 0, v.w != 0};
    int pos;
    Scan(tmp).ExclusiveSum(f[0] + f[1] + f[2] + f[3], pos);
    pos += tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (f[j]) out[pos++] = (int)(i0 + j);
}

// rows with a non-empty stamp segment (seg_end zeroed before k_mark_segments)
struct SegNonEmpty {
    const int* __restrict__ seg_end;
    __host__ __device__ __forceinline__ bool operator()(int r) const { return seg_end[r] > 0; }
};

// ---- stamp plan (driver-cached row order of the collision stamps, reused across the
// LG iterations of one pair set).  Plan entries are ordered by the merge key
// row << 34 | pair << 2 | slot, i.e. by free row and, within a row, in pair order
// (np.add.at order over the engaged pairs: entries of pairs that are not engaged carry
// w = 0 and are skipped by every consumer).
constexpr int kPlanRowShift = 34;

// merge keys of the row-sorted entries of a freshly built plan
// (+ the plan position of every entry slot: dst[src] = j, -1 elsewhere by a memset)
__global__ void k_plan_keys(const int* __restrict__ skey_s, const int* __restrict__ ssrc_s,
                            const int* __restrict__ sel, int m, unsigned long long* __restrict__ pkey,
                            int* __restrict__ dst) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int src = ssrc_s[j];
    pkey[j] = ((unsigned long long)skey_s[j] << kPlanRowShift) | ((unsigned long long)sel[src >> 2] << 2) |
              (unsigned long long)(src & 3);
    dst[src] = j;
}

// pair -> position in the plan's pair list (the rest stays -1 from a memset)
__global__ void k_plan_pair_u(const int* __restrict__ sel, int A, int* __restrict__ pair_u) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < A) pair_u[sel[a]] = a;
}

// pairs newly engaged during the plan's lifetime: appended to the plan's pair list
// (sel[U0 + j]); their four entries get merge keys (or the sentinel when the slot can
// never stamp: immovable endpoint or clipped barycentric weight 0, as k_collision_terms)
__global__ void k_plan_new(const int* __restrict__ newsel, int N, int U0, const int8_t* __restrict__ kind,
                           const int4* __restrict__ idx, const double* __restrict__ bary, int n_cloth,
                           const int* __restrict__ free_index, unsigned long long sentinel, int* __restrict__ sel,
                           int* __restrict__ pair_u, unsigned long long* __restrict__ nkey,
                           int* __restrict__ nsrc) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    const int i = newsel[j];
    sel[U0 + j] = i;
    pair_u[i] = U0 + j;
    const int kd = kind[i];
    const int4 id = idx[i];
    const double l1 = bary[2 * i], l2 = bary[2 * i + 1];
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
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int v = ids[k];
        const int row = v < n_cloth ? free_index[v] : -1;
        const bool ok = row >= 0 && clip01(gam[k]) > 0.0;
        nkey[4 * j + k] = ok ? (((unsigned long long)row << kPlanRowShift) | ((unsigned long long)i << 2) | k)
                             : sentinel;
        nsrc[4 * j + k] = 4 * (U0 + j) + k;
    }
}

// row segments + entry positions of a merged plan (sentinel entries trail and are ignored)
__global__ void k_plan_segments(const unsigned long long* __restrict__ pkey, const int* __restrict__ psrc, int m,
                                int nrows, int* __restrict__ seg_beg, int* __restrict__ seg_end,
                                int* __restrict__ dst, int side) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const unsigned long long r = pkey[j] >> kPlanRowShift;
    if (r >= (unsigned long long)nrows) return;
    dst[psrc[j]] = side ? -2 - j : j;  // plan_store encoding
    if (j == 0 || (pkey[j - 1] >> kPlanRowShift) != r) seg_beg[r] = j;
    if (j == m - 1 || (pkey[j + 1] >> kPlanRowShift) != r) seg_end[r] = j + 1;
}

// rows whose stamps carry weight (delta_i > 0): the reduced Gram's row list
__global__ void k_flag_positive(const double* __restrict__ v, int m, uint8_t* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flag[i] = v[i] > 0.0;
}

struct U64Less {
    __host__ __device__ __forceinline__ bool operator()(unsigned long long a, unsigned long long b) const {
        return a < b;
    }
};

// compaction helpers for the per-stage collision-terms entry point
// Stable compaction of the stamp entries on a free row (key < nf) with their keys,
// in entry order (replaces a flag select + key gather): tile counts over 256 pairs
// (4 entries each) per block, an exclusive scan, then each block writes its kept
// (entry, key) pairs at its offset.
constexpr int kKeptTile = 256;
__global__ void __launch_bounds__(kKeptTile) k_kept_tiles(const int* __restrict__ key, int64_t A, int nf,
                                                         int* __restrict__ tile_count) {
    using Reduce = cub::BlockReduce<int, kKeptTile>;
    __shared__ typename Reduce::TempStorage tmp;
    const int64_t a = (int64_t)blockIdx.x * kKeptTile + threadIdx.x;
    int c = 0;
    if (a < A) {
        const int4 k = reinterpret_cast<const int4*>(key)[a];
        c = (k.x < nf) + (k.y < nf) + (k.z < nf) + (k.w < nf);
    }
    const int t = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) tile_count[blockIdx.x] = t;
}
__global__ void __launch_bounds__(kKeptTile) k_kept_compact(const int* __restrict__ key, int64_t A, int nf,
                                                           const int* __restrict__ tile_off, int* __restrict__ src,
                                                           int* __restrict__ key_out) {
    using Scan = cub::BlockScan<int, kKeptTile>;
    __shared__ typename Scan::TempStorage tmp;
    const int64_t a = (int64_t)blockIdx.x * kKeptTile + threadIdx.x;
    int4 k = make_int4(nf, nf, nf, nf);
    if (a < A) k = reinterpret_cast<const int4*>(key)[a];
    const int kk[4] = {k.x, k.y, k.z, k.w};
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) c += kk[j] < nf;
    int pos;
    Scan(tmp).ExclusiveSum(c, pos);
    pos += tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (kk[j] < nf) {
            src[pos] = (int)(4 * a + j);
            key_out[pos] = kk[j];
            ++pos;
        }
}

__global__ void k_key_kept(const int* __restrict__ key, int m, int nf, uint8_t* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flag[i] = key[i] < nf ? 1 : 0;
}
__global__ void k_gather_terms(const int* __restrict__ pick, const int* __restrict__ count,
                               const int* __restrict__ sel, const int4* __restrict__ idx,
                               const double4* __restrict__ stamp, int* __restrict__ ids_out,
                               double* __restrict__ w_out, double* __restrict__ t_out) {
    const int n = count[0];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int o = pick[k];
        const int4 id = idx[sel[o >> 2]];
        const int slot = o & 3;
        ids_out[k] = slot == 0 ? id.x : (slot == 1 ? id.y : (slot == 2 ? id.z : id.w));
        const double4 st = ldg256(stamp + o);
        w_out[k] = st.w;
        t_out[3 * k] = st.x;
        t_out[3 * k + 1] = st.y;
        t_out[3 * k + 2] = st.z;
    }
}

// DBB baseline weights (pairs.py:83-99): -kappa (d - dh)^2 ln(d / dh) for d < dh, d =
// max(dist, 1e-12) (stepper.py:490); engaged = weight > 0.  numpy order: ((-kappa) sq) ln.
__global__ void k_dbb_weights(const double* __restrict__ dist, int64_t P, double dh, double kappa,
                              uint8_t* __restrict__ engaged, double* __restrict__ weight, int* __restrict__ count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool e = false;
    if (i < P) {
        const double d = np_max(dist[i], 1e-12);
        double w = 0.0;
        if (d < dh) {
            const double dd = d - dh;
            w = ((-kappa) * (dd * dd)) * log(d / dh);
        }
        weight[i] = w;
        e = w > 0.0;
        engaged[i] = e;
    }
    block_count(e, count);
}

__global__ void k_clamp_keys(int* __restrict__ k, int m, int cap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m && k[i] > cap) k[i] = cap;
}

__global__ void k_iota(int* __restrict__ a, int64_t m) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) a[i] = (int)i;
}

__global__ void k_fill_u64(unsigned long long* __restrict__ a, int64_t m, unsigned long long v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) a[i] = v;
}

__global__ void k_rf_weights(const double* __restrict__ dist, int64_t P, double d_hat, double k,
                             uint8_t* __restrict__ engaged, double* __restrict__ weight) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    const bool e = dist[i] < 2.0 * d_hat;
    engaged[i] = e;
    weight[i] = e ? k : 0.0;
}

__global__ void k_neg_gather(const double* __restrict__ g, const int* __restrict__ free_ids, int nf,
                             double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int v = free_ids[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[3 * i + c] = -g[3 * v + c];
}

}  // namespace cs

namespace cs {

// v = (x_final - x) / h  (stepper.py:597)
__global__ void k_velocity_update(const double* __restrict__ xfin, const double* __restrict__ x,
                                  double* __restrict__ v, int64_t m, double h) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) v[i] = (xfin[i] - x[i]) / h;
}

// delta_i = sum of stamp weights in np.add.at order (stepper.py:653-657)
__global__ void k_stamp_delta(int nf, const int* __restrict__ seg_beg, const int* __restrict__ seg_end,
                              const int* __restrict__ src, const double4* __restrict__ stamp,
                              double* __restrict__ delta) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    double d = 0.0;
    if (seg_beg != nullptr)
        for (int k = seg_beg[i]; k < seg_end[i]; ++k) {
            const double w = stamp[src[k]].w;
            if (w > 0.0) d = d + w;  // plan entries outside the engaged set carry w = 0
        }
    delta[i] = d;
}

// per-stage inputs (flat weights, targets) -> the driver's stamp records
__global__ void k_pack_stamps(const double* __restrict__ w, const double* __restrict__ t, int m,
                              double4* __restrict__ stamp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) stg256(stamp + i, t[3 * i], t[3 * i + 1], t[3 * i + 2], w[i]);
}

// stamp sort keys from cloth vertex ids: free row or sentinel (constraints.py:252-255)
__global__ void k_stamp_keys(const int* __restrict__ ids, int m, const int* __restrict__ free_index, int n,
                             int* __restrict__ key) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int v = ids[j];
    const int f = (v >= 0 && v < n) ? free_index[v] : -1;
    key[j] = f >= 0 ? f : 0x7fffffff;
}

__global__ void k_nonzero_flags(const double* __restrict__ d, int m, int* __restrict__ flags) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flags[i] = d[i] != 0.0;
}

}  // namespace cs
