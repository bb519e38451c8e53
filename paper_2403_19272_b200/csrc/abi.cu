// C ABI + native step driver for the sm_100a cloth pipeline.
//
// cs_step() is reference Simulation.step() (pkg/src/clothsim/stepper.py:454-624)
// in the NDB barrier mode: warm start -> CCD site -> outer/inner local-global
// loops (collision stamps, rhs, reduced correction, A-Jacobi smoothing, partial
// CCD + life-span update) -> CCD site per outer loop -> exit line search ->
// residual forwarding (:626-672).  All arithmetic runs in the kernels of
// narrow.cu / solver.cu / broad.cu / pairs.cu; the host only sequences launches
// and reads back one small scalar block at each data-dependent branch (the
// reference's own sync points: RMS exits, TOI clamps, pair counts).
//
// Single translation unit (unity build) so kernels stay in one module.
#include <cub/cub.cuh>
#include <cub/device/device_merge.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <thread>
#include <string>

#include "common.cuh"
#include "narrow.cu"
#include "solver.cu"
#include "broad.cu"
#include "pairs.cu"
#include "intersect.cu"
#include "../../include/clothsim_b200.h"

using namespace cs;

#define CS_TRY(expr)                                   \
    do {                                               \
        cudaError_t e_ = (expr);                       \
        if (e_ != cudaSuccess) return 1000 + (int)e_;  \
    } while (0)
#define CS_RET(expr)               \
    do {                           \
        int rc_ = (expr);          \
        if (rc_ != 0) return rc_;  \
    } while (0)

#include "stages.cu"  // scene-free stage kernels + their C entry points
#include "eigen.cu"   // device eigensolver block kernels (setup)

namespace {

// Stream the DBuf (re)allocations of the current call are ordered on.  Buffers come
// from the device's stream-ordered pool (cudaMallocAsync / cudaFreeAsync, release
// threshold raised at scene creation): a mid-run regrowth neither synchronises the
// device nor maps fresh memory once the pool has grown (a plain cudaFree/cudaMalloc
// pair of a few hundred MB costs tens of ms).
thread_local cudaStream_t t_alloc_stream = nullptr;

// The library's own stream-ordered pool per device (cudaMemPoolCreate): freed blocks
// stay mapped for the next regrowth, without touching the device's default pool that
// PyTorch / CuPy / other cudaMallocAsync users of the process share.
cudaMemPool_t lib_pool() {
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return pools[dev];
}

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool = lib_pool();
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    int ensure(size_t m, bool exact = false) {
        if (m <= n && p) return 0;
        if (p) cudaFreeAsync(p, t_alloc_stream);
        p = nullptr;
        // regrowth reserves 1.5x and a large first sizing 2x: per-step sizes (pairs, grid
        // entries, stamps) drift upward while the cloth settles; regrowth from the
        // library pool's slab costs microseconds, the headroom only saves the copies of
        // many small regrowths (and memory for many scenes per GPU matters more)
        size_t want = std::max<size_t>(m, 1);
        if (!exact) {
            if (n) want = std::max(want + want / 2, n + n / 2);
            else if (want > (1u << 16)) want *= 2;
        }
        static const bool trace = std::getenv("CS_TRACE_ALLOC") != nullptr;
        if (trace) std::fprintf(stderr, "[cs alloc] %zu -> %zu bytes\n", n * sizeof(T), want * sizeof(T));
        cudaError_t e = pool_alloc(reinterpret_cast<void**>(&p), want * sizeof(T), t_alloc_stream);
        if (e != cudaSuccess) {
            n = 0;
            p = nullptr;
            return 1000 + (int)e;
        }
        n = want;
        return 0;
    }
    // grow to >= m elements keeping the first `used` (stream-ordered copy)
    int grow_keep(size_t m, size_t used) {
        if (m <= n && p) return 0;
        T* old = p;
        p = nullptr;
        n = 0;
        CS_RET(ensure(2 * m, true));
        if (old) {
            if (used) {
                cudaError_t e = cudaMemcpyAsync(p, old, used * sizeof(T), cudaMemcpyDeviceToDevice, t_alloc_stream);
                if (e != cudaSuccess) return 1000 + (int)e;
            }
            cudaFreeAsync(old, t_alloc_stream);
        }
        return 0;
    }
    int upload(const T* host, size_t m) {
        CS_RET(ensure(m, true));
        if (m && host) {
            cudaError_t e = cudaStreamSynchronize(t_alloc_stream);
            if (e == cudaSuccess) e = cudaMemcpy(p, host, m * sizeof(T), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return 1000 + (int)e;
        }
        return 0;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// one hash-grid entry table (vertices, triangles or edges) of the broad phase
struct EntryBuf {
    int np = 0;
    unsigned T = 0;  // buckets (power of two)
    int log2T = 0;
    long long m = 0;  // entries
    int n_over_h = 0;
    DBuf<double> box, part, inv;
    DBuf<int> count, offset, prim, perm, perm_s, prim_s, run, n_run, bstart, bend, over, n_over, pcount, poffset;
    DBuf<int> lrows, lcount, loff, n_lrows;  // rows of long bucket runs (k_long_ee / k_long_vt)
    long long n_lrows_h = 0;
    DBuf<long long> iters, iter_off;
    DBuf<unsigned> masks;
    DBuf<unsigned> key, key_s;
    DBuf<unsigned long long> code, code_s;
    DBuf<uint8_t> is_over, head, zb, zb_s;
    int create(int n_prim, bool has_box) {
        np = n_prim;
        if (has_box) CS_RET(box.ensure(6LL * np));
        CS_RET(inv.ensure(1));
        CS_RET(count.ensure(np + 1));
        CS_RET(offset.ensure(np + 1));
        CS_RET(over.ensure(np));
        CS_RET(n_over.ensure(1));
        CS_RET(n_run.ensure(1));
        CS_RET(is_over.ensure(np));
        return 0;
    }
    void set_buckets(long long want) {
        T = 1024;
        log2T = 10;
        while ((long long)T < want) {
            T <<= 1;
            ++log2T;
        }
    }
    EntryTable view() const {
        return EntryTable{key_s.p, prim_s.p, code_s.p, zb_s.p, run.p, n_run.p, bstart.p, bend.p, (int)m};
    }
    void release() {
        for (DBuf<int>* b : {&lrows, &lcount, &loff, &n_lrows, &count, &offset, &prim, &perm, &perm_s, &prim_s, &run, &n_run, &bstart, &bend, &over,
                             &n_over, &pcount, &poffset})
            b->release();
        iters.release(); iter_off.release(); masks.release();
        box.release(); part.release(); inv.release(); key.release(); key_s.release(); code.release();
        code_s.release(); is_over.release(); head.release(); zb.release(); zb_s.release();
    }
};

struct PairBuf {
    long long P = 0;
    DBuf<int8_t> kind;
    DBuf<int4> idx;
    DBuf<unsigned long long> keys;
    DBuf<double> toi, filt, bary, dist, normal, weight;
    DBuf<int> life;
    DBuf<uint8_t> engaged;
    // near / far split for the partial CCD passes on this set (k_witness, EngageOut.split)
    DBuf<int> near_l;        // near pairs (pair order), then the far pairs (reversed)
    long long n_near = 0;    // read at the sync after engage (I_NEAR)
    bool split_valid = false;
    int reserve(long long m) {
        // first real sizing (from the 1024-row placeholder) takes 2x headroom, later
        // regrowth 1.5x: pair counts drift upward while the cloth settles
        if (m <= (long long)kind.n && kind.p) return 0;
        const bool first = kind.n <= 1024 && m > 1024;
        m = first ? 2 * m : m + m / 2;
        CS_RET(kind.ensure(m, true));
        CS_RET(idx.ensure(m, true));
        CS_RET(keys.ensure(m, true));
        CS_RET(toi.ensure(m, true));
        CS_RET(filt.ensure(m, true));
        CS_RET(bary.ensure(2 * m, true));
        CS_RET(dist.ensure(m, true));
        CS_RET(normal.ensure(3 * m, true));
        CS_RET(weight.ensure(m, true));
        CS_RET(life.ensure(m, true));
        CS_RET(engaged.ensure(m, true));
        return 0;
    }
    void release() {
        kind.release(); idx.release(); keys.release(); toi.release(); filt.release(); bary.release();
        dist.release(); normal.release(); weight.release(); life.release(); engaged.release();
        near_l.release();
        split_valid = false;
    }
};

// scalar slots (doubles) read back in one D2H copy
enum { S_SQ = 0, S_CLAMP_MIN = 1, S_CLAMP = 2, S_CLAMP_BAD = 3, S_NORM0 = 4, S_NORM1 = 5, S_NORM_F = 6,
       S_RES = 7, S_DFNORM = 8, S_DFSCALE = 9, S_MINBITS = 10, S_TOIEXIT = 11, S_COUNT = 16 };
// partial CCD near / far split margin, in units of d_hat (EngageOut.near_thresh; the
// far gate's per-pair displacement bound is what makes a far pair exact, this only
// sets which list a pair starts in: 0.05 and 0.25 were slower than 0)
constexpr double kFarDelta = 0.0;
enum { I_ENG = 0, I_BAD = 1, I_ROWS = 2, I_VT = 3, I_EE = 4, I_FALLBACK = 5, I_LIVE = 6, I_FLAG = 7, I_WLF = 8,
       I_NEW = 9, I_NEAR = 10, I_FARREST = 11, I_COUNT = 12 };

const int kStages = 8;
enum { T_WARM = 0, T_LOCAL, T_GLOBAL, T_SMOOTH, T_BROAD, T_PARTIAL, T_FULL, T_RF };

}  // namespace

struct cs_scene {
    // sizes
    int n = 0, nf = 0, npin = 0, nobs = 0, nw = 0, ne = 0, ns = 0, ntw = 0, new_ = 0, rb = 0, r = 0;
    cs_step_config cfg{};
    SamplePattern pat{};
    // static cloth data
    DBuf<int> free_ids, free_index, pin_ids, pin_slot;
    DBuf<double> mass, fext, mh2;
    DBuf<int> e0, e1, rinc_ptr, rinc, ginc_ptr, ginc, st, binc_ptr, binc;
    DBuf<double> erest, ew, bk, bw;
    DBuf<int> sell_ptr, sell_col, hfp_ptr, hfp_col;
    DBuf<double> sell_val, diag, hfp_val;
    int nslices = 0;
    bool has_fp = false;
    DBuf<double> U, V, lam;
    // world topology
    DBuf<int> wtris, wedges, edge_tris, edge_slot, patch, pslot;
    DBuf<uint8_t> tri_static, vert_static, vert_used, edge_static;
    DBuf<ulonglong2> eflip;
    EntryBuf vtab, ttab, etab;
    DBuf<int> ocount, ooffset;
    // state
    DBuf<double> x, v, xprev, df, obs;
    DBuf<double> dfn;  // residual-forwarding result, committed with the new state
    int step_index = 0;
    // work arrays
    DBuf<double> z, xs_w, xc_w, anchor_w, tmp_w, xf, xf0, b, t, delta, prev_outer, grad, fr;
    DBuf<double> pins_next_d, obs_next_d;
    DBuf<double> vlo, vhi, vdisp, tdisp, edisp;
    DBuf<float> fvbox, ftbox, febox;  // fp32 outward-rounded copies for the site filter
    double bmargin = 0.0;
    PairBuf pa, pb;  // current and next pair sets
    PairBuf* cur = &pa;
    PairBuf* nxt = &pb;
    DBuf<int> sel, skey, ssrc, skey_s, ssrc_s, seg_beg, seg_end, rowflag, rows_act, skey_c;  // rowflag: stage APIs
    DBuf<double4> stamp;  // collision stamps: target xyz + weight
    DBuf<unsigned long long> hkeys;
    DBuf<int> hvals;
    DBuf<double> part, part2, spart, rhs_red, gram_red, q, Xred, beta_red, norms;
    int pending_checks = 0;
    DBuf<int> fallback;
    DBuf<int> wl_full, wl_dist;
    DBuf<uint8_t> keep_flag;
    DBuf<unsigned> keep_bits;
    DBuf<int> tile_cnt, tile_off;
    // subset sites: a moving site served from the step's base site (subset_site)
    PairBuf basepr;
    DBuf<double> blo, bhi;
    DBuf<uint8_t> vviol, tviol, eviol;
    DBuf<int> vlist, tlist, elist, qcount, qoff;
    DBuf<unsigned long long> query_dbg;  // CS_TRACE_SITES counters
    bool base_valid = false;
    double base_margin = -1.0;
    int subset_fail = 0;  // consecutive outer-loop sites that refused the subset path
    DBuf<char> cub_tmp;
    DBuf<double> d_scal;
    DBuf<int> d_iscal;
    double* h_scal = nullptr;
    int* h_iscal = nullptr;
    double* h_stage = nullptr;  // pinned: [pins (3 npin) | obstacles (3 nobs)]
    static constexpr int kMaxNormChecks = 64;
    double* h_norms = nullptr;  // pinned: smoother residual norms (divergence check)
    cudaStream_t s = 0;
    long long launches = 0;
    // timing
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
    int active_stage = -1;
    cudaEvent_t stage_start{};
    int sm_count = 148;
    bool stamps_valid = false;   // seg_beg/seg_end hold stamps for the current rhs
    int n_stamp_rows = 0;
    // Stamp plan: the row order of the collision stamps of pair set plan_pr, cached across
    // its LG iterations.  A superset of the engaged set: pairs that leave it keep their
    // entries (w = 0, skipped by the rhs); pairs that join are appended by k_partial_ndb
    // (newsel) and merged in by key (row, pair, slot) = np.add.at order within a row.
    // Entries live in a main list (pkey / ssrc_s / seg_beg / seg_end / stamp_p) and a
    // small side list of recently joined pairs (skey_sd / ssrc_sd / sseg_* / stamp_sd)
    // that the rhs interleaves by key; the side list is folded into the main list when it
    // outgrows 1/8 of it.  pdst[4u + k] = plan position of entry k of plan pair u
    // (plan_store encoding); k_partial_ndb writes the next iteration's stamps there.
    bool plan_valid = false;
    const PairBuf* plan_pr = nullptr;
    long long plan_U = 0;        // pairs in the plan (sel[0, plan_U))
    long long plan_Umain = 0;    // sel[0, plan_Umain) have their entries in the main list
    long long plan_M = 0;        // main-list entries (row-sorted, incl. trailing sentinels)
    long long side_M = 0;        // side-list entries
    long long plan_new = 0;      // engaged pairs outside the plan at the last partial CCD
    long long plan_reuses = 0;
    bool fused_ok = false;       // k_partial_ndb wrote this plan's stamps at the candidate
    int last_loop_lg = 0;        // LG iterations of the last outer loop (plan worth building?)
    bool lazy_exit = std::getenv("CS_NO_LAZY_EXIT") == nullptr;  // read at scene creation
    bool far_pairs = std::getenv("CS_NO_FAR_PAIRS") == nullptr;  // partial CCD near / far split
    DBuf<double> vdn;  // per world vertex |candidate - anchor|
    DBuf<int> far_rest;
    DBuf<int> ktile;  // per-tile kept stamp-entry counts -> offsets (k_kept_tiles)
    long long live_known = -1;  // pairs with a nonzero life span after the last partial CCD (-1: unknown)
    DBuf<int> ftile;  // per-tile engaged-flag counts -> offsets (k_flag_tiles)  // far pairs the displacement bound does not settle (k_far_gate)
    bool rows_from_delta = false;  // rows_act must be rebuilt from delta after the rhs
    bool plan_enabled = std::getenv("CS_NO_STAMP_PLAN") == nullptr;  // read at scene creation
    DBuf<unsigned long long> pkey, pkey2, nkey, nkey_s, skey_sd, skey_sd2;
    DBuf<int> psrc2, nsrc, nsrc_s, newsel, pdst, pair_u, ssrc_sd, ssrc_sd2, sseg_beg, sseg_end;
    DBuf<double4> stamp_p, stamp_sd;  // stamps in plan order (main / side list)
    bool stamps_plan_order = false;   // the current rhs streams stamp_p instead of gathering stamp
    DBuf<uint8_t> rowpos;

    // ------------------------------------------------------------ utilities
    cudaEvent_t ev() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    void stage(int k) {  // switch the timed stage (-1 = none)
        if (active_stage == k) return;
        cudaEvent_t e = ev();
        cudaEventRecord(e, s);
        if (active_stage >= 0) spans.push_back({active_stage, {stage_start, e}});
        active_stage = k;
        stage_start = e;
    }
    int n_syncs = 0;  // host<->device synchronisations in the current cs_step
    cudaError_t hsync(int line = 0) {
        ++n_syncs;
        static const bool trace_sync = std::getenv("CS_TRACE_SYNC") != nullptr;
        if (trace_sync) std::fprintf(stderr, "[cs sync] abi.cu:%d\n", line);
        return cudaStreamSynchronize(s);
    }
    int sync_scalars(int line = 0) {
        // doubles [0, S_COUNT) and ints [0, I_COUNT) in one copy (the 4-double scratch
        // between them rides along; its host copy is only read right after its own
        // sync), plus the smoother's pending residual norms
        CS_TRY(cudaMemcpyAsync(h_scal, d_scal.p, (S_COUNT + 4) * sizeof(double) + I_COUNT * sizeof(int),
                               cudaMemcpyDeviceToHost, s));
        const int nchk = pending_checks >= 2 ? std::min(pending_checks, kMaxNormChecks) : 0;
        if (nchk) CS_TRY(cudaMemcpyAsync(h_norms, norms.p, sizeof(double) * nchk, cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(line));
        return check_divergence(nchk);
    }
    int grid(long long m, int bs = 256) { return (int)std::max<long long>(1, (m + bs - 1) / bs); }

    Sell sell() { return Sell{nf, nslices, sell_ptr.p, sell_col.p, sell_val.p}; }
    EdgeSet edges() { return EdgeSet{e0.p, e1.p, erest.p, ew.p}; }

    // ------------------------------------------------------------ reductions
    // slot = sqrt(sum (a[ids] - b)^2) over n rows (b may be null)
    int sqnorm(const double* a, const double* bb, int rows, const int* ids, int slot) {
        int g = std::min(grid(rows), 2 * sm_count);
        CS_RET(part.ensure(g));
        k_sqdiff_partial<<<g, 256, 0, s>>>(a, bb, rows, ids, part.p);
        k_norm_final<<<1, 256, 0, s>>>(part.p, g, d_scal.p + slot);
        launches += 2;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // ------------------------------------------------------------ solver stages
    // b, delta for cloth positions xcl (n,3) (pinned rows carry the pin targets)
    int assemble_rhs(const double* zc, const double* xcl, bool with_stamps) {
        const int* sb = with_stamps ? seg_beg.p : nullptr;
        k_assemble_rhs<<<grid(nf), 256, 0, s>>>(nf, free_ids.p, xcl, zc, mh2.p, edges(), rinc_ptr.p, rinc.p,
                                                has_fp ? hfp_ptr.p : nullptr, hfp_col.p, hfp_val.p, xcl, sb,
                                                seg_end.p, stamps_plan_order ? nullptr : ssrc_s.p,
                                                stamps_plan_order ? stamp_p.p : stamp.p, b.p, delta.p,
                                                with_stamps && stamps_plan_order && side_M > 0
                                                    ? StampSide{sseg_beg.p, sseg_end.p, skey_sd.p, stamp_sd.p, pkey.p}
                                                    : StampSide{});
        ++launches;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // rank-2 A-Jacobi on x (nf,3) in place (smoothing.py:23-66).  The residual
    // norms at k = 0, 10, 20, ... are kept on device and compared at the next
    // host sync (check_divergence): a diverging step is discarded either way.
    // The 2 x 16 SpMV passes (+ norm checks) of one smoothing call are captured once
    // per distinct argument set into a CUDA graph and replayed: back-to-back
    // dependent launches without per-launch host overhead or launch gaps.
    struct SmoothGraph {
        const double* bb;
        const double* xx;
        const double* dl;
        const double* part;
        const double* norms;
        int steps;
        double c;
        cudaGraphExec_t exec;
    };
    std::vector<SmoothGraph> smooth_graphs;
    cudaStream_t cap_stream = nullptr;
    // asynchronous frame snapshots (cs_frame_async): two device slots, a copy stream
    struct FrameSlot {
        DBuf<double> x;
        cudaEvent_t taken = nullptr, done = nullptr;
        bool used = false;
    };
    FrameSlot frame_slots[2];
    int frame_next = 0;
    cudaStream_t copy_stream = nullptr;

    void smooth_launch(cudaStream_t st, const double* bb, double* xx, int steps, double c, const double* dl) {
        const int g2 = grid(nf, 128);
        for (int k = 0; k < steps; ++k) {
            const bool chk = (k % 10) == 0;
            k_jacobi_a<<<g2, 128, 0, st>>>(sell(), diag.p, dl, bb, xx, t.p, chk ? spart.p : nullptr);
            if (chk) k_norm_final<<<1, 256, 0, st>>>(spart.p, g2, norms.p + k / 10);
            k_jacobi_b<<<g2, 128, 0, st>>>(sell(), diag.p, dl, t.p, c, xx);
        }
    }

    // Chebyshev-accelerated Jacobi (StepConfig.smoother = "chebyshev", opt-in): `iterations`
    // fused SELL passes (the same SpMV count as the A-Jacobi's rank-2 steps) over three
    // rotating x buffers; interval [max(1 - rho, 0.02), 1 + rho] from the Gershgorin
    // radius rho of D^-1 H (computed once per scene: delta >= 0 only shrinks it).
    double cheb_rho = -1.0;
    DBuf<double> cheb_b1, cheb_b2;
    void cheb_launch(cudaStream_t st, const double* bb, double* xx, int iterations, const double* dl) {
        const double lmax = 1.0 + cheb_rho, lmin = std::max(1.0 - cheb_rho, 0.02);
        const double g = 2.0 / (lmax + lmin), sg = (lmax - lmin) / (lmax + lmin);
        const int g2 = grid(nf, 128);
        double* buf[3] = {xx, cheb_b1.p, cheb_b2.p};
        double w = 1.0;
        int cur = 0, prev = 0;
        for (int k = 0; k < iterations; ++k) {
            if (k == 1) w = 1.0 / (1.0 - 0.5 * sg * sg);
            else if (k > 1) w = 1.0 / (1.0 - 0.25 * sg * sg * w);
            const int nxt = (cur + 1) % 3 == prev ? (cur + 2) % 3 : (cur + 1) % 3;
            const bool chk = (k % 20) == 0;
            k_cheb_step<<<g2, 128, 0, st>>>(sell(), diag.p, dl, bb, buf[cur], buf[prev], w, g, buf[nxt],
                                            chk ? spart.p : nullptr);
            if (chk) k_norm_final<<<1, 256, 0, st>>>(spart.p, g2, norms.p + k / 20);
            prev = cur;
            cur = nxt;
        }
        if (cur != 0) cudaMemcpyAsync(xx, buf[cur], sizeof(double) * 3 * nf, cudaMemcpyDeviceToDevice, st);
    }
    int cheb_bounds() {
        if (cheb_rho >= 0.0) return 0;
        const int g = grid(nf);
        CS_RET(part.ensure(g));
        k_gershgorin<<<g, 256, 0, s>>>(sell(), diag.p, part.p);
        CS_CHECK_LAUNCH();
        std::vector<double> hp(g);
        CS_TRY(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * g, cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        double rho = 0.0;
        for (double v : hp) rho = std::max(rho, v);
        cheb_rho = rho;
        return 0;
    }

    int smooth(const double* bb, double* xx, int iterations, double omega, const double* dl) {
        if (cfg.smoother == CS_SMOOTHER_CHEBYSHEV) return smooth_cheb(bb, xx, iterations, dl);
        const int steps = (iterations + 1) / 2;
        const double c = 1.0 - omega;
        CS_RET(spart.ensure(grid(nf, 128)));
        const int nchk = (steps + 9) / 10;
        CS_RET(norms.ensure(std::max(nchk, 1)));
        launches += 2LL * steps + nchk;
        pending_checks = nchk;
        for (auto& sg : smooth_graphs)
            if (sg.bb == bb && sg.xx == xx && sg.dl == dl && sg.part == spart.p && sg.norms == norms.p &&
                sg.steps == steps && sg.c == c) {
                CS_TRY(cudaGraphLaunch(sg.exec, s));
                return 0;
            }
        if (!cap_stream) CS_TRY(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        cudaGraph_t graph;
        CS_TRY(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
        smooth_launch(cap_stream, bb, xx, steps, c, dl);
        CS_TRY(cudaStreamEndCapture(cap_stream, &graph));
        cudaGraphExec_t exec;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        CS_TRY(e);
        if (smooth_graphs.size() >= 8) {
            cudaGraphExecDestroy(smooth_graphs.front().exec);
            smooth_graphs.erase(smooth_graphs.begin());
        }
        smooth_graphs.push_back(SmoothGraph{bb, xx, dl, spart.p, norms.p, steps, c, exec});
        CS_TRY(cudaGraphLaunch(exec, s));
        return 0;
    }

    int smooth_cheb(const double* bb, double* xx, int iterations, const double* dl) {
        CS_RET(cheb_bounds());
        CS_RET(spart.ensure(grid(nf, 128)));
        CS_RET(cheb_b1.ensure(3LL * nf));
        CS_RET(cheb_b2.ensure(3LL * nf));
        const int nchk = (iterations + 19) / 20;
        CS_RET(norms.ensure(std::max(nchk, 1)));
        launches += iterations + nchk;
        pending_checks = nchk;
        const double c = -1.0;  // graph-cache tag for the Chebyshev sequence
        for (auto& sg : smooth_graphs)
            if (sg.bb == bb && sg.xx == xx && sg.dl == dl && sg.part == spart.p && sg.norms == norms.p &&
                sg.steps == iterations && sg.c == c) {
                CS_TRY(cudaGraphLaunch(sg.exec, s));
                return 0;
            }
        if (!cap_stream) CS_TRY(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        cudaGraph_t graph;
        CS_TRY(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
        cheb_launch(cap_stream, bb, xx, iterations, dl);
        CS_TRY(cudaStreamEndCapture(cap_stream, &graph));
        cudaGraphExec_t exec;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        CS_TRY(e);
        if (smooth_graphs.size() >= 8) {
            cudaGraphExecDestroy(smooth_graphs.front().exec);
            smooth_graphs.erase(smooth_graphs.begin());
        }
        smooth_graphs.push_back(SmoothGraph{bb, xx, dl, spart.p, norms.p, iterations, c, exec});
        CS_TRY(cudaGraphLaunch(exec, s));
        return 0;
    }

    // smoothing.py:57-64: raise if a checked residual norm grew 10x (norms copied to
    // h_norms by the caller's sync)
    int check_divergence(int m) {
        pending_checks = 0;
        for (int i = 1; i < m; ++i)
            if (h_norms[i] > 10.0 * h_norms[i - 1]) return CS_DIVERGENCE;
        return 0;
    }

    // one value for every scene and thread (scenes stepped concurrently from host threads
    // must not race a smaller limit against a larger launch): the largest tile any basis
    // width up to 128 columns takes
    static cudaError_t proj_smem_attr() {
        size_t mx = 0;
        for (int w = 1; w <= 128; ++w) mx = std::max(mx, proj_smem(w));
        return cudaFuncSetAttribute(k_project_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    }

    // reduced correction in the reuse basis (subspace.py:165-186); x (nf,3) in place
    int reduced(const double* bb, double* xx, const double* dl, bool refactor, int n_rows_act_known) {
        const int g = std::min(cs_div_up(nf, proj_rows(r)), 3 * sm_count);
        CS_RET(part.ensure((size_t)g * 3 * r));
        CS_TRY(proj_smem_attr());
        k_project_partial<<<g, 256, proj_smem(r), s>>>(sell(), bb, xx, dl, V.p, r, part.p);
        k_reduce_partials<<<cs_div_up(3 * r, 32), 256, 0, s>>>(part.p, g, 3 * r, rhs_red.p);
        launches += 2;
        const double* gram = nullptr;
        if (refactor && n_rows_act_known > 0) {
            // grid from nf only: the row partition (hence the rounding) depends on the device
            // row count alone, whatever bound the host holds
            const int gg = std::min(cs_div_up(nf, 64), 2 * sm_count);
            CS_RET(part2.ensure((size_t)gg * r * r));
            k_gram_partial<<<gg, kGramThreads, 0, s>>>(rows_act.p, d_iscal.p + I_ROWS, dl, V.p, r, part2.p);
            k_reduce_partials<<<cs_div_up(r * r, 32), 256, 0, s>>>(part2.p, gg, r * r, gram_red.p);
            launches += 2;
            gram = gram_red.p;
        }
        ReducedState rs{Xred.p, beta_red.p, fallback.p};
        k_reduced_solve<<<1, 256, 0, s>>>(rhs_red.p, gram, lam.p, r, 0, refactor ? 1 : 0, rs, q.p);
        k_prolong<<<cs_div_up(nf, prolong_rows(r)), 128, prolong_rows(r) * (r | 1) * sizeof(double), s>>>(
            V.p, r, q.p, nf, xx);
        launches += 2;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // warm-start correction in the wide basis (subspace.py:189-192)
    int warm_correction(const double* bb, double* xx) {
        const int g = std::min(cs_div_up(nf, proj_rows(rb)), 3 * sm_count);
        CS_RET(part.ensure((size_t)g * 3 * rb));
        CS_TRY(proj_smem_attr());
        k_project_partial<<<g, 256, proj_smem(rb), s>>>(sell(), bb, xx, nullptr, U.p, rb, part.p);
        k_reduce_partials<<<cs_div_up(3 * rb, 32), 256, 0, s>>>(part.p, g, 3 * rb, rhs_red.p);
        ReducedState rs{Xred.p, beta_red.p, fallback.p};
        k_reduced_solve<<<1, 256, 0, s>>>(rhs_red.p, nullptr, lam.p, rb, 1, 0, rs, q.p);
        k_prolong<<<cs_div_up(nf, prolong_rows(rb)), 128, prolong_rows(rb) * (rb | 1) * sizeof(double), s>>>(
            U.p, rb, q.p, nf, xx);
        launches += 4;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // ------------------------------------------------------------ collision stages
    WorldTopo world() {
        WorldTopo w;
        w.nw = nw;
        w.tris = wtris.p;
        w.edges = wedges.p;
        w.tri_static = tri_static.p;
        w.vert_static = vert_static.p;
        w.vert_used = vert_used.p;
        w.edge_static = edge_static.p;
        w.edge_tris = edge_tris.p;
        w.edge_slot = edge_slot.p;
        w.patch = patch.p;
        w.pslot = pslot.p;
        w.flip = eflip.p;
        return w;
    }

    template <typename I>
    int scan(const I* in, I* out, int m) {
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, m, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceScan::ExclusiveSum(cub_tmp.p, bytes, in, out, m, s));
        return 0;
    }

    // hash-grid table stage 1: per-primitive cell counts, scan, oversize list
    int table_count(EntryBuf& G, BoxSrc src, const double* inv) {
        k_cell_count<<<grid(G.np), 256, 0, s>>>(src, inv, G.count.p, G.is_over.p);
        ++launches;
        CS_CHECK_LAUNCH();
        CS_TRY(cudaMemsetAsync(G.count.p + G.np, 0, sizeof(int), s));
        CS_RET(scan(G.count.p, G.offset.p, G.np + 1));
        size_t bytes = 0;
        cub::CountingInputIterator<int> it(0);
        cub::DeviceSelect::Flagged(nullptr, bytes, it, G.is_over.p, G.over.p, G.n_over.p, G.np, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, G.is_over.p, G.over.p, G.n_over.p, G.np, s));
        return 0;
    }
    // stage 2 (entry count m known on host): fill, stable radix sort by bucket,
    // sorted (primitive, code) arrays, run heads (+ dense bucket ranges if dense)
    int table_build(EntryBuf& G, BoxSrc src, const double* inv, bool dense) {
        const long long m = G.m;
        CS_RET(G.run.ensure(std::max<long long>(m, 1)));
        CS_TRY(cudaMemsetAsync(G.n_run.p, 0, sizeof(int), s));
        if (dense) {
            CS_RET(G.bstart.ensure(G.T));
            CS_RET(G.bend.ensure(G.T));
            CS_TRY(cudaMemsetAsync(G.bstart.p, 0, sizeof(int) * G.T, s));
            CS_TRY(cudaMemsetAsync(G.bend.p, 0, sizeof(int) * G.T, s));
        }
        if (m == 0) return 0;
        CS_RET(G.key.ensure(m));
        CS_RET(G.key_s.ensure(m));
        CS_RET(G.prim.ensure(m));
        CS_RET(G.prim_s.ensure(m));
        CS_RET(G.perm.ensure(m));
        CS_RET(G.perm_s.ensure(m));
        CS_RET(G.code.ensure(m));
        CS_RET(G.code_s.ensure(m));
        CS_RET(G.head.ensure(m));
        CS_RET(G.zb.ensure(m));
        CS_RET(G.zb_s.ensure(m));
        k_cell_fill<<<grid(8LL * G.np), 256, 0, s>>>(src, inv, G.T - 1, G.count.p, G.offset.p, G.key.p, G.prim.p,
                                               G.code.p, G.zb.p);
        k_iota<<<grid(m), 256, 0, s>>>(G.perm.p, m);
        launches += 2;
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, G.key.p, G.key_s.p, G.perm.p, G.perm_s.p, (int)m, 0, G.log2T,
                                        s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp.p, bytes, G.key.p, G.key_s.p, G.perm.p, G.perm_s.p, (int)m, 0,
                                               G.log2T, s));
        k_entries_sorted<<<grid(m), 256, 0, s>>>(G.perm_s.p, (int)m, G.prim.p, G.code.p, G.zb.p, G.key_s.p,
                                                 G.prim_s.p, G.code_s.p, G.zb_s.p, G.head.p, dense ? G.bstart.p : nullptr,
                                                 dense ? G.bend.p : nullptr);
        ++launches;
        bytes = 0;
        cub::CountingInputIterator<int> it(0);
        cub::DeviceSelect::Flagged(nullptr, bytes, it, G.head.p, G.run.p, G.n_run.p, (int)m, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, G.head.p, G.run.p, G.n_run.p, (int)m, s));
        CS_CHECK_LAUNCH();
        return 0;
    }
    // entries of long bucket runs (LongRow) into G.lrows, count in G.n_lrows (device)
    int long_rows(EntryBuf& G, const LongRow& pred) {
        CS_RET(G.n_lrows.ensure(1));
        CS_TRY(cudaMemsetAsync(G.n_lrows.p, 0, sizeof(int), s));
        if (!G.m) return 0;
        CS_RET(G.lrows.ensure(G.m));
        cub::CountingInputIterator<int> it(0);
        size_t bytes = 0;
        cub::DeviceSelect::If(nullptr, bytes, it, G.lrows.p, G.n_lrows.p, (int)G.m, pred, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::If(cub_tmp.p, bytes, it, G.lrows.p, G.n_lrows.p, (int)G.m, pred, s));
        ++launches;
        return 0;
    }

    int run_blocks(long long m) {
        return (int)std::max<long long>(1, std::min<long long>((m + kPairWarps - 1) / kPairWarps, 32LL * sm_count));
    }

    // broad phase into pr (bvh.py:207-292): entry tables -> bucket-pair count -> scan -> write; two host syncs
    int broad_phase(const double* xa, const double* xb, double margin, PairBuf& pr) {
        base_valid = false;  // the grid tables are rebuilt below
        k_vertex_boxes<<<grid(3LL * nw), 256, 0, s>>>(xa, xb, nw, margin, vlo.p, vhi.p, fvbox.p);
        k_vertex_disp<<<grid(nw), 256, 0, s>>>(xa, xb, nw, vdisp.p, fvbox.p);
        bmargin = margin;
        const int gt = grid(ntw), ge = grid(new_);
        CS_RET(ttab.part.ensure(4LL * gt));
        CS_RET(etab.part.ensure(4LL * ge));
        k_prim_boxes<3><<<gt, 256, 0, s>>>(wtris.p, ntw, tri_static.p, vlo.p, vhi.p, vdisp.p, ttab.box.p, tdisp.p,
                                           ttab.part.p, ftbox.p);
        static const double cell_scale = std::getenv("CS_CELL_SCALE") ? std::atof(std::getenv("CS_CELL_SCALE")) : 1.0;
        k_cell_size<<<1, 256, 0, s>>>(ttab.part.p, gt, ttab.inv.p, cell_scale);
        k_prim_boxes<2><<<ge, 256, 0, s>>>(wedges.p, new_, edge_static.p, vlo.p, vhi.p, vdisp.p, etab.box.p, edisp.p,
                                           etab.part.p, febox.p);
        k_cell_size<<<1, 256, 0, s>>>(etab.part.p, ge, etab.inv.p, cell_scale);
        k_prim_motion<3><<<gt, 256, 0, s>>>(wtris.p, ntw, xa, xb, ftbox.p);
        k_prim_motion<2><<<ge, 256, 0, s>>>(wedges.p, new_, xa, xb, febox.p);
        launches += 8;
        const BoxSrc vs{nullptr, vlo.p, vhi.p, vert_used.p, nw};
        const BoxSrc ts{ttab.box.p, nullptr, nullptr, nullptr, ntw};
        const BoxSrc es{etab.box.p, nullptr, nullptr, nullptr, new_};
        CS_RET(table_count(vtab, vs, ttab.inv.p));
        CS_RET(table_count(ttab, ts, ttab.inv.p));
        CS_RET(table_count(etab, es, etab.inv.p));
        EntryBuf* tabs[3] = {&vtab, &ttab, &etab};
        for (int k = 0; k < 3; ++k) {
            CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + k], tabs[k]->offset.p + tabs[k]->np, sizeof(int), cudaMemcpyDeviceToHost, s));
            CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 4 + k], tabs[k]->n_over.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        }
        CS_TRY(hsync(__LINE__));
        for (int k = 0; k < 3; ++k) {
            tabs[k]->m = h_iscal[I_COUNT + k];
            tabs[k]->n_over_h = h_iscal[I_COUNT + 4 + k];
        }
        vtab.set_buckets(std::max(vtab.m, ttab.m));
        ttab.T = vtab.T;
        ttab.log2T = vtab.log2T;
        etab.set_buckets(etab.m);
        // dense bucket ranges: the triangle table for k_pairs_vt, all three for
        // k_subset_query's cell walks
        CS_RET(table_build(vtab, vs, ttab.inv.p, true));
        CS_RET(table_build(ttab, ts, ttab.inv.p, true));
        CS_RET(table_build(etab, es, etab.inv.p, true));
        // ballot buffers: warp iterations per run, scanned (one more host sync)
        const EntryTable VT = vtab.view(), TT = ttab.view(), ET = etab.view();
        for (EntryBuf* G : {&vtab, &etab}) {
            CS_RET(G->iters.ensure(G->m + 1));
            CS_RET(G->iter_off.ensure(G->m + 1));
            CS_TRY(cudaMemsetAsync(G->iters.p, 0, sizeof(long long) * (G->m + 1), s));
        }
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_COUNT + 4, 0, 2 * sizeof(int), s));
        if (vtab.m) k_run_iters<<<grid(vtab.m), 256, 0, s>>>(VT, TT, 1, vtab.iters.p, d_iscal.p + I_COUNT + 4);
        if (etab.m) k_run_iters<<<grid(etab.m), 256, 0, s>>>(ET, ET, 0, etab.iters.p, d_iscal.p + I_COUNT + 5);
        launches += 2;
        CS_RET(scan(vtab.iters.p, vtab.iter_off.p, (int)vtab.m + 1));
        CS_RET(scan(etab.iters.p, etab.iter_off.p, (int)etab.m + 1));
        long long* hits_h = reinterpret_cast<long long*>(h_scal + S_COUNT);
        CS_TRY(cudaMemcpyAsync(&hits_h[0], vtab.iter_off.p + vtab.m, sizeof(long long), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&hits_h[1], etab.iter_off.p + etab.m, sizeof(long long), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 4], d_iscal.p + I_COUNT + 4, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                               s));
        CS_TRY(hsync(__LINE__));
        // rows of runs too long for one warp (dense piles): one thread each; only when
        // such runs exist (one more synchronisation for their count)
        const bool long_vt = vtab.m && h_iscal[I_COUNT + 4], long_ee = etab.m && h_iscal[I_COUNT + 5];
        vtab.n_lrows_h = etab.n_lrows_h = 0;
        if (long_vt || long_ee) {
            if (long_vt) CS_RET(long_rows(vtab, LongRow{VT.key, VT.bstart, VT.bend, TT.bstart, TT.bend}));
            if (long_ee) CS_RET(long_rows(etab, LongRow{ET.key, ET.bstart, ET.bend, nullptr, nullptr}));
            if (long_vt)
                CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 4], vtab.n_lrows.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            if (long_ee)
                CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 5], etab.n_lrows.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            CS_TRY(hsync(__LINE__));
            vtab.n_lrows_h = long_vt ? h_iscal[I_COUNT + 4] : 0;
            etab.n_lrows_h = long_ee ? h_iscal[I_COUNT + 5] : 0;
        }
        CS_RET(vtab.masks.ensure(std::max<long long>(hits_h[0], 1)));
        CS_RET(etab.masks.ensure(std::max<long long>(hits_h[1], 1)));
        // pair counts: [VT runs][VT oversize][EE runs][EE oversize]
        const int n_ovt = vtab.n_over_h + ttab.n_over_h, n_oee = etab.n_over_h;
        for (EntryBuf* G : {&vtab, &etab}) {
            CS_RET(G->pcount.ensure(G->m + 1));
            CS_RET(G->poffset.ensure(G->m + 1));
            CS_TRY(cudaMemsetAsync(G->pcount.p, 0, sizeof(int) * (G->m + 1), s));
        }
        CS_RET(ocount.ensure(n_ovt + n_oee + 2));
        CS_RET(ooffset.ensure(n_ovt + n_oee + 2));
        CS_TRY(cudaMemsetAsync(ocount.p, 0, sizeof(int) * (n_ovt + n_oee + 2), s));
        int* oc_vt = ocount.p;
        int* oc_ee = ocount.p + n_ovt + 1;
        int* oo_vt = ooffset.p;
        int* oo_ee = ooffset.p + n_ovt + 1;
        const WorldTopo W = world();
        PairOut O{};
        if (vtab.m) {
            O.counts = vtab.pcount.p;
            k_pairs_vt<0><<<run_blocks(vtab.m), 32 * kPairWarps, 0, s>>>(VT, TT, vlo.p, vhi.p, ttab.box.p, ttab.inv.p, W,
                                                                       vtab.iter_off.p, vtab.masks.p, O);
            ++launches;
        }
        if (n_ovt) {
            O.counts = oc_vt;
            k_over_vt<0><<<grid(n_ovt, 64), 64, 0, s>>>(vtab.over.p, vtab.n_over_h, ttab.over.p, ttab.n_over_h,
                                                         vtab.is_over.p, vlo.p, vhi.p, ttab.box.p, ntw, W, O);
            ++launches;
        }
        if (etab.m) {
            O.counts = etab.pcount.p;
            k_pairs_ee<0><<<run_blocks(etab.m), 32 * kPairWarps, 0, s>>>(ET, etab.box.p, etab.inv.p, W,
                                                                       etab.iter_off.p, etab.masks.p, O);
            ++launches;
        }
        if (n_oee) {
            O.counts = oc_ee;
            k_over_ee<0><<<grid(n_oee, 64), 64, 0, s>>>(etab.over.p, n_oee, etab.is_over.p, etab.box.p, new_, W, O);
            ++launches;
        }
        for (EntryBuf* G : {&vtab, &etab}) {
            CS_RET(G->lcount.ensure(G->n_lrows_h + 1));
            CS_RET(G->loff.ensure(G->n_lrows_h + 1));
            CS_TRY(cudaMemsetAsync(G->lcount.p, 0, sizeof(int) * (G->n_lrows_h + 1), s));
        }
        if (vtab.n_lrows_h) {
            O.counts = vtab.lcount.p;
            k_long_vt<0><<<grid(vtab.n_lrows_h, 128), 128, 0, s>>>(VT, TT, vlo.p, vhi.p, ttab.box.p, ttab.inv.p, W,
                                                                   vtab.lrows.p, vtab.n_lrows.p, O);
            ++launches;
        }
        if (etab.n_lrows_h) {
            O.counts = etab.lcount.p;
            k_long_ee<0><<<grid(etab.n_lrows_h, 128), 128, 0, s>>>(ET, etab.box.p, etab.inv.p, W, etab.lrows.p,
                                                                   etab.n_lrows.p, O);
            ++launches;
        }
        CS_CHECK_LAUNCH();
        CS_RET(scan(vtab.pcount.p, vtab.poffset.p, (int)vtab.m + 1));
        CS_RET(scan(oc_vt, oo_vt, n_ovt + 1));
        CS_RET(scan(etab.pcount.p, etab.poffset.p, (int)etab.m + 1));
        CS_RET(scan(oc_ee, oo_ee, n_oee + 1));
        CS_RET(scan(vtab.lcount.p, vtab.loff.p, (int)vtab.n_lrows_h + 1));
        CS_RET(scan(etab.lcount.p, etab.loff.p, (int)etab.n_lrows_h + 1));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 0], vtab.poffset.p + vtab.m, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 1], oo_vt + n_ovt, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 2], etab.poffset.p + etab.m, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 3], oo_ee + n_oee, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 4], vtab.loff.p + vtab.n_lrows_h, sizeof(int), cudaMemcpyDeviceToHost,
                               s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 5], etab.loff.p + etab.n_lrows_h, sizeof(int), cudaMemcpyDeviceToHost,
                               s));
        CS_TRY(hsync(__LINE__));
        // rows: [VT runs c0][VT long runs c4][VT oversize c1][EE runs c2][EE long runs c5][EE oversize c3]
        const long long c0 = h_iscal[I_COUNT + 0], c1 = h_iscal[I_COUNT + 1], c2 = h_iscal[I_COUNT + 2], c3 = h_iscal[I_COUNT + 3];
        const long long c4 = h_iscal[I_COUNT + 4], c5 = h_iscal[I_COUNT + 5];
        const long long P = c0 + c1 + c2 + c3 + c4 + c5;
        CS_RET(pr.reserve(std::max<long long>(P, 1)));
        auto out_at = [&](long long base, const int* offs) {
            return PairOut{nullptr, offs, pr.kind.p + base, pr.idx.p + base, pr.keys.p + base};
        };
        if (vtab.m && c0)
            k_pairs_vt<1><<<run_blocks(vtab.m), 32 * kPairWarps, 0, s>>>(VT, TT, vlo.p, vhi.p, ttab.box.p, ttab.inv.p, W,
                                                                       vtab.iter_off.p, vtab.masks.p,
                                                                       out_at(0, vtab.poffset.p));
        if (vtab.n_lrows_h && c4)
            k_long_vt<1><<<grid(vtab.n_lrows_h, 128), 128, 0, s>>>(VT, TT, vlo.p, vhi.p, ttab.box.p, ttab.inv.p, W,
                                                                   vtab.lrows.p, vtab.n_lrows.p,
                                                                   out_at(c0, vtab.loff.p));
        if (n_ovt && c1)
            k_over_vt<1><<<grid(n_ovt, 64), 64, 0, s>>>(vtab.over.p, vtab.n_over_h, ttab.over.p, ttab.n_over_h,
                                                         vtab.is_over.p, vlo.p, vhi.p, ttab.box.p, ntw, W,
                                                         out_at(c0 + c4, oo_vt));
        const long long e0 = c0 + c4 + c1;  // first EE row
        if (etab.m && c2)
            k_pairs_ee<1><<<run_blocks(etab.m), 32 * kPairWarps, 0, s>>>(ET, etab.box.p, etab.inv.p, W,
                                                                       etab.iter_off.p, etab.masks.p,
                                                                       out_at(e0, etab.poffset.p));
        if (etab.n_lrows_h && c5)
            k_long_ee<1><<<grid(etab.n_lrows_h, 128), 128, 0, s>>>(ET, etab.box.p, etab.inv.p, W, etab.lrows.p,
                                                                   etab.n_lrows.p, out_at(e0 + c2, etab.loff.p));
        if (n_oee && c3)
            k_over_ee<1><<<grid(n_oee, 64), 64, 0, s>>>(etab.over.p, n_oee, etab.is_over.p, etab.box.p, new_, W,
                                                        out_at(e0 + c2 + c5, oo_ee));
        launches += 6;
        if (c2 + c5 + c3) {
            k_ee_orient<<<grid(c2 + c5 + c3), 256, 0, s>>>(pr.keys.p + e0, pr.idx.p + e0, c2 + c5 + c3, W);
            ++launches;
        }
        CS_CHECK_LAUNCH();
        pr.P = P;
        return 0;
    }

    // fused keep + stable compaction, phase 1: tile bitmasks + counts + scan; the
    // kept total lands in h_iscal[slot] after the caller's next sync
    int keep_tiles(const PairBuf& src, const uint8_t* vv, const uint8_t* tv, const uint8_t* ev, int slot) {
        const long long P0 = src.P;
        const long long nt = (P0 + kKeepTile - 1) / kKeepTile;
        CS_RET(keep_bits.ensure(std::max<long long>(nt * (kKeepTile / 32), 1)));
        CS_RET(tile_cnt.ensure(nt + 1));
        CS_RET(tile_off.ensure(nt + 1));
        CS_TRY(cudaMemsetAsync(tile_cnt.p + nt, 0, sizeof(int), s));
        if (nt) {
            const KeepArgs A{src.keys.p, P0, vlo.p, vhi.p, ttab.box.p, etab.box.p, vv, tv, ev};
            k_keep_tiles<<<(int)nt, 256, 0, s>>>(A, keep_bits.p, tile_cnt.p);
            ++launches;
        }
        CS_RET(scan(tile_cnt.p, tile_off.p, (int)nt + 1));
        CS_TRY(cudaMemcpyAsync(&h_iscal[slot], tile_off.p + nt, sizeof(int), cudaMemcpyDeviceToHost, s));
        return 0;
    }
    // phase 2: the kept rows of src into dst[0, kept) in order
    int compact_tiles(const PairBuf& src, PairBuf& dst) {
        const long long nt = (src.P + kKeepTile - 1) / kKeepTile;
        if (nt) {
            k_compact_tiles<<<(int)nt, 256, 0, s>>>(keep_bits.p, tile_off.p, src.P, src.kind.p, src.idx.p,
                                                    src.keys.p, dst.kind.p, dst.idx.p, dst.keys.p);
            ++launches;
        }
        return 0;
    }

    // broad -> full CCD -> distance march -> clamp factor (stepper.py:426-452)
    // Motion-free site (xa == xb) right after a site whose pairs are in `prev`: when
    // the static boxes stay inside that site's boxes, the candidate set is the
    // subset of `prev` that still overlaps (order preserved).  ok = false -> caller
    // runs the full broad phase.  Two small host syncs instead of three.
    int broad_phase_static(const double* x, double margin, PairBuf& prev, PairBuf& pr, bool& ok) {
        ok = false;
        if (margin != bmargin || prev.P == 0) return 0;
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_FLAG, 0, sizeof(int), s));
        k_box_contained<<<grid(3LL * nw), 256, 0, s>>>(x, 3 * nw, margin, vlo.p, vhi.p, d_iscal.p + I_FLAG);
        ++launches;
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_FLAG], d_iscal.p + I_FLAG, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        if (h_iscal[I_FLAG]) return 0;
        // boxes of this site (static), then the surviving subset of prev
        k_vertex_boxes<<<grid(3LL * nw), 256, 0, s>>>(x, x, nw, margin, vlo.p, vhi.p, fvbox.p);
        k_vertex_disp<<<grid(nw), 256, 0, s>>>(x, x, nw, vdisp.p, fvbox.p);
        const int gt = grid(ntw), ge = grid(new_);
        k_prim_boxes<3><<<gt, 256, 0, s>>>(wtris.p, ntw, tri_static.p, vlo.p, vhi.p, vdisp.p, ttab.box.p, tdisp.p,
                                           ttab.part.p, ftbox.p);
        k_prim_boxes<2><<<ge, 256, 0, s>>>(wedges.p, new_, edge_static.p, vlo.p, vhi.p, vdisp.p, etab.box.p, edisp.p,
                                           etab.part.p, febox.p);
        k_prim_motion<3><<<gt, 256, 0, s>>>(wtris.p, ntw, x, x, ftbox.p);
        k_prim_motion<2><<<ge, 256, 0, s>>>(wedges.p, new_, x, x, febox.p);
        launches += 4;
        CS_RET(keep_tiles(prev, nullptr, nullptr, nullptr, I_FLAG));
        CS_TRY(hsync(__LINE__));
        const long long P = h_iscal[I_FLAG];
        CS_RET(pr.reserve(std::max<long long>(P, 1)));
        if (P) CS_RET(compact_tiles(prev, pr));
        CS_CHECK_LAUNCH();
        pr.P = P;
        ok = true;
        return 0;
    }

    // Base site: the step's first moving site runs the full broad phase with its
    // margin widened by a small slack into basepr and keeps its vertex boxes; the
    // grid tables stay valid until the next full broad phase.
    int build_base(const double* xa, const double* xb, double margin) {
        const char* env = std::getenv("CS_SITE_SLACK");
        const double slack = env ? std::atof(env) : 0.01;
        CS_RET(broad_phase(xa, xb, margin + slack * margin, basepr));
        CS_RET(blo.ensure(3LL * nw));
        CS_RET(bhi.ensure(3LL * nw));
        CS_TRY(cudaMemcpyAsync(blo.p, vlo.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
        CS_TRY(cudaMemcpyAsync(bhi.p, vhi.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
        base_valid = true;
        base_margin = margin;
        return 0;
    }

    // Subset site: a moving site whose candidate set is taken from the base site.
    // Pairs are "boxes overlap" (bvh.py:207-292), and every box is the union of its
    // vertices' boxes, so for primitives whose vertex boxes all lie inside their base
    // boxes ("non-violators") the pairs are the base pairs that still overlap.  Pairs
    // with a violator (a vertex box poking out, or left out of the base grid) are
    // found by k_subset_query: base-grid cell walks for non-violating partners, brute
    // force among violators.  Exactly the full broad phase's set
    // (CS_VERIFY_STATIC_SITE checks it); ok = false when violators are too many.
    int subset_site(const double* xa, const double* xb, double margin, PairBuf& pr, bool& ok) {
        ok = false;
        if (!base_valid || margin != base_margin) return 0;
        // boxes and filter records of this site
        k_vertex_boxes<<<grid(3LL * nw), 256, 0, s>>>(xa, xb, nw, margin, vlo.p, vhi.p, fvbox.p);
        k_vertex_disp<<<grid(nw), 256, 0, s>>>(xa, xb, nw, vdisp.p, fvbox.p);
        const int gt = grid(ntw), ge = grid(new_);
        k_prim_boxes<3><<<gt, 256, 0, s>>>(wtris.p, ntw, tri_static.p, vlo.p, vhi.p, vdisp.p, ttab.box.p, tdisp.p,
                                           ttab.part.p, ftbox.p);
        k_prim_boxes<2><<<ge, 256, 0, s>>>(wedges.p, new_, edge_static.p, vlo.p, vhi.p, vdisp.p, etab.box.p, edisp.p,
                                           etab.part.p, febox.p);
        k_prim_motion<3><<<gt, 256, 0, s>>>(wtris.p, ntw, xa, xb, ftbox.p);
        k_prim_motion<2><<<ge, 256, 0, s>>>(wedges.p, new_, xa, xb, febox.p);
        bmargin = margin;
        // violators
        CS_RET(vviol.ensure(nw));
        CS_RET(tviol.ensure(std::max(ntw, 1)));
        CS_RET(eviol.ensure(std::max(new_, 1)));
        CS_RET(vlist.ensure(nw));
        CS_RET(tlist.ensure(std::max(ntw, 1)));
        CS_RET(elist.ensure(std::max(new_, 1)));
        k_viol_vertices<<<grid(nw), 256, 0, s>>>(vlo.p, vhi.p, blo.p, bhi.p, nw, vert_used.p, vtab.is_over.p,
                                                vviol.p);
        k_viol_prims<3><<<gt, 256, 0, s>>>(wtris.p, ntw, vviol.p, ttab.is_over.p, tviol.p);
        k_viol_prims<2><<<ge, 256, 0, s>>>(wedges.p, new_, vviol.p, etab.is_over.p, eviol.p);
        launches += 9;
        cub::CountingInputIterator<int> it(0);
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, it, vviol.p, vlist.p, d_iscal.p + I_COUNT, nw, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, vviol.p, vlist.p, d_iscal.p + I_COUNT, nw, s));
        bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, it, tviol.p, tlist.p, d_iscal.p + I_COUNT + 1, ntw, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, tviol.p, tlist.p, d_iscal.p + I_COUNT + 1, ntw, s));
        bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, it, eviol.p, elist.p, d_iscal.p + I_COUNT + 2, new_, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, eviol.p, elist.p, d_iscal.p + I_COUNT + 2, new_, s));
        // violator counts decide first (nothing else is queued yet, so a refusal wastes
        // only the box and violator passes)
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT], d_iscal.p + I_COUNT, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        const int nv = h_iscal[I_COUNT], nt = h_iscal[I_COUNT + 1], ne = h_iscal[I_COUNT + 2];
        const long long nq = (long long)nv + nt + ne;
        // violator x violator tests: one warp walks a whole violator list, so the
        // longest list sets the kernel's latency chain, and the total is quadratic;
        // past these the full broad phase is cheaper
        if (std::max(nt, ne) > 16384 || (double)nv * nt + 0.5 * (double)ne * ne > 1e8) return 0;
        // surviving base pairs among non-violators (count lands with the query totals)
        const long long P0 = basepr.P;
        CS_RET(keep_tiles(basepr, vviol.p, tviol.p, eviol.p, I_COUNT + 3));
        // violator partners: count, scan, write
        CS_RET(qcount.ensure(nq + 1));
        CS_RET(qoff.ensure(nq + 1));
        CS_TRY(cudaMemsetAsync(qcount.p, 0, sizeof(int) * (nq + 1), s));
        const QueryArgs A{vlist.p, tlist.p, elist.p, nv, nt, ne, vviol.p, tviol.p, eviol.p, vlo.p, vhi.p,
                          ttab.box.p, etab.box.p, vtab.view(), ttab.view(), etab.view(), ttab.inv.p, etab.inv.p,
                          (unsigned)(vtab.T - 1), (unsigned)(etab.T - 1), ntw, new_, nullptr};
        static const bool trace_sites = std::getenv("CS_TRACE_SITES") != nullptr;
        QueryArgs Aq = A;
        if (trace_sites) {
            CS_RET(query_dbg.ensure(4));
            CS_TRY(cudaMemsetAsync(query_dbg.p, 0, 4 * sizeof(unsigned long long), s));
            Aq.big = query_dbg.p;
        }
        const WorldTopo W = world();
        const int gq = (int)std::max<long long>(1, (32 * nq + 127) / 128);
        if (nq) {
            k_subset_query<0><<<gq, 128, 0, s>>>(Aq, W, qcount.p, nullptr, PairOut{});
            ++launches;
        }
        CS_RET(scan(qcount.p, qoff.p, (int)nq + 1));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT], qoff.p + nq, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 1], qoff.p + nv + nt, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        const long long Q = h_iscal[I_COUNT], Qvt = h_iscal[I_COUNT + 1];
        const long long Pa = h_iscal[I_COUNT + 3];
        if (trace_sites) {
            unsigned long long bg[4];
            CS_TRY(cudaMemcpy(bg, query_dbg.p, sizeof(bg), cudaMemcpyDeviceToHost));
            std::fprintf(stderr,
                         "[cs subset] base pairs %lld kept %lld violators v %d t %d e %d query pairs %lld "
                         "big v %llu t %llu e %llu max cells %llu\n",
                         P0, Pa, nv, nt, ne, Q, bg[0], bg[1], bg[2], bg[3]);
        }
        CS_RET(pr.reserve(std::max<long long>(Pa + Q, 1)));
        if (Pa) CS_RET(compact_tiles(basepr, pr));
        if (Q) {
            k_subset_query<1><<<gq, 128, 0, s>>>(A, W, nullptr, qoff.p,
                                                PairOut{nullptr, nullptr, pr.kind.p + Pa, pr.idx.p + Pa,
                                                        pr.keys.p + Pa});
            ++launches;
            if (Q > Qvt) {
                k_ee_orient<<<grid(Q - Qvt), 256, 0, s>>>(pr.keys.p + Pa + Qvt, pr.idx.p + Pa + Qvt, Q - Qvt, W);
                ++launches;
            }
        }
        CS_CHECK_LAUNCH();
        pr.P = Pa + Q;
        ok = true;
        return 0;
    }

    // test hook (CS_VERIFY_STATIC_SITE): the subset path must give exactly the full
    // broad phase's key set; returns CS_INTERNAL on any difference
    int verify_static_site(const double* x, PairBuf& got) { return verify_site(x, x, got); }
    // The reference broad phase runs on a private set of grid tables, so the step's
    // base site (its tables, cell sizes and base_valid) survives the check and later
    // outer-loop sites of the same step still take -- and get checked on -- the
    // subset path.  The site boxes it recomputes are the same values (same xa, xb,
    // margin) the subset path just wrote.
    EntryBuf vtab_v, ttab_v, etab_v;
    int verify_site(const double* xa, const double* xb, PairBuf& got) {
        PairBuf full;
        if (vtab_v.np == 0) {
            CS_RET(vtab_v.create(nw, false));
            CS_RET(ttab_v.create(ntw, true));
            CS_RET(etab_v.create(new_, true));
        }
        const bool keep_valid = base_valid;
        std::swap(vtab, vtab_v);
        std::swap(ttab, ttab_v);
        std::swap(etab, etab_v);
        int brc = broad_phase(xa, xb, cfg.d_hat, full);
        std::swap(vtab, vtab_v);
        std::swap(ttab, ttab_v);
        std::swap(etab, etab_v);
        base_valid = keep_valid;
        CS_RET(brc);
        int rc = 0;
        if (full.P != got.P) {
            rc = CS_INTERNAL;
        } else if (full.P > 0) {
            DBuf<unsigned long long> a, b;
            CS_RET(a.ensure(full.P));
            CS_RET(b.ensure(full.P));
            size_t bytes = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, bytes, full.keys.p, a.p, (int)full.P, 0, 64, s);
            CS_RET(cub_tmp.ensure(bytes));
            CS_TRY(cub::DeviceRadixSort::SortKeys(cub_tmp.p, bytes, full.keys.p, a.p, (int)full.P, 0, 64, s));
            CS_TRY(cub::DeviceRadixSort::SortKeys(cub_tmp.p, bytes, got.keys.p, b.p, (int)full.P, 0, 64, s));
            std::vector<unsigned long long> ha(full.P), hb(full.P);
            CS_TRY(cudaMemcpyAsync(ha.data(), a.p, sizeof(unsigned long long) * full.P, cudaMemcpyDeviceToHost, s));
            CS_TRY(cudaMemcpyAsync(hb.data(), b.p, sizeof(unsigned long long) * full.P, cudaMemcpyDeviceToHost, s));
            CS_TRY(hsync(__LINE__));
            if (ha != hb) rc = CS_INTERNAL;
            a.release();
            b.release();
        }
        full.release();
        return rc;
    }

    // ---------------------------------------------------------- intersection check
    // all intersecting non-adjacent world-triangle pairs at positions xw (device)
    // (reference oracles.py:83-131); pairs: first `cap` as (lo, hi) rows, unsorted
    DBuf<int> isect_out;
    bool verify_on = false;
    long long last_isect = 0;
    std::vector<int> last_isect_pairs;

    int intersections(const double* xw, long long& count, int cap) {
        k_vertex_boxes<<<grid(3LL * nw), 256, 0, s>>>(xw, xw, nw, 0.0, vlo.p, vhi.p);
        const int gt = grid(ntw);
        CS_RET(ttab.part.ensure(4LL * gt));
        k_prim_boxes<3><<<gt, 256, 0, s>>>(wtris.p, ntw, tri_static.p, vlo.p, vhi.p, vdisp.p, ttab.box.p, tdisp.p,
                                           ttab.part.p);
        k_cell_size<<<1, 256, 0, s>>>(ttab.part.p, gt, ttab.inv.p);
        launches += 3;
        bmargin = -1.0;  // the site boxes are gone: no motion-free site may reuse them
        base_valid = false;
        const BoxSrc ts{ttab.box.p, nullptr, nullptr, nullptr, ntw};
        CS_RET(table_count(ttab, ts, ttab.inv.p));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT], ttab.offset.p + ttab.np, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 1], ttab.n_over.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        ttab.m = h_iscal[I_COUNT];
        ttab.n_over_h = h_iscal[I_COUNT + 1];
        ttab.set_buckets(ttab.m);
        CS_RET(table_build(ttab, ts, ttab.inv.p, false));
        CS_RET(isect_out.ensure(2LL * std::max(cap, 1)));
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_FLAG, 0, sizeof(int), s));
        if (ttab.m)
            k_tri_intersect<<<run_blocks(ttab.m), 128, 0, s>>>(ttab.view(), ttab.box.p, wtris.p, xw,
                                                               d_iscal.p + I_FLAG, isect_out.p, cap);
        if (ttab.n_over_h)
            k_tri_intersect_over<<<grid(ttab.n_over_h, 64), 64, 0, s>>>(ttab.over.p, ttab.n_over_h, ttab.is_over.p,
                                                                         ttab.box.p, ntw, wtris.p, xw,
                                                                         d_iscal.p + I_FLAG, isect_out.p, cap);
        launches += 2;
        CS_CHECK_LAUNCH();
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_FLAG], d_iscal.p + I_FLAG, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        count = h_iscal[I_FLAG];
        return 0;
    }

    // base: 0 full broad phase; 1 subset of the current base site if there is one
    // (else / on refusal the full broad phase); 2 this site becomes the base (first
    // moving site of a step)
    // defer: the clamp stays on the device (d_scal: S_CLAMP_MIN / S_CLAMP / S_CLAMP_BAD, as
    // k_clamp_from_min writes them) and is read at the caller's next synchronisation
    // (clamp is then NaN here); the lerp kernel takes t >= 1 as "no clamp" exactly
    int ccd_site(const double* xa, const double* xb, PairBuf& pr, cs_step_report* rep, double& clamp,
                 PairBuf* prev_site = nullptr, int base = 0, bool defer = false) {
        stage(T_BROAD);
        bool done = false;
        const bool no_subset = std::getenv("CS_NO_SUBSET_SITES") != nullptr;
        const bool verify = std::getenv("CS_VERIFY_STATIC_SITE") != nullptr;
        if (prev_site != nullptr && xa == xb) {
            CS_RET(broad_phase_static(xa, cfg.d_hat, *prev_site, pr, done));
            if (done && verify) CS_RET(verify_static_site(xa, pr));
            if (done && rep) rep->static_sites += 1;
            if (done && verify && rep) rep->verified_sites += 1;
        } else if (base == 2 && !no_subset) {
            // a base costs a widened broad phase + a compaction; skip it while outer-loop
            // sites keep refusing the subset path (retry every 8 steps)
            if (subset_fail < 2 || step_index % 8 == 0) {
                CS_RET(build_base(xa, xb, cfg.d_hat));
                CS_RET(subset_site(xa, xb, cfg.d_hat, pr, done));
                if (done && verify) CS_RET(verify_site(xa, xb, pr));
                if (done && verify && rep) rep->verified_sites += 1;
            }
        } else if (base == 1 && !no_subset && base_valid) {
            CS_RET(subset_site(xa, xb, cfg.d_hat, pr, done));
            subset_fail = done ? 0 : subset_fail + 1;
            if (done && rep) rep->subset_sites += 1;
            if (done && verify) CS_RET(verify_site(xa, xb, pr));
            if (done && verify && rep) rep->verified_sites += 1;
        }
        if (!done) CS_RET(broad_phase(xa, xb, cfg.d_hat, pr));
        stage(T_FULL);
        const long long P = pr.P;
        if (P > 0) {
            // filter pass settles the provably-NaN pairs; heavy kernels run over worklists;
            // the march minimum folds into an +inf-initialised slot
            unsigned long long* min_slot = reinterpret_cast<unsigned long long*>(d_scal.p + S_MINBITS);
            k_fill_u64<<<1, 32, 0, s>>>(min_slot, 1, 0x7ff0000000000000ull);
            CS_RET(wl_full.ensure(P));
            CS_RET(wl_dist.ensure(P));
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_WLF, 0, 2 * sizeof(int), s));
            const SiteBoxes SB{(const float4*)fvbox.p, (const float4*)ftbox.p, (const float4*)febox.p, bmargin};
            k_site_filter<<<grid(P), 256, 0, s>>>(pr.keys.p, P, SB, 1e-6, 1.0 - cfg.alpha, 64, pr.toi.p, pr.filt.p,
                                                  wl_full.p, wl_dist.p, d_iscal.p + I_WLF);
            const int gw = std::max(1, std::min(grid(P, 128), 16 * sm_count));
            k_full_ccd_wl<<<gw, 128, 0, s>>>(wl_full.p, d_iscal.p + I_WLF, pr.kind.p, pr.idx.p, xa, xb,
                                             P == 1 ? 1 : 0, 1e-6, pr.toi.p);
            k_distance_toi_wl<<<gw, 128, 0, s>>>(wl_dist.p, d_iscal.p + I_WLF + 1, pr.kind.p, pr.idx.p, xa, xb,
                                                 1.0 - cfg.alpha, 64, pr.filt.p, min_slot);
            k_clamp_from_min<<<1, 1, 0, s>>>(min_slot, cfg.alpha, d_scal.p + S_CLAMP_MIN);
            launches += 5;
            static const bool trace_sites = std::getenv("CS_TRACE_SITES") != nullptr;
            if (trace_sites) {
                int wl[2];
                cudaMemcpyAsync(wl, d_iscal.p + I_WLF, sizeof(wl), cudaMemcpyDeviceToHost, s);
                cudaStreamSynchronize(s);
                std::fprintf(stderr, "[cs site] pairs %lld full-ccd worklist %d march worklist %d\n", P, wl[0], wl[1]);
            }
            CS_CHECK_LAUNCH();
            if (defer) {
                clamp = NAN;
            } else {
                CS_RET(sync_scalars(__LINE__));
                if (trace_sites) std::fprintf(stderr, "[cs site] min march toi %.6g\n", h_scal[S_CLAMP_MIN]);
                if (h_scal[S_CLAMP_BAD] != 0.0) return CS_PENETRATION;
                clamp = h_scal[S_CLAMP];
            }
        } else {
            clamp = 1.0;
            if (defer) {  // no pairs: clamp 1, no penetration, on the device too
                unsigned long long* min_slot = reinterpret_cast<unsigned long long*>(d_scal.p + S_MINBITS);
                k_fill_u64<<<1, 32, 0, s>>>(min_slot, 1, 0x7ff0000000000000ull);
                k_clamp_from_min<<<1, 1, 0, s>>>(min_slot, cfg.alpha, d_scal.p + S_CLAMP_MIN);
                launches += 2;
                CS_CHECK_LAUNCH();
                clamp = NAN;
            }
        }
        if (rep) {
            rep->full_ccd_calls += 1;
            rep->pairs_last_site = P;
            rep->pairs_max_site = std::max(rep->pairs_max_site, P);
        }
        return 0;
    }

    int witness(PairBuf& pr, const double* xw) {
        if (pr.P == 0) return 0;
        k_witness<<<grid(pr.P, 128), 128, 0, s>>>(pr.kind.p, pr.idx.p, xw, pr.P, pr.bary.p, pr.dist.p,
                                                  pr.normal.p, nullptr, nullptr, EngageOut{});
        ++launches;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // witness refresh at the anchor + engaged set and weights of a fresh site (NDB: one
    // pass; the life spans must be in place: zeroed or carried); count lands in I_ENG
    int witness_engage(PairBuf& pr, const double* xw) {
        if (cfg.barrier_mode == CS_BARRIER_DBB) {
            CS_RET(witness(pr, xw));
            return engage(pr);
        }
        plan_valid = false;
        pr.split_valid = false;
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_ENG, 0, sizeof(int), s));
        if (pr.P == 0) return 0;
        // the near / far split rides along (the far-pair classification on the toi and
        // distance this pass has in registers)
        EngageOut eo{pr.toi.p, pr.life.p, cfg.d_hat, cfg.ndb_k, cfg.ndb_base, pr.engaged.p, pr.weight.p,
                     d_iscal.p + I_ENG, nullptr, nullptr, nullptr, 0.0};
        if (far_pairs) {
            CS_RET(pr.near_l.ensure(pr.P));
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_NEAR, 0, sizeof(int), s));
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_FARREST, 0, sizeof(int), s));
            eo.split = pr.near_l.p;
            eo.n_near = d_iscal.p + I_NEAR;
            eo.n_far = d_iscal.p + I_FARREST;
            eo.near_thresh = near_thresh();
        }
        k_witness<<<grid(pr.P, 128), 128, 0, s>>>(pr.kind.p, pr.idx.p, xw, pr.P, pr.bary.p, pr.dist.p,
                                                  pr.normal.p, nullptr, nullptr, eo);
        ++launches;
        CS_CHECK_LAUNCH();
        pr.split_valid = far_pairs;  // counts read at the caller's sync (I_NEAR)
        return 0;
    }

    double near_thresh() const { return (2.0 * cfg.d_hat + kFarDelta * cfg.d_hat) * (1.0 + 1e-6) + 1e-12; }

    // engaged set + weights after a site; count lands in I_ENG
    int engage(PairBuf& pr) {
        plan_valid = false;
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_ENG, 0, sizeof(int), s));
        if (pr.P == 0) return 0;
        if (cfg.barrier_mode == CS_BARRIER_DBB)  // log barrier of the witness distance (stepper.py:489-491)
            k_dbb_weights<<<grid(pr.P), 256, 0, s>>>(pr.dist.p, pr.P, 2.0 * cfg.d_hat, cfg.dbb_kappa, pr.engaged.p,
                                                     pr.weight.p, d_iscal.p + I_ENG);
        else
            k_engage_init<<<grid(pr.P), 256, 0, s>>>(pr.toi.p, pr.dist.p, pr.life.p, pr.P, cfg.d_hat, cfg.ndb_k,
                                                     cfg.ndb_base, pr.engaged.p, pr.weight.p, d_iscal.p + I_ENG);
        ++launches;
        pr.split_valid = false;  // DBB: no partial CCD classes, no split
        CS_CHECK_LAUNCH();
        return 0;
    }

    // life-span carry old -> new (stepper.py:300-305).  Only pairs with a nonzero
    // life span can carry anything, so the hash table holds just those (one
    // extra 4-byte read-back sizes it; nothing to do when no pair is alive).
    int carry(PairBuf& old, PairBuf& nw_) {
        if (nw_.P == 0) return 0;
        // life spans of the new set: zero unless the lookup below writes every one
        const auto zero_new = [&]() -> int {
            CS_TRY(cudaMemsetAsync(nw_.life.p, 0, sizeof(int) * nw_.P, s));
            return 0;
        };
        if (old.P == 0) return zero_new();
        long long live = live_known;
        if (live < 0) {  // not counted by the last partial CCD pass on this set
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_LIVE, 0, sizeof(int), s));
            k_count_nonzero<<<grid(old.P), 256, 0, s>>>(old.life.p, old.P, d_iscal.p + I_LIVE);
            ++launches;
            CS_TRY(cudaMemcpyAsync(&h_iscal[I_LIVE], d_iscal.p + I_LIVE, sizeof(int), cudaMemcpyDeviceToHost, s));
            CS_TRY(hsync(__LINE__));
            live = h_iscal[I_LIVE];
        }
        live_known = -1;
        if (live == 0) return zero_new();
        unsigned long long cap = 1024;
        while (cap < 2ull * (unsigned long long)live) cap <<= 1;
        CS_RET(hkeys.ensure(cap));
        CS_RET(hvals.ensure(cap));
        k_fill_u64<<<grid(cap), 256, 0, s>>>(hkeys.p, cap, CS_EMPTY_KEY);
        k_hash_insert<<<grid(old.P), 256, 0, s>>>(old.keys.p, old.life.p, old.P, hkeys.p, hvals.p, cap - 1);
        k_hash_lookup<<<grid(nw_.P), 256, 0, s>>>(nw_.keys.p, nw_.P, hkeys.p, hvals.p, cap - 1, nw_.life.p);  // all P
        launches += 3;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // collision stamps from engaged pairs at world positions xw (stepper.py:238-285);
    // A = number of engaged pairs (known on host).  Fills seg_beg/seg_end, rows_act.
    int stamps(PairBuf& pr, long long A, const double* xw) {
        if (plan_valid && plan_pr == &pr && A > 0 && stamps_valid) {
            long long from = fused_ok ? plan_U : 0;  // plan pairs whose stamps must be computed here
            if (plan_new > 0) {
                // a union drifting far from the engaged set costs more per iteration than a
                // rebuild; an overflowing append list means the list is incomplete
                if (plan_new <= (long long)newsel.n && plan_U + plan_new <= A + A / 2 + (1 << 16)) {
                    long long r0 = 0;
                    CS_RET(plan_extend(pr, plan_new, r0));
                    from = std::min(from, r0);
                } else {
                    plan_valid = false;
                }
                plan_new = 0;
            }
            fused_ok = false;
            if (plan_valid) {
                if (from < plan_U) {
                    k_collision_terms<<<grid(plan_U - from), 256, 0, s>>>(
                        sel.p + from, plan_U - from, pr.kind.p, pr.idx.p, xw, pr.bary.p, pr.normal.p, pr.weight.p,
                        cfg.d_hat, n, free_index.p, 0, nullptr, stamp_p.p, pdst.p + 4 * from, stamp_sd.p);
                    ++launches;
                    CS_CHECK_LAUNCH();
                }
                stamps_plan_order = true;
                ++plan_reuses;
                rows_from_delta = true;
                return 0;
            }
        }
        plan_valid = false;
        stamps_valid = false;
        stamps_plan_order = false;
        n_stamp_rows = 0;
        CS_TRY(cudaMemsetAsync(seg_beg.p, 0, sizeof(int) * nf, s));
        CS_TRY(cudaMemsetAsync(seg_end.p, 0, sizeof(int) * nf, s));
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_ROWS, 0, sizeof(int), s));
        if (A <= 0 || pr.P == 0) return 0;
        CS_RET(sel.ensure(A));
        const long long m = 4 * A;
        CS_RET(skey.ensure(m));
        CS_RET(ssrc.ensure(m));
        CS_RET(skey_s.ensure(m));
        CS_RET(ssrc_s.ensure(m));
        CS_RET(stamp.ensure(m));
        CS_RET(rows_act.ensure(m));
        // compact engaged pair ids in pair order (tile counts, scan, writes)
        size_t bytes = 0;
        cub::CountingInputIterator<int> it(0);
        {
            const long long nt = (pr.P + kFlagTile - 1) / kFlagTile;
            CS_RET(ftile.ensure(nt + 1));
            CS_TRY(cudaMemsetAsync(ftile.p + nt, 0, sizeof(int), s));
            k_flag_tiles<<<(int)nt, 256, 0, s>>>(pr.engaged.p, pr.P, ftile.p);
            CS_RET(scan(ftile.p, ftile.p, (int)nt + 1));
            k_flag_compact<<<(int)nt, 256, 0, s>>>(pr.engaged.p, pr.P, ftile.p, sel.p);
            launches += 3;
        }
        k_collision_terms<<<grid(A), 256, 0, s>>>(sel.p, A, pr.kind.p, pr.idx.p, xw, pr.bary.p, pr.normal.p,
                                                  pr.weight.p, cfg.d_hat, n, free_index.p, 0, skey.p, stamp.p,
                                                  nullptr, nullptr);
        ++launches;
        // entries on a free row (a third of them are not: obstacle / pinned endpoints,
        // zero weight), compacted in order with their keys (tile counts, scan, write)
        const long long ntile = (A + kKeptTile - 1) / kKeptTile;
        CS_RET(ktile.ensure(ntile + 1));
        CS_TRY(cudaMemsetAsync(ktile.p + ntile, 0, sizeof(int), s));
        k_kept_tiles<<<(int)ntile, kKeptTile, 0, s>>>(skey.p, A, nf, ktile.p);
        CS_RET(scan(ktile.p, ktile.p, (int)ntile + 1));
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_COUNT + 7], ktile.p + ntile, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_RET(skey_c.ensure(m));
        k_kept_compact<<<(int)ntile, kKeptTile, 0, s>>>(skey.p, A, nf, ktile.p, ssrc.p, skey_c.p);
        launches += 3;
        CS_TRY(hsync(__LINE__));
        const long long mc = h_iscal[I_COUNT + 7];
        static const bool trace_stamps = std::getenv("CS_TRACE_SITES") != nullptr;
        if (trace_stamps)
            std::fprintf(stderr, "[cs stamps] engaged %lld stamps %lld on free rows %lld\n", A, m, mc);
        if (mc == 0) return 0;
        // stable sort by free row keeps np.add.at's per-vertex order; only the bits a
        // row needs
        int bits = 1;
        while ((1LL << bits) <= (long long)nf) ++bits;
        bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, skey_c.p, skey_s.p, ssrc.p, ssrc_s.p, (int)mc, 0, bits, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp.p, bytes, skey_c.p, skey_s.p, ssrc.p, ssrc_s.p, (int)mc, 0,
                                               bits, s));
        k_mark_segments<<<grid(mc), 256, 0, s>>>(skey_s.p, (int)mc, nf, seg_beg.p, seg_end.p, nullptr);
        ++launches;
        // distinct rows, ascending = the rows with a non-empty segment (a select over the
        // nf rows instead of the mc sorted entries)
        bytes = 0;
        cub::DeviceSelect::If(nullptr, bytes, it, rows_act.p, d_iscal.p + I_ROWS, nf, SegNonEmpty{seg_end.p}, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::If(cub_tmp.p, bytes, it, rows_act.p, d_iscal.p + I_ROWS, nf, SegNonEmpty{seg_end.p},
                                     s));
        CS_CHECK_LAUNCH();
        stamps_valid = true;
        n_stamp_rows = (int)std::min<long long>(m, nf);  // upper bound; exact count read on device
        rows_from_delta = false;
        // (only when the last outer loop ran more than one LG iteration: with one
        // iteration per pair set the plan would never be reused)
        if (plan_enabled && last_loop_lg > 1 && cfg.barrier_mode != CS_BARRIER_DBB && &pr == cur) {
            // cache the plan for the next LG iterations on this pair set
            CS_RET(pkey.ensure(mc));
            CS_RET(pdst.ensure(m));
            CS_RET(pair_u.ensure(pr.P));
            CS_RET(stamp_p.ensure(mc));
            CS_TRY(cudaMemsetAsync(pdst.p, 0xff, sizeof(int) * m, s));
            CS_TRY(cudaMemsetAsync(pair_u.p, 0xff, sizeof(int) * pr.P, s));
            k_plan_keys<<<grid(mc), 256, 0, s>>>(skey_s.p, ssrc_s.p, sel.p, (int)mc, pkey.p, pdst.p);
            k_plan_pair_u<<<grid(A), 256, 0, s>>>(sel.p, (int)A, pair_u.p);
            CS_RET(newsel.ensure(std::max<long long>(pr.P / 8, 1 << 16)));
            launches += 2;
            CS_CHECK_LAUNCH();
            plan_valid = true;
            plan_pr = &pr;
            plan_U = plan_Umain = A;
            plan_M = mc;
            side_M = 0;
            plan_new = 0;
            fused_ok = false;
        }
        return 0;
    }

    // merge the N pairs that joined the engaged set into the cached plan: append them to
    // the plan's pair list, sort their entries by merge key and merge them into the side
    // list (or, once the side list outgrows 1/8 of the main list, fold both into the main
    // list); rebuild the affected row segments and plan positions.  r0 = first plan pair
    // whose stamps the positions change (their fused stamps are stale).
    int plan_extend(PairBuf& pr, long long N, long long& r0) {
        int rb = 1;
        while ((1LL << rb) <= (long long)nf) ++rb;
        const int end_bit = kPlanRowShift + rb;
        const unsigned long long sentinel = (1ull << end_bit) - 1;
        const long long m4 = 4 * N, U2 = plan_U + N;
        CS_RET(sel.grow_keep(U2, plan_U));
        CS_RET(pdst.grow_keep(4 * U2, 4 * plan_U));
        CS_RET(nkey.ensure(m4));
        CS_RET(nsrc.ensure(m4));
        CS_RET(nkey_s.ensure(m4));
        CS_RET(nsrc_s.ensure(m4));
        // the append order of newsel is arbitrary; the plan order is the merge key's
        k_plan_new<<<grid(N), 256, 0, s>>>(newsel.p, (int)N, (int)plan_U, pr.kind.p, pr.idx.p, pr.bary.p, n,
                                           free_index.p, sentinel, sel.p, pair_u.p, nkey.p, nsrc.p);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, nkey.p, nkey_s.p, nsrc.p, nsrc_s.p, (int)m4, 0, end_bit, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp.p, bytes, nkey.p, nkey_s.p, nsrc.p, nsrc_s.p, (int)m4, 0,
                                               end_bit, s));
        launches += 2;
        // side list + new entries
        const unsigned long long* k2 = nkey_s.p;
        const int* v2 = nsrc_s.p;
        long long n2 = m4;
        if (side_M > 0) {
            CS_RET(skey_sd2.ensure(side_M + m4));
            CS_RET(ssrc_sd2.ensure(side_M + m4));
            CS_RET(merge_keys(skey_sd.p, ssrc_sd.p, side_M, nkey_s.p, nsrc_s.p, m4, skey_sd2.p, ssrc_sd2.p));
            std::swap(skey_sd, skey_sd2);
            std::swap(ssrc_sd, ssrc_sd2);
            k2 = skey_sd.p;
            v2 = ssrc_sd.p;
            n2 = side_M + m4;
        }
        if (n2 <= std::max<long long>(plan_M / 8, 1 << 16)) {
            if (side_M == 0) {  // the sorted new entries become the side list
                CS_RET(skey_sd.ensure(m4));
                CS_RET(ssrc_sd.ensure(m4));
                CS_TRY(cudaMemcpyAsync(skey_sd.p, nkey_s.p, sizeof(unsigned long long) * m4, cudaMemcpyDeviceToDevice,
                                       s));
                CS_TRY(cudaMemcpyAsync(ssrc_sd.p, nsrc_s.p, sizeof(int) * m4, cudaMemcpyDeviceToDevice, s));
            }
            side_M = n2;
            CS_RET(sseg_beg.ensure(nf));
            CS_RET(sseg_end.ensure(nf));
            CS_RET(stamp_sd.ensure(side_M));
            CS_TRY(cudaMemsetAsync(sseg_beg.p, 0, sizeof(int) * nf, s));
            CS_TRY(cudaMemsetAsync(sseg_end.p, 0, sizeof(int) * nf, s));
            CS_TRY(cudaMemsetAsync(pdst.p + 4 * plan_Umain, 0xff, sizeof(int) * 4 * (U2 - plan_Umain), s));
            k_plan_segments<<<grid(side_M), 256, 0, s>>>(skey_sd.p, ssrc_sd.p, (int)side_M, nf, sseg_beg.p,
                                                         sseg_end.p, pdst.p, 1);
            r0 = plan_Umain;
        } else {
            // fold the side list (+ new entries) into the main list
            const long long M2 = plan_M + n2;
            CS_RET(pkey2.ensure(M2));
            CS_RET(psrc2.ensure(M2));
            CS_RET(merge_keys(pkey.p, ssrc_s.p, plan_M, k2, v2, n2, pkey2.p, psrc2.p));
            std::swap(pkey, pkey2);
            std::swap(ssrc_s, psrc2);
            plan_M = M2;
            side_M = 0;
            plan_Umain = U2;
            CS_RET(stamp_p.ensure(plan_M));
            CS_TRY(cudaMemsetAsync(seg_beg.p, 0, sizeof(int) * nf, s));
            CS_TRY(cudaMemsetAsync(seg_end.p, 0, sizeof(int) * nf, s));
            CS_TRY(cudaMemsetAsync(pdst.p, 0xff, sizeof(int) * 4 * U2, s));
            k_plan_segments<<<grid(plan_M), 256, 0, s>>>(pkey.p, ssrc_s.p, (int)plan_M, nf, seg_beg.p, seg_end.p,
                                                         pdst.p, 0);
            r0 = 0;
        }
        ++launches;
        CS_CHECK_LAUNCH();
        plan_U = U2;
        return 0;
    }

    int merge_keys(const unsigned long long* k1, const int* v1, long long n1, const unsigned long long* k2,
                   const int* v2, long long n2, unsigned long long* ko, int* vo) {
        size_t bytes = 0;
        cub::DeviceMerge::MergePairs(nullptr, bytes, k1, v1, (int)n1, k2, v2, (int)n2, ko, vo, U64Less{}, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceMerge::MergePairs(cub_tmp.p, bytes, k1, v1, (int)n1, k2, v2, (int)n2, ko, vo, U64Less{},
                                            s));
        ++launches;
        return 0;
    }

    // rows_act = rows with delta > 0 (a plan reused across iterations can hold rows
    // whose pairs all left the engaged set); same list as the fresh plan's
    int rows_act_from_delta() {
        CS_RET(rowpos.ensure(nf));
        CS_RET(rows_act.ensure(nf));
        k_flag_positive<<<grid(nf), 256, 0, s>>>(delta.p, nf, rowpos.p);
        size_t bytes = 0;
        cub::CountingInputIterator<int> it(0);
        cub::DeviceSelect::Flagged(nullptr, bytes, it, rowpos.p, rows_act.p, d_iscal.p + I_ROWS, nf, s);
        CS_RET(cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(cub_tmp.p, bytes, it, rowpos.p, rows_act.p, d_iscal.p + I_ROWS, nf, s));
        ++launches;
        CS_CHECK_LAUNCH();
        return 0;
    }

    // one local-global cycle (stepper.py:402-424) on the candidate cloth rows xc_w[:n]
    int inner_solve(long long A) {
        stage(T_LOCAL);
        CS_RET(stamps(*cur, A, xc_w.p));
        CS_RET(assemble_rhs(z.p, xc_w.p, stamps_valid));
        if (stamps_valid && rows_from_delta) CS_RET(rows_act_from_delta());
        k_gather_rows<<<grid(nf), 256, 0, s>>>(xc_w.p, free_ids.p, nf, xf0.p);
        CS_TRY(cudaMemcpyAsync(xf.p, xf0.p, sizeof(double) * 3 * nf, cudaMemcpyDeviceToDevice, s));
        ++launches;
        stage(T_GLOBAL);
        CS_RET(reduced(b.p, xf.p, delta.p, true, stamps_valid ? n_stamp_rows : 0));
        stage(T_SMOOTH);
        CS_RET(smooth(b.p, xf.p, cfg.smoothing_iterations, cfg.omega, delta.p));
        return 0;
    }

    int lerp_world(const double* a, const double* bb, const double* tptr, double* out) {
        k_lerp<<<grid(3LL * nw), 256, 0, s>>>(a, bb, tptr, 3LL * nw, out);
        ++launches;
        CS_CHECK_LAUNCH();
        return 0;
    }

    int set_clamp_value(double tval) {
        h_scal[S_CLAMP] = tval;
        CS_TRY(cudaMemcpyAsync(d_scal.p + S_CLAMP, &h_scal[S_CLAMP], sizeof(double), cudaMemcpyHostToDevice, s));
        return 0;
    }

    // ------------------------------------------------------------ step
    int step(const double* pin_next_h, const double* obs_next_h, cs_step_report* rep);
    int residual_forward(const double* x_final_w, cs_step_report* rep);
    int create(const cs_scene_desc* d, const cs_step_config* c, int want);
    int parts = 0;  // CS_PART_* present
    bool has(int need) const { return (parts & need) == need; }
    void set_pattern();
    void release();
};

void cs_scene::set_pattern() {
    static const double tri1[1][2] = {{1.0 / 3.0, 1.0 / 3.0}};
    static const double tri3[3][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0}};
    static const double tri6[6][2] = {{1.0 / 6.0, 1.0 / 6.0}, {2.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 2.0 / 3.0},
                                      {0.5, 0.25}, {0.25, 0.5}, {1.0 / 3.0, 1.0 / 3.0}};
    static const double box1[1][2] = {{0.5, 0.5}};
    static const double box3[3][2] = {{0.25, 0.25}, {0.5, 0.5}, {0.75, 0.75}};
    static const double box6[6][2] = {{0.25, 0.25}, {0.5, 0.5}, {0.75, 0.75}, {0.25, 0.75}, {0.75, 0.25}, {0.5, 0.25}};
    const int cnt = cfg.samples == 1 ? 1 : (cfg.samples == 6 ? 6 : 3);
    const double(*tp)[2] = cnt == 1 ? tri1 : (cnt == 6 ? tri6 : tri3);
    const double(*bp)[2] = cnt == 1 ? box1 : (cnt == 6 ? box6 : box3);
    pat.width = cnt;
    for (int k = 0; k < cnt; ++k) {
        pat.vt[k][0] = tp[k][0];
        pat.vt[k][1] = tp[k][1];
        pat.ee[k][0] = bp[k][0];
        pat.ee[k][1] = bp[k][1];
    }
}

int cs_scene::create(const cs_scene_desc* d, const cs_step_config* c, int want) {
    cfg = *c;
    parts = want;
    n = d->n_cloth;
    nf = d->n_free;
    npin = d->n_pinned;
    nobs = d->n_obstacle;
    nw = d->n_world;
    ne = d->n_edges;
    ns = d->n_stencils;
    ntw = d->n_world_tris;
    new_ = d->n_world_edges;
    rb = d->r_bar;
    r = d->r;
    const bool sys = want & CS_PART_SYSTEM, cloth = want & CS_PART_CLOTH, basis = want & CS_PART_BASIS,
               world = want & CS_PART_WORLD, state = (want & CS_PART_ALL) == CS_PART_ALL;
    if (cloth && !sys) return CS_BAD_ARGUMENT;
    if ((sys || basis) && nf <= 0) return CS_BAD_ARGUMENT;
    if (cloth && (n <= 0 || nf > n)) return CS_BAD_ARGUMENT;
    if (basis && (rb <= 0 || r <= 0 || r > rb || rb > 128 || r > 32)) return CS_BAD_ARGUMENT;
    if (world && (nw <= 0 || ntw <= 0 || new_ <= 0)) return CS_BAD_ARGUMENT;
    if (state && nw != n + nobs) return CS_BAD_ARGUMENT;
    set_pattern();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (cloth) {
        CS_RET(free_ids.upload(d->free_ids, nf));
        CS_RET(free_index.upload(d->free_index, n));
        CS_RET(pin_ids.upload(d->pin_ids, npin));
        CS_RET(mass.upload(d->mass, n));
        CS_RET(fext.upload(d->fext, 3LL * n));
        CS_RET(mh2.upload(d->mass_over_h2, nf));
        std::vector<int> a(ne), bb(ne), slot(n, -1);
        for (int i = 0; i < ne; ++i) {
            a[i] = d->edge_v[2 * i];
            bb[i] = d->edge_v[2 * i + 1];
        }
        for (int i = 0; i < npin; ++i) slot[d->pin_ids[i]] = i;
        CS_RET(e0.upload(a.data(), ne));
        CS_RET(e1.upload(bb.data(), ne));
        CS_RET(pin_slot.upload(slot.data(), n));
        CS_RET(erest.upload(d->edge_rest, ne));
        CS_RET(ew.upload(d->edge_w, ne));
        CS_RET(rinc_ptr.upload(d->rhs_inc_ptr, n + 1));
        CS_RET(rinc.upload(d->rhs_inc, d->rhs_inc_ptr[n]));
        CS_RET(ginc_ptr.upload(d->grad_inc_ptr, n + 1));
        CS_RET(ginc.upload(d->grad_inc, d->grad_inc_ptr[n]));
        CS_RET(st.upload(d->stencils, 4LL * ns));
        CS_RET(bk.upload(d->bend_k, 4LL * ns));
        CS_RET(bw.upload(d->bend_w, ns));
        CS_RET(binc_ptr.upload(d->bend_inc_ptr, n + 1));
        CS_RET(binc.upload(d->bend_inc, d->bend_inc_ptr[n]));
        CS_RET(hfp_ptr.upload(d->hfp_ptr, nf + 1));
        has_fp = npin > 0 && d->hfp_ptr != nullptr && d->hfp_ptr[nf] > 0;
        CS_RET(hfp_col.upload(d->hfp_col, std::max(d->hfp_ptr[nf], 1)));
        CS_RET(hfp_val.upload(d->hfp_val, std::max(d->hfp_ptr[nf], 1)));
    }
    if (sys) {
        nslices = d->sell_nslices;
        CS_RET(sell_ptr.upload(d->sell_slice_ptr, nslices + 1));
        CS_RET(sell_col.upload(d->sell_col, d->sell_slice_ptr[nslices]));
        CS_RET(sell_val.upload(d->sell_val, d->sell_slice_ptr[nslices]));
        CS_RET(diag.upload(d->diag, nf));
    }
    if (basis) {
        CS_RET(U.upload(d->U, (size_t)nf * rb));
        std::vector<double> vv((size_t)nf * r);
        for (long long i = 0; i < nf; ++i)
            for (int j = 0; j < r; ++j) vv[i * r + j] = d->U[i * rb + j];
        CS_RET(V.upload(vv.data(), vv.size()));
        CS_RET(lam.upload(d->eigenvalues, rb));
    }
    if (world) {
        CS_RET(wtris.upload(d->world_tris, 3LL * ntw));
        CS_RET(wedges.upload(d->world_edges, 2LL * new_));
        CS_RET(tri_static.upload(d->tri_static, ntw));
        CS_RET(vert_static.upload(d->vert_static, nw));
        CS_RET(vert_used.upload(d->vert_used, nw));
        CS_RET(edge_static.upload(d->edge_static, new_));
        CS_RET(edge_tris.upload(d->edge_tris, 2LL * new_));
        CS_RET(edge_slot.upload(d->edge_slot, 2LL * new_));
        CS_RET(patch.upload(d->patch, ntw));
        CS_RET(pslot.upload(d->patch_slot, ntw));
        CS_RET(eflip.ensure(new_));
        k_edge_flip_info<<<grid(new_), 256>>>(new_, edge_tris.p, edge_slot.p, tri_static.p, patch.p, pslot.p,
                                               eflip.p);
        CS_TRY(cudaGetLastError());
        CS_RET(vtab.create(nw, false));
        CS_RET(ttab.create(ntw, true));
        CS_RET(etab.create(new_, true));
        for (DBuf<double>* w : {&xs_w, &xc_w, &anchor_w, &tmp_w}) CS_RET(w->ensure(3LL * nw));
        CS_RET(vlo.ensure(3LL * nw));
        CS_RET(vhi.ensure(3LL * nw));
        CS_RET(vdisp.ensure(nw, true));
        CS_RET(fvbox.ensure(16LL * nw, true));
        CS_RET(ftbox.ensure(16LL * ntw, true));
        CS_RET(febox.ensure(16LL * new_, true));
        CS_RET(tdisp.ensure(ntw, true));
        CS_RET(edisp.ensure(new_, true));
    }
    if (state) {
        CS_RET(x.upload(d->x0, 3LL * n));
        CS_RET(xprev.upload(d->x0, 3LL * n));
        CS_RET(v.ensure(3LL * n));
        CS_RET(df.ensure(3LL * n));
        CS_TRY(cudaMemset(v.p, 0, sizeof(double) * 3 * n));
        CS_TRY(cudaMemset(df.p, 0, sizeof(double) * 3 * n));
        CS_RET(obs.upload(d->obstacle_x0, 3LL * std::max(nobs, 0)));
        CS_RET(obs.ensure(std::max(3LL * nobs, 1LL)));
        CS_RET(pins_next_d.ensure(std::max(3 * npin, 1)));
        CS_RET(obs_next_d.ensure(std::max(3 * nobs, 1)));
        // page-locked staging for the per-step pin / obstacle targets (a pageable
        // cudaMemcpyAsync stages through the driver and can stall the stream)
        CS_TRY(cudaMallocHost(&h_stage, sizeof(double) * (3 * npin + 3 * nobs + 1)));
    }
    if (cloth) for (DBuf<double>* w : {&z, &prev_outer, &grad, &dfn}) CS_RET(w->ensure(3LL * n));
    if (sys) {
        for (DBuf<double>* w : {&xf, &xf0, &b, &t, &fr}) CS_RET(w->ensure(3LL * nf));
        CS_RET(delta.ensure(nf));
        CS_RET(seg_beg.ensure(nf));
        CS_RET(seg_end.ensure(nf));
    }
    CS_RET(rhs_red.ensure(3 * 128));
    CS_RET(gram_red.ensure(32 * 32));
    CS_RET(q.ensure(3 * 128));
    CS_RET(Xred.ensure(32 * 32));
    CS_RET(beta_red.ensure(1));
    CS_RET(fallback.ensure(1));
    // scalar block, one allocation on each side so sync_scalars is a single copy:
    // [S_COUNT doubles | 4 doubles scratch | I_COUNT ints | 8 ints scratch]
    constexpr int kScalDoubles = S_COUNT + 4 + (I_COUNT + 8 + 1) / 2;
    CS_RET(d_scal.ensure(kScalDoubles, true));
    CS_TRY(cudaMemset(d_scal.p, 0, sizeof(double) * kScalDoubles));
    d_iscal.p = reinterpret_cast<int*>(d_scal.p + S_COUNT + 4);  // view into d_scal
    d_iscal.n = I_COUNT + 8;
    CS_TRY(cudaMallocHost(&h_scal, sizeof(double) * kScalDoubles));
    h_iscal = reinterpret_cast<int*>(h_scal + S_COUNT + 4);
    CS_TRY(cudaMallocHost(&h_norms, sizeof(double) * kMaxNormChecks));
    CS_RET(pa.reserve(1024));
    CS_RET(pb.reserve(1024));
    CS_TRY(cudaDeviceSynchronize());
    return 0;
}

void cs_scene::release() {
    for (auto& sg : smooth_graphs) cudaGraphExecDestroy(sg.exec);
    smooth_graphs.clear();
    if (cap_stream) cudaStreamDestroy(cap_stream);
    cap_stream = nullptr;
    for (FrameSlot& f : frame_slots) {
        if (f.used) cudaEventSynchronize(f.done);
        if (f.taken) cudaEventDestroy(f.taken);
        if (f.done) cudaEventDestroy(f.done);
        f.taken = f.done = nullptr;
        f.x.release();
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
    copy_stream = nullptr;
    for (auto e : ev_pool) cudaEventDestroy(e);
    ev_pool.clear();
    if (h_scal) cudaFreeHost(h_scal);  // h_iscal is a view into it
    if (h_norms) cudaFreeHost(h_norms);
    h_norms = nullptr;
    if (h_stage) cudaFreeHost(h_stage);
    h_stage = nullptr;
    h_scal = nullptr;
    h_iscal = nullptr;
    // DBuf members release through their owners
    DBuf<int>* ints[] = {&free_ids, &free_index, &pin_ids, &pin_slot, &e0, &e1, &rinc_ptr, &rinc, &ginc_ptr, &ginc,
                         &st, &binc_ptr, &binc, &sell_ptr, &sell_col, &hfp_ptr, &hfp_col, &wtris, &wedges,
                         &edge_tris, &edge_slot, &patch, &pslot, &sel, &skey, &ssrc, &skey_s,
                         &ssrc_s, &seg_beg, &seg_end, &rowflag, &rows_act, &skey_c, &hvals, &fallback, &wl_full, &wl_dist};
    d_iscal.p = nullptr;  // view into d_scal
    d_iscal.n = 0;
    for (auto* p : ints) p->release();
    DBuf<double>* dbl[] = {&mass, &fext, &mh2, &erest, &ew, &bk, &bw, &sell_val, &diag, &hfp_val, &U, &V, &lam,
                           &x, &v, &xprev, &df, &obs, &z, &xs_w, &xc_w, &anchor_w, &tmp_w, &xf, &xf0, &b, &t,
                           &delta, &prev_outer, &grad, &dfn, &fr, &pins_next_d, &obs_next_d, &vlo, &vhi, &vdisp, &tdisp, &edisp,
                           &part, &part2, &spart, &rhs_red, &gram_red, &q, &Xred, &beta_red, &d_scal, &norms};
    for (auto* p : dbl) p->release();
    tri_static.release();
    vert_static.release();
    vert_used.release();
    edge_static.release();
    eflip.release();
    keep_flag.release();
    keep_bits.release();
    tile_cnt.release();
    tile_off.release();
    basepr.release();
    blo.release();
    bhi.release();
    vviol.release();
    tviol.release();
    eviol.release();
    for (DBuf<int>* b : {&vlist, &tlist, &elist, &qcount, &qoff}) b->release();
    query_dbg.release();
    isect_out.release();
    fvbox.release();
    ftbox.release();
    febox.release();
    stamp.release();
    cheb_b1.release();
    cheb_b2.release();
    hkeys.release();
    cub_tmp.release();
    pa.release();
    pb.release();
    vtab.release();
    ttab.release();
    etab.release();
    vtab_v.release();
    ttab_v.release();
    etab_v.release();
    ocount.release();
    ooffset.release();
}

int cs_scene::step(const double* pin_next_h, const double* obs_next_h, cs_step_report* rep) {
    launches = 0;
    n_syncs = 0;
    live_known = -1;
    const long long plan_reuses0 = plan_reuses;
    ev_used = 0;
    spans.clear();
    active_stage = -1;
    const double h = cfg.h;
    // prescribed geometry at t + h (stepper.py:461-463): host callbacks evaluated by the caller
    // (the previous step ended with a stream synchronisation, so h_stage is free)
    if (npin) {
        if (pin_next_h) {
            std::memcpy(h_stage, pin_next_h, sizeof(double) * 3 * npin);
            static const bool trace_h = std::getenv("CS_TRACE_HOST") != nullptr;
            const auto tq0 = std::chrono::steady_clock::now();
            CS_TRY(cudaMemcpyAsync(pins_next_d.p, h_stage, sizeof(double) * 3 * npin, cudaMemcpyHostToDevice, s));
            if (trace_h)
                std::fprintf(stderr, "[cs host] pins H2D call %.1f us\n",
                             std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tq0).count());
        } else {
            k_gather_rows<<<grid(npin), 256, 0, s>>>(x.p, pin_ids.p, npin, pins_next_d.p);
            ++launches;
        }
    }
    const double* obs_next = obs.p;
    if (nobs && obs_next_h) {
        std::memcpy(h_stage + 3 * npin, obs_next_h, sizeof(double) * 3 * nobs);
        CS_TRY(cudaMemcpyAsync(obs_next_d.p, h_stage + 3 * npin, sizeof(double) * 3 * nobs, cudaMemcpyHostToDevice,
                               s));
        obs_next = obs_next_d.p;
    }
    stage(T_WARM);
    // z = inertia target (mesh.py:174-196)
    CS_TRY(cudaMemsetAsync(d_iscal.p + I_BAD, 0, sizeof(int), s));
    k_inertia_target<<<grid(n), 256, 0, s>>>(x.p, v.p, fext.p, df.p, mass.p, n, h, pin_slot.p, pins_next_d.p, z.p,
                                            d_iscal.p + I_BAD);
    ++launches;
    CS_CHECK_LAUNCH();
    // ---- warm start (stepper.py:384-400): x = z (pins already at pin_next)
    double* xcl = xc_w.p;  // cloth rows of the candidate world array
    CS_TRY(cudaMemcpyAsync(xcl, z.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    // the non-finite check of the inertia target is read at the warm start's first
    // synchronisation (nothing in between writes I_BAD; a failing step commits nothing)
    bool inertia_unchecked = true;
    // toi_exit on the device: min over the outer sites' clamps (stepper.py:556-558)
    k_set_scalar<<<1, 1, 0, s>>>(d_scal.p + S_TOIEXIT, 1.0);
    ++launches;
    int ws_iters = 0;
    for (int it = 0; it < cfg.warm_start_cap; ++it) {
        CS_RET(assemble_rhs(z.p, xcl, false));
        k_gather_rows<<<grid(nf), 256, 0, s>>>(xcl, free_ids.p, nf, xf0.p);
        CS_TRY(cudaMemcpyAsync(xf.p, xf0.p, sizeof(double) * 3 * nf, cudaMemcpyDeviceToDevice, s));
        ++launches;
        CS_RET(warm_correction(b.p, xf.p));
        CS_RET(sqnorm(xf.p, xf0.p, nf, nullptr, S_SQ));
        k_scatter_rows<<<grid(nf), 256, 0, s>>>(xf.p, free_ids.p, nf, xcl);
        ++launches;
        CS_RET(sync_scalars(__LINE__));
        if (inertia_unchecked && h_iscal[I_BAD]) return CS_NONFINITE;
        inertia_unchecked = false;
        ++ws_iters;
        const double dx = h_scal[S_SQ] / std::max(std::sqrt(3.0 * nf), 1.0);
        if (dx < cfg.eps_initial) break;
    }
    if (rep) rep->warm_start_iterations = ws_iters;

    // ---- world arrays: start = [x; obstacle_x], candidate = [x_cand; obs_next]
    CS_TRY(cudaMemcpyAsync(xs_w.p, x.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    if (nobs) {
        CS_TRY(cudaMemcpyAsync(xs_w.p + 3LL * n, obs.p, sizeof(double) * 3 * nobs, cudaMemcpyDeviceToDevice, s));
        CS_TRY(cudaMemcpyAsync(xc_w.p + 3LL * n, obs_next, sizeof(double) * 3 * nobs, cudaMemcpyDeviceToDevice, s));
    }
    double tc = 1.0;
    CS_RET(ccd_site(xs_w.p, xc_w.p, *cur, rep, tc, nullptr, 2, true));
    // x_acc = clamp; anchor = x_acc (stepper.py:475-480); the clamp factor is read on the
    // device, its penetration flag at the next synchronisation (below)
    CS_RET(lerp_world(xs_w.p, xc_w.p, d_scal.p + S_CLAMP, tmp_w.p));
    CS_TRY(cudaMemcpyAsync(xc_w.p, tmp_w.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
    CS_TRY(cudaMemcpyAsync(anchor_w.p, tmp_w.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
    stage(T_FULL);
    if (cur->P) CS_TRY(cudaMemsetAsync(cur->life.p, 0, sizeof(int) * cur->P, s));
    CS_RET(witness_engage(*cur, anchor_w.p));
    CS_TRY(cudaMemcpyAsync(prev_outer.p, xcl, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    CS_RET(sync_scalars(__LINE__));
    if (h_scal[S_CLAMP_BAD] != 0.0) return CS_PENETRATION;  // the first site (_clamp, stepper.py:445-452)
    if (inertia_unchecked && h_iscal[I_BAD]) return CS_NONFINITE;
    long long A = h_iscal[I_ENG];
    if (cur->split_valid) cur->n_near = h_iscal[I_NEAR];

    double dx_last = INFINITY;
    bool cap_hit = false;
    double toi_exit = 1.0;
    int lg = 0, outer_loops = 0, partial_calls = 0;
    int n_deltas = 0;
    for (int outer = 0; outer < cfg.outer_cap; ++outer) {
        int lg_loop = 0;
        for (int inner = 0; inner < cfg.inner_cap; ++inner) {
            ++lg_loop;
            last_loop_lg = std::max(last_loop_lg, lg_loop);
            CS_RET(inner_solve(A));
            // dx = rms(x_new[free] - x_cand[free]); write back (stepper.py:506-509)
            CS_RET(sqnorm(xf.p, xf0.p, nf, nullptr, S_SQ));
            k_scatter_rows<<<grid(nf), 256, 0, s>>>(xf.p, free_ids.p, nf, xcl);
            ++launches;
            ++lg;
            if (cfg.barrier_mode == CS_BARRIER_DBB) {
                // DBB baseline (stepper.py:524-538): the partial-CCD classes go unused;
                // distance march anchor -> candidate, clamp, witness at the candidate,
                // log-barrier weights
                ++partial_calls;
                double t_in = 1.0;
                stage(T_FULL);
                if (cur->P) {
                    k_distance_toi<<<grid(cur->P, 128), 128, 0, s>>>(cur->kind.p, cur->idx.p, anchor_w.p, xc_w.p,
                                                                     cur->P, 1.0 - cfg.alpha, 64, cur->filt.p);
                    const int g = std::min(grid(cur->P), 2 * sm_count);
                    CS_RET(part.ensure(g));
                    k_min_toi_partial<<<g, 256, 0, s>>>(cur->filt.p, cur->P, part.p);
                    k_min_toi_final<<<1, 256, 0, s>>>(part.p, g, cfg.alpha, d_scal.p + S_CLAMP_MIN);
                    launches += 3;
                    CS_CHECK_LAUNCH();
                }
                CS_RET(sync_scalars(__LINE__));
                dx_last = h_scal[S_SQ] / std::max(std::sqrt(3.0 * nf), 1.0);
                if (cur->P) {
                    if (h_scal[S_CLAMP_BAD] != 0.0) return CS_PENETRATION;
                    t_in = h_scal[S_CLAMP];
                }
                if (t_in < 1.0) {
                    CS_RET(lerp_world(anchor_w.p, xc_w.p, d_scal.p + S_CLAMP, tmp_w.p));
                    CS_TRY(cudaMemcpyAsync(xc_w.p, tmp_w.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
                }
                CS_RET(witness(*cur, xc_w.p));
                CS_RET(engage(*cur));
                CS_RET(sync_scalars(__LINE__));
                A = h_iscal[I_ENG];
                if (cfg.iteration_cap && lg >= cfg.iteration_cap) {
                    cap_hit = true;
                    break;
                }
                if (dx_last <= cfg.eps_inner) break;
                continue;
            }
            // partial CCD + NDB life-span update (stepper.py:511-523)
            stage(T_PARTIAL);
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_ENG, 0, sizeof(int), s));
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_NEW, 0, sizeof(int), s));
            CS_TRY(cudaMemsetAsync(d_iscal.p + I_LIVE, 0, sizeof(int), s));  // the carry's table size
            // collect pairs joining the stamp plan; write the plan's next stamps (fused terms)
            const bool track = plan_valid && plan_pr == cur;
            PlanView plan{};
            if (track)
                plan = PlanView{pair_u.p, d_iscal.p + I_NEW, newsel.p, (int)newsel.n, pdst.p, stamp_p.p,
                                side_M > 0 ? stamp_sd.p : nullptr, n, free_index.p};
            fused_ok = track;
            if (cur->P) {
                const NdbArgs na{cur->kind.p, cur->idx.p, anchor_w.p, xc_w.p, pat, cur->bary.p, cur->normal.p,
                                 cfg.d_hat, cfg.ndb_k, cfg.ndb_base, cur->life.p, cur->weight.p, cur->engaged.p,
                                 0, nullptr, 1, d_iscal.p + I_LIVE};
                if (cur->split_valid) {
                    // near list: the full classifier; far list (after it, reversed): gated on the
                    // largest vertex displacement anchor -> candidate (k_far_gate, then the rest through
                    // the classifier: k_partial_ndb_dyn)
                    const long long nn = cur->n_near, nfar = cur->P - cur->n_near;
                    CS_RET(vdn.ensure(nw));
                    k_vertex_disp_norm<<<grid(nw), 256, 0, s>>>(anchor_w.p, xc_w.p, nw, vdn.p);
                    if (nn > 0)
                        k_partial_ndb<<<grid(nn, 128), 128, 0, s>>>(na, nn, d_iscal.p + I_ENG, plan, cur->near_l.p);
                    if (nfar > 0) {
                        CS_RET(far_rest.ensure(nfar));
                        CS_TRY(cudaMemsetAsync(d_iscal.p + I_FARREST, 0, sizeof(int), s));
                        k_far_gate<<<grid(nfar), 256, 0, s>>>(na, nfar, plan, cur->near_l.p + nn, cur->dist.p, vdn.p,
                                                               far_rest.p, d_iscal.p + I_FARREST);
                        k_partial_ndb_dyn<<<6 * sm_count, 128, 0, s>>>(na, d_iscal.p + I_FARREST, d_iscal.p + I_ENG,
                                                                        plan, far_rest.p);
                        ++launches;
                    }
                    launches += 3;
                } else {
                    k_partial_ndb<<<grid(cur->P, 128), 128, 0, s>>>(na, cur->P, d_iscal.p + I_ENG, plan, nullptr);
                    ++launches;
                }
                CS_CHECK_LAUNCH();
            }
            ++partial_calls;
            CS_RET(sync_scalars(__LINE__));
            dx_last = h_scal[S_SQ] / std::max(std::sqrt(3.0 * nf), 1.0);
            A = h_iscal[I_ENG];
            plan_new = h_iscal[I_NEW];
            live_known = cur->P ? h_iscal[I_LIVE] : -1;

            if (cfg.iteration_cap && lg >= cfg.iteration_cap) {
                cap_hit = true;
                break;
            }
            if (dx_last <= cfg.eps_inner) break;
        }
        ++outer_loops;
        last_loop_lg = lg_loop;
        // fresh pair set + line-search filter at the end of every outer loop (stepper.py:547-570)
        double tout = 1.0;
        CS_RET(ccd_site(anchor_w.p, xc_w.p, *nxt, rep, tout, nullptr, 1, true));
        // truncation with the device clamp (k_lerp: t >= 1 keeps the candidate exactly),
        // toi_exit folded on the device; the penetration flag is read at this loop's sync
        CS_RET(lerp_world(anchor_w.p, xc_w.p, d_scal.p + S_CLAMP, tmp_w.p));
        CS_TRY(cudaMemcpyAsync(xc_w.p, tmp_w.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
        k_min_scalar<<<1, 1, 0, s>>>(d_scal.p + S_TOIEXIT, d_scal.p + S_CLAMP);
        ++launches;
        CS_TRY(cudaMemcpyAsync(anchor_w.p, xc_w.p, sizeof(double) * 3 * nw, cudaMemcpyDeviceToDevice, s));
        stage(T_FULL);
        // life spans carried first (keys only), then witness + engagement in one pass
        if (cfg.barrier_mode != CS_BARRIER_DBB) CS_RET(carry(*cur, *nxt));
        CS_RET(witness_engage(*nxt, anchor_w.p));
        std::swap(cur, nxt);
        // outer progress (stepper.py:574-578)
        CS_RET(sqnorm(xcl, prev_outer.p, nf, free_ids.p, S_SQ));
        // prev_outer holds cloth rows; compare over free rows only
        CS_TRY(cudaMemcpyAsync(prev_outer.p, xcl, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
        CS_RET(sync_scalars(__LINE__));
        if (h_scal[S_CLAMP_BAD] != 0.0) return CS_PENETRATION;  // this loop's site
        toi_exit = h_scal[S_TOIEXIT];
        A = h_iscal[I_ENG];
        if (cur->split_valid) cur->n_near = h_iscal[I_NEAR];
        const double d_out = h_scal[S_SQ] / std::max(std::sqrt(3.0 * nf), 1.0);
        if (rep && n_deltas < 64) rep->outer_deltas[n_deltas++] = d_out;
        if (cap_hit || d_out <= cfg.eps_outer) break;
    }
    // ---- exit line search (stepper.py:580-592)
    const long long active_pairs = cur->P ? A : 0;
    double tfin = 1.0;
    // anchor_w == xc_w here (the last outer site set the anchor to the clamped
    // candidate): a motion-free site whose pairs are a subset of that site's (*cur).
    // With zero motion its distance march returns 0 for a pair at distance 0 and NaN
    // for every other pair (L = 0, ccd.py:246-266), and its full-CCD results are never
    // read (stepper.py:587-592): the site reduces to "is some pair at distance 0", and
    // every such pair is in *cur, whose witness distances were computed at this very
    // anchor (same closest-point routines as the march's d0).  The pair set itself is
    // only needed by residual forwarding (stepper.py:604-610), whose trigger does not
    // depend on this site unless it reports penetration; so it is materialised only
    // then (or when sites are being verified, CS_VERIFY_STATIC_SITE).
    const bool rf_pre = toi_exit < cfg.eps_toi || (cap_hit && dx_last > cfg.eps_outer);
    if (!rf_pre && lazy_exit && std::getenv("CS_VERIFY_STATIC_SITE") == nullptr) {
        stage(T_FULL);
        CS_TRY(cudaMemsetAsync(d_iscal.p + I_FLAG, 0, sizeof(int), s));
        if (cur->P) {
            k_any_nonpositive<<<grid(cur->P), 256, 0, s>>>(cur->dist.p, cur->P, d_iscal.p + I_FLAG);
            ++launches;
            CS_CHECK_LAUNCH();
        }
        CS_RET(sync_scalars(__LINE__));
        if (h_iscal[I_FLAG]) return CS_PENETRATION;
        if (rep) {
            rep->full_ccd_calls += 1;
            rep->lazy_exit_sites += 1;
        }
    } else {
        CS_RET(ccd_site(anchor_w.p, anchor_w.p, *nxt, rep, tfin, cur));
    }
    CS_RET(set_clamp_value(tfin));
    CS_RET(lerp_world(anchor_w.p, xc_w.p, d_scal.p + S_CLAMP, tmp_w.p));  // tmp_w = x_final_w
    toi_exit = std::min(toi_exit, tfin);
    stage(-1);
    // ---- verify mode (stepper.py:614-621): the device intersection check replaces the
    // injected oracle; a failing step leaves the state untouched
    if (verify_on) {
        long long bad = 0;
        const int cap = 1024;
        CS_RET(intersections(tmp_w.p, bad, cap));
        last_isect = bad;
        last_isect_pairs.assign(2 * (size_t)std::min<long long>(bad, cap), 0);
        if (bad) {
            CS_TRY(cudaMemcpy(last_isect_pairs.data(), isect_out.p, sizeof(int) * last_isect_pairs.size(),
                              cudaMemcpyDeviceToHost));
            return CS_PENETRATION;
        }
    }
    // ---- residual forwarding (stepper.py:604-610) into the scratch dfn: it can
    // still fail (smoother divergence, allocation), and the reference raises
    // before `self.state = new_state`, leaving the state untouched
    const bool needs_rf = toi_exit < cfg.eps_toi || (cap_hit && dx_last > cfg.eps_outer);
    if (needs_rf) {
        stage(T_RF);
        CS_RET(residual_forward(tmp_w.p, rep));
        stage(-1);
    }
    // ---- new state (stepper.py:594-602), committed only after every check passed
    CS_TRY(cudaMemcpyAsync(xprev.p, x.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    k_velocity_update<<<grid(3LL * n), 256, 0, s>>>(tmp_w.p, x.p, v.p, 3LL * n, h);
    ++launches;
    CS_TRY(cudaMemcpyAsync(x.p, tmp_w.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    if (needs_rf)
        CS_TRY(cudaMemcpyAsync(df.p, dfn.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    else
        CS_TRY(cudaMemsetAsync(df.p, 0, sizeof(double) * 3 * n, s));
    if (nobs) CS_TRY(cudaMemcpyAsync(obs.p, tmp_w.p + 3LL * n, sizeof(double) * 3 * nobs, cudaMemcpyDeviceToDevice, s));
    CS_CHECK_LAUNCH();
    ++step_index;
    if (rep) {
        rep->lg_iterations = lg;
        rep->outer_loops = outer_loops;
        rep->partial_ccd_calls = partial_calls;
        rep->toi_exit = toi_exit;
        rep->cap_hit = cap_hit ? 1 : 0;
        rep->rf_triggered = needs_rf ? 1 : 0;
        rep->active_pairs = (int)active_pairs;
        rep->n_outer_deltas = n_deltas;
        rep->gpu_launches = launches;
        CS_TRY(hsync(__LINE__));
        rep->host_syncs = n_syncs;
        rep->stamp_plan_reuses = (int)(plan_reuses - plan_reuses0);
        double acc[kStages] = {0};
        for (auto& sp : spans) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, sp.second.first, sp.second.second);
            acc[sp.first] += ms;
        }
        rep->t_warm_start = acc[T_WARM];
        rep->t_local = acc[T_LOCAL];
        rep->t_global = acc[T_GLOBAL];
        rep->t_smoothing = acc[T_SMOOTH];
        rep->t_broad = acc[T_BROAD];
        rep->t_narrow_partial = acc[T_PARTIAL];
        rep->t_narrow_full = acc[T_FULL];
        rep->t_rf = acc[T_RF];
    }
    return 0;
}

int cs_scene::residual_forward(const double* xfw, cs_step_report* rep) {
    // exit pairs live in *nxt: witness at x_final_w, frozen weights (stepper.py:626-642)
    PairBuf& ex = *nxt;
    long long A = 0;
    CS_TRY(cudaMemsetAsync(d_iscal.p + I_ENG, 0, sizeof(int), s));
    if (ex.P) {
        CS_RET(witness(ex, xfw));
        k_rf_weights<<<grid(ex.P), 256, 0, s>>>(ex.dist.p, ex.P, cfg.d_hat, cfg.ndb_k, ex.engaged.p, ex.weight.p);
        k_count_true<<<grid(ex.P), 256, 0, s>>>(ex.engaged.p, ex.P, d_iscal.p + I_ENG);
        launches += 2;
        CS_RET(sync_scalars(__LINE__));
        A = h_iscal[I_ENG];
    }
    CS_RET(stamps(ex, A, xfw));
    // f_r = -grad E at x_final (quad collision form), delta from stamps
    // cloth rows of x_final_w (the state is not committed yet)
    k_energy_grad<<<grid(n), 256, 0, s>>>(n, xfw, z.p, mass.p, cfg.h, edges(), ginc_ptr.p, ginc.p,
                                          BendSet{st.p, bk.p, bw.p}, binc_ptr.p, binc.p, free_index.p,
                                          stamps_valid ? seg_beg.p : nullptr, seg_end.p, ssrc_s.p, stamp.p,
                                          grad.p);
    k_neg_gather<<<grid(nf), 256, 0, s>>>(grad.p, free_ids.p, nf, fr.p);
    k_stamp_delta<<<grid(nf), 256, 0, s>>>(nf, stamps_valid ? seg_beg.p : nullptr, seg_end.p, ssrc_s.p, stamp.p,
                                           delta.p);
    launches += 3;
    CS_CHECK_LAUNCH();
    CS_TRY(cudaMemsetAsync(xf.p, 0, sizeof(double) * 3 * nf, s));
    CS_RET(sqnorm(fr.p, nullptr, nf, nullptr, S_NORM_F));
    for (int it = 0; it < cfg.rf_iterations; ++it) {
        CS_RET(reduced(fr.p, xf.p, delta.p, it == 0, stamps_valid ? n_stamp_rows : 0));
        CS_RET(smooth(fr.p, xf.p, cfg.smoothing_iterations, cfg.omega, delta.p));
        // resid = f_r - H dx - delta dx ; ||resid|| <= tol * max(||f_r||, 1e-30)
        k_residual<<<grid(nf), 256, 0, s>>>(sell(), fr.p, xf.p, delta.p, t.p);
        ++launches;
        CS_RET(sqnorm(t.p, nullptr, nf, nullptr, S_RES));
        CS_RET(sync_scalars(__LINE__));
        if (h_scal[S_RES] <= cfg.rf_tolerance * std::max(h_scal[S_NORM_F], 1e-30)) break;
    }
    CS_TRY(cudaMemsetAsync(dfn.p, 0, sizeof(double) * 3 * n, s));
    k_forward_force<<<grid(nf), 256, 0, s>>>(xf.p, free_ids.p, nf, mass.p, cfg.h, dfn.p);
    ++launches;
    CS_RET(sqnorm(dfn.p, nullptr, n, nullptr, S_DFNORM));
    CS_RET(sync_scalars(__LINE__));
    const double nrm = h_scal[S_DFNORM];
    if (nrm > cfg.delta_f_cap) {
        h_scal[S_DFSCALE] = cfg.delta_f_cap / nrm;
        CS_TRY(cudaMemcpyAsync(d_scal.p + S_DFSCALE, &h_scal[S_DFSCALE], sizeof(double), cudaMemcpyHostToDevice, s));
        k_scale<<<grid(3LL * n), 256, 0, s>>>(dfn.p, 3LL * n, d_scal.p + S_DFSCALE);
        ++launches;
    }
    CS_CHECK_LAUNCH();
    if (rep) {
        CS_TRY(cudaMemcpyAsync(&h_iscal[I_FALLBACK], fallback.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CS_TRY(hsync(__LINE__));
        rep->reduced_fallbacks += h_iscal[I_FALLBACK];
    }
    return 0;
}

// ============================================================ C ABI
extern "C" {

const char* cs_version(void) { return "clothsim_b200 0.1 sm_100a fp64"; }

// OBJ vertex block "v %.9f %.9f %.9f\n" (reference mesh.py:220-226; glibc printf and
// Python's float formatting both round correctly, so the text is identical),
// formatted by up to 16 host threads.  Returns the byte count, or -1 if cap is short.
long long cs_format_obj_vertices(const double* v, long long n, char* out, long long cap) {
    if (n < 0 || (n > 0 && (!v || !out))) return -1;
    const int nt = (int)std::max<long long>(1, std::min<long long>(16, n / 8192));
    std::vector<std::string> parts(nt);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            const long long a = n * t / nt, b = n * (t + 1) / nt;
            std::string& o = parts[t];
            o.reserve((size_t)(b - a) * 48);
            char line[160];
            for (long long i = a; i < b; ++i) {
                const int k = std::snprintf(line, sizeof(line), "v %.9f %.9f %.9f\n", v[3 * i], v[3 * i + 1],
                                            v[3 * i + 2]);
                o.append(line, (size_t)std::min<int>(k, (int)sizeof(line) - 1));
            }
        });
    for (auto& t : th) t.join();
    long long total = 0;
    for (auto& p : parts) total += (long long)p.size();
    if (total > cap) return -1;
    long long o = 0;
    for (auto& p : parts) {
        std::memcpy(out + o, p.data(), p.size());
        o += (long long)p.size();
    }
    return total;
}

cs_scene* cs_scene_create(const cs_scene_desc* desc, const cs_step_config* cfg, int* status) {
    if (desc) {
        // map a slab into the library pool once per process and device, so pair-buffer
        // regrowth under contact is served without mapping fresh memory (a mapping of a few
        // GB stalls the stream for hundreds of ms): ~32 KB per world primitive (pair sets
        // of up to ~50 M pairs, grid tables, stamps and the stamp plan at the bench's
        // contact density), at most a third of the free memory; CS_POOL_RESERVE_GB
        // overrides (0 = none)
        static bool reserved[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool = lib_pool();
        if (pool && dev >= 0 && dev < 64 && !reserved[dev]) {
            reserved[dev] = true;
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            const char* env = std::getenv("CS_POOL_RESERVE_GB");
            const size_t prims = (size_t)std::max(desc->n_world_tris, 0) + (size_t)std::max(desc->n_world_edges, 0);
            size_t want = env ? (size_t)(std::atof(env) * (1ull << 30)) : std::min<size_t>(32768 * prims, free_b / 3);
            void* slab = nullptr;
            if (want && cudaMallocFromPoolAsync(&slab, want, pool, nullptr) == cudaSuccess) {
                cudaFreeAsync(slab, nullptr);
                cudaStreamSynchronize(nullptr);
            }
            cudaGetLastError();
        }
    }
    return cs_scene_create_parts(desc, cfg, CS_PART_ALL, status);
}

cs_scene* cs_scene_create_parts(const cs_scene_desc* desc, const cs_step_config* cfg, int parts, int* status) {
    if (!desc || !cfg) {
        if (status) *status = CS_BAD_ARGUMENT;
        return nullptr;
    }
    t_alloc_stream = nullptr;
    cs_scene* sc = new cs_scene();
    int rc = sc->create(desc, cfg, parts);
    if (status) *status = rc;
    if (rc != 0) {
        sc->release();
        delete sc;
        return nullptr;
    }
    return sc;
}

void cs_scene_destroy(cs_scene* scene) {
    if (!scene) return;
    cudaDeviceSynchronize();
    scene->release();
    delete scene;
}

int cs_scene_set_config(cs_scene* scene, const cs_step_config* cfg) {
    if (!scene || !cfg) return CS_BAD_ARGUMENT;
    scene->cfg = *cfg;
    scene->set_pattern();
    return 0;
}

int cs_step(cs_scene* scene, const double* pin_next, const double* obstacle_next, cs_step_report* report,
            void* stream) {
    if (scene && !scene->has(CS_PART_ALL)) return CS_BAD_ARGUMENT;
    if (!scene) return CS_BAD_ARGUMENT;
    static const bool trace_host = std::getenv("CS_TRACE_HOST") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (report) std::memset(report, 0, sizeof(*report));
    scene->s = (cudaStream_t)stream;
    t_alloc_stream = scene->s;
    int rc = scene->step(pin_next, obstacle_next, report);
    scene->stage(-1);
    if (trace_host) {
        const auto t1 = std::chrono::steady_clock::now();
        static auto last = t1;
        std::fprintf(stderr, "[cs host] step %.1f us, since previous exit %.1f us\n",
                     std::chrono::duration<double, std::micro>(t1 - t0).count(),
                     std::chrono::duration<double, std::micro>(t0 - last).count());
        last = t1;
    }
    return rc;
}

int cs_get_state(cs_scene* sc, double* x, double* x_dot, double* x_prev, double* delta_f, double* obstacle_x,
                 int* step_index, void* stream) {
    if (sc && !sc->has(CS_PART_ALL)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    const size_t nb = sizeof(double) * 3 * sc->n;
    if (x) CS_TRY(cudaMemcpyAsync(x, sc->x.p, nb, cudaMemcpyDeviceToHost, s));
    if (x_dot) CS_TRY(cudaMemcpyAsync(x_dot, sc->v.p, nb, cudaMemcpyDeviceToHost, s));
    if (x_prev) CS_TRY(cudaMemcpyAsync(x_prev, sc->xprev.p, nb, cudaMemcpyDeviceToHost, s));
    if (delta_f) CS_TRY(cudaMemcpyAsync(delta_f, sc->df.p, nb, cudaMemcpyDeviceToHost, s));
    if (obstacle_x && sc->nobs)
        CS_TRY(cudaMemcpyAsync(obstacle_x, sc->obs.p, sizeof(double) * 3 * sc->nobs, cudaMemcpyDeviceToHost, s));
    if (step_index) *step_index = sc->step_index;
    CS_TRY(cudaStreamSynchronize(s));
    return 0;
}

int cs_set_state(cs_scene* sc, const double* x, const double* x_dot, const double* x_prev, const double* delta_f,
                 const double* obstacle_x, int step_index, void* stream) {
    if (sc && !sc->has(CS_PART_ALL)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    const size_t nb = sizeof(double) * 3 * sc->n;
    if (x) CS_TRY(cudaMemcpyAsync(sc->x.p, x, nb, cudaMemcpyHostToDevice, s));
    if (x_dot) CS_TRY(cudaMemcpyAsync(sc->v.p, x_dot, nb, cudaMemcpyHostToDevice, s));
    if (x_prev) CS_TRY(cudaMemcpyAsync(sc->xprev.p, x_prev, nb, cudaMemcpyHostToDevice, s));
    if (delta_f) CS_TRY(cudaMemcpyAsync(sc->df.p, delta_f, nb, cudaMemcpyHostToDevice, s));
    if (obstacle_x && sc->nobs)
        CS_TRY(cudaMemcpyAsync(sc->obs.p, obstacle_x, sizeof(double) * 3 * sc->nobs, cudaMemcpyHostToDevice, s));
    if (step_index >= 0) sc->step_index = step_index;
    CS_TRY(cudaStreamSynchronize(s));
    return 0;
}

int cs_state_device(cs_scene* sc, double** x, double** x_dot, double** delta_f, double** obstacle_x) {
    if (sc && !sc->has(CS_PART_ALL)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    if (x) *x = sc->x.p;
    if (x_dot) *x_dot = sc->v.p;
    if (delta_f) *delta_f = sc->df.p;
    if (obstacle_x) *obstacle_x = sc->obs.p;
    return 0;
}

// Frame output without stalling the step loop (reference cli.py:64-98 writes a
// frame every frame_stride steps): the positions are snapshotted on the caller's
// stream into one of two device slots (an 8 MB D2D at config 4), and the slot is
// copied to the caller's page-locked buffer on a separate copy stream while the
// next steps run.  cs_frame_wait(ticket) blocks until that copy has landed.
int cs_frame_async(cs_scene* sc, double* host_x, int* ticket, void* stream) {
    if (sc && !sc->has(CS_PART_ALL)) return CS_BAD_ARGUMENT;
    if (!sc || !host_x || !ticket) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    if (!sc->copy_stream) CS_TRY(cudaStreamCreateWithFlags(&sc->copy_stream, cudaStreamNonBlocking));
    const int k = sc->frame_next;
    cs_scene::FrameSlot& f = sc->frame_slots[k];
    if (!f.taken) {
        CS_TRY(cudaEventCreateWithFlags(&f.taken, cudaEventDisableTiming));
        CS_TRY(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
    }
    const size_t nb = sizeof(double) * 3 * sc->n;
    CS_RET(f.x.ensure(3LL * sc->n, true));
    if (f.used) CS_TRY(cudaStreamWaitEvent(s, f.done, 0));  // the slot's previous copy has left it
    CS_TRY(cudaMemcpyAsync(f.x.p, sc->x.p, nb, cudaMemcpyDeviceToDevice, s));
    CS_TRY(cudaEventRecord(f.taken, s));
    CS_TRY(cudaStreamWaitEvent(sc->copy_stream, f.taken, 0));
    CS_TRY(cudaMemcpyAsync(host_x, f.x.p, nb, cudaMemcpyDeviceToHost, sc->copy_stream));
    CS_TRY(cudaEventRecord(f.done, sc->copy_stream));
    f.used = true;
    sc->frame_next = k ^ 1;
    *ticket = k;
    return 0;
}

int cs_frame_wait(cs_scene* sc, int ticket) {
    if (!sc || ticket < 0 || ticket > 1) return CS_BAD_ARGUMENT;
    cs_scene::FrameSlot& f = sc->frame_slots[ticket];
    if (f.used) CS_TRY(cudaEventSynchronize(f.done));
    return 0;
}

int cs_full_ccd(const int8_t* kind, const int* idx4, const double* x_start, const double* x_end, long long P,
                double tol, double* toi, void* stream) {
    if (P < 0) return CS_BAD_ARGUMENT;
    if (P == 0) return 0;
    k_full_ccd<<<(int)((P + 127) / 128), 128, 0, (cudaStream_t)stream>>>(kind, (const int4*)idx4, x_start, x_end, P,
                                                                         P == 1 ? 1 : 0, tol, toi);
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_distance_toi(const int8_t* kind, const int* idx4, const double* x_start, const double* x_end, long long P,
                    double floor_frac, int max_iterations, double* toi, void* stream) {
    if (P < 0) return CS_BAD_ARGUMENT;
    if (P == 0) return 0;
    k_distance_toi<<<(int)((P + 127) / 128), 128, 0, (cudaStream_t)stream>>>(kind, (const int4*)idx4, x_start, x_end,
                                                                             P, floor_frac, max_iterations, toi);
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_partial_ccd(const int8_t* kind, const int* idx4, const double* x_start, const double* x_end, long long P,
                   int samples, uint8_t* active, void* stream) {
    if (P < 0 || (samples != 1 && samples != 3 && samples != 6)) return CS_BAD_ARGUMENT;
    if (P == 0) return 0;
    cs_scene tmp;
    tmp.cfg.samples = samples;
    tmp.set_pattern();
    // classification only: feed an impossible gap so the NDB half leaves `active` untouched
    DBuf<double> bary, normal, weight;
    DBuf<int> life;
    DBuf<uint8_t> eng;
    CS_RET(bary.ensure(2 * P));
    CS_RET(normal.ensure(3 * P));
    CS_RET(weight.ensure(P));
    CS_RET(life.ensure(P));
    CS_RET(eng.ensure(P));
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    CS_TRY(cudaMemsetAsync(bary.p, 0, sizeof(double) * 2 * P, s));
    CS_TRY(cudaMemsetAsync(normal.p, 0, sizeof(double) * 3 * P, s));
    CS_TRY(cudaMemsetAsync(life.p, 0, sizeof(int) * P, s));
    const NdbArgs na{kind, (const int4*)idx4, x_start, x_end, tmp.pat, bary.p, normal.p, -1.0, 1.0, 2.0,
                     life.p, weight.p, eng.p, 1, active, 0, nullptr};
    k_partial_ndb<<<(int)((P + 127) / 128), 128, 0, s>>>(na, P, nullptr, PlanView{}, nullptr);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(s));
    bary.release();
    normal.release();
    weight.release();
    life.release();
    eng.release();
    return 0;
}

int cs_pair_witness(const int8_t* kind, const int* idx4, const double* x, long long P, double* p1, double* p2,
                    double* bary, double* dist, double* normal, void* stream) {
    if (P < 0) return CS_BAD_ARGUMENT;
    if (P == 0) return 0;
    k_witness<<<(int)((P + 127) / 128), 128, 0, (cudaStream_t)stream>>>(kind, (const int4*)idx4, x, P, bary, dist,
                                                                        normal, p1, p2, EngageOut{});
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_broad_phase(cs_scene* sc, const double* x_start_w, const double* x_end_w, double margin, long long* count,
                   void* stream) {
    if (sc && !sc->has(CS_PART_WORLD)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    CS_RET(sc->broad_phase(x_start_w, x_end_w, margin, *sc->cur));
    if (count) *count = sc->cur->P;
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

int cs_ccd_site(cs_scene* sc, const double* x_start_w, const double* x_end_w, long long* count, double* clamp,
                void* stream) {
    if (sc && !sc->has(CS_PART_WORLD)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    double c = 1.0;
    const int rc = sc->ccd_site(x_start_w, x_end_w, *sc->cur, nullptr, c);
    if (count) *count = sc->cur->P;
    if (clamp) *clamp = c;
    CS_TRY(cudaStreamSynchronize(sc->s));
    return rc;
}

int cs_scene_pair_results(cs_scene* sc, double* toi, double* toi_filter, void* stream) {
    if (sc && !sc->has(CS_PART_WORLD)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    const long long P = sc->cur->P;
    if (P == 0) return 0;
    if (toi) CS_TRY(cudaMemcpyAsync(toi, sc->cur->toi.p, sizeof(double) * P, cudaMemcpyDeviceToDevice, s));
    if (toi_filter) CS_TRY(cudaMemcpyAsync(toi_filter, sc->cur->filt.p, sizeof(double) * P, cudaMemcpyDeviceToDevice, s));
    return 0;
}

int cs_scene_set_verify(cs_scene* sc, int on) {
    if (!sc) return CS_BAD_ARGUMENT;
    sc->verify_on = on != 0;
    return 0;
}

int cs_intersections(cs_scene* sc, const double* x_world, long long* count, int* pairs, int cap, void* stream) {
    if (sc && !sc->has(CS_PART_WORLD)) return CS_BAD_ARGUMENT;
    if (!sc || cap < 0) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    const double* xw = x_world;
    if (!xw) {  // current world state
        CS_TRY(cudaMemcpyAsync(sc->tmp_w.p, sc->x.p, sizeof(double) * 3 * sc->n, cudaMemcpyDeviceToDevice, sc->s));
        if (sc->nobs)
            CS_TRY(cudaMemcpyAsync(sc->tmp_w.p + 3LL * sc->n, sc->obs.p, sizeof(double) * 3 * sc->nobs,
                                   cudaMemcpyDeviceToDevice, sc->s));
        xw = sc->tmp_w.p;
    }
    long long bad = 0;
    CS_RET(sc->intersections(xw, bad, cap));
    if (count) *count = bad;
    if (pairs && bad)
        CS_TRY(cudaMemcpy(pairs, sc->isect_out.p, sizeof(int) * 2 * std::min<long long>(bad, cap),
                          cudaMemcpyDeviceToHost));
    return 0;
}

int cs_last_intersections(cs_scene* sc, long long* count, int* pairs, int cap, double* x_final) {
    if (!sc || cap < 0) return CS_BAD_ARGUMENT;
    if (count) *count = sc->last_isect;
    if (pairs) {
        const size_t k = std::min<size_t>(sc->last_isect_pairs.size() / 2, (size_t)cap);
        std::memcpy(pairs, sc->last_isect_pairs.data(), sizeof(int) * 2 * k);
    }
    if (x_final) CS_TRY(cudaMemcpy(x_final, sc->tmp_w.p, sizeof(double) * 3 * sc->n, cudaMemcpyDeviceToHost));
    return 0;
}

int cs_scene_pairs(cs_scene* sc, int8_t* kind, int* idx4, void* stream) {
    if (sc && !sc->has(CS_PART_WORLD)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    t_alloc_stream = s;
    const long long P = sc->cur->P;
    if (P == 0) return 0;
    if (kind) CS_TRY(cudaMemcpyAsync(kind, sc->cur->kind.p, P, cudaMemcpyDeviceToDevice, s));
    if (idx4) CS_TRY(cudaMemcpyAsync(idx4, sc->cur->idx.p, sizeof(int4) * P, cudaMemcpyDeviceToDevice, s));
    return 0;
}

int cs_assemble_rhs(cs_scene* sc, const double* z, const double* x, const double* pins, const int* coll_ids,
                    const double* coll_w, const double* coll_t, int n_coll, double* b, double* delta, void* stream) {
    if (sc && !sc->has(CS_PART_CLOTH | CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    cudaStream_t s = sc->s;
    bool with = false;
    CS_TRY(cudaMemsetAsync(sc->seg_beg.p, 0, sizeof(int) * sc->nf, s));
    CS_TRY(cudaMemsetAsync(sc->seg_end.p, 0, sizeof(int) * sc->nf, s));
    if (n_coll > 0) {
        const int m = n_coll;
        CS_RET(sc->skey.ensure(m));
        CS_RET(sc->ssrc.ensure(m));
        CS_RET(sc->skey_s.ensure(m));
        CS_RET(sc->ssrc_s.ensure(m));
        sc->plan_valid = false;
        CS_RET(sc->stamp.ensure(m));
        CS_RET(sc->rowflag.ensure(m));
        k_pack_stamps<<<sc->grid(m), 256, 0, s>>>(coll_w, coll_t, m, sc->stamp.p);
        k_stamp_keys<<<sc->grid(m), 256, 0, s>>>(coll_ids, m, sc->free_index.p, sc->n, sc->skey.p);
        k_iota<<<sc->grid(m), 256, 0, s>>>(sc->ssrc.p, m);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, sc->skey.p, sc->skey_s.p, sc->ssrc.p, sc->ssrc_s.p, m, 0, 31, s);
        CS_RET(sc->cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceRadixSort::SortPairs(sc->cub_tmp.p, bytes, sc->skey.p, sc->skey_s.p, sc->ssrc.p,
                                               sc->ssrc_s.p, m, 0, 31, s));
        CS_TRY(cudaMemsetAsync(sc->rowflag.p, 0, sizeof(int) * m, s));
        k_mark_segments<<<sc->grid(m), 256, 0, s>>>(sc->skey_s.p, m, sc->nf, sc->seg_beg.p, sc->seg_end.p, sc->rowflag.p);
        CS_CHECK_LAUNCH();
        with = true;
    }
    k_assemble_rhs<<<sc->grid(sc->nf), 256, 0, s>>>(sc->nf, sc->free_ids.p, x, z, sc->mh2.p, sc->edges(),
                                                    sc->rinc_ptr.p, sc->rinc.p, sc->has_fp ? sc->hfp_ptr.p : nullptr,
                                                    sc->hfp_col.p, sc->hfp_val.p, pins ? pins : x,
                                                    with ? sc->seg_beg.p : nullptr, sc->seg_end.p, sc->ssrc_s.p,
                                                    sc->stamp.p, b, delta, StampSide{});
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(s));
    return 0;
}

int cs_collision_terms(cs_scene* sc, const int8_t* kind, const int* idx4, const double* bary, const double* normal,
                       const double* weight, const uint8_t* engaged, long long P, const double* x_world, int* ids,
                       double* w, double* targets, long long* count, void* stream) {
    if (sc && !sc->has(CS_PART_CLOTH | CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc || P < 0) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    cudaStream_t s = sc->s;
    if (count) *count = 0;
    if (P == 0) return 0;
    // engaged & weight > 0, in pair order (stepper.py:245)
    CS_RET(sc->keep_flag.ensure(P));
    CS_TRY(cudaMemsetAsync(sc->d_iscal.p + I_FLAG, 0, sizeof(int), s));
    k_flag_engaged<<<sc->grid(P), 256, 0, s>>>(engaged, weight, P, sc->keep_flag.p, sc->d_iscal.p + I_FLAG);
    CS_RET(sc->sel.ensure(P));
    size_t bytes = 0;
    cub::CountingInputIterator<int> it(0);
    cub::DeviceSelect::Flagged(nullptr, bytes, it, sc->keep_flag.p, sc->sel.p, sc->d_iscal.p + I_FLAG, (int)P, s);
    CS_RET(sc->cub_tmp.ensure(bytes));
    CS_TRY(cub::DeviceSelect::Flagged(sc->cub_tmp.p, bytes, it, sc->keep_flag.p, sc->sel.p, sc->d_iscal.p + I_FLAG,
                                      (int)P, s));
    CS_TRY(cudaMemcpyAsync(&sc->h_iscal[I_FLAG], sc->d_iscal.p + I_FLAG, sizeof(int), cudaMemcpyDeviceToHost, s));
    CS_TRY(cudaStreamSynchronize(s));
    const long long A = sc->h_iscal[I_FLAG];
    if (A == 0) return 0;
    const long long m = 4 * A;
    CS_RET(sc->skey.ensure(m));
    sc->plan_valid = false;
    CS_RET(sc->stamp.ensure(m));
    CS_RET(sc->rowflag.ensure(m));
    CS_RET(sc->rows_act.ensure(m));
    k_collision_terms<<<sc->grid(A), 256, 0, s>>>(sc->sel.p, A, kind, (const int4*)idx4, x_world, bary, normal, weight,
                                                  sc->cfg.d_hat, sc->n, sc->free_index.p, 0, sc->skey.p,
                                                  sc->stamp.p, nullptr, nullptr);
    CS_RET(sc->keep_flag.ensure(m));
    k_key_kept<<<sc->grid(m), 256, 0, s>>>(sc->skey.p, (int)m, sc->nf, sc->keep_flag.p);
    bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, bytes, it, sc->keep_flag.p, sc->rows_act.p, sc->d_iscal.p + I_FLAG, (int)m, s);
    CS_RET(sc->cub_tmp.ensure(bytes));
    CS_TRY(cub::DeviceSelect::Flagged(sc->cub_tmp.p, bytes, it, sc->keep_flag.p, sc->rows_act.p,
                                      sc->d_iscal.p + I_FLAG, (int)m, s));
    k_gather_terms<<<std::max(1, std::min(sc->grid(m), 16 * sc->sm_count)), 256, 0, s>>>(
        sc->rows_act.p, sc->d_iscal.p + I_FLAG, sc->sel.p, (const int4*)idx4, sc->stamp.p, ids, w, targets);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaMemcpyAsync(&sc->h_iscal[I_FLAG], sc->d_iscal.p + I_FLAG, sizeof(int), cudaMemcpyDeviceToHost, s));
    CS_TRY(cudaStreamSynchronize(s));
    if (count) *count = sc->h_iscal[I_FLAG];
    return 0;
}

int cs_residual(cs_scene* sc, const double* b, const double* x, const double* delta, double* r, void* stream) {
    if (sc && !sc->has(CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc || !delta) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    k_residual<<<sc->grid(sc->nf), 256, 0, sc->s>>>(sc->sell(), b, x, delta, r);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

int cs_ajacobi_smooth(cs_scene* sc, const double* b, double* x, int iterations, double omega, const double* delta,
                      void* stream) {
    if (sc && !sc->has(CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    const double* dl = delta;
    if (dl == nullptr) {
        CS_TRY(cudaMemsetAsync(sc->delta.p, 0, sizeof(double) * sc->nf, sc->s));
        dl = sc->delta.p;
    }
    CS_RET(sc->smooth(b, x, iterations, omega, dl));
    return sc->sync_scalars();  // includes the residual-norm divergence check
}

int cs_reduced_correction(cs_scene* sc, const double* b, double* x, const double* delta, int reuse, void* stream) {
    if (sc && !sc->has(CS_PART_SYSTEM | CS_PART_BASIS)) return CS_BAD_ARGUMENT;
    if (!sc || !delta) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    int rows = 0;
    if (!reuse) {
        // active rows = flatnonzero(delta) (subspace.py:182)
        CS_RET(sc->rows_act.ensure(sc->nf));
        CS_RET(sc->rowflag.ensure(sc->nf));
        k_nonzero_flags<<<sc->grid(sc->nf), 256, 0, sc->s>>>(delta, sc->nf, sc->rowflag.p);
        size_t bytes = 0;
        cub::CountingInputIterator<int> it(0);
        cub::DeviceSelect::Flagged(nullptr, bytes, it, sc->rowflag.p, sc->rows_act.p, sc->d_iscal.p + I_ROWS, sc->nf,
                                   sc->s);
        CS_RET(sc->cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceSelect::Flagged(sc->cub_tmp.p, bytes, it, sc->rowflag.p, sc->rows_act.p,
                                          sc->d_iscal.p + I_ROWS, sc->nf, sc->s));
        rows = sc->nf;
    }
    CS_RET(sc->reduced(b, x, delta, !reuse, rows));
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

// jacobi_step (smoothing.py:69-78): out = x + (1 - omega) D^-1 (b - (H + delta) x)
int cs_jacobi_step(cs_scene* sc, const double* b, const double* x, double omega, const double* delta, double* out,
                   void* stream) {
    if (sc && !sc->has(CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    const double* dl = delta;
    if (dl == nullptr) {
        CS_TRY(cudaMemsetAsync(sc->delta.p, 0, sizeof(double) * sc->nf, sc->s));
        dl = sc->delta.p;
    }
    k_jacobi_a<<<sc->grid(sc->nf, 128), 128, 0, sc->s>>>(sc->sell(), sc->diag.p, dl, b, x, sc->t.p, nullptr);
    k_axpy_step<<<sc->grid(3LL * sc->nf), 256, 0, sc->s>>>(x, sc->t.p, 1.0 - omega, 3LL * sc->nf, out);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

// reduced_update (subspace.py:97-106): G (r*r) = sum_j w_j V_j V_j^T over rows[j] (DEVICE)
int cs_reduced_update(cs_scene* sc, const int* rows, const double* weights, int m, double* G, void* stream) {
    if (sc && !sc->has(CS_PART_BASIS)) return CS_BAD_ARGUMENT;
    if (!sc || m < 0) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    const int r = sc->r;
    if (m == 0) {
        CS_TRY(cudaMemsetAsync(G, 0, sizeof(double) * r * r, sc->s));
        return 0;
    }
    CS_TRY(cudaMemcpyAsync(sc->d_iscal.p + I_FLAG, &m, sizeof(int), cudaMemcpyHostToDevice, sc->s));
    const int gg = std::min(cs_div_up(m, 64), 2 * sc->sm_count);
    CS_RET(sc->part2.ensure((size_t)gg * r * r));
    k_gram_partial<<<gg, kGramThreads, 0, sc->s>>>(rows, sc->d_iscal.p + I_FLAG, nullptr, sc->V.p, r, sc->part2.p,
                                                   weights);
    k_reduce_partials<<<cs_div_up(r * r, 32), 256, 0, sc->s>>>(sc->part2.p, gg, r * r, G);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

// build_reduced (subspace.py:122-140): A = diag(lambda_r) + G (G DEVICE r*r, may be NULL),
// beta = rhs_scale (1 if <= 0), inverse X with A X = I / beta (LU, pinv fallback) ->
// inverse (DEVICE r*r); beta / fallback (HOST).  The context keeps it as its current
// reduced system (cs_reduced_correction with reuse != 0 applies it).
int cs_build_reduced(cs_scene* sc, const double* G, double rhs_scale, double* inverse, double* beta, int* fallback,
                     void* stream) {
    if (sc && !sc->has(CS_PART_BASIS)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    ReducedState rs{sc->Xred.p, sc->beta_red.p, sc->fallback.p};
    k_reduced_solve<<<1, 256, 0, sc->s>>>(sc->rhs_red.p, G, sc->lam.p, sc->r, 0, 1, rs, sc->q.p,
                                           rhs_scale > 0.0 ? rhs_scale : 0.0);
    CS_CHECK_LAUNCH();
    return cs_reduced_get(sc, inverse, beta, fallback, stream);
}

// the context's current reduced system (after cs_reduced_correction / cs_build_reduced)
int cs_reduced_get(cs_scene* sc, double* inverse, double* beta, int* fallback, void* stream) {
    if (sc && !sc->has(CS_PART_BASIS)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    const int r = sc->r;
    if (inverse) CS_TRY(cudaMemcpyAsync(inverse, sc->Xred.p, sizeof(double) * r * r, cudaMemcpyDeviceToDevice, s));
    if (beta) CS_TRY(cudaMemcpyAsync(beta, sc->beta_red.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (fallback) CS_TRY(cudaMemcpyAsync(fallback, sc->fallback.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CS_TRY(cudaStreamSynchronize(s));
    return 0;
}

int cs_warmstart_correction(cs_scene* sc, const double* b, double* x, void* stream) {
    if (sc && !sc->has(CS_PART_SYSTEM | CS_PART_BASIS)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    CS_RET(sc->warm_correction(b, x));
    CS_TRY(cudaStreamSynchronize(sc->s));
    return 0;
}

int cs_energy_gradient(cs_scene* sc, const double* x, const double* z, const int* q_ids, const double* q_w,
                       const double* q_t, int n_q, double* grad, void* stream) {
    if (sc && !sc->has(CS_PART_CLOTH | CS_PART_SYSTEM)) return CS_BAD_ARGUMENT;
    if (!sc) return CS_BAD_ARGUMENT;
    sc->s = (cudaStream_t)stream;
    t_alloc_stream = sc->s;
    cudaStream_t s = sc->s;
    bool with = false;
    CS_TRY(cudaMemsetAsync(sc->seg_beg.p, 0, sizeof(int) * sc->nf, s));
    CS_TRY(cudaMemsetAsync(sc->seg_end.p, 0, sizeof(int) * sc->nf, s));
    if (n_q > 0) {
        const int m = n_q;
        CS_RET(sc->skey.ensure(m));
        CS_RET(sc->ssrc.ensure(m));
        CS_RET(sc->skey_s.ensure(m));
        CS_RET(sc->ssrc_s.ensure(m));
        sc->plan_valid = false;
        CS_RET(sc->stamp.ensure(m));
        CS_RET(sc->rowflag.ensure(m));
        k_pack_stamps<<<sc->grid(m), 256, 0, s>>>(q_w, q_t, m, sc->stamp.p);
        k_stamp_keys<<<sc->grid(m), 256, 0, s>>>(q_ids, m, sc->free_index.p, sc->n, sc->skey.p);
        k_iota<<<sc->grid(m), 256, 0, s>>>(sc->ssrc.p, m);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, sc->skey.p, sc->skey_s.p, sc->ssrc.p, sc->ssrc_s.p, m, 0, 31, s);
        CS_RET(sc->cub_tmp.ensure(bytes));
        CS_TRY(cub::DeviceRadixSort::SortPairs(sc->cub_tmp.p, bytes, sc->skey.p, sc->skey_s.p, sc->ssrc.p,
                                               sc->ssrc_s.p, m, 0, 31, s));
        CS_TRY(cudaMemsetAsync(sc->rowflag.p, 0, sizeof(int) * m, s));
        k_mark_segments<<<sc->grid(m), 256, 0, s>>>(sc->skey_s.p, m, sc->nf, sc->seg_beg.p, sc->seg_end.p, sc->rowflag.p);
        with = true;
    }
    k_energy_grad<<<sc->grid(sc->n), 256, 0, s>>>(sc->n, x, z, sc->mass.p, sc->cfg.h, sc->edges(), sc->ginc_ptr.p,
                                                  sc->ginc.p, BendSet{sc->st.p, sc->bk.p, sc->bw.p}, sc->binc_ptr.p,
                                                  sc->binc.p, sc->free_index.p, with ? sc->seg_beg.p : nullptr,
                                                  sc->seg_end.p, sc->ssrc_s.p, sc->stamp.p, grad);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(s));
    return 0;
}

}  // extern "C"

// ------------------------------------------------------------------ device eigensolver (setup)
// Block kernels of the Chebyshev-filtered subspace iteration (eigen.cu) on an opaque
// context holding H (CSR) and nb row-major n x pp blocks; eigen.py drives it.
struct cs_eig {
    int n = 0, p = 0, pp = 0;
    DBuf<int> indptr, indices;
    DBuf<double> data, part, red, S, w;
    std::vector<DBuf<double>> blk;
    cudaStream_t s = nullptr;
    int grid_rows(int rows_per_block) const { return std::max(1, (n + rows_per_block - 1) / rows_per_block); }
    int spmm(int src, int dst, int prev, int mode, double c, double s1, double s2) {
        const int g = std::max(1, (int)(((long long)n * 32 + 255) / 256));
        const double* X = blk[src].p;
        const double* Xp = prev >= 0 ? blk[prev].p : nullptr;
        double* Y = blk[dst].p;
#define CS_EIG_SPMM(NQ)                                                                                           \
    if (pp == 32 * NQ) {                                                                                          \
        if (mode == 0) k_blk_spmm<NQ, 0><<<g, 256, 0, s>>>(n, indptr.p, indices.p, data.p, X, Xp, pp, c, s1, s2, Y); \
        else if (mode == 1) k_blk_spmm<NQ, 1><<<g, 256, 0, s>>>(n, indptr.p, indices.p, data.p, X, Xp, pp, c, s1, s2, Y); \
        else k_blk_spmm<NQ, 2><<<g, 256, 0, s>>>(n, indptr.p, indices.p, data.p, X, Xp, pp, c, s1, s2, Y);     \
        return 0;                                                                                                 \
    }
        CS_EIG_SPMM(1) CS_EIG_SPMM(2) CS_EIG_SPMM(3) CS_EIG_SPMM(4) CS_EIG_SPMM(5) CS_EIG_SPMM(6) CS_EIG_SPMM(7)
        CS_EIG_SPMM(8)
#undef CS_EIG_SPMM
        return CS_BAD_ARGUMENT;
    }
};

extern "C" {

cs_eig* cs_eig_create(int n, const int* indptr, const int* indices, const double* data, int p, int nblocks,
                      int* status) {
    auto fail = [&](int st, cs_eig* e) -> cs_eig* {
        if (status) *status = st;
        delete e;
        return nullptr;
    };
    if (n <= 0 || p <= 0 || p > 256 || nblocks <= 0 || !indptr || !indices || !data) return fail(CS_BAD_ARGUMENT, nullptr);
    cs_eig* e = new cs_eig();
    e->n = n;
    e->p = p;
    e->pp = (p + 31) / 32 * 32;
    t_alloc_stream = nullptr;
    const long long nnz = indptr[n];
    int st = 0;
    if ((st = e->indptr.upload(indptr, (size_t)n + 1)) || (st = e->indices.upload(indices, (size_t)nnz)) ||
        (st = e->data.upload(data, (size_t)nnz)))
        return fail(st, e);
    e->blk.resize(nblocks);
    for (auto& b : e->blk) {
        if ((st = b.ensure((size_t)n * e->pp, true))) return fail(st, e);
        if (cudaMemset(b.p, 0, sizeof(double) * (size_t)n * e->pp) != cudaSuccess) return fail(CS_INTERNAL, e);
    }
    if ((st = e->S.ensure((size_t)e->pp * e->pp, true)) || (st = e->w.ensure(e->pp, true))) return fail(st, e);
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(CS_INTERNAL, e);
    if (status) *status = 0;
    return e;
}

int cs_eig_destroy(cs_eig* e) {
    if (!e) return 0;
    cudaDeviceSynchronize();
    for (auto& b : e->blk) b.release();
    e->indptr.release();
    e->indices.release();
    e->data.release();
    e->part.release();
    e->red.release();
    e->S.release();
    e->w.release();
    delete e;
    return 0;
}

static bool eig_ok(cs_eig* e, int b) { return e && b >= 0 && b < (int)e->blk.size(); }

// block <- host (n x p row-major); padding columns zero
int cs_eig_set(cs_eig* e, int b, const double* host, void* stream) {
    if (!eig_ok(e, b) || !host) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    CS_TRY(cudaMemsetAsync(e->blk[b].p, 0, sizeof(double) * (size_t)e->n * e->pp, e->s));
    CS_TRY(cudaMemcpy2DAsync(e->blk[b].p, sizeof(double) * e->pp, host, sizeof(double) * e->p, sizeof(double) * e->p,
                             e->n, cudaMemcpyHostToDevice, e->s));
    CS_TRY(cudaStreamSynchronize(e->s));
    return 0;
}

// host (n x cols row-major) <- first cols columns of block b
int cs_eig_get(cs_eig* e, int b, int cols, double* host, void* stream) {
    if (!eig_ok(e, b) || !host || cols <= 0 || cols > e->p) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    CS_TRY(cudaMemcpy2DAsync(host, sizeof(double) * cols, e->blk[b].p, sizeof(double) * e->pp, sizeof(double) * cols,
                             e->n, cudaMemcpyDeviceToHost, e->s));
    CS_TRY(cudaStreamSynchronize(e->s));
    return 0;
}

// dst = H src
int cs_eig_spmm(cs_eig* e, int src, int dst, void* stream) {
    if (!eig_ok(e, src) || !eig_ok(e, dst) || src == dst) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    CS_RET(e->spmm(src, dst, -1, 0, 0.0, 1.0, 0.0));
    CS_CHECK_LAUNCH();
    return 0;
}

// Chebyshev filter of degree `degree` damping [a, lam_max] (scaled at a0) applied to
// block x in place; w1, w2: scratch blocks (eigen.py: Y1 = (H X - c X) sigma / e,
// Y_{d+1} = (H Y_d - c Y_d) 2 s / e - sigma s Y_{d-1})
int cs_eig_filter(cs_eig* e, int x, int w1, int w2, int degree, double a, double lam_max, double a0, void* stream) {
    if (!eig_ok(e, x) || !eig_ok(e, w1) || !eig_ok(e, w2) || x == w1 || x == w2 || w1 == w2 || degree < 1)
        return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    const double ee = (lam_max - a) / 2.0, c = (lam_max + a) / 2.0;
    double sigma = ee / (a0 - c);
    const double tau = 2.0 / sigma;
    int bufs[3] = {x, w1, w2};
    int prev = 0, cur = 1;
    CS_RET(e->spmm(bufs[prev], bufs[cur], -1, 1, c, sigma / ee, 0.0));
    for (int d = 2; d <= degree; ++d) {
        const double s_new = 1.0 / (tau - sigma);
        const int nxt = 3 - prev - cur;
        CS_RET(e->spmm(bufs[cur], bufs[nxt], bufs[prev], 2, c, 2.0 * s_new / ee, sigma * s_new));
        prev = cur;
        cur = nxt;
        sigma = s_new;
    }
    if (bufs[cur] != x)
        CS_TRY(cudaMemcpyAsync(e->blk[x].p, e->blk[bufs[cur]].p, sizeof(double) * (size_t)e->n * e->pp,
                               cudaMemcpyDeviceToDevice, e->s));
    CS_CHECK_LAUNCH();
    return 0;
}

// exchange two block slots (no data movement)
int cs_eig_swap(cs_eig* e, int a, int b) {
    if (!eig_ok(e, a) || !eig_ok(e, b)) return CS_BAD_ARGUMENT;
    std::swap(e->blk[a], e->blk[b]);
    return 0;
}

// out (HOST p x p) = A^T B
int cs_eig_gram(cs_eig* e, int a, int b, double* out, void* stream) {
    if (!eig_ok(e, a) || !eig_ok(e, b) || !out) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    t_alloc_stream = e->s;
    const int pp = e->pp, nt = pp / 32;
    const int chunks = std::max(1, std::min(64, (e->n + 4095) / 4096));
    const int rpc = (e->n + chunks - 1) / chunks;
    CS_RET(e->part.ensure((size_t)chunks * pp * pp));
    CS_RET(e->red.ensure((size_t)pp * pp));
    k_blk_gram_partial<<<dim3(chunks, nt * nt), 256, 0, e->s>>>(e->n, pp, e->blk[a].p, e->blk[b].p, rpc, e->part.p);
    k_reduce_partials<<<cs_div_up(pp * pp, 32), 256, 0, e->s>>>(e->part.p, chunks, pp * pp, e->red.p);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaMemcpy2DAsync(out, sizeof(double) * e->p, e->red.p, sizeof(double) * pp, sizeof(double) * e->p, e->p,
                             cudaMemcpyDeviceToHost, e->s));
    CS_TRY(cudaStreamSynchronize(e->s));
    return 0;
}

// dst = src S (S HOST p x p row-major)
int cs_eig_mul(cs_eig* e, int src, const double* S, int dst, void* stream) {
    if (!eig_ok(e, src) || !eig_ok(e, dst) || src == dst || !S) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    const int pp = e->pp;
    CS_TRY(cudaMemsetAsync(e->S.p, 0, sizeof(double) * pp * pp, e->s));
    CS_TRY(cudaMemcpy2DAsync(e->S.p, sizeof(double) * pp, S, sizeof(double) * e->p, sizeof(double) * e->p, e->p,
                             cudaMemcpyHostToDevice, e->s));
    const size_t smem = sizeof(double) * pp * 33;
    CS_TRY(cudaFuncSetAttribute(k_blk_mul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int gx = std::min(e->grid_rows(8), 4 * 148);
    k_blk_mul<<<dim3(gx, pp / 32), 256, smem, e->s>>>(e->n, pp, e->blk[src].p, e->S.p, e->blk[dst].p);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaStreamSynchronize(e->s));
    return 0;
}

// out (HOST, cols) = |HX_j - w_j X_j|^2 per column j < cols (w HOST, p)
int cs_eig_residuals(cs_eig* e, int hx, int x, const double* w, int cols, double* out, void* stream) {
    if (!eig_ok(e, hx) || !eig_ok(e, x) || !w || !out || cols <= 0 || cols > e->p) return CS_BAD_ARGUMENT;
    e->s = (cudaStream_t)stream;
    t_alloc_stream = e->s;
    const int pp = e->pp;
    CS_TRY(cudaMemsetAsync(e->w.p, 0, sizeof(double) * pp, e->s));
    CS_TRY(cudaMemcpyAsync(e->w.p, w, sizeof(double) * e->p, cudaMemcpyHostToDevice, e->s));
    const int g = std::min(e->grid_rows(8), 2 * 148);
    CS_RET(e->part.ensure((size_t)g * pp));
    CS_RET(e->red.ensure((size_t)pp * pp));
    k_blk_resid<<<g, 256, 0, e->s>>>(e->n, pp, e->blk[hx].p, e->blk[x].p, e->w.p, e->part.p);
    k_reduce_partials<<<cs_div_up(pp, 32), 256, 0, e->s>>>(e->part.p, g, pp, e->red.p);
    CS_CHECK_LAUNCH();
    CS_TRY(cudaMemcpyAsync(out, e->red.p, sizeof(double) * cols, cudaMemcpyDeviceToHost, e->s));
    CS_TRY(cudaStreamSynchronize(e->s));
    return 0;
}

}  // extern "C"
