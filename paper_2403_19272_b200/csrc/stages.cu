// Scene-free per-pair stage kernels behind the reference's module-level helpers
// (clothsim.collision.__init__ / clothsim.oracles): each reproduces the reference
// function's arithmetic in numpy's evaluation order on the device.
//   k_tri_tri_sat      tri_tri_intersect        oracles.py:33-48
//   k_coplanarity      coplanarity_coefficients collision/ccd.py:36-44
//   k_query_q          query_q                  collision/partial.py:117-146
//   k_swept_boxes      swept_boxes              collision/bvh.py:140-143
//   k_dbb_weight       dbb_weight / _gradient   collision/pairs.py:83-108
#include "common.cuh"

namespace cs {

__global__ void k_tri_tri_sat(const double* __restrict__ p, const double* __restrict__ q, int64_t m,
                              uint8_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    d3 a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = ld3(p, 3 * i + k);
        b[k] = ld3(q, 3 * i + k);
    }
    out[i] = tri_tri_intersect_dev(a, b) ? 1 : 0;
}

__global__ void k_coplanarity(const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                              const double* __restrict__ x0, const double* __restrict__ x1, int64_t P, int single,
                              double* __restrict__ coef) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    const int4 id = idx[i];
    const Corners a = gather4(x0, id), b = gather4(x1, id);
    double c[4];
    coplanarity_fit(kind[i], a, b, single, c);
#pragma unroll
    for (int j = 0; j < 4; ++j) coef[4 * i + j] = c[j];
}

// trajectory endpoints p1(lam), p2(lam) of one pair at positions q (partial.py:117-130):
// VT p1 = x_v, p2 = t0 + l1 (t1 - t0) + l2 (t2 - t0); EE p1 = a0 + l1 (a1 - a0),
// p2 = b0 + l2 (b1 - b0)
__device__ __forceinline__ void param_points(int kd, const Corners& q, double l1, double l2, d3& p1, d3& p2) {
    if (kd == CS_VT) {
        p1 = q.p[0];
        p2 = (q.p[1] + l1 * (q.p[2] - q.p[1])) + l2 * (q.p[3] - q.p[1]);
    } else {
        p1 = q.p[0] + l1 * (q.p[1] - q.p[0]);
        p2 = q.p[2] + l2 * (q.p[3] - q.p[2]);
    }
}

// lam: (P, k, 2) per pair, or (k, 2) shared (shared != 0); out (P, k)
__global__ void k_query_q(const int8_t* __restrict__ kind, const int4* __restrict__ idx,
                          const double* __restrict__ x0, const double* __restrict__ x1, int64_t P,
                          const double* __restrict__ lam, int k, int shared, double* __restrict__ out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= P * k) return;
    const int64_t i = t / k;
    const int j = (int)(t - i * k);
    const double* l = shared ? lam + 2 * j : lam + 2 * t;
    const int4 id = idx[i];
    const int kd = kind[i];
    const Corners a = gather4(x0, id), b = gather4(x1, id);
    d3 p10, p20, p11, p21;
    param_points(kd, a, l[0], l[1], p10, p20);
    param_points(kd, b, l[0], l[1], p11, p21);
    out[t] = dot3(p21 - p11, p20 - p10);
}

// points (m, k, 3): lo/hi (m, 3) = min/max over the k points at both ends -/+ margin
__global__ void k_swept_boxes(const double* __restrict__ ps, const double* __restrict__ pe, int64_t m, int k,
                              double margin, double* __restrict__ lo, double* __restrict__ hi) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 3 * m) return;
    const int64_t i = t / 3;
    const int c = (int)(t - 3 * i);
    double a = ps[(i * k) * 3 + c], b = a, e = pe[(i * k) * 3 + c], f = e;
    for (int j = 1; j < k; ++j) {
        const double u = ps[(i * k + j) * 3 + c], v = pe[(i * k + j) * 3 + c];
        a = np_min(a, u);
        b = np_max(b, u);
        e = np_min(e, v);
        f = np_max(f, v);
    }
    lo[t] = np_min(a, e) - margin;
    hi[t] = np_max(b, f) + margin;
}

// -kappa (d - d_hat)^2 ln(d / d_hat) for 0 < d < d_hat (numpy order ((-kappa) sq) ln);
// gradient -kappa (2 (d - d_hat) ln(d / d_hat) + (d - d_hat)^2 / d); flag d <= 0 (weight)
__global__ void k_dbb_weight(const double* __restrict__ d, int64_t m, double d_hat, double kappa, int gradient,
                             double* __restrict__ out, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double x = d[i];
    double w = 0.0;
    if (!gradient) {
        if (!(x > 0.0)) atomicOr(bad, 1);
        if (x < d_hat) {
            const double u = x - d_hat;
            w = ((-kappa) * (u * u)) * log(x / d_hat);
        }
    } else if (x > 0.0 && x < d_hat) {
        const double u = x - d_hat;
        w = (-kappa) * (((2.0 * u) * log(x / d_hat)) + (u * u) / x);
    }
    out[i] = w;
}

}  // namespace cs

extern "C" {

int cs_tri_tri_intersect(const double* p, const double* q, long long m, uint8_t* out, void* stream) {
    if (m < 0 || (m && (!p || !q || !out))) return CS_BAD_ARGUMENT;
    if (m == 0) return 0;
    cs::k_tri_tri_sat<<<(int)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(p, q, m, out);
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_coplanarity_coefficients(const int8_t* kind, const int* idx4, const double* x_start, const double* x_end,
                                long long P, double* coef, void* stream) {
    if (P < 0) return CS_BAD_ARGUMENT;
    if (P == 0) return 0;
    cs::k_coplanarity<<<(int)((P + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        kind, (const int4*)idx4, x_start, x_end, P, P == 1 ? 1 : 0, coef);
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_query_q(const int8_t* kind, const int* idx4, const double* x_start, const double* x_end, long long P,
               const double* lam, int k, int shared, double* out, void* stream) {
    if (P < 0 || k < 0) return CS_BAD_ARGUMENT;
    if (P == 0 || k == 0) return 0;
    const long long n = P * k;
    cs::k_query_q<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(kind, (const int4*)idx4, x_start, x_end,
                                                                             P, lam, k, shared, out);
    CS_CHECK_LAUNCH();
    return 0;
}

int cs_swept_boxes(const double* points_start, const double* points_end, long long m, int k, double margin,
                   double* lo, double* hi, void* stream) {
    if (m < 0 || k <= 0) return CS_BAD_ARGUMENT;
    if (m == 0) return 0;
    cs::k_swept_boxes<<<(int)((3 * m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(points_start, points_end, m, k,
                                                                                     margin, lo, hi);
    CS_CHECK_LAUNCH();
    return 0;
}

// status CS_NONFINITE when a distance is <= 0 (pairs.py:92-93 raises FloatingPointError)
int cs_dbb_weight(const double* d, long long m, double d_hat, double kappa, int gradient, double* out, int* flag,
                  void* stream) {
    if (m < 0 || !flag || (!gradient && (!(d_hat > 0.0) || !(kappa > 0.0)))) return CS_BAD_ARGUMENT;
    cudaStream_t s = (cudaStream_t)stream;
    CS_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
    if (m == 0) return 0;
    cs::k_dbb_weight<<<(int)((m + 255) / 256), 256, 0, s>>>(d, m, d_hat, kappa, gradient, out, flag);
    CS_CHECK_LAUNCH();
    int h = 0;
    CS_TRY(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CS_TRY(cudaStreamSynchronize(s));
    return h ? CS_NONFINITE : 0;
}

}  // extern "C"
