// pairs.cu — the reference's public DTW utilities on the device, in float64
// with the reference's operation order (dtw.py:239-284):
//   dtw_distance  -> ssh_dtw_pairs64   (_dtw_band_sq, dtw.py:83-121)
//   build_envelope-> ssh_envelope64    (_envelope_into, dtw.py:124-151)
//   lb_keogh(2)   -> ssh_lb_keogh64    (_lb_keogh_sq, dtw.py:154-168)
//   lb_kim        -> ssh_lb_kim64      (dtw.py:252-260)
// Batched over rows; inputs and outputs are device f64 arrays.
#include <math.h>

#include "common.cuh"
#include "dtw_warp.cuh"

#define PR_WARPS 4

// one warp per pair: X row xrow[p] (or p) against Y row yrow[p] (or p)
template <int C>
__global__ void __launch_bounds__(32 * PR_WARPS)
dtw_pairs64_kernel(const double *__restrict__ X, const double *__restrict__ Y, const int64_t *__restrict__ xrow,
                   const int64_t *__restrict__ yrow, int64_t npair, int m, int r, double abandon_sq,
                   double *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * PR_WARPS + (threadIdx.x >> 5);
    if (p >= npair) return;
    const int64_t a = xrow ? xrow[p] : p, b = yrow ? yrow[p] : p;
    const double v = dtw_warp_band64<double, C>(X + a * m, Y + b * m, m, r, abandon_sq);
    if ((threadIdx.x & 31) == 0) out[p] = v;
}

// bands wider than 32 x 32 cells: one thread per pair, rolling rows in
// global scratch (2 m per pair), the reference's loop as written
__global__ void dtw_pairs64_rows_kernel(const double *__restrict__ X, const double *__restrict__ Y,
                                        const int64_t *__restrict__ xrow, const int64_t *__restrict__ yrow,
                                        int64_t npair, int m, int r, double abandon_sq, double *__restrict__ scratch,
                                        double *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npair) return;
    const double *x = X + (xrow ? xrow[p] : p) * m;
    const double *y = Y + (yrow ? yrow[p] : p) * m;
    double *prev = scratch + p * 2 * m, *curr = prev + m;
    const double inf = (double)INFINITY;
    for (int j = 0; j < m; j++) prev[j] = curr[j] = inf;
    for (int i = 0; i < m; i++) {
        const int lo = max(i - r, 0), hi = min(i + r, m - 1);
        if (lo > 0) curr[lo - 1] = inf;
        double row_min = inf;
        for (int j = lo; j <= hi; j++) {
            double d = __dsub_rn(x[i], y[j]);
            d = __dmul_rn(d, d);
            double c;
            if (i == 0 && j == 0) {
                c = d;
            } else {
                double best = prev[j];
                if (j > 0) {
                    if (curr[j - 1] < best) best = curr[j - 1];
                    if (prev[j - 1] < best) best = prev[j - 1];
                }
                c = __dadd_rn(d, best);
            }
            curr[j] = c;
            if (c < row_min) row_min = c;
        }
        if (abandon_sq >= 0.0 && row_min > abandon_sq) {
            out[p] = inf;
            return;
        }
        double *t = prev;
        prev = curr;
        curr = t;
    }
    out[p] = prev[m - 1];
}

extern "C" int ssh_dtw_pairs64(const double *X, const double *Y, const int64_t *xrow, const int64_t *yrow,
                               int64_t npair, int32_t m, int32_t r, double abandon_sq, double *out_sq,
                               void *stream) {
    SSH_REQUIRE(npair >= 0 && m >= 1 && r >= 0, SSH_ERR_INVALID, "ssh_dtw_pairs64: bad sizes");
    if (npair == 0) return SSH_OK;
    SSH_REQUIRE(X && Y && out_sq, SSH_ERR_INVALID, "ssh_dtw_pairs64: NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int C = dtw_warp_chunk(r);
    if (C) {
        const unsigned g = (unsigned)ssh_div_up(npair, PR_WARPS);
#define PR_CALL(CC) \
    dtw_pairs64_kernel<CC><<<g, 32 * PR_WARPS, 0, st>>>(X, Y, xrow, yrow, npair, m, r, abandon_sq, out_sq)
        DTW_WARP_DISPATCH(C, PR_CALL)
#undef PR_CALL
        SSH_CHECK_LAUNCH();
        return SSH_OK;
    }
    double *scratch = nullptr;
    SSH_CUDA(cudaMallocAsync(&scratch, sizeof(double) * 2 * (size_t)m * npair, st));
    dtw_pairs64_rows_kernel<<<(unsigned)ssh_div_up(npair, 64), 64, 0, st>>>(X, Y, xrow, yrow, npair, m, r,
                                                                           abandon_sq, scratch, out_sq);
    ssh_count_launch();
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return ssh_cuda_fail(e, "dtw_pairs64_rows_kernel", __FILE__, __LINE__);
    return SSH_OK;
}

// running max / min over [i - r, i + r] (the values the reference's deques
// select; max/min are exact), one thread per (row, i)
__global__ void envelope64_kernel(const double *__restrict__ X, int64_t n, int m, int r, double *__restrict__ U,
                                  double *__restrict__ Lo) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * m) return;
    const int64_t row = t / m;
    const int i = (int)(t - row * m);
    const double *x = X + row * m;
    const int lo = max(i - r, 0), hi = min(i + r, m - 1);
    double u = x[lo], l = x[lo];
    for (int j = lo + 1; j <= hi; j++) {
        const double v = x[j];
        u = v >= u ? v : u;
        l = v <= l ? v : l;
    }
    U[t] = u;
    Lo[t] = l;
}

extern "C" int ssh_envelope64(const double *X, int64_t n, int32_t m, int32_t r, double *upper, double *lower,
                              void *stream) {
    SSH_REQUIRE(n >= 0 && m >= 1 && r >= 0, SSH_ERR_INVALID, "ssh_envelope64: bad sizes");
    if (n == 0) return SSH_OK;
    SSH_REQUIRE(X && upper && lower, SSH_ERR_INVALID, "ssh_envelope64: NULL pointer");
    envelope64_kernel<<<(unsigned)ssh_div_up(n * m, 256), 256, 0, (cudaStream_t)stream>>>(X, n, m, r, upper,
                                                                                        lower);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

// sum of squared excursions of c outside [lower, upper], sequential in i
// (_lb_keogh_sq with abandon disabled), one thread per row
__global__ void lb_keogh64_kernel(const double *__restrict__ Cs, const double *__restrict__ U,
                                  const double *__restrict__ Lo, int64_t n, int m, int env_rows,
                                  double *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double *c = Cs + p * m;
    const int64_t eb = env_rows == 1 ? 0 : p * m;
    double total = 0.0;
    for (int i = 0; i < m; i++) {
        const double v = c[i], u = U[eb + i], l = Lo[eb + i];
        if (v > u) {
            const double d = __dsub_rn(v, u);
            total = __dadd_rn(total, __dmul_rn(d, d));
        } else if (v < l) {
            const double d = __dsub_rn(l, v);
            total = __dadd_rn(total, __dmul_rn(d, d));
        }
    }
    out[p] = total;
}

extern "C" int ssh_lb_keogh64(const double *Cs, const double *U, const double *Lo, int64_t n, int32_t m,
                              int32_t env_rows, double *out_sq, void *stream) {
    SSH_REQUIRE(n >= 0 && m >= 1 && (env_rows == 1 || env_rows == n), SSH_ERR_INVALID,
                "ssh_lb_keogh64: bad sizes");
    if (n == 0) return SSH_OK;
    SSH_REQUIRE(Cs && U && Lo && out_sq, SSH_ERR_INVALID, "ssh_lb_keogh64: NULL pointer");
    lb_keogh64_kernel<<<(unsigned)ssh_div_up(n, 128), 128, 0, (cudaStream_t)stream>>>(Cs, U, Lo, n, m, env_rows,
                                                                                   out_sq);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

// sqrt(d0^2 + d_{m-1}^2) of the first and last point pairs (dtw.py:252-260)
__global__ void lb_kim64_kernel(const double *__restrict__ X, const double *__restrict__ Y, int64_t n, int m,
                                double *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double *x = X + p * m, *y = Y + p * m;
    const double d0 = __dsub_rn(x[0], y[0]);
    const double dm = __dsub_rn(x[m - 1], y[m - 1]);
    out[p] = __dsqrt_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(dm, dm)));
}

extern "C" int ssh_lb_kim64(const double *X, const double *Y, int64_t n, int32_t m, double *out, void *stream) {
    SSH_REQUIRE(n >= 0 && m >= 1, SSH_ERR_INVALID, "ssh_lb_kim64: bad sizes");
    if (n == 0) return SSH_OK;
    SSH_REQUIRE(X && Y && out, SSH_ERR_INVALID, "ssh_lb_kim64: NULL pointer");
    lb_kim64_kernel<<<(unsigned)ssh_div_up(n, 128), 128, 0, (cudaStream_t)stream>>>(X, Y, n, m, out);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}
