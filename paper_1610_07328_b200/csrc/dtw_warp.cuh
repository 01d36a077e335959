// dtw_warp.cuh — warp-cooperative banded DTW for any radius: one warp per
// (series, query) pair, the band split across the lanes, rows swept as a
// skewed wavefront with warp-shuffle neighbour exchange (SURVEY.md §7 iii).
//
// Band coordinates (dtw.py:83-121): row i = candidate sample, column
// j = i + k - r for k in [0, 2r]; cell (i, k) reads diag (i-1, k), up
// (i-1, k+1) and left (i, k-1); cells with j outside [0, m) or k outside
// [0, 2r] are +inf (the reference's rolling rows hold +inf there).
//
// Lane l owns the C consecutive offsets k = lC + c (C = ceil((2r+1)/32) >= 2)
// as registers band[c] and works on row i = s - l at step s.  In one step a
// lane updates its C cells in place in ascending k:
//   diag = band[c] (row i-1), up = band[c+1] (row i-1), left = band[c-1]
//   (row i, just written); the lane's first cell takes `left` from lane l-1,
//   which finished row i one step earlier (shfl_up of its band[C-1]); its
//   last cell takes `up` = (i-1, (l+1)C) from lane l+1, which computes that
//   cell as the first cell of ITS step-s row i-1 (shfl_down after sub-step 0;
//   hence C >= 2).
// The lane's samples are register windows: x_i arrives from lane l-1 (it had
// row i one step earlier); the C query samples y[j] slide by one per step and
// the new one comes from lane l+1's second window entry; lane 0 / lane 31 read
// x / y from 32-sample blocks loaded once per 32 steps.  Row minima (early
// abandon, dtw.py:114-115) travel along the skew with the left edge: lane 31
// holds the full minimum of row s - 31.
//
// T = double with EXACT: every cell is the reference's d = x - y; d = d*d;
// c = d + min(up, left, diag) with _rn intrinsics (no FMA contraction), so
// the result has the reference's bits.  A virtual row -1 holding 0 at k = r
// gives D(0, 0) = d exactly as the reference's i == j == 0 case.
#pragma once

template <typename T>
__device__ __forceinline__ T dw_shfl_up(T v, int d) { return __shfl_up_sync(0xFFFFFFFFu, v, d); }
template <typename T>
__device__ __forceinline__ T dw_shfl_down(T v, int d) { return __shfl_down_sync(0xFFFFFFFFu, v, d); }
template <typename T>
__device__ __forceinline__ T dw_shfl(T v, int s) { return __shfl_sync(0xFFFFFFFFu, v, s); }

__device__ __forceinline__ double dw_cell(double xi, double yj, double up, double left, double dg) {
    double d = __dsub_rn(xi, yj);
    d = __dmul_rn(d, d);
    return __dadd_rn(d, fmin(fmin(up, left), dg));
}

// Squared banded DTW of x (row, length m) against y (length m), radius r,
// C cells per lane (C >= 2, 32 C >= 2 r + 1).  abandon_sq >= 0 enables the
// reference's row-minimum abandon (returns +inf).  Every lane returns the
// result.  TX: float or double samples in global memory.
template <typename TX, int C>
__device__ double dtw_warp_band64(const TX *__restrict__ x, const TX *__restrict__ y, int m, int r,
                                  double abandon_sq) {
    const int lane = threadIdx.x & 31;
    const double inf = (double)INFINITY;
    const int nk = 2 * r + 1;
    double band[C];
    double yw[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
        band[c] = (lane * C + c == r) ? 0.0 : inf;  // virtual row -1
        const int j = lane * (C - 1) - r + c;        // window at step 0
        yw[c] = (j >= 0 && j < m) ? (double)y[j] : inf;
    }
    double xi = 0.0, rmin = inf, res = inf;
    double xblk = 0.0, yblk = inf;
    const int steps = m + 31;
    const int k_res = r - lane * C;  // this lane's cell index of k = r (if in [0, C))
    for (int s = 0; s < steps; s++) {
        const int sl = s & 31;
        if (sl == 0) {
            const int ix = s + lane;
            xblk = ix < m ? (double)x[ix] : 0.0;
            // lane 31's new window entry at step s + 1 + t is y[s + t + 32 C - 31 - r]
            const int jy = s + lane + 32 * C - 31 - r;
            yblk = (jy >= 0 && jy < m) ? (double)y[jy] : inf;
        }
        const double x0 = dw_shfl(xblk, sl);
        const double ynew31 = dw_shfl(yblk, sl);
        const double xprev = dw_shfl_up(xi, 1);
        double leftv = dw_shfl_up(band[C - 1], 1);
        double pm = dw_shfl_up(rmin, 1);
        xi = lane == 0 ? x0 : xprev;
        if (lane == 0) {
            leftv = inf;
            pm = inf;
        }
        const int i = s - lane;
        const bool act = i >= 0 && i < m;
        // sub-step 0
        double lm;
        {
            const double up = band[1];
            double v = dw_cell(xi, yw[0], up, leftv, band[0]);
            if (lane * C >= nk) v = inf;
            if (act) band[0] = v;
        }
        double upr = dw_shfl_down(band[0], 1);
        if (lane == 31) upr = inf;
        lm = band[0];
#pragma unroll
        for (int c = 1; c < C; c++) {
            const double up = (c + 1 < C) ? band[c + 1] : upr;
            double v = dw_cell(xi, yw[c], up, band[c - 1], band[c]);
            if (lane * C + c >= nk) v = inf;
            if (act) band[c] = v;
            lm = fmin(lm, band[c]);
        }
        rmin = fmin(pm, lm);
        if (i == m - 1 && k_res >= 0 && k_res < C) {
#pragma unroll
            for (int c = 0; c < C; c++)
                if (c == k_res) res = band[c];
        }
        if (abandon_sq >= 0.0) {
            const double fm = dw_shfl(rmin, 31);
            const int i31 = s - 31;
            if (i31 >= 0 && i31 < m && fm > abandon_sq) return inf;
        }
        // slide the query window: new last entry from lane l + 1's yw[1]
        double yn = dw_shfl_down(yw[1], 1);
        if (lane == 31) yn = ynew31;
#pragma unroll
        for (int c = 0; c + 1 < C; c++) yw[c] = yw[c + 1];
        yw[C - 1] = yn;
    }
    const int owner = r / C;
    return dw_shfl(res, owner);
}

// cells per lane for radius r (0 when the warp kernel does not cover r)
static inline int dtw_warp_chunk(int r) {
    int c = (2 * r + 1 + 31) / 32;
    if (c < 2) c = 2;
    return c <= 32 ? c : 0;
}

// chunk sizes 2..16 only (radius <= 255): the query-path kernels
#define DTW_WARP_DISPATCH16(C_, CALL)                                              \
    switch (C_) {                                                                  \
        case 2: CALL(2); break;   case 3: CALL(3); break;   case 4: CALL(4); break;    \
        case 5: CALL(5); break;   case 6: CALL(6); break;   case 7: CALL(7); break;    \
        case 8: CALL(8); break;   case 9: CALL(9); break;   case 10: CALL(10); break;  \
        case 11: CALL(11); break; case 12: CALL(12); break; case 13: CALL(13); break;  \
        case 14: CALL(14); break; case 15: CALL(15); break; case 16: CALL(16); break;  \
        default: break;                                                            \
    }

// switch over the instantiated chunk sizes: FN<C>(args...) for C = chunk
#define DTW_WARP_DISPATCH(C_, CALL)                                                \
    switch (C_) {                                                                  \
        case 2: CALL(2); break;   case 3: CALL(3); break;   case 4: CALL(4); break;    \
        case 5: CALL(5); break;   case 6: CALL(6); break;   case 7: CALL(7); break;    \
        case 8: CALL(8); break;   case 9: CALL(9); break;   case 10: CALL(10); break;  \
        case 11: CALL(11); break; case 12: CALL(12); break; case 13: CALL(13); break;  \
        case 14: CALL(14); break; case 15: CALL(15); break; case 16: CALL(16); break;  \
        case 17: CALL(17); break; case 18: CALL(18); break; case 19: CALL(19); break;  \
        case 20: CALL(20); break; case 21: CALL(21); break; case 22: CALL(22); break;  \
        case 23: CALL(23); break; case 24: CALL(24); break; case 25: CALL(25); break;  \
        case 26: CALL(26); break; case 27: CALL(27); break; case 28: CALL(28); break;  \
        case 29: CALL(29); break; case 30: CALL(30); break; case 31: CALL(31); break;  \
        case 32: CALL(32); break;                                                  \
        default: break;                                                            \
    }
