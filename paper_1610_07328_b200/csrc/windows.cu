// windows.cu — §8f item 3: make_dataset (core.py:162-169) on the device:
// extract_subsequences (core.py:138-146, every window of length t, here with
// an optional stride) fused with z_normalize_dataset (core.py:127-135).  The
// row mean and population std follow numpy's float64 reductions bit for bit:
// np.sum along a contiguous axis is numpy's pairwise summation (blocks of <=
// 128 with 8 interleaved accumulators, recursive halving at multiples of 8),
// mean = sum / t, std = sqrt(sum((x - mean)^2) / t); rows with std < 1e-12
// become zeros; out = (x - mean) / std.  One thread per window.
#include "common.cuh"

// numpy pairwise_sum of f(a[0..n)) in float64 (f = identity or (x - mu)^2)
template <bool SQ>
__device__ double np_pairwise(const double *a, int64_t stride, int n, double mu) {
    auto val = [&](int i) {
        const double v = a[(int64_t)i * stride];
        if (!SQ) return v;
        const double d = __dsub_rn(v, mu);
        return __dmul_rn(d, d);
    };
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, val(i));
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = val(j);
        int i = 8;
        for (; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], val(i + j));
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, val(i));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise<SQ>(a, stride, n2, mu), np_pairwise<SQ>(a + (int64_t)n2 * stride, stride, n - n2, mu));
}

__global__ void windows_kernel(const double *__restrict__ rec, int t, int64_t stride, int64_t count,
                               int normalize, float *__restrict__ out32, double *__restrict__ out64) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < count;
         w += (int64_t)gridDim.x * blockDim.x) {
        const double *a = rec + w * stride;
        double mu = 0.0, sd = 1.0;
        bool flat = false;
        if (normalize) {
            mu = __ddiv_rn(np_pairwise<false>(a, 1, t, 0.0), (double)t);
            sd = __dsqrt_rn(__ddiv_rn(np_pairwise<true>(a, 1, t, mu), (double)t));
            flat = sd < 1e-12;
        }
        for (int i = 0; i < t; i++) {
            double v = a[i];
            if (normalize) v = flat ? 0.0 : __ddiv_rn(__dsub_rn(v, mu), sd);
            if (out32) out32[w * t + i] = (float)v;
            if (out64) out64[w * t + i] = v;
        }
    }
}

extern "C" int ssh_windows(const double *rec, int64_t len, int32_t t, int64_t stride, int32_t normalize,
                           float *out32, double *out64, int64_t *count_out, void *stream) {
    SSH_REQUIRE(rec && count_out && (out32 || out64), SSH_ERR_INVALID, "ssh_windows: NULL argument");
    SSH_REQUIRE(t >= 1, SSH_ERR_INVALID, "subsequence length must be >= 1, got %d", t);
    SSH_REQUIRE(t <= len, SSH_ERR_INVALID, "subsequence length %d exceeds series length %lld", t, (long long)len);
    SSH_REQUIRE(stride >= 1, SSH_ERR_INVALID, "window stride must be >= 1, got %lld", (long long)stride);
    const int64_t count = (len - t) / stride + 1;
    *count_out = count;
    const int grid = (int)std::min<int64_t>((count + 127) / 128, 148 * 32);
    windows_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(rec, t, stride, count, normalize, out32, out64);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}
