// srp.cu — §8f item 4: signed random projection baseline, srp_matrix
// (index.py:420-423): bit[i][j] = [x_i . v_j >= 0] (+1 else -1, int8), with
// v_j = default_rng([seed, j]).standard_normal(m) drawn on the host.
// A tiled fp32 FFMA product decides every sign whose |value| exceeds the
// fp32 error bound (m + 2) u * sum|x_k v_jk| (accumulated alongside); the
// rest are re-evaluated as a sequential fp64 dot product.  (numpy's BLAS
// matmul has its own summation order, so signs of projections within a few
// f64 ulps of zero are the only place the two can differ.)
#include "common.cuh"

#define SRP_TM 64
#define SRP_TN 64
#define SRP_TK 32

__global__ void __launch_bounds__(256)
srp_kernel(const float *__restrict__ X, int64_t N, int m, const float *__restrict__ V32,
           const double *__restrict__ V64, int bits, int8_t *__restrict__ out, unsigned long long *nrecheck) {
    __shared__ float xs[SRP_TK][SRP_TM + 1];
    __shared__ float vs[SRP_TK][SRP_TN + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
    const int64_t r0 = (int64_t)blockIdx.x * SRP_TM;
    const int c0 = blockIdx.y * SRP_TN;
    float acc[4][4] = {}, mag[4][4] = {};
    for (int k0 = 0; k0 < m; k0 += SRP_TK) {
        for (int e = threadIdx.x; e < SRP_TK * SRP_TM; e += 256) {
            const int kk = e % SRP_TK, rr = e / SRP_TK;
            const int64_t row = r0 + rr;
            xs[kk][rr] = (row < N && k0 + kk < m) ? X[row * m + k0 + kk] : 0.f;
        }
        for (int e = threadIdx.x; e < SRP_TK * SRP_TN; e += 256) {
            const int kk = e % SRP_TK, cc = e / SRP_TK;
            vs[kk][cc] = (c0 + cc < bits && k0 + kk < m) ? V32[(int64_t)(c0 + cc) * m + k0 + kk] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < SRP_TK; kk++) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; i++) a[i] = xs[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; j++) b[j] = vs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
                    mag[i][j] = fmaf(fabsf(a[i]), fabsf(b[j]), mag[i][j]);
                }
        }
        __syncthreads();
    }
    const float tol = (float)(m + 4) * 1.2e-7f;  // (m + 2) u32 plus the f32-rounded taps
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t row = r0 + ty + 16 * i;
            const int col = c0 + tx + 16 * j;
            if (row >= N || col >= bits) continue;
            int8_t bit;
            if (fabsf(acc[i][j]) > tol * mag[i][j] * 2.f + 1e-30f) {
                bit = acc[i][j] >= 0.f ? 1 : -1;
            } else {
                double s = 0.0;
                const float *x = X + row * m;
                const double *v = V64 + (int64_t)col * m;
                for (int k = 0; k < m; k++) s = __dadd_rn(s, __dmul_rn((double)x[k], v[k]));
                bit = s >= 0.0 ? 1 : -1;
                if (nrecheck) atomicAdd(nrecheck, 1ULL);
            }
            out[row * bits + col] = bit;
        }
}

extern "C" int ssh_srp(const float *X, int64_t N, int32_t m, const float *V32, const double *V64, int32_t bits,
                       int8_t *out, unsigned long long *nrecheck, void *stream) {
    SSH_REQUIRE(X && V32 && V64 && out, SSH_ERR_INVALID, "ssh_srp: NULL argument");
    SSH_REQUIRE(N >= 0 && m >= 1 && bits >= 1, SSH_ERR_INVALID, "ssh_srp: bad shape");
    if (N == 0) return SSH_OK;
    dim3 g((unsigned)((N + SRP_TM - 1) / SRP_TM), (unsigned)((bits + SRP_TN - 1) / SRP_TN));
    srp_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(X, N, m, V32, V64, bits, out, nrecheck);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}
