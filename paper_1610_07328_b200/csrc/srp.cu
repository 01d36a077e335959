// srp.cu — §8f item 4: signed random projection baseline, srp_matrix
// (index.py:420-423): bit[i][j] = [x_i . v_j >= 0] (+1 else -1, int8), with
// v_j = default_rng([seed, j]).standard_normal(m) drawn on the host.
//
// The product X V^T is the one dense contraction of the reference, so it runs
// on the 5th-generation tensor cores: tcgen05.mma kind::tf32 (A = a 128-row
// tile of X, B = all the projections, both K-major in shared memory, the
// fp32 accumulator tile in TMEM), issued by one thread per CTA, completion
// signalled through an mbarrier (tcgen05.commit), the accumulator read back
// with tcgen05.ld.  The signs are then screened with a rigorous error bound:
// TF32 keeps 10 mantissa bits (|x - tf32(x)| <= 2^-10 |x|) and the fp32
// accumulation adds at most (m + 8) 2^-24 sum|x v|, so with Cauchy-Schwarz
//     |fl_tc(x . v) - x . v| <= (2^-8 + (m + 8) 2^-23) ||x|| ||v||  =: tol
// (both terms with a 2x margin; the norms are f64, rounded up).  A value with
// |acc| > tol has the exact product's sign; the rest (a few percent) are
// re-evaluated as a sequential fp64 dot product of the ORIGINAL values (f64
// inputs stay f64).  numpy's BLAS matmul has its own summation order, so signs
// of projections within a few f64 ulps of zero are the only place the two can
// differ.  The SIMT fp32 kernel below is kept for shapes outside the tensor-
// core path (bits > 256).
#include "common.cuh"

#define SRP_TM 64
#define SRP_TN 64
#define SRP_TK 32

__global__ void __launch_bounds__(256)
srp_kernel(const float *__restrict__ X, int64_t N, int m, const float *__restrict__ V32,
           const double *__restrict__ V64, int bits, int8_t *__restrict__ out, unsigned long long *nrecheck,
           const double *__restrict__ X64) {
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
    // (m + 2) u32 plus the f32-rounded taps, and the f32 rounding of f64 inputs
    const float tol = (float)(m + 6) * 1.2e-7f;
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
                const double *v = V64 + (int64_t)col * m;
                if (X64) {
                    const double *x = X64 + row * m;
                    for (int k = 0; k < m; k++) s = __dadd_rn(s, __dmul_rn(x[k], v[k]));
                } else {
                    const float *x = X + row * m;
                    for (int k = 0; k < m; k++) s = __dadd_rn(s, __dmul_rn((double)x[k], v[k]));
                }
                bit = s >= 0.0 ? 1 : -1;
                if (nrecheck) atomicAdd(nrecheck, 1ULL);
            }
            out[row * bits + col] = bit;
        }
}

// ---------------------------------------------------------------- tcgen05
#define ST_M 128     // rows of X per CTA (UMMA_M)
#define ST_BK 32     // K (floats) per shared-memory stage: 128 B per row
#define ST_THREADS 128

// f64 L2 norm of each row of an (n, m) matrix (f32 or f64), rounded up
__global__ void srp_rownorm_kernel(const float *__restrict__ X32, const double *__restrict__ X64, int64_t n, int m,
                                   double *__restrict__ nrm) {
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    double s = 0.0;
    for (int k = lane; k < m; k += 32) {
        const double v = X64 ? X64[r * m + k] : (double)X32[r * m + k];
        s = fma(v, v, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0) nrm[r] = sqrt(s) * (1.0 + 1e-12);
}

__device__ __forceinline__ uint32_t st_smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no-swizzle UMMA shared-memory descriptor: core matrices of 8 rows
// x 16 B stored contiguously (128 B); LBO = byte stride between the two core
// matrices of one MMA's K extent (32 B of tf32 = 2 cores), SBO = byte stride
// between 8-row groups; version 1 (sm_100), layout type 0 (SWIZZLE_NONE).
__device__ __forceinline__ uint64_t st_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;
}

// Instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, N x M.
__host__ __device__ constexpr uint32_t st_idesc(int n, int mrows) {
    return (1u << 4)                        // c_format = F32
           | (2u << 7) | (2u << 10)         // a_format = b_format = TF32
           | ((uint32_t)(n >> 3) << 17)     // N >> 3
           | ((uint32_t)(mrows >> 4) << 24);  // M >> 4
}

// Stage rows [0, rows) x K block [k0, k0 + ST_BK) of a row-major (ld = m)
// matrix into the core-matrix layout: element (r, k) of the stage at byte
// ((r / 8) * 8 + k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4; zeros outside.
__device__ __forceinline__ void st_stage(float *sm, const float *__restrict__ src, int64_t r0, int64_t nrows,
                                         int rows, int m, int k0, bool vec) {
    for (int e = threadIdx.x; e < rows * (ST_BK / 4); e += ST_THREADS) {
        const int r = e >> 3, c = e & 7;  // c: 16-byte chunk within the 128-byte row block
        const int64_t gr = r0 + r;
        const int k = k0 + 4 * c;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gr < nrows) {
            const float *p = src + gr * (int64_t)m + k;
            if (vec && k + 4 <= m) {
                v = __ldg(reinterpret_cast<const float4 *>(p));
            } else {
                v.x = k < m ? p[0] : 0.f;
                v.y = k + 1 < m ? p[1] : 0.f;
                v.z = k + 2 < m ? p[2] : 0.f;
                v.w = k + 3 < m ? p[3] : 0.f;
            }
        }
        *reinterpret_cast<float4 *>(reinterpret_cast<unsigned char *>(sm) + (((r >> 3) * 8 + c) * 128 + (r & 7) * 16)) = v;
    }
}

template <int NB>  // projections padded to a multiple of 16 (<= 256): the UMMA N
__global__ void __launch_bounds__(ST_THREADS)
srp_tc_kernel(const float *__restrict__ X32, const double *__restrict__ X64, int64_t N, int m,
              const float *__restrict__ V32, const double *__restrict__ V64, int bits, const double *__restrict__ xn,
              const double *__restrict__ vn, int8_t *__restrict__ out, unsigned long long *__restrict__ nrecheck) {
    constexpr int TCOLS = NB <= 32 ? 32 : NB <= 64 ? 64 : NB <= 128 ? 128 : 256;
    extern __shared__ __align__(1024) unsigned char st_sm[];
    float *sa = reinterpret_cast<float *>(st_sm);                    // ST_M x ST_BK
    float *sb = reinterpret_cast<float *>(st_sm + ST_M * ST_BK * 4);  // NB x ST_BK
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * ST_M;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                     ::"r"(st_smem_u32(&tmem_base)), "n"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(st_smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    const bool vec = (m & 3) == 0;
    constexpr uint32_t IDESC = st_idesc(NB, ST_M);
    uint32_t phase = 0;
    for (int k0 = 0; k0 < m; k0 += ST_BK) {
        st_stage(sa, X32, r0, N, ST_M, m, k0, vec);
        st_stage(sb, V32, 0, bits, NB, m, k0, vec);
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;\n");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t a0 = st_smem_u32(sa), b0 = st_smem_u32(sb);
#pragma unroll
            for (int kk = 0; kk < ST_BK / 8; kk++) {  // UMMA_K = 8 tf32 = 32 B = 2 core matrices
                const uint64_t ad = st_desc(a0 + kk * 256, 128, 1024);
                const uint64_t bd = st_desc(b0 + kk * 256, 128, 1024);
                const uint32_t acc = (k0 > 0 || kk > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                         ::"r"(st_smem_u32(&mbar)));
        }
        // the stage's MMAs have completed (and read shared memory) once the barrier flips
        {
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(st_smem_u32(&mbar)), "r"(phase));
            }
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        __syncthreads();
    }
    // epilogue: warp w owns TMEM lanes [32 w, 32 w + 32) = rows r0 + 32 w + lane
    const int64_t row = r0 + 32 * warp + lane;
    const double xnorm = row < N ? xn[row] : 0.0;
    const double eps = 1.0 / 256.0 + (double)(m + 8) * (1.0 / 8388608.0);
#pragma unroll 1
    for (int c0 = 0; c0 < NB; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        if (row < N) {
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const int col = c0 + j;
                if (col >= bits) continue;
                const float a = __uint_as_float(v[j]);
                const double tol = eps * xnorm * vn[col];
                int8_t bit;
                if ((double)fabsf(a) > tol) {
                    bit = a >= 0.f ? 1 : -1;
                } else {
                    double s = 0.0;
                    const double *vv = V64 + (int64_t)col * m;
                    if (X64) {
                        const double *x = X64 + row * m;
                        for (int k = 0; k < m; k++) s = __dadd_rn(s, __dmul_rn(x[k], vv[k]));
                    } else {
                        const float *x = X32 + row * m;
                        for (int k = 0; k < m; k++) s = __dadd_rn(s, __dmul_rn((double)x[k], vv[k]));
                    }
                    bit = s >= 0.0 ? 1 : -1;
                    if (nrecheck) atomicAdd(nrecheck, 1ULL);
                }
                out[row * bits + col] = bit;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
}

template <int NB>
static int launch_srp_tc(const float *X32, const double *X64, int64_t N, int m, const float *V32, const double *V64,
                         int bits, const double *xn, const double *vn, int8_t *out, unsigned long long *nrecheck,
                         cudaStream_t st) {
    const size_t smem = (size_t)(ST_M + NB) * ST_BK * 4;
    SSH_CUDA(cudaFuncSetAttribute(srp_tc_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    srp_tc_kernel<NB><<<(unsigned)((N + ST_M - 1) / ST_M), ST_THREADS, smem, st>>>(X32, X64, N, m, V32, V64, bits, xn,
                                                                                    vn, out, nrecheck);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

extern "C" int ssh_srp(const float *X, int64_t N, int32_t m, const float *V32, const double *V64, int32_t bits,
                       int8_t *out, unsigned long long *nrecheck, void *stream) {
    return ssh_srp2(X, nullptr, N, m, V32, V64, bits, out, nrecheck, 1, stream);
}

extern "C" int ssh_srp2(const float *X, const double *X64, int64_t N, int32_t m, const float *V32, const double *V64,
                        int32_t bits, int8_t *out, unsigned long long *nrecheck, int32_t tensor_cores, void *stream) {
    SSH_REQUIRE(X && V32 && V64 && out, SSH_ERR_INVALID, "ssh_srp: NULL argument");
    SSH_REQUIRE(N >= 0 && m >= 1 && bits >= 1, SSH_ERR_INVALID, "ssh_srp: bad shape");
    if (N == 0) return SSH_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = (bits + 15) / 16 * 16;
    if (tensor_cores && nb <= 256) {
        double *norms = nullptr;
        SSH_CUDA(cudaMallocAsync((void **)&norms, sizeof(double) * (size_t)(N + bits), st));
        srp_rownorm_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(X, X64, N, m, norms);
        ssh_count_launch();
        srp_rownorm_kernel<<<(unsigned)((bits + 7) / 8), 256, 0, st>>>(nullptr, V64, bits, m, norms + N);
        ssh_count_launch();
        int rc = SSH_OK;
#define SRP_TC(NBV) \
    case NBV: rc = launch_srp_tc<NBV>(X, X64, N, m, V32, V64, bits, norms, norms + N, out, nrecheck, st); break;
        switch (nb) {
            SRP_TC(16) SRP_TC(32) SRP_TC(48) SRP_TC(64) SRP_TC(80) SRP_TC(96) SRP_TC(112) SRP_TC(128)
            SRP_TC(144) SRP_TC(160) SRP_TC(176) SRP_TC(192) SRP_TC(208) SRP_TC(224) SRP_TC(240) SRP_TC(256)
            default: rc = SSH_ERR_UNSUPPORTED; break;
        }
#undef SRP_TC
        cudaFreeAsync(norms, st);
        return rc;
    }
    dim3 g((unsigned)((N + SRP_TM - 1) / SRP_TM), (unsigned)((bits + SRP_TN - 1) / SRP_TN));
    srp_kernel<<<g, 256, 0, st>>>(X, N, m, V32, V64, bits, out, nrecheck, X64);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}
