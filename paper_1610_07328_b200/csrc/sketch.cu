// sketch.cu — K1: sliding random-filter sign sketch (sketch.py:51-61, 69-89).
//
// bit_i = [ sum_{k<W} w_k x_{i*delta+k} >= 0 ].  The reference evaluates the
// dot in f64, sequentially in k, mul then add (numpy's non-BLAS matmul loop;
// SURVEY.md §0 item 6).  The device evaluates an f32 screen and re-evaluates
// exactly that f64 sequence only for windows whose screen value is within
// the a-priori error bound of zero:
//   |fl32(sum x w32) - fl64(sum x w)| <= (W+2) 2^-24 sum|x_k||w_k|
//                                    <= screen_c * max|x|      (ctx.cu)
// so every emitted bit equals the reference bit.
//
// Layout/roofline: one CTA stages a tile of ST series from HBM with
// coalesced float4 loads into a polyphase shared-memory layout
// x_b[j] = x[j*delta + b] (b < delta), padded by one float per 8 so that
// threads owning 8 consecutive windows read with a bank-conflict-free stride
// of 9.  With W, delta compile-time, each thread keeps a sliding register
// window and the taps come from the constant bank: 8 FFMA per LDS.  The
// kernel is HBM-bound: 4m bytes in + 8*words bytes out per series.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

#define SK_THREADS 256
#define SK_J 8

struct SketchW {
    float w[SSH_MAX_W];
};

struct SketchGeom {
    int m, nb, words, G, ST, PB, P, W, delta;
    int64_t N, ld;
    float screen_c;
};

__device__ __forceinline__ int poly_off(int j) { return j + (j >> 3); }

// byte offset of the packed-bit staging buffer after the series tile (16-byte aligned)
__host__ __device__ __forceinline__ size_t bits_offset(const SketchGeom &g) {
    return ((size_t)g.ST * g.P * 4 + 15) & ~(size_t)15;
}
__host__ __device__ __forceinline__ size_t sketch_smem(const SketchGeom &g) {
    return bits_offset(g) + (size_t)g.ST * g.words * 8;
}

// Stage up to ST series [s0, s0+ns) into polyphase smem; record max|x| per series.
template <int DELTA_T>
__device__ __forceinline__ void stage_tile(const float *__restrict__ X, const SketchGeom &g,
                                           int64_t s0, int ns, float *xs, unsigned *maxabs) {
    const int delta = DELTA_T > 0 ? DELTA_T : g.delta;
    const int m = g.m;
    const int tid = threadIdx.x;
    const bool vec = ((g.ld & 3) == 0) && ((m & 3) == 0) && ((((uintptr_t)X) & 15) == 0);
    if (vec) {
        const int m4 = m >> 2;
        const int total = ns * m4;
        for (int f = tid; f < total; f += SK_THREADS) {
            int s = f / m4;
            int p4 = f - s * m4;
            float4 v = __ldg(reinterpret_cast<const float4 *>(X + (s0 + s) * g.ld) + p4);
            float *xr = xs + s * g.P;
            float vv[4] = {v.x, v.y, v.z, v.w};
            float mx = 0.f;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                int p = 4 * p4 + e;
                int b = p % delta, j = p / delta;
                xr[b * g.PB + poly_off(j)] = vv[e];
                mx = fmaxf(mx, fabsf(vv[e]));
            }
            atomicMax(&maxabs[s], __float_as_uint(mx));
        }
    } else {
        const int total = ns * m;
        for (int f = tid; f < total; f += SK_THREADS) {
            int s = f / m;
            int p = f - s * m;
            float v = __ldg(X + (s0 + s) * g.ld + p);
            int b = p % delta, j = p / delta;
            xs[s * g.P + b * g.PB + poly_off(j)] = v;
            atomicMax(&maxabs[s], __float_as_uint(fabsf(v)));
        }
    }
}

// Exact reference-order f64 dot of window i (sketch.py:60): acc = acc + x*w, k ascending.
// (es = float stride of the polyphase elements: 1, or 2 for the paired layout)
__device__ __noinline__ double exact_window_dot(const float *xr, const SketchGeom &g, int i,
                                                const double *w64, int es) {
    double acc = 0.0;
    for (int k = 0; k < g.W; k++) {
        int b = k % g.delta, j = i + k / g.delta;
        double prod = __dmul_rn((double)xr[es * (b * g.PB + poly_off(j))], w64[k]);
        acc = __dadd_rn(acc, prod);
    }
    return acc;
}

__device__ __forceinline__ unsigned decide_bits(const float *acc, int i0, const float *xr,
                                                const SketchGeom &g, float thr,
                                                const double *w64, long long *stats, int es = 1) {
    unsigned byte = 0;
#pragma unroll
    for (int c = 0; c < SK_J; c++) {
        int i = i0 + c;
        if (i < g.nb) {
            bool pos;
            if (fabsf(acc[c]) > thr) {
                pos = acc[c] > 0.f;
            } else {
                double d = exact_window_dot(xr, g, i, w64, es);
                pos = d >= 0.0;
                if (stats) {
                    atomicAdd(reinterpret_cast<unsigned long long *>(&stats[0]), 1ULL);
                    if (fabs(d) < 1e-9)
                        atomicAdd(reinterpret_cast<unsigned long long *>(&stats[1]), 1ULL);
                }
            }
            byte |= (unsigned)pos << c;
        }
    }
    return byte;
}

// W, DELTA compile-time: polyphase sliding-register kernel.
template <int W, int DELTA>
__global__ void __launch_bounds__(SK_THREADS)
sketch_poly_kernel(const float *__restrict__ X, SketchGeom g, const SketchW wp,
                   const double *__restrict__ w64g, uint64_t *__restrict__ bits,
                   long long *stats) {
    extern __shared__ __align__(16) unsigned char sk_smem[];
    float *xs = reinterpret_cast<float *>(sk_smem);
    uint64_t *bs = reinterpret_cast<uint64_t *>(sk_smem + bits_offset(g));
    __shared__ unsigned maxabs[64];
    __shared__ double w64[W];
    for (int k = threadIdx.x; k < W; k += SK_THREADS) w64[k] = w64g[k];

    const int64_t ntiles = (g.N + g.ST - 1) / g.ST;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t s0 = tile * g.ST;
        const int ns = (int)min((int64_t)g.ST, g.N - s0);
        for (int e = threadIdx.x; e < ns * g.words; e += SK_THREADS) bs[e] = 0ULL;
        if (threadIdx.x < ns) maxabs[threadIdx.x] = 0u;
        __syncthreads();
        stage_tile<DELTA>(X, g, s0, ns, xs, maxabs);
        __syncthreads();
        const int item = threadIdx.x;
        if (item < ns * g.G) {
            const int s = item / g.G;
            const int gi = item - s * g.G;
            const float *xr = xs + s * g.P;
            float acc[SK_J];
#pragma unroll
            for (int c = 0; c < SK_J; c++) acc[c] = 0.f;
#pragma unroll
            for (int b = 0; b < DELTA; b++) {
                constexpr int AMAX = (W + DELTA - 1) / DELTA;
                const int A = (W - b + DELTA - 1) / DELTA;
                const float *xb = xr + b * g.PB + 9 * gi;
                float win[SK_J];
#pragma unroll
                for (int c = 0; c < SK_J; c++) win[c] = xb[c];
#pragma unroll
                for (int a = 0; a < AMAX; a++) {
                    if (a < A) {
                        const float wk = wp.w[a * DELTA + b];
#pragma unroll
                        for (int c = 0; c < SK_J; c++) acc[c] = fmaf(win[c], wk, acc[c]);
                        if (a + 1 < A) {
#pragma unroll
                            for (int c = 0; c < SK_J - 1; c++) win[c] = win[c + 1];
                            const int jn = a + SK_J;
                            win[SK_J - 1] = xb[jn + (jn >> 3)];
                        }
                    }
                }
            }
            const float thr = g.screen_c * __uint_as_float(maxabs[s]) + 2e-9f;
            unsigned byte = decide_bits(acc, gi * SK_J, xr, g, thr, w64, stats);
            reinterpret_cast<unsigned char *>(bs)[s * g.words * 8 + gi] = (unsigned char)byte;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ns * g.words; e += SK_THREADS)
            bits[s0 * g.words + e] = bs[e];
        __syncthreads();
    }
}

// W, DELTA compile-time, float4-aligned rows: series are processed in pairs
// so that the f32x2 FMA pipe (FFMA2) does two series' windows per
// instruction.  Pair ps stores element (b, j) of its two series as one float2
// {x_b[j] of series 2ps, of series 2ps + 1} at float index
// 2 (b PB + poly_off(j)) (+ ps * 2P), so the sliding register window moves by
// whole float2 values (no repacking) and each step is one LDS.64 + 8 FFMA2
// for 16 windows.  Each product/sum is the same IEEE f32 fma as in
// sketch_poly_kernel, so screen values and bits are bit-identical.
struct SketchW2 {
    float2 w[SSH_MAX_W];  // {w_k, w_k}
};

#ifndef SK_PAIR_MINB
#define SK_PAIR_MINB 3
#endif
#ifndef SK_LB
#define SK_LB 4
#endif
template <int W, int DELTA>
__global__ void __launch_bounds__(SK_THREADS, SK_PAIR_MINB)
sketch_pair_kernel(const float *__restrict__ X, SketchGeom g, const SketchW2 wp,
                   const double *__restrict__ w64g, uint64_t *__restrict__ bits,
                   long long *stats, unsigned m4magic) {
    extern __shared__ __align__(16) unsigned char sk_smem[];
    float *xs = reinterpret_cast<float *>(sk_smem);  // ST/2 pairs x 2P floats
    uint64_t *bs = reinterpret_cast<uint64_t *>(sk_smem + bits_offset(g));
    __shared__ unsigned maxabs[64];
    __shared__ double w64[W];
    for (int k = threadIdx.x; k < W; k += SK_THREADS) w64[k] = w64g[k];
    const int tid = threadIdx.x;
    const int m4 = g.m >> 2;
    const int64_t ntiles = (g.N + g.ST - 1) / g.ST;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t s0 = tile * g.ST;
        const int ns = (int)min((int64_t)g.ST, g.N - s0);
        for (int e = tid; e < ns * g.words; e += SK_THREADS) bs[e] = 0ULL;
        if (tid < ns) maxabs[tid] = 0u;
        __syncthreads();
        const int total = ns * m4;
        // SK_LB loads in flight per thread before their scatters
        for (int f0 = tid; f0 < total; f0 += SK_LB * SK_THREADS) {
            float4 v4[SK_LB];
#pragma unroll
            for (int u = 0; u < SK_LB; u++) {
                const int f = f0 + u * SK_THREADS;
                if (f < total) {
                    const int s = __umulhi((unsigned)f, m4magic);
                    v4[u] = __ldg(reinterpret_cast<const float4 *>(X + (s0 + s) * g.ld) + (f - s * m4));
                }
            }
#pragma unroll
            for (int u = 0; u < SK_LB; u++) {
                const int f = f0 + u * SK_THREADS;
                if (f < total) {
                    const int s = __umulhi((unsigned)f, m4magic);
                    const int p0 = 4 * (f - s * m4);
                    float *xr = xs + (s >> 1) * 2 * g.P + (s & 1);
                    const float vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
                    float mx = 0.f;
                    int j = p0 / DELTA, b = p0 - j * DELTA;
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        xr[2 * (b * g.PB + poly_off(j))] = vv[e];
                        mx = fmaxf(mx, fabsf(vv[e]));
                        if (++b == DELTA) { b = 0; j++; }
                    }
                    // one smem atomic per warp when its lanes share the series
                    // (lanes hitting one address would serialise 32-fold)
                    const unsigned am = __activemask();
                    const int lead = __ffs(am) - 1;
                    if (__all_sync(am, s == __shfl_sync(am, s, lead))) {
                        const unsigned v = __reduce_max_sync(am, __float_as_uint(mx));
                        if ((int)(threadIdx.x & 31) == lead) atomicMax(&maxabs[s], v);
                    } else {
                        atomicMax(&maxabs[s], __float_as_uint(mx));
                    }
                }
            }
        }
        __syncthreads();
        const int np = (ns + 1) >> 1;
        const int item = tid;
        if (item < np * g.G) {
            const int ps = item / g.G;
            const int gi = item - ps * g.G;
            const float *xr = xs + ps * 2 * g.P;
            float2 acc[SK_J];  // {series 2ps, series 2ps + 1} for windows 8 gi + c
#pragma unroll
            for (int c = 0; c < SK_J; c++) acc[c] = make_float2(0.f, 0.f);
#pragma unroll
            for (int b = 0; b < DELTA; b++) {
                constexpr int AMAX = (W + DELTA - 1) / DELTA;
                const int A = (W - b + DELTA - 1) / DELTA;
                // poly_off(8 gi + k) = 9 gi + k + (k >> 3)
                const float2 *xg = reinterpret_cast<const float2 *>(xr) + b * g.PB + 9 * gi;
                float2 win[SK_J];
#pragma unroll
                for (int c = 0; c < SK_J; c++) win[c] = xg[c];
#pragma unroll
                for (int a = 0; a < AMAX; a++) {
                    if (a < A) {
                        const float2 wk = wp.w[a * DELTA + b];
#pragma unroll
                        for (int c = 0; c < SK_J; c++) acc[c] = __ffma2_rn(win[c], wk, acc[c]);
                        if (a + 1 < A) {
#pragma unroll
                            for (int c = 0; c < SK_J - 1; c++) win[c] = win[c + 1];
                            const int jn = a + SK_J;
                            win[SK_J - 1] = xg[jn + (jn >> 3)];
                        }
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int s = 2 * ps + h;
                if (s < ns) {
                    float accs[SK_J];
#pragma unroll
                    for (int c = 0; c < SK_J; c++) accs[c] = h ? acc[c].y : acc[c].x;
                    const float thr = g.screen_c * __uint_as_float(maxabs[s]) + 2e-9f;
                    unsigned byte = decide_bits(accs, gi * SK_J, xr + h, g, thr, w64, stats, 2);
                    reinterpret_cast<unsigned char *>(bs)[s * g.words * 8 + gi] = (unsigned char)byte;
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < ns * g.words; e += SK_THREADS)
            bits[s0 * g.words + e] = bs[e];
    }
}

// Generic W, delta: one thread per window, taps from shared memory.
__global__ void __launch_bounds__(SK_THREADS)
sketch_generic_kernel(const float *__restrict__ X, SketchGeom g, const SketchW wp,
                      const double *__restrict__ w64g, uint64_t *__restrict__ bits,
                      long long *stats) {
    extern __shared__ __align__(16) unsigned char sk_smem[];
    float *xs = reinterpret_cast<float *>(sk_smem);
    uint64_t *bs = reinterpret_cast<uint64_t *>(sk_smem + bits_offset(g));
    __shared__ unsigned maxabs[64];
    __shared__ double w64[SSH_MAX_W];
    __shared__ float w32[SSH_MAX_W];
    for (int k = threadIdx.x; k < g.W; k += SK_THREADS) {
        w64[k] = w64g[k];
        w32[k] = wp.w[k];
    }
    const int64_t ntiles = (g.N + g.ST - 1) / g.ST;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t s0 = tile * g.ST;
        const int ns = (int)min((int64_t)g.ST, g.N - s0);
        for (int e = threadIdx.x; e < ns * g.words; e += SK_THREADS) bs[e] = 0ULL;
        if (threadIdx.x < ns) maxabs[threadIdx.x] = 0u;
        __syncthreads();
        stage_tile<0>(X, g, s0, ns, xs, maxabs);
        __syncthreads();
        for (int item = threadIdx.x; item < ns * g.nb; item += SK_THREADS) {
            const int s = item / g.nb;
            const int i = item - s * g.nb;
            const float *xr = xs + s * g.P;
            float acc = 0.f;
            for (int k = 0; k < g.W; k++) {
                int b = k % g.delta, j = i + k / g.delta;
                acc = fmaf(xr[b * g.PB + poly_off(j)], w32[k], acc);
            }
            const float thr = g.screen_c * __uint_as_float(maxabs[s]) + 2e-9f;
            bool pos;
            if (fabsf(acc) > thr) {
                pos = acc > 0.f;
            } else {
                double d = exact_window_dot(xr, g, i, w64, 1);
                pos = d >= 0.0;
                if (stats) {
                    atomicAdd(reinterpret_cast<unsigned long long *>(&stats[0]), 1ULL);
                    if (fabs(d) < 1e-9)
                        atomicAdd(reinterpret_cast<unsigned long long *>(&stats[1]), 1ULL);
                }
            }
            if (pos)
                atomicOr(reinterpret_cast<unsigned long long *>(&bs[s * g.words + (i >> 6)]),
                         1ULL << (i & 63));
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ns * g.words; e += SK_THREADS)
            bits[s0 * g.words + e] = bs[e];
        __syncthreads();
    }
}

template <int W, int D>
static bool try_poly(ssh_ctx *ctx, const float *X, SketchGeom &g, const SketchW &wp,
                     uint64_t *bits, int64_t *stats, cudaStream_t st, int *rc) {
    if (g.W != W || g.delta != D) return false;
    size_t smem = sketch_smem(g);
    auto kern = sketch_poly_kernel<W, D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { *rc = ssh_cuda_fail(e, "cudaFuncSetAttribute(sketch)", __FILE__, __LINE__); return true; }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SK_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t ntiles = (g.N + g.ST - 1) / g.ST;
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * per_sm);
    kern<<<grid, SK_THREADS, smem, st>>>(X, g, wp, ctx->d_w64, bits, (long long *)stats); ssh_count_launch();
    e = cudaGetLastError();
    *rc = e == cudaSuccess ? SSH_OK : ssh_cuda_fail(e, "sketch_poly_kernel", __FILE__, __LINE__);
    return true;
}

template <int W, int D>
static bool try_pair(ssh_ctx *ctx, const float *X, const SketchGeom &g0, uint64_t *bits, int64_t *stats,
                     cudaStream_t st, int *rc) {
    if (g0.W != W || g0.delta != D) return false;
    const bool vec = ((g0.ld & 3) == 0) && ((g0.m & 3) == 0) && ((((uintptr_t)X) & 15) == 0);
    static const bool off = [] {
        const char *e = getenv("SSH_SKETCH_PAIR");
        return e && e[0] == '0';
    }();
    if (!vec || off) return false;
    SketchGeom g = g0;
    g.ST = 2 * (SK_THREADS / g.G);  // pairs of series
    if (g.ST < 2 || g.ST > 64) return false;
    const int m4 = g.m >> 2;
    if ((int64_t)g.ST * m4 >= 65536) return false;
    size_t smem = sketch_smem(g);
    if (smem > 200 * 1024) return false;
    // floor(f / m4) = umulhi(f, floor(2^32 / m4) + 1) for f * m4 < 2^32
    const unsigned magic = (unsigned)((1ULL << 32) / (unsigned long long)m4 + 1ULL);
    SketchW2 wp;
    for (int k = 0; k < W; k++) wp.w[k] = make_float2(ctx->h_w32[k], ctx->h_w32[k]);
    auto kern = sketch_pair_kernel<W, D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { *rc = ssh_cuda_fail(e, "cudaFuncSetAttribute(sketch)", __FILE__, __LINE__); return true; }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SK_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t ntiles = (g.N + g.ST - 1) / g.ST;
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * per_sm);
    kern<<<grid, SK_THREADS, smem, st>>>(X, g, wp, ctx->d_w64, bits, (long long *)stats, magic);
    ssh_count_launch();
    e = cudaGetLastError();
    *rc = e == cudaSuccess ? SSH_OK : ssh_cuda_fail(e, "sketch_pair_kernel", __FILE__, __LINE__);
    return true;
}

int ssh_launch_sketch(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
                      int64_t *stats, cudaStream_t st) {
    const ssh_params &p = ctx->p;
    SketchGeom g;
    g.m = p.m; g.nb = ctx->nb; g.words = ctx->words; g.W = p.W; g.delta = p.delta;
    g.N = N; g.ld = ld; g.screen_c = ctx->screen_c;
    g.G = (ctx->nb + SK_J - 1) / SK_J;
    g.ST = SK_THREADS / g.G;
    if (g.ST < 1) g.ST = 1;
    if (g.ST > 64) g.ST = 64;
    // polyphase block: covers j up to 8G + ceil(W/delta) (sliding-window over-read)
    int amax = (p.W + p.delta - 1) / p.delta;
    int jmax = SK_J * g.G + amax + SK_J;
    int jcap = (p.m + p.delta - 1) / p.delta;
    if (jmax < jcap) jmax = jcap;
    g.PB = jmax + (jmax >> 3) + 2;
    int P = p.delta * g.PB;
    while (((P - 9 * g.G) % 32 + 32) % 32 != 0) P++;
    g.P = P;
    size_t smem = sketch_smem(g);
    SSH_REQUIRE(smem <= 200 * 1024, SSH_ERR_UNSUPPORTED,
                "series length %d too long for the sketch kernel's shared-memory tile", p.m);
    SketchW wp;
    memcpy(wp.w, ctx->h_w32, sizeof(float) * p.W);
    int rc = SSH_OK;
    if (p.m >= 4 * SK_J) {
        if (try_pair<80, 3>(ctx, X, g, bits, stats, st, &rc)) return rc;
        if (try_poly<80, 3>(ctx, X, g, wp, bits, stats, st, &rc)) return rc;
        if (try_poly<30, 5>(ctx, X, g, wp, bits, stats, st, &rc)) return rc;
        if (try_poly<30, 4>(ctx, X, g, wp, bits, stats, st, &rc)) return rc;
        if (try_poly<30, 2>(ctx, X, g, wp, bits, stats, st, &rc)) return rc;
        if (try_poly<30, 1>(ctx, X, g, wp, bits, stats, st, &rc)) return rc;
    }
    // generic path: one thread per window
    g.ST = max(1, min(64, 2048 / max(1, ctx->nb)));
    smem = sketch_smem(g);
    SSH_REQUIRE(smem <= 200 * 1024, SSH_ERR_UNSUPPORTED,
                "series length %d too long for the sketch kernel's shared-memory tile", p.m);
    SSH_CUDA(cudaFuncSetAttribute(sketch_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sketch_generic_kernel, SK_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t ntiles = (N + g.ST - 1) / g.ST;
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * per_sm);
    sketch_generic_kernel<<<grid, SK_THREADS, smem, st>>>(X, g, wp, ctx->d_w64, bits,
                                                          (long long *)stats);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}
