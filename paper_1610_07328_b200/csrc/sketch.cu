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
// Kernels (dispatch in ssh_launch_sketch):
//  * sketch_stream_kernel<80,3,20> (float4-aligned rows, m <= ~1500): rows
//    staged by the bulk-copy engine into a ring of shared-memory stages
//    (warp-specialised producer, mbarriers), FFMA2 window pairs with
//    broadcast samples; 4.2 TB/s (64% of HBM) at configs[1].
//  * sketch_pair_kernel / sketch_poly_kernel: polyphase shared-memory layout
//    x_b[j] = x[j*delta + b] (padded by one float per 8, conflict-free stride
//    9) staged by LDG + scatter; used for longer rows (configs[3]).
//  * sketch_generic_kernel: any W, delta.
// All are HBM-bound by design: 4m bytes in + 8*words bytes out per series.
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

// ---------------------------------------------------------------------------
// sketch_stream_kernel<W, D, J>: TMA-staged rows, no polyphase scatter.
//
// A tile of ST series is copied row by row into shared memory by the bulk
// copy engine (cp.async.bulk, one mbarrier per stage, two stages per CTA), so
// the SMs spend no instructions on staging.  Rows keep the HBM layout with a
// stride of an odd number of 16-byte units, so the 8 lanes of each LDS.128
// phase (8 consecutive series, same offset) hit 8 distinct bank quads.
// Thread (s, t) owns windows [J t, J t + J) of series s: J/2 accumulator
// pairs {acc_2q, acc_2q+1}.  Window 2q uses x[6q + d] with tap d and window
// 2q+1 the same sample with tap d - D, so one FFMA2 with the sample broadcast
// and the tap pair WP[d] = {w_d, w_{d-D}} (zero outside [0, W)) advances both
// windows.  Loops run weight-block stationary (blocks of 2D taps, uniform
// registers) over a sliding register window of samples.  Every product/sum is
// an IEEE f32 fma of exact products of f32 inputs and f32 taps, so the same
// (W+2) u sum|x||w| screen bound as sketch_poly_kernel holds (summation order
// does not enter it); the per-thread max|x| over its own sample range bounds
// every window it decides, and the zero tail beyond m only meets zero taps of
// real windows or windows >= nb that are never emitted.
// ---------------------------------------------------------------------------
#ifndef SKS_ST_DEFAULT
#define SKS_ST_DEFAULT 16
#endif

template <int W, int D>
struct SketchWP {
    float2 w[((W + D) + 2 * D - 1) / (2 * D) * (2 * D)];  // {w_d, w_{d-D}}
};

struct StreamGeom {
    int m, nb, words, stride, tps, nstages, ngroups, gthreads;
    int64_t N, ld;
    float screen_c;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
        "[%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ float fmin_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// Exact reference-order f64 dot over a contiguous row window (sketch.py:60).
__device__ __noinline__ double exact_row_dot(const float *x, const double *w64, int W) {
    double d = 0.0;
    for (int k = 0; k < W; k++) d = __dadd_rn(d, __dmul_rn((double)x[k], w64[k]));
    return d;
}

#define SKS_MAXSTAGES 8
#define SKS_MAXG 4

// Warp-specialised pipeline: warp 0 produces (bulk row copies into a ring of
// ns_stages tiles, one full/empty mbarrier pair per stage); consumer groups of
// gthreads threads (ST series x tps window slots) take tiles round-robin, so
// up to ns_stages - ngroups tiles are in flight from HBM while the others are
// computed.
template <int W, int D, int J, int SKS_ST>
__global__ void __launch_bounds__(544)
sketch_stream_kernel(const float *__restrict__ X, StreamGeom g, const SketchWP<W, D> wp,
                     const double *__restrict__ w64g, uint64_t *__restrict__ bits, long long *stats) {
    constexpr int S2 = 2 * D;                        // sample shift between window pairs
    constexpr int NWB = (W + D + S2 - 1) / S2;       // weight blocks of S2 tap pairs
    constexpr int NQ = J / 2;                        // accumulator pairs
    constexpr int NXB = NWB + NQ - 1;                // sample blocks a thread reads
    static_assert(J % 2 == 0, "J even");
    static_assert((J * D) % 4 == 0, "thread sample bases must be 16-byte aligned");
    extern __shared__ __align__(128) unsigned char sks_smem[];
    __shared__ uint64_t full[SKS_MAXSTAGES], empty[SKS_MAXSTAGES];
    __shared__ double w64[W];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int NS = g.nstages, NG = g.ngroups;
    const int stage_floats = SKS_ST * g.stride;
    float *xs = reinterpret_cast<float *>(sks_smem);
    // after the stages: per group, two packed-bit buffers of ST x words
    unsigned long long *wbits_all = reinterpret_cast<unsigned long long *>(xs + (size_t)NS * stage_floats);
    for (int k = tid; k < W; k += nthr) w64[k] = w64g[k];
    // zero tails of every stage (never written by the bulk copies)
    const int tail = g.stride - g.m;
    for (int e = tid; e < NS * SKS_ST * tail; e += nthr) {
        const int r = e / tail;
        xs[r * g.stride + g.m + (e - r * tail)] = 0.f;
    }
    if (tid == 0) {
        for (int i = 0; i < NS; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ntiles = (g.N + SKS_ST - 1) / SKS_ST;
    // this CTA's tiles: blockIdx.x + k gridDim.x, k = 0, 1, ...
    const int64_t nmine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (tid < 32) {
        // producer warp
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
        const unsigned row_bytes = (unsigned)g.m * 4u;
        const int lane = tid;
        for (int64_t k = 0; k < nmine; k++) {
            const int stg = (int)(k % NS);
            if (k >= NS) mbar_wait(&empty[stg], (unsigned)((k / NS) - 1) & 1u);
            const int64_t s0 = (blockIdx.x + k * gridDim.x) * SKS_ST;
            const int ns = (int)min((int64_t)SKS_ST, g.N - s0);
            if (lane == 0) mbar_expect_tx(&full[stg], row_bytes * (unsigned)ns);
            __syncwarp();
            if (lane < ns)
                bulk_g2s(xs + stg * stage_floats + lane * g.stride, X + (s0 + lane) * g.ld, row_bytes,
                         &full[stg], policy);
        }
        return;
    }
    const int ctid = tid - 32;
    const int grp = ctid / g.gthreads;
    if (grp >= NG) return;
    const int gtid = ctid - grp * g.gthreads;
    const int s = gtid % SKS_ST;
    const int t = gtid / SKS_ST;
    const int wpr = g.words;
    int par = 0;
    for (int64_t k = grp; k < nmine; k += NG, par ^= 1) {
        const int stg = (int)(k % NS);
        const int64_t s0 = (blockIdx.x + k * gridDim.x) * SKS_ST;
        const int ns = (int)min((int64_t)SKS_ST, g.N - s0);
        unsigned long long *wbits = wbits_all + (size_t)(2 * grp + par) * SKS_ST * wpr;
        for (int e = gtid; e < SKS_ST * wpr; e += g.gthreads) wbits[e] = 0ULL;
        mbar_wait(&full[stg], (unsigned)(k / NS) & 1u);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(g.gthreads) : "memory");
        if (s < ns && t < g.tps) {
            const float *xr = xs + stg * stage_floats + s * g.stride;
            const float *xt = xr + t * (J * D);
            float2 acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; q++) acc[q] = make_float2(0.f, 0.f);
            float xv[NXB * S2 + 4];  // fully unrolled: registers hold a sliding subset
            float mx = 0.f;
#pragma unroll
            for (int e = 0; e < NQ * S2; e += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(xt + e);
                xv[e] = v.x; xv[e + 1] = v.y; xv[e + 2] = v.z; xv[e + 3] = v.w;
            }
#pragma unroll
            for (int b = 0; b < NWB; b++) {
                // samples of block b + NQ - 1 (the newest block this step needs)
                const int lo = (b + NQ - 1) * S2;
                if (b > 0) {
#pragma unroll
                    for (int e = 0; e < S2; e++) {
                        const int p = lo + e;
                        if ((p & 3) == 0) {
                            const float4 v = *reinterpret_cast<const float4 *>(xt + p);
                            xv[p] = v.x; xv[p + 1] = v.y; xv[p + 2] = v.z; xv[p + 3] = v.w;
                        }
                    }
                }
#pragma unroll
                for (int e = 0; e < S2; e++) {
                    const float2 wk = wp.w[b * S2 + e];
#pragma unroll
                    for (int q = 0; q < NQ; q++) {
                        const float xq = xv[(b + q) * S2 + e];
                        acc[q] = __ffma2_rn(make_float2(xq, xq), wk, acc[q]);
                    }
                }
                // max|x| over the block that leaves the window
#pragma unroll
                for (int e = 0; e < S2; e++) mx = fmaxf(mx, fabsf(xv[b * S2 + e]));
            }
#pragma unroll
            for (int e = NWB * S2; e < NXB * S2; e++) mx = fmaxf(mx, fabsf(xv[e]));
            const float thr = g.screen_c * mx + 2e-9f;
            // branch-free common case: sign bits of the screen values and the NaN-propagating
            // minimum |value| over the thread's valid windows; the exact path runs only when
            // some window is within the screen bound (or NaN)
            const int nval = min(J, g.nb - t * J);
            unsigned neg = 0;
            float amin = __int_as_float(0x7f800000);
            if (nval == J) {
#pragma unroll
                for (int c = 0; c < J; c++) {
                    const float a = (c & 1) ? acc[c >> 1].y : acc[c >> 1].x;
                    neg |= (__float_as_uint(a) >> 31) << c;
                    amin = fmin_nan(amin, fabsf(a));
                }
            } else {
#pragma unroll
                for (int c = 0; c < J; c++) {
                    const float a = (c & 1) ? acc[c >> 1].y : acc[c >> 1].x;
                    if (c < nval) {
                        neg |= (__float_as_uint(a) >> 31) << c;
                        amin = fmin_nan(amin, fabsf(a));
                    }
                }
            }
            unsigned msk = ~neg & (nval >= 32 ? 0xffffffffu : ((1u << nval) - 1u));
            if (!(amin > thr)) {
#pragma unroll
                for (int c = 0; c < J; c++) {
                    const float a = (c & 1) ? acc[c >> 1].y : acc[c >> 1].x;
                    if (c < nval && !(fabsf(a) > thr)) {
                        const int i = t * J + c;
                        const double d = exact_row_dot(xr + i * D, w64, W);
                        msk = d >= 0.0 ? (msk | (1u << c)) : (msk & ~(1u << c));
                        if (stats) {
                            atomicAdd(reinterpret_cast<unsigned long long *>(&stats[0]), 1ULL);
                            if (fabs(d) < 1e-9)
                                atomicAdd(reinterpret_cast<unsigned long long *>(&stats[1]), 1ULL);
                        }
                    }
                }
            }
            const int i0 = t * J;
            const unsigned long long lo = (unsigned long long)msk << (i0 & 63);
            if (lo) atomicOr(&wbits[s * wpr + (i0 >> 6)], lo);
            if ((i0 & 63) + J > 64) {
                const unsigned long long hi = (unsigned long long)msk >> (64 - (i0 & 63));
                if (hi) atomicOr(&wbits[s * wpr + (i0 >> 6) + 1], hi);
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(g.gthreads) : "memory");
        // every thread of the group is done with the stage: release it
        if (gtid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stg])) : "memory");
        for (int e = gtid; e < ns * wpr; e += g.gthreads) bits[s0 * wpr + e] = wbits[e];
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

template <int W, int D, int J, int SKS_ST>
static bool try_stream(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
                       int64_t *stats, cudaStream_t st, int *rc) {
    const ssh_params &p = ctx->p;
    if (p.W != W || p.delta != D) return false;
    static const bool off = [] {
        const char *e = getenv("SSH_SKETCH_STREAM");
        return e && e[0] == '0';
    }();
    const bool vec = ((ld & 3) == 0) && ((p.m & 3) == 0) && ((((uintptr_t)X) & 15) == 0);
    if (off || !vec || N <= 0) return false;
    constexpr int S2 = 2 * D;
    constexpr int NWB = (W + D + S2 - 1) / S2;
    constexpr int NXB = NWB + J / 2 - 1;
    StreamGeom g;
    g.m = p.m; g.nb = ctx->nb; g.words = ctx->words; g.N = N; g.ld = ld; g.screen_c = ctx->screen_c;
    g.tps = (g.nb + J - 1) / J;
    if (g.words > 16) return false;
    g.gthreads = (SKS_ST * g.tps + 31) / 32 * 32;
    if (g.gthreads > 512) return false;
    int need = (g.tps - 1) * J * D + NXB * S2 + 4;
    int stride = std::max(need, g.m);
    stride = (stride + 3) & ~3;
    if (((stride >> 2) & 1) == 0) stride += 4;  // odd number of 16-byte units
    g.stride = stride;
    const size_t stage_bytes = (size_t)SKS_ST * stride * 4;
    static const int env_groups = [] {
        const char *e = getenv("SSH_SKETCH_GROUPS");
        return e ? atoi(e) : 0;
    }();
    g.ngroups = env_groups > 0 ? env_groups : std::max(1, 512 / g.gthreads);
    g.ngroups = std::min(g.ngroups, std::min(SKS_MAXG, 512 / g.gthreads));
    if (g.ngroups < 1) return false;
    const size_t wbits_bytes = (size_t)g.ngroups * 2 * SKS_ST * g.words * 8;
    const size_t smem_cap = 232448 - 4096 - wbits_bytes;
    g.nstages = (int)std::min<size_t>(SKS_MAXSTAGES, smem_cap / stage_bytes);
    if (g.nstages < g.ngroups + 1) return false;
    const int threads = 32 + g.ngroups * g.gthreads;
    const size_t smem = (size_t)g.nstages * stage_bytes + wbits_bytes;
    SketchWP<W, D> wp;
    constexpr int NWP = sizeof(wp.w) / sizeof(wp.w[0]);
    for (int d = 0; d < NWP; d++) {
        const float a = d < W ? ctx->h_w32[d] : 0.f;
        const float b = (d >= D && d - D < W) ? ctx->h_w32[d - D] : 0.f;
        wp.w[d] = make_float2(a, b);
    }
    auto kern = sketch_stream_kernel<W, D, J, SKS_ST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { *rc = ssh_cuda_fail(e, "cudaFuncSetAttribute(sketch_stream)", __FILE__, __LINE__); return true; }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t ntiles = (N + SKS_ST - 1) / SKS_ST;
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * per_sm);
    (void)threads;
    kern<<<grid, threads, smem, st>>>(X, g, wp, ctx->d_w64, bits, (long long *)stats);
    ssh_count_launch();
    e = cudaGetLastError();
    *rc = e == cudaSuccess ? SSH_OK : ssh_cuda_fail(e, "sketch_stream_kernel", __FILE__, __LINE__);
    return true;
}

int ssh_launch_sketch(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
                      int64_t *stats, cudaStream_t st) {
    {
        int rc = SSH_OK;
        if (ctx->p.m >= 64) {
            // J = 20 windows per thread measured best against J = 12 and 16 (configs[1]/[2])
            if (try_stream<80, 3, 20, SKS_ST_DEFAULT>(ctx, X, N, ld, bits, stats, st, &rc)) return rc;
            // long rows (configs[3], m = 2048): 8-series tiles keep a 3-stage ring
            if (try_stream<80, 3, 20, 8>(ctx, X, N, ld, bits, stats, st, &rc)) return rc;
        }
    }
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
