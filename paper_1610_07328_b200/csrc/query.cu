// query.cu — K5..K10: query_index (index.py:204-273) for a batch of queries.
//
// Reference semantics: R = deduplicated union of the L probed buckets
// (index.py:184-190); the result is the exact top-k of R by (DTW^2, id)
// (_cascade_search dtw.py:171-236 visits candidates in (lb, id) order with
// strict pruning, so its result is visit-order independent; SURVEY.md §8a
// A14).  Distances are the reference's f64 values (dtw.py:83-121, FMA-free).
//
// Device pipeline per query batch (all queries in flight at once):
//   probe     binary search of each query key in each table's sorted keys
//   bitmap    membership bitmap of R (warp-aggregated atomicOr over buckets)
//   seeds     LB_PAA (segment-mean envelope bound, from the L2-resident PAA
//             summary of the shard) of every member -> per-query histogram
//             -> the S0 members with the smallest LB_PAA; their fp32 DTW
//             gives thr0 >= the exact k-th best
//   filter    per member: LB_PAA, LB_Kim, then early-abandoning LB_Keogh
//             (query envelope) against thr0; survivors keep their LB_Keogh
//   waves     wave 1 = the W1 smallest-LB survivors (fp32 DTW) -> thr1;
//             wave 2 = remaining survivors with LB <= thr1.  The fp32 DTW
//             abandons on row-min + the remaining rows' LB_Keogh terms
//             (the UCR-suite cumulative bound)
//   rescore   T_k = k-th smallest fp32 DTW; every candidate with
//             d32 <= T_k (1 + eps) is re-evaluated in exact f64
//             (__dsub_rn/__dmul_rn/__dadd_rn in reference order)
//   top-k     (d64, id) order -> ids / squared distances
// eps = (8m + 64) 2^-24 bounds the relative error of every fp32 bound and
// DTW value against the f64 reference values; bounds built on
// stored segment means subtract an explicit absolute error term.  No member
// of the exact top-k is ever pruned, abandoned or left unrescored.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "dtw_warp.cuh"

#define MB_THREADS 256
#define MB_WARPS (MB_THREADS / 32)
#define MB_SLICE_WORDS 256
#define MB_WARP_BYTES (1024 * 6)  // per warp: 1024 u16 member slots + 1024 f32 partial sums
#define NBINS 2048
#define U32_EPS (1.0f / 16777216.0f)

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ unsigned lb_bin(float v) { return min(__float_as_uint(v) >> 20, (unsigned)(NBINS - 1)); }

__device__ int block_sum(int c, int *red) {
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
    return s;
}

// count of entries (over up to two arrays) whose bit pattern is <= v
template <typename U>
__device__ int block_count_le2(const U *a, int na, const U *b, int nb, U v, int *red) {
    int c = 0;
    for (int e = threadIdx.x; e < na; e += blockDim.x) c += a[e] <= v;
    for (int e = threadIdx.x; e < nb; e += blockDim.x) c += b[e] <= v;
    return block_sum(c, red);
}

// smallest v with count(<= v) >= kk over the two arrays (non-negative float/double bits)
template <typename U>
__device__ U block_kth2(const U *a, int na, const U *b, int nb, int kk, U hi, int *red) {
    U lo = 0;
    while (lo < hi) {
        U mid = lo + (hi - lo) / 2;
        if (block_count_le2<U>(a, na, b, nb, mid, red) >= kk) hi = mid; else lo = mid + 1;
    }
    return lo;
}

template <typename K>
__device__ void block_sort_pairs(K *key, uint32_t *val, int P2) {
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = threadIdx.x; idx < (P2 >> 1); idx += blockDim.x) {
                int i = 2 * idx - (idx & (j - 1));
                int l = i + j;
                K a = key[i], b = key[l];
                uint32_t va = val[i], vb = val[l];
                bool gt = (a > b) || (a == b && va > vb);
                bool up = (i & k) == 0;
                if (gt == up) {
                    key[i] = b; key[l] = a;
                    val[i] = vb; val[l] = va;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ float thr_from(float t, float eps) {
    return isinf(t) ? INFINITY : (float)((double)t * (1.0 + (double)eps));
}

// ------------------------------------------------------------------ probe
__global__ void probe_kernel(const uint64_t *__restrict__ qsig, int nq, int L,
                             const uint64_t *__restrict__ keys, const uint32_t *__restrict__ offsets,
                             const int64_t *__restrict__ nbk, const int64_t *__restrict__ kbase,
                             int64_t N, uint64_t *__restrict__ bstart, uint32_t *__restrict__ blen) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq * L) return;
    int q = t / L, j = t - q * L;
    uint64_t key = qsig[(int64_t)q * L + j];
    int64_t nb = nbk[j], kb = kbase[j];
    const uint64_t *kk = keys + kb;
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (kk[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo < nb && kk[lo] == key) {
        uint32_t o0 = offsets[kb + j + lo], o1 = offsets[kb + j + lo + 1];
        bstart[t] = (uint64_t)j * N + o0;
        blen[t] = o1 - o0;
    } else {
        bstart[t] = 0;
        blen[t] = 0;
    }
}

// membership bitmap: blockIdx.x = q*L + j, blockIdx.y strides the bucket
__global__ void bitmap_kernel(const uint32_t *__restrict__ ids, const uint64_t *__restrict__ bstart,
                              const uint32_t *__restrict__ blen, int L, int64_t NW,
                              uint32_t *__restrict__ bitmap) {
    const int qj = blockIdx.x;
    const int q = qj / L;
    const uint32_t len = blen[qj];
    if (len == 0) return;
    const uint32_t *b = ids + bstart[qj];
    uint32_t *bm = bitmap + (int64_t)q * NW;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.y * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.y * blockDim.x + (threadIdx.x & ~31); base < len;
         base += stride) {
        int64_t e = base + lane;
        bool valid = e < len;
        uint32_t row = valid ? b[e] : 0u;
        uint32_t word = valid ? (row >> 5) : 0xFFFFFFFFu;
        unsigned peers = __match_any_sync(0xFFFFFFFFu, word);
        uint32_t bit = valid ? (1u << (row & 31)) : 0u;
        uint32_t all = __reduce_or_sync(peers, bit);
        if (valid && (peers & ((1u << lane) - 1u)) == 0) atomicOr(&bm[word], all);
    }
}


// membership bitmap, one CTA per (query, slice of <= BM_SLICE_WORDS words):
// the slice is built with shared-memory atomics from the sub-range of each
// probed bucket that falls into it (bucket ids are ascending, so two binary
// searches per bucket bound it), then stored with coalesced writes
#define BM_SLICE_WORDS 32768  // 1M rows, 128 KB of shared memory
__global__ void __launch_bounds__(1024)
bitmap_smem_kernel(const uint32_t *__restrict__ ids, const uint64_t *__restrict__ bstart,
                   const uint32_t *__restrict__ blen, int L, int64_t N, int64_t NW, uint32_t *__restrict__ bitmap) {
    extern __shared__ uint32_t bmsm[];
    __shared__ uint32_t slo[64], shi[64];
    const int q = blockIdx.y;
    const int64_t w0 = (int64_t)blockIdx.x * BM_SLICE_WORDS;
    const int nw = (int)min((int64_t)BM_SLICE_WORDS, NW - w0);
    const uint32_t r0 = (uint32_t)(w0 * 32), r1 = (uint32_t)min(N, (w0 + nw) * 32);
    for (int w = threadIdx.x; w < nw; w += blockDim.x) bmsm[w] = 0u;
    if (threadIdx.x < L) {
        const int j = threadIdx.x;
        const uint32_t len = blen[(int64_t)q * L + j];
        const uint32_t *b = ids + bstart[(int64_t)q * L + j];
        // (a slice starting at row 0 / ending at N needs no search on that side:
        // at configs[1] one slice covers the whole shard)
        uint32_t lo = 0, hi = len;
        while (r0 > 0 && lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (b[mid] < r0) lo = mid + 1; else hi = mid;
        }
        slo[j] = lo;
        hi = len;
        uint32_t l2 = (int64_t)r1 >= N ? len : lo;
        while (l2 < hi) {
            const uint32_t mid = (l2 + hi) >> 1;
            if (b[mid] < r1) l2 = mid + 1; else hi = mid;
        }
        shi[j] = l2;
    }
    __syncthreads();
    for (int j = 0; j < L; j++) {
        const uint32_t a = slo[j], e = shi[j];
        if (a >= e) continue;
        const uint32_t *b = ids + bstart[(int64_t)q * L + j];
        for (uint32_t i = a + threadIdx.x; i < e; i += blockDim.x) {
            const uint32_t id = b[i] - r0;
            atomicOr(&bmsm[id >> 5], 1u << (id & 31));
        }
    }
    __syncthreads();
    uint32_t *out = bitmap + (int64_t)q * NW + w0;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) out[w] = bmsm[w];
}

// |R| per query; with fallback, an empty R becomes the whole shard
__global__ void count_kernel(uint32_t *__restrict__ bitmap, int64_t NW, int64_t N,
                             const uint32_t *__restrict__ blen, int L, int fallback,
                             long long *__restrict__ n_cand, int *__restrict__ is_fallback) {
    const int q = blockIdx.x;
    uint32_t *bm = bitmap + (int64_t)q * NW;
    __shared__ int empty;
    if (threadIdx.x == 0) {
        uint64_t s = 0;
        for (int j = 0; j < L; j++) s += blen[(int64_t)q * L + j];
        empty = (s == 0);
        is_fallback[q] = (s == 0 && fallback) ? 1 : 0;
    }
    __syncthreads();
    if (empty && fallback) {
        for (int64_t w = threadIdx.x; w < NW; w += blockDim.x) {
            int64_t rem = N - w * 32;
            bm[w] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
        }
        __syncthreads();
    }
    unsigned long long c = 0;
    for (int64_t w = threadIdx.x; w < NW; w += blockDim.x) c += __popc(bm[w]);
    __shared__ unsigned long long red[32];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
        n_cand[q] = (long long)s;
    }
}

// query envelope (dtw.py:124-151 semantics: max/min over [i-r, i+r]) and its
// per-segment means for the PAA bound, rounded outward past the f64 error
// (Useg >= mean U, Lseg <= mean L; by convexity of max(.,0)^2,
// sum_seg max(x_i - U_i, 0)^2 >= len * max(mean x - mean U, 0)^2).
__global__ void envelope_kernel(const float *__restrict__ Q, int m, int r, int seg, int nseg,
                                float *__restrict__ U, float *__restrict__ Lo,
                                float *__restrict__ Useg, float *__restrict__ Lseg) {
    extern __shared__ float esm[];
    float *su = esm, *sl = esm + m;
    __shared__ float red[32];
    const int q = blockIdx.x;
    const float *y = Q + (int64_t)q * m;
    float amax = 0.f;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        int lo = max(0, i - r), hi = min(m - 1, i + r);
        float mx = y[lo], mn = y[lo];
        for (int j = lo + 1; j <= hi; j++) {
            float v = y[j];
            mx = fmaxf(mx, v);
            mn = fminf(mn, v);
        }
        su[i] = mx;
        sl[i] = mn;
        amax = fmaxf(amax, fmaxf(fabsf(mx), fabsf(mn)));
        U[(int64_t)q * m + i] = mx;
        Lo[(int64_t)q * m + i] = mn;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double mg = (double)red[0] * 0x1p-36;
    for (int s = threadIdx.x; s < nseg; s += blockDim.x) {
        const int a = s * seg, b = min(m, a + seg);
        double su_ = 0.0, sl_ = 0.0;
        for (int i = a; i < b; i++) {
            su_ += (double)su[i];
            sl_ += (double)sl[i];
        }
        Useg[(int64_t)q * nseg + s] = __double2float_ru(su_ / (double)(b - a) + mg);
        Lseg[(int64_t)q * nseg + s] = __double2float_rd(sl_ / (double)(b - a) - mg);
    }
}

// ------------------------------------------------------ shard summaries
// Rerank summaries of every row (layout in common.cuh): one warp per row.
// The row is staged in the warp's shared-memory slice; the per-row grid is
// lo = min x, sc ~ (max x - lo) / 254 with dec(255) >= max x verified; sample
// codes and PAA codes are chosen and verified with the same fp32 dec() the
// query kernels use, so every stored interval provably contains its value.
// The envelope codes come from the sample codes: over the window
// [i - r, i + r] (dtw.py:124-151), U8 = max c + 1 and L8 = min c bracket the
// exact running max / min (dec(c_j) <= x_j <= dec(c_j + 1)), computed by
// byte-packed log-step doubling (__vmaxu4 on the codes and their complements).
__device__ __forceinline__ float sdec(int c, float sc, float lo) { return fmaf((float)c, sc, lo); }

// c in [0, 254] with dec(c) <= v <= dec(c + 1)
__device__ __forceinline__ int code_in(float v, float lo, float sc, float inv) {
    // estimate, then verify both ends with the decoder's own arithmetic
    const float cf = fminf(fmaxf(floorf((v - lo) * inv), 0.f), 254.f);
    if (fmaf(cf, sc, lo) <= v && fmaf(cf + 1.f, sc, lo) >= v) return (int)cf;
    int c = (int)cf;
    for (int it = 0; it < 256 && c > 0 && sdec(c, sc, lo) > v; it++) c--;
    for (int it = 0; it < 256 && c < 254 && sdec(c + 1, sc, lo) < v; it++) c++;
    return c;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

// running max doubling of one padded u16 code array held in registers
// (two codes per word, native VIMNMX.U16x2): lane owns words
// [lane * WPL, lane * WPL + WPL); a word shifted by 2^l elements comes from
// the lane's own registers or, via shuffles, from the next lanes
// (compile-time offsets).  Words at or past padw are 0 (neutral).  A shuffle
// past lane 31 returns the caller's own word; after the levels that garbage
// reaches down to word 32 WPL - 2^(lev-1) at most, so the caller guarantees
// 32 WPL >= padw + 2^(lev-1) and every word written back or read later is exact.  Reads the array from shared memory and
// writes it back.
template <int WPL>
__device__ __forceinline__ void env_doubling16(uint32_t *arr, int padw, int lev, int lane) {
    uint32_t v[WPL];
    const int w0 = lane * WPL;
#pragma unroll
    for (int j = 0; j < WPL; j++) v[j] = w0 + j < padw ? arr[w0 + j] : 0u;
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 12; l++) {
        if (l < lev) {
            const int d = 1 << l;
            const int dq = d >> 1;
            uint32_t nv[WPL];
#pragma unroll
            for (int j = 0; j < WPL; j++) {
                const int k0 = j + dq;
                const uint32_t a0 = k0 < WPL ? v[k0] : __shfl_down_sync(0xFFFFFFFFu, v[k0 % WPL], k0 / WPL);
                uint32_t sh = a0;
                if (d == 1) {  // odd shift: halves of words j and j + 1
                    const int k1 = j + 1;
                    const uint32_t a1 = k1 < WPL ? v[k1] : __shfl_down_sync(0xFFFFFFFFu, v[k1 % WPL], k1 / WPL);
                    sh = __byte_perm(a0, a1, 0x5432u);
                }
                nv[j] = __vmaxu2(v[j], sh);
            }
#pragma unroll
            for (int j = 0; j < WPL; j++) v[j] = nv[j];
        }
    }
#pragma unroll
    for (int j = 0; j < WPL; j++)
        if (w0 + j < padw) arr[w0 + j] = v[j];
    __syncwarp();
}

// element e of a u16 array held as words: the word starting at element e
__device__ __forceinline__ uint32_t u16_word_at(const uint32_t *arr, int e) {
    const int q = e >> 1;
    return (e & 1) ? __byte_perm(arr[q], arr[q + 1], 0x5432u) : arr[q];
}

struct SumArgs {
    const float *X;
    int64_t N, ld, cstride;
    int m, r, lev, pad, seg, nseg, mp, warp_bytes;
    int single;  // one row buffer per warp: the next row streams in while the envelope codes are computed
    uint4 *rec;
    uint8_t *codes;
};

// GEN: the general form (single row buffer and / or odd radius); !GEN is the
// even-radius, double-buffered form with those paths compiled out (configs[1])
template <int WPL, bool GEN>
__global__ void __launch_bounds__(256, (WPL > 0 && WPL <= 13) ? 4 : 1) summaries_kernel(SumArgs a) {
    const bool single = GEN && a.single != 0;
    extern __shared__ __align__(16) unsigned char xsmb[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int m = a.m, pad = a.pad, padw = pad >> 1;
    unsigned char *base = xsmb + (size_t)w * a.warp_bytes;
    const int mq = (m + 3) & ~3;
    float *xbuf = reinterpret_cast<float *>(base);                    // 2 x mq samples (double buffer), or 1 x mq
    uint32_t *cmx = reinterpret_cast<uint32_t *>(xbuf + (single ? 1 : 2) * mq);  // pad u16: codes, 0 outside
    uint32_t *cmn = cmx + padw;                                       // pad u16: 255 - codes, 0 outside
    uint8_t *prec = reinterpret_cast<uint8_t *>(cmn + padw);          // 64-byte record staging
    uint16_t *bmx = reinterpret_cast<uint16_t *>(cmx), *bmn = reinterpret_cast<uint16_t *>(cmn);
    const int win = 2 * a.r + 1;
    const int shw = win - (1 << a.lev);
    const int64_t nwarps = (int64_t)gridDim.x * nwb;
    const bool v16 = ((m & 3) == 0) && ((a.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
    // rows stream into the warp's double buffer with cp.async, one row ahead
    auto prefetch = [&](int64_t rw, float *dst) {
        if (rw < a.N) {
            const float *src = a.X + rw * a.ld;
            if (v16)
                for (int i = 4 * lane; i < m; i += 128) cp_async16(dst + i, src + i);
            else
                for (int i = lane; i < m; i += 32) cp_async4(dst + i, src + i);
        }
        cp_async_commit();
    };
    int64_t row = (int64_t)blockIdx.x * nwb + w;
    prefetch(row, xbuf);
    for (int buf = 0; row < a.N; row += nwarps, buf ^= 1) {
        float *xs = single ? xbuf : xbuf + buf * mq;
        if (single) {
            cp_async_wait0();
        } else {
            prefetch(row + nwarps, xbuf + (buf ^ 1) * mq);
            cp_async_wait1();
        }
        __syncwarp();
        float vmin = INFINITY, vmax = -INFINITY;
        bool fin = true;
        for (int i = lane; i < m; i += 32) {
            const float v = xs[i];
            fin = fin && isfinite(v);
            vmin = fminf(vmin, v);
            vmax = fmaxf(vmax, v);
        }
        for (int t = lane; t < padw; t += 32) {
            cmx[t] = 0u;
            cmn[t] = 0u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            vmin = fminf(vmin, __shfl_xor_sync(0xFFFFFFFFu, vmin, o));
            vmax = fmaxf(vmax, __shfl_xor_sync(0xFFFFFFFFu, vmax, o));
        }
        fin = __all_sync(0xFFFFFFFFu, fin);
        __syncwarp();
        const float lo = vmin;
        float sc = (vmax - lo) * (1.0f / 254.0f);
        if (fin && isfinite(sc)) {
            for (int it = 0; it < 64 && sdec(255, sc, lo) < vmax; it++) sc = nextafterf(sc, INFINITY);
        }
        if (!fin || !isfinite(sc) || sdec(255, sc, lo) < vmax) sc = __int_as_float(0x7FC00000);  // NaN
        const float inv = 1.0f / sc;
        // sample codes, 4 per lane per 128-sample chunk (global) + padded byte arrays (smem)
        uint8_t *cr = a.codes + row * a.cstride;
        // sample j sits at padded element j + rp, rp = r rounded up to even, so whole
        // quads store as aligned u16 pairs for any radius; the window of sample i,
        // [i - r, i + r], is the padded range [i + ro, i + ro + win) with ro = rp - r
        const int ro = GEN ? (a.r & 1) : 0, rp = a.r + ro;
        for (int i4 = 4 * lane; i4 < a.mp; i4 += 128) {
            uint32_t pk = 0;
            if (i4 + 4 <= m) {
                // whole quad: one LDS.128, codes packed as u16 pairs (4-byte aligned: rp even)
                const float4 x4 = *reinterpret_cast<const float4 *>(xs + i4);
                const int c0 = code_in(x4.x, lo, sc, inv), c1 = code_in(x4.y, lo, sc, inv);
                const int c2 = code_in(x4.z, lo, sc, inv), c3 = code_in(x4.w, lo, sc, inv);
                pk = (uint32_t)c0 | ((uint32_t)c1 << 8) | ((uint32_t)c2 << 16) | ((uint32_t)c3 << 24);
                const uint32_t w01 = (uint32_t)c0 | ((uint32_t)c1 << 16), w23 = (uint32_t)c2 | ((uint32_t)c3 << 16);
                const int wi = (rp + i4) >> 1;
                cmx[wi] = w01;
                cmx[wi + 1] = w23;
                cmn[wi] = 0x00FF00FFu - w01;
                cmn[wi + 1] = 0x00FF00FFu - w23;
            } else {
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int i = i4 + t;
                    if (i < m) {
                        const int c = code_in(xs[i], lo, sc, inv);
                        pk |= (uint32_t)c << (8 * t);
                        bmx[rp + i] = (uint16_t)c;
                        bmn[rp + i] = (uint16_t)(255 - c);
                    }
                }
            }
            *reinterpret_cast<uint32_t *>(cr + i4) = pk;
        }
        // PAA codes of the segment means (f64 sums); a mean with a grid point
        // within its f64 error margin makes the row's PAA codes unusable (flag)
        const double amax = fmax(fabs((double)lo), fabs((double)vmax));
        const double mg = amax * 0x1p-36;
        bool ambiguous = false;
        for (int s = lane; s < SSH_REC_CODES; s += 32) {
            int c = 0;
            if (s < a.nseg) {
                const int b0 = s * a.seg, b1 = min(m, b0 + a.seg);
                double sum = 0.0;
                for (int i = b0; i < b1; i++) sum += (double)xs[i];
                const double md = sum / (double)(b1 - b0);
                c = __double2int_rd((md - (double)lo) * (double)inv);
                c = min(max(c, 0), 254);
                for (int it = 0; it < 256 && c > 0 && (double)sdec(c, sc, lo) > md - mg; it++) c--;
                for (int it = 0; it < 256 && c < 254 && (double)sdec(c + 1, sc, lo) < md - mg; it++) c++;
                if ((c > 0 && (double)sdec(c, sc, lo) > md - mg) ||
                    (c < 254 && (double)sdec(c + 1, sc, lo) < md + mg))
                    ambiguous = true;  // a grid point within the f64 error of the mean
            }
            prec[16 + s] = (uint8_t)c;
        }
        // a row with an ambiguous segment mean carries -sc: its PAA codes are
        // not used (the key falls back to LB_Kim); decoders take |sc|
        ambiguous = __any_sync(0xFFFFFFFFu, ambiguous);
        if (lane == 0) *reinterpret_cast<float4 *>(prec) = make_float4(lo, ambiguous ? -sc : sc, xs[0], xs[m - 1]);
        __syncwarp();
        if (lane < 4) a.rec[row * 4 + lane] = reinterpret_cast<const uint4 *>(prec)[lane];
        // long rows keep one row buffer (more resident warps): the samples are not
        // read again, so the next row streams in under the envelope stage
        if (single) prefetch(row + nwarps, xbuf);
        // running max of the codes and of their complements (= running min) over
        // [t, t + 2^lev) by byte-packed log-step doubling
        if (WPL > 0) {
            env_doubling16<(WPL > 0 ? WPL : 1)>(cmx, padw, a.lev, lane);
            env_doubling16<(WPL > 0 ? WPL : 1)>(cmn, padw, a.lev, lane);
        } else {
            for (int l = 0; l < a.lev; l++) {
                const int d = 1 << l, dq = d >> 1;
                const unsigned sel = d & 1 ? 0x5432u : 0x3210u;
                for (int t0 = 0; t0 < padw; t0 += 32 * 8) {
                    uint32_t va[8], vb[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int t = t0 + u * 32 + lane;
                        if (t < padw) {
                            const int q0 = t + dq;
                            const uint32_t a0 = q0 < padw ? cmx[q0] : 0u, a1 = q0 + 1 < padw ? cmx[q0 + 1] : 0u;
                            const uint32_t b0 = q0 < padw ? cmn[q0] : 0u, b1 = q0 + 1 < padw ? cmn[q0 + 1] : 0u;
                            va[u] = __vmaxu2(cmx[t], __byte_perm(a0, a1, sel));
                            vb[u] = __vmaxu2(cmn[t], __byte_perm(b0, b1, sel));
                        }
                    }
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int t = t0 + u * 32 + lane;
                        if (t < padw) {
                            cmx[t] = va[u];
                            cmn[t] = vb[u];
                        }
                    }
                    __syncwarp();
                }
            }
        }
        // envelope codes of samples i4..i4+3: window [i - r, i + r] = padded
        // [i, i + win) = max over [i, i + 2^lev) and [i + shw, i + shw + 2^lev);
        // U8 = max code + 1 (dec(c + 1) >= x), L8 = min code (dec(c) <= x)
        {
            for (int i4 = 4 * lane; i4 < a.mp; i4 += 128) {
                uint2 out = make_uint2(0x00FF00FFu, 0x00FF00FFu);  // U8 = 255, L8 = 0
                if (i4 < m) {
                    // padded element i of sample i (window [i - r, i + r] -> [i, i + win))
                    const int e4 = i4 + ro;  // window start of sample i4 (see rp above)
                    uint32_t a01, a23, b01, b23;  // the words at the window start (aligned when r is even)
                    if (ro == 0) {
                        a01 = cmx[i4 >> 1]; a23 = cmx[(i4 >> 1) + 1];
                        b01 = cmn[i4 >> 1]; b23 = cmn[(i4 >> 1) + 1];
                    } else {
                        a01 = u16_word_at(cmx, e4); a23 = u16_word_at(cmx, e4 + 2);
                        b01 = u16_word_at(cmn, e4); b23 = u16_word_at(cmn, e4 + 2);
                    }
                    const uint32_t u01 = __vmaxu2(a01, u16_word_at(cmx, e4 + shw)) + 0x00010001u;
                    const uint32_t u23 = __vmaxu2(a23, u16_word_at(cmx, e4 + 2 + shw)) + 0x00010001u;
                    const uint32_t l01 = __vmaxu2(b01, u16_word_at(cmn, e4 + shw)) ^ 0x00FF00FFu;
                    const uint32_t l23 = __vmaxu2(b23, u16_word_at(cmn, e4 + 2 + shw)) ^ 0x00FF00FFu;
                    out = make_uint2(__byte_perm(u01, l01, 0x6240u), __byte_perm(u23, l23, 0x6240u));
                }
                *reinterpret_cast<uint2 *>(cr + a.mp + 2 * i4) = out;
            }
        }
        __syncwarp();
    }
}

struct SumGeom {
    int seg, nseg, mp, lev, pad, warp_bytes, nwb, single;
};

static int summaries_geom(const ssh_ctx *ctx, SumGeom &g) {
    const int m = ctx->p.m, r = ctx->p.radius;
    g.seg = (m + SSH_REC_CODES - 1) / SSH_REC_CODES;
    g.nseg = (m + g.seg - 1) / g.seg;
    g.mp = ((m + 127) / 128) * 128;
    g.lev = 0;
    while ((2 << g.lev) <= 2 * r + 1) g.lev++;
    // padded u16 code arrays: sample j at element j + r; the last doubling read
    // reaches element (m - 1) + 2r + 2^lev + 3; 4 pad % 16 == 0 keeps the record aligned
    g.pad = ((m + 2 * r + (1 << g.lev) + 12 + (r & 1)) + 7) & ~7;  // + 1: odd radii shift the samples by one element
    // rows longer than 512 samples keep a single row buffer per warp (see the kernel);
    // SSH_SUM_SINGLE=0/1 forces either form
    g.single = m > 512;
    if (const char *ev = getenv("SSH_SUM_SINGLE")) g.single = atoi(ev) != 0;
    g.warp_bytes = (((m + 3) & ~3) * (g.single ? 4 : 8) + 4 * g.pad + 64 + 15) & ~15;
    g.nwb = (int)std::min<size_t>(8, (200 * 1024) / (size_t)g.warp_bytes);
    // two or three blocks per SM when the rows are too long for 8 warps of one block
    {
        const int fit = (int)((200 * 1024) / (size_t)g.warp_bytes);  // warps per SM by shared memory
        if (fit >= 10 && fit < 16) g.nwb = fit / 2;                  // two smaller blocks (registers allow it)
    }
    SSH_REQUIRE(g.nwb >= 1, SSH_ERR_UNSUPPORTED, "series too long for the summaries kernel (m=%d, r=%d)", m, r);
    return SSH_OK;
}

int ssh_alloc_summaries(ssh_ctx *ctx, ssh_index *ix, int64_t N, cudaStream_t st) {
    SumGeom g;
    int rc = summaries_geom(ctx, g);
    if (rc) return rc;
    if (!ix->rec) {
        SSH_CUDA(cudaMallocAsync(&ix->rec, (size_t)64 * N, st));
        cudaError_t e = cudaMallocAsync((void **)&ix->codes, (size_t)3 * g.mp * N, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(ix->rec, st);
            ix->rec = nullptr;
            return ssh_cuda_fail(e, "rerank summaries (3 m bytes per series)", __FILE__, __LINE__);
        }
    }
    ix->seg = g.seg;
    ix->nseg = g.nseg;
    ix->mp = g.mp;
    ix->cstride = (int64_t)3 * g.mp;
    return SSH_OK;
}

int ssh_launch_summaries_rows(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t r0, int64_t n, int64_t ld,
                              cudaStream_t st) {
    if (n <= 0) return SSH_OK;
    SumGeom g;
    int rc = summaries_geom(ctx, g);
    if (rc) return rc;
    const int m = ctx->p.m, r = ctx->p.radius;
    SumArgs a{X, n, ld, ix->cstride, m, r, g.lev, g.pad, g.seg, g.nseg, g.mp, g.warp_bytes, g.single,
              (uint4 *)ix->rec + r0 * 4, ix->codes + r0 * ix->cstride};
    const size_t smem = (size_t)g.warp_bytes * g.nwb;
    // envelope doubling in registers when the padded array fits 32 x WPL words
    // (zero margin of 2^(lev-1) words past padw: see env_doubling16)
    const int need = g.pad / 2 + (1 << g.lev) / 2;
    // odd words-per-lane: lane l's chunk starts at word l * WPL, and an odd stride
    // spreads the 32 lanes over all banks (WPL = 48 was a 16-way conflict on every
    // shared-memory access of the doubling, 24 an 8-way one)
    const bool gen = g.single || (r & 1);
    auto kern = need <= 32 * 10 ? (gen ? summaries_kernel<10, true> : summaries_kernel<10, false>)
                : need <= 32 * 11 ? (gen ? summaries_kernel<11, true> : summaries_kernel<11, false>)
                : need <= 32 * 13 ? (gen ? summaries_kernel<13, true> : summaries_kernel<13, false>)
                : need <= 32 * 25 ? summaries_kernel<25, true>
                : need <= 32 * 49 ? summaries_kernel<49, true> : summaries_kernel<0, true>;
    SSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * g.nwb, smem);
    if (const char *ev = getenv("SSH_SUM_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(ev)));
    const int grid = (int)std::min<int64_t>((n + g.nwb - 1) / g.nwb, (int64_t)ctx->num_sms * std::max(1, per_sm));
    kern<<<grid, 32 * g.nwb, smem, st>>>(a);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

int ssh_launch_summaries(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t N, int64_t ld,
                         cudaStream_t st) {
    int rc = ssh_alloc_summaries(ctx, ix, N, st);
    if (rc) return rc;
    return ssh_launch_summaries_rows(ctx, ix, X, 0, N, ld, st);
}

extern "C" int ssh_index_copy_summaries(const ssh_index *ix, int64_t r0, int64_t n, void *rec_out,
                                        void *codes_out, int32_t *mp, int64_t *cstride, void *stream) {
    SSH_REQUIRE(ix, SSH_ERR_INVALID, "ssh_index_copy_summaries: NULL index");
    SSH_REQUIRE(ix->rec && ix->codes, SSH_ERR_STATE, "ssh_index_copy_summaries: index has no summaries");
    SSH_REQUIRE(r0 >= 0 && n >= 0 && r0 + n <= ix->N, SSH_ERR_INVALID,
                "ssh_index_copy_summaries: rows [%lld, %lld) outside [0, %lld)", (long long)r0,
                (long long)(r0 + n), (long long)ix->N);
    SSH_CUDA(cudaSetDevice(ix->device));
    if (mp) *mp = ix->mp;
    if (cstride) *cstride = ix->cstride;
    cudaStream_t st = (cudaStream_t)stream;
    if (rec_out && n)
        SSH_CUDA(cudaMemcpyAsync(rec_out, (const uint8_t *)ix->rec + 64 * r0, (size_t)64 * n,
                                 cudaMemcpyDefault, st));
    if (codes_out && n)
        SSH_CUDA(cudaMemcpyAsync(codes_out, ix->codes + ix->cstride * r0, (size_t)ix->cstride * n,
                                 cudaMemcpyDefault, st));
    SSH_CUDA(cudaStreamSynchronize(st));
    return SSH_OK;
}

extern "C" int ssh_index_summarize(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t ld,
                                   void *stream) {
    SSH_REQUIRE(ctx && ix && X, SSH_ERR_INVALID, "ssh_index_summarize: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_index_summarize: params not set");
    SSH_REQUIRE(ld >= ctx->p.m, SSH_ERR_INVALID, "ssh_index_summarize: ld < m");
    SSH_CUDA(cudaSetDevice(ctx->device));
    int rc = ssh_launch_summaries(ctx, ix, X, ix->N, ld, (cudaStream_t)stream);
    if (rc == SSH_OK) ssh_index_touch(ix, (cudaStream_t)stream);
    return rc;
}

// --------------------------------------------------- LB_PAA of every member
// One CTA per (query, slice of MB_SLICE_WORDS bitmap words).  A warp turns 32
// words into a member list in shared memory and evaluates lane-per-member the
// summary key from the member's 64-byte record (L2-resident for shards up to
// ~2M rows):
//   LB_PAA = shrink * sum_seg len * max(dec(c) - Useg, Lseg - dec(c+1), 0)^2
//   LB_Kim = (x_0 - q_0)^2 + (x_last - q_last)^2            (dtw.py:154-160)
//   key    = max(LB_PAA, LB_Kim), bit 0 = "LB_Kim is the larger" (the key is
//            first lowered by >= 1 ulp, so setting the bit keeps it a bound)
// shrink = 1 - (3 nseg + 8) u absorbs the fp32 evaluation error.
// SAMPLE: members of every 8th bitmap word only; their key bins go to a
// per-query histogram (cutoff choice).  Otherwise members whose key bin lies
// in [binlo_q, binhi_q] are appended to the query's list; the LB_PAA sum is
// abandoned once a partial sum passes the upper bin (a partial sum is a lower
// bound of the key).
struct PaaArgs {
    const float *Useg, *Lseg, *Q;
    const uint4 *rec;
    const uint32_t *bitmap;
    const int64_t *roff;  // per-query CSR offset of the member list
    uint32_t *rows;
    float *lb;
    int *cnt;
    const int *binlo, *binhi;  // per query (full pass)
    unsigned *hist;            // [q][NBINS] (sample pass)
    int64_t NW;
    int m, seg, nseg;
};

// 256-bit read-only global load (sm_100 LDG.E.ENL2.256): p 32-byte aligned
struct __align__(32) U32x8 {
    uint32_t v[8];
};
__device__ __forceinline__ U32x8 ldg256(const void *p) {
    U32x8 r;
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
    return r;
}

__device__ __forceinline__ float code_f(uint32_t w, int t) {
    // byte t of w as an exact float (0x4B0000cc = 2^23 + cc)
    return __uint_as_float(__byte_perm(w, 0x4B000000u, (unsigned)t | 0x7440u)) - 8388608.f;
}

#ifndef SAMPLE_SHIFT
#define SAMPLE_SHIFT 5  // sample pass: bitmap words w with w % 32 == 0 (3: 27.9 ms, 4: 27.3, 5: 27.0 per 1000-query batch)
#endif

template <bool SAMPLE>
__global__ void __launch_bounds__(MB_THREADS) paa_members_kernel(PaaArgs a) {
    extern __shared__ __align__(16) unsigned char msm[];
    __shared__ float2 sUL[SSH_REC_CODES];  // {-Useg, Lseg}
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nseg = a.nseg;
    // member slots hold the bit position within the warp's 32-word chunk
    // (lane of the word * 32 + bit), 2 bytes each: 6 KB per warp, 4 blocks/SM
    uint16_t *list = reinterpret_cast<uint16_t *>(msm) + w * 1024;
    float *accb = reinterpret_cast<float *>(msm + MB_WARPS * 2048) + w * 1024;
    unsigned *shist = reinterpret_cast<unsigned *>(msm + MB_WARPS * MB_WARP_BYTES);  // SAMPLE: NBINS
    int blo = 0, bhi = NBINS - 1;
    if (!SAMPLE) {
        blo = a.binlo[q];
        bhi = a.binhi[q];
        if (blo > bhi) return;  // block-uniform: nothing to collect for this query
    }
    for (int s = threadIdx.x; s < SSH_REC_CODES; s += MB_THREADS) {
        // unused segments contribute max(dec - inf, -inf - dec, 0) = 0
        sUL[s] = s < nseg ? make_float2(-a.Useg[(int64_t)q * nseg + s], a.Lseg[(int64_t)q * nseg + s])
                          : make_float2(-INFINITY, -INFINITY);
    }
    if (SAMPLE)
        for (int b = threadIdx.x; b < NBINS; b += MB_THREADS) shist[b] = 0u;
    __syncthreads();
    const float q0 = a.Q[(int64_t)q * a.m], ql = a.Q[(int64_t)q * a.m + a.m - 1];
    const float segf = (float)a.seg;
    const float lastlen = (float)(a.m - (nseg - 1) * a.seg);
    // fp32 evaluation error of the weighted sum, including the last-segment
    // correction (cancellation relative to seg / lastlen)
    const float shrink = 1.f - (3.f * nseg + 12.f + 4.f * segf / lastlen) * U32_EPS;
    const float wseg = segf;
    // smallest key value in bin bhi + 1: keys at or above it are dropped
    const float edge = bhi >= NBINS - 1 ? INFINITY : __uint_as_float((uint32_t)(bhi + 1) << 20);
    const uint32_t *bm = a.bitmap + (int64_t)q * a.NW;
    const int64_t base_q = a.roff[q];
    // a sample block covers 2^SAMPLE_SHIFT slices (same sampled words per block)
    const int64_t slice = SAMPLE ? ((int64_t)MB_SLICE_WORDS << SAMPLE_SHIFT) : MB_SLICE_WORDS;
    const int64_t s0 = (int64_t)blockIdx.x * slice;
    const int64_t s1 = min(a.NW, s0 + slice);
    const int wstep = SAMPLE ? (32 << SAMPLE_SHIFT) : 32;
    for (int64_t wb = s0 + (int64_t)wstep * w; wb < s1; wb += (int64_t)wstep * MB_WARPS) {
        const int64_t wd = wb + (SAMPLE ? ((int64_t)lane << SAMPLE_SHIFT) : lane);
        uint32_t word = wd < s1 ? bm[wd] : 0u;
        const int c = __popc(word);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (total == 0) continue;
        int pos = incl - c;
        while (word) {
            int b = __ffs(word) - 1;
            word &= word - 1;
            SSH_DASSERT(pos < 1024);
            list[pos++] = (uint16_t)(lane * 32 + b);
        }
        __syncwarp();
        // slot -> series row (the sample pass strides its words by 2^SAMPLE_SHIFT)
        const int64_t row0 = wb * 32;
        auto slot_row = [&](uint32_t sl) -> uint32_t {
            return (uint32_t)(row0 + (SAMPLE ? ((int64_t)(sl >> 5) << (5 + SAMPLE_SHIFT)) + (sl & 31u) : (int64_t)sl));
        };
        // three passes over the list, one 16-segment group each; after each
        // pass the members still below the edge are compacted in place (rows
        // in list, partial sums in accb) so every pass runs on full warps
        int n = total;
        for (int g = 0; g < 3 && n > 0; g++) {
            int nk = 0;
            // the next 32 members' records are loaded one iteration ahead (L2
            // latency overlaps this iteration's arithmetic); compaction only
            // writes list/accb below e0 + 32, ahead of the prefetched entries
            uint32_t rowN = 0, slN = 0;
            float accN = 0.f;
            float4 hN = make_float4(0.f, 0.f, 0.f, 0.f);  // lo, sc, x_0, x_last
            uint4 cgN = make_uint4(0u, 0u, 0u, 0u);
            auto fetch = [&](int e) {
                if (e < n) {
                    slN = list[e];
                    rowN = slot_row(slN);
                    accN = g ? accb[e] : 0.f;
                    const uint4 *rp = a.rec + (int64_t)rowN * 4;
                    if (g == 0) {
                        // header and the first code group share the record's first 32-byte
                        // sector: one 256-bit gather instead of two (the kernel is bound by
                        // the L1 tag stage of these scattered loads)
                        const U32x8 v = ldg256(rp);
                        hN = make_float4(__uint_as_float(v.v[0]), __uint_as_float(v.v[1]), 0.f, 0.f);
                        cgN = make_uint4(v.v[4], v.v[5], v.v[6], v.v[7]);
                    } else if (g == 1) {
                        const float2 h2 = __ldg(reinterpret_cast<const float2 *>(rp));
                        hN = make_float4(h2.x, h2.y, 0.f, 0.f);
                        cgN = __ldg(rp + 2);
                    } else {
                        // the last pass also needs x_0 / x_last (LB_Kim): the whole header in one gather
                        hN = __ldg(reinterpret_cast<const float4 *>(rp));
                        cgN = __ldg(rp + 3);
                    }
                }
            };
            fetch(lane);
            for (int e0 = 0; e0 < n; e0 += 32) {
                const int e = e0 + lane;
                bool keep = false;
                float acc = accN, key = 0.f;
                const uint32_t row = rowN, sl = slN;
                const float4 h = hN;
                const uint4 cg = cgN;
                fetch(e + 32);
                if (e < n) {
                    const uint4 *rp = a.rec + (int64_t)row * 4;
                    // flagged rows (-sc): NaN scale -> every PAA term max(NaN, ..., 0) = 0
                    const float lo = h.x, sc = h.y >= 0.f ? h.y : __int_as_float(0x7FC00000);
                    const uint32_t cw[4] = {cg.x, cg.y, cg.z, cg.w};
                    // packed f32x2, the same IEEE operations as the scalar
                    // forms: {xa, xb} = fma({c, c + 1}, sc, lo) and
                    // {xa - U, L - xb} = fma({xa, xb}, {1, -1}, {-U, L})
                    // upper end: fma(c, sc, lo_hi) with lo_hi = RU(lo + sc) is never below
                    // dec(c + 1) = fma(c + 1, sc, lo) (c sc + lo_hi >= (c + 1) sc + lo before
                    // the one rounding), so it still brackets the mean from above; one scalar
                    // FADD converts the code instead of an f32x2 add with a constant pair
                    const float2 sc2 = make_float2(sc, sc), loh = make_float2(lo, __fadd_ru(lo, sc));
                    const float2 pm = make_float2(1.f, -1.f);
                    float2 acc2 = make_float2(acc, 0.f);
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        float ev[2];
#pragma unroll
                        for (int u = 0; u < 2; u++) {
                            const int jj = j + u;
                            const float r = __uint_as_float(__byte_perm(cw[jj >> 2], 0x4B000000u,
                                                                        (unsigned)(jj & 3) | 0x7440u));
                            const float cf = r - 8388608.f;
                            const float2 x = __ffma2_rn(make_float2(cf, cf), sc2, loh);
                            const float2 df = __ffma2_rn(x, pm, sUL[16 * g + jj]);
                            ev[u] = fmaxf(fmaxf(df.x, df.y), 0.f);
                        }
                        // weight seg for every segment; the last is fixed below
                        acc2 = __ffma2_rn(make_float2(ev[0], ev[1]), make_float2(ev[0], ev[1]), acc2);
                    }
                    acc = acc2.x + acc2.y;
                    if (g < 2) {
                        keep = SAMPLE || acc * wseg * shrink * (1.f - 4.f * U32_EPS) < edge;
                    } else {
                        // the last segment has lastlen <= seg samples: remove its excess weight
                        const int sg = nseg - 1;
                        // its code word is in this pass's group when sg >= 32 (no extra gather)
                        const int wi = (sg >> 2) - 8;
                        const uint32_t lw = wi < 0 ? __ldg(reinterpret_cast<const uint32_t *>(rp) + 4 + (sg >> 2))
                                            : wi == 0 ? cg.x : wi == 1 ? cg.y : wi == 2 ? cg.z : cg.w;
                        const float cf = code_f(lw, sg & 3);
                        const float ev = fmaxf(fmaxf(fmaf(cf, sc, lo) + sUL[sg].x, sUL[sg].y - fmaf(cf + 1.f, sc, lo)), 0.f);
                        const float paa = fmaxf(fmaf(-(segf - lastlen) * ev, ev, acc * segf), 0.f) * shrink;
                        const float d0 = h.z - q0, dl = h.w - ql;
                        const float kim = a.m >= 2 ? fmaf(dl, dl, d0 * d0) : d0 * d0;
                        if (kim > paa) key = __uint_as_float(__float_as_uint(kim * (1.f - 2.f * U32_EPS)) | 1u);
                        else key = __uint_as_float(__float_as_uint(paa) & ~1u);
                        const int kb = (int)lb_bin(key);
                        keep = kb >= blo && kb <= bhi;
                    }
                }
                if (g < 2) {
                    const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
                    __syncwarp();
                    if (keep) {
                        const int p = nk + __popc(km & ((1u << lane) - 1u));
                        list[p] = (uint16_t)sl;
                        accb[p] = acc;
                    }
                    nk += __popc(km);
                    __syncwarp();
                } else if (SAMPLE) {
                    const unsigned bin = keep ? lb_bin(key) : 0xFFFFFFFFu;
                    const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
                    if (keep && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&shist[bin], (unsigned)__popc(peers));
                } else {
                    // kept members compact in place like the earlier passes (rows in
                    // list, keys in accb); the chunk's kept run is reserved with one
                    // atomic and copied out after the pass
                    const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
                    __syncwarp();
                    if (keep) {
                        const int p = nk + __popc(km & ((1u << lane) - 1u));
                        list[p] = (uint16_t)sl;
                        accb[p] = key;
                    }
                    nk += __popc(km);
                    __syncwarp();
                }
            }
            if (!SAMPLE && g == 2 && nk > 0) {
                int dst = 0;
                if (lane == 0) dst = atomicAdd(&a.cnt[q], nk);
                dst = __shfl_sync(0xFFFFFFFFu, dst, 0);
                SSH_DASSERT(base_q + dst + nk <= a.roff[q + 1]);
                for (int e = lane; e < nk; e += 32) {
                    a.rows[base_q + dst + e] = slot_row(list[e]);
                    a.lb[base_q + dst + e] = accb[e];
                }
            }
            n = nk;
        }
        __syncwarp();
    }
    if (SAMPLE) {
        __syncthreads();
        for (int b = threadIdx.x; b < NBINS; b += MB_THREADS)
            if (shist[b]) atomicAdd(&a.hist[(int64_t)q * NBINS + b], shist[b]);
    }
}

// Per-query member cutoff from the sampled key histogram: the smallest bin b
// whose sampled cumulative count reaches target >> SAMPLE_SHIFT (all bins when
// the sample is smaller).  Round 0 keeps bins [0, b]; overflow rounds [b+1, ...).
__global__ void cutoff_kernel(const unsigned *__restrict__ hist, int target, int *__restrict__ binlo,
                              int *__restrict__ binhi) {
    __shared__ unsigned part[256];
    const int q = blockIdx.x;
    constexpr int PER = NBINS / 256;
    const unsigned *hq = hist + (int64_t)q * NBINS;
    unsigned loc = 0;
    for (int i = 0; i < PER; i++) loc += hq[threadIdx.x * PER + i];
    part[threadIdx.x] = loc;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const unsigned v = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    // at least one sampled member: need = 0 would leave binhi unset
    const unsigned need = max(1u, (unsigned)(target >> SAMPLE_SHIFT));
    const unsigned before = part[threadIdx.x] - loc;
    if (threadIdx.x == 0) {
        binlo[q] = 0;
        if (part[255] < need) binhi[q] = NBINS - 1;
    }
    if (part[255] >= need && before < need && part[threadIdx.x] >= need) {
        unsigned run = before;
        int b = threadIdx.x * PER;
        for (int i = 0; i < PER; i++) {
            run += hq[threadIdx.x * PER + i];
            if (run >= need) {
                b = threadIdx.x * PER + i;
                break;
            }
        }
        binhi[q] = b;
    }
}

// overflow round: queries whose round-0 list ran out below their threshold get
// the bins above their cutoff; the others get an empty window
__global__ void overflow_window_kernel(const int *__restrict__ overflow, int nq, int *__restrict__ binlo,
                                       int *__restrict__ binhi) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    if (overflow[q]) {
        binlo[q] = binhi[q] + 1;
        binhi[q] = NBINS - 1;
    } else {
        binlo[q] = NBINS;
        binhi[q] = NBINS - 1;
    }
}

// Per query: members reordered by LB bin (float bits >> 20, ~12% wide) with a
// counting sort; within a bin the order is arbitrary (the wave loop relies
// only on non-decreasing bins).
__global__ void __launch_bounds__(1024)
binsort_kernel(const uint32_t *__restrict__ rows_in, const float *__restrict__ lb_in,
               const int64_t *__restrict__ roff, const int *__restrict__ cnt,
               uint32_t *__restrict__ rows_out, float *__restrict__ lb_out) {
    __shared__ uint32_t h[NBINS];
    __shared__ uint32_t part[1024];
    const int q = blockIdx.x;
    const int64_t o = roff[q];
    const int n = cnt[q];
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // warp-aggregated counting: LB values cluster in few bins
    for (int e0 = 0; e0 < n; e0 += blockDim.x) {
        const int e = e0 + threadIdx.x;
        const unsigned bin = e < n ? lb_bin(lb_in[o + e]) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        if (e < n && (peers & lt) == 0) atomicAdd(&h[bin], (uint32_t)__popc(peers));
    }
    __syncthreads();
    const int per = NBINS / blockDim.x;
    uint32_t loc = 0;
    for (int i = 0; i < per; i++) loc += h[threadIdx.x * per + i];
    part[threadIdx.x] = loc;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        uint32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - loc;
    for (int i = 0; i < per; i++) {
        uint32_t c = h[threadIdx.x * per + i];
        h[threadIdx.x * per + i] = run;
        run += c;
    }
    __syncthreads();
    for (int e0 = 0; e0 < n; e0 += blockDim.x) {
        const int e = e0 + threadIdx.x;
        const float v = e < n ? lb_in[o + e] : 0.f;
        const unsigned bin = e < n ? lb_bin(v) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        const int leader = __ffs(peers) - 1;
        uint32_t basep = 0;
        if (e < n && lane == leader) basep = atomicAdd(&h[bin], (uint32_t)__popc(peers));
        basep = __shfl_sync(0xFFFFFFFFu, basep, leader);
        if (e < n) {
            const uint32_t p = basep + __popc(peers & lt);
            SSH_DASSERT(p < (uint32_t)n);
            rows_out[o + p] = rows_in[o + e];
            lb_out[o + p] = v;
        }
    }
}


// Multi-block version of the per-query bin sort (large lists): chunks of
// BS_CHUNK members per block; per-(query, bin, chunk) counts -> per-query
// exclusive scan (bin-major) -> scatter.  Order inside a bin is arbitrary.
#define BS_CHUNK 32768
__global__ void __launch_bounds__(1024)
bs_hist_kernel(const float *__restrict__ lb_in, const int64_t *__restrict__ roff, const int *__restrict__ cnt,
               int nch, uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[NBINS];
    const int q = blockIdx.y, ch = blockIdx.x;
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    const int n = cnt[q];
    const int64_t o = roff[q];
    const int e0 = ch * BS_CHUNK, e1 = min(n, e0 + BS_CHUNK);
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = e0; b0 < e1; b0 += blockDim.x) {
        const int e = b0 + threadIdx.x;
        const unsigned bin = e < e1 ? lb_bin(lb_in[o + e]) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        if (e < e1 && (peers & lt) == 0) atomicAdd(&h[bin], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) hist[((int64_t)q * NBINS + b) * nch + ch] = h[b];
}

// exclusive scan of hist[q][*] (NBINS * nch entries, a multiple of 4), one
// block per query: coalesced 16-byte loads over per-warp segments, a warp
// scan of the segment totals, then in-lane prefix of 4 + shuffle scans
__global__ void __launch_bounds__(1024) bs_scan_kernel(uint32_t *__restrict__ hist, int nch) {
    static_assert(NBINS % 4 == 0, "");
    __shared__ uint32_t wtot[32];
    const int q = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint4 *h = reinterpret_cast<uint4 *>(hist + (int64_t)q * NBINS * nch);
    const int64_t n4 = (int64_t)NBINS * nch / 4;
    const int64_t seg = ((n4 + 31) / 32 + 31) / 32 * 32;
    const int64_t b = (int64_t)w * seg, e = min(n4, b + seg);
    uint32_t s = 0;
#pragma unroll 4
    for (int64_t i = b + lane; i < e; i += 32) {
        const uint4 v = h[i];
        s += v.x + v.y + v.z + v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0) wtot[w] = s;
    __syncthreads();
    uint32_t run;
    {
        const uint32_t t = wtot[lane];
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        run = __shfl_sync(0xFFFFFFFFu, x - t, w);
    }
    for (int64_t c = b; c < e; c += 32) {
        const int64_t i = c + lane;
        const uint4 v = i < e ? h[i] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t p1 = v.x, p2 = p1 + v.y, p3 = p2 + v.z, tot = p3 + v.w;
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t base = run + x - tot;
        if (i < e) h[i] = make_uint4(base, base + p1, base + p2, base + p3);
        run += __shfl_sync(0xFFFFFFFFu, x, 31);
    }
}

__global__ void __launch_bounds__(1024)
bs_scatter_kernel(const uint32_t *__restrict__ rows_in, const float *__restrict__ lb_in,
                  const int64_t *__restrict__ roff, const int *__restrict__ cnt, int nch,
                  const uint32_t *__restrict__ hist, uint32_t *__restrict__ rows_out, float *__restrict__ lb_out) {
    __shared__ uint32_t h[NBINS];
    const int q = blockIdx.y, ch = blockIdx.x;
    const int n = cnt[q];
    const int e0 = ch * BS_CHUNK, e1 = min(n, e0 + BS_CHUNK);
    if (e0 >= e1) return;
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) h[b] = hist[((int64_t)q * NBINS + b) * nch + ch];
    __syncthreads();
    const int64_t o = roff[q];
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = e0; b0 < e1; b0 += blockDim.x) {
        const int e = b0 + threadIdx.x;
        const float v = e < e1 ? lb_in[o + e] : 0.f;
        const unsigned bin = e < e1 ? lb_bin(v) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
        const int leader = __ffs(peers) - 1;
        uint32_t basep = 0;
        if (e < e1 && lane == leader) basep = atomicAdd(&h[bin], (uint32_t)__popc(peers));
        basep = __shfl_sync(0xFFFFFFFFu, basep, leader);
        if (e < e1) {
            const uint32_t p = basep + __popc(peers & lt);
            rows_out[o + p] = rows_in[o + e];
            lb_out[o + p] = v;
        }
    }
}

// One wave, part 1: members [pos_q, pos_q + wave) of the key-sorted list.
// A warp takes 32 consecutive members (coalesced key/row loads, ballot of
// key <= thr) and walks the live ones with the next member's first
// 512-sample block of envelope codes prefetched while the current one is
// evaluated.  Per member: LB_Keogh2 = LB_Keogh(q, env(x)) over the member's
// envelope codes (dec(U8) >= U, dec(L8) <= L: each term is a lower bound of
// the exact one), then LB_Keogh(x, env(q)) over its sample codes
// (dec(c) <= x <= dec(c+1)), each abandoning after any 512-sample block whose
// partial sum exceeds thr (dtw.py:154-168, 206-215).  Survivors go to the
// wave's DTW list.
struct WaveLbArgs {
    const float *Q, *U, *Lo;
    const uint4 *rec;
    const uint8_t *codes;
    int64_t cstride;
    const uint32_t *srows;
    const float *slbp;
    const int64_t *roff;
    const int *cnt, *pos, *done;
    const float *thr;
    const int *act;  // active queries: block row y works on query act[y] (slot y)
    uint32_t *wrows;  // per-slot wave lists [slot][wcap]
    float2 *wlb;  // (LB_Keogh, LB_Keogh2) totals of each DTW-list entry
    int *wcnt;
    long long *counters;
    unsigned long long *dbg;  // profiling: [1] key skips, [2] LB_Keogh prunes, [3] visited, [4] bytes
    int m, mp, wave, wcap;
};

#define WL_BLK 512  // samples per block of loads (4 chunks of 128, one per lane each)

// bytes t0, t1 of w as exact floats {c0, c1} (0x4B0000cc = 2^23 + cc)
__device__ __forceinline__ float2 code_f2(uint32_t w, int t0, int t1) {
    const float a = __uint_as_float(__byte_perm(w, 0x4B000000u, (unsigned)t0 | 0x7440u));
    const float b = __uint_as_float(__byte_perm(w, 0x4B000000u, (unsigned)t1 | 0x7440u));
    return __fadd2_rn(make_float2(a, b), make_float2(-8388608.f, -8388608.f));
}

__device__ __forceinline__ void wl_load_env(const uint8_t *cr, int mp, int base, uint2 (&v)[4]) {
    const uint2 *p = reinterpret_cast<const uint2 *>(cr + mp + 2 * base) + (threadIdx.x & 31);
#pragma unroll
    for (int c = 0; c < 4; c++) v[c] = base + 128 * c < mp ? __ldg(p + 32 * c) : make_uint2(0u, 0u);
}

// partial LB_Keogh2 over chunks [C0, C1) of one 512-sample block (tails: sqn =
// NaN -> term 0).  Packed f32x2: {ue, le} = fma({cU, cL}, sc, lo) and
// {ue - q, le - q} = {ue, le} + (-q) (broadcast addend), so the terms
// max(q - ue, le - q, 0) = max(-(ue - q), le - q, 0) are the same IEEE values
// as the scalar forms (round-to-nearest is sign-symmetric; dtw.py:154-168
// terms, fp32 screen).  sqn holds -q_i: one 16-byte LDS per 4 samples.
template <int C0, int C1>
__device__ __forceinline__ float wl_env_chunks(const uint2 (&v)[4], const float *sqn, int base, int mp, float sc,
                                               float lo) {
    const int lane = threadIdx.x & 31;
    float2 acc = make_float2(0.f, 0.f);
    const float2 sc2 = make_float2(sc, sc), lo2 = make_float2(lo, lo);
#pragma unroll
    for (int c = C0; c < C1; c++) {
        const int i0 = base + 128 * c + 4 * lane;
        if (base + 128 * c < mp) {
            const float4 qn = *reinterpret_cast<const float4 *>(sqn + i0);
            const float nq[4] = {qn.x, qn.y, qn.z, qn.w};
            float dd[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const uint32_t wv = t < 2 ? v[c].x : v[c].y;
                const int bu = 2 * (t & 1);
                const float2 ul = __ffma2_rn(code_f2(wv, bu, bu + 1), sc2, lo2);
                const float2 df = __fadd2_rn(ul, make_float2(nq[t], nq[t]));
                dd[t] = fmaxf(fmaxf(-df.x, df.y), 0.f);
            }
            acc = __ffma2_rn(make_float2(dd[0], dd[1]), make_float2(dd[0], dd[1]), acc);
            acc = __ffma2_rn(make_float2(dd[2], dd[3]), make_float2(dd[2], dd[3]), acc);
        }
    }
    return acc.x + acc.y;
}

__device__ __forceinline__ void wl_load_smp(const uint8_t *cr, int mp, int base, uint32_t (&v)[4]) {
    const uint32_t *p = reinterpret_cast<const uint32_t *>(cr + base) + (threadIdx.x & 31);
#pragma unroll
    for (int c = 0; c < 4; c++) v[c] = base + 128 * c < mp ? __ldg(p + 32 * c) : 0u;
}

// partial LB_Keogh of one 512-sample block over sample codes (tails: U = inf,
// L = -inf -> 0); sul[i] = {-U_i, L_i}.  {xa, xb} = fma({c, c + 1}, sc, lo)
// and {xa - U, L - xb} = fma({xa, xb}, {1, -1}, {-U, L}) (same IEEE ops).
__device__ __forceinline__ float wl_smp_block(const uint32_t (&cw)[4], const float2 *sul, int base,
                                              int mp, float sc, float lo) {
    const int lane = threadIdx.x & 31;
    float2 acc = make_float2(0.f, 0.f);
    const float2 sc2 = make_float2(sc, sc), lo2 = make_float2(lo, lo), pm = make_float2(1.f, -1.f);
    const float2 off = make_float2(-8388608.f, -8388607.f);  // {c, c + 1}
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const int i0 = base + 128 * c + 4 * lane;
        if (base + 128 * c < mp) {
            const float4 p01 = *reinterpret_cast<const float4 *>(sul + i0);
            const float4 p23 = *reinterpret_cast<const float4 *>(sul + i0 + 2);
            const float2 ul[4] = {make_float2(p01.x, p01.y), make_float2(p01.z, p01.w),
                                  make_float2(p23.x, p23.y), make_float2(p23.z, p23.w)};
            float dd[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const float r = __uint_as_float(__byte_perm(cw[c], 0x4B000000u, (unsigned)t | 0x7440u));
                const float2 x = __ffma2_rn(__fadd2_rn(make_float2(r, r), off), sc2, lo2);
                const float2 df = __ffma2_rn(x, pm, ul[t]);
                dd[t] = fmaxf(fmaxf(df.x, df.y), 0.f);
            }
            acc = __ffma2_rn(make_float2(dd[0], dd[1]), make_float2(dd[0], dd[1]), acc);
            acc = __ffma2_rn(make_float2(dd[2], dd[3]), make_float2(dd[2], dd[3]), acc);
        }
    }
    return acc.x + acc.y;
}

// First-chunk screen, 8 lanes per member (4 members per warp instruction):
// the partial LB_Keogh2 over samples [0, WL_F) of the member whose codes row is
// cr; lane l8 of the group reads 16 contiguous code bytes (8 samples) per
// 64-sample chunk, so a group reads 128 contiguous bytes per load.  Same
// per-sample IEEE operations as wl_env_chunks; returns the group's sum on
// every lane of the group (xor-shuffle over the 8 lanes).
#define WL_F 256
__device__ __forceinline__ float wl_env_first8(const uint8_t *cr, const float *sqn, int mp, float sc, float lo) {
    const int l8 = threadIdx.x & 7;
    float2 acc = make_float2(0.f, 0.f);
    const float2 sc2 = make_float2(sc, sc), lo2 = make_float2(lo, lo);
    const uint4 *p = reinterpret_cast<const uint4 *>(cr + mp) + l8;
    uint4 v[WL_F / 64];
#pragma unroll
    for (int c = 0; c < WL_F / 64; c++) v[c] = 64 * c < mp ? __ldg(p + 8 * c) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int c = 0; c < WL_F / 64; c++) {
        if (64 * c < mp) {
            const int i0 = 64 * c + 8 * l8;
            const float4 qa = *reinterpret_cast<const float4 *>(sqn + i0);
            const float4 qb = *reinterpret_cast<const float4 *>(sqn + i0 + 4);
            const float nq[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
            const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
            float dd[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
                const int bu = 2 * (t & 1);
                const float2 ul = __ffma2_rn(code_f2(wv[t >> 1], bu, bu + 1), sc2, lo2);
                const float2 df = __fadd2_rn(ul, make_float2(nq[t], nq[t]));
                dd[t] = fmaxf(fmaxf(-df.x, df.y), 0.f);
            }
#pragma unroll
            for (int t = 0; t < 8; t += 2)
                acc = __ffma2_rn(make_float2(dd[t], dd[t + 1]), make_float2(dd[t], dd[t + 1]), acc);
        }
    }
    float s = acc.x + acc.y;
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
    return s;
}

__global__ void __launch_bounds__(256, 4) wave_lb_kernel(WaveLbArgs a) {  // 64 registers, 32 warps/SM (72 registers, 24 warps: 8.0 vs 7.3 ms per configs[1] batch)
    extern __shared__ __align__(16) float wsm[];
    const int slot = blockIdx.y;
    const int q = a.act[slot];
    const int m = a.m, mp = a.mp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int start = a.pos[q];
    const int end = min(a.cnt[q], start + a.wave);
    if (start + (int)blockIdx.x * nw * 32 >= end) return;
    float2 *sul = reinterpret_cast<float2 *>(wsm);       // {-U_i, L_i}
    float *sqn = reinterpret_cast<float *>(reinterpret_cast<float2 *>(wsm) + mp);  // -q_i
    for (int i = threadIdx.x; i < mp; i += blockDim.x) {
        const bool in = i < m;
        sul[i] = in ? make_float2(-a.U[(int64_t)q * m + i], a.Lo[(int64_t)q * m + i])
                    : make_float2(-INFINITY, -INFINITY);
        const float qv = in ? a.Q[(int64_t)q * m + i] : __int_as_float(0x7FC00000);
        sqn[i] = -qv;
    }
    __syncthreads();
    const float T = a.thr[q];
    const int64_t o = a.roff[q];
    int paa = 0, kim = 0, keo = 0, keo2 = 0, nvis = 0;
    long long nbytes = 0;
    for (int b0 = start + (blockIdx.x * nw + w) * 32; b0 < end; b0 += gridDim.x * nw * 32) {
        const int e = b0 + lane;
        float key = INFINITY;
        uint32_t row = 0;
        if (e < end) {
            key = a.slbp[o + e];
            row = a.srows[o + e];
            nvis++;
            if (key > T) {
                if (__float_as_uint(key) & 1u) kim++; else paa++;
            }
        }
        unsigned live = __ballot_sync(0xFFFFFFFFu, e < end && key <= T);
        if (!live) continue;
        // stage 1: LB_Keogh2 over the first WL_F samples, 4 members at a time
        // (8 lanes each); most members are pruned here.  Survivors keep their
        // partial sum (p1 on the member's own lane) for the warp-wide pass.
        float p1 = 0.f;
        {
            unsigned todo = live, surv = 0u;
            while (todo) {
                int js[4];
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    js[g] = todo ? __ffs(todo) - 1 : -1;
                    if (todo) todo &= todo - 1;
                }
                const int gi = lane >> 3;
                const int jm = gi == 0 ? js[0] : gi == 1 ? js[1] : gi == 2 ? js[2] : js[3];
                const uint32_t rm = __shfl_sync(0xFFFFFFFFu, row, jm < 0 ? 0 : jm);
                float part = 0.f;
                if (jm >= 0) {
                    float2 h = __ldg(reinterpret_cast<const float2 *>(a.rec + (int64_t)rm * 4));
                    part = wl_env_first8(a.codes + (int64_t)rm * a.cstride, sqn, mp, fabsf(h.y), h.x);
                } else {
                    part = wl_env_first8(a.codes, sqn, 0, 0.f, 0.f);  // idle group: no loads (mp = 0)
                }
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    const float pg = __shfl_sync(0xFFFFFFFFu, part, 8 * g);
                    if (js[g] >= 0) {
                        if (lane == js[g]) p1 = pg;
                        if (pg > T) keo2++;
                        else surv |= 1u << js[g];
                        nbytes += 2 * min(WL_F, mp);
                    }
                }
            }
            live = surv;
        }
        if (!live) continue;
        int j = __ffs(live) - 1;
        live &= live - 1;
        int jc = j;
        uint32_t rc = __shfl_sync(0xFFFFFFFFu, row, j);
        float2 hc = __ldg(reinterpret_cast<const float2 *>(a.rec + (int64_t)rc * 4));
        hc.y = fabsf(hc.y);  // sign = PAA-codes flag, not part of the scale
        uint2 vc[4];
        wl_load_env(a.codes + (int64_t)rc * a.cstride, mp, 0, vc);
        for (;;) {
            // prefetch the next live member's header and first block
            const bool more = live != 0;
            uint32_t rn = 0;
            float2 hn = make_float2(0.f, 0.f);
            uint2 vn[4];
            if (more) {
                j = __ffs(live) - 1;
                live &= live - 1;
                rn = __shfl_sync(0xFFFFFFFFu, row, j);
                hn = __ldg(reinterpret_cast<const float2 *>(a.rec + (int64_t)rn * 4));
                hn.y = fabsf(hn.y);
                wl_load_env(a.codes + (int64_t)rn * a.cstride, mp, 0, vn);
            }
            const uint8_t *cr = a.codes + (int64_t)rc * a.cstride;
            const float lo = hc.x, sc = hc.y;
            bool pruned = false;
            // samples [0, WL_F) were summed by the stage-1 screen (p1 of lane jc)
            const float pre = __shfl_sync(0xFFFFFFFFu, p1, jc);
            float acc = lane == 0 ? pre : 0.f, tot2 = pre, tot1 = 0.f;
            // abandon checks after every 256 samples (partial sums are lower bounds)
            for (int base = 0; base < mp; base += WL_BLK) {
                if (base) {
                    wl_load_env(cr, mp, base, vc);
                    nbytes += 2 * min(WL_BLK, mp - base);
                    acc += wl_env_chunks<0, 2>(vc, sqn, base, mp, sc, lo);
                    tot2 = warp_sum(acc);
                    if (tot2 > T) { pruned = true; break; }
                } else {
                    nbytes += 2 * max(0, min(WL_BLK, mp) - WL_F);
                }
                if (base + 256 < mp) {
                    acc += wl_env_chunks<2, 4>(vc, sqn, base, mp, sc, lo);
                    tot2 = warp_sum(acc);
                    if (tot2 > T) { pruned = true; break; }
                }
            }
            if (pruned) {
                keo2++;
            } else {
                acc = 0.f;
                for (int base = 0; base < mp; base += WL_BLK) {
                    uint32_t cw[4];
                    wl_load_smp(cr, mp, base, cw);
                    nbytes += min(WL_BLK, mp - base);
                    acc += wl_smp_block(cw, sul, base, mp, sc, lo);
                    tot1 = warp_sum(acc);
                    if (tot1 > T) { pruned = true; break; }
                }
                if (pruned) {
                    keo++;
                } else if (lane == 0) {
                    const int p = atomicAdd(&a.wcnt[slot], 1);
                    if (p < a.wcap) {
                        a.wrows[(int64_t)slot * a.wcap + p] = rc;
                        a.wlb[(int64_t)slot * a.wcap + p] = make_float2(tot1, tot2);
                    }
                }
            }
            if (!more) break;
            rc = rn;
            jc = j;
            hc = hn;
#pragma unroll
            for (int c = 0; c < 4; c++) vc[c] = vn[c];
        }
    }
    // per-lane key counts, per-warp (lane-uniform) LB counts
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        paa += __shfl_xor_sync(0xFFFFFFFFu, paa, off);
        kim += __shfl_xor_sync(0xFFFFFFFFu, kim, off);
        nvis += __shfl_xor_sync(0xFFFFFFFFu, nvis, off);
    }
    if (lane == 0) {
        if (kim) atomicAdd((unsigned long long *)&a.counters[q * 5 + 0], (unsigned long long)kim);
        if (paa + keo) atomicAdd((unsigned long long *)&a.counters[q * 5 + 1], (unsigned long long)(paa + keo));
        if (keo2) atomicAdd((unsigned long long *)&a.counters[q * 5 + 2], (unsigned long long)keo2);
        if (a.dbg) {
            atomicAdd(&a.dbg[1], (unsigned long long)(paa + kim));
            atomicAdd(&a.dbg[2], (unsigned long long)keo);
            atomicAdd(&a.dbg[3], (unsigned long long)nvis);
            atomicAdd(&a.dbg[4], (unsigned long long)nbytes);
        }
    }
}

// ------------------------------------------------------------ fp32 DTW
// Candidate list of one DTW launch: per query the entries
// [off_q, min(cnt_q, off_q + wave)) of rows[q][*]; an entry whose lower bound
// lbs[q][e] exceeds thr_q is skipped (result +inf).
struct DtwList {
    const uint32_t *rows;
    int64_t stride;
    const int *cnt;     // per-query entry count (NULL: stride)
    const int *off;     // per-query first entry (NULL: 0)
    int wave;           // entries per query in this launch
    const float *lbs;   // per-entry lower bound (NULL: none)
    float *out;         // result at the same index
    unsigned long long *abandoned;  // per query (NULL ok)
    int *computed;      // per query DTWs evaluated (NULL ok)
    const int *act;     // block row y -> query act[y]; rows/lbs/out/cnt/off are per slot y (NULL: identity)
};

__device__ __forceinline__ void dtw_list_range(const DtwList &L, int slot, int &start, int &end) {
    start = L.off ? L.off[slot] : 0;
    const int total = L.cnt ? L.cnt[slot] : (int)L.stride;
    end = min(total, start + L.wave);
}

// Lane-per-candidate banded DTW; band[k][lane] in shared memory, the query
// padded with +inf outside [0, m) so out-of-band cells are +inf without
// branches.  With a finite threshold the lane abandons once
//   row_min + sum_{i' > i} LB_Keogh_i'(x, env(q)) - slack > thr
// (every remaining row contributes at least its envelope excursion).
__global__ void dtw32_kernel(const float *__restrict__ X, int m, int r, const float *__restrict__ Q,
                             const float *__restrict__ U, const float *__restrict__ Lo, DtwList L,
                             const float *__restrict__ thr, int warps,
                             unsigned long long *__restrict__ cells) {
    extern __shared__ float dsm[];
    const int q = L.act ? L.act[blockIdx.y] : blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int B = 2 * r + 2;
    const int ypadn = (m + 2 * r + 3) & ~3;
    float *ypad = dsm;  // m + 2r
    float *su = dsm + ypadn;
    float *sl = su + m;
    float *band = sl + m + (size_t)w * B * 32;
    const int slot = blockIdx.y;
    int start, end;
    dtw_list_range(L, slot, start, end);
    if (start + (int)blockIdx.x * warps * 32 >= end) return;  // block-uniform: no work
    const float *y = Q + (int64_t)q * m;
    for (int j = threadIdx.x; j < m + 2 * r; j += blockDim.x) {
        int jj = j - r;
        ypad[j] = (jj >= 0 && jj < m) ? y[jj] : INFINITY;
    }
    const float T = thr ? thr[q] : INFINITY;
    const bool cb = !isinf(T) && U != nullptr;
    if (cb)
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            su[i] = U[(int64_t)q * m + i];
            sl[i] = Lo[(int64_t)q * m + i];
        }
    __syncthreads();
    const int e = start + (blockIdx.x * warps + w) * 32 + lane;
    if (start + (blockIdx.x * warps + w) * 32 >= end) return;
    uint32_t row = e < end ? L.rows[(int64_t)slot * L.stride + e] : 0xFFFFFFFFu;
    bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)slot * L.stride + e] > T));
    {
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        if (L.computed && lane == 0 && vm) atomicAdd(&L.computed[q], __popc(vm));
    }
    const float *x = X + (int64_t)(valid ? row : 0) * m;
    float rem = 0.f, slack = 0.f;
    if (cb) {
        for (int i = 0; i < m; i++) {
            float cv = x[i];
            float v = fmaxf(fmaxf(cv - su[i], sl[i] - cv), 0.f);
            rem = fmaf(v, v, rem);
        }
        slack = rem * (float)(2 * m + 8) * U32_EPS;
    }
    for (int k = 0; k < B; k++) band[k * 32 + lane] = INFINITY;
    band[r * 32 + lane] = 0.f;
    bool alive = valid;
    int rows = 0;
    for (int i = 0; i < m; i++) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;
        rows += alive;
        const float xi = x[i];
        float left = INFINITY;
        float diag = band[lane];
        float rmin = INFINITY;
        const float *yr = ypad + i;
        for (int k = 0; k <= 2 * r; k++) {
            float up = band[(k + 1) * 32 + lane];
            float d = xi - yr[k];
            float best = fminf(fminf(diag, up), left);
            float c = fmaf(d, d, best);
            band[k * 32 + lane] = c;
            rmin = fminf(rmin, c);
            left = c;
            diag = up;
        }
        float bound = rmin;
        if (cb) {
            float v = fmaxf(fmaxf(xi - su[i], sl[i] - xi), 0.f);
            rem = fmaf(-v, v, rem);
            bound = rmin + fmaxf(rem - slack, 0.f);
        }
        if (alive && bound > T) alive = false;
    }
    if (e < end) {
        float res = (valid && alive) ? band[r * 32 + lane] : INFINITY;
        L.out[(int64_t)slot * L.stride + e] = res;
        if (L.abandoned && valid && !alive) atomicAdd(&L.abandoned[q], 1ULL);
    }
    if (cells) {
        unsigned long long c = (unsigned long long)rows * (unsigned long long)(2 * r + 1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        if (lane == 0 && c) atomicAdd(cells, c);
    }
}

// Wide-band wave DTW (fp32 screen): the band-chunked warp wavefront of
// dtw_warp.cuh, one warp per candidate.  Lane l owns the C band offsets
// k = lC + c in registers and sweeps row i = s - l at step s (cell update
// in place, ascending k; left edge from lane l - 1 by shfl_up, up edge from
// lane l + 1's first cell of the same step by shfl_down).  The query (padded
// with +inf) is staged once per block; each lane's query samples are a
// register window sliding one sample per step (the new one from lane l + 1);
// its series sample x[s - l] is a coalesced load per step from L1 (the row
// was just read by the vectorised LB-prefix pass).  Per cell: FADD + FMNMX3 +
// FFMA.  Groups of C steps come in three variants: ramp-up (lanes whose row is
// still negative keep the virtual row -1 by selects), main (no checks), and
// ramp-down (sample indices checked; rows >= m produce values no in-range
// cell reads).
//
// Abandon (UCR-suite cumulative bound, dtw.py:206-215) on a skewed cut: after
// step s the lanes hold the cells with i + floor(k / C) = s.  Along any
// warping path f = i + floor(k / C) grows by 0 or 1 per move, from
// floor(r / C) at (0, 0) to m - 1 + floor(r / C), so for s in that range every
// path crosses the cut; the path's remaining rows are all > s - 31 ... s, so
//   DTW >= min_cut D + sum_{i' > s} LB_Keogh term(i')
// (lane 0 holds row s).  The test runs once per group of C steps with the same
// fp32 slack as the row test: cut_min + max(remK - slack, 0) > thr.
// remK = total - prefix(s) with the exact-x LB_Keogh terms (query envelope)
// summed by a warp scan while the candidate is first read.
#define DW_WARPS 8
#ifndef DW_MINB
#define DW_MINB 3
#endif
// one step of the wide-band wavefront (see dtw32w_kernel); MASK: lanes whose
// row is still negative keep their virtual row -1 (ramp-up steps only)
template <int C, int U, bool MASK>
__device__ __forceinline__ void dw_step(float (&band)[C], float (&yw)[C], const float xi, const int i,
                                        const int lane, const int own, const int cst, const float y31) {
    const float inf = INFINITY;
    float leftv = __shfl_up_sync(0xFFFFFFFFu, band[C - 1], 1);
    if (lane == 0) leftv = inf;
    const bool act = !MASK || i >= 0;
    {
        const float d = xi - yw[U % C];
        float v = fmaf(d, d, fminf(fminf(band[0], band[1]), leftv));
        if (cst == 0 && lane == own) v = inf;
        band[0] = act ? v : band[0];
    }
    float upr = __shfl_down_sync(0xFFFFFFFFu, band[0], 1);
    if (lane == 31) upr = inf;
#pragma unroll
    for (int c = 1; c < C; c++) {
        const float up = (c + 1 < C) ? band[c + 1] : upr;
        const float d = xi - yw[(U + c) % C];
        float v = fmaf(d, d, fminf(fminf(band[c], up), band[c - 1]));
        if (cst == c && lane == own) v = inf;
        band[c] = act ? v : band[c];
    }
    // slide the query window: logical 0 (phys U) expires, the new last sample
    // comes from lane l + 1's logical 1 (lane 31: from the staged query)
    float yn = __shfl_down_sync(0xFFFFFFFFu, yw[(U + 1) % C], 1);
    if (lane == 31) yn = y31;
    yw[U % C] = yn;
}

// C steps from s0 (a multiple of C): MASK during ramp-up; CHECK: some lane's
// sample index s - lane lies outside [0, m) (ramp-up / ramp-down groups)
template <int C, int U, bool MASK, bool CHECK>
__device__ __forceinline__ void dw_group(float (&band)[C], float (&yw)[C], const float *__restrict__ x,
                                         const float *yb, const int s0, const int lane, const int own,
                                         const int cst, const int rown, const int rcc, const int m, float &res) {
    if constexpr (U < C) {
        const int s = s0 + U;
        const int ix = s - lane;
        float xi;
        if (CHECK) xi = (unsigned)ix < (unsigned)m ? __ldg(x + ix) : 0.f;
        else xi = __ldg(x + ix);
        dw_step<C, U, MASK>(band, yw, xi, ix, lane, own, cst, yb[U]);
        if (CHECK && ix == m - 1 && lane == rown) {
#pragma unroll
            for (int c = 0; c < C; c++)
                if (c == rcc) res = band[c];
        }
        dw_group<C, U + 1, MASK, CHECK>(band, yw, x, yb, s0, lane, own, cst, rown, rcc, m, res);
    }
}
template <int C, int RF>
__global__ void __launch_bounds__(32 * DW_WARPS, DW_MINB)
dtw32w_kernel(const float *__restrict__ X, int m, int r_rt, const float *__restrict__ Q,
              const float *__restrict__ U, const float *__restrict__ Lo, DtwList L,
              const float *__restrict__ thr, unsigned long long *__restrict__ cells) {
    const int r = RF >= 0 ? RF : r_rt;
    const int nk = 2 * r + 1;
    const int own = nk / C, cst = nk - own * C;  // cell k = nk (forced +inf): lane own, index cst
    const int rown = r / C, rcc = r - rown * C;   // result cell k = r
    const int G = (m + 31 + C - 1) / C;          // step groups
    const int YP = (r + m + 33 * C + 64 + 3) & ~3;  // keeps su / sl 16-byte aligned
    extern __shared__ __align__(16) float wsm[];
    float *yq = wsm;          // yq[j + r] = y[j], +inf outside [0, m)
    float *su = yq + YP;      // query envelope
    float *sl = su + m;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float *pre = sl + m + (size_t)w * (G + 1);  // prefix of LB_Keogh terms at group ends
    const int q = L.act ? L.act[blockIdx.y] : blockIdx.y;
    const int slot = blockIdx.y;
    int start, end;
    dtw_list_range(L, slot, start, end);
    if (start + (int)blockIdx.x * DW_WARPS >= end) return;  // block-uniform
    const float *y = Q + (int64_t)q * m;
    for (int t = threadIdx.x; t < YP; t += blockDim.x) {
        const int j = t - r;
        yq[t] = (j >= 0 && j < m) ? y[j] : INFINITY;
    }
    const float T = thr ? thr[q] : INFINITY;
    const bool cb = !isinf(T) && U != nullptr;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        su[i] = cb ? U[(int64_t)q * m + i] : INFINITY;
        sl[i] = cb ? Lo[(int64_t)q * m + i] : -INFINITY;
    }
    __syncthreads();
    const float inf = INFINITY;
    const int f_lo = r / C, f_hi = m - 1 + r / C;  // cut steps every path crosses
    // groups [g_main0, g_main1) need no index checks (0 <= s - lane < m - 1 for
    // every lane; the result row m - 1 is always reached in a checked group)
    const int g_main0 = (31 + C - 1) / C, g_main1 = max(g_main0, (m - 1) / C);
    const bool vec = (m & 3) == 0;
    unsigned long long my_cells = 0;
    for (int e = start + (int)blockIdx.x * DW_WARPS + w; e < end; e += (int)gridDim.x * DW_WARPS) {
        const uint32_t row = L.rows[(int64_t)slot * L.stride + e];
        const bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)slot * L.stride + e] > T));
        if (!valid) {  // warp-uniform
            if (lane == 0) L.out[(int64_t)slot * L.stride + e] = inf;
            continue;
        }
        if (L.computed && lane == 0) atomicAdd(&L.computed[q], 1);
        const float *x = X + (int64_t)row * m;
        __syncwarp();
        // prefix sums of the LB_Keogh terms (exact x vs the query envelope) at
        // the group-end steps s = (g + 1) C - 1: 4 consecutive samples per
        // lane per 128 (independent vector loads; the row then sits in L1 for
        // the sweep)
        float carry = 0.f;
        if (vec) {
#pragma unroll 4
            for (int i0 = 0; i0 < G * C; i0 += 128) {
                const int i = i0 + 4 * lane;
                float v2[4] = {0.f, 0.f, 0.f, 0.f};
                if (i < m) {
                    const float4 xv = __ldg(reinterpret_cast<const float4 *>(x + i));
                    const float4 uv = *reinterpret_cast<const float4 *>(su + i);
                    const float4 lv = *reinterpret_cast<const float4 *>(sl + i);
                    const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
                    const float ua[4] = {uv.x, uv.y, uv.z, uv.w};
                    const float la[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const float v = fmaxf(fmaxf(xa[t] - ua[t], la[t] - xa[t]), 0.f);
                        v2[t] = v * v;
                    }
                }
                v2[1] += v2[0];
                v2[2] += v2[1];
                v2[3] += v2[2];
                float sc = v2[3];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xFFFFFFFFu, sc, o);
                    if (lane >= o) sc += t;
                }
                const float base = carry + sc - v2[3];
#pragma unroll
                for (int t = 0; t < 4; t++)
                    if ((i + t + 1) % C == 0 && i + t < G * C) pre[(i + t + 1) / C - 1] = base + v2[t];
                carry = __shfl_sync(0xFFFFFFFFu, carry + sc, 31);
            }
        } else {
            for (int i0 = 0; i0 < G * C; i0 += 32) {
                const int i = i0 + lane;
                float v2 = 0.f;
                if (i < m) {
                    const float xv = __ldg(x + i);
                    const float v = fmaxf(fmaxf(xv - su[i], sl[i] - xv), 0.f);
                    v2 = v * v;
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xFFFFFFFFu, v2, o);
                    if (lane >= o) v2 += t;
                }
                const float P = carry + v2;
                if ((i + 1) % C == 0) pre[(i + 1) / C - 1] = P;
                carry = __shfl_sync(0xFFFFFFFFu, P, 31);
            }
        }
        const float total = carry;
        const float slack = total * (float)(2 * m + 8) * U32_EPS;
        __syncwarp();
        float band[C], yw[C];
#pragma unroll
        for (int c = 0; c < C; c++) {
            band[c] = (lane * C + c == r) ? 0.f : inf;  // virtual row -1: D(0, 0) = d(0, 0)
            yw[c] = yq[lane * (C - 1) + c];
        }
        float res = inf;
        bool dead = false;
        int g = 0;
        for (; g < G; g++) {
            const int s0 = g * C;
            const float *yb = yq + s0 + 32 * C - 31;
            SSH_DASSERT(s0 + 32 * C - 31 + C <= YP);
            if (g < g_main0)
                dw_group<C, 0, true, true>(band, yw, x, yb, s0, lane, own, cst, rown, rcc, m, res);
            else if (g < g_main1)
                dw_group<C, 0, false, false>(band, yw, x, yb, s0, lane, own, cst, rown, rcc, m, res);
            else
                dw_group<C, 0, false, true>(band, yw, x, yb, s0, lane, own, cst, rown, rcc, m, res);
            // cut test after step s = s0 + C - 1
            const int s = s0 + C - 1;
            if (cb && s >= f_lo && s <= f_hi) {
                const int i = s - lane;
                float cm = inf;
                if (i >= 0 && i < m) {
#pragma unroll
                    for (int c = 0; c < C; c++)
                        if (lane * C + c < nk) cm = fminf(cm, band[c]);
                }
                const unsigned cmb = __reduce_min_sync(0xFFFFFFFFu, __float_as_uint(cm));
                SSH_DASSERT(g < G);
                const float remk = fmaxf(total - pre[g] - slack, 0.f);
                if (__uint_as_float(cmb) + remk > T) {
                    dead = true;
                    break;
                }
            }
        }
        res = __shfl_sync(0xFFFFFFFFu, res, rown);
        if (lane == 0) {
            L.out[(int64_t)slot * L.stride + e] = dead ? inf : res;
            if (dead && L.abandoned) atomicAdd(&L.abandoned[q], 1ULL);
        }
        if (cells) {
            // in-band cells of the rows lane 31 completed
            const long long rows = dead ? (long long)min(m, max(0, (g + 1) * C - 31)) : (long long)m;
            long long c = rows * nk;
            const long long a = min(rows, (long long)r);  // rows i < r lose r - i cells
            c -= a * r - a * (a - 1) / 2;
            const long long b0 = max(0LL, (long long)(m - r));  // rows i >= m - r lose i + r - m + 1
            if (rows > b0) {
                const long long nb = rows - b0;
                c -= nb * (b0 + r - m + 1) + nb * (nb - 1) / 2;
            }
            my_cells += (unsigned long long)c;
        }
    }
    if (cells && lane == 0 && my_cells) atomicAdd(cells, my_cells);
}

// Wide-band wave DTW, paired form: the warp wavefront above with 64 VIRTUAL
// lanes, two per physical lane, so every cell update is half of an f32x2 pair.
// Virtual lane v owns the C2 band offsets k = v C2 + c and sweeps row s - v at
// step s; physical lane l hosts A = virtual 2l (row s - 2l) and B = virtual
// 2l + 1 (row s - 2l - 1, offsets right after A's), pair c = {A_c, B_c}.  In
// one step, ascending c, A_c and B_c update together:
//   A_c = d_A^2 + min(A_c, A_{c+1} | B_0 (new), A_{c-1} (new) | lane l-1's
//         B_{C2-1} from the previous step (shfl_up; +inf on lane 0))
//   B_c = d_B^2 + min(B_c, B_{c+1} | lane l+1's new A_0 (shfl_down after pair
//         0; +inf on lane 31), B_{c-1} (new) | A_{C2-1} from the previous step)
// d = {x_A, x_B} + {-y_A, -y_B} is one FADD2 and the cells one FFMA2 per pair
// (the same IEEE operations as the scalar fmaf(d, d, min3) recurrence), so a
// cell costs half an FADD2, half an FFMA2 and one FMNMX3.  Query samples are a
// sliding register window of 2 C2 - 1 negated samples held as pairs
// {Y[c], Y[c + C2 - 1]} (pair c serves A_c and B_c); one new sample per step
// comes from lane l + 1 (lane 31: the staged query).  x_B is the previous
// step's x_A.  Abandon: the skewed-cut cumulative bound of dtw32w_kernel with
// 64 virtual lanes (virtual lane 0 holds row s).
#ifndef DV_WARPS
#define DV_WARPS 8
#endif
#ifndef DV_MINB
#define DV_MINB 2
#endif
// f32x2 helpers on packed 64-bit registers (the PTX f32x2 operand type), so
// the query-window pairs stay register pairs across the window rotation
__device__ __forceinline__ unsigned long long dv_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float dv_hi(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ float dv_lo(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ unsigned long long dv_add2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float2 dv_sqadd2(unsigned long long d, float mA, float mB) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(d), "l"(dv_pack(mA, mB)));
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}

// window: NY[(U + c) % C2] = {-Y[c], -Y[c + C2 - 1]} (pair c serves A_c and B_c)
template <int C2, int U, bool MASK>
__device__ __forceinline__ void dv_step(float2 (&P)[C2], unsigned long long (&NY)[C2], float &xb, const float xa,
                                        const int iA, const int lane, const int olane, const int ocomp,
                                        const int cst, const float y31) {
    const float inf = INFINITY;
    float lA = __shfl_up_sync(0xFFFFFFFFu, P[C2 - 1].y, 1);  // lane l-1's B_{C2-1}, previous step
    if (lane == 0) lA = inf;
    const float lB = P[C2 - 1].x;                           // own A_{C2-1}, previous step
    const unsigned long long XP = dv_pack(xa, xb);
    const bool actA = !MASK || iA >= 0, actB = !MASK || iA >= 1;
    float upr = inf;
#pragma unroll
    for (int c = 0; c < C2; c++) {
        const float2 old = P[c];
        const float upA = (c + 1 < C2) ? P[c + 1].x : P[0].y;
        const float upB = (c + 1 < C2) ? P[c + 1].y : upr;
        const float leftA = c == 0 ? lA : P[c - 1].x;
        const float leftB = c == 0 ? lB : P[c - 1].y;
        const float mA = fminf(fminf(old.x, upA), leftA);
        const float mB = fminf(fminf(old.y, upB), leftB);
        float2 v = dv_sqadd2(dv_add2(XP, NY[(U + c) % C2]), mA, mB);
        if (c == cst && lane == olane) {  // first out-of-band offset k = 2r + 1 stays +inf
            if (ocomp) v.y = inf;
            else v.x = inf;
        }
        if (MASK) {
            v.x = actA ? v.x : old.x;
            v.y = actB ? v.y : old.y;
        }
        P[c] = v;
        if (c == 0) {
            upr = __shfl_down_sync(0xFFFFFFFFu, v.x, 1);
            if (lane == 31) upr = inf;
        }
    }
    xb = xa;
    // slide: pair 0 expires; the new last pair is {Y[C2] (own pair 1's high
    // half), Y[2 C2 - 1] (lane l + 1's Y[1] = its pair 1's low half)}
    float yn = __shfl_down_sync(0xFFFFFFFFu, dv_lo(NY[(U + 1) % C2]), 1);
    if (lane == 31) yn = y31;
    NY[U % C2] = dv_pack(dv_hi(NY[(U + 1) % C2]), yn);
}

// C2 steps from s0 (window phase 0): MASK during ramp-up; CHECK: some lane's
// row index lies outside [0, m)
template <int C2, int U, bool MASK, bool CHECK>
__device__ __forceinline__ void dv_group(float2 (&P)[C2], unsigned long long (&NY)[C2], float &xb,
                                         const float *__restrict__ xg, const float *nyb, const int s0,
                                         const int lane, const int olane, const int ocomp, const int cst,
                                         const int rlane, const int rcomp, const int rcc, const int m, float &res) {
    if constexpr (U < C2) {
        const int iA = s0 + U - 2 * lane;
        float xa;
        if (CHECK) xa = (unsigned)iA < (unsigned)m ? __ldg(xg + U) : 0.f;
        else xa = __ldg(xg + U);
        const float y31 = nyb[U];
        dv_step<C2, U, MASK>(P, NY, xb, xa, iA, lane, olane, ocomp, cst, y31);
        if (CHECK && lane == rlane && iA - rcomp == m - 1) {
#pragma unroll
            for (int c = 0; c < C2; c++)
                if (c == rcc) res = rcomp ? P[c].y : P[c].x;
        }
        dv_group<C2, U + 1, MASK, CHECK>(P, NY, xb, xg, nyb, s0, lane, olane, ocomp, cst, rlane, rcomp, rcc, m,
                                         res);
    }
}

template <int C2, int RF>
__global__ void __launch_bounds__(32 * DV_WARPS, DV_MINB)
dtw32v_kernel(const float *__restrict__ X, int m, int r_rt, const float *__restrict__ Q,
              const float *__restrict__ U, const float *__restrict__ Lo, DtwList L,
              const float *__restrict__ thr, unsigned long long *__restrict__ cells) {
    const int r = RF >= 0 ? RF : r_rt;
    const int nk = 2 * r + 1;
    const int ov = nk / C2, cst = nk - ov * C2;  // cell k = nk (forced +inf): virtual lane ov, pair cst
    const int olane = ov < 64 ? ov >> 1 : -1, ocomp = ov & 1;
    const int rv = r / C2, rcc = r - rv * C2;    // result cell k = r
    const int rlane = rv >> 1, rcomp = rv & 1;
    constexpr int GS = C2;                       // steps per group (one window rotation)
    const int NS = m + 63;                       // steps: virtual lane 63 finishes row m - 1 at m + 62
    const int G = (NS + GS - 1) / GS;            // step groups
    const int YP = (r + m + 64 * C2 + 2 * GS + 64 + 3) & ~3;
    extern __shared__ __align__(16) float vsm[];
    float *nyq = vsm;         // nyq[j + r] = -y[j], -inf outside [0, m)
    float *su = nyq + YP;     // query envelope
    float *sl = su + m;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float *pre = sl + m + (size_t)w * (G + 1);  // prefix of LB_Keogh terms at group ends
    const int q = L.act ? L.act[blockIdx.y] : blockIdx.y;
    const int slot = blockIdx.y;
    int start, end;
    dtw_list_range(L, slot, start, end);
    if (start + (int)blockIdx.x * DV_WARPS >= end) return;  // block-uniform
    const float *y = Q + (int64_t)q * m;
    for (int t = threadIdx.x; t < YP; t += blockDim.x) {
        const int j = t - r;
        nyq[t] = (j >= 0 && j < m) ? -y[j] : -INFINITY;
    }
    const float T = thr ? thr[q] : INFINITY;
    const bool cb = !isinf(T) && U != nullptr;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        su[i] = cb ? U[(int64_t)q * m + i] : INFINITY;
        sl[i] = cb ? Lo[(int64_t)q * m + i] : -INFINITY;
    }
    __syncthreads();
    const float inf = INFINITY;
    const int f_lo = r / C2, f_hi = m - 1 + r / C2;  // cut steps every path crosses
    // groups [g_main0, g_main1): every virtual lane's row in [0, m - 1)
    const int g_main0 = (63 + GS - 1) / GS, g_main1 = max(g_main0, (m - 1) / GS);
    const bool vec = (m & 3) == 0;
    unsigned long long my_cells = 0;
    for (int e = start + (int)blockIdx.x * DV_WARPS + w; e < end; e += (int)gridDim.x * DV_WARPS) {
        const uint32_t row = L.rows[(int64_t)slot * L.stride + e];
        const bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)slot * L.stride + e] > T));
        if (!valid) {  // warp-uniform
            if (lane == 0) L.out[(int64_t)slot * L.stride + e] = inf;
            continue;
        }
        if (L.computed && lane == 0) atomicAdd(&L.computed[q], 1);
        const float *x = X + (int64_t)row * m;
        __syncwarp();
        // prefix sums of the LB_Keogh terms (exact x vs the query envelope) at
        // the group-end steps s = (g + 1) C2 - 1 (rows >= m add nothing)
        float carry = 0.f;
        if (vec) {
#pragma unroll 1
            for (int i0 = 0; i0 < G * GS; i0 += 128) {
                const int i = i0 + 4 * lane;
                float v2[4] = {0.f, 0.f, 0.f, 0.f};
                if (i < m) {
                    const float4 xv = __ldg(reinterpret_cast<const float4 *>(x + i));
                    const float4 uv = *reinterpret_cast<const float4 *>(su + i);
                    const float4 lv = *reinterpret_cast<const float4 *>(sl + i);
                    const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
                    const float ua[4] = {uv.x, uv.y, uv.z, uv.w};
                    const float la[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const float v = fmaxf(fmaxf(xa[t] - ua[t], la[t] - xa[t]), 0.f);
                        v2[t] = v * v;
                    }
                }
                v2[1] += v2[0];
                v2[2] += v2[1];
                v2[3] += v2[2];
                float sc = v2[3];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xFFFFFFFFu, sc, o);
                    if (lane >= o) sc += t;
                }
                const float base = carry + sc - v2[3];
#pragma unroll
                for (int t = 0; t < 4; t++)
                    if ((i + t + 1) % GS == 0 && i + t < G * GS) pre[(i + t + 1) / GS - 1] = base + v2[t];
                carry = __shfl_sync(0xFFFFFFFFu, carry + sc, 31);
            }
        } else {
            for (int i0 = 0; i0 < G * GS; i0 += 32) {
                const int i = i0 + lane;
                float v2 = 0.f;
                if (i < m) {
                    const float xv = __ldg(x + i);
                    const float v = fmaxf(fmaxf(xv - su[i], sl[i] - xv), 0.f);
                    v2 = v * v;
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xFFFFFFFFu, v2, o);
                    if (lane >= o) v2 += t;
                }
                const float P0 = carry + v2;
                if ((i + 1) % GS == 0) pre[(i + 1) / GS - 1] = P0;
                carry = __shfl_sync(0xFFFFFFFFu, P0, 31);
            }
        }
        const float total = carry;
        const float slack = total * (float)(2 * m + 8) * U32_EPS;
        __syncwarp();
        float2 P[C2];
        unsigned long long NY[C2];
        float xb = 0.f;
        const int wy = 2 * lane * (C2 - 1);  // nyq index of Y[0] at step 0
#pragma unroll
        for (int c = 0; c < C2; c++) {
            // virtual row -1: 0 at k = r (D(0, 0) = d(0, 0)), +inf elsewhere
            P[c] = make_float2((2 * lane * C2 + c == r) ? 0.f : inf, ((2 * lane + 1) * C2 + c == r) ? 0.f : inf);
            NY[c] = dv_pack(nyq[wy + c], nyq[wy + c + C2 - 1]);
        }
        const float *xl = x - 2 * lane;
        float res = inf;
        bool dead = false;
        int g = 0;
        for (; g < G; g++) {
            const int s0 = g * GS;
            // lane 31's new sample when sliding after step s: Y_31[2 C2 - 1] = nyq[s + 64 C2 - 63]
            const float *nyb = nyq + s0 + 64 * C2 - 63;
            const float *xg = xl + s0;
            if (g < g_main0)
                dv_group<C2, 0, true, true>(P, NY, xb, xg, nyb, s0, lane, olane, ocomp, cst, rlane, rcomp, rcc, m,
                                            res);
            else if (g < g_main1)
                dv_group<C2, 0, false, false>(P, NY, xb, xg, nyb, s0, lane, olane, ocomp, cst, rlane, rcomp, rcc,
                                              m, res);
            else
                dv_group<C2, 0, false, true>(P, NY, xb, xg, nyb, s0, lane, olane, ocomp, cst, rlane, rcomp, rcc, m,
                                             res);
            // cut test after step s = s0 + GS - 1
            const int s = s0 + GS - 1;
            if (cb && s >= f_lo && s <= f_hi) {
                const int iA = s - 2 * lane;
                const bool okA = iA >= 0 && iA < m, okB = iA >= 1 && iA <= m;
                float cm = inf;
#pragma unroll
                for (int c = 0; c < C2; c++) cm = fminf(fminf(cm, okA ? P[c].x : inf), okB ? P[c].y : inf);
                const unsigned cmb = __reduce_min_sync(0xFFFFFFFFu, __float_as_uint(cm));
                const float remk = fmaxf(total - pre[g] - slack, 0.f);
                if (__uint_as_float(cmb) + remk > T) {
                    dead = true;
                    break;
                }
            }
        }
        res = __shfl_sync(0xFFFFFFFFu, res, rlane);
        if (lane == 0) {
            L.out[(int64_t)slot * L.stride + e] = dead ? inf : res;
            if (dead && L.abandoned) atomicAdd(&L.abandoned[q], 1ULL);
        }
        if (cells) {
            // in-band cells of the rows virtual lane 63 completed
            const long long rows = dead ? (long long)min(m, max(0, (g + 1) * GS - 63)) : (long long)m;
            long long c = rows * nk;
            const long long a = min(rows, (long long)r);  // rows i < r lose r - i cells
            c -= a * r - a * (a - 1) / 2;
            const long long b0 = max(0LL, (long long)(m - r));  // rows i >= m - r lose i + r - m + 1
            if (rows > b0) {
                const long long nb = rows - b0;
                c -= nb * (b0 + r - m + 1) + nb * (nb - 1) / 2;
            }
            my_cells += (unsigned long long)c;
        }
    }
    if (cells && lane == 0 && my_cells) atomicAdd(cells, my_cells);
}

// Register-resident band (radius R compile-time): band[k], k = j - i + R, lives
// in registers and is updated in place k-ascending (diag = old band[k], up =
// old band[k+1], left = new band[k-1]).  The query is staged in 4 copies
// shifted by 0..3 samples so every LDS.128 (warp-uniform broadcast) feeds 4
// cells; x_i is prefetched 4 rows at a time.  Per cell: FADD + FMNMX3 + FFMA
// + 1/2 FMNMX3 (row min) + 1/4 LDS.128.
template <int R>
__global__ void __launch_bounds__(128)
dtw32r_kernel(const float *__restrict__ X, int m, const float *__restrict__ Q,
              const float *__restrict__ U, const float *__restrict__ Lo, DtwList L,
              const float *__restrict__ thr, int warps, unsigned long long *__restrict__ cells) {
    constexpr int NB = 2 * R + 1;
    constexpr int NT = (NB + 3) / 4;
    extern __shared__ __align__(16) float rsm[];
    const int q = L.act ? L.act[blockIdx.y] : blockIdx.y;
    const int slot = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int YP = ((m + 2 * R + 8) + 3) & ~3;
    float *yc = rsm;           // 4 x YP
    float *su = rsm + 4 * YP;  // m
    float *sl = su + m;        // m
    int start, end;
    dtw_list_range(L, slot, start, end);
    if (start + (int)blockIdx.x * warps * 32 >= end) return;  // block-uniform: no work
    const float *y = Q + (int64_t)q * m;
    for (int t = threadIdx.x; t < 4 * YP; t += blockDim.x) {
        int c = t / YP, jj = (t - c * YP) + c - R;
        yc[t] = (jj >= 0 && jj < m) ? y[jj] : INFINITY;
    }
    const float T = thr ? thr[q] : INFINITY;
    const bool cb = !isinf(T) && U != nullptr;
    if (cb)
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            su[i] = U[(int64_t)q * m + i];
            sl[i] = Lo[(int64_t)q * m + i];
        }
    __syncthreads();
    const int e = start + (blockIdx.x * warps + w) * 32 + lane;
    if (start + (blockIdx.x * warps + w) * 32 >= end) return;
    const uint32_t row = e < end ? L.rows[(int64_t)slot * L.stride + e] : 0xFFFFFFFFu;
    const bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)slot * L.stride + e] > T));
    {
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        if (L.computed && lane == 0 && vm) atomicAdd(&L.computed[q], __popc(vm));
    }
    const float *x = X + (int64_t)(valid ? row : 0) * m;
    const bool vec = (m & 3) == 0;
    float rem = 0.f, slack = 0.f;
    if (cb) {
        for (int i = 0; i < m; i++) {
            float cv = x[i];
            float v = fmaxf(fmaxf(cv - su[i], sl[i] - cv), 0.f);
            rem = fmaf(v, v, rem);
        }
        slack = rem * (float)(2 * m + 8) * U32_EPS;
    }
    float band[NB];
#pragma unroll
    for (int k = 0; k < NB; k++) band[k] = INFINITY;
    band[R] = 0.f;
    bool alive = valid;
    int rows = 0;
    float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < m; i++) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;
        rows += alive;
        const int c = i & 3;
        float xi;
        if (vec) {
            if (c == 0) xv = __ldg(reinterpret_cast<const float4 *>(x + i));
            xi = c == 0 ? xv.x : c == 1 ? xv.y : c == 2 ? xv.z : xv.w;
        } else {
            xi = __ldg(x + i);
        }
        const float4 *yr = reinterpret_cast<const float4 *>(yc + c * YP + (i - c));
        float left = INFINITY, diag = band[0], rmin = INFINITY;
#pragma unroll
        for (int t = 0; t < NT; t++) {
            const float4 yv = yr[t];
            const float ys[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = 4 * t + u;
                if (k < NB) {
                    const float up = (k + 1 < NB) ? band[k + 1] : INFINITY;
                    const float d = xi - ys[u];
                    const float cv = fmaf(d, d, fminf(fminf(diag, up), left));
                    band[k] = cv;
                    rmin = fminf(rmin, cv);
                    left = cv;
                    diag = up;
                }
            }
        }
        float bound = rmin;
        if (cb) {
            float v = fmaxf(fmaxf(xi - su[i], sl[i] - xi), 0.f);
            rem = fmaf(-v, v, rem);
            bound = rmin + fmaxf(rem - slack, 0.f);
        }
        if (alive && bound > T) alive = false;
    }
    if (e < end) {
        L.out[(int64_t)slot * L.stride + e] = (valid && alive) ? band[R] : INFINITY;
        if (L.abandoned && valid && !alive) atomicAdd(&L.abandoned[q], 1ULL);
    }
    if (cells) {
        unsigned long long cc = (unsigned long long)rows * (unsigned long long)NB;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xFFFFFFFFu, cc, o);
        if (lane == 0 && cc) atomicAdd(cells, cc);
    }
}

// Wave DTW list (per active-query slot) handed to the pooled DTW launcher.
struct DtwWave {
    const uint32_t *rows;
    const float2 *lbs;  // (LB_Keogh, LB_Keogh2) totals per entry
    int64_t stride;
    const int *cnt;
    float *out;
    unsigned long long *abandoned;
    int *computed;
    const uint4 *rec;
    const uint8_t *codes;
    int64_t cstride;
    int mp;
    const int *act;  // block row y -> query act[y]; rows/lbs/out/cnt per slot y
};

// ----------------------------------------------- pooled wave fp32 DTW
// The wave's candidates of all queries run through row passes [0,8),
// [8,16), [16,32), ... .  The first pass works per query slot straight from
// the wave lists; every later pass takes the survivors of all queries from a
// shared pool (state in global memory, SoA), so warps are always full and no
// lane waits for a slower candidate beyond the end of a pass.  Lanes of one
// warp may serve different queries: query samples, envelope and threshold are
// per-lane loads (L1/L2-resident).  Per row block of 4 rows: the band lives
// in registers, the 4 rows interleave with a one-cell lag (all four need the
// same query sample at a step).  Abandon test after row i (UCR-suite
// cumulative bounds, dtw.py:206-215):
//   rmin_i + max(remK_i - slackK, rem2_i - slack2, 0) > thr
//   remK_i = LBK total - sum_{i' <= i} LB_Keogh term of row i'     (rows left)
//   rem2_i = LBK2 total - sum_{j <= i + R} LB_Keogh2 term of col j (columns
//            no path through row i has reached)
// with the totals from the wave LB kernel (code-based terms; the exact-x row
// terms subtracted here are never smaller, so remK stays a lower bound) and
// slack = total * (2m + 8) u for the fp32 running sums.
struct DtwPool {
    int *q;          // local query index
    uint32_t *row;   // series row
    int64_t *out;    // index into the wave's d32 array
    float *st;       // [6][cap]: remK, rem2, slackK, slack2, lo, sc
    float *band;     // [NB][cap]
    int *count;
    int64_t cap;
};

struct DtwCommon {
    const float *X;
    const float *qpad;  // [nq][YP]: y[j] at j + R, +inf outside [0, m)
    const float *U, *Lo;
    const float *thr;
    const uint8_t *codes;
    int64_t cstride;
    int m, mp, YP;
    float *out;  // the wave's d32 array
    unsigned long long *abandoned;
    int *computed;
    unsigned long long *cells;  // profiling: [0] alive lane-cells, [5] executed lane-cells
};

#define DP_WARPS 4
#ifndef DTWP_PAIRED
#define DTWP_PAIRED 1
#endif
#ifndef DTWP_MINB
#define DTWP_MINB 1
#endif
#ifndef DTWP_MINB_NARROW
#define DTWP_MINB_NARROW 3  // radii <= 26: 3 blocks/SM at 168 registers (6.44 vs 6.77 ms per configs[1] batch at 1)
#endif
#ifndef DTWP_BLOCKCUT
#define DTWP_BLOCKCUT 1  // one cut test per 4-row block on the band minimum (else per row)
#endif
#define DP_MAXPASS 64  // longest pooled row pass
#ifndef SSH_DTW_B0
#define SSH_DTW_B0 32  // rows of the first (per query slot) pass: 8 -> 32 saves two pool round trips (configs[1] DTW 6.38 -> 5.71 ms)
#endif
#ifndef SSH_DTW_PASS_DOUBLING
#define SSH_DTW_PASS_DOUBLING 0
#endif

// in-band cells (0 <= j < m, |i - j| <= R) of rows [i0, i0 + n) (profiling counters)
__device__ __forceinline__ unsigned long long dtw_band_cells(int i0, int n, int R, int m) {
    unsigned long long c = 0;
    for (int i = i0; i < i0 + n && i < m; i++) c += (unsigned long long)(min(m - 1, i + R) - max(0, i - R) + 1);
    return c;
}

// rows [a, b) of one lane's candidate; returns whether it is still alive
template <int R>
__device__ __forceinline__ bool dtwp_rows(const DtwCommon &C, int q, uint32_t row, float (&band)[2 * R + 1],
                                          float &remk, float &rem2, float slk, float sl2, float lo, float sc,
                                          float T, int a, int b, bool alive, unsigned long long &cal,
                                          unsigned long long &cex, unsigned long long &nab) {
    constexpr int NB = 2 * R + 1;
    const int m = C.m;
    const float *yq = C.qpad + (int64_t)q * C.YP;
    const float *uq = C.U + (int64_t)q * m, *lq = C.Lo + (int64_t)q * m;
    const float4 *xp = reinterpret_cast<const float4 *>(C.X + (int64_t)row * m);
    const uint8_t *env = C.codes + (int64_t)row * C.cstride + C.mp;
    float4 xn = alive ? __ldg(xp + (a >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i0 = a; i0 < b; i0 += 4) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;
        if (alive && C.cells) cal += dtw_band_cells(i0, 4, R, m);  // in-band cells of rows i0 .. i0 + 3
        cex += 4 * NB;
        const float4 xc = xn;
        if (i0 + 4 < b && alive) xn = __ldg(xp + (i0 >> 2) + 1);
        const int jb = (i0 + R) & ~3;
        uint2 e0 = make_uint2(0u, 0u), e1 = make_uint2(0u, 0u);
        if (alive && jb < m) e0 = __ldg(reinterpret_cast<const uint2 *>(env + 2 * jb));
        if (alive && jb + 4 < m) e1 = __ldg(reinterpret_cast<const uint2 *>(env + 2 * jb + 8));
        const float xr[4] = {xc.x, xc.y, xc.z, xc.w};
        float lft[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
        float rmn[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#if DTWP_PAIRED
        // Row u runs two steps behind row u - 1 (step t: band offset k = t - 2u,
        // query sample i0 + t - u), so rows (u + 1, u) never touch each other's
        // fresh cells within a step and advance together as one f32x2 pair:
        // d = fma(y, -1, x) = x - y and cv = fma(d, d, min3) are the same IEEE
        // operations as the scalar recurrence (in-place band: row u + 1 reads
        // offsets k - 2, k - 1 that row u wrote one and two steps earlier).
        // Rows (1, 0) take the query pair {y_(t-1), y_t}, rows (3, 2) {y_(t-3), y_(t-2)}.
        // No per-cell row minimum: after the block the band IS row i0 + 3, and
        // its minimum feeds one cut test per block (below).
        constexpr int NSTEP = NB + 6;
        const float2 xp01 = make_float2(xr[1], xr[0]), xp23 = make_float2(xr[3], xr[2]);
        const float2 neg1 = make_float2(-1.f, -1.f);
        float yw[NSTEP + 4];
        const float4 *yp4 = reinterpret_cast<const float4 *>(yq + i0);
#if !DTWP_BLOCKCUT
        float cvp[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#endif
#pragma unroll
        for (int t = 0; t < NSTEP; t++) {
            // query samples: one 16-byte load per 4 steps (per-sample 8-byte pair
            // loads from a pre-paired copy measured 1.2-1.8x slower: L1-bound)
            if ((t & 3) == 0 && t < NB + 3) {
                const float4 v = __ldg(yp4 + (t >> 2));
                yw[t] = v.x; yw[t + 1] = v.y; yw[t + 2] = v.z; yw[t + 3] = v.w;
            }
            const float2 ypr[2] = {make_float2(t >= 1 ? yw[t - 1] : 0.f, yw[t]),
                                   make_float2(t >= 3 ? yw[t - 3] : 0.f, t >= 2 ? yw[t - 2] : 0.f)};
            float cvs[4];
            bool val[4];
#pragma unroll
            for (int u = 0; u < 4; u++) val[u] = t - 2 * u >= 0 && t - 2 * u < NB;
#pragma unroll
            for (int pr = 0; pr < 2; pr++) {
                const int ua = 2 * pr, ub = 2 * pr + 1;  // rows (ub, ua) -> pair {.x = ub, .y = ua}
                const int ka = t - 2 * ua, kb = t - 2 * ub;
                if (val[ua] && val[ub]) {
                    const float upa = (ka + 1 < NB) ? band[ka + 1] : INFINITY;
                    const float ma = fminf(fminf(band[ka], upa), lft[ua]);
                    const float mb = fminf(fminf(band[kb], band[kb + 1]), lft[ub]);
                    const float2 d = __ffma2_rn(ypr[pr], neg1, pr ? xp23 : xp01);
                    const float2 cv = __ffma2_rn(d, d, make_float2(mb, ma));
                    cvs[ua] = cv.y;
                    cvs[ub] = cv.x;
                } else {
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int u = h ? ub : ua;
                        const int k = t - 2 * u;
                        if (val[u]) {
                            const float up = (k + 1 < NB) ? band[k + 1] : INFINITY;
                            const float d = xr[u] - (h ? ypr[pr].x : ypr[pr].y);
                            cvs[u] = fmaf(d, d, fminf(fminf(band[k], up), lft[u]));
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = t - 2 * u;
                if (val[u]) {
                    band[k] = cvs[u];
                    lft[u] = cvs[u];
#if !DTWP_BLOCKCUT
                    if (k & 1) rmn[u] = fminf(fminf(rmn[u], cvp[u]), cvs[u]);
                    else cvp[u] = cvs[u];
#endif
                }
            }
        }
#if DTWP_BLOCKCUT
        {
            float bm = band[0];
#pragma unroll
            for (int k = 1; k + 1 < NB; k += 2) bm = fminf(fminf(bm, band[k]), band[k + 1]);
            if (!(NB & 1)) bm = fminf(bm, band[NB - 1]);
            rmn[3] = bm;
        }
#else
#pragma unroll
        for (int u = 0; u < 4; u++) rmn[u] = fminf(rmn[u], cvp[u]);  // NB odd: the last cell
#endif
#else
        const float4 *yp = reinterpret_cast<const float4 *>(yq + i0);
#pragma unroll
        for (int s4 = 0; s4 < (NB + 3 + 3) / 4; s4++) {
            const float4 yv4 = __ldg(yp + s4);
            const float yv[4] = {yv4.x, yv4.y, yv4.z, yv4.w};
#pragma unroll
            for (int sv = 0; sv < 4; sv++) {
                const int stp = 4 * s4 + sv;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int k = stp - u;
                    if (k >= 0 && k < NB) {
                        const float up = (k + 1 < NB) ? band[k + 1] : INFINITY;
                        const float d = xr[u] - yv[sv];
                        const float cv = fmaf(d, d, fminf(fminf(band[k], up), lft[u]));
                        band[k] = cv;
                        lft[u] = cv;
                        rmn[u] = fminf(rmn[u], cv);
                    }
                }
            }
        }
#endif
        const float4 u4 = __ldg(reinterpret_cast<const float4 *>(uq + i0));
        const float4 l4 = __ldg(reinterpret_cast<const float4 *>(lq + i0));
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w}, ll[4] = {l4.x, l4.y, l4.z, l4.w};
        bool cut = false;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const float v = fmaxf(fmaxf(xr[u] - uu[u], ll[u] - xr[u]), 0.f);
            remk = fmaf(-v, v, remk);
            const int jj = i0 + u + R;
            if (jj < m) {
                const int off = (R & 3) + u;  // column jj within the 8-column window
                const uint32_t wv = off < 2 ? e0.x : off < 4 ? e0.y : off < 6 ? e1.x : e1.y;
                const int bu = 2 * (off & 1);
                const float qj = __ldg(yq + jj + R);
                const float ue = fmaf(code_f(wv, bu), sc, lo), le = fmaf(code_f(wv, bu + 1), sc, lo);
                const float dd = fmaxf(fmaxf(qj - ue, le - qj), 0.f);
                rem2 = fmaf(-dd, dd, rem2);
            }
#if !(DTWP_PAIRED && DTWP_BLOCKCUT)
            cut = cut || (rmn[u] + fmaxf(fmaxf(remk - slk, rem2 - sl2), 0.f) > T);
#endif
        }
#if DTWP_PAIRED && DTWP_BLOCKCUT
        cut = rmn[3] + fmaxf(fmaxf(remk - slk, rem2 - sl2), 0.f) > T;
#endif
        if (alive && cut) {
            alive = false;
            nab++;
        }
    }
    return alive;
}

// survivors of a pass -> pool (warp-aggregated append); finished -> d32
template <int R>
__device__ __forceinline__ void dtwp_emit(const DtwCommon &C, const DtwPool &P, bool alive, bool last, int q,
                                          uint32_t row, int64_t oi, const float (&band)[2 * R + 1], float remk,
                                          float rem2, float slk, float sl2, float lo, float sc) {
    constexpr int NB = 2 * R + 1;
    const int lane = threadIdx.x & 31;
    const unsigned am = __ballot_sync(0xFFFFFFFFu, alive && !last);
    int base = 0;
    if (am) {
        if (lane == 0) base = atomicAdd(P.count, __popc(am));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
    }
    if (!alive) return;
    if (last) {
        C.out[oi] = band[R];
        return;
    }
    const int64_t d = base + __popc(am & ((1u << lane) - 1u));
    SSH_DASSERT(d < P.cap);
    if (d >= P.cap) return;  // cannot happen: the pool holds every wave candidate
    P.q[d] = q;
    P.row[d] = row;
    P.out[d] = oi;
    P.st[0 * P.cap + d] = remk;
    P.st[1 * P.cap + d] = rem2;
    P.st[2 * P.cap + d] = slk;
    P.st[3 * P.cap + d] = sl2;
    P.st[4 * P.cap + d] = lo;
    P.st[5 * P.cap + d] = sc;
#pragma unroll
    for (int k = 0; k < NB; k++) P.band[(int64_t)k * P.cap + d] = band[k];
}

__device__ __forceinline__ void dtwp_flush(const DtwCommon &C, unsigned long long cal, unsigned long long cex) {
    if (!C.cells) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cal += __shfl_xor_sync(0xFFFFFFFFu, cal, o);
        cex += __shfl_xor_sync(0xFFFFFFFFu, cex, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (cal) atomicAdd(C.cells, cal);
        if (cex) atomicAdd(C.cells + 5, cex);
    }
}

// first pass, per query slot: wave list entries -> rows [0, b) -> pool
template <int R>
__global__ void __launch_bounds__(32 * DP_WARPS, (R <= 26 ? DTWP_MINB_NARROW : DTWP_MINB))
dtwp_first_kernel(DtwCommon C, const int *__restrict__ act, const uint32_t *__restrict__ wrows,
                  const float2 *__restrict__ wlb, const int *__restrict__ wcnt, int64_t wcap,
                  const uint4 *__restrict__ rec, int b, DtwPool P) {
    constexpr int NB = 2 * R + 1;
    const int slot = blockIdx.y;
    const int q = act[slot];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int total = min(wcnt[slot], (int)wcap);
    const int e0 = (blockIdx.x * DP_WARPS + w) * 32;
    if (e0 >= total) return;
    const int e = e0 + lane;
    const bool have = e < total;
    if (lane == 0 && C.computed) atomicAdd(&C.computed[q], min(32, total - e0));
    const int64_t oi = (int64_t)slot * wcap + e;
    uint32_t row = 0;
    float remk = 0.f, rem2 = 0.f, slk = 0.f, sl2 = 0.f, lo = 0.f, sc = 0.f;
    const float slf = (float)(2 * C.m + 8) * U32_EPS;
    if (have) {
        row = wrows[oi];
        const float2 lb = wlb[oi];
        float2 h = __ldg(reinterpret_cast<const float2 *>(rec + (int64_t)row * 4));
        h.y = fabsf(h.y);
        C.out[oi] = INFINITY;
        remk = lb.x;
        rem2 = lb.y;
        slk = lb.x * slf;
        sl2 = lb.y * slf;
        lo = h.x;
        sc = h.y;
        // columns j < R leave the LB_Keogh2 remainder before row 0
        const uint8_t *env = C.codes + (int64_t)row * C.cstride + C.mp;
        const float *yq = C.qpad + (int64_t)q * C.YP;
        uint2 ev = make_uint2(0u, 0u);
        for (int j = 0; j < min(R, C.m); j++) {
            if ((j & 3) == 0) ev = __ldg(reinterpret_cast<const uint2 *>(env + 2 * j));
            const uint32_t wv = (j & 2) ? ev.y : ev.x;
            const int bu = 2 * (j & 1);
            const float qj = __ldg(yq + j + R);
            const float ue = fmaf(code_f(wv, bu), sc, lo), le = fmaf(code_f(wv, bu + 1), sc, lo);
            const float d = fmaxf(fmaxf(qj - ue, le - qj), 0.f);
            rem2 = fmaf(-d, d, rem2);
        }
    }
    float band[NB];
#pragma unroll
    for (int k = 0; k < NB; k++) band[k] = k == R ? 0.f : INFINITY;
    unsigned long long cal = 0, cex = 0, nab = 0;
    const bool alive = dtwp_rows<R>(C, q, row, band, remk, rem2, slk, sl2, lo, sc, C.thr[q], 0, b, have, cal,
                                    cex, nab);
    if (nab && C.abandoned) atomicAdd(&C.abandoned[q], nab);
    dtwp_emit<R>(C, P, alive, b >= C.m, q, row, oi, band, remk, rem2, slk, sl2, lo, sc);
    dtwp_flush(C, cal, cex);
}

// later passes over the pooled survivors of all queries (persistent grid)
template <int R>
__device__ __forceinline__ void dtwp_pass_body(const DtwCommon &C, const DtwPool &in, const DtwPool &P, int a, int b,
                                               int n) {
    constexpr int NB = 2 * R + 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long cal = 0, cex = 0;
    for (int e0 = (blockIdx.x * DP_WARPS + w) * 32; e0 < n; e0 += gridDim.x * DP_WARPS * 32) {
        const int e = e0 + lane;
        const bool have = e < n;
        int q = 0;
        uint32_t row = 0;
        int64_t oi = 0;
        float remk = 0.f, rem2 = 0.f, slk = 0.f, sl2 = 0.f, lo = 0.f, sc = 0.f;
        float band[NB];
        if (have) {
            q = in.q[e];
            row = in.row[e];
            oi = in.out[e];
            remk = in.st[0 * in.cap + e];
            rem2 = in.st[1 * in.cap + e];
            slk = in.st[2 * in.cap + e];
            sl2 = in.st[3 * in.cap + e];
            lo = in.st[4 * in.cap + e];
            sc = in.st[5 * in.cap + e];
#pragma unroll
            for (int k = 0; k < NB; k++) band[k] = in.band[(int64_t)k * in.cap + e];
        } else {
#pragma unroll
            for (int k = 0; k < NB; k++) band[k] = INFINITY;
        }
        unsigned long long nab = 0;
        const bool alive = dtwp_rows<R>(C, q, row, band, remk, rem2, slk, sl2, lo, sc, have ? C.thr[q] : 0.f,
                                        a, b, have, cal, cex, nab);
        if (nab && C.abandoned) atomicAdd(&C.abandoned[q], nab);
        dtwp_emit<R>(C, P, alive, b >= C.m, q, row, oi, band, remk, rem2, slk, sl2, lo, sc);
    }
    dtwp_flush(C, cal, cex);
}

// Tail of a pooled wave: once fewer than `lim` candidates are left, the
// remaining rows [a, m) of each run in one launch, one warp per candidate,
// as an anti-diagonal wavefront (lane l owns rows a + l, a + l + 32, ...,
// starting two steps behind lane l - 1 and computing two band cells per step,
// so a row of NB = 2R + 1 cells takes R + 1 steps and a round of 32 rows 64).
// The cell above arrives by shuffle from lane l - 1 (lane 0: lane 31 of the
// previous round, or the pooled band of row a - 1 in the first round).  Cells
// are the pooled kernel's fmaf(d, d, min(diag, up, left)), so the distance is
// the same fp32 value; a lane checks the cumulative bound of dtwp_rows when
// its row ends, with the LB_Keogh / LB_Keogh2 remainders of its row taken from
// warp prefix sums of the row / column terms at the start of each round.
#define DT_WARPS 4
#ifndef SSH_DTW_TAIL
#define SSH_DTW_TAIL 2048  // pooled candidates below which the tail kernel takes over
#endif

__device__ __forceinline__ float warp_incl_scan(float v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float u = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

template <int R>
__device__ __forceinline__ void dtwt_body(const DtwCommon &C, const DtwPool &in, int a, int n, float *dtsm) {
    constexpr int NB = 2 * R + 1, NP = R + 1;  // pairs per row; the last pair's second cell is out of band
    static_assert(NP <= 63, "a row must end before its lane's next round");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int m = C.m, YP = C.YP;
    const int stride = YP + 2 * 64 + 4;
    float *ys = dtsm + (size_t)w * stride;
    float *bs = ys + YP;
    const int rows = m - a, rounds = (rows + 31) >> 5;
    const int last_t = 64 * (rounds - 1) + 62 + NP - 1;
    const int owner = (m - 1 - a) & 31;
    unsigned long long cal = 0, cex = 0;
    for (int e = blockIdx.x * DT_WARPS + w; e < n; e += gridDim.x * DT_WARPS) {
        const int q = in.q[e];
        const uint32_t row = in.row[e];
        const int64_t oi = in.out[e];
        float remk = in.st[0 * in.cap + e], rem2 = in.st[1 * in.cap + e];
        const float slk = in.st[2 * in.cap + e], sl2 = in.st[3 * in.cap + e];
        const float lo = in.st[4 * in.cap + e], sc = in.st[5 * in.cap + e];
        const float T = C.thr[q];
        const float *yq = C.qpad + (int64_t)q * YP;
        __syncwarp();
        for (int t = lane; t < YP; t += 32) ys[t] = __ldg(yq + t);
        for (int k = lane; k < 2 * 64 + 4; k += 32) bs[k] = k < NB ? in.band[(int64_t)k * in.cap + e] : INFINITY;
        __syncwarp();
        const float *xp = C.X + (int64_t)row * m;
        const uint8_t *env = C.codes + (int64_t)row * C.cstride + C.mp;
        const float *uq = C.U + (int64_t)q * m, *lq = C.Lo + (int64_t)q * m;
        // row / column inputs of this lane's row in the next round (prefetched a round ahead)
        float xn = 0.f, un = 0.f, ln = 0.f;
        uint32_t en = 0;
        auto fetch = [&](int i) {
            xn = 0.f;
            un = 0.f;
            ln = 0.f;
            en = 0;
            if (i < m) {
                xn = __ldg(xp + i);
                un = __ldg(uq + i);
                ln = __ldg(lq + i);
                if (i + R < m) en = *reinterpret_cast<const unsigned short *>(env + 2 * (i + R));
            }
        };
        fetch(a + lane);
        float xr = 0.f, rk = 0.f, r2 = 0.f;
        float2 rp = lane == 0 ? make_float2(bs[0], bs[1]) : make_float2(INFINITY, INFINITY);
        float c0 = INFINITY, c1 = INFINITY, left = INFINITY, rmn = INFINITY, res = INFINITY;
        bool cut = false, ab = false;
        const int kend = (last_t + 64) >> 6;  // rows of the last round drain into one more
        for (int k = 0; k < kend; k++) {
            // round k: LB_Keogh / LB_Keogh2 remainders after rows a + 32 k + lane
            const int ik = a + 32 * k + lane;
            const float xrn = xn;
            float kt = 0.f, ct = 0.f;
            if (ik < m) {
                const float g = fmaxf(fmaxf(xn - un, ln - xn), 0.f);
                kt = g * g;
                if (ik + R < m) {
                    const float qj = ys[ik + 2 * R];
                    const float ue = fmaf((float)(en & 0xFFu), sc, lo), le = fmaf((float)(en >> 8), sc, lo);
                    const float dd = fmaxf(fmaxf(qj - ue, le - qj), 0.f);
                    ct = dd * dd;
                }
            }
            fetch(ik + 32);
            kt = warp_incl_scan(kt);
            ct = warp_incl_scan(ct);
            const float rkn = remk - kt, r2n = rem2 - ct;
            remk -= __shfl_sync(0xFFFFFFFFu, kt, 31);
            rem2 -= __shfl_sync(0xFFFFFFFFu, ct, 31);
            const int send = min(64, last_t + 1 - 64 * k);
            for (int s0 = 0; s0 < send; s0 += 8) {
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int s = s0 + u;
                    // the pair lane - 1 produced last step (lane 0, first round: the pooled
                    // band of row a - 1 while its row a needs it, s < NP; from step NP on it
                    // carries lane 31's row a + 31 into round 1 like every later round)
                    const float2 bb = reinterpret_cast<const float2 *>(bs)[min(s + 1, 63)];
                    const bool fromb = (k == 0) & (lane == 0) & (s < NP);
                    float rx = __shfl_sync(0xFFFFFFFFu, c0, (lane + 31) & 31);
                    float ry = __shfl_sync(0xFFFFFFFFu, c1, (lane + 31) & 31);
                    rx = fromb ? bb.x : rx;
                    ry = fromb ? bb.y : ry;
                    const int d = s - 2 * lane;  // >= 0: this round's row, else the previous round's
                    const int sp = d & 63;
                    const int i = ik - (d < 0 ? 32 : 0);
                    const bool act = (s < send) & (sp < NP) & (i < m) & (i >= a);
                    const bool st0 = d == 0;
                    xr = st0 ? xrn : xr;
                    rk = st0 ? rkn : rk;
                    r2 = st0 ? r2n : r2;
                    left = st0 ? INFINITY : left;
                    rmn = st0 ? INFINITY : rmn;
                    const int yi = act ? i + 2 * sp : 0;
                    SSH_DASSERT(yi + 1 < YP);
                    const float d0 = xr - ys[yi], d1 = xr - ys[yi + 1];
                    const float n0 = fmaf(d0, d0, fminf(fminf(rp.x, rp.y), left));
                    const float n1 = fmaf(d1, d1, fminf(fminf(rp.y, rx), n0));
                    c0 = act ? n0 : INFINITY;
                    c1 = (act && sp < NP - 1) ? n1 : INFINITY;
                    left = c1;
                    rmn = fminf(rmn, fminf(c0, c1));
                    res = (act & (i == m - 1) & (sp == (R >> 1))) ? ((R & 1) ? c1 : c0) : res;
                    cut |= act & (sp == NP - 1) & (rmn + fmaxf(fmaxf(rk - slk, r2 - sl2), 0.f) > T);
                    if (C.cells && act && sp == NP - 1) cal += dtw_band_cells(i, 1, R, m);  // row i complete
                    rp = make_float2(rx, ry);
                }
                if (__any_sync(0xFFFFFFFFu, cut)) {
                    ab = true;
                    cex += 2 * (64 * k + s0 + 8);
                    break;
                }
            }
            if (ab) break;
        }
        if (ab) {
            if (lane == 0 && C.abandoned) atomicAdd(&C.abandoned[q], 1ull);
        } else {
            cex += 2 * (last_t + 1);
            res = __shfl_sync(0xFFFFFFFFu, res, owner);
            if (lane == 0) C.out[oi] = res;
        }
    }
    dtwp_flush(C, cal, cex);
}

// one pooled level: rows [a, b) of every pooled candidate, or, once fewer
// than lim are left, all remaining rows [a, m) in the wavefront tail
template <int R>
__global__ void __launch_bounds__(32 * DP_WARPS, (R <= 26 ? DTWP_MINB_NARROW : DTWP_MINB))
dtwp_level_kernel(DtwCommon C, DtwPool in, DtwPool P, int a, int b, int lim) {
    extern __shared__ __align__(16) float dtsm[];
    const int n = min(*in.count, (int)in.cap);
    if (n == 0) return;
    if (n < lim) dtwt_body<R>(C, in, a, n, dtsm);
    else dtwp_pass_body<R>(C, in, P, a, b, n);
}

// padded query copies for the pooled DTW: qpad[q][t] = y[t - R] (+inf outside)
__global__ void qpad_kernel(const float *__restrict__ Q, int m, int R, int YP, float *__restrict__ qpad) {
    const int q = blockIdx.x;
    for (int t = threadIdx.x; t < YP; t += blockDim.x) {
        const int j = t - R;
        qpad[(int64_t)q * YP + t] = (j >= 0 && j < m) ? Q[(int64_t)q * m + j] : INFINITY;
    }
}


// Exact f64 rescoring, register band (radius R) with 4 rows interleaved per
// lane (one-cell lag, as in the fp32 kernels): the reference recurrence
// d = x - y; d = d * d; c = d + min(diag, up, left) (dtw.py:100-113) with
// _rn intrinsics, out-of-band / out-of-range cells +inf (the query is padded
// with +inf, so such cells evaluate to +inf exactly).  One query per block row.
template <int R>
__global__ void __launch_bounds__(128)
dtw64r_kernel(const float *__restrict__ X, int m, const float *__restrict__ Q, const uint32_t *__restrict__ list,
              int64_t list_stride, const int *__restrict__ list_cnt, double *__restrict__ out) {
    constexpr int NB = 2 * R + 1;
    extern __shared__ __align__(16) double ysm[];
    const int q = blockIdx.y;
    const int cnt = list_cnt[q];
    if ((int)(blockIdx.x * blockDim.x) >= cnt) return;
    const int YP = m + 2 * R + 8;
    for (int t = threadIdx.x; t < YP; t += blockDim.x) {
        const int j = t - R;
        ysm[t] = (j >= 0 && j < m) ? (double)Q[(int64_t)q * m + j] : (double)INFINITY;
    }
    __syncthreads();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= cnt) return;
    const float4 *xp = reinterpret_cast<const float4 *>(X + (int64_t)list[(int64_t)q * list_stride + e] * m);
    double band[NB];
#pragma unroll
    for (int k = 0; k < NB; k++) band[k] = k == R ? 0.0 : (double)INFINITY;
    for (int i0 = 0; i0 < m; i0 += 4) {
        const float4 xv = __ldg(xp + (i0 >> 2));
        const double xr[4] = {(double)xv.x, (double)xv.y, (double)xv.z, (double)xv.w};
        double lft[4] = {(double)INFINITY, (double)INFINITY, (double)INFINITY, (double)INFINITY};
        const double *yp = ysm + i0;
#pragma unroll
        for (int st = 0; st < NB + 3; st++) {
            const double yv = yp[st];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = st - u;
                if (k >= 0 && k < NB) {
                    const double up = (k + 1 < NB) ? band[k + 1] : (double)INFINITY;
                    double d = __dsub_rn(xr[u], yv);
                    d = __dmul_rn(d, d);
                    const double c = __dadd_rn(d, fmin(fmin(up, lft[u]), band[k]));
                    band[k] = c;
                    lft[u] = c;
                }
            }
        }
    }
    out[(int64_t)q * list_stride + e] = band[R];
}


// Exact f64 DTW, one warp per pair, anti-diagonal wavefront over rows: lane l
// owns rows l, l + 32, ...; within a round it walks its row's band left to
// right, two steps behind lane l - 1, so the cell above arrives by a shuffle
// from lane l - 1 one step earlier (its diagonal one step before that) and
// lane 0 continues after lane 31 (period 64 steps, 2 r + 1 busy).  Every
// cell is the reference recurrence d = x - y; d = d * d; c = d + min(up,
// left, diag) (dtw.py:100-113) with _rn intrinsics, so the result is the
// same bits as a sequential evaluation; cells outside the band or the series
// are +inf.  Needs 2 r + 1 <= 64 (a lane's row must end before its next
// round starts).  The query (as f64, padded with +inf) is staged per warp.
// Pairs: list mode (blockIdx.y = query, list[q][e]) or explicit (qrow, xrow).
#define D64W_WARPS 4
__global__ void __launch_bounds__(32 * D64W_WARPS)
dtw64w_kernel(const float *__restrict__ X, int m, int r, const float *__restrict__ Q,
              const int32_t *__restrict__ qrow, const uint32_t *__restrict__ list, int64_t list_stride,
              const int *__restrict__ list_cnt, const int64_t *__restrict__ xrow64, int64_t npair,
              double *__restrict__ out) {
    extern __shared__ double ysm64[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int YP = m + 2 * r + 2;
    double *yq = ysm64 + (size_t)w * YP;  // yq[j + r] = y[j]
    int64_t e, row;
    int q;
    if (list) {
        q = blockIdx.y;
        e = (int64_t)blockIdx.x * D64W_WARPS + w;
        if (e >= list_cnt[q]) return;  // warp-uniform
        row = list[(int64_t)q * list_stride + e];
    } else {
        e = (int64_t)blockIdx.x * D64W_WARPS + w;
        if (e >= npair) return;
        q = qrow[e];
        row = xrow64[e];
    }
    const double inf = (double)INFINITY;
    const float *y = Q + (int64_t)q * m;
    for (int t = lane; t < YP; t += 32) {
        const int j = t - r;
        yq[t] = (j >= 0 && j < m) ? (double)y[j] : inf;
    }
    __syncwarp();
    const float *x = X + row * m;
    const int NB = 2 * r + 1;
    const int rounds = (m + 31) / 32;
    const int last_t = 64 * (rounds - 1) + 2 * 31 + NB;  // last active step of lane 31
    double cur = inf;     // value this lane produced in the previous step (shared to lane + 1)
    double diag_in = inf; // value received one step ago (= diag for this step)
    double left = inf;
    double xi = 0.0;
    double res = inf;
    for (int t = 0; t <= last_t; t++) {
        // value from lane - 1 (lane 0: lane 31, previous round) produced at step t - 1
        const double up_in = __shfl_sync(0xFFFFFFFFu, cur, (lane + 31) & 31);
        const int tl = t - 2 * lane;
        double c = inf;
        if (tl >= 0) {
            const int k = tl >> 6, sstep = tl & 63;
            const int i = 32 * k + lane;
            if (sstep < NB && i < m) {
                if (sstep == 0) {
                    xi = (double)x[i];
                    left = inf;
                }
                const int j = i - r + sstep;
                double up = up_in, dg = diag_in;
                if (i == 0) {
                    up = inf;
                    dg = (j == 0) ? 0.0 : inf;
                } else if (sstep == NB - 1) {
                    up = inf;  // D(i - 1, i + r) lies outside row i - 1's band
                }
                if (j >= 0 && j < m) {
                    double d = __dsub_rn(xi, yq[j + r]);
                    d = __dmul_rn(d, d);
                    double best = up;
                    if (left < best) best = left;
                    if (dg < best) best = dg;
                    c = __dadd_rn(d, best);
                }
                left = c;
                if (i == m - 1 && j == m - 1) res = c;
            }
        }
        diag_in = up_in;
        cur = c;
    }
    // the lane owning row m - 1 holds the result
    const int owner = (m - 1) & 31;
    res = __shfl_sync(0xFFFFFFFFu, res, owner);
    if (lane == 0) {
        if (list) out[(int64_t)q * list_stride + e] = res;
        else out[e] = res;
    }
}

// Exact f64 DTW for bands wider than the lane-per-row wavefront covers
// (2 r + 1 > 64): the band-chunked warp wavefront of dtw_warp.cuh, one warp
// per pair (list mode: blockIdx.y = query, list[q][e]; or explicit pairs).
#define D64B_WARPS 4
template <int C>
__global__ void __launch_bounds__(32 * D64B_WARPS)
dtw64band_kernel(const float *__restrict__ X, int m, int r, const float *__restrict__ Q,
                 const int32_t *__restrict__ qrow, const uint32_t *__restrict__ list, int64_t list_stride,
                 const int *__restrict__ list_cnt, const int64_t *__restrict__ xrow64, int64_t npair,
                 double *__restrict__ out) {
    const int w = threadIdx.x >> 5;
    const int64_t e = (int64_t)blockIdx.x * D64B_WARPS + w;
    int q;
    int64_t row;
    if (list) {
        q = blockIdx.y;
        if (e >= list_cnt[q]) return;  // warp-uniform
        row = list[(int64_t)q * list_stride + e];
    } else {
        if (e >= npair) return;
        q = qrow[e];
        row = xrow64[e];
    }
    const double res = dtw_warp_band64<float, C>(X + row * m, Q + (int64_t)q * m, m, r, -1.0);
    if ((threadIdx.x & 31) == 0) {
        if (list) out[(int64_t)q * list_stride + e] = res;
        else out[e] = res;
    }
}

static int launch_dtw64band(const float *X, int m, int r, const float *Q, const int32_t *qrow,
                            const uint32_t *list, int64_t stride, const int *cnt, const int64_t *xrow,
                            int64_t n, int nq, double *out, cudaStream_t st, bool *done) {
    *done = false;
    const int C = dtw_warp_chunk(r);
    if (C == 0 || C > 16) return SSH_OK;
    dim3 grid((unsigned)ssh_div_up(n, D64B_WARPS), (unsigned)(list ? nq : 1));
#define D64B_CALL(CC) \
    dtw64band_kernel<CC><<<grid, 32 * D64B_WARPS, 0, st>>>(X, m, r, Q, qrow, list, stride, cnt, xrow, n, out)
    DTW_WARP_DISPATCH16(C, D64B_CALL)
#undef D64B_CALL
    SSH_CHECK_LAUNCH();
    *done = true;
    return SSH_OK;
}

// ------------------------------------------------------------ fp64 DTW
// exact reference arithmetic (dtw.py:100-113): d = x - y; d = d*d; c = d + min(...)
__global__ void dtw64_kernel(const float *__restrict__ X, int m, int r, const float *__restrict__ Q,
                             const int32_t *__restrict__ qrow, const uint32_t *__restrict__ list,
                             int64_t list_stride, const int *__restrict__ list_cnt,
                             const int64_t *__restrict__ xrow64, int64_t npair,
                             double *__restrict__ out) {
    extern __shared__ double bsm[];
    const int B = 2 * r + 2;
    const int nt = blockDim.x;
    double *band = bsm + threadIdx.x;  // band[k * nt]
    int64_t e;
    int q;
    int64_t row;
    if (list) {  // per-query list mode: blockIdx.y = q
        q = blockIdx.y;
        e = (int64_t)blockIdx.x * nt + threadIdx.x;
        int cnt = list_cnt[q];
        if (e >= cnt) return;
        row = list[(int64_t)q * list_stride + e];
    } else {  // explicit pairs
        e = (int64_t)blockIdx.x * nt + threadIdx.x;
        if (e >= npair) return;
        q = qrow[e];
        row = xrow64[e];
    }
    const float *x = X + row * m;
    const float *y = Q + (int64_t)q * m;
    const double inf = (double)INFINITY;
    for (int k = 0; k < B; k++) band[k * nt] = inf;
    band[r * nt] = 0.0;
    for (int i = 0; i < m; i++) {
        const double xi = (double)x[i];
        double left = inf;
        double diag = band[0];
        for (int k = 0; k <= 2 * r; k++) {
            double up = band[(k + 1) * nt];
            int j = i + k - r;
            double c = inf;
            if (j >= 0 && j < m) {
                double d = __dsub_rn(xi, (double)y[j]);
                d = __dmul_rn(d, d);
                double best = up;
                if (left < best) best = left;
                if (diag < best) best = diag;
                c = __dadd_rn(d, best);
            }
            band[k * nt] = c;
            left = c;
            diag = up;
        }
    }
    double res = band[r * nt];
    if (list) out[(int64_t)q * list_stride + e] = res;
    else out[e] = res;
}

// ------------------------------------------------------- thresholds / waves
// One wave, part 3: fold the wave's fp32 DTWs into the per-query k smallest
// (topk), tighten thr = min(thr, kth (1 + eps)), keep every evaluated
// candidate with d32 <= thr (only those can reach the final rescoring set,
// since thr never increases and always stays >= the final kth (1 + eps)),
// advance the wave start and decide whether the query is done (next member's
// LB_PAA bin above thr's bin => every remaining LB_PAA exceeds thr).
__global__ void wave_update_kernel(const int *__restrict__ act, const float *__restrict__ wd32,
                                   const uint32_t *__restrict__ wrows,
                                   int *__restrict__ wcnt, int wcap, const float *__restrict__ slbp,
                                   const int64_t *__restrict__ roff, const int *__restrict__ cnt,
                                   const int *__restrict__ binhi,
                                   int wave, int k, float eps, float *__restrict__ topk,
                                   float *__restrict__ thr, int *__restrict__ pos,
                                   int *__restrict__ done, int *__restrict__ overflow,
                                   uint32_t *__restrict__ keep_rows, float *__restrict__ keep_d32,
                                   int *__restrict__ keep_cnt, int kcap) {
    __shared__ int red[32];
    extern __shared__ uint32_t tmp[];  // k entries
    __shared__ int npos;
    const int slot = blockIdx.x;
    const int q = act[slot];
    const int nw = min(wcnt[slot], wcap);
    const uint32_t *wb = reinterpret_cast<const uint32_t *>(wd32 + (int64_t)slot * wcap);
    uint32_t *tb = reinterpret_cast<uint32_t *>(topk + (int64_t)q * k);
    const int nfin = block_count_le2<uint32_t>(tb, k, wb, nw, 0x7F7FFFFFu, red);
    float T = thr[q];
    if (nfin >= k) {
        const uint32_t kv = block_kth2<uint32_t>(tb, k, wb, nw, k, 0x7F7FFFFFu, red);
        if (threadIdx.x == 0) npos = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < k; e += blockDim.x)
            if (tb[e] < kv) tmp[atomicAdd(&npos, 1)] = tb[e];
        for (int e = threadIdx.x; e < nw; e += blockDim.x)
            if (wb[e] < kv) tmp[atomicAdd(&npos, 1)] = wb[e];
        __syncthreads();
        const int c = npos;
        for (int e = threadIdx.x; e < k; e += blockDim.x) tb[e] = e < c ? tmp[e] : kv;
        T = fminf(T, thr_from(__uint_as_float(kv), eps));
    } else {
        if (threadIdx.x == 0) {
            int c = 0;
            for (int e = 0; e < k; e++) c += tb[e] <= 0x7F7FFFFFu;
            npos = c;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nw; e += blockDim.x)
            if (wb[e] <= 0x7F7FFFFFu) tb[atomicAdd(&npos, 1)] = wb[e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nw; e += blockDim.x) {
        const float v = wd32[(int64_t)slot * wcap + e];
        if (v <= T) {
            const int p = atomicAdd(&keep_cnt[q], 1);
            if (p < kcap) {
                keep_rows[(int64_t)q * kcap + p] = wrows[(int64_t)slot * wcap + e];
                keep_d32[(int64_t)q * kcap + p] = v;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        thr[q] = T;
        wcnt[slot] = 0;
        const int total = cnt[q];
        const int end = min(total, pos[q] + wave);
        pos[q] = end;
        const bool fin = end >= total || lb_bin(slbp[roff[q] + end]) > lb_bin(T);
        done[q] = fin;
        // list exhausted while thr still reaches past the cutoff: members in
        // the dropped bins may still beat thr -> overflow round
        if (end >= total && lb_bin(T) > (unsigned)binhi[q]) overflow[q] = 1;
    }
}

// compact list of the queries still in the wave loop (order irrelevant)
__global__ void compact_active_kernel(const int *__restrict__ done, int nq, int *__restrict__ act,
                                      int *__restrict__ nact) {
    __shared__ int n;
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int q0 = 0; q0 < nq; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        const bool a = q < nq && !done[q];
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, a);
        int base = 0;
        if (lane == 0 && bm) base = atomicAdd(&n, __popc(bm));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (a) act[base + __popc(bm & ((1u << lane) - 1u))] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) *nact = n;
}

// Rescoring set: kept candidates with d32 <= T_k (1 + eps), T_k = k-th
// smallest kept d32 (the kept set contains the k smallest of all evaluated).
__global__ void select_kernel(const uint32_t *__restrict__ keep_rows, const float *__restrict__ keep_d32,
                              const int *__restrict__ keep_cnt, int kcap, int k, float eps,
                              uint32_t *__restrict__ resc, int *__restrict__ resc_cnt,
                              long long *__restrict__ counters, const int *__restrict__ cnt,
                              const int *__restrict__ pos) {
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    const int n = min(keep_cnt[q], kcap);
    const uint32_t *b = reinterpret_cast<const uint32_t *>(keep_d32 + (int64_t)q * kcap);
    const int nfin = block_count_le2<uint32_t>(b, n, nullptr, 0, 0x7F7FFFFFu, red);
    const int kk = min(k, nfin);
    float bound = -1.f;
    if (kk > 0) bound = thr_from(__uint_as_float(block_kth2<uint32_t>(b, n, nullptr, 0, kk, 0x7F7FFFFFu, red)), eps);
    if (threadIdx.x == 0) npos = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        if (keep_d32[(int64_t)q * kcap + e] <= bound)
            resc[(int64_t)q * kcap + atomicAdd(&npos, 1)] = keep_rows[(int64_t)q * kcap + e];
    __syncthreads();
    if (threadIdx.x == 0) {
        resc_cnt[q] = npos;
        counters[q * 5 + 1] += cnt[q] - pos[q];  // never visited: LB_PAA > thr
    }
}

// exact top-k by (d64, id) of the rescored set; P2 >= k power of two
__global__ void topk_kernel(const uint32_t *__restrict__ resc, const double *__restrict__ d64,
                            const int *__restrict__ resc_cnt, int RS, int P2, int k,
                            int64_t id_base, const long long *__restrict__ n_cand,
                            long long *__restrict__ out_ids, double *__restrict__ out_d2,
                            int *__restrict__ n_out) {
    extern __shared__ double ksm[];
    double *key = ksm;
    uint32_t *val = reinterpret_cast<uint32_t *>(ksm + P2);
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    const int cnt = n_cand[q] > 0 ? min(resc_cnt[q], RS) : 0;
    const int n = min(k, cnt);
    const uint64_t *bits = reinterpret_cast<const uint64_t *>(d64 + (int64_t)q * RS);
    const uint32_t *ids = resc + (int64_t)q * RS;
    uint64_t V = 0x7FF0000000000000ULL;
    uint32_t idcut = 0xFFFFFFFFu;
    if (n > 0 && cnt > n) {
        V = block_kth2<uint64_t>(bits, cnt, nullptr, 0, n, 0x7FF0000000000000ULL, red);
        int nless = V ? block_count_le2<uint64_t>(bits, cnt, nullptr, 0, V - 1, red) : 0;
        int need = n - nless;
        uint32_t lo = 0, hi = 0xFFFFFFFFu;
        while (lo < hi) {  // need-th smallest id among entries equal to V
            uint32_t mid = lo + (hi - lo) / 2;
            int c = 0;
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) c += (bits[e] == V && ids[e] <= mid);
            if (block_sum(c, red) >= need) hi = mid; else lo = mid + 1;
        }
        idcut = lo;
    }
    if (threadIdx.x == 0) npos = 0;
    for (int e = threadIdx.x; e < P2; e += blockDim.x) {
        key[e] = (double)INFINITY;
        val[e] = 0xFFFFFFFFu;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        uint64_t b = bits[e];
        if (cnt <= n || b < V || (b == V && ids[e] <= idcut)) {
            int p = atomicAdd(&npos, 1);
            if (p < P2) {
                key[p] = __longlong_as_double((long long)b);
                val[p] = ids[e];
            }
        }
    }
    __syncthreads();
    block_sort_pairs<double>(key, val, P2);
    for (int e = threadIdx.x; e < k; e += blockDim.x) {
        out_ids[(int64_t)q * k + e] = e < n ? (long long)val[e] + id_base : -1LL;
        out_d2[(int64_t)q * k + e] = e < n ? key[e] : (double)INFINITY;
    }
    if (threadIdx.x == 0) n_out[q] = n;
}

__global__ void finalize_counters(const int *__restrict__ computed,
                                  const unsigned long long *__restrict__ abandoned, int nq,
                                  const long long *__restrict__ n_cand,
                                  const int *__restrict__ is_fb, long long *__restrict__ counters,
                                  int *__restrict__ status) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    counters[q * 5 + 3] = computed[q];
    counters[q * 5 + 4] = (long long)abandoned[q];
    // every member not pruned by LB_Kim / LB_Keogh2 nor DTW-evaluated was
    // pruned by a query-envelope bound (LB_PAA key, cutoff, LB_Keogh)
    counters[q * 5 + 1] = n_cand[q] - counters[q * 5 + 0] - counters[q * 5 + 2] - computed[q];
    status[q] = n_cand[q] == 0 ? 1 : (is_fb[q] ? 2 : 0);
}

__global__ void wave_init_kernel(int nq, int k, int round, const int *__restrict__ cnt,
                                 int *__restrict__ overflow, float *__restrict__ thr,
                                 float *__restrict__ topk, int *__restrict__ pos, int *__restrict__ done,
                                 int *__restrict__ wcnt, int *__restrict__ keep_cnt,
                                 int *__restrict__ computed, unsigned long long *__restrict__ aband) {
    const int64_t n = (int64_t)nq * k;
    if (round == 0)
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
            reinterpret_cast<uint32_t *>(topk)[e] = 0xFFFFFFFFu;  // NaN bits: above every finite value
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        pos[q] = 0;
        wcnt[q] = 0;
        if (round == 0) {
            thr[q] = INFINITY;
            done[q] = cnt[q] == 0;
            keep_cnt[q] = 0;
            computed[q] = 0;
            aband[q] = 0ULL;
        } else {
            // overflow round: only the flagged queries continue, with their state
            done[q] = !overflow[q] || cnt[q] == 0;
        }
        overflow[q] = 0;
    }
}

// ------------------------------------------------------------------ host
namespace {
struct Arena {
    std::vector<void *> ptrs;
    cudaStream_t st;
    cudaError_t err = cudaSuccess;
    template <typename T>
    T *get(size_t n) {
        void *p = nullptr;
        if (err != cudaSuccess) return nullptr;
        err = cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st);
        if (err != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return (T *)p;
    }
    ~Arena() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
};

// bump carving of one ctx slot (a first pass with base == nullptr sizes it)
struct Carver {
    unsigned char *base = nullptr;
    size_t off = 0;
    template <typename T>
    T *take(size_t n) {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += std::max<size_t>(n, 1) * sizeof(T);
        return p;
    }
};

#define SSH_MEMBER_BUDGET ((int64_t)1 << 29)  // members per sub-range (8 GiB of lists)
#define SSH_MEMBER_TARGET 65536               // round-0 members per query (sampled cutoff)
#ifndef SSH_WAVE_GROWTH
#define SSH_WAVE_GROWTH 8                     // wave size multiplier
#endif

struct QueryBufs {
    uint64_t *qsig, *qbits, *bstart;
    uint32_t *blen;
    int64_t *roff;
    int *isfb, *mcnt, *pos, *done, *active, *wcnt, *keep_cnt, *rcnt, *computed, *act, *nact;
    int *binlo, *binhi, *overflow;
    float *U, *Lo, *Useg, *Lseg, *thr;
    unsigned long long *aband;

    void carve(Carver &c, int nc, int L, int words, int m, int nseg) {
        qsig = c.take<uint64_t>((size_t)nc * L);
        qbits = c.take<uint64_t>((size_t)nc * words);
        bstart = c.take<uint64_t>((size_t)nc * L);
        blen = c.take<uint32_t>((size_t)nc * L);
        roff = c.take<int64_t>(nc + 1);
        isfb = c.take<int>(nc);
        mcnt = c.take<int>(nc);
        pos = c.take<int>(nc);
        done = c.take<int>(nc);
        active = c.take<int>(1);
        nact = c.take<int>(1);
        act = c.take<int>(nc);
        binlo = c.take<int>(nc);
        binhi = c.take<int>(nc);
        overflow = c.take<int>(nc);
        wcnt = c.take<int>(nc);
        keep_cnt = c.take<int>(nc);
        rcnt = c.take<int>(nc);
        computed = c.take<int>(nc);
        U = c.take<float>((size_t)nc * m);
        Lo = c.take<float>((size_t)nc * m);
        Useg = c.take<float>((size_t)nc * nseg);
        Lseg = c.take<float>((size_t)nc * nseg);
        thr = c.take<float>(nc);
        aband = c.take<unsigned long long>(nc);
    }

    // view of queries [qa, ...): per-query arrays advanced by qa (roff and the
    // scalar flags stay shared; roff is rewritten per sub-range)
    QueryBufs shifted(int qa, int L, int words, int m, int nseg) const {
        QueryBufs o = *this;
        o.qsig += (size_t)qa * L;
        o.qbits += (size_t)qa * words;
        o.bstart += (size_t)qa * L;
        o.blen += (size_t)qa * L;
        o.isfb += qa;
        o.mcnt += qa;
        o.pos += qa;
        o.done += qa;
        o.act += qa;
        o.binlo += qa;
        o.binhi += qa;
        o.overflow += qa;
        o.wcnt += qa;
        o.keep_cnt += qa;
        o.rcnt += qa;
        o.computed += qa;
        o.U += (size_t)qa * m;
        o.Lo += (size_t)qa * m;
        o.Useg += (size_t)qa * nseg;
        o.Lseg += (size_t)qa * nseg;
        o.thr += qa;
        o.aband += qa;
        return o;
    }
};

// CUDA-event timing of a launch group into ctx->prof[slot] (profiling only)
struct Prof {
    ssh_ctx *ctx;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    bool on;
    float last = 0.f;
    Prof(ssh_ctx *c, cudaStream_t s) : ctx(c), st(s), on(c->profile != 0) {
        if (on) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
        }
    }
    void begin() {
        if (on) cudaEventRecord(a, st);
    }
    void end(int slot) {
        if (!on) return;
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        ctx->prof[slot] += ms;
        last = ms;
    }
    ~Prof() {
        if (on) {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    }
};



int next_pow2(int v) {
    int p = 32;
    while (p < v) p <<= 1;
    return p;
}

float rescore_eps(int m) { return (float)((8.0 * m + 64.0) * ldexp(1.0, -24)); }

size_t dtw32_smem(int m, int r, int warps) {
    size_t yb = (size_t)((m + 2 * r + 3) & ~3) * 4 + (size_t)2 * m * 4;
    return yb + (size_t)(2 * r + 2) * 32 * 4 * warps;
}

int dtw32_warps(int m, int r, size_t *smem) {
    int w = 4;
    while (w > 1 && dtw32_smem(m, r, w) > 200 * 1024) w--;
    *smem = dtw32_smem(m, r, w);
    return w;
}

int dtw64_threads(int r, size_t *smem) {
    size_t per = (size_t)(2 * r + 2) * 8;
    int t = 64;
    while (t > 1 && per * t > 200 * 1024) t >>= 1;
    *smem = per * t;
    return t;
}


}  // namespace

template <int R>
static int launch_dtw32r(ssh_ctx *ctx, const float *X, const float *Q, const float *U,
                         const float *Lo, const DtwList &L, const float *thr, int nq,
                         cudaStream_t st) {
    const int m = ctx->p.m;
    const int warps = 4;
    const int YP = ((m + 2 * R + 8) + 3) & ~3;
    size_t smem = (size_t)(4 * YP + 2 * m) * sizeof(float);
    SSH_CUDA(cudaFuncSetAttribute(dtw32r_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (L.wave <= 0) return SSH_OK;
    dim3 grid((unsigned)ssh_div_up(L.wave, 32 * warps), (unsigned)nq);
    dtw32r_kernel<R><<<grid, 32 * warps, smem, st>>>(X, m, Q, U, Lo, L, thr, warps,
                                                     ctx->profile ? ctx->d_cells : nullptr);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

// wave fp32 DTW: compacting register-band kernel for the common radii, the
// generic lane-per-candidate kernel otherwise
static int launch_dtw32_wave(ssh_ctx *ctx, const float *X, const float *Q, const float *U, const float *Lo,
                             const DtwWave &W, const DtwList &Lg, const DtwCommon &C, const float *thr, int nq,
                             int wave, cudaStream_t st);

// wide-band wave DTW (band-chunked warp wavefront); *done = false when r is
// outside its range (C = ceil((2r+1)/32) in [3, 32])
static int launch_dtw32w(ssh_ctx *ctx, const float *X, const float *Q, const float *U, const float *Lo,
                         const DtwList &L, const float *thr, int nq, cudaStream_t st, bool *done) {
    *done = false;
    const int m = ctx->p.m, r = ctx->p.radius;
    {
        // paired 64-virtual-lane form (dtw32v_kernel) for C2 = ceil((2r+1)/64) in [3, 8]
        // A/B only (measured slower than dtw32w at r = 205: 3.4 vs 4.4 T cells/s,
        // fewer resident warps): SSH_DTW_PAIRED_WIDE=1
        static const bool paired = getenv("SSH_DTW_PAIRED_WIDE") != nullptr;
        const int C2 = (2 * r + 1 + 63) / 64;
        if (paired && C2 >= 2 && C2 <= 8) {
            // must match dtw32v_kernel's layout: YP + 2m + DV_WARPS (G + 1), groups of C2 steps
            const int NS = m + 63, G = (NS + C2 - 1) / C2;
            const size_t smem = sizeof(float) * ((size_t)((r + m + 64 * C2 + 2 * C2 + 64 + 3) & ~3) +
                                                 2 * (size_t)m + (size_t)DV_WARPS * (G + 1));
            if (smem <= 200 * 1024) {
                *done = true;
                if (L.wave <= 0 || nq <= 0) return SSH_OK;
                dim3 grid((unsigned)ssh_div_up(L.wave, DV_WARPS * 4), (unsigned)nq);
                unsigned long long *cells = ctx->profile ? ctx->d_cells : nullptr;
#define DV_LAUNCH(CC, RR)                                                                                   \
    do {                                                                                                  \
        SSH_CUDA(cudaFuncSetAttribute(dtw32v_kernel<CC, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)smem));                                                        \
        dtw32v_kernel<CC, RR><<<grid, 32 * DV_WARPS, smem, st>>>(X, m, r, Q, U, Lo, L, thr, cells);        \
    } while (0)
                switch (r == 205 ? -1 : C2) {
                    case -1: DV_LAUNCH(7, 205); break;
                    case 2: DV_LAUNCH(2, -1); break;
                    case 3: DV_LAUNCH(3, -1); break;
                    case 4: DV_LAUNCH(4, -1); break;
                    case 5: DV_LAUNCH(5, -1); break;
                    case 6: DV_LAUNCH(6, -1); break;
                    case 7: DV_LAUNCH(7, -1); break;
                    case 8: DV_LAUNCH(8, -1); break;
                    default: break;
                }
#undef DV_LAUNCH
                SSH_CHECK_LAUNCH();
                return SSH_OK;
            }
        }
    }
    const int C = dtw_warp_chunk(r);
    if (C < 3 || C > 16) return SSH_OK;
    const int G = (m + 31 + C - 1) / C;
    const size_t smem = sizeof(float) * ((size_t)((r + m + 33 * C + 64 + 3) & ~3) + 2 * (size_t)m +
                                         (size_t)DW_WARPS * (G + 1));
    if (smem > 200 * 1024) return SSH_OK;
    *done = true;
    if (L.wave <= 0 || nq <= 0) return SSH_OK;
    // about 4 candidates per warp; the grid covers the longest list
    dim3 grid((unsigned)ssh_div_up(L.wave, DW_WARPS * 4), (unsigned)nq);
    unsigned long long *cells = ctx->profile ? ctx->d_cells : nullptr;
#define DW_LAUNCH(CC, RR)                                                                                   \
    do {                                                                                                  \
        SSH_CUDA(cudaFuncSetAttribute(dtw32w_kernel<CC, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                      (int)smem));                                                        \
        dtw32w_kernel<CC, RR><<<grid, 32 * DW_WARPS, smem, st>>>(X, m, r, Q, U, Lo, L, thr, cells);        \
    } while (0)
    if (r == 205) {
        DW_LAUNCH(13, 205);
    } else if (r == 51) {
        DW_LAUNCH(4, 51);
    } else {
#define DW_CALL(CC) DW_LAUNCH(CC, -1)
        DTW_WARP_DISPATCH16(C, DW_CALL)
#undef DW_CALL
    }
#undef DW_LAUNCH
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

// fp32 DTW of a candidate list (register band for the common radii, shared-memory band otherwise)
static int launch_dtw32(ssh_ctx *ctx, const float *X, const float *Q, const float *U,
                        const float *Lo, const DtwList &L, const float *thr, int nq,
                        cudaStream_t st) {
    const int m = ctx->p.m, r = ctx->p.radius;
    {
        static const bool no_wide = getenv("SSH_DEBUG_DTW_NO_WAVEFRONT") != nullptr;
        bool done = false;
        if (!no_wide) {
            int rc = launch_dtw32w(ctx, X, Q, U, Lo, L, thr, nq, st, &done);
            if (rc || done) return rc;
        }
    }
#define DTWR(RR) \
    case RR: return launch_dtw32r<RR>(ctx, X, Q, U, Lo, L, thr, nq, st);
    switch (r) {
        DTWR(3) DTWR(6) DTWR(13) DTWR(26) DTWR(51)
        default: break;
    }
#undef DTWR
    size_t smem;
    int warps = dtw32_warps(m, r, &smem);
    SSH_REQUIRE(smem <= 227 * 1024, SSH_ERR_UNSUPPORTED, "DTW band too wide (r=%d)", r);
    SSH_CUDA(cudaFuncSetAttribute(dtw32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (L.wave <= 0) return SSH_OK;
    dim3 grid((unsigned)ssh_div_up(L.wave, 32 * warps), (unsigned)nq);
    dtw32_kernel<<<grid, 32 * warps, smem, st>>>(X, m, r, Q, U, Lo, L, thr, warps,
                                                 ctx->profile ? ctx->d_cells : nullptr);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

template <int R>
static int launch_dtw_pooled(ssh_ctx *ctx, const DtwCommon &C, const int *act, const uint32_t *wrows,
                             const float2 *wlb, const int *wcnt, int64_t wcap, const uint4 *rec, int nact,
                             int wave, cudaStream_t st);

static int launch_dtw32_wave(ssh_ctx *ctx, const float *X, const float *Q, const float *U, const float *Lo,
                             const DtwWave &W, const DtwList &Lg, const DtwCommon &C, const float *thr, int nq,
                             int wave, cudaStream_t st) {
    const int m = ctx->p.m, r = ctx->p.radius;
    static const bool legacy = getenv("SSH_DEBUG_DTW_LEGACY") != nullptr;
#define DTWP(RR) \
    case RR:     \
        return launch_dtw_pooled<RR>(ctx, C, W.act, W.rows, W.lbs, W.cnt, W.stride, W.rec, nq, wave, st);
    // SSH_DEBUG_DTW_WAVEFRONT: the warp wavefront also for the pooled radii (A/B)
    static const bool wavefront = getenv("SSH_DEBUG_DTW_WAVEFRONT") != nullptr;
    // SSH_DTW_POOLED_MAXR: largest radius served by the pooled kernels (A/B)
    static const int pooled_maxr = getenv("SSH_DTW_POOLED_MAXR") ? atoi(getenv("SSH_DTW_POOLED_MAXR")) : 51;
    if (!legacy && !wavefront && (m & 3) == 0 && C.qpad && r <= pooled_maxr) switch (r) {
        DTWP(3) DTWP(6) DTWP(13) DTWP(26) DTWP(51)
        default: break;
    }
#undef DTWP
    return launch_dtw32(ctx, X, Q, U, Lo, Lg, thr, nq, st);
}


// pooled wave DTW (register band, radius R): first pass per slot, then
// pooled passes over the survivors of all queries
template <int R>
static int launch_dtw_pooled(ssh_ctx *ctx, const DtwCommon &C, const int *act, const uint32_t *wrows,
                             const float2 *wlb, const int *wcnt, int64_t wcap, const uint4 *rec, int nact,
                             int wave, cudaStream_t st) {
    constexpr int NB = 2 * R + 1;
    if (wave <= 0 || nact <= 0) return SSH_OK;
    const int64_t cap = (int64_t)nact * wave;
    const size_t per = 4 + 4 + 8 + 6 * 4 + NB * 4;
    DtwPool pool[2];
    for (int i = 0; i < 2; i++) {
        unsigned char *base = (unsigned char *)ssh_slot(ctx, i ? SLOT_Q_POOLB : SLOT_Q_POOLA, per * (size_t)cap + 64, st);
        if (!base) return SSH_ERR_OOM;
        pool[i].out = reinterpret_cast<int64_t *>(base);
        pool[i].q = reinterpret_cast<int *>(pool[i].out + cap);
        pool[i].row = reinterpret_cast<uint32_t *>(pool[i].q + cap);
        pool[i].st = reinterpret_cast<float *>(pool[i].row + cap);
        pool[i].band = pool[i].st + 6 * cap;
        pool[i].cap = cap;
    }
    int *cnt = (int *)ssh_slot(ctx, SLOT_Q_POOLCNT, 64 * sizeof(int), st);
    if (!cnt) return SSH_ERR_OOM;
    const int m = C.m;
    // pass ends 8, 16, 32, 64, then every DP_MAXPASS rows (or doubling)
    auto next_end = [&](int a) {
        return std::min(m, (a < DP_MAXPASS || SSH_DTW_PASS_DOUBLING) ? 2 * a : a + DP_MAXPASS);
    };
    static const int b0_env = getenv("SSH_DTW_B0") ? atoi(getenv("SSH_DTW_B0")) : SSH_DTW_B0;
    const int b0 = std::min(m, b0_env);
    int nlev = 1;
    for (int a = b0; a < m; a = next_end(a)) nlev++;
    SSH_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * nlev, st));
    pool[0].count = cnt;
    dim3 g1((unsigned)ssh_div_up(wave, 32 * DP_WARPS), (unsigned)nact);
    dtwp_first_kernel<R><<<g1, 32 * DP_WARPS, 0, st>>>(C, act, wrows, wlb, wcnt, wcap, rec, b0, pool[0]);
    SSH_CHECK_LAUNCH();
    // the wavefront tail (per-warp staged query + band) once fewer than lim are left
    const size_t tail_smem = sizeof(float) * (size_t)DT_WARPS * (C.YP + 2 * 64 + 4);
    const int lim = tail_smem <= 160 * 1024 ? SSH_DTW_TAIL : 0;
    const size_t lsmem = lim ? tail_smem : 0;
    static size_t attr_smem = 0;
    static int per_sm = 0;
    static size_t per_sm_smem = ~(size_t)0;
    if (lsmem > attr_smem) {
        SSH_CUDA(cudaFuncSetAttribute(dtwp_level_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem));
        attr_smem = lsmem;
    }
    if (per_sm_smem != lsmem) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dtwp_level_kernel<R>, 32 * DP_WARPS, lsmem);
        per_sm = std::max(1, per_sm);
        per_sm_smem = lsmem;
    }
    static const bool dbg = getenv("SSH_DEBUG_DTW_PASSES") != nullptr;
    cudaEvent_t ev[66];
    if (dbg) {
        for (int i = 0; i <= nlev; i++) cudaEventCreate(&ev[i]);
        cudaEventRecord(ev[0], st);
    }
    int lev = 1;
    for (int a = b0; a < m; lev++) {
        const int b = next_end(a);
        DtwPool in = pool[(lev - 1) & 1], out = pool[lev & 1];
        in.count = cnt + lev - 1;
        out.count = cnt + lev;
        if (dbg) cudaEventRecord(ev[lev], st);
        dtwp_level_kernel<R><<<ctx->num_sms * per_sm, 32 * DP_WARPS, lsmem, st>>>(C, in, out, a, b, lim);
        SSH_CHECK_LAUNCH();
        a = b;
    }
    if (dbg) {
        cudaEventRecord(ev[lev], st);
        cudaEventSynchronize(ev[lev]);
        std::vector<int> hc(nlev);
        cudaMemcpy(hc.data(), cnt, sizeof(int) * nlev, cudaMemcpyDeviceToHost);
        fprintf(stderr, "dtw pooled: nact %d wave %d |", nact, wave);
        for (int i = 1; i < lev; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            fprintf(stderr, " [%d items %.3f ms]", hc[i - 1], ms);
        }
        float f0 = 0.f;
        cudaEventElapsedTime(&f0, ev[0], ev[1]);
        fprintf(stderr, " first %.3f ms\n", f0);
        for (int i = 0; i <= nlev; i++) cudaEventDestroy(ev[i]);
    }
    return SSH_OK;
}

template <int R>
static int launch_dtw64r(const float *X, int m, const float *Q, const uint32_t *list, int64_t stride,
                         const int *cnt, int maxcnt, double *out, int nq, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)(m + 2 * R + 8);
    SSH_CUDA(cudaFuncSetAttribute(dtw64r_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)ssh_div_up(maxcnt, 128), (unsigned)nq);
    dtw64r_kernel<R><<<grid, 128, smem, st>>>(X, m, Q, list, stride, cnt, out);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

static int launch_dtw64_list(const float *X, int m, int r, const float *Q, const uint32_t *list,
                             int64_t stride, const int *cnt, int maxcnt, double *out, int nq,
                             cudaStream_t st) {
    if (maxcnt <= 0) return SSH_OK;
    const size_t smem = sizeof(double) * (size_t)(m + 2 * r + 2) * D64W_WARPS;
    if (2 * r + 1 <= 64 && smem <= 200 * 1024) {  // wavefront period 64 >= band width
        SSH_CUDA(cudaFuncSetAttribute(dtw64w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid((unsigned)ssh_div_up(maxcnt, D64W_WARPS), (unsigned)nq);
        dtw64w_kernel<<<grid, 32 * D64W_WARPS, smem, st>>>(X, m, r, Q, nullptr, list, stride, cnt, nullptr, 0, out);
        SSH_CHECK_LAUNCH();
        return SSH_OK;
    }
    {
        bool done = false;
        int rc = launch_dtw64band(X, m, r, Q, nullptr, list, stride, cnt, nullptr, maxcnt, nq, out, st, &done);
        if (rc || done) return rc;
    }
    size_t smem2;
    int t = dtw64_threads(r, &smem2);
    SSH_CUDA(cudaFuncSetAttribute(dtw64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    dim3 grid((unsigned)ssh_div_up(maxcnt, t), (unsigned)nq);
    dtw64_kernel<<<grid, t, smem2, st>>>(X, m, r, Q, nullptr, list, stride, cnt, nullptr, 0, out);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

extern "C" int ssh_dtw_exact(ssh_ctx *ctx, const float *X, const float *Q, const int32_t *qrow,
                             const int64_t *xrow, int64_t npair, double *d2, void *stream) {
    SSH_REQUIRE(ctx && ctx->have_params, SSH_ERR_STATE, "ssh_dtw_exact: params not set");
    if (npair == 0) return SSH_OK;
    SSH_REQUIRE(X && Q && qrow && xrow && d2, SSH_ERR_INVALID, "ssh_dtw_exact: NULL pointer");
    SSH_CUDA(cudaSetDevice(ctx->device));
    int m = ctx->p.m, r = ctx->p.radius;
    const size_t smem = sizeof(double) * (size_t)(m + 2 * r + 2) * D64W_WARPS;
    if (2 * r + 1 <= 64 && smem <= 200 * 1024) {  // wavefront period 64 >= band width
        SSH_CUDA(cudaFuncSetAttribute(dtw64w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dtw64w_kernel<<<(unsigned)ssh_div_up(npair, D64W_WARPS), 32 * D64W_WARPS, smem, (cudaStream_t)stream>>>(
            X, m, r, Q, qrow, nullptr, 0, nullptr, xrow, npair, d2);
        SSH_CHECK_LAUNCH();
        return SSH_OK;
    }
    {
        bool done = false;
        int rc = launch_dtw64band(X, m, r, Q, qrow, nullptr, 0, nullptr, xrow, npair, 1, d2,
                                  (cudaStream_t)stream, &done);
        if (rc || done) return rc;
    }
    size_t smem2;
    int t = dtw64_threads(r, &smem2);
    SSH_CUDA(cudaFuncSetAttribute(dtw64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    dtw64_kernel<<<(unsigned)ssh_div_up(npair, t), t, smem2, (cudaStream_t)stream>>>(
        X, m, r, Q, qrow, nullptr, 0, nullptr, xrow, npair, d2);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

static int qsig_batch(ssh_ctx *ctx, const float *Q, int nq, uint64_t *qsig, uint64_t *qbits,
                      cudaStream_t st) {
    int rc = ssh_launch_sketch(ctx, Q, nq, ctx->p.m, qbits, nullptr, st);
    if (rc) return rc;
    return ssh_launch_shingle_cws(ctx, qbits, nullptr, nullptr, nullptr, nq, nullptr, nullptr,
                                  nullptr, nullptr, qsig, SIG_MODE_FUSED, st);
}

static int probe_and_bitmap(const ssh_index *ix, const uint64_t *qsig, int nq, int fallback,
                            uint64_t *bstart, uint32_t *blen, uint32_t *bitmap, long long *n_cand,
                            int *is_fb, cudaStream_t st, bool exact = false) {
    const int L = ix->L;
    const int64_t N = ix->N, NW = (N + 31) / 32;
    if (exact || !ix->keys) {
        // exact search: no probe; every query's R is the whole shard (count_kernel fills it)
        SSH_CUDA(cudaMemsetAsync(blen, 0, sizeof(uint32_t) * (size_t)nq * L, st));
        SSH_CUDA(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (size_t)nq * NW, st));
        count_kernel<<<nq, 256, 0, st>>>(bitmap, NW, N, blen, L, 1, n_cand, is_fb);
        SSH_CHECK_LAUNCH();
        return SSH_OK;
    }
    probe_kernel<<<ssh_div_up((int64_t)nq * L, 128), 128, 0, st>>>(
        qsig, nq, L, ix->keys, ix->offsets, ix->d_nb, ix->d_kbase, N, bstart, blen);
    SSH_CHECK_LAUNCH();
    if (L <= 64) {
        const int sw = (int)std::min<int64_t>(NW, BM_SLICE_WORDS);
        SSH_CUDA(cudaFuncSetAttribute(bitmap_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(uint32_t) * sw)));
        dim3 g((unsigned)ssh_div_up(NW, BM_SLICE_WORDS), (unsigned)nq);
        bitmap_smem_kernel<<<g, 1024, sizeof(uint32_t) * sw, st>>>(ix->ids, bstart, blen, L, N, NW, bitmap);
    } else {
        SSH_CUDA(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (size_t)nq * NW, st));
        dim3 g((unsigned)(nq * L), 8);
        bitmap_kernel<<<g, 256, 0, st>>>(ix->ids, bstart, blen, L, NW, bitmap);
    }
    SSH_CHECK_LAUNCH();
    count_kernel<<<nq, 256, 0, st>>>(bitmap, NW, N, blen, L, fallback, n_cand, is_fb);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

extern "C" int ssh_probe(ssh_ctx *ctx, const ssh_index *ix, const uint64_t *qsig, int32_t nq,
                         uint32_t *bitmap, int64_t *n_cand, void *stream) {
    SSH_REQUIRE(ctx && ix && qsig && bitmap && n_cand, SSH_ERR_INVALID, "ssh_probe: NULL argument");
    SSH_REQUIRE(ix->keys != nullptr, SSH_ERR_STATE, "ssh_probe: index has no bucket tables");
    SSH_REQUIRE(nq >= 0 && ix->L == ctx->p.L, SSH_ERR_INVALID, "ssh_probe: bad arguments");
    if (nq == 0) return SSH_OK;
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    Arena A;
    A.st = st;
    uint64_t *bstart = A.get<uint64_t>((size_t)nq * ix->L);
    uint32_t *blen = A.get<uint32_t>((size_t)nq * ix->L);
    int *isfb = A.get<int>(nq);
    if (A.err) return ssh_cuda_fail(A.err, "ssh_probe scratch", __FILE__, __LINE__);
    int rc = probe_and_bitmap(ix, qsig, nq, 0, bstart, blen, bitmap, (long long *)n_cand, isfb, st);
    if (rc == SSH_OK) ssh_index_touch(ix, st);
    return rc;
}

// fold the last chunk's rerank span [qev[2], qev[3]] into ctx->qphase[2]
static int fold_rerank(ssh_ctx *ctx) {
    if (!ctx->qpending) return SSH_OK;
    SSH_CUDA(cudaEventSynchronize(ctx->qev[3]));
    float ms = 0.f;
    SSH_CUDA(cudaEventElapsedTime(&ms, ctx->qev[2], ctx->qev[3]));
    ctx->qphase[2] += ms;
    ctx->qpending = false;
    return SSH_OK;
}

extern "C" int ssh_query_phase_ms(ssh_ctx *ctx, double *out3) {
    SSH_REQUIRE(ctx && out3, SSH_ERR_INVALID, "ssh_query_phase_ms: NULL argument");
    SSH_CUDA(cudaSetDevice(ctx->device));
    int rc = fold_rerank(ctx);
    if (rc) return rc;
    for (int i = 0; i < 3; i++) out3[i] = ctx->qphase[i];
    return SSH_OK;
}

static int max_of(const int *d, int n, cudaStream_t st, int *out) {
    std::vector<int> h(n);
    SSH_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    SSH_CUDA(cudaStreamSynchronize(st));
    *out = n ? *std::max_element(h.begin(), h.end()) : 0;
    return SSH_OK;
}

extern "C" int ssh_query_batch(ssh_ctx *ctx, const ssh_index *ix, const float *X, const float *Q,
                               int32_t nq, int32_t k, int32_t flags, int64_t *out_ids,
                               double *out_d2, int32_t *n_out, int64_t *n_cand,
                               int64_t *counters, int32_t *status, void *stream) {
    SSH_REQUIRE(ctx && ix, SSH_ERR_INVALID, "ssh_query_batch: NULL ctx/index");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_query_batch: params not set");
    SSH_REQUIRE(ix->L == ctx->p.L, SSH_ERR_INVALID, "ssh_query_batch: index/ctx table count mismatch");
    SSH_REQUIRE(k >= 1, SSH_ERR_INVALID, "k must be >= 1, got %d", k);
    SSH_REQUIRE(k <= SSH_MAX_K, SSH_ERR_UNSUPPORTED, "k=%d exceeds the device limit %d", k, SSH_MAX_K);
    SSH_REQUIRE(nq >= 0, SSH_ERR_INVALID, "nq must be >= 0");
    if (nq == 0) return SSH_OK;
    SSH_REQUIRE(X && Q && out_ids && out_d2 && n_out && n_cand && counters && status, SSH_ERR_INVALID,
                "ssh_query_batch: NULL pointer");
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    for (int i = 0; i < 4; i++)
        if (!ctx->qev[i]) SSH_CUDA(cudaEventCreate(&ctx->qev[i]));
    ctx->qpending = false;
    ctx->qphase[0] = ctx->qphase[1] = ctx->qphase[2] = 0.0;
    ssh_index *mix = const_cast<ssh_index *>(ix);
    if (!mix->rec) {
        int rc = ssh_index_summarize(ctx, mix, X, ctx->p.m, stream);
        if (rc) return rc;
    }
    const int m = ctx->p.m, r = ctx->p.radius, L = ix->L, nseg = ix->nseg;
    const int64_t N = ix->N, NW = (N + 31) / 32;
    const float eps = rescore_eps(m);
#ifndef SSH_W0
#define SSH_W0 64
#endif
    const int W0 = ((std::max(SSH_W0, 2 * k) + 31) / 32) * 32;
    const int WCAP = std::max(W0, 16384);
    int KCAP = 4096 + 4 * k;  // per-query rescoring-list capacity; grows (and the slice reruns) when ties overflow it
    const int fallback = (flags & SSH_QUERY_FALLBACK_ON_EMPTY) ? 1 : 0;
    const bool exact = (flags & SSH_QUERY_EXACT) != 0 || !ix->keys;
    // query chunk: membership bitmaps <= 1 GiB; within a chunk, sub-ranges of
    // queries whose actual member lists (16 B per member) fit SSH_MEMBER_BUDGET
    int64_t qc64 = std::min<int64_t>(nq, 32768);
    qc64 = std::min<int64_t>(qc64, ((int64_t)1 << 28) / std::max<int64_t>(1, NW));
    const int qc = (int)std::max<int64_t>(1, qc64);
    SSH_CUDA(cudaMemsetAsync(counters, 0, sizeof(int64_t) * 5 * (size_t)nq, st));
    SSH_CUDA(cudaFuncSetAttribute(wave_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(uint32_t) * SSH_MAX_K)));
    SSH_CUDA(cudaFuncSetAttribute(paa_members_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(MB_WARPS * MB_WARP_BYTES)));
    SSH_CUDA(cudaFuncSetAttribute(paa_members_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(MB_WARPS * MB_WARP_BYTES + NBINS * 4)));
    for (int q0 = 0; q0 < nq; q0 += qc) {
        const int nc = std::min(qc, nq - q0);
        const float *Qc = Q + (int64_t)q0 * m;
        long long *ncand = (long long *)n_cand + q0;
        long long *cnt5 = (long long *)counters + (int64_t)q0 * 5;
        Carver sizer;
        QueryBufs B;
        B.carve(sizer, nc, L, ctx->words, m, nseg);
        Carver cv;
        cv.base = (unsigned char *)ssh_slot(ctx, SLOT_Q_FIXED, sizer.off, st);
        if (!cv.base) return SSH_ERR_OOM;
        B.carve(cv, nc, L, ctx->words, m, nseg);
        uint32_t *bitmap = (uint32_t *)ssh_slot(ctx, SLOT_Q_BITMAP, sizeof(uint32_t) * (size_t)nc * NW, st);
        if (!bitmap) return SSH_ERR_OOM;
        Prof pf(ctx, st);
        // K5: query signatures
        pf.begin();
        int rc = fold_rerank(ctx);  // previous chunk (its events are re-recorded below)
        if (rc) return rc;
        SSH_CUDA(cudaEventRecord(ctx->qev[0], st));
        rc = qsig_batch(ctx, Qc, nc, B.qsig, B.qbits, st);
        if (rc) return rc;
        SSH_CUDA(cudaEventRecord(ctx->qev[1], st));
        pf.end(0);
        // K6: probe + candidate bitmap; member counts -> CSR offsets
        pf.begin();
        rc = probe_and_bitmap(ix, B.qsig, nc, fallback, B.bstart, B.blen, bitmap, ncand, B.isfb, st, exact);
        if (rc) return rc;
        envelope_kernel<<<nc, 256, 2 * m * sizeof(float), st>>>(Qc, m, r, ix->seg, nseg, B.U, B.Lo, B.Useg, B.Lseg);
        SSH_CHECK_LAUNCH();
        // padded query copies for the pooled wave DTW
        const int qYP = ((m + 2 * r + 8) + 3) & ~3;
        float *qpad = (float *)ssh_slot(ctx, SLOT_Q_QPAD, sizeof(float) * (size_t)nc * qYP, st);
        if (!qpad) return SSH_ERR_OOM;
        qpad_kernel<<<nc, 256, 0, st>>>(Qc, m, r, qYP, qpad);
        SSH_CHECK_LAUNCH();
        SSH_CUDA(cudaEventRecord(ctx->qev[2], st));
        std::vector<long long> hc(nc);
        SSH_CUDA(cudaMemcpyAsync(hc.data(), ncand, sizeof(long long) * nc, cudaMemcpyDeviceToHost, st));
        SSH_CUDA(cudaStreamSynchronize(st));
        {
            float a = 0.f, b = 0.f;
            SSH_CUDA(cudaEventElapsedTime(&a, ctx->qev[0], ctx->qev[1]));
            SSH_CUDA(cudaEventElapsedTime(&b, ctx->qev[1], ctx->qev[2]));
            ctx->qphase[0] += a;
            ctx->qphase[1] += b;
        }
        pf.end(1);
        // sub-ranges of the chunk whose actual member lists fit the budget
        // (SSH_DEBUG_MEMBER_BUDGET overrides it, for tests of the split path)
        int64_t budget = SSH_MEMBER_BUDGET;
        if (const char *ev = getenv("SSH_DEBUG_MEMBER_BUDGET")) budget = std::max<int64_t>(1, atoll(ev));
        // (SSH_DEBUG_MEMBER_TARGET lowers the round-0 cutoff, for tests of the overflow round)
        int member_target = SSH_MEMBER_TARGET;
        if (const char *ev = getenv("SSH_DEBUG_MEMBER_TARGET")) member_target = std::max(8, atoi(ev));
        for (int sa = 0; sa < nc;) {
            int sb = sa;
            int64_t total = 0;
            while (sb < nc && (sb == sa || total + hc[sb] <= budget)) total += hc[sb++];
            const int ns = sb - sa;
            int64_t maxcand = 0;
            for (int q = sa; q < sb; q++) maxcand = std::max<int64_t>(maxcand, hc[q]);
            QueryBufs S = B.shifted(sa, L, ctx->words, m, nseg);
            const float *Qs = Qc + (int64_t)sa * m;
            uint32_t *bms = bitmap + (int64_t)sa * NW;
            long long *ncs = ncand + sa;
            long long *c5s = cnt5 + (int64_t)sa * 5;
            const int qs0 = q0 + sa;
            {
                std::vector<int64_t> hoff(ns + 1);
                hoff[0] = 0;
                for (int q = 0; q < ns; q++) hoff[q + 1] = hoff[q] + hc[sa + q];
                SSH_CUDA(cudaMemcpyAsync(S.roff, hoff.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice, st));
            }
            // K7 lists: members with their summary key, sorted by key bin.  Round 0
            // keeps the bins up to a per-query cutoff chosen from a 1/8 sample of
            // the keys (about SSH_MEMBER_TARGET members); a query whose list runs
            // out while its threshold is still above the cutoff takes an overflow
            // round over the remaining bins, continuing the same top-k state.
            pf.begin();
            uint32_t *rows_u = (uint32_t *)ssh_slot(ctx, SLOT_Q_SURV, sizeof(uint32_t) * (size_t)std::max<int64_t>(total, 1), st);
            float *lb_u = (float *)ssh_slot(ctx, SLOT_Q_SURV_LB, sizeof(float) * (size_t)std::max<int64_t>(total, 1), st);
            uint32_t *rows_s = (uint32_t *)ssh_slot(ctx, SLOT_Q_W2, sizeof(uint32_t) * (size_t)std::max<int64_t>(total, 1), st);
            float *lb_s = (float *)ssh_slot(ctx, SLOT_Q_D2, sizeof(float) * (size_t)std::max<int64_t>(total, 1), st);
            unsigned *khist = (unsigned *)ssh_slot(ctx, SLOT_Q_KHIST, sizeof(unsigned) * (size_t)ns * NBINS, st);
            if (!rows_u || !lb_u || !rows_s || !lb_s || !khist) return SSH_ERR_OOM;
            const dim3 gm((unsigned)ssh_div_up(NW, MB_SLICE_WORDS), (unsigned)ns);
            PaaArgs pa{S.Useg, S.Lseg, Qs, (const uint4 *)ix->rec, bms, S.roff, rows_u, lb_u, S.mcnt,
                       S.binlo, S.binhi, khist, NW, m, ix->seg, nseg};
            {
                SSH_CUDA(cudaMemsetAsync(khist, 0, sizeof(unsigned) * (size_t)ns * NBINS, st));
                const dim3 gs((unsigned)ssh_div_up(NW, (int64_t)MB_SLICE_WORDS << SAMPLE_SHIFT), (unsigned)ns);
                paa_members_kernel<true><<<gs, MB_THREADS, MB_WARPS * MB_WARP_BYTES + NBINS * 4, st>>>(pa);
                SSH_CHECK_LAUNCH();
                cutoff_kernel<<<ns, 256, 0, st>>>(khist, member_target, S.binlo, S.binhi);
                SSH_CHECK_LAUNCH();
            }
            pf.end(2);
            uint32_t *wrows = (uint32_t *)ssh_slot(ctx, SLOT_Q_RESC, sizeof(uint32_t) * (size_t)ns * WCAP, st);
            float *wd32 = (float *)ssh_slot(ctx, SLOT_Q_D32, sizeof(float) * (size_t)ns * WCAP, st);
            float2 *wlb = (float2 *)ssh_slot(ctx, SLOT_Q_WLB, sizeof(float2) * (size_t)ns * WCAP, st);
            float *topk = (float *)ssh_slot(ctx, SLOT_Q_TOPK, sizeof(float) * (size_t)ns * k, st);
            uint32_t *keep_rows = (uint32_t *)ssh_slot(ctx, SLOT_Q_KEEP, sizeof(uint32_t) * (size_t)ns * KCAP, st);
            float *keep_d32 = (float *)ssh_slot(ctx, SLOT_Q_KEEP_D, sizeof(float) * (size_t)ns * KCAP, st);
            uint32_t *resc = (uint32_t *)ssh_slot(ctx, SLOT_Q_HIST, sizeof(uint32_t) * (size_t)ns * KCAP, st);
            double *d64 = (double *)ssh_slot(ctx, SLOT_Q_D64, sizeof(double) * (size_t)ns * KCAP, st);
            if (!wrows || !wd32 || !wlb || !topk || !keep_rows || !keep_d32 || !resc || !d64) return SSH_ERR_OOM;
            std::vector<float> thr0h;
            const int64_t pool = (int64_t)ns * WCAP;
            const int wl_warps = 8;
            const size_t wl_smem = (size_t)4 * ix->mp * sizeof(float);
            SSH_CUDA(cudaFuncSetAttribute(wave_lb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wl_smem));
            for (int round = 0; round < 2; round++) {
                pf.begin();
                if (round == 1) {
                    overflow_window_kernel<<<ssh_div_up(ns, 256), 256, 0, st>>>(S.overflow, ns, S.binlo, S.binhi);
                    SSH_CHECK_LAUNCH();
                }
                SSH_CUDA(cudaMemsetAsync(S.mcnt, 0, sizeof(int) * ns, st));
                paa_members_kernel<false><<<gm, MB_THREADS, MB_WARPS * MB_WARP_BYTES, st>>>(pa);
                SSH_CHECK_LAUNCH();
                if (round == 0) {
                    binsort_kernel<<<ns, 1024, 0, st>>>(rows_u, lb_u, S.roff, S.mcnt, rows_s, lb_s);
                } else {
                    // overflow lists are long: chunked multi-block sort
                    const int nch = (int)std::max<int64_t>(1, (maxcand + BS_CHUNK - 1) / BS_CHUNK);
                    uint32_t *bsh = (uint32_t *)ssh_slot(ctx, SLOT_Q_BSHIST, sizeof(uint32_t) * (size_t)ns * NBINS * nch, st);
                    if (!bsh) return SSH_ERR_OOM;
                    dim3 gb((unsigned)nch, (unsigned)ns);
                    bs_hist_kernel<<<gb, 1024, 0, st>>>(lb_u, S.roff, S.mcnt, nch, bsh);
                    SSH_CHECK_LAUNCH();
                    bs_scan_kernel<<<ns, 1024, 0, st>>>(bsh, nch);
                    SSH_CHECK_LAUNCH();
                    bs_scatter_kernel<<<gb, 1024, 0, st>>>(rows_u, lb_u, S.roff, S.mcnt, nch, bsh, rows_s, lb_s);
                }
                SSH_CHECK_LAUNCH();
                pf.end(2);
                // K7/K8: waves in key order: LB_Keogh2/LB_Keogh -> fp32 DTW -> threshold
                wave_init_kernel<<<ssh_div_up(std::max<int64_t>((int64_t)ns * k, ns), 256), 256, 0, st>>>(
                    ns, k, round, S.mcnt, S.overflow, S.thr, topk, S.pos, S.done, S.wcnt, S.keep_cnt, S.computed,
                    S.aband);
                SSH_CHECK_LAUNCH();
                // waves over the active queries only: block row y = slot y = query
                // act[y]; the per-wave lists share one pool, so the per-slot
                // capacity grows as queries finish
                compact_active_kernel<<<1, 1024, 0, st>>>(S.done, ns, S.act, S.nact);
                SSH_CHECK_LAUNCH();
                int nact = 0;
                SSH_CUDA(cudaMemcpyAsync(&nact, S.nact, sizeof(int), cudaMemcpyDeviceToHost, st));
                SSH_CUDA(cudaStreamSynchronize(st));
                if (nact == 0) break;
                WaveLbArgs wl{Qs, S.U, S.Lo, (const uint4 *)ix->rec, ix->codes, ix->cstride, rows_s, lb_s, S.roff,
                              S.mcnt, S.pos, S.done, S.thr, S.act, wrows, wlb, S.wcnt, c5s,
                              ctx->profile ? ctx->d_cells : nullptr, m, ix->mp, W0, WCAP};
                for (int wave = W0, it = 0; nact > 0; wave *= SSH_WAVE_GROWTH, it++) {
                    const int wcap = (int)std::min<int64_t>((int64_t)1 << 20, (pool / nact) & ~(int64_t)255);
                    wave = std::min(wave, wcap);
                    pf.begin();
                    {
                        dim3 g((unsigned)std::min(ssh_div_up(wave, 32 * wl_warps), 512), (unsigned)nact);
                        wl.wave = wave;
                        wl.wcap = wcap;
                        wave_lb_kernel<<<g, 32 * wl_warps, wl_smem, st>>>(wl);
                        SSH_CHECK_LAUNCH();
                    }
                    pf.end(3);
                    const float lb_ms = pf.last;
                    pf.begin();
                    {
                        DtwList dl{wrows, wcap, S.wcnt, nullptr, wave, nullptr, wd32, S.aband, S.computed, S.act};
                        DtwWave dw{wrows, wlb, wcap, S.wcnt, wd32, S.aband, S.computed, (const uint4 *)ix->rec,
                                   ix->codes, ix->cstride, ix->mp, S.act};
                        DtwCommon dc{X, qpad ? qpad + (int64_t)sa * qYP : nullptr, S.U, S.Lo, S.thr, ix->codes,
                                     ix->cstride, m, ix->mp, qYP, wd32, S.aband, S.computed,
                                     ctx->profile ? ctx->d_cells : nullptr};
                        rc = launch_dtw32_wave(ctx, X, Qs, S.U, S.Lo, dw, dl, dc, S.thr, nact, wave, st);
                        if (rc) return rc;
                    }
                    pf.end(4);
                    if (ctx->profile && getenv("SSH_DEBUG_WAVES"))
                        fprintf(stderr, "round %d wave %d: active %d wave %d cap %d | LB %.3f ms DTW %.3f ms\n", round,
                                it, nact, wave, wcap, lb_ms, pf.last);
                    wave_update_kernel<<<nact, 256, sizeof(uint32_t) * (size_t)k, st>>>(S.act, wd32, wrows, S.wcnt, wcap, lb_s, S.roff, S.mcnt,
                                                             S.binhi, wave, k, eps, topk, S.thr, S.pos, S.done,
                                                             S.overflow, keep_rows, keep_d32, S.keep_cnt, KCAP);
                    SSH_CHECK_LAUNCH();
                    compact_active_kernel<<<1, 1024, 0, st>>>(S.done, ns, S.act, S.nact);
                    SSH_CHECK_LAUNCH();
                    if (ctx->profile && it == 0 && round == 0) {
                        thr0h.resize(ns);
                        cudaMemcpyAsync(thr0h.data(), S.thr, sizeof(float) * ns, cudaMemcpyDeviceToHost, st);
                    }
                    SSH_CUDA(cudaMemcpyAsync(&nact, S.nact, sizeof(int), cudaMemcpyDeviceToHost, st));
                    SSH_CUDA(cudaStreamSynchronize(st));
                    if (ctx->profile) {
                        ctx->prof[16] += 1;
                        ctx->prof[17] += nact;
                    }
                }
                if (round == 0) {
                    int nover = 0;
                    rc = max_of(S.overflow, ns, st, &nover);
                    if (rc) return rc;
                    if (ctx->profile) ctx->prof[18] += 1;
                    if (!nover) break;
                    if (ctx->profile) ctx->prof[19] += 1;
                }
            }
            int maxkeep = 0;
            rc = max_of(S.keep_cnt, ns, st, &maxkeep);
            if (rc) return rc;
            if (maxkeep > KCAP) {
                // massively tied distances (e.g. thousands of duplicate series): more
                // candidates within the rescoring margin than the keep lists hold.  The
                // reference cascade always answers (dtw.py:171-236), so the slice is
                // searched again with lists that hold every such candidate
                // (keep_cnt counted all of them, an upper bound of the rerun's need).
                SSH_REQUIRE((int64_t)maxkeep <= N + 1, SSH_ERR_STATE,
                            "ssh_query_batch: keep count %d exceeds the shard size", maxkeep);
                KCAP = (maxkeep + 1023) & ~1023;
                SSH_CUDA(cudaMemsetAsync(c5s, 0, sizeof(long long) * 5 * (size_t)ns, st));
                if (ctx->profile) ctx->prof[21] += 1;  // reruns with larger rescoring lists
                continue;  // sa unchanged: same slice, larger lists
            }
            // K9/K10: rescoring set, exact f64 DTW, top-k by (d64, id)
            pf.begin();
            select_kernel<<<ns, 256, 0, st>>>(keep_rows, keep_d32, S.keep_cnt, KCAP, k, eps, resc, S.rcnt, c5s,
                                              S.mcnt, S.pos);
            SSH_CHECK_LAUNCH();
            int maxr = 0;
            rc = max_of(S.rcnt, ns, st, &maxr);
            if (rc) return rc;
            rc = launch_dtw64_list(X, m, r, Qs, resc, KCAP, S.rcnt, maxr, d64, ns, st);
            if (rc) return rc;
            const int P2k = next_pow2(k);
            size_t stk = (size_t)P2k * (sizeof(double) + sizeof(uint32_t));
            SSH_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stk));
            topk_kernel<<<ns, 256, stk, st>>>(resc, d64, S.rcnt, KCAP, P2k, k, ix->id_base, ncs,
                                              (long long *)out_ids + (int64_t)qs0 * k,
                                              out_d2 + (int64_t)qs0 * k, n_out + qs0);
            SSH_CHECK_LAUNCH();
            finalize_counters<<<ssh_div_up(ns, 128), 128, 0, st>>>(S.computed, S.aband, ns, ncs, S.isfb, c5s,
                                                                   status + qs0);
            SSH_CHECK_LAUNCH();
            pf.end(5);
            if (ctx->profile) {
                std::vector<int> h(ns);
                cudaMemcpy(h.data(), S.computed, sizeof(int) * ns, cudaMemcpyDeviceToHost);
                for (int v : h) ctx->prof[8] += v;
                cudaMemcpy(h.data(), S.rcnt, sizeof(int) * ns, cudaMemcpyDeviceToHost);
                for (int v : h) ctx->prof[9] += v;
                std::vector<float> thr1h(ns);
                std::vector<double> dk((size_t)ns * k);
                cudaMemcpy(thr1h.data(), S.thr, sizeof(float) * ns, cudaMemcpyDeviceToHost);
                cudaMemcpy(dk.data(), out_d2 + (int64_t)qs0 * k, sizeof(double) * ns * k, cudaMemcpyDeviceToHost);
                for (int q = 0; q < ns; q++) {
                    double d = dk[(size_t)q * k + k - 1];
                    if (d > 0 && std::isfinite(d) && !thr0h.empty() && std::isfinite(thr0h[q])) {
                        ctx->prof[13] += thr0h[q] / d;
                        ctx->prof[14] += thr1h[q] / d;
                        ctx->prof[15] += 1;
                    }
                }
            }
            sa = sb;
        }
        SSH_CUDA(cudaEventRecord(ctx->qev[3], st));
        ctx->qpending = true;
    }
    ssh_index_touch(ix, st);
    return SSH_OK;
}
