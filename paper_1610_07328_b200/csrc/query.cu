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

#include <algorithm>
#include <vector>

#include "common.cuh"

#define Q_SURV_CAP0 4096
#define Q_SEED_CAND 4096
#define MB_THREADS 256
#define MB_WARPS (MB_THREADS / 32)
#define MB_SLICE_WORDS 256
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
// per-segment max/min for the PAA bound
__global__ void envelope_kernel(const float *__restrict__ Q, int m, int r, int nseg,
                                float *__restrict__ U, float *__restrict__ Lo,
                                float *__restrict__ Useg, float *__restrict__ Lseg) {
    extern __shared__ float esm[];
    float *su = esm, *sl = esm + m;
    const int q = blockIdx.x;
    const float *y = Q + (int64_t)q * m;
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
        U[(int64_t)q * m + i] = mx;
        Lo[(int64_t)q * m + i] = mn;
    }
    __syncthreads();
    for (int s = threadIdx.x; s < nseg; s += blockDim.x) {
        int a = s * SSH_PAA_SEG, b = min(m, a + SSH_PAA_SEG);
        float mx = su[a], mn = sl[a];
        for (int i = a + 1; i < b; i++) {
            mx = fmaxf(mx, su[i]);
            mn = fminf(mn, sl[i]);
        }
        Useg[(int64_t)q * nseg + s] = mx;
        Lseg[(int64_t)q * nseg + s] = mn;
    }
}

// ------------------------------------------------------ shard summaries
// PAA segment means (f64 sum, stored f32) of every row + max|x| over the shard
__global__ void paa_kernel(const float *__restrict__ X, int64_t N, int m, int64_t ld, int nseg,
                           float *__restrict__ paa, unsigned *__restrict__ maxabs) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    float mx = 0.f;
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < N; row += nw) {
        const float *x = X + row * ld;
        for (int s = lane; s < nseg; s += 32) {
            int a = s * SSH_PAA_SEG, b = min(m, a + SSH_PAA_SEG);
            double sum = 0.0;
            for (int i = a; i < b; i++) {
                float v = x[i];
                sum += (double)v;
                mx = fmaxf(mx, fabsf(v));
            }
            paa[row * nseg + s] = (float)(sum / (double)(b - a));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) atomicMax(maxabs, __float_as_uint(mx));
}

extern "C" int ssh_index_summarize(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t ld,
                                   void *stream) {
    SSH_REQUIRE(ctx && ix && X, SSH_ERR_INVALID, "ssh_index_summarize: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_index_summarize: params not set");
    SSH_REQUIRE(ld >= ctx->p.m, SSH_ERR_INVALID, "ssh_index_summarize: ld < m");
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int m = ctx->p.m;
    const int nseg = (m + SSH_PAA_SEG - 1) / SSH_PAA_SEG;
    if (!ix->paa) {
        SSH_CUDA(cudaMallocAsync((void **)&ix->paa, sizeof(float) * (size_t)ix->N * nseg, st));
        SSH_CUDA(cudaMallocAsync((void **)&ix->d_maxabs, sizeof(unsigned), st));
    }
    ix->nseg = nseg;
    SSH_CUDA(cudaMemsetAsync(ix->d_maxabs, 0, sizeof(unsigned), st));
    int grid = (int)std::min<int64_t>((ix->N + 7) / 8, (int64_t)ctx->num_sms * 16);
    paa_kernel<<<grid, 256, 0, st>>>(X, ix->N, m, ld, nseg, ix->paa, ix->d_maxabs);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

// --------------------------------------------------- member stream kernel
// One CTA per (query, slice of MB_SLICE_WORDS bitmap words).  A warp turns 32
// words into a member list in shared memory, evaluates LB_PAA lane-per-member
// (L2-resident summaries), and
//   MODE_HIST    histograms LB_PAA (seed threshold),
//   MODE_COLLECT lists members with LB_PAA below the per-query threshold,
//   MODE_FILTER  keeps members with LB_PAA <= thr and runs LB_Kim + the
//                early-abandoning LB_Keogh warp-cooperatively; survivors are
//                appended with their LB_Keogh value.
enum { MODE_HIST = 0, MODE_COLLECT = 1, MODE_FILTER = 2 };

struct MemberArgs {
    const float *X;
    const float *Q;
    const float *U, *Lo, *Useg, *Lseg;
    const float *paa;
    const unsigned *maxabs;
    const uint32_t *bitmap;
    const float *thr;
    const uint32_t *ts;
    uint32_t *hist;
    uint32_t *out;
    float *out_lb;
    int *out_cnt;
    long long *counters;
    unsigned long long *dbg;  // profiling counters (ctx->d_cells) or NULL
    int64_t NW;
    int m, nseg, cap;
};

template <int MODE>
__global__ void __launch_bounds__(MB_THREADS) members_kernel(MemberArgs a) {
    extern __shared__ __align__(16) unsigned char msm[];
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int m = a.m, nseg = a.nseg;
    float *sUs = reinterpret_cast<float *>(msm);
    float *sLs = sUs + nseg;
    uint32_t *lists = reinterpret_cast<uint32_t *>(sLs + nseg);  // MB_WARPS x 1024
    uint32_t *shist = lists + MB_WARPS * 1024;                   // NBINS (HIST)
    float *su = reinterpret_cast<float *>(lists + MB_WARPS * 1024);  // m (FILTER)
    float *sl = su + m;
    for (int s = threadIdx.x; s < nseg; s += MB_THREADS) {
        sUs[s] = a.Useg[(int64_t)q * nseg + s];
        sLs[s] = a.Lseg[(int64_t)q * nseg + s];
    }
    if (MODE == MODE_HIST)
        for (int b = threadIdx.x; b < NBINS; b += MB_THREADS) shist[b] = 0u;
    if (MODE == MODE_FILTER)
        for (int i = threadIdx.x; i < m; i += MB_THREADS) {
            su[i] = a.U[(int64_t)q * m + i];
            sl[i] = a.Lo[(int64_t)q * m + i];
        }
    __syncthreads();
    // |stored mean - exact mean| <= 2u max|x|; products/sums: relative (2 nseg + 8) u
    const float delta = 2.f * U32_EPS * __uint_as_float(*a.maxabs) + 1e-30f;
    const float shrink = 1.f - (2.f * nseg + 8.f) * U32_EPS;
    const float lastlen = (float)(m - (nseg - 1) * SSH_PAA_SEG);
    const float T = MODE == MODE_FILTER ? a.thr[q] : 0.f;
    const uint32_t TS = MODE == MODE_COLLECT ? a.ts[q] : 0u;
    const float q0 = a.Q[(int64_t)q * m], ql = a.Q[(int64_t)q * m + m - 1];
    const uint32_t *bm = a.bitmap + (int64_t)q * a.NW;
    uint32_t *list = lists + w * 1024;
    int paa_pr = 0, kim = 0, keo = 0, nvisit = 0;
    const int64_t s0 = (int64_t)blockIdx.x * MB_SLICE_WORDS;
    const int64_t s1 = min(a.NW, s0 + MB_SLICE_WORDS);
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t wb = s0 + 32 * w; wb < s1; wb += 32 * MB_WARPS) {
        const int64_t wd = wb + lane;
        uint32_t word = wd < s1 ? bm[wd] : 0u;
        int c = __popc(word);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        nvisit += lane == 0 ? total : 0;
        int pos = incl - c;
        while (word) {
            int b = __ffs(word) - 1;
            word &= word - 1;
            list[pos++] = (uint32_t)(wd * 32 + b);
        }
        __syncwarp();
        // stage A: LB_PAA, lane per member
        int kept = 0;
        for (int base = 0; base < total; base += 32) {
            const int e = base + lane;
            bool keep = false;
            uint32_t row = 0;
            if (e < total) {
                row = list[e];
                const float *p = a.paa + (int64_t)row * nseg;
                float acc = 0.f;
                for (int s = 0; s < nseg; s++) {
                    float xb = __ldg(p + s);
                    float ev = fmaxf(fmaxf(xb - sUs[s] - delta, sLs[s] - xb - delta), 0.f);
                    float len = s + 1 < nseg ? (float)SSH_PAA_SEG : lastlen;
                    acc = fmaf(len * ev, ev, acc);
                }
                const float lb = acc * shrink;
                if (MODE == MODE_HIST) {
                    atomicAdd(&shist[lb_bin(lb)], 1u);
                } else if (MODE == MODE_COLLECT) {
                    if (__float_as_uint(lb) < TS) {
                        int p2 = atomicAdd(&a.out_cnt[q], 1);
                        if (p2 < a.cap) {
                            a.out[(int64_t)q * a.cap + p2] = row;
                            a.out_lb[(int64_t)q * a.cap + p2] = lb;
                        }
                    }
                } else {
                    keep = !(lb > T);
                    paa_pr += !keep;
                }
            }
            if (MODE == MODE_FILTER) {
                unsigned msk = __ballot_sync(0xFFFFFFFFu, keep);
                if (keep) list[kept + __popc(msk & lt)] = row;
                kept += __popc(msk);
                __syncwarp();
            }
        }
        if (MODE == MODE_FILTER) {
            // stage B: LB_Kim + early-abandoning LB_Keogh, warp per member
            for (int e = 0; e < kept; e++) {
                const uint32_t row = list[e];
                const float *x = a.X + (int64_t)row * m;
                if (m >= 2) {
                    float d0 = x[0] - q0, dl = x[m - 1] - ql;
                    if (fmaf(dl, dl, d0 * d0) > T) { kim++; continue; }
                }
                float acc = 0.f, tot = 0.f;
                bool pruned = false;
                for (int base = 0; base < m; base += 128) {
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        int i = base + k * 32 + lane;
                        if (i < m) {
                            float cv = __ldg(x + i);
                            float v = fmaxf(fmaxf(cv - su[i], sl[i] - cv), 0.f);
                            acc = fmaf(v, v, acc);
                        }
                    }
                    tot = warp_sum(acc);
                    if (tot > T) { pruned = true; break; }
                }
                if (pruned) { keo++; continue; }
                if (lane == 0) {
                    int p2 = atomicAdd(&a.out_cnt[q], 1);
                    if (p2 < a.cap) {
                        a.out[(int64_t)q * a.cap + p2] = row;
                        a.out_lb[(int64_t)q * a.cap + p2] = tot;
                    }
                }
            }
        }
        __syncwarp();
    }
    if (MODE == MODE_HIST) {
        __syncthreads();
        for (int b = threadIdx.x; b < NBINS; b += MB_THREADS) {
            uint32_t v = shist[b];
            if (v) atomicAdd(&a.hist[(int64_t)q * NBINS + b], v);
        }
    }
    if (MODE == MODE_FILTER) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) paa_pr += __shfl_xor_sync(0xFFFFFFFFu, paa_pr, o);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nvisit += __shfl_xor_sync(0xFFFFFFFFu, nvisit, o);
        if (lane == 0) {
            long long k1 = kim, k2 = (long long)keo + paa_pr;
            if (k1) atomicAdd((unsigned long long *)&a.counters[q * 5 + 0], (unsigned long long)k1);
            if (k2) atomicAdd((unsigned long long *)&a.counters[q * 5 + 1], (unsigned long long)k2);
            if (a.dbg) {
                atomicAdd(&a.dbg[1], (unsigned long long)paa_pr);
                atomicAdd(&a.dbg[2], (unsigned long long)keo);
                atomicAdd(&a.dbg[3], (unsigned long long)nvisit);
            }
        }
    }
}

// per query: LB_PAA bin threshold holding >= S0 members
__global__ void seed_thresh_kernel(const uint32_t *__restrict__ hist, int S0, uint32_t *__restrict__ ts) {
    __shared__ uint32_t part[NBINS / 8];
    const int q = blockIdx.x;
    const uint32_t *h = hist + (int64_t)q * NBINS;
    uint32_t s = 0;
    for (int b = 0; b < 8; b++) s += h[threadIdx.x * 8 + b];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t cum = 0;
        uint32_t out = 0xFFFFFFFFu;
        for (int t = 0; t < NBINS / 8 && out == 0xFFFFFFFFu; t++) {
            if (cum + part[t] >= (uint32_t)S0) {
                for (int b = 0; b < 8; b++) {
                    cum += h[t * 8 + b];
                    if (cum >= (uint32_t)S0) {
                        int bin = t * 8 + b;
                        out = bin + 1 >= NBINS ? 0xFFFFFFFFu : ((uint32_t)(bin + 1) << 20);
                        break;
                    }
                }
            } else {
                cum += part[t];
            }
        }
        ts[q] = out;
    }
}

// per query: the S0 collected members with the smallest LB_PAA -> seeds
__global__ void seed_select_kernel(const uint32_t *__restrict__ cand, const float *__restrict__ cand_lb,
                                   const int *__restrict__ cand_cnt, int cap, int S0,
                                   uint32_t *__restrict__ seeds, int *__restrict__ nseed) {
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    uint32_t *out = seeds + (int64_t)q * S0;
    const int n = min(cand_cnt[q], cap);
    const uint32_t *bits = reinterpret_cast<const uint32_t *>(cand_lb + (int64_t)q * cap);
    uint32_t V = 0xFFFFFFFFu;
    if (n > S0) V = block_kth2<uint32_t>(bits, n, nullptr, 0, S0, 0x7F800000u, red);
    if (threadIdx.x == 0) npos = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        if (n <= S0 || bits[e] < V) out[atomicAdd(&npos, 1)] = cand[(int64_t)q * cap + e];
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        if (n > S0 && bits[e] == V) {
            int p = atomicAdd(&npos, 1);
            if (p < S0) out[p] = cand[(int64_t)q * cap + e];
        }
    __syncthreads();
    const int c = min(npos, S0);
    for (int e = c + threadIdx.x; e < S0; e += blockDim.x) out[e] = 0xFFFFFFFFu;
    if (threadIdx.x == 0) nseed[q] = c;
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
};

__device__ __forceinline__ void dtw_list_range(const DtwList &L, int q, int &start, int &end) {
    start = L.off ? L.off[q] : 0;
    const int total = L.cnt ? L.cnt[q] : (int)L.stride;
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
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int B = 2 * r + 2;
    const int ypadn = (m + 2 * r + 3) & ~3;
    float *ypad = dsm;  // m + 2r
    float *su = dsm + ypadn;
    float *sl = su + m;
    float *band = sl + m + (size_t)w * B * 32;
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
    int start, end;
    dtw_list_range(L, q, start, end);
    const int e = start + (blockIdx.x * warps + w) * 32 + lane;
    if (start + (blockIdx.x * warps + w) * 32 >= end) return;
    uint32_t row = e < end ? L.rows[(int64_t)q * L.stride + e] : 0xFFFFFFFFu;
    bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)q * L.stride + e] > T));
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
        L.out[(int64_t)q * L.stride + e] = res;
        if (L.abandoned && valid && !alive) atomicAdd(&L.abandoned[q], 1ULL);
    }
    if (cells) {
        unsigned long long c = (unsigned long long)rows * (unsigned long long)(2 * r + 1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        if (lane == 0 && c) atomicAdd(cells, c);
    }
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
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int YP = ((m + 2 * R + 8) + 3) & ~3;
    float *yc = rsm;           // 4 x YP
    float *su = rsm + 4 * YP;  // m
    float *sl = su + m;        // m
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
    int start, end;
    dtw_list_range(L, q, start, end);
    const int e = start + (blockIdx.x * warps + w) * 32 + lane;
    if (start + (blockIdx.x * warps + w) * 32 >= end) return;
    const uint32_t row = e < end ? L.rows[(int64_t)q * L.stride + e] : 0xFFFFFFFFu;
    const bool valid = row != 0xFFFFFFFFu && (!L.lbs || !(L.lbs[(int64_t)q * L.stride + e] > T));
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
        L.out[(int64_t)q * L.stride + e] = (valid && alive) ? band[R] : INFINITY;
        if (L.abandoned && valid && !alive) atomicAdd(&L.abandoned[q], 1ULL);
    }
    if (cells) {
        unsigned long long cc = (unsigned long long)rows * (unsigned long long)NB;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xFFFFFFFFu, cc, o);
        if (lane == 0 && cc) atomicAdd(cells, cc);
    }
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
// thr0 from the seed DTWs (k-th smallest of distinct seeds)
__global__ void tau_kernel(const float *__restrict__ sd32, int S0, const int *__restrict__ nseed,
                           int k, float eps, float *__restrict__ thr) {
    __shared__ int red[32];
    const int q = blockIdx.x;
    const int ns = nseed[q];
    const uint32_t *bits = reinterpret_cast<const uint32_t *>(sd32 + (int64_t)q * S0);
    float t = INFINITY;
    if (k <= ns) {
        int nfin = block_count_le2<uint32_t>(bits, ns, nullptr, 0, 0x7F7FFFFFu, red);
        if (nfin >= k) t = __uint_as_float(block_kth2<uint32_t>(bits, ns, nullptr, 0, k, 0x7F7FFFFFu, red));
    }
    if (threadIdx.x == 0) thr[q] = thr_from(t, eps);
}

// Per query: survivors reordered by LB_Keogh bin (float bits >> 20, ~12% wide)
// with a counting sort.  Within a bin the order is arbitrary; the wave loop
// only relies on bins being non-decreasing.
__global__ void __launch_bounds__(1024)
lbsort_kernel(const uint32_t *__restrict__ surv, const float *__restrict__ slb,
              const int *__restrict__ surv_cnt, int cap, uint32_t *__restrict__ srow,
              float *__restrict__ slbs) {
    __shared__ uint32_t h[NBINS];
    const int q = blockIdx.x;
    const int cnt = min(surv_cnt[q], cap);
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    const float *lb = slb + (int64_t)q * cap;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) atomicAdd(&h[lb_bin(lb[e])], 1u);
    __syncthreads();
    // exclusive scan of NBINS (= 2 per thread at 1024 threads)
    __shared__ uint32_t part[1024];
    const int per = NBINS / blockDim.x;
    uint32_t loc = 0;
    for (int i = 0; i < per; i++) loc += h[threadIdx.x * per + i];
    part[threadIdx.x] = loc;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
        uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
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
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        const float v = lb[e];
        const uint32_t p = atomicAdd(&h[lb_bin(v)], 1u);
        srow[(int64_t)q * cap + p] = surv[(int64_t)q * cap + e];
        slbs[(int64_t)q * cap + p] = v;
    }
}

// After a wave: fold its fp32 DTWs into the per-query k smallest (topk),
// tighten thr = min(thr, kth (1 + eps)), advance the wave start and decide
// whether the query is done (next entry's LB bin above thr's bin => every
// remaining LB exceeds thr).  Sets *active if any query continues.
__global__ void wave_update_kernel(const float *__restrict__ d32, const float *__restrict__ slbs,
                                   const int *__restrict__ cnt, int cap, int wave, int k, float eps,
                                   float *__restrict__ topk, float *__restrict__ thr,
                                   int *__restrict__ pos, int *__restrict__ done,
                                   int *__restrict__ active) {
    __shared__ int red[32];
    const int q = blockIdx.x;
    if (done[q]) return;
    const int start = pos[q];
    const int total = min(cnt[q], cap);
    const int end = min(total, start + wave);
    const uint32_t *wb = reinterpret_cast<const uint32_t *>(d32 + (int64_t)q * cap + start);
    uint32_t *tb = reinterpret_cast<uint32_t *>(topk + (int64_t)q * k);
    const int nw = end - start;
    const int nfin = block_count_le2<uint32_t>(tb, k, wb, nw, 0x7F7FFFFFu, red);
    float T = thr[q];
    if (nfin >= k) {
        const uint32_t kv = block_kth2<uint32_t>(tb, k, wb, nw, k, 0x7F7FFFFFu, red);
        // new topk: values < kv, padded with kv
        __shared__ int npos;
        __shared__ uint32_t tmp[2048];
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
        // fewer than k finite values so far: append the wave's finite values
        __shared__ int npos2;
        if (threadIdx.x == 0) {
            int c = 0;
            for (int e = 0; e < k; e++) c += tb[e] <= 0x7F7FFFFFu;
            npos2 = c;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nw; e += blockDim.x)
            if (wb[e] <= 0x7F7FFFFFu) tb[atomicAdd(&npos2, 1)] = wb[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        thr[q] = T;
        pos[q] = end;
        const bool fin = end >= total || lb_bin(slbs[(int64_t)q * cap + end]) > lb_bin(T);
        done[q] = fin;
        if (!fin) atomicOr(active, 1);
    }
}

// rescoring set over every wave: d32 <= T_k (1 + eps)
__global__ void select_kernel(const uint32_t *__restrict__ srow, const float *__restrict__ d32,
                              const int *__restrict__ pos, int cap, int k, float eps,
                              uint32_t *__restrict__ resc, int *__restrict__ resc_cnt,
                              long long *__restrict__ counters, const int *__restrict__ cnt,
                              const int *__restrict__ computed) {
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    const int n = pos[q];
    const uint32_t *b = reinterpret_cast<const uint32_t *>(d32 + (int64_t)q * cap);
    const int nfin = block_count_le2<uint32_t>(b, n, nullptr, 0, 0x7F7FFFFFu, red);
    const int kk = min(k, nfin);
    float bound = -1.f;
    if (kk > 0) bound = thr_from(__uint_as_float(block_kth2<uint32_t>(b, n, nullptr, 0, kk, 0x7F7FFFFFu, red)), eps);
    if (threadIdx.x == 0) npos = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        if (d32[(int64_t)q * cap + e] <= bound) resc[(int64_t)q * cap + atomicAdd(&npos, 1)] = srow[(int64_t)q * cap + e];
    __syncthreads();
    if (threadIdx.x == 0) {
        resc_cnt[q] = npos;
        // survivors never evaluated were excluded by LB_Keogh > thr
        counters[q * 5 + 1] += min(cnt[q], cap) - computed[q];
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

__global__ void finalize_counters(const int *__restrict__ nseed, const int *__restrict__ computed,
                                  const unsigned long long *__restrict__ abandoned, int nq,
                                  const long long *__restrict__ n_cand,
                                  const int *__restrict__ is_fb, long long *__restrict__ counters,
                                  int *__restrict__ status) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    counters[q * 5 + 3] = (long long)nseed[q] + computed[q];
    counters[q * 5 + 4] = (long long)abandoned[q];
    status[q] = n_cand[q] == 0 ? 1 : (is_fb[q] ? 2 : 0);
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

struct QueryBufs {
    uint64_t *qsig, *qbits, *bstart;
    uint32_t *blen, *seeds, *w1, *ts, *cand;
    int *isfb, *nseed, *scnt, *c1, *c2, *rcnt, *ccnt, *done, *active;
    float *U, *Lo, *Useg, *Lseg, *sd32, *thr, *d1, *cand_lb;
    unsigned long long *aband;

    void carve(Carver &c, int nc, int L, int words, int S0, int W1, int m, int nseg) {
        qsig = c.take<uint64_t>((size_t)nc * L);
        qbits = c.take<uint64_t>((size_t)nc * words);
        bstart = c.take<uint64_t>((size_t)nc * L);
        blen = c.take<uint32_t>((size_t)nc * L);
        seeds = c.take<uint32_t>((size_t)nc * S0);
        w1 = c.take<uint32_t>((size_t)nc * W1);
        ts = c.take<uint32_t>(nc);
        cand = c.take<uint32_t>((size_t)nc * Q_SEED_CAND);
        isfb = c.take<int>(nc);
        nseed = c.take<int>(nc);
        scnt = c.take<int>(nc);
        c1 = c.take<int>(nc);
        c2 = c.take<int>(nc);
        rcnt = c.take<int>(nc);
        ccnt = c.take<int>(nc);
        done = c.take<int>(nc);
        active = c.take<int>(1);
        U = c.take<float>((size_t)nc * m);
        Lo = c.take<float>((size_t)nc * m);
        Useg = c.take<float>((size_t)nc * nseg);
        Lseg = c.take<float>((size_t)nc * nseg);
        sd32 = c.take<float>((size_t)nc * S0);
        thr = c.take<float>(nc);
        d1 = c.take<float>((size_t)nc * W1);
        cand_lb = c.take<float>((size_t)nc * Q_SEED_CAND);
        aband = c.take<unsigned long long>(nc);
    }
};

struct PhaseTimer {
    ssh_ctx *ctx;
    cudaStream_t st;
    cudaEvent_t ev[8];
    int n = 0;
    bool on;
    PhaseTimer(ssh_ctx *c, cudaStream_t s) : ctx(c), st(s), on(c->profile != 0) {
        if (on)
            for (int i = 0; i < 8; i++) cudaEventCreate(&ev[i]);
    }
    void mark() {
        if (on && n < 8) cudaEventRecord(ev[n++], st);
    }
    void flush() {
        if (!on || n == 0) return;
        cudaEventSynchronize(ev[n - 1]);
        for (int i = 1; i < n; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            ctx->prof[i - 1] += ms;
        }
        n = 0;
    }
    ~PhaseTimer() {
        if (on)
            for (int i = 0; i < 8; i++) cudaEventDestroy(ev[i]);
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

size_t members_smem(int mode, int m, int nseg) {
    size_t b = (size_t)2 * nseg * 4 + (size_t)MB_WARPS * 1024 * 4;
    if (mode == MODE_HIST) b += NBINS * 4;
    if (mode == MODE_FILTER) b += (size_t)2 * m * 4;
    return b;
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

// fp32 DTW of a candidate list (register band for the common radii, shared-memory band otherwise)
static int launch_dtw32(ssh_ctx *ctx, const float *X, const float *Q, const float *U,
                        const float *Lo, const DtwList &L, const float *thr, int nq,
                        cudaStream_t st) {
    const int m = ctx->p.m, r = ctx->p.radius;
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

static int launch_dtw64_list(const float *X, int m, int r, const float *Q, const uint32_t *list,
                             int64_t stride, const int *cnt, int maxcnt, double *out, int nq,
                             cudaStream_t st) {
    size_t smem;
    int t = dtw64_threads(r, &smem);
    SSH_CUDA(cudaFuncSetAttribute(dtw64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (maxcnt <= 0) return SSH_OK;
    dim3 grid((unsigned)ssh_div_up(maxcnt, t), (unsigned)nq);
    dtw64_kernel<<<grid, t, smem, st>>>(X, m, r, Q, nullptr, list, stride, cnt, nullptr, 0, out);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

template <int MODE>
static int launch_members(const MemberArgs &a, int nq, cudaStream_t st) {
    size_t smem = members_smem(MODE, a.m, a.nseg);
    SSH_CUDA(cudaFuncSetAttribute(members_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    dim3 g((unsigned)ssh_div_up(a.NW, MB_SLICE_WORDS), (unsigned)nq);
    members_kernel<MODE><<<g, MB_THREADS, smem, st>>>(a);
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
    size_t smem;
    int t = dtw64_threads(r, &smem);
    SSH_CUDA(cudaFuncSetAttribute(dtw64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dtw64_kernel<<<(unsigned)ssh_div_up(npair, t), t, smem, (cudaStream_t)stream>>>(
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
                            int *is_fb, cudaStream_t st) {
    const int L = ix->L;
    const int64_t N = ix->N, NW = (N + 31) / 32;
    probe_kernel<<<ssh_div_up((int64_t)nq * L, 128), 128, 0, st>>>(
        qsig, nq, L, ix->keys, ix->offsets, ix->d_nb, ix->d_kbase, N, bstart, blen);
    SSH_CHECK_LAUNCH();
    SSH_CUDA(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (size_t)nq * NW, st));
    dim3 g((unsigned)(nq * L), 8);
    bitmap_kernel<<<g, 256, 0, st>>>(ix->ids, bstart, blen, L, NW, bitmap);
    SSH_CHECK_LAUNCH();
    count_kernel<<<nq, 256, 0, st>>>(bitmap, NW, N, blen, L, fallback, n_cand, is_fb);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

extern "C" int ssh_probe(ssh_ctx *ctx, const ssh_index *ix, const uint64_t *qsig, int32_t nq,
                         uint32_t *bitmap, int64_t *n_cand, void *stream) {
    SSH_REQUIRE(ctx && ix && qsig && bitmap && n_cand, SSH_ERR_INVALID, "ssh_probe: NULL argument");
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
    return probe_and_bitmap(ix, qsig, nq, 0, bstart, blen, bitmap, (long long *)n_cand, isfb, st);
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
    SSH_REQUIRE(k <= 2048, SSH_ERR_UNSUPPORTED, "k=%d exceeds the device limit 2048", k);
    SSH_REQUIRE(nq >= 0, SSH_ERR_INVALID, "nq must be >= 0");
    if (nq == 0) return SSH_OK;
    SSH_REQUIRE(X && Q && out_ids && out_d2 && n_out && n_cand && counters && status, SSH_ERR_INVALID,
                "ssh_query_batch: NULL pointer");
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    ssh_index *mix = const_cast<ssh_index *>(ix);
    if (!mix->paa) {
        int rc = ssh_index_summarize(ctx, mix, X, ctx->p.m, stream);
        if (rc) return rc;
    }
    const int m = ctx->p.m, r = ctx->p.radius, L = ix->L, nseg = ix->nseg;
    const int64_t N = ix->N, NW = (N + 31) / 32;
    const float eps = rescore_eps(m);
    const int S0 = ((std::max(64, 2 * k) + 31) / 32) * 32;
    const int W1 = S0;
    const int fallback = (flags & SSH_QUERY_FALLBACK_ON_EMPTY) ? 1 : 0;
    // query chunk: keep the membership bitmaps under ~1 GiB
    int qc = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(nq, 32768),
                                                         ((int64_t)1 << 28) / std::max<int64_t>(1, NW)));
    SSH_CUDA(cudaMemsetAsync(counters, 0, sizeof(int64_t) * 5 * (size_t)nq, st));
    int cap = std::max(Q_SURV_CAP0, ctx->surv_cap);
    PhaseTimer pt(ctx, st);
    for (int q0 = 0; q0 < nq; q0 += qc) {
        const int nc = std::min(qc, nq - q0);
        const float *Qc = Q + (int64_t)q0 * m;
        long long *ncand = (long long *)n_cand + q0;
        long long *cnt5 = (long long *)counters + (int64_t)q0 * 5;
        Carver sizer;
        QueryBufs B;
        B.carve(sizer, nc, L, ctx->words, S0, W1, m, nseg);
        Carver cv;
        cv.base = (unsigned char *)ssh_slot(ctx, SLOT_Q_FIXED, sizer.off, st);
        if (!cv.base) return SSH_ERR_OOM;
        B.carve(cv, nc, L, ctx->words, S0, W1, m, nseg);
        uint32_t *bitmap = (uint32_t *)ssh_slot(ctx, SLOT_Q_BITMAP, sizeof(uint32_t) * (size_t)nc * NW, st);
        uint32_t *hist = (uint32_t *)ssh_slot(ctx, SLOT_Q_HIST, sizeof(uint32_t) * (size_t)nc * NBINS, st);
        if (!bitmap || !hist) return SSH_ERR_OOM;
        SSH_CUDA(cudaMemsetAsync(B.aband, 0, sizeof(unsigned long long) * nc, st));
        pt.mark();
        // K5: query signatures
        int rc = qsig_batch(ctx, Qc, nc, B.qsig, B.qbits, st);
        if (rc) return rc;
        pt.mark();
        // K6: probe + candidate bitmap
        rc = probe_and_bitmap(ix, B.qsig, nc, fallback, B.bstart, B.blen, bitmap, ncand, B.isfb, st);
        if (rc) return rc;
        pt.mark();
        // seeds: the S0 members with the smallest LB_PAA -> fp32 DTW -> thr0
        envelope_kernel<<<nc, 256, 2 * m * sizeof(float), st>>>(Qc, m, r, nseg, B.U, B.Lo, B.Useg, B.Lseg);
        ssh_count_launch();
        MemberArgs ma;
        ma.X = X; ma.Q = Qc; ma.U = B.U; ma.Lo = B.Lo; ma.Useg = B.Useg; ma.Lseg = B.Lseg;
        ma.paa = ix->paa; ma.maxabs = ix->d_maxabs; ma.bitmap = bitmap; ma.thr = B.thr; ma.ts = B.ts;
        ma.hist = hist; ma.counters = cnt5; ma.NW = NW; ma.m = m; ma.nseg = nseg;
        ma.dbg = nullptr;
        ma.out = nullptr; ma.out_lb = nullptr; ma.out_cnt = nullptr; ma.cap = 0;
        SSH_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)nc * NBINS, st));
        rc = launch_members<MODE_HIST>(ma, nc, st);
        if (rc) return rc;
        seed_thresh_kernel<<<nc, NBINS / 8, 0, st>>>(hist, S0, B.ts);
        SSH_CHECK_LAUNCH();
        SSH_CUDA(cudaMemsetAsync(B.ccnt, 0, sizeof(int) * nc, st));
        ma.out = B.cand; ma.out_lb = B.cand_lb; ma.out_cnt = B.ccnt; ma.cap = Q_SEED_CAND;
        rc = launch_members<MODE_COLLECT>(ma, nc, st);
        if (rc) return rc;
        seed_select_kernel<<<nc, 256, 0, st>>>(B.cand, B.cand_lb, B.ccnt, Q_SEED_CAND, S0, B.seeds,
                                               B.nseed);
        SSH_CHECK_LAUNCH();
        {
            DtwList dl{B.seeds, S0, B.nseed, nullptr, S0, nullptr, B.sd32, nullptr, nullptr};
            rc = launch_dtw32(ctx, X, Qc, nullptr, nullptr, dl, nullptr, nc, st);
        }
        if (rc) return rc;
        tau_kernel<<<nc, 256, 0, st>>>(B.sd32, S0, B.nseed, k, eps, B.thr);
        SSH_CHECK_LAUNCH();
        std::vector<float> thr0h;
        if (ctx->profile) {
            thr0h.resize(nc);
            cudaMemcpyAsync(thr0h.data(), B.thr, sizeof(float) * nc, cudaMemcpyDeviceToHost, st);
        }
        pt.mark();
        // K7: member filter (retried with a larger per-query capacity on overflow)
        uint32_t *surv = nullptr;
        float *slb = nullptr;
        int maxs = 0;
        for (;;) {
            surv = (uint32_t *)ssh_slot(ctx, SLOT_Q_SURV, sizeof(uint32_t) * (size_t)nc * cap, st);
            slb = (float *)ssh_slot(ctx, SLOT_Q_SURV_LB, sizeof(float) * (size_t)nc * cap, st);
            if (!surv || !slb) return SSH_ERR_OOM;
            SSH_CUDA(cudaMemsetAsync(B.scnt, 0, sizeof(int) * nc, st));
            SSH_CUDA(cudaMemsetAsync(cnt5, 0, sizeof(long long) * 5 * nc, st));
            ma.out = surv; ma.out_lb = slb; ma.out_cnt = B.scnt; ma.cap = cap;
            ma.dbg = ctx->profile ? ctx->d_cells : nullptr;
            rc = launch_members<MODE_FILTER>(ma, nc, st);
            if (rc) return rc;
            rc = max_of(B.scnt, nc, st, &maxs);
            if (rc) return rc;
            if (maxs <= cap) break;
            cap = next_pow2(maxs + maxs / 4);
            ctx->surv_cap = cap;
        }
        pt.mark();
        // K8: DTW waves in LB order (survivors bucket-sorted by LB; growing waves)
        uint32_t *srow = (uint32_t *)ssh_slot(ctx, SLOT_Q_W2, sizeof(uint32_t) * (size_t)nc * cap, st);
        float *slbs = (float *)ssh_slot(ctx, SLOT_Q_D2, sizeof(float) * (size_t)nc * cap, st);
        float *d32 = (float *)ssh_slot(ctx, SLOT_Q_D32, sizeof(float) * (size_t)nc * cap, st);
        uint32_t *resc = (uint32_t *)ssh_slot(ctx, SLOT_Q_RESC, sizeof(uint32_t) * (size_t)nc * cap, st);
        double *d64 = (double *)ssh_slot(ctx, SLOT_Q_D64, sizeof(double) * (size_t)nc * cap, st);
        float *topk = (float *)ssh_slot(ctx, SLOT_Q_TOPK, sizeof(float) * (size_t)nc * k, st);
        if (!srow || !slbs || !d32 || !resc || !d64 || !topk) return SSH_ERR_OOM;
        lbsort_kernel<<<nc, 1024, 0, st>>>(surv, slb, B.scnt, cap, srow, slbs);
        SSH_CHECK_LAUNCH();
        SSH_CUDA(cudaMemsetAsync(topk, 0xFF, sizeof(float) * (size_t)nc * k, st));  // NaN bits > any finite
        SSH_CUDA(cudaMemsetAsync(B.c1, 0, sizeof(int) * nc, st));    // wave start
        SSH_CUDA(cudaMemsetAsync(B.c2, 0, sizeof(int) * nc, st));    // DTWs evaluated
        SSH_CUDA(cudaMemsetAsync(B.done, 0, sizeof(int) * nc, st));
        int wave = W1;
        for (int it = 0; maxs > 0; it++) {
            SSH_CUDA(cudaMemsetAsync(B.active, 0, sizeof(int), st));
            DtwList dl{srow, cap, B.scnt, B.c1, std::min(wave, maxs), slbs, d32, B.aband, B.c2};
            rc = launch_dtw32(ctx, X, Qc, B.U, B.Lo, dl, B.thr, nc, st);
            if (rc) return rc;
            wave_update_kernel<<<nc, 256, 0, st>>>(d32, slbs, B.scnt, cap, std::min(wave, maxs), k, eps,
                                                   topk, B.thr, B.c1, B.done, B.active);
            SSH_CHECK_LAUNCH();
            int act = 0;
            SSH_CUDA(cudaMemcpyAsync(&act, B.active, sizeof(int), cudaMemcpyDeviceToHost, st));
            SSH_CUDA(cudaStreamSynchronize(st));
            if (!act) break;
            wave = std::min(wave * 2, 1 << 14);
        }
        pt.mark();
        // K9/K10: rescoring set, exact f64 DTW, top-k by (d64, id)
        const int RS = cap;
        select_kernel<<<nc, 256, 0, st>>>(srow, d32, B.c1, cap, k, eps, resc, B.rcnt, cnt5, B.scnt, B.c2);
        SSH_CHECK_LAUNCH();
        int maxr = 0;
        rc = max_of(B.rcnt, nc, st, &maxr);
        if (rc) return rc;
        rc = launch_dtw64_list(X, m, r, Qc, resc, RS, B.rcnt, maxr, d64, nc, st);
        if (rc) return rc;
        const int P2k = next_pow2(k);
        size_t stk = (size_t)P2k * (sizeof(double) + sizeof(uint32_t));
        SSH_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stk));
        topk_kernel<<<nc, 256, stk, st>>>(resc, d64, B.rcnt, RS, P2k, k, ix->id_base, ncand,
                                          (long long *)out_ids + (int64_t)q0 * k,
                                          out_d2 + (int64_t)q0 * k, n_out + q0);
        SSH_CHECK_LAUNCH();
        finalize_counters<<<ssh_div_up(nc, 128), 128, 0, st>>>(B.nseed, B.c2, B.aband, nc, ncand,
                                                               B.isfb, cnt5, status + q0);
        SSH_CHECK_LAUNCH();
        pt.mark();
        if (ctx->profile) {
            pt.flush();
            std::vector<int> h(nc);
            cudaMemcpy(h.data(), B.scnt, sizeof(int) * nc, cudaMemcpyDeviceToHost);
            for (int v : h) ctx->prof[8] += v;
            cudaMemcpy(h.data(), B.rcnt, sizeof(int) * nc, cudaMemcpyDeviceToHost);
            for (int v : h) ctx->prof[9] += v;
            // threshold quality: thr0 / d_k and thr1 / d_k (d_k = exact k-th squared distance)
            std::vector<float> thr1h(nc);
            std::vector<double> dk((size_t)nc * k);
            cudaMemcpy(thr1h.data(), B.thr, sizeof(float) * nc, cudaMemcpyDeviceToHost);
            cudaMemcpy(dk.data(), out_d2 + (int64_t)q0 * k, sizeof(double) * nc * k, cudaMemcpyDeviceToHost);
            for (int q = 0; q < nc; q++) {
                double d = dk[(size_t)q * k + k - 1];
                if (d > 0 && std::isfinite(d) && std::isfinite(thr0h[q])) {
                    ctx->prof[13] += thr0h[q] / d;
                    ctx->prof[14] += thr1h[q] / d;
                    ctx->prof[15] += 1;
                }
            }
        }
    }
    return SSH_OK;
}
