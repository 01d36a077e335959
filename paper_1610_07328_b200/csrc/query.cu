// query.cu — K5..K10: query_index (index.py:204-273) for a batch of queries.
//
// Reference semantics: R = deduplicated union of the L probed buckets
// (index.py:184-190); the result is the exact top-k of R by (DTW^2, id)
// (_cascade_search dtw.py:171-236 visits candidates in (lb, id) order with
// strict pruning, so its result is visit-order independent; SURVEY.md §8a
// A14).  Distances are the reference's f64 values (dtw.py:83-121, FMA-free).
//
// Device pipeline per query batch (all queries in flight at once):
//   probe      binary search of each query key in each table's sorted keys
//   bitmap     membership bitmap of R (warp-aggregated atomicOr over buckets)
//   seeds      up to S0 distinct members taken from the smallest probed
//              buckets first; their fp32 DTW gives tau_q >= true k-th best
//   lb_filter  LB_Kim then early-abandoning LB_Keogh (fp32) of every member
//              against thr_q = tau_q (1 + eps); survivors listed per query
//   dtw32      lane-per-candidate banded DTW (fp32, row-min abandon at thr_q)
//   select     T_k = k-th smallest fp32 DTW; rescoring set = d32 <= T_k(1+eps)
//   dtw64      exact f64 DTW (__dsub_rn/__dmul_rn/__dadd_rn, reference order)
//   topk       sort by (d64, id) -> ids / d2
// eps = (8m + 64) 2^-24 bounds the relative error of every fp32 bound and
// DTW value against the f64 reference values, so no member of
// the exact top-k is ever pruned, abandoned or left unrescored.
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

#define Q_SURV_CAP0 4096
#define LB_THREADS 256
#define LB_WARPS (LB_THREADS / 32)
#define LB_WORDS 64

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
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

// membership bitmap: blockIdx.y = q*L + j
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

// query envelope (dtw.py:124-151 semantics: max/min over [i-r, i+r])
__global__ void envelope_kernel(const float *__restrict__ Q, int m, int r, float *__restrict__ U,
                                float *__restrict__ Lo) {
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
        U[(int64_t)q * m + i] = mx;
        Lo[(int64_t)q * m + i] = mn;
    }
}

// seeds: distinct members from the smallest non-empty probed buckets first
__global__ void seed_kernel(const uint32_t *__restrict__ ids, const uint64_t *__restrict__ bstart,
                            const uint32_t *__restrict__ blen, int L, int S0, int64_t N,
                            const int *__restrict__ is_fallback, uint32_t *__restrict__ seeds,
                            int *__restrict__ nseed) {
    const int q = blockIdx.x;
    const int lane = threadIdx.x;
    extern __shared__ uint32_t hset[];  // 2*S0 hash slots, then L used-flags
    const int H = 2 * S0;
    uint32_t *used = hset + H;
    for (int e = lane; e < H; e += 32) hset[e] = 0xFFFFFFFFu;
    for (int j = lane; j < L; j += 32) used[j] = blen[(int64_t)q * L + j] == 0;
    __syncwarp();
    uint32_t *out = seeds + (int64_t)q * S0;
    int cnt = 0;
    if (is_fallback[q]) {
        int n = (int)((int64_t)S0 < N ? (int64_t)S0 : N);
        for (int e = lane; e < S0; e += 32) out[e] = e < n ? (uint32_t)e : 0xFFFFFFFFu;
        if (lane == 0) nseed[q] = n;
        return;
    }
    const unsigned lt = (1u << lane) - 1u;
    while (cnt < S0) {
        // smallest unused non-empty bucket (ties -> lowest table)
        uint64_t mn = ~0ULL;
        for (int j = lane; j < L; j += 32)
            if (!used[j]) {
                uint64_t key = ((uint64_t)blen[(int64_t)q * L + j] << 16) | (uint64_t)j;
                mn = key < mn ? key : mn;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t o2 = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
            mn = o2 < mn ? o2 : mn;
        }
        if (mn == ~0ULL) break;
        int jsel = (int)(mn & 0xFFFF);
        uint32_t len = (uint32_t)(mn >> 16);
        __syncwarp();
        if (lane == 0) used[jsel] = 1;
        __syncwarp();
        const uint32_t *b = ids + bstart[(int64_t)q * L + jsel];
        for (uint32_t base = 0; base < len && cnt < S0; base += 32) {
            uint32_t e = base + lane;
            bool ins = false;
            uint32_t row = 0;
            if (e < len) {
                row = b[e];
                uint32_t h = (row * 2654435761u) % (uint32_t)H;
                while (true) {
                    uint32_t prev = atomicCAS(&hset[h], 0xFFFFFFFFu, row);
                    if (prev == 0xFFFFFFFFu) { ins = true; break; }
                    if (prev == row) break;
                    h = (h + 1) % (uint32_t)H;
                }
            }
            unsigned msk = __ballot_sync(0xFFFFFFFFu, ins);
            int pos = cnt + __popc(msk & lt);
            if (ins && pos < S0) out[pos] = row;
            cnt = min(S0, cnt + __popc(msk));
            __syncwarp();
        }
    }
    for (int e = cnt + lane; e < S0; e += 32) out[e] = 0xFFFFFFFFu;
    if (lane == 0) nseed[q] = cnt;
}

// ------------------------------------------------------------ fp32 DTW
// lane-per-candidate banded DTW; band[k][lane] in shared memory, query padded
// with +inf outside [0, m) so out-of-band cells are +inf without branches.
__global__ void dtw32_kernel(const float *__restrict__ X, int m, int r, const float *__restrict__ Q,
                             const uint32_t *__restrict__ list, int64_t list_stride,
                             const int *__restrict__ list_cnt, int cap, const float *__restrict__ thr,
                             float *__restrict__ out, unsigned long long *__restrict__ abandoned,
                             int warps) {
    extern __shared__ float dsm[];
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int B = 2 * r + 2;
    float *ypad = dsm;                           // m + 2r
    float *band = dsm + ((m + 2 * r + 3) & ~3) + (size_t)w * B * 32;
    const float *y = Q + (int64_t)q * m;
    for (int j = threadIdx.x; j < m + 2 * r; j += blockDim.x) {
        int jj = j - r;
        ypad[j] = (jj >= 0 && jj < m) ? y[jj] : INFINITY;
    }
    __syncthreads();
    const int cnt = min(list_cnt ? list_cnt[q] : (int)list_stride, cap);
    const int e = (blockIdx.x * warps + w) * 32 + lane;
    if ((blockIdx.x * warps + w) * 32 >= cnt) return;
    uint32_t row = e < cnt ? list[(int64_t)q * list_stride + e] : 0xFFFFFFFFu;
    bool valid = row != 0xFFFFFFFFu;
    const float T = thr ? thr[q] : INFINITY;
    for (int k = 0; k < B; k++) band[k * 32 + lane] = INFINITY;
    band[r * 32 + lane] = 0.f;
    const float *x = X + (int64_t)(valid ? row : 0) * m;
    bool alive = valid;
    for (int i = 0; i < m; i++) {
        if (!__any_sync(0xFFFFFFFFu, alive)) break;
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
        if (alive && rmin > T) alive = false;
    }
    if (e < cnt) {
        float res = (valid && alive) ? band[r * 32 + lane] : INFINITY;
        out[(int64_t)q * list_stride + e] = res;
        if (abandoned && valid && !alive) atomicAdd(&abandoned[q], 1ULL);
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

// ------------------------------------------------------- LB filter
__global__ void __launch_bounds__(LB_THREADS)
lb_filter_kernel(const float *__restrict__ X, int m, const float *__restrict__ Q,
                 const float *__restrict__ U, const float *__restrict__ Lo,
                 const uint32_t *__restrict__ bitmap, int64_t NW, const float *__restrict__ thr,
                 uint32_t *__restrict__ surv, int cap, int *__restrict__ surv_cnt,
                 long long *__restrict__ counters) {
    extern __shared__ float lsm[];
    float *su = lsm, *sl = lsm + m;
    const int q = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < m; i += LB_THREADS) {
        su[i] = U[(int64_t)q * m + i];
        sl[i] = Lo[(int64_t)q * m + i];
    }
    __syncthreads();
    const float T = thr[q];
    const float q0 = Q[(int64_t)q * m], ql = Q[(int64_t)q * m + m - 1];
    const uint32_t *bm = bitmap + (int64_t)q * NW;
    int kim = 0, keo = 0;
    const int64_t w0 = (int64_t)blockIdx.x * LB_WORDS;
    const int64_t w1 = min(NW, w0 + LB_WORDS);
    for (int64_t wd = w0 + w; wd < w1; wd += LB_WARPS) {
        uint32_t bits = bm[wd];
        while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t row = wd * 32 + b;
            const float *x = X + row * m;
            if (m >= 2) {
                float d0 = x[0] - q0, dl = x[m - 1] - ql;
                float kv = fmaf(dl, dl, d0 * d0);
                if (kv > T) { kim++; continue; }
            }
            float acc = 0.f, tot = 0.f;
            bool pruned = false;
            for (int base = 0; base < m; base += 128) {
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    int i = base + e * 32 + lane;
                    if (i < m) {
                        float c = x[i];
                        float a = c - su[i], bb = sl[i] - c;
                        float v = fmaxf(fmaxf(a, bb), 0.f);
                        acc = fmaf(v, v, acc);
                    }
                }
                tot = warp_sum(acc);
                if (tot > T) { pruned = true; break; }
            }
            if (pruned) { keo++; continue; }
            if (lane == 0) {
                int pos = atomicAdd(&surv_cnt[q], 1);
                if (pos < cap) surv[(int64_t)q * cap + pos] = (uint32_t)row;
            }
        }
    }
    if (lane == 0 && (kim | keo)) {
        if (kim) atomicAdd((unsigned long long *)&counters[q * 5 + 0], (unsigned long long)kim);
        if (keo) atomicAdd((unsigned long long *)&counters[q * 5 + 1], (unsigned long long)keo);
    }
}

// ------------------------------------------------------- block sort helper
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

// tau_q = k-th smallest seed DTW (seeds are distinct rows of R)
__global__ void tau_kernel(const float *__restrict__ sd32, int S0, const int *__restrict__ nseed,
                           int k, float eps, float *__restrict__ thr) {
    extern __shared__ float tsm[];
    float *key = tsm;
    uint32_t *val = reinterpret_cast<uint32_t *>(tsm + S0);
    const int q = blockIdx.x;
    const int ns = nseed[q];
    for (int e = threadIdx.x; e < S0; e += blockDim.x) {
        key[e] = e < ns ? sd32[(int64_t)q * S0 + e] : INFINITY;
        val[e] = e;
    }
    __syncthreads();
    block_sort_pairs<float>(key, val, S0);
    if (threadIdx.x == 0) {
        float t = (k <= ns) ? key[k - 1] : INFINITY;
        thr[q] = isinf(t) ? INFINITY : (float)((double)t * (1.0 + (double)eps));
    }
}

// block-wide count of entries with key-bits <= v (non-negative floats/doubles
// order like their bit patterns)
template <typename U>
__device__ int block_count_le(const U *bits, int n, U v, int *red) {
    int c = 0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) c += bits[e] <= v;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
    return s;
}

// smallest v with count(bits <= v) >= kk (kk >= 1, kk <= n)
template <typename U>
__device__ U block_kth(const U *bits, int n, int kk, U hi, int *red) {
    U lo = 0;
    while (lo < hi) {
        U mid = lo + (hi - lo) / 2;
        if (block_count_le<U>(bits, n, mid, red) >= kk) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// rescoring set: d32 <= T_k (1 + eps), T_k = k-th smallest finite survivor d32
__global__ void select_kernel(const uint32_t *__restrict__ surv, const float *__restrict__ d32,
                              const int *__restrict__ surv_cnt, int cap, int k, float eps,
                              uint32_t *__restrict__ resc, int *__restrict__ resc_cnt) {
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    const int cnt = min(surv_cnt[q], cap);
    const uint32_t *bits = reinterpret_cast<const uint32_t *>(d32 + (int64_t)q * cap);
    const uint32_t INF = 0x7F800000u;
    const int nfin = block_count_le<uint32_t>(bits, cnt, INF - 1, red);
    const int kk = min(k, nfin);
    float bound = -1.f;
    if (kk > 0) {
        uint32_t t = block_kth<uint32_t>(bits, cnt, kk, INF - 1, red);
        bound = (float)((double)__uint_as_float(t) * (1.0 + (double)eps));
    }
    if (threadIdx.x == 0) npos = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        float v = d32[(int64_t)q * cap + e];
        if (v <= bound) {
            int p = atomicAdd(&npos, 1);
            resc[(int64_t)q * cap + p] = surv[(int64_t)q * cap + e];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) resc_cnt[q] = npos;
}

// exact top-k by (d64, id) of the rescored set; P2 >= k power of two
__global__ void topk_kernel(const uint32_t *__restrict__ resc, const double *__restrict__ d64,
                            const int *__restrict__ resc_cnt, int cap, int P2, int k,
                            int64_t id_base, const long long *__restrict__ n_cand,
                            long long *__restrict__ out_ids, double *__restrict__ out_d2,
                            int *__restrict__ n_out) {
    extern __shared__ double ksm[];
    double *key = ksm;
    uint32_t *val = reinterpret_cast<uint32_t *>(ksm + P2);
    __shared__ int red[32];
    __shared__ int npos;
    const int q = blockIdx.x;
    const int cnt = n_cand[q] > 0 ? min(resc_cnt[q], cap) : 0;
    const int n = min(k, cnt);
    const uint64_t *bits = reinterpret_cast<const uint64_t *>(d64 + (int64_t)q * cap);
    const uint32_t *ids = resc + (int64_t)q * cap;
    // V = n-th smallest d64; then the smallest ids among entries equal to V
    uint64_t V = 0;
    uint32_t idcut = 0xFFFFFFFFu;
    if (n > 0 && cnt > n) {
        V = block_kth<uint64_t>(bits, cnt, n, 0x7FF0000000000000ULL, red);
        int nless = V ? block_count_le<uint64_t>(bits, cnt, V - 1, red) : 0;
        int need = n - nless;
        // idcut = need-th smallest id among entries with bits == V
        uint32_t lo = 0, hi = 0xFFFFFFFFu;
        while (lo < hi) {
            uint32_t mid = lo + (hi - lo) / 2;
            int c = 0;
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) c += (bits[e] == V && ids[e] <= mid);
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
            __syncthreads();
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
            __syncthreads();
            int s = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
            if (s >= need) hi = mid; else lo = mid + 1;
        }
        idcut = lo;
    } else {
        V = 0x7FF0000000000000ULL;
    }
    if (threadIdx.x == 0) npos = 0;
    for (int e = threadIdx.x; e < P2; e += blockDim.x) {
        key[e] = (double)INFINITY;
        val[e] = 0xFFFFFFFFu;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        uint64_t b = bits[e];
        bool take = (cnt <= n) || b < V || (b == V && ids[e] <= idcut);
        if (take) {
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

__global__ void finalize_counters(const int *__restrict__ surv_cnt,
                                  const unsigned long long *__restrict__ abandoned, int nq,
                                  const long long *__restrict__ n_cand,
                                  const int *__restrict__ is_fb, long long *__restrict__ counters,
                                  int *__restrict__ status) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    counters[q * 5 + 3] = surv_cnt[q];
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

int next_pow2(int v) {
    int p = 32;
    while (p < v) p <<= 1;
    return p;
}

float rescore_eps(int m) { return (float)((8.0 * m + 64.0) * ldexp(1.0, -24)); }

int dtw32_warps(int m, int r, size_t *smem) {
    size_t yb = (size_t)((m + 2 * r + 3) & ~3) * 4;
    size_t per = (size_t)(2 * r + 2) * 32 * 4;
    int w = 4;
    while (w > 1 && yb + per * w > 200 * 1024) w--;
    *smem = yb + per * w;
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

static int launch_dtw32(const float *X, int m, int r, const float *Q, const uint32_t *list,
                        int64_t stride, const int *cnt, int cap, int maxcnt, const float *thr,
                        float *out, unsigned long long *aband, int nq, cudaStream_t st) {
    size_t smem;
    int warps = dtw32_warps(m, r, &smem);
    SSH_REQUIRE(smem <= 227 * 1024, SSH_ERR_UNSUPPORTED, "DTW band too wide (r=%d)", r);
    SSH_CUDA(cudaFuncSetAttribute(dtw32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (maxcnt <= 0) return SSH_OK;
    dim3 grid((unsigned)ssh_div_up(maxcnt, 32 * warps), (unsigned)nq);
    dtw32_kernel<<<grid, 32 * warps, smem, st>>>(X, m, r, Q, list, stride, cnt, cap, thr, out, aband,
                                                 warps);
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

static int probe_and_bitmap(ssh_ctx *ctx, const ssh_index *ix, const uint64_t *qsig, int nq,
                            int fallback, uint64_t *bstart, uint32_t *blen, uint32_t *bitmap,
                            long long *n_cand, int *is_fb, cudaStream_t st) {
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
    return probe_and_bitmap(ctx, ix, qsig, nq, 0, bstart, blen, bitmap, (long long *)n_cand, isfb, st);
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
    const int m = ctx->p.m, r = ctx->p.radius, L = ix->L;
    const int64_t N = ix->N, NW = (N + 31) / 32;
    const float eps = rescore_eps(m);
    const int S0 = ((std::max(64, 2 * k) + 31) / 32) * 32;
    const int fallback = (flags & SSH_QUERY_FALLBACK_ON_EMPTY) ? 1 : 0;
    // query chunk: keep the membership bitmaps under ~1 GiB
    int qc = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(nq, 32768),
                                                         ((int64_t)1 << 28) / std::max<int64_t>(1, NW)));
    SSH_CUDA(cudaMemsetAsync(counters, 0, sizeof(int64_t) * 5 * (size_t)nq, st));
    int cap = Q_SURV_CAP0;
    for (int q0 = 0; q0 < nq; q0 += qc) {
        const int nc = std::min(qc, nq - q0);
        const float *Qc = Q + (int64_t)q0 * m;
        long long *ncand = (long long *)n_cand + q0;
        long long *cnt5 = (long long *)counters + (int64_t)q0 * 5;
        Arena A;
        A.st = st;
        uint64_t *qsig = A.get<uint64_t>((size_t)nc * L);
        uint64_t *qbits = A.get<uint64_t>((size_t)nc * ctx->words);
        uint64_t *bstart = A.get<uint64_t>((size_t)nc * L);
        uint32_t *blen = A.get<uint32_t>((size_t)nc * L);
        uint32_t *bitmap = A.get<uint32_t>((size_t)nc * NW);
        int *isfb = A.get<int>(nc);
        float *U = A.get<float>((size_t)nc * m);
        float *Lo = A.get<float>((size_t)nc * m);
        uint32_t *seeds = A.get<uint32_t>((size_t)nc * S0);
        int *nseed = A.get<int>(nc);
        float *sd32 = A.get<float>((size_t)nc * S0);
        float *thr = A.get<float>(nc);
        int *scnt = A.get<int>(nc);
        int *rcnt = A.get<int>(nc);
        unsigned long long *aband = A.get<unsigned long long>(nc);
        if (A.err) return ssh_cuda_fail(A.err, "query scratch", __FILE__, __LINE__);
        int rc = qsig_batch(ctx, Qc, nc, qsig, qbits, st);
        if (rc) return rc;
        rc = probe_and_bitmap(ctx, ix, qsig, nc, fallback, bstart, blen, bitmap, ncand, isfb, st);
        if (rc) return rc;
        envelope_kernel<<<nc, 256, 0, st>>>(Qc, m, r, U, Lo);
        seed_kernel<<<nc, 32, sizeof(uint32_t) * (2 * S0 + L), st>>>(ix->ids, bstart, blen, L, S0, N, isfb,
                                                               seeds, nseed);
        SSH_CHECK_LAUNCH();
        rc = launch_dtw32(X, m, r, Qc, seeds, S0, nseed, S0, S0, nullptr, sd32, nullptr, nc, st);
        if (rc) return rc;
        tau_kernel<<<nc, 256, (sizeof(float) + sizeof(uint32_t)) * S0, st>>>(sd32, S0, nseed, k, eps, thr);
        SSH_CHECK_LAUNCH();
        // LB filter (retried with a larger per-query capacity on overflow)
        uint32_t *surv = nullptr;
        std::vector<int> hcnt(nc);
        SSH_CUDA(cudaFuncSetAttribute(lb_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(8 * m)));
        for (int attempt = 0;; attempt++) {
            surv = A.get<uint32_t>((size_t)nc * cap);
            if (A.err) return ssh_cuda_fail(A.err, "survivor buffer", __FILE__, __LINE__);
            SSH_CUDA(cudaMemsetAsync(scnt, 0, sizeof(int) * nc, st));
            SSH_CUDA(cudaMemsetAsync(cnt5, 0, sizeof(long long) * 5 * nc, st));
            dim3 g((unsigned)ssh_div_up(NW, LB_WORDS), (unsigned)nc);
            lb_filter_kernel<<<g, LB_THREADS, 8 * m, st>>>(X, m, Qc, U, Lo, bitmap, NW, thr, surv, cap,
                                                         scnt, cnt5);
            SSH_CHECK_LAUNCH();
            SSH_CUDA(cudaMemcpyAsync(hcnt.data(), scnt, sizeof(int) * nc, cudaMemcpyDeviceToHost, st));
            SSH_CUDA(cudaStreamSynchronize(st));
            int mx = *std::max_element(hcnt.begin(), hcnt.end());
            if (mx <= cap) break;
            cap = next_pow2(mx);
        }
        int maxs = *std::max_element(hcnt.begin(), hcnt.end());
        float *d32 = A.get<float>((size_t)nc * cap);
        uint32_t *resc = A.get<uint32_t>((size_t)nc * cap);
        double *d64 = A.get<double>((size_t)nc * cap);
        if (A.err) return ssh_cuda_fail(A.err, "rerank buffers", __FILE__, __LINE__);
        SSH_CUDA(cudaMemsetAsync(aband, 0, sizeof(unsigned long long) * nc, st));
        rc = launch_dtw32(X, m, r, Qc, surv, cap, scnt, cap, maxs, thr, d32, aband, nc, st);
        if (rc) return rc;
        select_kernel<<<nc, 256, 0, st>>>(surv, d32, scnt, cap, k, eps, resc, rcnt);
        SSH_CHECK_LAUNCH();
        std::vector<int> hr(nc);
        SSH_CUDA(cudaMemcpyAsync(hr.data(), rcnt, sizeof(int) * nc, cudaMemcpyDeviceToHost, st));
        SSH_CUDA(cudaStreamSynchronize(st));
        int maxr = *std::max_element(hr.begin(), hr.end());
        rc = launch_dtw64_list(X, m, r, Qc, resc, cap, rcnt, maxr, d64, nc, st);
        if (rc) return rc;
        const int P2k = next_pow2(k);
        size_t stk = (size_t)P2k * (sizeof(double) + sizeof(uint32_t));
        SSH_CUDA(cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stk));
        topk_kernel<<<nc, 256, stk, st>>>(resc, d64, rcnt, cap, P2k, k, ix->id_base, ncand,
                                          (long long *)out_ids + (int64_t)q0 * k,
                                          out_d2 + (int64_t)q0 * k, n_out + q0);
        SSH_CHECK_LAUNCH();
        finalize_counters<<<ssh_div_up(nc, 128), 128, 0, st>>>(scnt, aband, nc, ncand, isfb, cnt5,
                                                               status + q0);
        SSH_CHECK_LAUNCH();
    }
    return SSH_OK;
}
