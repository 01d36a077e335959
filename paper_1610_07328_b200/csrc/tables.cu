// tables.cu — K4: LSH bucket tables (index.py:141-156, _tables_from_signatures).
//
// Reference: per table j, order = argsort(sig[:, j], kind="stable"); buckets
// are runs of equal keys, ids ascending inside a bucket.  Device: per table,
// an LSD radix sort of (key u64, row u32) with 8-bit digits (8 passes, all L
// tables in one launch per pass via blockIdx.y), stable by construction
// (per-warp ordered ranking with __match_any_sync), tiles staged in shared
// memory so each digit run is written contiguously.  Then a run-length pass
// emits CSR: sorted unique keys, u32 offsets, u32 rows.  Bytes per
// (series, table): 8 B key read + 8 B key + 4 B row written per pass.
#include <limits.h>

#include <algorithm>

#include "common.cuh"

#define RS_THREADS 256
#define RS_WARPS (RS_THREADS / 32)
#define RS_ITEMS 12
#define RS_TILE (RS_THREADS * RS_ITEMS)
#define RS_BINS 256

// sig [N][L] row-major -> keys [L][N], rows [L][N] = 0..N-1
__global__ void rs_transpose(const uint64_t *__restrict__ sig, int64_t N, int L,
                             uint64_t *__restrict__ keys, uint32_t *__restrict__ rows) {
    __shared__ uint64_t tile[32][33];
    int64_t r0 = (int64_t)blockIdx.x * 32;
    int j0 = blockIdx.y * 32;
    int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int yy = ty; yy < 32; yy += 8) {
        int64_t r = r0 + yy;
        int j = j0 + tx;
        if (r < N && j < L) tile[yy][tx] = sig[r * L + j];
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        int j = j0 + yy;
        int64_t r = r0 + tx;
        if (r < N && j < L) {
            keys[(int64_t)j * N + r] = tile[tx][yy];
            rows[(int64_t)j * N + r] = (uint32_t)r;
        }
    }
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
rs_hist(const K *__restrict__ keys, int64_t N, int shift, int ntiles,
        uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[RS_BINS];
    const int j = blockIdx.y;
    const int tile = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const K *k = keys + (int64_t)j * N;
    int64_t base = (int64_t)tile * RS_TILE;
#pragma unroll 4
    for (int it = 0; it < RS_ITEMS; it++) {
        int64_t i = base + it * RS_THREADS + threadIdx.x;
        if (i < N) atomicAdd(&h[(k[i] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    // digit-major layout: hist[j][digit][tile]
    hist[((int64_t)j * RS_BINS + threadIdx.x) * ntiles + tile] = h[threadIdx.x];
}

// exclusive scan of hist[j][*] (RS_BINS * ntiles entries, a multiple of 4), one
// block per table: each warp owns a contiguous segment read with coalesced
// 16-byte loads; pass 1 sums the segments, a warp scan of the 32 totals gives
// the segment offsets, pass 2 scans each 128-entry chunk (in-lane prefix of 4
// + warp shuffle scan) and writes it back.
__global__ void __launch_bounds__(1024) rs_scan(uint32_t *__restrict__ hist, int ntiles) {
    __shared__ uint32_t wtot[32];
    const int j = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint4 *h = reinterpret_cast<uint4 *>(hist + (int64_t)j * RS_BINS * ntiles);
    const int64_t n4 = (int64_t)RS_BINS * ntiles / 4;
    const int64_t seg = ((n4 + 31) / 32 + 31) / 32 * 32;  // uint4 per warp, a multiple of 32
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
    uint32_t run = 0;
    {
        const uint32_t t = wtot[lane];
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        run = __shfl_sync(0xFFFFFFFFu, x - t, w);  // exclusive offset of this warp's segment
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

template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
rs_scatter(const K *__restrict__ kin, const uint32_t *__restrict__ rin, int64_t N,
           int shift, int ntiles, const uint32_t *__restrict__ gofs, K *__restrict__ kout,
           uint32_t *__restrict__ rout) {
    __shared__ uint32_t wcnt[RS_WARPS][RS_BINS];
    __shared__ uint32_t dstart[RS_BINS];
    __shared__ K skey[RS_TILE];
    __shared__ uint32_t srow[RS_TILE];
    const int j = blockIdx.y;
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int e = threadIdx.x; e < RS_WARPS * RS_BINS; e += RS_THREADS) (&wcnt[0][0])[e] = 0;
    __syncthreads();
    const K *k = kin + (int64_t)j * N;
    const uint32_t *r = rin + (int64_t)j * N;
    // warp w owns the contiguous sub-tile [w*32*ITEMS, (w+1)*32*ITEMS) of the tile
    const int64_t wbase = (int64_t)tile * RS_TILE + (int64_t)w * 32 * RS_ITEMS;
    K key[RS_ITEMS];
    uint32_t row[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
#pragma unroll
    for (int it = 0; it < RS_ITEMS; it++) {
        int64_t i = wbase + it * 32 + lane;
        bool valid = i < N;
        key[it] = valid ? k[i] : (K)0;
        row[it] = valid ? r[i] : 0u;
        unsigned d = valid ? (unsigned)((key[it] >> shift) & 0xFF) : RS_BINS;
        unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        unsigned before = valid ? wcnt[w][d] : 0u;
        rank[it] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wcnt[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps per digit; digit totals
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ww++) {
            uint32_t t = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += t;
        }
        dstart[d] = run;
    }
    __syncthreads();
    // exclusive scan over digits (256 entries, one thread each)
    {
        const int d = threadIdx.x;
        uint32_t v = dstart[d];
        // warp-level inclusive scan then cross-warp fixup
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        __shared__ uint32_t wsum[RS_WARPS];
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        uint32_t add = 0;
        for (int ww = 0; ww < w; ww++) add += wsum[ww];
        __syncthreads();
        dstart[d] = x - v + add;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < RS_ITEMS; it++) {
        int64_t i = wbase + it * 32 + lane;
        if (i < N) {
            unsigned d = (unsigned)((key[it] >> shift) & 0xFF);
            uint32_t pos = dstart[d] + wcnt[w][d] + rank[it];
            skey[pos] = key[it];
            srow[pos] = row[it];
        }
    }
    __syncthreads();
    const int64_t tbase = (int64_t)tile * RS_TILE;
    const int nvalid = (int)min((int64_t)RS_TILE, N - tbase);
    const uint32_t *go = gofs + (int64_t)j * RS_BINS * ntiles;
    for (int e = threadIdx.x; e < nvalid; e += RS_THREADS) {
        K kk = skey[e];
        unsigned d = (unsigned)((kk >> shift) & 0xFF);
        int64_t dst = (int64_t)go[(int64_t)d * ntiles + tile] + (e - dstart[d]);
        kout[(int64_t)j * N + dst] = kk;
        rout[(int64_t)j * N + dst] = srow[e];
    }
}

// run starts per tile: count flags
__global__ void __launch_bounds__(RS_THREADS)
rle_count(const uint64_t *__restrict__ keys, int64_t N, int ntiles, uint32_t *__restrict__ bcnt) {
    const int j = blockIdx.y, tile = blockIdx.x;
    const uint64_t *k = keys + (int64_t)j * N;
    uint32_t c = 0;
    for (int it = 0; it < RS_ITEMS; it++) {
        int64_t i = (int64_t)tile * RS_TILE + it * RS_THREADS + threadIdx.x;
        if (i < N && (i == 0 || k[i] != k[i - 1])) c++;
    }
    __shared__ uint32_t red[RS_WARPS];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < RS_WARPS; w++) s += red[w];
        bcnt[(int64_t)j * ntiles + tile] = s;
    }
}

// per table: exclusive scan of tile counts; nb[j] = total
__global__ void rle_scan(uint32_t *__restrict__ bcnt, int ntiles, int64_t *__restrict__ nb) {
    const int j = blockIdx.x;
    if (threadIdx.x != 0) return;
    uint32_t *b = bcnt + (int64_t)j * ntiles;
    uint32_t run = 0;
    for (int t = 0; t < ntiles; t++) {
        uint32_t v = b[t];
        b[t] = run;
        run += v;
    }
    nb[j] = run;
}

__global__ void __launch_bounds__(RS_THREADS)
rle_emit(const uint64_t *__restrict__ keys, int64_t N, int ntiles, const uint32_t *__restrict__ bofs,
         const int64_t *__restrict__ kbase, const int64_t *__restrict__ nb,
         uint64_t *__restrict__ ukeys, uint32_t *__restrict__ offsets) {
    const int j = blockIdx.y, tile = blockIdx.x;
    const uint64_t *k = keys + (int64_t)j * N;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __shared__ uint32_t wsum[RS_WARPS];
    __shared__ uint32_t running;
    if (threadIdx.x == 0) running = bofs[(int64_t)j * ntiles + tile];
    __syncthreads();
    uint64_t *uk = ukeys + kbase[j];
    uint32_t *of = offsets + kbase[j] + j;
    for (int it = 0; it < RS_ITEMS; it++) {
        int64_t i = (int64_t)tile * RS_TILE + it * RS_THREADS + threadIdx.x;
        bool f = i < N && (i == 0 || k[i] != k[i - 1]);
        unsigned m = __ballot_sync(0xFFFFFFFFu, f);
        if (lane == 0) wsum[w] = __popc(m);
        __syncthreads();
        uint32_t before = running;
        for (int ww = 0; ww < w; ww++) before += wsum[ww];
        if (f) {
            uint32_t pos = before + __popc(m & ((1u << lane) - 1u));
            uk[pos] = k[i];
            of[pos] = (uint32_t)i;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t s = 0;
            for (int ww = 0; ww < RS_WARPS; ww++) s += wsum[ww];
            running += s;
        }
        __syncthreads();
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) of[nb[j]] = (uint32_t)N;
}

// Stable LSD radix sort (8 x 8-bit passes) of the L columns of a row-major
// [N][L] u64 matrix, each column independently; rows_out [L][N] receives the
// original row of every sorted position, *keys_sorted the sorted keys [L][N]
// (a ctx scratch slot).  Ties keep ascending row order.
int ssh_sort_columns(ssh_ctx *ctx, const uint64_t *rowmajor, int64_t N, int L, uint32_t *rows_out,
                     uint64_t **keys_sorted, cudaStream_t st) {
    const int ntiles = ssh_div_up(N, RS_TILE);
    size_t kbytes = sizeof(uint64_t) * (size_t)L * N;
    size_t rbytes = sizeof(uint32_t) * (size_t)L * N;
    size_t hbytes = sizeof(uint32_t) * (size_t)L * RS_BINS * ntiles;
    uint64_t *kA = (uint64_t *)ssh_slot(ctx, SLOT_RS_KEYS_A, kbytes, st);
    uint64_t *kB = (uint64_t *)ssh_slot(ctx, SLOT_RS_KEYS_B, kbytes, st);
    uint32_t *rB = (uint32_t *)ssh_slot(ctx, SLOT_RS_ROWS_B, rbytes, st);
    uint32_t *hist = (uint32_t *)ssh_slot(ctx, SLOT_RS_HIST, hbytes, st);
    if (!kA || !kB || !rB || !hist) return SSH_ERR_OOM;
    uint32_t *rA = rows_out;  // 8 passes (even): the sorted rows land back in rA
    {
        dim3 g((unsigned)ssh_div_up(N, 32), (unsigned)ssh_div_up(L, 32));
        rs_transpose<<<g, 256, 0, st>>>(rowmajor, N, L, kA, rA); ssh_count_launch();
    }
    uint64_t *kin = kA, *kout = kB;
    uint32_t *rin = rA, *rout = rB;
    dim3 grid((unsigned)ntiles, (unsigned)L);
    for (int pass = 0; pass < 8; pass++) {
        int shift = 8 * pass;
        rs_hist<uint64_t><<<grid, RS_THREADS, 0, st>>>(kin, N, shift, ntiles, hist); ssh_count_launch();
        rs_scan<<<L, 1024, 0, st>>>(hist, ntiles); ssh_count_launch();
        rs_scatter<uint64_t><<<grid, RS_THREADS, 0, st>>>(kin, rin, N, shift, ntiles, hist, kout, rout);
        ssh_count_launch();
        uint64_t *tk = kin; kin = kout; kout = tk;
        uint32_t *tr = rin; rin = rout; rout = tr;
    }
    SSH_CUDA(cudaGetLastError());
    *keys_sorted = kin;
    return SSH_OK;
}


// sig [N][L] -> full keys kT [L][N], high halves hi [L][N], rows [L][N] = 0..N-1
__global__ void rs_transpose_hi(const uint64_t *__restrict__ sig, int64_t N, int L, uint64_t *__restrict__ keys,
                                uint32_t *__restrict__ hi, uint32_t *__restrict__ rows) {
    __shared__ uint64_t tile[32][33];
    int64_t r0 = (int64_t)blockIdx.x * 32;
    int j0 = blockIdx.y * 32;
    int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int yy = ty; yy < 32; yy += 8) {
        int64_t r = r0 + yy;
        int j = j0 + tx;
        if (r < N && j < L) tile[yy][tx] = sig[r * L + j];
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        int j = j0 + yy;
        int64_t r = r0 + tx;
        if (r < N && j < L) {
            const uint64_t k = tile[tx][yy];
            keys[(int64_t)j * N + r] = k;
            hi[(int64_t)j * N + r] = (uint32_t)(k >> 32);
            rows[(int64_t)j * N + r] = (uint32_t)r;
        }
    }
}

// full keys in (hi-sorted) order; a position whose high half equals the
// previous one's but whose key differs lies in a run of equal high halves that
// needs a fix-up; its bounds come from binary searches on the sorted high
// halves (duplicates are removed by rs_dedup_runs).
__global__ void rs_gather_dirty(const uint64_t *__restrict__ kT, const uint32_t *__restrict__ rows,
                                const uint32_t *__restrict__ hs, int64_t N, int L, uint64_t *__restrict__ ks,
                                int4 *__restrict__ runs, int *__restrict__ nruns, int maxruns) {
    const int j = blockIdx.y;
    const uint64_t *kt = kT + (int64_t)j * N;
    const uint32_t *rw = rows + (int64_t)j * N;
    const uint32_t *h = hs + (int64_t)j * N;
    uint64_t *ko = ks + (int64_t)j * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = kt[rw[i]];
        ko[i] = k;
        if (i == 0 || h[i - 1] != h[i]) continue;
        if (kt[rw[i - 1]] == k) continue;
        const uint32_t hv = h[i];
        int64_t lo = 0, hi = i;  // first position with h == hv
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (h[mid] < hv) lo = mid + 1; else hi = mid;
        }
        const int64_t s = lo;
        lo = i;
        hi = N;  // first position with h > hv
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (h[mid] <= hv) lo = mid + 1; else hi = mid;
        }
        const int slot = atomicAdd(nruns, 1);
        if (slot < maxruns) runs[slot] = make_int4(j, (int)s, (int)(lo - s), 0);
    }
}

// one block: sort the reported runs by (table, start) and drop duplicates
__global__ void __launch_bounds__(1024) rs_dedup_runs(int4 *__restrict__ runs, int *__restrict__ nruns, int maxruns) {
    extern __shared__ int4 rsm[];
    const int n = min(*nruns, maxruns);
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) rsm[i] = i < n ? runs[i] : make_int4(INT_MAX, INT_MAX, 0, 0);
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int idx = threadIdx.x; idx < (P >> 1); idx += blockDim.x) {
                const int i = 2 * idx - (idx & (jj - 1)), l = i + jj;
                const int4 x = rsm[i], y = rsm[l];
                const bool gt = x.x > y.x || (x.x == y.x && x.y > y.y);
                if (gt == ((i & k) == 0)) {
                    rsm[i] = y;
                    rsm[l] = x;
                }
            }
            __syncthreads();
        }
    __shared__ int cnt;
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < n; i++)
            if (i == 0 || rsm[i].x != rsm[i - 1].x || rsm[i].y != rsm[i - 1].y) rsm[c++] = rsm[i];
        cnt = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) runs[i] = rsm[i];
    if (threadIdx.x == 0) *nruns = cnt;
}

// stable sort of each dirty run by the full key (rows ascending inside a
// key): one block per run, 4 LSD passes over the low halves through scratch
__global__ void __launch_bounds__(1024)
rs_fix_runs(uint64_t *__restrict__ ks, uint32_t *__restrict__ rows, int64_t N, const int4 *__restrict__ runs,
            const int *__restrict__ nruns, int maxruns, uint64_t *__restrict__ kscr, uint32_t *__restrict__ rscr) {
    __shared__ uint32_t hist[256], wcnt[32][256];
    __shared__ uint32_t carry[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nr = min(*nruns, maxruns);
    for (int ri = blockIdx.x; ri < nr; ri += gridDim.x) {
        const int4 rr = runs[ri];
        const int64_t off = (int64_t)rr.x * N + rr.y;
        const int len = rr.z;
        uint64_t *ka = ks + off, *kb = kscr + off;
        uint32_t *ra = rows + off, *rb = rscr + off;
        for (int pass = 0; pass < 4; pass++) {
            const int shift = 8 * pass;
            for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < len; i += blockDim.x) atomicAdd(&hist[(ka[i] >> shift) & 0xFF], 1u);
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t run = 0;
                for (int b = 0; b < 256; b++) {
                    carry[b] = run;
                    run += hist[b];
                }
            }
            __syncthreads();
            // tiles of blockDim elements in order; inside a tile: warp order,
            // then lane order (match_any peers) -> stable
            for (int t0 = 0; t0 < len; t0 += blockDim.x) {
                const int i = t0 + threadIdx.x;
                const bool valid = i < len;
                const uint64_t k = valid ? ka[i] : 0ULL;
                const uint32_t rw = valid ? ra[i] : 0u;
                const unsigned d = valid ? (unsigned)((k >> shift) & 0xFF) : 256u;
                for (int b = lane; b < 256; b += 32) wcnt[w][b] = 0;
                __syncthreads();
                const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
                const unsigned lt = (1u << lane) - 1u;
                if (valid && (peers & lt) == 0) wcnt[w][d] = __popc(peers);
                __syncthreads();
                uint32_t before = 0;
                if (valid)
                    for (int ww = 0; ww < w; ww++) before += wcnt[ww][d];
                __syncthreads();
                if (valid) {
                    const uint32_t p = carry[d] + before + __popc(peers & lt);
                    kb[p] = k;
                    rb[p] = rw;
                }
                __syncthreads();
                // advance carries by this tile's digit counts
                for (int b = threadIdx.x; b < 256; b += blockDim.x) {
                    uint32_t c = 0;
                    for (int ww = 0; ww < 32; ww++) c += wcnt[ww][b];
                    carry[b] += c;
                }
                __syncthreads();
            }
            uint64_t *tk = ka; ka = kb; kb = tk;
            uint32_t *tr = ra; ra = rb; rb = tr;
            __syncthreads();
        }
        // 4 passes (even): the result is back in ks/rows
    }
}

// Stable sort of every table column of sig by the full u64 key: 4 LSD passes
// over the high 32 bits (16 B moved per element and pass instead of 24 for
// 8 passes over the whole key), then runs whose keys share the high half but
// differ are fixed up by a per-run stable sort.  rows_out [L][N] receives the
// rows, *keys_sorted [L][N] the full keys (ctx slot).
int ssh_sort_columns_hi(ssh_ctx *ctx, const uint64_t *rowmajor, int64_t N, int L, uint32_t *rows_out,
                        uint64_t **keys_sorted, cudaStream_t st) {
    const int ntiles = ssh_div_up(N, RS_TILE);
    const size_t kbytes = sizeof(uint64_t) * (size_t)L * N;
    const size_t hbytes32 = sizeof(uint32_t) * (size_t)L * N;
    const size_t hbytes = sizeof(uint32_t) * (size_t)L * RS_BINS * ntiles;
    const int MAXRUNS = 8192;  // reported high-half collision runs per build (expected ~10 per table)
    uint64_t *kT = (uint64_t *)ssh_slot(ctx, SLOT_RS_KEYS_A, kbytes, st);
    uint64_t *ks = (uint64_t *)ssh_slot(ctx, SLOT_RS_KEYS_B, kbytes + 2 * hbytes32 + 16 + sizeof(int4) * MAXRUNS, st);
    uint32_t *rB = (uint32_t *)ssh_slot(ctx, SLOT_RS_ROWS_B, hbytes32, st);
    uint32_t *hist = (uint32_t *)ssh_slot(ctx, SLOT_RS_HIST, hbytes, st);
    if (!kT || !ks || !rB || !hist) return SSH_ERR_OOM;
    uint32_t *hA = reinterpret_cast<uint32_t *>(ks + (size_t)L * N);
    uint32_t *hB = hA + (size_t)L * N;
    int *nruns = reinterpret_cast<int *>(hB + (size_t)L * N);
    int4 *runs = reinterpret_cast<int4 *>(reinterpret_cast<unsigned char *>(nruns) + 16);
    uint32_t *rA = rows_out;  // 4 passes (even): the sorted rows land back in rA
    {
        dim3 g((unsigned)ssh_div_up(N, 32), (unsigned)ssh_div_up(L, 32));
        rs_transpose_hi<<<g, 256, 0, st>>>(rowmajor, N, L, kT, hA, rA);
        ssh_count_launch();
    }
    uint32_t *kin = hA, *kout = hB;
    uint32_t *rin = rA, *rout = rB;
    dim3 grid((unsigned)ntiles, (unsigned)L);
    for (int pass = 0; pass < 4; pass++) {
        const int shift = 8 * pass;
        rs_hist<uint32_t><<<grid, RS_THREADS, 0, st>>>(kin, N, shift, ntiles, hist); ssh_count_launch();
        rs_scan<<<L, 1024, 0, st>>>(hist, ntiles); ssh_count_launch();
        rs_scatter<uint32_t><<<grid, RS_THREADS, 0, st>>>(kin, rin, N, shift, ntiles, hist, kout, rout);
        ssh_count_launch();
        uint32_t *tk = kin; kin = kout; kout = tk;
        uint32_t *tr = rin; rin = rout; rout = tr;
    }
    SSH_CUDA(cudaMemsetAsync(nruns, 0, sizeof(int), st));
    {
        dim3 g((unsigned)std::min<int64_t>(ssh_div_up(N, 256), 1024), (unsigned)L);
        rs_gather_dirty<<<g, 256, 0, st>>>(kT, rA, kin, N, L, ks, runs, nruns, MAXRUNS);
        ssh_count_launch();
    }
    int hn = 0;
    SSH_CUDA(cudaMemcpyAsync(&hn, nruns, sizeof(int), cudaMemcpyDeviceToHost, st));
    SSH_CUDA(cudaStreamSynchronize(st));
    if (hn > MAXRUNS)  // more high-half collisions than the fix-up list holds: full-key sort
        return ssh_sort_columns(ctx, rowmajor, N, L, rows_out, keys_sorted, st);
    if (hn == 0) {
        *keys_sorted = ks;
        return SSH_OK;
    }
    SSH_CUDA(cudaFuncSetAttribute(rs_dedup_runs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(int4) * MAXRUNS)));
    rs_dedup_runs<<<1, 1024, sizeof(int4) * MAXRUNS, st>>>(runs, nruns, MAXRUNS);
    ssh_count_launch();
    // scratch for the fix-ups: the transposed keys and the spare row buffer
    rs_fix_runs<<<256, 1024, 0, st>>>(ks, rA, N, runs, nruns, MAXRUNS, kT, rB);
    ssh_count_launch();
    SSH_CUDA(cudaGetLastError());
    *keys_sorted = ks;
    return SSH_OK;
}

// Per-slot ranks of ln_a1 (order by (value, token)): rank[token][slot].
__global__ void lna1_orderable_kernel(const double *__restrict__ lna1, size_t n, uint64_t *__restrict__ keys) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        uint64_t b = (uint64_t)__double_as_longlong(lna1[e]);
        keys[e] = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
    }
}

template <typename RT>
__global__ void rank_scatter_kernel(const uint32_t *__restrict__ rows, int64_t T, int S, RT *__restrict__ rank) {
    const int64_t n = T * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / T, p = e - j * T;
        rank[(int64_t)rows[e] * S + j] = (RT)p;
    }
}

// ln_a and t of a count-2 token (wmh.py:74-76, reference op order):
// t = floor(fl(fl(ln 2 / r) + beta)), ln_a = (ln_c - r (t - beta)) - r.
__device__ __forceinline__ double lna_count2(double rr, double lnc, double b, double ln2, double &t) {
    t = floor(__dadd_rn(__ddiv_rn(ln2, rr), b));
    const double lny = __dmul_rn(rr, __dsub_rn(t, b));
    return __dsub_rn(__dsub_rn(lnc, lny), rr);
}

// Orderable keys of the combined (token, count in {1, 2}) rows: row 2 tok + (count - 1).
__global__ void comb_orderable_kernel(const double *__restrict__ r, const double *__restrict__ lnc,
                                      const double *__restrict__ beta, const double *__restrict__ lna1,
                                      double ln2, size_t n, int S, uint64_t *__restrict__ keys) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const size_t tok = e / S, s = e - tok * S;
        double t2;
        const double v2 = lna_count2(r[e], lnc[e], beta[e], ln2, t2);
        const double v[2] = {lna1[e], v2};
#pragma unroll
        for (int c = 0; c < 2; c++) {
            const uint64_t bb = (uint64_t)__double_as_longlong(v[c]);
            keys[(2 * tok + c) * S + s] = (bb >> 63) ? ~bb : (bb | 0x8000000000000000ULL);
        }
    }
}

// Order-free CWS tables (signature.cu, cws_fast): padded u16 ranks per
// combined row (count-1 and count-2 tokens share one per-slot order by
// (ln_a, row) = (ln_a, token): a token has one count per series), the winner
// record per (slot, rank), and the packed variates.
__global__ void rank_fast_kernel(const uint32_t *__restrict__ rows, int64_t T2, int S, int SP,
                                 const double *__restrict__ r, const double *__restrict__ lnc,
                                 const double *__restrict__ beta, const double *__restrict__ lna1,
                                 double ln2, uint16_t *__restrict__ rankp, uint4 *__restrict__ byrank,
                                 double *__restrict__ rlcb) {
    const int64_t n2 = T2 * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / T2, p = e - j * T2;
        const uint32_t row = rows[e];
        const uint32_t tok = row >> 1;
        rankp[(int64_t)row * SP + j] = (uint16_t)p;
        const int64_t te = (int64_t)tok * S + j;
        double v, t;
        if (row & 1u) {
            v = lna_count2(r[te], lnc[te], beta[te], ln2, t);
        } else {
            v = lna1[te];
            t = floor(beta[te]);  // beta in (0, 1]: 0 or 1
        }
        byrank[e] = make_uint4((uint32_t)__double2loint(v), (uint32_t)__double2hiint(v),
                               tok | ((uint32_t)t << 16), 0u);
    }
    const int64_t n = (T2 / 2) * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const double rr = r[e];
        double *q = rlcb + 4 * e;
        q[0] = rr;
        q[1] = __drcp_rn(rr);
        q[2] = lnc[e];
        q[3] = beta[e];
    }
}

// {ln_a, t} for the all-zero and all-one tokens at every count (wmh.py:74-76,
// reference op order): e = (which * (maxc + 1) + count) * S + slot.
__global__ void edge_table_kernel(const double *__restrict__ r, const double *__restrict__ lnc,
                                  const double *__restrict__ beta, const double *__restrict__ lnw,
                                  int n, int S, int maxc, double2 *__restrict__ out) {
    const int64_t total = 2LL * (maxc + 1) * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(e % S);
        const int64_t wc = e / S;
        const int c = (int)(wc % (maxc + 1));
        const int which = (int)(wc / (maxc + 1));
        if (c < 1) { out[e] = make_double2(INFINITY, 0.0); continue; }
        const int64_t te = (int64_t)(which ? ((1 << n) - 1) : 0) * S + s;
        const double rr = r[te], b = beta[te];
        const double t = floor(__dadd_rn(__ddiv_rn(lnw[c], rr), b));
        const double lny = __dmul_rn(rr, __dsub_rn(t, b));
        out[e] = make_double2(__dsub_rn(__dsub_rn(lnc[te], lny), rr), t);
    }
}

static int pick_rank_ql(int S) {
    const int q = (S + 15) / 16;
    if (q <= 6) return q;
    if (q <= 8) return 8;
    return 0;
}

int ssh_build_ranks(ssh_ctx *ctx, cudaStream_t st) {
    const int64_t T = (int64_t)1 << ctx->p.n;
    const int S = ctx->S;
    const size_t n = (size_t)T * S;
    uint64_t *keys = nullptr;
    uint32_t *rows = nullptr;
    SSH_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * n));
    SSH_CUDA(cudaMalloc(&rows, sizeof(uint32_t) * n));
    int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)ctx->num_sms * 16);
    lna1_orderable_kernel<<<grid, 256, 0, st>>>(ctx->d_lna1, n, keys);
    SSH_CHECK_LAUNCH();
    uint64_t *sorted = nullptr;
    int rc = ssh_sort_columns(ctx, keys, T, S, rows, &sorted, st);
    if (rc == SSH_OK) {
        if (ctx->p.n <= 16) {
            rank_scatter_kernel<uint16_t><<<grid, 256, 0, st>>>(rows, T, S, (uint16_t *)ctx->d_rank);
        } else {
            rank_scatter_kernel<uint32_t><<<grid, 256, 0, st>>>(rows, T, S, (uint32_t *)ctx->d_rank);
        }
        ssh_count_launch();
        const int ql = ctx->p.n <= 15 ? pick_rank_ql(S) : 0;
        if (ql > 0) {
            const int SP = 16 * ql;
            const int64_t T2 = 2 * T;
            const size_t n2 = (size_t)T2 * S;
            uint64_t *keys2 = nullptr;
            uint32_t *rows2 = nullptr;
            cudaError_t e = cudaMalloc(&keys2, sizeof(uint64_t) * n2);
            if (e == cudaSuccess) e = cudaMalloc(&rows2, sizeof(uint32_t) * n2);
            if (e == cudaSuccess) {
                comb_orderable_kernel<<<grid, 256, 0, st>>>(ctx->d_r, ctx->d_lnc, ctx->d_beta, ctx->d_lna1,
                                                            ctx->h_ln2, n, S, keys2);
                ssh_count_launch();
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) {
                uint64_t *sorted2 = nullptr;
                const int rc2 = ssh_sort_columns(ctx, keys2, T2, S, rows2, &sorted2, st);
                if (rc2 != SSH_OK) e = cudaErrorUnknown;
            }
            if (e == cudaSuccess) e = cudaMalloc(&ctx->d_rankp, sizeof(uint16_t) * (size_t)T2 * SP);
            if (e == cudaSuccess) e = cudaMalloc(&ctx->d_byrank, sizeof(uint4) * n2);
            if (e == cudaSuccess) e = cudaMalloc(&ctx->d_rlcb, 4 * sizeof(double) * n);
            const char *ee = getenv("SSH_CWS_EDGE");
            const bool wante = !(ee && ee[0] == '0');
            const size_t nedge = 2 * (size_t)(ctx->max_count + 1) * S;
            if (e == cudaSuccess && wante) e = cudaMalloc(&ctx->d_edge, 2 * sizeof(double) * nedge);
            if (e == cudaSuccess && wante) {
                const int g2 = (int)std::min<size_t>((nedge + 255) / 256, (size_t)ctx->num_sms * 8);
                edge_table_kernel<<<g2, 256, 0, st>>>(ctx->d_r, ctx->d_lnc, ctx->d_beta, ctx->d_lnw, ctx->p.n, S,
                                                      ctx->max_count, reinterpret_cast<double2 *>(ctx->d_edge));
                ssh_count_launch();
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaMemsetAsync(ctx->d_rankp, 0xFF, sizeof(uint16_t) * (size_t)T2 * SP, st);
            if (e == cudaSuccess) {
                const int g3 = (int)std::min<size_t>((n2 + 255) / 256, (size_t)ctx->num_sms * 16);
                rank_fast_kernel<<<g3, 256, 0, st>>>(rows2, T2, S, SP, ctx->d_r, ctx->d_lnc, ctx->d_beta,
                                                     ctx->d_lna1, ctx->h_ln2, ctx->d_rankp, ctx->d_byrank,
                                                     ctx->d_rlcb);
                ssh_count_launch();
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            cudaFree(keys2);
            cudaFree(rows2);
            if (e != cudaSuccess) rc = ssh_cuda_fail(e, "ssh_build_ranks(fast tables)", __FILE__, __LINE__);
            else ctx->rank_ql = ql;
        }
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess && rc == SSH_OK) rc = ssh_cuda_fail(e, "ssh_build_ranks", __FILE__, __LINE__);
    }
    cudaFree(keys);
    cudaFree(rows);
    return rc;
}

extern "C" int ssh_index_build(ssh_ctx *ctx, const uint64_t *sig, int64_t N, int64_t id_base,
                               ssh_index **out, void *stream) {
    SSH_REQUIRE(ctx && out, SSH_ERR_INVALID, "ssh_index_build: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_index_build: ssh_ctx_set_params not called");
    SSH_REQUIRE(N >= 1 && N < (int64_t)0xFFFFFFFF, SSH_ERR_INVALID,
                "ssh_index_build: N=%lld outside [1, 2^32-1)", (long long)N);
    SSH_REQUIRE(sig != nullptr, SSH_ERR_INVALID, "ssh_index_build: sig is NULL");
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int L = ctx->p.L;
    const int ntiles = ssh_div_up(N, RS_TILE);
    ssh_index *ix = new ssh_index();
    ix->L = L; ix->N = N; ix->id_base = id_base; ix->device = ctx->device;
    int rc = SSH_OK;
    cudaError_t e;
    uint64_t *kin = nullptr;
    size_t rbytes = sizeof(uint32_t) * (size_t)L * N;
    e = cudaMallocAsync((void **)&ix->ids, rbytes, st);
    if (e != cudaSuccess) { delete ix; return ssh_cuda_fail(e, "cudaMallocAsync(ids)", __FILE__, __LINE__); }
    rc = ssh_sort_columns_hi(ctx, sig, N, L, ix->ids, &kin, st);
    if (rc) goto fail;
    {
    uint32_t *hist = (uint32_t *)ctx->slot_ptr[SLOT_RS_HIST];
    dim3 grid((unsigned)ntiles, (unsigned)L);
    // sorted keys in kin, rows in ix->ids
    // run-length encode -> CSR
    e = cudaMallocAsync((void **)&ix->d_nb, sizeof(int64_t) * 2 * L, st);
    if (e != cudaSuccess) { rc = ssh_cuda_fail(e, "cudaMallocAsync(nb)", __FILE__, __LINE__); goto fail; }
    ix->d_kbase = ix->d_nb + L;
    rle_count<<<grid, RS_THREADS, 0, st>>>(kin, N, ntiles, hist); ssh_count_launch();
    rle_scan<<<L, 32, 0, st>>>(hist, ntiles, ix->d_nb); ssh_count_launch();
    ix->h_nb = new int64_t[2 * L];
    ix->h_kbase = ix->h_nb + L;
    e = cudaMemcpyAsync(ix->h_nb, ix->d_nb, sizeof(int64_t) * L, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { rc = ssh_cuda_fail(e, "bucket count readback", __FILE__, __LINE__); goto fail; }
    {
        int64_t tot = 0;
        for (int j = 0; j < L; j++) { ix->h_kbase[j] = tot; tot += ix->h_nb[j]; }
        ix->total_buckets = tot;
        e = cudaMemcpyAsync(ix->d_kbase, ix->h_kbase, sizeof(int64_t) * L, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMallocAsync((void **)&ix->keys, sizeof(uint64_t) * tot, st);
        if (e == cudaSuccess) e = cudaMallocAsync((void **)&ix->offsets, sizeof(uint32_t) * (tot + L), st);
        if (e != cudaSuccess) { rc = ssh_cuda_fail(e, "CSR allocation", __FILE__, __LINE__); goto fail; }
        rle_emit<<<grid, RS_THREADS, 0, st>>>(kin, N, ntiles, hist, ix->d_kbase, ix->d_nb,
                                              ix->keys, ix->offsets);
        ssh_count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) { rc = ssh_cuda_fail(e, "rle_emit", __FILE__, __LINE__); goto fail; }
    }
    }
    ssh_index_touch(ix, st);
    *out = ix;
    return SSH_OK;
fail:
    cudaStreamSynchronize(st);
    ssh_index_destroy(ix);
    return rc;
}

void ssh_index_touch(const ssh_index *ix, cudaStream_t st) {
    ssh_index *m = const_cast<ssh_index *>(ix);
    if (!m->last_use && cudaEventCreateWithFlags(&m->last_use, cudaEventDisableTiming) != cudaSuccess) {
        m->last_use = nullptr;
        return;
    }
    cudaEventRecord(m->last_use, st);
}

extern "C" int ssh_index_destroy(ssh_index *ix) {
    if (!ix) return SSH_OK;
    cudaSetDevice(ix->device);
    // stream-ordered frees on the legacy stream: memory returns to the pool
    // without a device-wide synchronisation, after the index's last use on
    // whatever stream the caller ran it (ssh_index_touch)
    cudaStream_t st = 0;
    if (ix->last_use) {
        cudaStreamWaitEvent(st, ix->last_use, 0);
        cudaEventDestroy(ix->last_use);
    }
    if (ix->keys) cudaFreeAsync(ix->keys, st);
    if (ix->offsets) cudaFreeAsync(ix->offsets, st);
    if (ix->ids) cudaFreeAsync(ix->ids, st);
    if (ix->d_nb) cudaFreeAsync(ix->d_nb, st);
    if (ix->rec) cudaFreeAsync(ix->rec, st);
    if (ix->codes) cudaFreeAsync(ix->codes, st);
    if (ix->d_sketch_stats) cudaFreeAsync(ix->d_sketch_stats, st);
    delete[] ix->h_nb;
    delete ix;
    return SSH_OK;
}

extern "C" int ssh_index_num_buckets(const ssh_index *ix, int table, int64_t *nb) {
    SSH_REQUIRE(ix && nb, SSH_ERR_INVALID, "ssh_index_num_buckets: NULL argument");
    SSH_REQUIRE(table >= 0 && table < ix->L, SSH_ERR_INVALID, "table %d out of range", table);
    *nb = ix->h_nb[table];
    return SSH_OK;
}

extern "C" int64_t ssh_index_size(const ssh_index *ix) { return ix ? ix->N : -1; }

extern "C" int ssh_index_sketch_stats(const ssh_index *ix, int64_t *out2, void *stream) {
    SSH_REQUIRE(ix && out2, SSH_ERR_INVALID, "ssh_index_sketch_stats: NULL argument");
    out2[0] = out2[1] = 0;
    if (!ix->d_sketch_stats) return SSH_OK;  // built from signatures: no sketch ran
    SSH_CUDA(cudaSetDevice(ix->device));
    cudaStream_t st = (cudaStream_t)stream;
    SSH_CUDA(cudaMemcpyAsync(out2, ix->d_sketch_stats, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SSH_CUDA(cudaStreamSynchronize(st));
    return SSH_OK;
}

extern "C" int ssh_index_export(const ssh_index *ix, int table, uint64_t *keys, int64_t *offsets,
                                int64_t *ids, void *stream) {
    SSH_REQUIRE(ix && keys && offsets && ids, SSH_ERR_INVALID, "ssh_index_export: NULL argument");
    SSH_REQUIRE(table >= 0 && table < ix->L, SSH_ERR_INVALID, "table %d out of range", table);
    SSH_CUDA(cudaSetDevice(ix->device));
    cudaStream_t st = (cudaStream_t)stream;
    int64_t nb = ix->h_nb[table], kb = ix->h_kbase[table], N = ix->N;
    uint32_t *of = new uint32_t[nb + 1];
    uint32_t *rw = new uint32_t[N];
    cudaError_t e = cudaMemcpyAsync(keys, ix->keys + kb, sizeof(uint64_t) * nb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(of, ix->offsets + kb + table, sizeof(uint32_t) * (nb + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(rw, ix->ids + (int64_t)table * N, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        for (int64_t b = 0; b <= nb; b++) offsets[b] = of[b];
        for (int64_t i = 0; i < N; i++) ids[i] = (int64_t)rw[i] + ix->id_base;
    }
    delete[] of;
    delete[] rw;
    if (e != cudaSuccess) return ssh_cuda_fail(e, "ssh_index_export", __FILE__, __LINE__);
    return SSH_OK;
}

// K1 -> K4 in one call: build_index (index.py:159-172), plus the rerank
// summaries of every row (they depend only on X: computed on the side stream,
// concurrently with the latency-bound signature kernels, joined at the end).
extern "C" int ssh_build_index(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, int64_t id_base,
                               uint64_t *sig_out, ssh_index **out, void *stream) {
    SSH_REQUIRE(ctx && X && out, SSH_ERR_INVALID, "ssh_build_index: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_build_index: ssh_ctx_set_params not called");
    SSH_REQUIRE(N >= 1 && ld >= ctx->p.m, SSH_ERR_INVALID, "ssh_build_index: bad shape N=%lld ld=%lld",
                (long long)N, (long long)ld);
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *bits = (uint64_t *)ssh_slot(ctx, SLOT_BITS, sizeof(uint64_t) * (size_t)N * ctx->words, st);
    uint64_t *sig = sig_out ? sig_out
                            : (uint64_t *)ssh_slot(ctx, SLOT_SIG, sizeof(uint64_t) * (size_t)N * ctx->p.L, st);
    if (!bits || !sig) return SSH_ERR_OOM;
    ssh_index summ;
    summ.N = N;
    // allocate on the caller's stream (where earlier indexes were freed, so the
    // pool reuses their memory), then summarise on the side stream
    int rc = ssh_alloc_summaries(ctx, &summ, N, st);
    if (rc) return rc;
    int64_t *skst = nullptr;  // near-zero sign-tie counters of this build (ssh_index_sketch_stats)
    if (cudaMallocAsync((void **)&skst, 2 * sizeof(int64_t), st) != cudaSuccess ||
        cudaMemsetAsync(skst, 0, 2 * sizeof(int64_t), st) != cudaSuccess) {
        if (skst) cudaFreeAsync(skst, st);
        cudaFreeAsync(summ.rec, st);
        cudaFreeAsync(summ.codes, st);
        return ssh_cuda_fail(cudaErrorMemoryAllocation, "cudaMallocAsync(sketch stats)", __FILE__, __LINE__);
    }
    // sketch + CWS first (CWS fills every SM), then the summaries on the side
    // stream run alongside the bucket-table sorts (memory-bound kernels with
    // host syncs for the bucket counts between them); joined at the end
    rc = ssh_launch_sketch(ctx, X, N, ld, bits, skst, st);
    if (rc == SSH_OK)
        rc = ssh_launch_shingle_cws(ctx, bits, nullptr, nullptr, nullptr, N, nullptr, nullptr, nullptr,
                                    nullptr, sig, SIG_MODE_FUSED, st);
    if (rc == SSH_OK) rc = cudaEventRecord(ctx->ev_fork, st) == cudaSuccess ? SSH_OK : SSH_ERR_CUDA;
    if (rc == SSH_OK) rc = cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0) == cudaSuccess ? SSH_OK : SSH_ERR_CUDA;
    if (rc == SSH_OK) rc = ssh_launch_summaries_rows(ctx, &summ, X, 0, N, ld, ctx->side);
    if (rc == SSH_OK) rc = cudaEventRecord(ctx->ev_join, ctx->side) == cudaSuccess ? SSH_OK : SSH_ERR_CUDA;
    if (rc == SSH_OK) rc = ssh_index_build(ctx, sig, N, id_base, out, stream);
    if (rc == SSH_OK) rc = cudaStreamWaitEvent(st, ctx->ev_join, 0) == cudaSuccess ? SSH_OK : SSH_ERR_CUDA;
    if (rc != SSH_OK) {
        cudaStreamWaitEvent(st, ctx->ev_join, 0);
        if (summ.rec) cudaFreeAsync(summ.rec, st);
        if (summ.codes) cudaFreeAsync(summ.codes, st);
        cudaFreeAsync(skst, st);
        return rc;
    }
    (*out)->d_sketch_stats = skst;
    (*out)->rec = summ.rec;
    (*out)->codes = summ.codes;
    (*out)->seg = summ.seg;
    (*out)->nseg = summ.nseg;
    (*out)->mp = summ.mp;
    (*out)->cstride = summ.cstride;
    ssh_index_touch(*out, st);
    return SSH_OK;
}

// build_index from HOST series (index.py:159-172 with the H2D copy inside):
// rows are copied in chunks on the copy stream into X_dev (the caller's device
// buffer, N x ld f32, which the index then uses for DTW) while the previous
// chunk is sketched, signed and summarised on `stream`; bucket tables last.
extern "C" int ssh_build_index_host(ssh_ctx *ctx, const float *X_host, int64_t N, int64_t ld, int64_t id_base,
                                    float *X_dev, uint64_t *sig_out, ssh_index **out, void *stream) {
    SSH_REQUIRE(ctx && X_host && X_dev && sig_out && out, SSH_ERR_INVALID, "ssh_build_index_host: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_build_index_host: ssh_ctx_set_params not called");
    SSH_REQUIRE(N >= 1 && ld >= ctx->p.m, SSH_ERR_INVALID, "ssh_build_index_host: bad shape N=%lld ld=%lld",
                (long long)N, (long long)ld);
    SSH_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t CH = 65536;
    uint64_t *bits = (uint64_t *)ssh_slot(ctx, SLOT_BITS, sizeof(uint64_t) * (size_t)std::min(N, CH) * ctx->words, st);
    if (!bits) return SSH_ERR_OOM;
    ssh_index summ;
    summ.N = N;
    int rc = ssh_alloc_summaries(ctx, &summ, N, st);
    if (rc) return rc;
    int64_t *skst = nullptr;
    if (cudaMallocAsync((void **)&skst, 2 * sizeof(int64_t), st) != cudaSuccess ||
        cudaMemsetAsync(skst, 0, 2 * sizeof(int64_t), st) != cudaSuccess) {
        if (skst) cudaFreeAsync(skst, st);
        cudaFreeAsync(summ.rec, st);
        cudaFreeAsync(summ.codes, st);
        return ssh_cuda_fail(cudaErrorMemoryAllocation, "cudaMallocAsync(sketch stats)", __FILE__, __LINE__);
    }
    // the copy stream may only write X_dev after the caller's prior work on it
    SSH_CUDA(cudaEventRecord(ctx->ev_fork, st));
    SSH_CUDA(cudaStreamWaitEvent(ctx->copy, ctx->ev_fork, 0));
    for (int64_t r0 = 0; r0 < N && rc == SSH_OK; r0 += CH) {
        const int64_t n = std::min(CH, N - r0);
        cudaError_t e = cudaMemcpyAsync(X_dev + r0 * ld, X_host + r0 * ld, sizeof(float) * (size_t)(n * ld),
                                        cudaMemcpyHostToDevice, ctx->copy);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_copy, ctx->copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->ev_copy, 0);
        if (e != cudaSuccess) {
            rc = ssh_cuda_fail(e, "ssh_build_index_host copy", __FILE__, __LINE__);
            break;
        }
        const float *Xc = X_dev + r0 * ld;
        rc = ssh_launch_sketch(ctx, Xc, n, ld, bits, skst, st);
        if (rc == SSH_OK)
            rc = ssh_launch_shingle_cws(ctx, bits, nullptr, nullptr, nullptr, n, nullptr, nullptr, nullptr,
                                        nullptr, sig_out + r0 * ctx->p.L, SIG_MODE_FUSED, st);
        if (rc == SSH_OK) rc = ssh_launch_summaries_rows(ctx, &summ, Xc, r0, n, ld, st);
    }
    if (rc == SSH_OK) rc = ssh_index_build(ctx, sig_out, N, id_base, out, stream);
    if (rc != SSH_OK) {
        if (summ.rec) cudaFreeAsync(summ.rec, st);
        if (summ.codes) cudaFreeAsync(summ.codes, st);
        cudaFreeAsync(skst, st);
        return rc;
    }
    (*out)->d_sketch_stats = skst;
    (*out)->rec = summ.rec;
    (*out)->codes = summ.codes;
    (*out)->seg = summ.seg;
    (*out)->nseg = summ.nseg;
    (*out)->mp = summ.mp;
    (*out)->cstride = summ.cstride;
    ssh_index_touch(*out, st);
    return SSH_OK;
}

// An index without bucket tables (exact search over the whole shard): the
// series summaries only.  ssh_query_batch treats every query's R as the shard.
extern "C" int ssh_index_create_bare(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, int64_t id_base,
                                     ssh_index **out, void *stream) {
    SSH_REQUIRE(ctx && X && out, SSH_ERR_INVALID, "ssh_index_create_bare: NULL argument");
    SSH_REQUIRE(ctx->have_params, SSH_ERR_STATE, "ssh_index_create_bare: params not set");
    SSH_REQUIRE(N >= 1 && N < (int64_t)0xFFFFFFFF && ld >= ctx->p.m, SSH_ERR_INVALID,
                "ssh_index_create_bare: bad shape N=%lld ld=%lld", (long long)N, (long long)ld);
    SSH_CUDA(cudaSetDevice(ctx->device));
    ssh_index *ix = new ssh_index();
    ix->L = ctx->p.L;
    ix->N = N;
    ix->id_base = id_base;
    ix->device = ctx->device;
    int rc = ssh_launch_summaries(ctx, ix, X, N, ld, (cudaStream_t)stream);
    if (rc != SSH_OK) {
        ssh_index_destroy(ix);
        return rc;
    }
    ssh_index_touch(ix, (cudaStream_t)stream);
    *out = ix;
    return SSH_OK;
}
