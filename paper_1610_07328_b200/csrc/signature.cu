// signature.cu — K2 shingle + K3 consistent weighted sampling (one warp per series).
//
// K2 (shingle.py:56-75, index.py:118): tokens t_i = bits[i..i+n-1] with the
// first bit most significant, and their multiplicities.  A warp extracts its
// series' T tokens from the packed bit row (word shuffles + __brev) and
// counts them in a per-warp shared-memory hash set (atomicCAS/atomicAdd),
// then compacts the distinct (token, count) pairs with ballots.  The stage
// API (ssh_shingle) additionally bitonic-sorts them to reproduce
// np.unique's ascending order; the fused build path does not need the order.
//
// K3 (wmh.py:52-81 + signature(concat=K) wmh.py:107-125): for every slot s
// of S = K*L, argmin over the distinct tokens of
//     ln_a = ln_c - r*(floor(ln_w/r + beta) - beta) - r
// with ties broken toward the lowest token (np.argmin's first occurrence over
// the sorted tokens), key = mix64(tok ^ mix64(t ^ SALT_KEY)), then the K-fold
// acc = mix64(acc ^ key).  The variates come from host tables (np.log bits);
// the device does only IEEE operations in the reference order with explicit
// _rn intrinsics, so keys are bit-exact:
//   * count-1 tokens (76-84% of all) read the precomputed ln_a1 table;
//   * larger counts need t = floor(fl(fl(ln_w / r) + beta)).  It is taken from
//     an approximate quotient (rcp.approx + two Newton steps, relative error
//     < 2^-48) whenever that sum is farther than 1e-12 (relative) from an
//     integer, which pins the floor; otherwise the exact IEEE division is
//     evaluated.  ln_y and ln_a then follow with _rn operations.
// Lanes own slots s = lane + 32*i, so every gather is a contiguous 256-byte
// segment of the [token][slot] tables (L2-resident: 2^15 x 80 x 8 B = 21 MB).
#include <float.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

#define SG_WARPS 8
#ifndef SG_FAST_MINB
#define SG_FAST_MINB 4
#endif
#ifndef SG_CWS_U2
#define SG_CWS_U2 0
#endif
#define SG_EMPTY 0xFFFFFFFFu

struct SigArgs {
    const uint64_t *bits;
    const uint32_t *tok_in;
    const uint16_t *cnt_in;
    const int32_t *len_in;
    uint32_t *tok_out;
    uint16_t *cnt_out;
    int32_t *len_out;
    uint64_t *keys_out;
    uint64_t *sig_out;
    const double *lna1, *tr, *tlnc, *tbeta, *lnw;
    const void *rank;  // per-slot rank of ln_a1: u16 (n <= 16) or u32
    const uint16_t *rankp;  // order-free path: u16 ranks, 16*QL slots per (2 token + count - 1) row
    const uint4 *byrank;    // order-free path: (slot << (n+1) | rank) -> {ln_a, token | t << 16}, counts 1-2
    const double2 *rlcb;    // order-free path: (token, slot) -> {r, 1/r}, {ln c, beta}
    const double2 *edge;    // order-free path: (token 0 | 2^n-1, count, slot) -> {ln_a, t} (or null)
    int maxc;
    int64_t N;
    int words, nb, n, T, P2, H, S, L, K;
    int warp_smem;  // bytes per warp
};

__global__ void lna1_kernel(const double *__restrict__ r, const double *__restrict__ lnc,
                            const double *__restrict__ beta, double *__restrict__ out,
                            size_t n) {
    // ln_w = log(1) = 0: t = floor(0/r + beta) = floor(beta) (beta may round to 1.0),
    // ln_a = (ln_c - r*(t - beta)) - r  — wmh.py:74-76 with the same op order.
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x) {
        double b = beta[e], rr = r[e];
        double t = floor(__dadd_rn(__ddiv_rn(0.0, rr), b));
        double lny = __dmul_rn(rr, __dsub_rn(t, b));
        out[e] = __dsub_rn(__dsub_rn(lnc[e], lny), rr);
    }
}

int ssh_launch_lna1(ssh_ctx *ctx, cudaStream_t st) {
    size_t n = ctx->tab_entries;
    int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)ctx->num_sms * 16);
    lna1_kernel<<<grid, 256, 0, st>>>(ctx->d_r, ctx->d_lnc, ctx->d_beta, ctx->d_lna1, n);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

struct WarpSmem {
    uint64_t *keys;     // S
    uint32_t *hkey;     // H   (hash set; aliases the sort buffer)
    uint32_t *hcnt;     // H
    uint32_t *sortbuf;  // P2  (ssh_shingle only)
    uint32_t *utok;     // T   distinct tokens (stage API)
    uint32_t *ukey;     // T   packed (token << 12 | count), aliases utok
    uint16_t *ucnt;     // T
    uint16_t *ustart;   // T+1 (ssh_shingle only)
};

__host__ __device__ __forceinline__ int warp_smem_bytes(int S, int P2, int H, int T) {
    int region = 8 * H > 4 * P2 ? 8 * H : 4 * P2;
    int b = 8 * S + region + 4 * T + 2 * T + 2 * (T + 1);
    return (b + 15) & ~15;
}

__device__ __forceinline__ WarpSmem carve(unsigned char *base, const SigArgs &a) {
    WarpSmem w;
    unsigned char *p = base;
    w.keys = reinterpret_cast<uint64_t *>(p); p += 8 * a.S;
    w.hkey = reinterpret_cast<uint32_t *>(p);
    w.hcnt = w.hkey + a.H;
    w.sortbuf = w.hkey;
    p += (8 * a.H > 4 * a.P2) ? 8 * a.H : 4 * a.P2;
    w.utok = reinterpret_cast<uint32_t *>(p); p += 4 * a.T;
    w.ukey = w.utok;
    w.ucnt = reinterpret_cast<uint16_t *>(p); p += 2 * a.T;
    w.ustart = reinterpret_cast<uint16_t *>(p);
    return w;
}

// token i of the packed bit row: bits i..i+n-1, first bit most significant
__device__ __forceinline__ uint32_t token_at(uint64_t myword, int i, int words, int n) {
    const int wi = min(i >> 6, 31);
    const int sh = i & 63;
    uint64_t w0 = __shfl_sync(0xFFFFFFFFu, myword, wi);
    uint64_t w1 = __shfl_sync(0xFFFFFFFFu, myword, min(wi + 1, 31));
    if (wi + 1 >= words) w1 = 0ULL;
    uint64_t v = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
    const uint32_t nmask = (n == 32) ? 0xFFFFFFFFu : ((1u << n) - 1u);
    return __brev((uint32_t)v & nmask) >> (32 - n);
}

// Warp bitonic sort of 32*V u32 keys held V per lane (element e = lane*V + v).
template <int V>
__device__ __forceinline__ void warp_sort_regs(uint32_t (&x)[V], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * V; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= V) {
                const int lj = j / V;
                const bool lower = (lane & lj) == 0;
#pragma unroll
                for (int v = 0; v < V; v++) {
                    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x[v], lj);
                    const bool up = ((lane * V + v) & k) == 0;
                    x[v] = (lower == up) ? min(x[v], y) : max(x[v], y);
                }
            } else {
#pragma unroll
                for (int v = 0; v < V; v++) {
                    if ((v & j) == 0) {
                        const bool up = ((lane * V + v) & k) == 0;
                        const uint32_t p = x[v], q = x[v + j];
                        x[v] = up ? min(p, q) : max(p, q);
                        x[v + j] = up ? max(p, q) : min(p, q);
                    }
                }
            }
        }
    }
}

template <int V>
__device__ __forceinline__ void sort_keys_regs(uint32_t *keys, int D, int lane) {
    uint32_t x[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        const int e = lane * V + v;
        x[v] = e < D ? keys[e] : 0xFFFFFFFFu;
    }
    __syncwarp();
    warp_sort_regs<V>(x, lane);
#pragma unroll
    for (int v = 0; v < V; v++) {
        const int e = lane * V + v;
        if (e < D) keys[e] = x[v];
    }
    __syncwarp();
}

// ascending sort of D packed keys in smem (buf: scratch of P2 >= D entries)
__device__ void sort_keys(uint32_t *keys, int D, uint32_t *buf, int P2, int lane) {
    if (D <= 1) return;
    if (D <= 32) { sort_keys_regs<1>(keys, D, lane); return; }
    if (D <= 64) { sort_keys_regs<2>(keys, D, lane); return; }
    if (D <= 128) { sort_keys_regs<4>(keys, D, lane); return; }
    if (D <= 256) { sort_keys_regs<8>(keys, D, lane); return; }
    int P = 512;
    while (P < D) P <<= 1;
    for (int e = lane; e < P; e += 32) buf[e] = e < D ? keys[e] : 0xFFFFFFFFu;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = lane; idx < (P >> 1); idx += 32) {
                int i = 2 * idx - (idx & (j - 1));
                int l = i + j;
                uint32_t x = buf[i], y = buf[l];
                bool up = (i & k) == 0;
                if ((x > y) == up) {
                    buf[i] = y;
                    buf[l] = x;
                }
            }
            __syncwarp();
        }
    }
    for (int e = lane; e < D; e += 32) keys[e] = buf[e];
    __syncwarp();
}


// Distinct tokens + counts by a register sort (T <= 32 V): the row's bit
// words are staged in shared memory, each lane builds V tokens (element
// e = lane * V + v), a warp bitonic sort orders them, and run starts give the
// np.unique order directly: w.ukey[d] = token << 12 | count.  Returns D.
template <int V>
__device__ int warp_dedup_sort(const SigArgs &a, int64_t row, const WarpSmem &w, int lane) {
    uint64_t *wsm = reinterpret_cast<uint64_t *>(w.hkey);  // >= 8 words of scratch (8 H bytes)
    for (int i = lane; i < a.words; i += 32) wsm[i] = a.bits[row * a.words + i];
    __syncwarp();
    const uint32_t nmask = (a.n == 32) ? 0xFFFFFFFFu : ((1u << a.n) - 1u);
    uint32_t x[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        const int e = lane * V + v;
        uint32_t tok = 0xFFFFFFFFu;
        if (e < a.T) {
            const int wi = e >> 6, sh = e & 63;
            const uint64_t w0 = wsm[wi], w1 = wi + 1 < a.words ? wsm[wi + 1] : 0ULL;
            const uint64_t bitsv = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
            tok = __brev((uint32_t)bitsv & nmask) >> (32 - a.n);
        }
        x[v] = tok;
    }
    __syncwarp();
    warp_sort_regs<V>(x, lane);
    // run starts
    const uint32_t pv = __shfl_up_sync(0xFFFFFFFFu, x[V - 1], 1);
    unsigned smask = 0;
    int c = 0;
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint32_t prev = v ? x[v - 1] : pv;
        const bool st = x[v] != 0xFFFFFFFFu && (lane * V + v == 0 || x[v] != prev);
        smask |= (unsigned)st << v;
        c += st;
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    const int D = __shfl_sync(0xFFFFFFFFu, incl, 31);
    int d = incl - c;
#pragma unroll
    for (int v = 0; v < V; v++) {
        if ((smask >> v) & 1u) {
            w.utok[d] = x[v];
            w.ustart[d] = (uint16_t)(lane * V + v);
            d++;
        }
    }
    if (lane == 0) w.ustart[D] = (uint16_t)a.T;
    __syncwarp();
    for (int k = lane; k < D; k += 32) {
        const uint32_t cnt = (uint32_t)w.ustart[k + 1] - (uint32_t)w.ustart[k];
        w.ukey[k] = (w.utok[k] << 12) | cnt;
    }
    __syncwarp();
    return D;
}

// Distinct tokens + counts via the per-warp hash set, as packed keys
// (token << 12 | count) sorted ascending (= np.unique order); returns D.
// The hash table is left empty again for the next series.
__device__ int warp_dedup(const SigArgs &a, int64_t row, const WarpSmem &w, int lane) {
    const uint64_t myword = lane < a.words ? a.bits[row * a.words + lane] : 0ULL;
    const uint32_t hmask = (uint32_t)a.H - 1u;
    const unsigned lt0 = (1u << lane) - 1u;
    for (int base = 0; base < a.T; base += 32) {
        const int i = base + lane;
        const uint32_t t0 = token_at(myword, i, a.words, a.n);  // all lanes shuffle
        const uint32_t tok = i < a.T ? t0 : SG_EMPTY;
        // identical tokens of this round insert once (runs are common)
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, tok);
        if (tok != SG_EMPTY && (peers & lt0) == 0) {
            const uint32_t add = __popc(peers);
            uint32_t h = (tok * 0x9E3779B1u) & hmask;
            while (true) {
                uint32_t prev = atomicCAS(&w.hkey[h], SG_EMPTY, tok);
                if (prev == SG_EMPTY || prev == tok) {
                    atomicAdd(&w.hcnt[h], add);
                    break;
                }
                h = (h + 1) & hmask;
            }
        }
    }
    __syncwarp();
    int D = 0;
    for (int base = 0; base < a.H; base += 32) {
        const int h = base + lane;
        const uint32_t k = w.hkey[h];
        const bool occ = k != SG_EMPTY;
        const unsigned msk = __ballot_sync(0xFFFFFFFFu, occ);
        if (occ) {
            w.ukey[D + __popc(msk & lt0)] = (k << 12) | w.hcnt[h];
            w.hkey[h] = SG_EMPTY;
            w.hcnt[h] = 0u;
        }
        D += __popc(msk);
    }
    __syncwarp();
    sort_keys(w.ukey, D, w.hkey, a.H, lane);
    if (D > 256) {  // the smem sort used the hash table as scratch
        for (int h = lane; h < a.H; h += 32) w.hkey[h] = SG_EMPTY;
        __syncwarp();
    }
    return D;
}

// Sorted distinct tokens + counts (np.unique order) for the stage API; returns D.
__device__ int warp_shingle_sorted(const SigArgs &a, int64_t row, const WarpSmem &w, int lane) {
    const uint64_t myword = lane < a.words ? a.bits[row * a.words + lane] : 0ULL;
    for (int base = 0; base < a.P2; base += 32) {
        const int i = base + lane;
        const uint32_t tok = token_at(myword, i, a.words, a.n);
        w.sortbuf[i] = i < a.T ? tok : 0xFFFFFFFFu;
    }
    __syncwarp();
    for (int k = 2; k <= a.P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = lane; idx < (a.P2 >> 1); idx += 32) {
                int i = 2 * idx - (idx & (j - 1));
                int l = i + j;
                uint32_t x = w.sortbuf[i], y = w.sortbuf[l];
                bool up = (i & k) == 0;
                if ((x > y) == up) {
                    w.sortbuf[i] = y;
                    w.sortbuf[l] = x;
                }
            }
            __syncwarp();
        }
    }
    int D = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < a.T; base += 32) {
        int i = base + lane;
        uint32_t v = i < a.T ? w.sortbuf[i] : 0u;
        uint32_t pv = (i > 0 && i < a.T) ? w.sortbuf[i - 1] : ~v;
        bool f = i < a.T && v != pv;
        unsigned msk = __ballot_sync(0xFFFFFFFFu, f);
        if (f) {
            int pos = D + __popc(msk & lt);
            w.utok[pos] = v;
            w.ustart[pos] = (uint16_t)i;
        }
        D += __popc(msk);
    }
    __syncwarp();
    for (int d = lane; d < D; d += 32) {
        int e = d + 1 < D ? w.ustart[d + 1] : a.T;
        w.ucnt[d] = (uint16_t)(e - w.ustart[d]);
    }
    __syncwarp();
    // restore the hash-set invariant (sortbuf aliases it)
    for (int h = lane; h < a.H; h += 32) {
        w.hkey[h] = SG_EMPTY;
        w.hcnt[h] = 0u;
    }
    __syncwarp();
    return D;
}

// t = floor(fl(fl(lw / r) + b)) exactly (see header): approximate quotient,
// exact IEEE division only when the sum is within 1e-12 of an integer.
__device__ __forceinline__ double cws_t(double lw, double r, double b) {
    double rc;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(r));
    double e = fma(-r, rc, 1.0);
    rc = fma(rc, e, rc);
    e = fma(-r, rc, 1.0);
    rc = fma(rc, e, rc);
    const double s1 = fma(lw, rc, b);
    const double fl = floor(s1);
    const double tol = s1 * 1e-12;
    if (s1 - fl > tol && (fl + 1.0) - s1 > tol) return fl;
    return floor(__dadd_rn(__ddiv_rn(lw, r), b));
}

// cws_t with a tabulated reciprocal 1/r = fl(1/r): fma(lw, 1/r, b) is within
// 4u(lw/r + b) of fl(fl(lw/r) + b), far inside the 1e-12 relative guard.
__device__ __forceinline__ double cws_t_inv(double lw, double r, double rinv, double b) {
    const double s1 = fma(lw, rinv, b);
    const double fl = floor(s1);
    const double tol = s1 * 1e-12;
    if (s1 - fl > tol && (fl + 1.0) - s1 > tol) return fl;
    return floor(__dadd_rn(__ddiv_rn(lw, r), b));
}

__device__ __forceinline__ double cws_lna(double t, double r, double lnc, double b) {
    const double lny = __dmul_rn(r, __dsub_rn(t, b));
    return __dsub_rn(__dsub_rn(lnc, lny), r);
}

// argmin over the D distinct tokens (packed keys in ascending token order),
// K-fold, signature row.  Count-1 and count>1 tokens run in separate
// branch-free loops (index lists keep ascending order); the count-1 loop keeps
// U independent min-chains per slot so the compare/select chain does not
// serialise on latency.  Chains are merged by (value, index): ties go to the
// lower index = lower token, i.e. np.argmin's first occurrence.
__device__ __forceinline__ void take_min(double v, int d, double &bv, int &bd) {
    if (v < bv || (v == bv && d < bd)) {
        bv = v;
        bd = d;
    }
}

template <int NS, typename RT>
__device__ void warp_cws(const SigArgs &a, int64_t row, const WarpSmem &w, int D, int lane) {
    constexpr int U = 4;
    const int S = a.S;
    const RT *rank = reinterpret_cast<const RT *>(a.rank);
    // split indices: count-1 into list1 (ustart storage), count>1 into listm (ucnt storage)
    uint16_t *list1 = w.ustart;
    uint16_t *listm = w.ucnt;
    int n1 = 0, nm = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < D; base += 32) {
        const int d = base + lane;
        const uint32_t key = d < D ? w.ukey[d] : 0u;
        const bool one = d < D && (key & 0xFFFu) == 1u;
        const bool many = d < D && (key & 0xFFFu) > 1u;
        const unsigned m1 = __ballot_sync(0xFFFFFFFFu, one);
        const unsigned mm = __ballot_sync(0xFFFFFFFFu, many);
        if (one) list1[n1 + __popc(m1 & lt)] = (uint16_t)d;
        if (many) listm[nm + __popc(mm & lt)] = (uint16_t)d;
        n1 += __popc(m1);
        nm += __popc(mm);
    }
    __syncwarp();
    // count-1 tokens: ln_a1 ranks are a total order by (value, token), so the
    // argmin is an integer min over (rank << 12 | index); U independent chains.
    uint32_t bk[U][NS];  // rank < 2^20, index < 2^12
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
        for (int i = 0; i < NS; i++) bk[u][i] = 0xFFFFFFFFu;
    for (int e0 = 0; e0 < n1; e0 += U) {
        int dd[U];
        uint32_t rv[U][NS];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool ok = e0 + u < n1;
            dd[u] = ok ? list1[e0 + u] : 0;
            const size_t base = (size_t)(w.ukey[dd[u]] >> 12) * S;
#pragma unroll
            for (int i = 0; i < NS; i++) {
                const int s = lane + 32 * i;
                rv[u][i] = (ok && s < S) ? (uint32_t)__ldg(rank + base + s) : 0xFFFFFu;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int i = 0; i < NS; i++) {
                bk[u][i] = min(bk[u][i], (rv[u][i] << 12) | (uint32_t)dd[u]);
            }
    }
    double best[1][NS];
    int bd[1][NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
        uint32_t k0 = bk[0][i];
#pragma unroll
        for (int u = 1; u < U; u++) k0 = min(k0, bk[u][i]);
        const int s = lane + 32 * i;
        if (n1 > 0 && s < S) {
            bd[0][i] = (int)(k0 & 0xFFFu);
            best[0][i] = __ldg(a.lna1 + (size_t)(w.ukey[bd[0][i]] >> 12) * S + s);
        } else {
            bd[0][i] = 0x7FFFFFFF;
            best[0][i] = (double)INFINITY;
        }
    }
    // count>1 tokens: full formula (wmh.py:74-76), one more chain
    double bestm[NS];
    int bdm[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
        bestm[i] = (double)INFINITY;
        bdm[i] = 0x7FFFFFFF;
    }
    for (int f = 0; f < nm; f++) {
        const int d = listm[f];
        const uint32_t key = w.ukey[d];
        const size_t base = (size_t)(key >> 12) * S;
        const double lw = __ldg(a.lnw + (key & 0xFFFu));
#pragma unroll
        for (int i = 0; i < NS; i++) {
            const int s = lane + 32 * i;
            if (s < S) {
                const double r = __ldg(a.tr + base + s);
                const double lnc = __ldg(a.tlnc + base + s), b = __ldg(a.tbeta + base + s);
                const double v = cws_lna(cws_t(lw, r, b), r, lnc, b);
                const bool l = v < bestm[i];  // ascending indices: strict < keeps the first
                bestm[i] = l ? v : bestm[i];
                bdm[i] = l ? d : bdm[i];
            }
        }
    }
    // merge chains, winners -> keys (wmh.py:79-81)
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const int s = lane + 32 * i;
        double bv = bestm[i];
        int bi = bdm[i];
        take_min(best[0][i], bd[0][i], bv, bi);
        if (s < S && D > 0) {
            const uint32_t key = w.ukey[bi];
            const uint32_t tok = key >> 12, cnt = key & 0xFFFu;
            const size_t ent = (size_t)tok * S + s;
            const double b = __ldg(a.tbeta + ent);
            double t;
            if (cnt == 1u) t = floor(b);  // fl(0/r + b) = b
            else t = cws_t(__ldg(a.lnw + cnt), __ldg(a.tr + ent), b);
            const uint64_t tt = (uint64_t)(int64_t)t;
            const uint64_t k64 = ssh_mix64((uint64_t)tok ^ ssh_mix64(tt ^ SSH_SALT_KEY));
            w.keys[s] = k64;
            if (a.keys_out) a.keys_out[row * S + s] = k64;
        }
    }
    __syncwarp();
    for (int j = lane; j < a.L; j += 32) {
        uint64_t acc = w.keys[j * a.K];
        for (int i = 1; i < a.K; i++) acc = ssh_mix64(acc ^ w.keys[j * a.K + i]);
        a.sig_out[row * a.L + j] = acc;
    }
    __syncwarp();
}

// ---------------------------------------------------------------- order-free CWS
// The argmin of every slot only needs the distinct tokens and their counts,
// not np.unique's order: ties are broken by comparing tokens (lowest wins =
// np.argmin's first occurrence over sorted tokens), and the count-1 argmin is
// an integer min over ln_a1 ranks, which are a total order by (value, token).
// This path (n <= 15, S = K*L <= 16*QL, T <= 1024) therefore
//   * dedups without a global sort: the first 32V tokens are sorted in
//     registers (run starts give their counts), the remaining tokens are
//     merged 32 at a time (match_any inside the chunk, binary search in the
//     sorted part, linear search among tokens appended earlier);
//   * takes the count-1 minimum with two lanes per token row (lane half h
//     loads 8*QL u16 ranks as QL 16-byte vectors) and packed u16x2 minima,
//     then a reduce-scatter across the 16 token lanes; the winning rank maps
//     back to its token through the inverse table, and its ln_a1 seeds the
//     per-slot best;
//   * evaluates count > 1 tokens with the full formula (wmh.py:74-76) with
//     lanes owning slots, as before.

template <int V>
__device__ int warp_dedup_split(const SigArgs &a, int64_t row, const WarpSmem &w, int lane) {
    uint64_t *wsm = reinterpret_cast<uint64_t *>(w.hkey);
    for (int i = lane; i < a.words; i += 32) wsm[i] = a.bits[row * a.words + i];
    __syncwarp();
    const uint32_t nmask = (1u << a.n) - 1u;  // n <= 15 on this path
    const int TM = min(a.T, 32 * V);
    const unsigned lt0 = (1u << lane) - 1u;
    uint32_t x[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        const int e = lane * V + v;
        uint32_t tok = 0xFFFFFFFFu;
        if (e < TM) {
            const int wi = e >> 6, sh = e & 63;
            const uint64_t w0 = wsm[wi], w1 = wi + 1 < a.words ? wsm[wi + 1] : 0ULL;
            const uint64_t bitsv = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
            tok = __brev((uint32_t)bitsv & nmask) >> (32 - a.n);
        }
        x[v] = tok;
    }
    warp_sort_regs<V>(x, lane);
    const uint32_t pv = __shfl_up_sync(0xFFFFFFFFu, x[V - 1], 1);
    unsigned smask = 0;
    int c = 0;
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint32_t prev = v ? x[v - 1] : pv;
        const bool st = x[v] != 0xFFFFFFFFu && (lane * V + v == 0 || x[v] != prev);
        smask |= (unsigned)st << v;
        c += st;
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    int D = __shfl_sync(0xFFFFFFFFu, incl, 31);
    int d = incl - c;
#pragma unroll
    for (int v = 0; v < V; v++) {
        if ((smask >> v) & 1u) {
            w.utok[d] = x[v];
            w.ustart[d] = (uint16_t)(lane * V + v);
            d++;
        }
    }
    if (lane == 0) w.ustart[D] = (uint16_t)TM;
    __syncwarp();
    for (int k = lane; k < D; k += 32) {
        const uint32_t cnt = (uint32_t)w.ustart[k + 1] - (uint32_t)w.ustart[k];
        w.ukey[k] = (w.utok[k] << 12) | cnt;
    }
    __syncwarp();
    const int Dm = D;
    for (int c0 = 32 * V; c0 < a.T; c0 += 32) {
        const int e = c0 + lane;
        uint32_t tok = 0xFFFFFFFFu;
        if (e < a.T) {
            const int wi = e >> 6, sh = e & 63;
            const uint64_t w0 = wsm[wi], w1 = wi + 1 < a.words ? wsm[wi + 1] : 0ULL;
            const uint64_t bitsv = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
            tok = __brev((uint32_t)bitsv & nmask) >> (32 - a.n);
        }
        // every lane looks its token up and counts it with a shared-memory atomic
        // (same-address atomics are cheap; __match_any_sync on every round was the
        // larger part of this loop); only rounds that meet a new token take the
        // match to insert each new token once
        bool need = false;
        if (tok != 0xFFFFFFFFu) {
            int lo = 0, hi = Dm;  // first entry with token >= tok
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((w.ukey[mid] >> 12) < tok) lo = mid + 1;
                else hi = mid;
            }
            int pos = -1;
            if (lo < Dm && (w.ukey[lo] >> 12) == tok) pos = lo;
            for (int q = Dm; pos < 0 && q < D; q++)
                if ((w.ukey[q] >> 12) == tok) pos = q;
            if (pos >= 0) atomicAdd(&w.ukey[pos], 1u);
            else need = true;
        }
        if (__any_sync(0xFFFFFFFFu, need)) {
            const unsigned peers = __match_any_sync(0xFFFFFFFFu, need ? tok : 0xFFFFFFFFu);
            const bool lead = need && (peers & lt0) == 0;
            const unsigned nm = __ballot_sync(0xFFFFFFFFu, lead);
            if (lead) w.ukey[D + __popc(nm & lt0)] = (tok << 12) | __popc(peers);
            D += __popc(nm);
        }
        __syncwarp();
    }
    return D;
}

// reduce-scatter of A packed u16x2 minima over the lane bits M, M/2, .., 1:
// halve while A is even (a lane keeps the half selected by its bit), then a
// full butterfly on the rest.  base = original index of x[0].
__host__ __device__ constexpr int rs_final(int A, int M) {
    return (M == 0 || (A & 1)) ? A : rs_final(A / 2, M / 2);
}
__host__ __device__ constexpr int rs_group(int A, int M) {  // lanes sharing a result
    return M == 0 ? 1 : ((A & 1) ? 2 * M : rs_group(A / 2, M / 2));
}

template <int A, int M>
__device__ __forceinline__ void rs_reduce(uint32_t (&x)[A], int lane, int &base) {
    if constexpr (M == 0) {
        return;
    } else if constexpr ((A & 1) == 0) {
        constexpr int H = A / 2;
        const bool hi = (lane & M) != 0;
        uint32_t y[H];
#pragma unroll
        for (int i = 0; i < H; i++) {
            const uint32_t send = hi ? x[i] : x[i + H];
            const uint32_t keep = hi ? x[i + H] : x[i];
            y[i] = __vminu2(keep, __shfl_xor_sync(0xFFFFFFFFu, send, M));
        }
        if (hi) base += H;
        rs_reduce<H, M / 2>(y, lane, base);
#pragma unroll
        for (int i = 0; i < H; i++) x[i] = y[i];
    } else {
#pragma unroll
        for (int mm = M; mm >= 1; mm >>= 1)
#pragma unroll
            for (int i = 0; i < A; i++) x[i] = __vminu2(x[i], __shfl_xor_sync(0xFFFFFFFFu, x[i], mm));
    }
}

template <int QL>
__device__ void warp_cws_fast(const SigArgs &a, int64_t row, const WarpSmem &w, int D, int lane) {
    constexpr int NS = (16 * QL + 31) / 32;
    constexpr int A = 4 * QL;
    const int S = a.S;
    uint16_t *list1 = w.ustart;                // count-1 and count-2 tokens (combined ranks)
    uint16_t *listm = w.ucnt;                  // count > 2 tokens
    int n1 = 0, nm = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < D; base += 32) {
        const int d = base + lane;
        const uint32_t key = d < D ? w.ukey[d] : 0u;
        const uint32_t c = key & 0xFFFu;
        const bool one = d < D && c <= 2u;
        const bool many = d < D && c > 2u;
        const unsigned m1 = __ballot_sync(0xFFFFFFFFu, one);
        const unsigned mm = __ballot_sync(0xFFFFFFFFu, many);
        if (one) list1[n1 + __popc(m1 & lt)] = (uint16_t)d;
        if (many) listm[nm + __popc(mm & lt)] = (uint16_t)d;
        n1 += __popc(m1);
        nm += __popc(mm);
    }
    __syncwarp();
    // count-1 tokens: packed u16x2 rank minima, lane = (row half h, token j)
    const int h = lane >> 4, j = lane & 15;
    uint32_t acc[A];
#pragma unroll
    for (int i = 0; i < A; i++) acc[i] = 0xFFFFFFFFu;
    const uint4 *rp = reinterpret_cast<const uint4 *>(a.rankp);
    for (int e0 = 0; e0 < n1; e0 += 16) {
        const int ea = e0 + j;
        if (ea < n1) {
            const uint32_t kk = w.ukey[list1[ea]];
            const size_t ba = (size_t)(((kk >> 12) << 1) | ((kk & 0xFFFu) - 1u)) * (2 * QL) + h * QL;
#pragma unroll
            for (int q = 0; q < QL; q++) {
                const uint4 va = __ldg(rp + ba + q);
                acc[4 * q + 0] = __vminu2(acc[4 * q + 0], va.x);
                acc[4 * q + 1] = __vminu2(acc[4 * q + 1], va.y);
                acc[4 * q + 2] = __vminu2(acc[4 * q + 2], va.z);
                acc[4 * q + 3] = __vminu2(acc[4 * q + 3], va.w);
            }
        }
    }
    int rbase = 0;
    rs_reduce<A, 8>(acc, lane, rbase);
    constexpr int AF = rs_final(A, 8);
    constexpr int G = rs_group(A, 8);
    double *bv = reinterpret_cast<double *>(w.keys);  // S entries, rewritten as keys below
    uint32_t *bt = w.hkey;                              // S entries: token | t1 << 16
#pragma unroll
    for (int l = 0; l < 2 * AF; l++) {
        if (l % G == (j & (G - 1))) {
            const int r = rbase + (l >> 1), hw = l & 1;
            const int s = 8 * QL * h + 2 * r + hw;
            if (s < S) {
                const uint32_t rk = (acc[l >> 1] >> (16 * hw)) & 0xFFFFu;
                double v = (double)INFINITY;
                uint32_t tt = 0xFFFFu;
                if (n1 > 0) {  // every slot then has a real minimum (0xFFFF is a valid rank)
                    const uint4 br = __ldg(a.byrank + (((size_t)s << (a.n + 1)) | rk));
                    v = __hiloint2double((int)br.y, (int)br.x);
                    tt = br.z;
                }
                bv[s] = v;
                bt[s] = tt;
            }
        }
    }
    __syncwarp();
    double best[NS], bestt[NS];
    uint32_t btok[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const int s = lane + 32 * i;
        const uint32_t tt = s < S ? bt[s] : 0xFFFFu;
        best[i] = s < S ? bv[s] : (double)INFINITY;
        btok[i] = tt & 0xFFFFu;
        bestt[i] = (double)(tt >> 16);
    }
    // count > 1 tokens: full formula, ties toward the lower token; two tokens
    // per step keep their twelve variate loads in flight together
    auto eval = [&](uint32_t tok, double lw, int i, double2 p0, double2 p1) {
        const double r = p0.x, rinv = p0.y, lnc = p1.x, b = p1.y;
        const double t = cws_t_inv(lw, r, rinv, b);
        const double v = cws_lna(t, r, lnc, b);
        const bool l = v < best[i] || (v == best[i] && tok < btok[i]);
        best[i] = l ? v : best[i];
        btok[i] = l ? tok : btok[i];
        bestt[i] = l ? t : bestt[i];
    };
    const uint32_t tmax = (1u << a.n) - 1u;
    for (int f = 0; f < nm; f++) {
        const uint32_t ka = w.ukey[listm[f]];
        const uint32_t ta = ka >> 12;
        if (a.edge && (ta == 0u || ta == tmax)) {
            // all-zero / all-one tokens (sign runs; most counts > 2): tabulated
            // {ln_a, t} per (count, slot), same exact formula
            const double2 *er = a.edge + ((size_t)(ta ? 1 : 0) * (a.maxc + 1) + (ka & 0xFFFu)) * S;
#pragma unroll
            for (int i = 0; i < NS; i++) {
                const int s = lane + 32 * i;
                if (s < S) {
                    const double2 v = __ldg(er + s);
                    const bool l = v.x < best[i] || (v.x == best[i] && ta < btok[i]);
                    best[i] = l ? v.x : best[i]; btok[i] = l ? ta : btok[i]; bestt[i] = l ? v.y : bestt[i];
                }
            }
            continue;
        }
        const double lwa = __ldg(a.lnw + (ka & 0xFFFu));
#pragma unroll
        for (int i = 0; i < NS; i++) {
            const int s = lane + 32 * i;
            if (s < S) {
                const size_t ea = 2 * ((size_t)ta * S + s);
                eval(ta, lwa, i, __ldg(a.rlcb + ea), __ldg(a.rlcb + ea + 1));
            }
        }
    }
    // winners -> keys (wmh.py:79-81); bv is dead from here on
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const int s = lane + 32 * i;
        if (s < S) {
            const uint64_t tt = (uint64_t)(int64_t)bestt[i];
            const uint64_t k64 = ssh_mix64((uint64_t)btok[i] ^ ssh_mix64(tt ^ SSH_SALT_KEY));
            w.keys[s] = k64;
            if (a.keys_out) a.keys_out[row * S + s] = k64;
        }
    }
    __syncwarp();
    for (int jj = lane; jj < a.L; jj += 32) {
        uint64_t acc64 = w.keys[jj * a.K];
        for (int i = 1; i < a.K; i++) acc64 = ssh_mix64(acc64 ^ w.keys[jj * a.K + i]);
        a.sig_out[row * a.L + jj] = acc64;
    }
    __syncwarp();
}

template <int MODE, int QL, int V>
__global__ void __launch_bounds__(32 * SG_WARPS, SG_FAST_MINB) cws_fast_kernel(SigArgs a, int warps) {
    extern __shared__ __align__(16) unsigned char sg_smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpSmem w = carve(sg_smem + (size_t)wid * a.warp_smem, a);
    const int64_t nwarps = (int64_t)gridDim.x * warps;
    for (int64_t row = (int64_t)blockIdx.x * warps + wid; row < a.N; row += nwarps) {
        int D;
        if (MODE == SIG_MODE_CWS_FROM_SETS) {
            D = a.len_in[row];
            for (int d = lane; d < D; d += 32)
                w.ukey[d] = (a.tok_in[row * a.T + d] << 12) | (uint32_t)a.cnt_in[row * a.T + d];
            __syncwarp();
        } else {
            D = warp_dedup_split<V>(a, row, w, lane);
        }
        warp_cws_fast<QL>(a, row, w, D, lane);
    }
}

template <int MODE, int QL, int V>
static int launch_fast(ssh_ctx *ctx, const SigArgs &a, int64_t N, cudaStream_t st) {
    auto kern = cws_fast_kernel<MODE, QL, V>;
    int warps = SG_WARPS;
    while (warps > 1 && (size_t)a.warp_smem * warps > 200 * 1024) warps--;
    size_t smem = (size_t)a.warp_smem * warps;
    SSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (N + warps - 1) / warps;
    const int grid = (int)std::min<int64_t>(nblk, (int64_t)ctx->num_sms * per_sm);
    kern<<<grid, 32 * warps, smem, st>>>(a, warps);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

template <int MODE, int QL>
static int launch_fast_v(ssh_ctx *ctx, const SigArgs &a, int64_t N, cudaStream_t st) {
    if (MODE == SIG_MODE_CWS_FROM_SETS) return launch_fast<MODE, QL, 1>(ctx, a, N, st);
    int v = a.T / 32;
    // SSH_CWS_V caps the register-sorted part (32 V tokens; the rest merges 32 at a time): A/B switch
    if (const char *ev = getenv("SSH_CWS_V")) v = std::min(v, std::max(1, atoi(ev)));
    // 256 register-sorted tokens at most: at T = 643 (configs[3]) sorting 512 and merging 131
    // measured 35.6 ms per 1M-row build against 32.0 ms for 256 + 387 (V = 4: 35.0 ms)
    if (v >= 8) return launch_fast<MODE, QL, 8>(ctx, a, N, st);
    if (v >= 4) return launch_fast<MODE, QL, 4>(ctx, a, N, st);
    if (v >= 2) return launch_fast<MODE, QL, 2>(ctx, a, N, st);
    return launch_fast<MODE, QL, 1>(ctx, a, N, st);
}

// 1: launched on the order-free path, 0: not applicable, <0: error
template <int MODE>
static int try_fast(ssh_ctx *ctx, const SigArgs &a, int64_t N, cudaStream_t st) {
    if (ctx->rank_ql == 0 || a.T > 1024 || ctx->p.n > 15) return 0;
    const int region = 8 * a.H > 4 * a.P2 ? 8 * a.H : 4 * a.P2;
    if (4 * a.S > region) return 0;
    int rc;
    switch (ctx->rank_ql) {
        case 2: rc = launch_fast_v<MODE, 2>(ctx, a, N, st); break;
        case 5: rc = launch_fast_v<MODE, 5>(ctx, a, N, st); break;
        default: return 0;
    }
    return rc == SSH_OK ? 1 : rc;
}

template <int MODE, int NS>
__global__ void __launch_bounds__(32 * SG_WARPS, 4) shingle_cws_kernel(SigArgs a, int warps) {
    extern __shared__ __align__(16) unsigned char sg_smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpSmem w = carve(sg_smem + (size_t)wid * a.warp_smem, a);
    for (int h = lane; h < a.H; h += 32) {
        w.hkey[h] = SG_EMPTY;
        w.hcnt[h] = 0u;
    }
    __syncwarp();
    const int64_t nwarps = (int64_t)gridDim.x * warps;
    for (int64_t row = (int64_t)blockIdx.x * warps + wid; row < a.N; row += nwarps) {
        int D;
        if (MODE == SIG_MODE_CWS_FROM_SETS) {
            D = a.len_in[row];
            for (int d = lane; d < D; d += 32)
                w.ukey[d] = (a.tok_in[row * a.T + d] << 12) | (uint32_t)a.cnt_in[row * a.T + d];
            __syncwarp();
        } else if (MODE == SIG_MODE_SHINGLE) {
            D = warp_shingle_sorted(a, row, w, lane);
        } else if (a.T <= 128) {
            D = warp_dedup_sort<4>(a, row, w, lane);
        } else if (a.T <= 256) {
            D = warp_dedup_sort<8>(a, row, w, lane);
        } else if (a.T <= 512) {
            D = warp_dedup_sort<16>(a, row, w, lane);
        } else {
            D = warp_dedup(a, row, w, lane);
        }
        if (MODE == SIG_MODE_SHINGLE) {
            for (int d = lane; d < a.T; d += 32) {
                a.tok_out[row * a.T + d] = d < D ? w.utok[d] : 0u;
                a.cnt_out[row * a.T + d] = d < D ? w.ucnt[d] : (uint16_t)0;
            }
            if (lane == 0) a.len_out[row] = D;
            __syncwarp();
        } else {
            if (a.n <= 16) warp_cws<NS, uint16_t>(a, row, w, D, lane);
            else warp_cws<NS, uint32_t>(a, row, w, D, lane);
        }
    }
}

template <int MODE, int NS>
static int launch_sig(ssh_ctx *ctx, const SigArgs &a, int64_t N, cudaStream_t st) {
    auto kern = shingle_cws_kernel<MODE, NS>;
    int warps = SG_WARPS;
    while (warps > 1 && (size_t)a.warp_smem * warps > 200 * 1024) warps--;
    size_t smem = (size_t)a.warp_smem * warps;
    SSH_REQUIRE(smem <= 220 * 1024, SSH_ERR_UNSUPPORTED,
                "signature kernel needs %zu bytes of shared memory (T=%d)", smem, a.T);
    SSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  (int)cudaSharedmemCarveoutMaxShared));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (N + warps - 1) / warps;
    const int grid = (int)std::min<int64_t>(nblk, (int64_t)ctx->num_sms * per_sm);
    kern<<<grid, 32 * warps, smem, st>>>(a, warps);
    SSH_CHECK_LAUNCH();
    return SSH_OK;
}

template <int MODE>
static int launch_sig_ns(ssh_ctx *ctx, const SigArgs &a, int64_t N, cudaStream_t st) {
    switch ((a.S + 31) / 32) {
        case 1: return launch_sig<MODE, 1>(ctx, a, N, st);
        case 2: return launch_sig<MODE, 2>(ctx, a, N, st);
        case 3: return launch_sig<MODE, 3>(ctx, a, N, st);
        case 4: return launch_sig<MODE, 4>(ctx, a, N, st);
        case 5: return launch_sig<MODE, 5>(ctx, a, N, st);
        case 6: return launch_sig<MODE, 6>(ctx, a, N, st);
        case 7: return launch_sig<MODE, 7>(ctx, a, N, st);
        default: return launch_sig<MODE, 8>(ctx, a, N, st);
    }
}

// SSH_CWS_FAST=0 selects the sorted-set kernel (A/B comparisons, tests)
static bool ssh_cws_fast_disabled() {
    static const int off = [] {
        const char *e = getenv("SSH_CWS_FAST");
        return (e && e[0] == '0') ? 1 : 0;
    }();
    return off != 0;
}

int ssh_launch_shingle_cws(ssh_ctx *ctx, const uint64_t *bits, const uint32_t *tok_in,
                           const uint16_t *cnt_in, const int32_t *len_in, int64_t N,
                           uint32_t *tok_out, uint16_t *cnt_out, int32_t *len_out,
                           uint64_t *keys_out, uint64_t *sig_out, int mode, cudaStream_t st) {
    SigArgs a;
    a.bits = bits; a.tok_in = tok_in; a.cnt_in = cnt_in; a.len_in = len_in;
    a.tok_out = tok_out; a.cnt_out = cnt_out; a.len_out = len_out;
    a.keys_out = keys_out; a.sig_out = sig_out;
    a.lna1 = ctx->d_lna1; a.tr = ctx->d_r; a.tlnc = ctx->d_lnc; a.tbeta = ctx->d_beta;
    a.lnw = ctx->d_lnw;
    a.rank = ctx->d_rank;
    a.rankp = ctx->d_rankp;
    a.byrank = ctx->d_byrank;
    a.rlcb = reinterpret_cast<const double2 *>(ctx->d_rlcb);
    a.edge = reinterpret_cast<const double2 *>(ctx->d_edge);
    a.maxc = ctx->max_count;
    a.N = N; a.words = ctx->words; a.nb = ctx->nb; a.n = ctx->p.n; a.T = ctx->T;
    int P2 = 32;
    while (P2 < ctx->T) P2 <<= 1;
    a.P2 = P2;
    a.H = P2;  // D <= T <= P2/2 + 1: load factor <= ~1/2
    a.S = ctx->S; a.L = ctx->p.L; a.K = ctx->p.K;
    a.warp_smem = warp_smem_bytes(a.S, a.P2, a.H, a.T);
    if (mode == SIG_MODE_SHINGLE) return launch_sig<SIG_MODE_SHINGLE, 1>(ctx, a, N, st);
    if (!ssh_cws_fast_disabled()) {
        const int f = mode == SIG_MODE_CWS_FROM_SETS ? try_fast<SIG_MODE_CWS_FROM_SETS>(ctx, a, N, st)
                                                     : try_fast<SIG_MODE_FUSED>(ctx, a, N, st);
        if (f != 0) return f > 0 ? SSH_OK : f;
    }
    if (mode == SIG_MODE_CWS_FROM_SETS) return launch_sig_ns<SIG_MODE_CWS_FROM_SETS>(ctx, a, N, st);
    return launch_sig_ns<SIG_MODE_FUSED>(ctx, a, N, st);
}
