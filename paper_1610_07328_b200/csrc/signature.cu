// signature.cu — K2 shingle + K3 consistent weighted sampling (one warp per series).
//
// K2 (shingle.py:56-75, index.py:118): tokens t_i = bits[i..i+n-1] with the
// first bit most significant, then the distinct tokens ascending with their
// counts (np.unique(return_counts=True)).  A warp extracts its series' T
// tokens from the packed bit row (word shuffles + __brev), bitonic-sorts
// them in shared memory and run-length encodes with ballots.
//
// K3 (wmh.py:52-81 + signature(concat=K) wmh.py:107-125): for every slot s
// of S = K*L, argmin over the distinct tokens of
//     ln_a = ln_c - r*(floor(ln_w/r + beta) - beta) - r
// (first occurrence = lowest token on ties), key = mix64(tok ^ mix64(t ^ SALT_KEY)),
// then the K-fold acc = mix64(acc ^ key).  The variates come from host tables
// (np.log bits); the device does only IEEE div/add/sub/mul/floor in the
// reference order with explicit _rn intrinsics, so keys are bit-exact.
// Count-1 tokens (76-84% of all) use the precomputed ln_a1 table (one 8-byte
// gather per (token, slot)); larger counts evaluate the full formula.
// Lanes own slots s = lane + 32*i, so every gather is a contiguous 256-byte
// segment of the [token][slot] table (L2-resident: 2^15 x 80 x 8 B = 21 MB).
#include <float.h>

#include <algorithm>

#include "common.cuh"

#define SG_WARPS 8
#define SG_NS_MAX (SSH_MAX_SLOTS / 32)

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
    int64_t N;
    int words, nb, n, T, P2, S, L, K;
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
    uint32_t *sortbuf;  // P2
    uint32_t *utok;     // T
    uint16_t *ucnt;     // T
    uint16_t *ustart;   // T+1
    uint16_t *list1;    // T  indices of count-1 tokens
    uint16_t *listm;    // T  indices of count>1 tokens
    uint64_t *keys;     // S
};

__device__ __forceinline__ WarpSmem carve(unsigned char *base, const SigArgs &a) {
    WarpSmem w;
    unsigned char *p = base;
    w.keys = reinterpret_cast<uint64_t *>(p); p += 8 * a.S;
    w.sortbuf = reinterpret_cast<uint32_t *>(p); p += 4 * a.P2;
    w.utok = reinterpret_cast<uint32_t *>(p); p += 4 * a.T;
    w.ucnt = reinterpret_cast<uint16_t *>(p); p += 2 * a.T;
    w.ustart = reinterpret_cast<uint16_t *>(p); p += 2 * (a.T + 1);
    w.list1 = reinterpret_cast<uint16_t *>(p); p += 2 * a.T;
    w.listm = reinterpret_cast<uint16_t *>(p);
    return w;
}

// Tokens of one series -> distinct sorted tokens + counts in smem; returns D.
__device__ int warp_shingle(const SigArgs &a, int64_t row, const WarpSmem &w, int lane) {
    const uint64_t *brow = a.bits + row * a.words;
    uint64_t myword = lane < a.words ? brow[lane] : 0ULL;
    const uint32_t nmask = (a.n == 32) ? 0xFFFFFFFFu : ((1u << a.n) - 1u);
    for (int base = 0; base < a.P2; base += 32) {
        int i = base + lane;
        int wi = min(i >> 6, 31);
        int sh = i & 63;
        uint64_t w0 = __shfl_sync(0xFFFFFFFFu, myword, wi);
        uint64_t w1 = __shfl_sync(0xFFFFFFFFu, myword, min(wi + 1, 31));
        if (wi + 1 >= a.words) w1 = 0ULL;
        uint64_t v = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
        uint32_t fwd = (uint32_t)v & nmask;                  // bit j = sketch bit i+j
        uint32_t tok = __brev(fwd) >> (32 - a.n);             // first bit most significant
        w.sortbuf[i] = i < a.T ? tok : 0xFFFFFFFFu;
    }
    __syncwarp();
    // bitonic sort (ascending) of P2 entries
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
    // run-length encode
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
    return D;
}

__device__ __forceinline__ void upd(double v, int d, double &best, int &bd) {
    if (v < best || (v == best && d < bd)) {
        best = v;
        bd = d;
    }
}

// CWS argmin over the D distinct tokens in smem, K-fold, write signature row.
__device__ void warp_cws(const SigArgs &a, int64_t row, const WarpSmem &w, int D, int lane) {
    const int S = a.S;
    const int NS = (S + 31) >> 5;
    // split count-1 / count>1 token indices (ascending)
    int n1 = 0, nm = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < D; base += 32) {
        int d = base + lane;
        bool valid = d < D;
        bool one = valid && w.ucnt[d] == 1;
        bool many = valid && !one;
        unsigned m1 = __ballot_sync(0xFFFFFFFFu, one);
        unsigned mm = __ballot_sync(0xFFFFFFFFu, many);
        if (one) w.list1[n1 + __popc(m1 & lt)] = (uint16_t)d;
        if (many) w.listm[nm + __popc(mm & lt)] = (uint16_t)d;
        n1 += __popc(m1);
        nm += __popc(mm);
    }
    __syncwarp();
    double best[SG_NS_MAX];
    int bd[SG_NS_MAX];
#pragma unroll
    for (int i = 0; i < SG_NS_MAX; i++) {
        best[i] = (double)INFINITY;
        bd[i] = 0x7FFFFFFF;
    }
    // count-1 tokens: one gather of the precomputed ln_a1 per (token, slot)
    int e = 0;
    for (; e + 4 <= n1; e += 4) {
        int d0 = w.list1[e], d1 = w.list1[e + 1], d2 = w.list1[e + 2], d3 = w.list1[e + 3];
        const double *p0 = a.lna1 + (size_t)w.utok[d0] * S;
        const double *p1 = a.lna1 + (size_t)w.utok[d1] * S;
        const double *p2 = a.lna1 + (size_t)w.utok[d2] * S;
        const double *p3 = a.lna1 + (size_t)w.utok[d3] * S;
#pragma unroll
        for (int i = 0; i < SG_NS_MAX; i++) {
            if (i < NS) {
                int s = lane + 32 * i;
                if (s < S) {
                    double v0 = __ldg(p0 + s), v1 = __ldg(p1 + s), v2 = __ldg(p2 + s),
                           v3 = __ldg(p3 + s);
                    upd(v0, d0, best[i], bd[i]);
                    upd(v1, d1, best[i], bd[i]);
                    upd(v2, d2, best[i], bd[i]);
                    upd(v3, d3, best[i], bd[i]);
                }
            }
        }
    }
    for (; e < n1; e++) {
        int d0 = w.list1[e];
        const double *p0 = a.lna1 + (size_t)w.utok[d0] * S;
#pragma unroll
        for (int i = 0; i < SG_NS_MAX; i++) {
            int s = lane + 32 * i;
            if (i < NS && s < S) upd(__ldg(p0 + s), d0, best[i], bd[i]);
        }
    }
    // count>1 tokens: full formula, reference op order (wmh.py:74-76)
    for (int f = 0; f < nm; f++) {
        int d0 = w.listm[f];
        size_t base = (size_t)w.utok[d0] * S;
        double lw = __ldg(a.lnw + w.ucnt[d0]);
#pragma unroll
        for (int i = 0; i < SG_NS_MAX; i++) {
            int s = lane + 32 * i;
            if (i < NS && s < S) {
                double r = __ldg(a.tr + base + s);
                double lnc = __ldg(a.tlnc + base + s);
                double b = __ldg(a.tbeta + base + s);
                double t = floor(__dadd_rn(__ddiv_rn(lw, r), b));
                double lny = __dmul_rn(r, __dsub_rn(t, b));
                double v = __dsub_rn(__dsub_rn(lnc, lny), r);
                upd(v, d0, best[i], bd[i]);
            }
        }
    }
    // winners -> keys (wmh.py:79-81)
#pragma unroll
    for (int i = 0; i < SG_NS_MAX; i++) {
        int s = lane + 32 * i;
        if (i < NS && s < S) {
            int d0 = bd[i];
            uint32_t tok = w.utok[d0];
            int c = w.ucnt[d0];
            size_t ent = (size_t)tok * S + s;
            double b = __ldg(a.tbeta + ent);
            double r = __ldg(a.tr + ent);
            double t = floor(__dadd_rn(__ddiv_rn(__ldg(a.lnw + c), r), b));
            uint64_t tt = (uint64_t)(int64_t)t;
            uint64_t key = ssh_mix64((uint64_t)tok ^ ssh_mix64(tt ^ SSH_SALT_KEY));
            w.keys[s] = key;
            if (a.keys_out) a.keys_out[row * S + s] = key;
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

template <int MODE>
__global__ void __launch_bounds__(32 * SG_WARPS) shingle_cws_kernel(SigArgs a) {
    extern __shared__ __align__(16) unsigned char sg_smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    WarpSmem w = carve(sg_smem + (size_t)wid * a.warp_smem, a);
    const int64_t nwarps = (int64_t)gridDim.x * SG_WARPS;
    for (int64_t row = (int64_t)blockIdx.x * SG_WARPS + wid; row < a.N; row += nwarps) {
        int D;
        if (MODE == SIG_MODE_CWS_FROM_SETS) {
            D = a.len_in[row];
            for (int d = lane; d < D; d += 32) {
                w.utok[d] = a.tok_in[row * a.T + d];
                w.ucnt[d] = a.cnt_in[row * a.T + d];
            }
            __syncwarp();
        } else {
            D = warp_shingle(a, row, w, lane);
        }
        if (MODE == SIG_MODE_SHINGLE) {
            for (int d = lane; d < a.T; d += 32) {
                a.tok_out[row * a.T + d] = d < D ? w.utok[d] : 0u;
                a.cnt_out[row * a.T + d] = d < D ? w.ucnt[d] : (uint16_t)0;
            }
            if (lane == 0) a.len_out[row] = D;
            __syncwarp();
        } else {
            warp_cws(a, row, w, D, lane);
        }
    }
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
    a.N = N; a.words = ctx->words; a.nb = ctx->nb; a.n = ctx->p.n; a.T = ctx->T;
    int P2 = 32;
    while (P2 < ctx->T) P2 <<= 1;
    a.P2 = P2;
    a.S = ctx->S; a.L = ctx->p.L; a.K = ctx->p.K;
    int ws = 8 * a.S + 4 * P2 + 4 * a.T + 2 * a.T + 2 * (a.T + 1) + 2 * a.T + 2 * a.T;
    ws = (ws + 15) & ~15;
    a.warp_smem = ws;
    size_t smem = (size_t)ws * SG_WARPS;
    SSH_REQUIRE(smem <= 220 * 1024, SSH_ERR_UNSUPPORTED,
                "signature kernel needs %zu bytes of shared memory (T=%d)", smem, a.T);
    int per_sm = 1;
    int64_t nblk = (N + SG_WARPS - 1) / SG_WARPS;
#define LAUNCH_SIG(MODE_)                                                                     \
    do {                                                                                      \
        auto kern = shingle_cws_kernel<MODE_>;                                                \
        SSH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                      (int)smem));                                            \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * SG_WARPS, smem);    \
        if (per_sm < 1) per_sm = 1;                                                           \
        int grid = (int)std::min<int64_t>(nblk, (int64_t)ctx->num_sms * per_sm);                   \
        kern<<<grid, 32 * SG_WARPS, smem, st>>>(a);                                           \
        SSH_CHECK_LAUNCH();                                                                   \
    } while (0)
    if (mode == SIG_MODE_SHINGLE) LAUNCH_SIG(SIG_MODE_SHINGLE);
    else if (mode == SIG_MODE_CWS_FROM_SETS) LAUNCH_SIG(SIG_MODE_CWS_FROM_SETS);
    else LAUNCH_SIG(SIG_MODE_FUSED);
#undef LAUNCH_SIG
    return SSH_OK;
}
