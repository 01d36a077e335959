// common.cuh — shared device/host helpers for libsshgpu (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/sshgpu.h"

#define SSH_MAX_W 256
#define SSH_MAX_N 20          // table-based CWS: 2^n x S variates resident in HBM
#define SSH_MAX_SLOTS 256     // K*L
#define SSH_MAX_K 16384       // top-k per query (shared-memory top-k state: 12 B per next_pow2(k))
#define SSH_SALT_KEY 0xEB44ACCAB455D165ULL

// --------------------------------------------------------------- errors
void ssh_set_error(const char *fmt, ...);
int ssh_cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define SSH_CUDA(call)                                                           \
    do {                                                                         \
        cudaError_t _e = (call);                                                 \
        if (_e != cudaSuccess) return ssh_cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

void ssh_count_launch();
// Device-side bounds assertions of the checked build (-DSSH_CHECKED; the
// sanitizers are not available on the GPU pool): a failed check traps the
// kernel, which surfaces as a CUDA error at the next call.  No code otherwise.
#ifdef SSH_CHECKED
#define SSH_DASSERT(cond)                                                                       \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("SSH_DASSERT failed: %s at %s:%d (block %d, thread %d)\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define SSH_DASSERT(cond) \
    do {                  \
    } while (0)
#endif

#define SSH_CHECK_LAUNCH()          \
    do {                            \
        ssh_count_launch();         \
        SSH_CUDA(cudaGetLastError()); \
    } while (0)

#define SSH_REQUIRE(cond, code, ...)       \
    do {                                   \
        if (!(cond)) {                     \
            ssh_set_error(__VA_ARGS__);    \
            return (code);                 \
        }                                  \
    } while (0)

// --------------------------------------------------------------- context
struct ssh_ctx {
    int device = 0;
    int num_sms = 148;
    bool have_params = false;
    ssh_params p{};
    int nb = 0;      // sketch bits per series
    int words = 0;   // u64 words per bit row
    int T = 0;       // tokens per series
    int S = 0;       // K*L slots
    int max_count = 0;
    double h_ln2 = 0.0;  // host ln(2) from the uploaded ln(count) table
    float screen_c = 0.f;  // |dot32 - dot64| <= screen_c * max|x|  (sketch.cu)
    float h_w32[SSH_MAX_W];  // filter rounded to f32 (host copy, passed as kernel params)
    double *d_w64 = nullptr;  // filter f64[W]
    float *d_w32 = nullptr;   // filter rounded to f32
    double *d_r = nullptr, *d_lnc = nullptr, *d_beta = nullptr, *d_lna1 = nullptr;
    double *d_lnw = nullptr;  // ln(count)
    void *d_rank = nullptr;   // per-slot rank of ln_a1 by (value, token): u16 (n <= 16) or u32
    // order-free CWS path (n <= 15, S <= 128; signature.cu):
    //  rankp  u16 ranks padded to 16*rank_ql slots per token row (pad = 0xFFFF)
    //  byrank per (slot, rank): {f64 ln_a1, u32 token | floor(beta) << 16, pad}
    //  rlcb   per (token, slot): f64 {r, 1/r, ln c, beta}
    uint16_t *d_rankp = nullptr;
    uint4 *d_byrank = nullptr;
    double *d_rlcb = nullptr;
    double *d_edge = nullptr;  // per (token 0 | 2^n-1, count, slot): {ln_a, t} (order-free CWS)  // per (token, slot): ln_a for count 2 (order-free CWS)
    int rank_ql = 0;  // 0: path unavailable
    size_t tab_entries = 0;
    // profiling (ssh_ctx_set_profiling)
    int profile = 0;
    double prof[24] = {0};
    unsigned long long *d_cells = nullptr;  // device counters: [0] DTW cells evaluated,
                                            // [1] LB_PAA prunes, [2] LB_Keogh prunes,
                                            // [3] members visited by the filter
    // side stream for independent build work (candidate envelopes), joined by events
    cudaStream_t side = nullptr;
    cudaStream_t copy = nullptr;  // host->device series chunks (ssh_build_index_host)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_copy = nullptr;
    // phase clock of the last ssh_query_batch (query_index timings "hash",
    // "probe", "rerank", index.py:235,265): events at the phase boundaries of
    // every query chunk, accumulated without extra host syncs
    cudaEvent_t qev[4] = {nullptr, nullptr, nullptr, nullptr};
    double qphase[3] = {0, 0, 0};
    bool qpending = false;  // the last chunk's rerank span is not folded in yet
    // named grow-only scratch slots reused across calls (stream-ordered)
    void *slot_ptr[32] = {nullptr};
    size_t slot_bytes[32] = {0};
};

enum {
    SLOT_BITS = 0,       // ssh_signatures: packed sketch bits
    SLOT_RS_KEYS_A,      // ssh_index_build radix sort
    SLOT_RS_KEYS_B,
    SLOT_RS_ROWS_B,
    SLOT_RS_HIST,
    SLOT_Q_FIXED,        // ssh_query_batch: per-query fixed-size arrays
    SLOT_Q_BITMAP,
    SLOT_Q_SURV,
    SLOT_Q_SURV_LB,
    SLOT_Q_W2,
    SLOT_Q_D2,
    SLOT_Q_RESC,
    SLOT_Q_D64,
    SLOT_Q_HIST,
    SLOT_Q_D32,
    SLOT_Q_TOPK,
    SLOT_SIG,
    SLOT_Q_KEEP,
    SLOT_Q_KEEP_D,
    SLOT_Q_WLB,
    SLOT_Q_KHIST,
    SLOT_Q_POOLA,
    SLOT_Q_POOLB,
    SLOT_Q_POOLCNT,
    SLOT_Q_QPAD,
    SLOT_Q_BSHIST,
    SLOT_COUNT
};

struct ssh_index {
    int L = 0;
    // rerank summaries (ssh_index_summarize / ssh_build_index), one per row:
    //  rec[row]   64 B: {lo, sc, x0, x_last} + u8 PAA codes of the segment
    //             means (seg samples per segment, nseg <= SSH_REC_CODES)
    //  codes[row] cstride B: u8 sample codes x8[mp] then (U8, L8)[mp] pairs of
    //             the row's +-radius envelope
    // Decoding is dec(c) = fmaf(c, sc, lo) (fp32); every code brackets its
    // value exactly: dec(x8) <= x <= dec(x8 + 1), dec(U8) >= U, dec(L8) <= L,
    // and dec(pc) <= segment mean <= dec(pc + 1).  Rows with non-finite
    // values have sc = NaN, which turns every bound on them into 0; a row
    // where some segment mean lies within the f64 error margin of a grid
    // point stores -sc (decoders use |sc|; the PAA key then ignores its codes).
    void *rec = nullptr;
    uint8_t *codes = nullptr;
    int seg = 0, nseg = 0, mp = 0;
    int64_t cstride = 0;
    int64_t N = 0;
    int64_t id_base = 0;
    int device = 0;
    uint64_t *keys = nullptr;     // concatenated unique keys, table j at kbase[j]
    uint32_t *offsets = nullptr;  // concatenated offsets, table j at kbase[j] + j (nb+1 entries)
    uint32_t *ids = nullptr;      // L x N local row ids
    int64_t *h_nb = nullptr;      // host: buckets per table
    int64_t *h_kbase = nullptr;   // host: bucket base per table
    int64_t *d_nb = nullptr;      // device copies
    int64_t *d_kbase = nullptr;
    int64_t total_buckets = 0;
    // last stream-ordered use (build, summaries, probe, query): destroy makes
    // its frees wait on it, so a caller working on any stream can drop the
    // index while its last query is still in flight
    cudaEvent_t last_use = nullptr;
    // sketch statistics of the build (device i64[2], ssh_build_index*):
    // [0] windows re-evaluated in exact f64, [1] of those |dot| < 1e-9
    int64_t *d_sketch_stats = nullptr;
};

// record ix's last use on `st` (see ssh_index::last_use)
void ssh_index_touch(const ssh_index *ix, cudaStream_t st);

// grow-only named scratch slot; returns pointer or nullptr (error set)
void *ssh_slot(ssh_ctx *ctx, int slot, size_t bytes, cudaStream_t st);

#define SSH_REC_CODES 48  // PAA codes per 64-byte series record

// rerank summaries of N rows into ix (allocates rec/codes if needed)
int ssh_launch_summaries(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t N, int64_t ld, cudaStream_t st);
// allocate ix's summaries for N rows / summarise rows [r0, r0 + n) of X (row r0 at X)
int ssh_alloc_summaries(ssh_ctx *ctx, ssh_index *ix, int64_t N, cudaStream_t st);
int ssh_launch_summaries_rows(ssh_ctx *ctx, ssh_index *ix, const float *X, int64_t r0, int64_t n, int64_t ld,
                              cudaStream_t st);

// ----------------------------------------------------------- device math
__host__ __device__ __forceinline__ uint64_t ssh_mix64(uint64_t x) {
    // splitmix64 finalizer (wmh.py:34-44)
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline int ssh_div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// kernel launchers implemented per translation unit
int ssh_launch_sketch(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
                      int64_t *stats, cudaStream_t st);
int ssh_launch_shingle_cws(ssh_ctx *ctx, const uint64_t *bits, const uint32_t *tok_in,
                           const uint16_t *cnt_in, const int32_t *len_in, int64_t N,
                           uint32_t *tok_out, uint16_t *cnt_out, int32_t *len_out,
                           uint64_t *keys_out, uint64_t *sig_out, int mode, cudaStream_t st);
int ssh_launch_lna1(ssh_ctx *ctx, cudaStream_t st);
int ssh_build_ranks(ssh_ctx *ctx, cudaStream_t st);
int ssh_sort_columns(ssh_ctx *ctx, const uint64_t *rowmajor, int64_t N, int L, uint32_t *rows_out,
                     uint64_t **keys_sorted, cudaStream_t st);

enum { SIG_MODE_SHINGLE = 1, SIG_MODE_CWS_FROM_SETS = 2, SIG_MODE_FUSED = 3 };
