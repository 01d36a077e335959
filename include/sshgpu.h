/*
 * sshgpu.h — C-ABI of the B200-native SSH (Sketch, Shingle & Hash) hot path.
 *
 * One shared library, libsshgpu.so (sm_100a, static cudart), exports these
 * entry points.  Signatures use plain pointers and sizes only: device
 * pointers are caller-owned (the Python host allocates them with PyTorch),
 * `stream` is a cudaStream_t passed as void*, and every call is
 * stream-ordered.  Functions return SSH_OK (0) or a negative error code;
 * ssh_last_error() returns a thread-local message for the last failure.
 *
 * Each entry point names the reference function it replaces
 * (/root/reference/pkg/src/sshts/<file>:<line>).  The reference itself has
 * no C ABI — it is a Python package — so the "binding a maintainer would
 * add" is a ctypes stub; paper_1610_07328_b200/_native.py
 * is exactly that binding.
 */
#ifndef SSHGPU_H
#define SSHGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSHGPU_ABI_VERSION 1

enum {
    SSH_OK = 0,
    SSH_ERR_INVALID = -1,     /* bad argument (message names it)            */
    SSH_ERR_CUDA = -2,        /* CUDA runtime failure                        */
    SSH_ERR_OOM = -3,         /* device allocation failed                    */
    SSH_ERR_UNSUPPORTED = -4, /* parameter outside the device path's range   */
    SSH_ERR_STATE = -5        /* call order violated (e.g. params not set)   */
};

/* Pipeline parameters: SshParams (index.py:32-56) + K (concatenation order,
 * wmh.py:107-125) + the series length and the DTW radius
 * r = int(round(band * m)) (dtw.py:38-39), resolved by the host. */
typedef struct ssh_params {
    int32_t m;      /* series length t                            */
    int32_t W;      /* filter length                              */
    int32_t delta;  /* filter step                                */
    int32_t n;      /* shingle length (device path: 1..20)        */
    int32_t L;      /* number of tables (SshParams.d)             */
    int32_t K;      /* CWS samples concatenated per table key     */
    uint64_t seed;  /* master seed (filter + CWS)                 */
    int32_t radius; /* Sakoe-Chiba radius r                       */
    int32_t reserved;
} ssh_params;

typedef struct ssh_ctx ssh_ctx;     /* per device: params, filter, CWS tables */
typedef struct ssh_index ssh_index; /* per shard: L CSR bucket tables          */

const char *ssh_last_error(void);
int ssh_abi_version(void);
/* Kernels launched by this library so far (process-wide, monotonic). */
int64_t ssh_launch_count(void);

/* Context for `device`; owns the uploaded filter and CWS tables. */
int ssh_ctx_create(int device, ssh_ctx **out);
int ssh_ctx_destroy(ssh_ctx *ctx);

/* Upload parameters and host tables (all HOST pointers):
 *   filter  f64[W]              make_filter (sketch.py:36-43), index.py:162
 *   tab_r, tab_lnc, tab_beta    f64[2^n][L*K], layout [token][slot]: the CWS
 *                               variates r, ln c, beta of wmh.py:60-72
 *   ln_w    f64[max_count+1]    np.log(count) of wmh.py:72 (entry 0 unused)
 * Replaces the stateless variate evaluation inside _cws_keys (wmh.py:52-81):
 * the device never evaluates log(), so keys are bit-identical to the
 * reference for the host's numpy. */
int ssh_ctx_set_params(ssh_ctx *ctx, const ssh_params *p, const double *filter,
                       const double *tab_r, const double *tab_lnc, const double *tab_beta,
                       const double *ln_w, int32_t max_count);

/* Optional per-phase device timing of ssh_query_batch (CUDA events; adds no
 * host syncs beyond the batch's own).  ssh_ctx_profile fills up to n (<= 24)
 * values, accumulated since profiling was enabled:
 * [0] query signatures ms, [1] probe + bitmap ms, [2] member keys + sort ms,
 * [3] wave LB ms, [4] wave fp32 DTW ms, [5] rescore + top-k ms,
 * [6] DTW cells evaluated (alive lane-rows x band), [7] bytes read by the
 * wave LB, [8] fp32 DTWs started, [9] rescored pairs, [10] key prunes
 * (LB_PAA / LB_Kim), [11] LB_Keogh prunes, [12] members visited,
 * [13]/[14]/[15] sum of first-wave / final thr over the exact k-th distance
 * and their count, [16] waves, [17] sum over waves of active queries,
 * [18] query sub-ranges, [19] overflow rounds, [20] DTW lane-cells executed. */
int ssh_ctx_set_profiling(ssh_ctx *ctx, int on);
int ssh_ctx_profile(const ssh_ctx *ctx, double *out, int n);

/* Sizes derived from the parameters. */
int ssh_num_sketch_bits(const ssh_ctx *ctx);   /* N_B  (sketch.py:46-48)      */
int ssh_sketch_words(const ssh_ctx *ctx);      /* ceil(N_B/64)                */
int ssh_tokens_per_series(const ssh_ctx *ctx); /* N_B - n + 1                 */

/* K1 — sketch_matrix (sketch.py:69-89) / sketch_values (sketch.py:51-61).
 * X: f32[N][ld] device.  bits: u64[N][words], bit i of a row = window i
 * has dot >= 0 (+1).  stats (device i64[2] or NULL, accumulated):
 * [0] windows re-evaluated in exact f64, [1] windows with |dot| < 1e-9. */
int ssh_sketch(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
               int64_t *stats, void *stream);

/* K2 — tokenize_bits + np.unique(return_counts) (shingle.py:56-75,
 * index.py:118).  Per series: distinct tokens ascending with counts, in rows
 * of T = N_B-n+1 slots; set_len[i] = number of distinct tokens. */
int ssh_shingle(ssh_ctx *ctx, const uint64_t *bits, int64_t N, uint32_t *tokens,
                uint16_t *counts, int32_t *set_len, void *stream);

/* K3 — _cws_keys + signature(concat=K) (wmh.py:52-81, 107-125).
 * keys: u64[N][L*K] raw slot keys (or NULL); sig: u64[N][L] folded keys. */
int ssh_cws(ssh_ctx *ctx, const uint32_t *tokens, const uint16_t *counts,
            const int32_t *set_len, int64_t N, uint64_t *keys, uint64_t *sig, void *stream);

/* K1->K3 fused — compute_signatures (index.py:123-138) with the K fold and
 * query_signature (index.py:175-181).  sig: u64[N][L]. */
int ssh_signatures(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *sig,
                   int64_t *stats, void *stream);

/* K4 — _tables_from_signatures (index.py:141-156): per table a stable
 * radix sort of (key, id) -> CSR (sorted unique keys, offsets, ids ascending
 * within each bucket).  Ids are id_base + row.  Synchronises `stream` once
 * to read back bucket counts. */
int ssh_index_build(ssh_ctx *ctx, const uint64_t *sig, int64_t N, int64_t id_base,
                    ssh_index **out, void *stream);
/* K1 -> K4 fused — build_index (index.py:159-172): signatures (written to
 * sig_out u64[N][L] when non-NULL), bucket tables and the shard's rerank
 * summaries (64-byte series records + u8 sample/envelope codes, computed on a
 * side stream).  X stays owned by the caller and is read by later queries. */
int ssh_build_index(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, int64_t id_base,
                    uint64_t *sig_out, ssh_index **out, void *stream);
/* Same from HOST series (pinned memory for copy/compute overlap): rows are
 * copied in 65536-row chunks into the caller's device buffer X_dev (N x ld
 * f32, kept for queries) while the previous chunk is sketched, signed and
 * summarised; sig_out (u64[N][L], device) is required. */
int ssh_build_index_host(ssh_ctx *ctx, const float *X_host, int64_t N, int64_t ld, int64_t id_base,
                         float *X_dev, uint64_t *sig_out, ssh_index **out, void *stream);
int ssh_index_destroy(ssh_index *idx);
/* An index without bucket tables over N series (summaries only): queries on
 * it search the whole shard exactly — exact_search (dtw.py:293-326). */
int ssh_index_create_bare(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, int64_t id_base,
                          ssh_index **out, void *stream);
/* make_dataset (core.py:162-169) on the device: windows of length t every
 * `stride` samples of the f64 recording rec[len] (stride 1 = the reference's
 * extract_subsequences, core.py:138-146), z-normalised per window exactly as
 * numpy's float64 mean/std (z_normalize_dataset, core.py:127-135) when
 * normalize != 0; written as f32 (out32) and/or f64 (out64) [count][t] with
 * count = (len - t) / stride + 1. */
int ssh_windows(const double *rec, int64_t len, int32_t t, int64_t stride, int32_t normalize, float *out32,
                double *out64, int64_t *count, void *stream);
/* srp_matrix (index.py:420-423): out i8[N][bits] = +1 if X[i] . V[j] >= 0
 * else -1; V64 f64[bits][m] (default_rng([seed, j]) rows, host-drawn) and
 * V32 its f32 rounding.  fp32 tiled product with an error bound, fp64
 * sequential recheck of the undecided signs (counted in *nrecheck). */
int ssh_srp(const float *X, int64_t N, int32_t m, const float *V32, const double *V64, int32_t bits,
            int8_t *out, unsigned long long *nrecheck, void *stream);
/* srp_matrix (index.py:420-423) with the f32 product on the tensor cores
 * (tcgen05.mma kind::tf32, accumulator in TMEM) when tensor_cores != 0 and
 * bits <= 256, else SIMT fp32; signs within the rigorous product error bound
 * are re-evaluated as a sequential f64 dot of the original values: X64
 * (device f64 [N][m], may be NULL) when the input was float64, else X.
 * nrecheck (device u64, may be NULL) counts the re-evaluated signs. */
int ssh_srp2(const float *X, const double *X64, int64_t N, int32_t m, const float *V32, const double *V64,
             int32_t bits, int8_t *out, unsigned long long *nrecheck, int32_t tensor_cores, void *stream);
/* Host-only: parse the per-table section of an SSHI index file
 * (index.py:279-396, load_index) starting at byte `off` into the signature
 * matrix sig u64[N][L] (signatures[ids, j] = key), checking ids in [0, N) and
 * every id exactly once per table.  Returns 0, 1 (truncated) or 2 (invalid)
 * with a message in msg; *end_off = offset after the last table. */
int ssh_sshi_parse_tables(const uint8_t *buf, int64_t len, int64_t off, int32_t L, int64_t N, uint64_t *sig,
                          int64_t *end_off, char *msg, int32_t msg_len);
int ssh_index_num_buckets(const ssh_index *idx, int table, int64_t *n_buckets);
int64_t ssh_index_size(const ssh_index *idx);
/* Sketch statistics of the build that made idx (ssh_build_index /
 * ssh_build_index_host; zeros for an index built from signatures), copied to
 * HOST out2[2] after synchronising `stream`: [0] windows whose f32 screen was
 * undecided and were re-evaluated with the reference's exact f64 sequence,
 * [1] of those, windows with |dot| < 1e-9 (near-zero sign ties, counted and
 * reported per BASELINE.json's north star; sign(0) = +1 as sketch.py:60). */
int ssh_index_sketch_stats(const ssh_index *idx, int64_t *out2, void *stream);
/* Cross-shard top-k merge (multi-GPU query): the exact
 * global top-k_out of a series-sharded index from the per-shard lists.
 * ids i64 / d2 f64 [lists][nq][k_in] (device; the all_gather layout), each
 * list sorted by (d2, id) and padded with id -1 / d2 +inf; out_ids /
 * out_d2 [nq][k_out] and n_out[nq] (may be NULL) on the device.  Order:
 * (d2, id) lexicographic, as the reference's final lexsort (index.py:249).
 * lists <= 32.  Replaces the per-query sort of the merged lists. */
int ssh_merge_topk(const int64_t *ids, const double *d2, int32_t nq, int32_t lists, int32_t k_in,
                   int32_t k_out, int64_t *out_ids, double *out_d2, int32_t *n_out, void *stream);
/* Copy table `table` to HOST arrays: keys u64[nb], offsets i64[nb+1],
 * ids i64[N] (global ids).  The reference's dict view (index.py:151-154). */
int ssh_index_export(const ssh_index *idx, int table, uint64_t *keys, int64_t *offsets,
                     int64_t *ids, void *stream);

/* Rerank summaries of the shard (device): PAA segment means of every row
 * (32-sample segments, f64 sums stored f32) and max|x|.  They feed the
 * LB_PAA bound of ssh_query_batch; build_index computes them right after
 * the tables (ssh_query_batch computes them lazily if absent).  X is the
 * shard the index was built over, f32[N][ld] device. */
int ssh_index_summarize(ssh_ctx *ctx, ssh_index *idx, const float *X, int64_t ld, void *stream);

/* Copy the rerank summaries of rows [r0, r0 + n) out of the index (inspection
 * and tests): rec_out receives 64 B per row, codes_out *cstride B per row
 * (u8 sample codes x8[mp], then (U8, L8) pairs).  Either buffer may be NULL;
 * both may be host or device memory.  *mp, *cstride report the layout. */
int ssh_index_copy_summaries(const ssh_index *idx, int64_t r0, int64_t n, void *rec_out,
                             void *codes_out, int32_t *mp, int64_t *cstride, void *stream);

/* K6 — probe_candidates (index.py:184-190) for a batch: membership bitmap
 * u32[nq][ceil(N/32)] of the deduplicated bucket union (bit = local row),
 * and n_cand[nq] = |R|.  qsig: u64[nq][L] device. */
int ssh_probe(ssh_ctx *ctx, const ssh_index *idx, const uint64_t *qsig, int32_t nq,
              uint32_t *bitmap, int64_t *n_cand, void *stream);

/* K5..K10 — query_index (index.py:204-273) for a batch of nq queries:
 * hash, probe, LB_Kim/LB_Keogh/LB_Keogh2-gated banded DTW (fp32) and exact
 * fp64 rescoring of the top-k boundary set.  X: f32[N][m] device (the
 * shard), Q: f32[nq][m] device.  Outputs (device): ids i64[nq][k] (global,
 * -1 padded), d2 f64[nq][k] squared DTW (bit-identical to dtw.py:83-121),
 * n_out i32[nq], n_cand i64[nq] (|R|), counters i64[nq][5] =
 * [kim_pruned, keogh_pruned, keogh2_pruned, dtw_computed, dtw_abandoned]
 * (SearchStats, dtw.py:50-72; batch-order semantics),
 * status i32[nq] = 0 "ok", 1 "no-candidates", 2 "fallback" (index.py:99).
 * 1 <= k <= 16384 (larger: SSH_ERR_UNSUPPORTED); k > N answers with N entries.
 * Any number of tied candidates is answered (the rescoring lists grow and the
 * query slice reruns), as the reference cascade does (dtw.py:171-236). */
#define SSH_QUERY_FALLBACK_ON_EMPTY 1 /* empty R -> exact search over the shard
                                         (query_index(fallback_on_empty=True),
                                         index.py:239-243) */
#define SSH_QUERY_EXACT 2             /* R = the whole shard, no probe (exact_search,
                                         dtw.py:293-326); implied for bare indexes */
int ssh_query_batch(ssh_ctx *ctx, const ssh_index *idx, const float *X, const float *Q,
                    int32_t nq, int32_t k, int32_t flags, int64_t *ids, double *d2,
                    int32_t *n_out, int64_t *n_cand, int64_t *counters, int32_t *status,
                    void *stream);

/* Device time (ms) of the phases of the last ssh_query_batch on ctx,
 * summed over its query chunks: [0] query signatures ("hash"), [1] probe +
 * candidate bitmap ("probe"), [2] bounds + DTW rerank + top-k ("rerank") —
 * the phases of query_index's timings dict (index.py:224-235,265).  Waits
 * for the batch's last event. */
int ssh_query_phase_ms(ssh_ctx *ctx, double *out3);

/* Exact f64 banded DTW (dtw.py:83-121, FMA-free, no abandon) of npair
 * (query row, series row) pairs; rows index X / Q.  d2: f64[npair]. */
int ssh_dtw_exact(ssh_ctx *ctx, const float *X, const float *Q, const int32_t *qrow,
                  const int64_t *xrow, int64_t npair, double *d2, void *stream);

/* ---- the reference's public DTW utilities (dtw.py:239-284), float64 on the
 * device in the reference's operation order.  All arrays are device f64,
 * row-major [rows][m]; row index arrays may be NULL (= identity). */

/* dtw_distance (dtw.py:239-250) / _dtw_band_sq (dtw.py:83-121): squared
 * banded DTW of X[xrow[p]] vs Y[yrow[p]]; abandon_sq >= 0 enables the
 * row-minimum abandon (+inf).  Band-chunked warp wavefront (any radius). */
int ssh_dtw_pairs64(const double *X, const double *Y, const int64_t *xrow, const int64_t *yrow,
                    int64_t npair, int32_t m, int32_t r, double abandon_sq, double *out_sq, void *stream);
/* build_envelope (dtw.py:262-268) / _envelope_into (dtw.py:124-151): running
 * max / min over [i - r, i + r] of each row. */
int ssh_envelope64(const double *X, int64_t n, int32_t m, int32_t r, double *upper, double *lower,
                   void *stream);
/* lb_keogh (dtw.py:271-276) / _lb_keogh_sq (dtw.py:154-168): squared
 * excursion of each row of C outside the envelope (one envelope shared by
 * every row when env_rows == 1, else one per row). */
int ssh_lb_keogh64(const double *C, const double *U, const double *Lo, int64_t n, int32_t m,
                   int32_t env_rows, double *out_sq, void *stream);
/* lb_kim (dtw.py:252-260): sqrt of the first and last squared differences. */
int ssh_lb_kim64(const double *X, const double *Y, int64_t n, int32_t m, double *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SSHGPU_H */
