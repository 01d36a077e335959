// ctx.cu — context, parameter/table upload, error reporting, stage wrappers.
#include <math.h>
#include <stdarg.h>

#include <new>

#include "common.cuh"

#include <atomic>

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void ssh_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" int64_t ssh_launch_count(void) { return g_launches.load(); }

extern "C" int ssh_ctx_set_profiling(ssh_ctx *ctx, int on) {
    SSH_REQUIRE(ctx != nullptr, SSH_ERR_INVALID, "ssh_ctx_set_profiling: ctx is NULL");
    SSH_CUDA(cudaSetDevice(ctx->device));
    if (on && !ctx->d_cells) SSH_CUDA(cudaMalloc(&ctx->d_cells, 8 * sizeof(unsigned long long)));
    if (ctx->d_cells) SSH_CUDA(cudaMemset(ctx->d_cells, 0, 8 * sizeof(unsigned long long)));
    for (int i = 0; i < 24; i++) ctx->prof[i] = 0.0;
    ctx->profile = on;
    return SSH_OK;
}

extern "C" int ssh_ctx_profile(const ssh_ctx *ctx, double *out, int n) {
    SSH_REQUIRE(ctx && out, SSH_ERR_INVALID, "ssh_ctx_profile: NULL argument");
    for (int i = 0; i < n && i < 24; i++) out[i] = ctx->prof[i];
    if (n > 6 && ctx->d_cells) {
        unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        SSH_CUDA(cudaMemcpy(c, ctx->d_cells, sizeof(c), cudaMemcpyDeviceToHost));
        out[6] = (double)c[0];
        if (n > 12) {
            out[10] = (double)c[1];
            out[11] = (double)c[2];
            out[12] = (double)c[3];
        }
        if (n > 7) out[7] = (double)c[4];  // bytes of codes read by the wave LB
        if (n > 20) out[20] = (double)c[5];  // DTW lane-cells executed (incl. idle lanes)
    }
    return SSH_OK;
}

void ssh_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int ssh_cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    ssh_set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    return e == cudaErrorMemoryAllocation ? SSH_ERR_OOM : SSH_ERR_CUDA;
}

extern "C" const char *ssh_last_error(void) { return g_err; }
extern "C" int ssh_abi_version(void) { return SSHGPU_ABI_VERSION; }

void *ssh_slot(ssh_ctx *ctx, int slot, size_t bytes, cudaStream_t st) {
    if (bytes <= ctx->slot_bytes[slot]) return ctx->slot_ptr[slot];
    if (ctx->slot_ptr[slot]) cudaFreeAsync(ctx->slot_ptr[slot], st);
    ctx->slot_ptr[slot] = nullptr;
    ctx->slot_bytes[slot] = 0;
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMallocAsync(&ctx->slot_ptr[slot], want, st);
    if (e != cudaSuccess) {
        ssh_cuda_fail(e, "cudaMallocAsync(scratch slot)", __FILE__, __LINE__);
        ctx->slot_ptr[slot] = nullptr;
        return nullptr;
    }
    ctx->slot_bytes[slot] = want;
    return ctx->slot_ptr[slot];
}

extern "C" int ssh_ctx_create(int device, ssh_ctx **out) {
    SSH_REQUIRE(out != nullptr, SSH_ERR_INVALID, "ssh_ctx_create: out is NULL");
    int ndev = 0;
    SSH_CUDA(cudaGetDeviceCount(&ndev));
    SSH_REQUIRE(device >= 0 && device < ndev, SSH_ERR_INVALID,
                "ssh_ctx_create: device %d out of range [0, %d)", device, ndev);
    SSH_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    SSH_CUDA(cudaGetDeviceProperties(&prop, device));
    SSH_REQUIRE(prop.major == 10, SSH_ERR_UNSUPPORTED,
                "ssh_ctx_create: device %d is sm_%d%d; libsshgpu is built for sm_100a only",
                device, prop.major, prop.minor);
    // keep freed stream-ordered allocations cached in the device pool
    // (the query batch and the table build allocate scratch per call)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    ssh_ctx *c = new (std::nothrow) ssh_ctx();
    SSH_REQUIRE(c != nullptr, SSH_ERR_OOM, "ssh_ctx_create: host allocation failed");
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return ssh_cuda_fail(cudaGetLastError(), "ssh_ctx_create streams", __FILE__, __LINE__);
    }
    *out = c;
    return SSH_OK;
}

static void free_tables(ssh_ctx *c) {
    cudaFree(c->d_w64); cudaFree(c->d_w32);
    cudaFree(c->d_r); cudaFree(c->d_lnc); cudaFree(c->d_beta); cudaFree(c->d_lna1);
    cudaFree(c->d_lnw);
    cudaFree(c->d_rank);
    c->d_rank = nullptr;
    cudaFree(c->d_rankp); cudaFree(c->d_byrank); cudaFree(c->d_rlcb);
    cudaFree(c->d_edge);
    c->d_edge = nullptr;
    c->d_rankp = nullptr; c->d_byrank = nullptr; c->d_rlcb = nullptr;
    c->rank_ql = 0;
    c->d_w64 = nullptr; c->d_w32 = nullptr; c->d_r = c->d_lnc = c->d_beta = c->d_lna1 = nullptr;
    c->d_lnw = nullptr;
}

extern "C" int ssh_ctx_destroy(ssh_ctx *ctx) {
    if (!ctx) return SSH_OK;
    cudaSetDevice(ctx->device);
    free_tables(ctx);
    cudaDeviceSynchronize();
    for (int i = 0; i < 32; i++)
        if (ctx->slot_ptr[i]) cudaFree(ctx->slot_ptr[i]);
    if (ctx->d_cells) cudaFree(ctx->d_cells);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    for (int i = 0; i < 4; i++)
        if (ctx->qev[i]) cudaEventDestroy(ctx->qev[i]);
    delete ctx;
    return SSH_OK;
}

extern "C" int ssh_ctx_set_params(ssh_ctx *ctx, const ssh_params *p, const double *filter,
                                  const double *tab_r, const double *tab_lnc,
                                  const double *tab_beta, const double *ln_w,
                                  int32_t max_count) {
    SSH_REQUIRE(ctx && p && filter && tab_r && tab_lnc && tab_beta && ln_w, SSH_ERR_INVALID,
                "ssh_ctx_set_params: NULL argument");
    // index.py:44-68 validation (messages mirror the reference's ConfigError)
    SSH_REQUIRE(p->W >= 1 && p->W <= SSH_MAX_W, SSH_ERR_UNSUPPORTED,
                "filter length W must be in [1, %d] on device, got %d", SSH_MAX_W, p->W);
    SSH_REQUIRE(p->delta >= 1, SSH_ERR_INVALID, "step size delta must be >= 1, got %d", p->delta);
    SSH_REQUIRE(p->n >= 1 && p->n <= SSH_MAX_N, SSH_ERR_UNSUPPORTED,
                "shingle length n must be in [1, %d] on device, got %d", SSH_MAX_N, p->n);
    SSH_REQUIRE(p->L >= 1 && p->K >= 1 && (int64_t)p->L * p->K <= SSH_MAX_SLOTS,
                SSH_ERR_UNSUPPORTED, "K*L must be in [1, %d] on device, got K=%d L=%d",
                SSH_MAX_SLOTS, p->K, p->L);
    SSH_REQUIRE(p->m >= p->W, SSH_ERR_INVALID, "series length t=%d violates t >= W (W=%d)",
                p->m, p->W);
    int nb = (p->m - p->W) / p->delta + 1;
    SSH_REQUIRE(nb >= p->n, SSH_ERR_INVALID,
                "sketch length floor((t-W)/delta)+1 = %d violates >= n (t=%d, W=%d, delta=%d, n=%d)",
                nb, p->m, p->W, p->delta, p->n);
    SSH_REQUIRE(p->radius >= 0, SSH_ERR_INVALID, "radius must be >= 0, got %d", p->radius);
    int T = nb - p->n + 1;
    SSH_REQUIRE(max_count >= T, SSH_ERR_INVALID,
                "ln_w table must cover counts up to %d (got max_count=%d)", T, max_count);
    SSH_REQUIRE(T <= 4095, SSH_ERR_UNSUPPORTED,
                "tokens per series %d exceeds the device limit 4095 (series too long)", T);
    SSH_CUDA(cudaSetDevice(ctx->device));
    free_tables(ctx);
    ctx->have_params = false;
    ctx->p = *p;
    ctx->nb = nb;
    ctx->words = (nb + 63) / 64;
    ctx->T = T;
    ctx->S = p->K * p->L;
    ctx->max_count = max_count;
    ctx->h_ln2 = max_count >= 2 ? ln_w[2] : 0.0;
    double l1 = 0.0;
    float w32[SSH_MAX_W];
    for (int k = 0; k < p->W; k++) {
        l1 += fabs(filter[k]);
        w32[k] = (float)filter[k];
        ctx->h_w32[k] = w32[k];
    }
    // |fl32(sum x*w32) - fl64(sum x*w)| <= (W+2) u sum|x||w| (1+1e-4), u = 2^-24;
    // 1% slack absorbs the f32 evaluation of this bound (sketch.cu).
    ctx->screen_c = (float)((p->W + 2) * ldexp(1.0, -24) * 1.01 * l1);

    size_t ent = ((size_t)1 << p->n) * (size_t)ctx->S;
    ctx->tab_entries = ent;
    SSH_CUDA(cudaMalloc(&ctx->d_w64, sizeof(double) * p->W));
    SSH_CUDA(cudaMalloc(&ctx->d_w32, sizeof(float) * p->W));
    SSH_CUDA(cudaMalloc(&ctx->d_r, sizeof(double) * ent));
    SSH_CUDA(cudaMalloc(&ctx->d_lnc, sizeof(double) * ent));
    SSH_CUDA(cudaMalloc(&ctx->d_beta, sizeof(double) * ent));
    SSH_CUDA(cudaMalloc(&ctx->d_lna1, sizeof(double) * ent));
    SSH_CUDA(cudaMalloc(&ctx->d_lnw, sizeof(double) * (max_count + 1)));
    SSH_CUDA(cudaMemcpy(ctx->d_w64, filter, sizeof(double) * p->W, cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMemcpy(ctx->d_w32, w32, sizeof(float) * p->W, cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMemcpy(ctx->d_r, tab_r, sizeof(double) * ent, cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMemcpy(ctx->d_lnc, tab_lnc, sizeof(double) * ent, cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMemcpy(ctx->d_beta, tab_beta, sizeof(double) * ent, cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMemcpy(ctx->d_lnw, ln_w, sizeof(double) * (max_count + 1),
                        cudaMemcpyHostToDevice));
    SSH_CUDA(cudaMalloc(&ctx->d_rank, (p->n <= 16 ? 2 : 4) * ent));
    int rc = ssh_launch_lna1(ctx, 0);
    if (rc) return rc;
    rc = ssh_build_ranks(ctx, 0);
    if (rc) return rc;
    SSH_CUDA(cudaDeviceSynchronize());
    ctx->have_params = true;
    return SSH_OK;
}

extern "C" int ssh_num_sketch_bits(const ssh_ctx *ctx) { return ctx && ctx->have_params ? ctx->nb : -1; }
extern "C" int ssh_sketch_words(const ssh_ctx *ctx) { return ctx && ctx->have_params ? ctx->words : -1; }
extern "C" int ssh_tokens_per_series(const ssh_ctx *ctx) { return ctx && ctx->have_params ? ctx->T : -1; }

#define REQUIRE_PARAMS(ctx, fn)                                                          \
    SSH_REQUIRE((ctx) != nullptr, SSH_ERR_INVALID, fn ": ctx is NULL");                 \
    SSH_REQUIRE((ctx)->have_params, SSH_ERR_STATE, fn ": ssh_ctx_set_params not called"); \
    SSH_CUDA(cudaSetDevice((ctx)->device))

extern "C" int ssh_sketch(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *bits,
                          int64_t *stats, void *stream) {
    REQUIRE_PARAMS(ctx, "ssh_sketch");
    SSH_REQUIRE(N >= 0 && ld >= ctx->p.m, SSH_ERR_INVALID,
                "ssh_sketch: bad shape N=%lld ld=%lld (m=%d)", (long long)N, (long long)ld, ctx->p.m);
    if (N == 0) return SSH_OK;
    SSH_REQUIRE(X && bits, SSH_ERR_INVALID, "ssh_sketch: NULL pointer");
    return ssh_launch_sketch(ctx, X, N, ld, bits, stats, (cudaStream_t)stream);
}

extern "C" int ssh_shingle(ssh_ctx *ctx, const uint64_t *bits, int64_t N, uint32_t *tokens,
                           uint16_t *counts, int32_t *set_len, void *stream) {
    REQUIRE_PARAMS(ctx, "ssh_shingle");
    if (N == 0) return SSH_OK;
    SSH_REQUIRE(bits && tokens && counts && set_len, SSH_ERR_INVALID, "ssh_shingle: NULL pointer");
    return ssh_launch_shingle_cws(ctx, bits, nullptr, nullptr, nullptr, N, tokens, counts, set_len,
                                  nullptr, nullptr, SIG_MODE_SHINGLE, (cudaStream_t)stream);
}

extern "C" int ssh_cws(ssh_ctx *ctx, const uint32_t *tokens, const uint16_t *counts,
                       const int32_t *set_len, int64_t N, uint64_t *keys, uint64_t *sig,
                       void *stream) {
    REQUIRE_PARAMS(ctx, "ssh_cws");
    if (N == 0) return SSH_OK;
    SSH_REQUIRE(tokens && counts && set_len && sig, SSH_ERR_INVALID, "ssh_cws: NULL pointer");
    return ssh_launch_shingle_cws(ctx, nullptr, tokens, counts, set_len, N, nullptr, nullptr,
                                  nullptr, keys, sig, SIG_MODE_CWS_FROM_SETS, (cudaStream_t)stream);
}

extern "C" int ssh_signatures(ssh_ctx *ctx, const float *X, int64_t N, int64_t ld, uint64_t *sig,
                              int64_t *stats, void *stream) {
    REQUIRE_PARAMS(ctx, "ssh_signatures");
    SSH_REQUIRE(N >= 0 && ld >= ctx->p.m, SSH_ERR_INVALID, "ssh_signatures: bad shape");
    if (N == 0) return SSH_OK;
    SSH_REQUIRE(X && sig, SSH_ERR_INVALID, "ssh_signatures: NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *bits = (uint64_t *)ssh_slot(ctx, SLOT_BITS, sizeof(uint64_t) * (size_t)N * ctx->words, st);
    if (!bits) return SSH_ERR_OOM;
    int rc = ssh_launch_sketch(ctx, X, N, ld, bits, stats, st);
    if (rc) return rc;
    return ssh_launch_shingle_cws(ctx, bits, nullptr, nullptr, nullptr, N, nullptr, nullptr,
                                  nullptr, nullptr, sig, SIG_MODE_FUSED, st);
}
