// merge.cu — cross-shard top-k merge: the exact global top-k
// of a series-sharded index is the (d2, id)-lexicographic merge of the
// per-shard top-k lists (each already sorted by (d2, id), padded with
// id -1 / d2 +inf), as the reference's final lexsort over R would order them
// (index.py:249-268).  One warp per query: lane j holds the head of list j and
// every output slot is a warp argmin over the heads (lists <= 32).
#include "common.cuh"

namespace {

// (d2, id) key with padding (id < 0) after every real entry, ids ascending
__device__ __forceinline__ bool mk_less(double da, long long ia, double db, long long ib) {
    const unsigned long long ua = ia < 0 ? ~0ULL : (unsigned long long)ia;
    const unsigned long long ub = ib < 0 ? ~0ULL : (unsigned long long)ib;
    return da < db || (da == db && ua < ub);
}

__global__ void merge_topk_kernel(const long long *__restrict__ ids, const double *__restrict__ d2, int nq,
                                  int lists, int k_in, int k_out, long long *__restrict__ out_ids,
                                  double *__restrict__ out_d2, int *__restrict__ n_out) {
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q >= nq) return;
    // list j of query q: ids[(j * nq + q) * k_in + t] (all_gather layout)
    const bool have = lane < lists;
    const long long *li = ids + ((int64_t)lane * nq + q) * k_in;
    const double *ld = d2 + ((int64_t)lane * nq + q) * k_in;
    int pos = 0;
    double hd = INFINITY;
    long long hi = -1;
    auto load = [&]() {
        if (have && pos < k_in) {
            hi = li[pos];
            hd = hi < 0 ? INFINITY : ld[pos];
        } else {
            hi = -1;
            hd = INFINITY;
        }
    };
    load();
    int n = 0;
    for (int t = 0; t < k_out; t++) {
        double bd = hd;
        long long bi = hi;
        int bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
            const long long oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
            const int ol = __shfl_xor_sync(0xFFFFFFFFu, bl, o);
            if (mk_less(od, oi, bd, bi) || (od == bd && oi == bi && ol < bl)) {
                bd = od;
                bi = oi;
                bl = ol;
            }
        }
        if (lane == 0) {
            out_ids[(int64_t)q * k_out + t] = bi;
            out_d2[(int64_t)q * k_out + t] = bi < 0 ? INFINITY : bd;
        }
        n += bi >= 0;
        if (lane == bl) {
            pos++;
            load();
        }
    }
    if (lane == 0 && n_out) n_out[q] = n;
}

}  // namespace

extern "C" int ssh_merge_topk(const int64_t *ids, const double *d2, int32_t nq, int32_t lists, int32_t k_in,
                              int32_t k_out, int64_t *out_ids, double *out_d2, int32_t *n_out, void *stream) {
    SSH_REQUIRE(nq >= 0 && lists >= 1 && lists <= 32 && k_in >= 1 && k_out >= 1, SSH_ERR_INVALID,
                "ssh_merge_topk: nq=%d lists=%d (1..32) k_in=%d k_out=%d", nq, lists, k_in, k_out);
    SSH_REQUIRE(nq == 0 || (ids && d2 && out_ids && out_d2), SSH_ERR_INVALID, "ssh_merge_topk: NULL argument");
    if (nq == 0) return SSH_OK;
    const int warps = 4;
    merge_topk_kernel<<<(nq + warps - 1) / warps, 32 * warps, 0, (cudaStream_t)stream>>>(
        (const long long *)ids, d2, nq, lists, k_in, k_out, (long long *)out_ids, out_d2, n_out);
    ssh_count_launch();
    SSH_CUDA(cudaGetLastError());
    return SSH_OK;
}
