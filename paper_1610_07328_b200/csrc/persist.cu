// persist.cu — host-side parsing of the SSHI index file's table section
// (index.py:279-396, load_index): per table a bucket count u64, then per
// bucket key u64, id count u64, ids u64[count].  The reference walks this
// with a Python loop per bucket; here one pass per table rebuilds the
// signature column (signatures[ids, j] = key, index.py:379-389) with the same
// validity checks: ids inside [0, N) and every id exactly once per table.
// No device work: callable without a GPU.
#include <stdio.h>
#include <string.h>

#include <vector>

#include "common.cuh"

extern "C" int ssh_sshi_parse_tables(const uint8_t *buf, int64_t len, int64_t off, int32_t L, int64_t N,
                                     uint64_t *sig, int64_t *end_off, char *msg, int32_t msg_len) {
    SSH_REQUIRE(buf && sig && end_off && msg && msg_len > 0, SSH_ERR_INVALID, "ssh_sshi_parse_tables: NULL argument");
    msg[0] = 0;
    std::vector<uint8_t> seen((size_t)N);
    auto word = [&](int64_t at) {
        uint64_t v;
        memcpy(&v, buf + at, 8);  // little-endian host (x86-64 / aarch64)
        return v;
    };
    for (int j = 0; j < L; j++) {
        if (off + 8 > len) {
            snprintf(msg, msg_len, "truncated index file (needed 8 bytes at offset %lld)", (long long)off);
            return 1;
        }
        const uint64_t nb = word(off);
        off += 8;
        std::fill(seen.begin(), seen.end(), 0);
        int64_t total = 0;
        for (uint64_t b = 0; b < nb; b++) {
            if (off + 16 > len) {
                snprintf(msg, msg_len, "truncated index file (needed 16 bytes at offset %lld)", (long long)off);
                return 1;
            }
            const uint64_t key = word(off), cnt = word(off + 8);
            off += 16;
            if (cnt > (uint64_t)(len - off) / 8) {
                snprintf(msg, msg_len, "truncated index file (needed %llu bytes at offset %lld)",
                         (unsigned long long)(cnt * 8), (long long)off);
                return 1;
            }
            for (uint64_t e = 0; e < cnt; e++) {
                const int64_t id = (int64_t)word(off + 8 * (int64_t)e);
                if (id < 0 || id >= N) {
                    snprintf(msg, msg_len, "table %d references ids outside [0, %lld)", j, (long long)N);
                    return 2;
                }
                if (seen[(size_t)id]) {
                    snprintf(msg, msg_len, "table %d holds id %lld more than once", j, (long long)id);
                    return 2;
                }
                seen[(size_t)id] = 1;
                sig[(size_t)id * L + j] = key;
            }
            off += 8 * (int64_t)cnt;
            total += (int64_t)cnt;
        }
        if (total != N) {
            snprintf(msg, msg_len, "table %d holds %lld ids, expected every id exactly once (%lld)", j,
                     (long long)total, (long long)N);
            return 2;
        }
    }
    *end_off = off;
    return SSH_OK;
}
