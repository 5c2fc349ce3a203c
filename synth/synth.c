/* synth.c -- seeded synthetic inputs shared by the oracle tests and the CUDA path.
 *
 * This module holds none of ES-SpMM's arithmetic (no sampling, no SpMM).  It only
 * draws the column indices of a CSR graph for a given degree sequence and the
 * dense feature matrix B, both from a counter-based generator so the output is
 * independent of the thread count and chunking.
 *
 *   col draw: row i draws d_i DISTINCT columns with
 *   probability proportional to the column node's degree (Chung-Lu popularity),
 *   sorted ascending (SPEC.md:L82 canonical order).
 *   B[j, c] = (mix64(seed + G*(j*F + c + 1)) >> 40) * 2^-24, in [0, 1).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC synth.c -o libsynth.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

uint64_t synth_mix64(uint64_t x) { return mix64(x); }

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* first index j with cumw[j] > u  (cumw inclusive prefix sums, strictly increasing
 * when every weight >= 1) */
static inline int32_t upper_bound_i64(const int64_t* cumw, int64_t n, uint64_t u) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)cumw[mid] > u) hi = mid; else lo = mid + 1;
    }
    return (int32_t)lo;
}

static int64_t unique_sorted(int32_t* a, int64_t n) {
    if (n == 0) return 0;
    int64_t m = 1;
    for (int64_t i = 1; i < n; ++i)
        if (a[i] != a[m - 1]) a[m++] = a[i];
    return m;
}

/* Returns 0 on success, -1 if some row asks for more distinct columns than exist. */
int synth_columns(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                  const int64_t* cumw, uint64_t seed, int32_t* colind) {
    int64_t maxd = 0;
    for (int64_t i = 0; i < n_rows; ++i) {
        int64_t d = rowptr[i + 1] - rowptr[i];
        if (d > maxd) maxd = d;
    }
    if (maxd > n_cols) return -1;
    const uint64_t total = (uint64_t)cumw[n_cols - 1];
    int failed = 0;
#pragma omp parallel
    {
        int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * maxd + 1));
        unsigned char* used = NULL;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n_rows; ++i) {
            int64_t d = rowptr[i + 1] - rowptr[i];
            int32_t* out = colind + rowptr[i];
            if (d == 0) continue;
            if (d == n_cols) {            /* complete row */
                for (int64_t j = 0; j < d; ++j) out[j] = (int32_t)j;
                continue;
            }
            const uint64_t base = mix64(seed + GOLDEN * (uint64_t)(i + 1));
            uint64_t ctr = 0;
            int64_t m = 0;
            int rounds = 0;
            while (m < d && rounds < 256) {
                for (int64_t j = m; j < d; ++j) {
                    uint64_t r = mix64(base + GOLDEN * (++ctr));
                    uint64_t u = (uint64_t)(((unsigned __int128)r * total) >> 64);
                    buf[j] = upper_bound_i64(cumw, n_cols, u);
                }
                qsort(buf, (size_t)d, sizeof(int32_t), cmp_i32);
                m = unique_sorted(buf, d);
                ++rounds;
            }
            if (m < d) {                  /* pathological weights: top up uniformly-unused */
                if (!used) used = (unsigned char*)malloc((size_t)n_cols);
                if (!used) { failed = 1; continue; }
                memset(used, 0, (size_t)n_cols);
                for (int64_t j = 0; j < m; ++j) used[buf[j]] = 1;
                for (int64_t c = 0; c < n_cols && m < d; ++c)
                    if (!used[c]) buf[m++] = (int32_t)c;
                qsort(buf, (size_t)d, sizeof(int32_t), cmp_i32);
            }
            memcpy(out, buf, sizeof(int32_t) * (size_t)d);
        }
        free(buf);
        free(used);
    }
    return failed ? -2 : 0;
}

/* B[j, c] for j < n, c < f; columns f..ld-1 are zero padding. */
void synth_dense(int64_t n, int64_t f, int64_t ld, uint64_t seed, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        float* row = out + j * ld;
        for (int64_t c = 0; c < f; ++c) {
            uint64_t r = mix64(seed + GOLDEN * (uint64_t)(j * f + c + 1));
            row[c] = (float)(r >> 40) * (1.0f / 16777216.0f);
        }
        for (int64_t c = f; c < ld; ++c) row[c] = 0.0f;
    }
}

/* Seeded keys for a node-id permutation (argsort of keys = permutation). */
void synth_perm_keys(int64_t n, uint64_t seed, uint64_t* keys) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) keys[i] = mix64(seed + GOLDEN * (uint64_t)(i + 1));
}
