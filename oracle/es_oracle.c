/* es_oracle.c -- CPU ORACLE for ES-SpMM's sampled SpMM.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this.  It shares no code with the CUDA path (paper_2104_10716_b200/).
 *
 * Plain, slow, obviously correct: one loop over rows (OpenMP over independent rows
 * only; the per-row arithmetic is sequential), fp64 accumulation in slot order,
 * rounded once to fp32.  Every function cites the passage it follows (PAPER.md
 * line numbers, Doc B unless noted; DESIGN.md "Readings" for the silent parts).
 *
 *   Alg. 1 "Pseudo Code of CacheSample"
 *   S = min(row_nnz, shmem_width)            Alg. 1 l.6, L961; "If S exceeds the NNZ of that
 *                                            row, then the whole row is fetched", L986
 *   Bucket: "picks the first S"              L1042-1047
 *   FastRand Eq. 2:
 *     sample_idx = (shmem_idx x P') mod row_nnz, P' = 577     L1064-1067, L1058
 *   acc += sh_data[j] * B[sh_cols[j], col_id]                 Alg. 1 l.13-15, L969-972
 *   in-kernel normalisation by degree (mean)                  L1570-1575 (reading R5: k_i)
 *   sampling rate = sum min(d_i,s) / nnz                      L1290-1303
 *
 * Pins: tests/test_oracle_pins.py (closed forms, SPEC.md worked examples, the paper's
 * Table sample_rate, scipy for s >= max degree, dense brute force on tiny graphs).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC es_oracle.c -o libesoracle.so   (no -ffast-math)
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_BUCKET 1
#define ORACLE_FASTRAND 2
#define ORACLE_SUM 0
#define ORACLE_MEAN 1
#define ORACLE_PRIME 577ull /* P' = 577 */

/* splitmix64 finalizer (reading R6: seeded FastRand offset). */
static uint64_t oracle_mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

uint64_t oracle_hash(uint64_t x) { return oracle_mix64(x); }

/* Reading R6: seed == 0 is exactly Eq. 2; seed != 0 rotates row i's FastRand
 * sequence by off_i = mix64(seed + G*(i+1)) mod d_i, i the GLOBAL row id. */
int64_t oracle_offset(uint64_t seed, int64_t row, int64_t d) {
    if (seed == 0 || d <= 0) return 0;
    uint64_t h = oracle_mix64(seed + 0x9E3779B97F4A7C15ull * (uint64_t)(row + 1));
    return (int64_t)(h % (uint64_t)d);
}

/* Position within the row of sampled slot j (0 <= j < k <= d).
 *   Bucket:   p_j = j                                    (L1043 "first S")
 *   FastRand: p_j = (off + j * P') mod d                 (Eq. 2; off per R6)
 * P' = 577 (L1058) unless overridden (NEXT-4 sensitivity variant; prime <= 0 means 577).
 * 64-bit unsigned arithmetic: j*P' < 2^64 for the sizes used here. */
int64_t oracle_position_p(int32_t strategy, int64_t j, int64_t d, int64_t off, int64_t prime) {
    uint64_t pp = prime > 0 ? (uint64_t)prime : ORACLE_PRIME;
    if (strategy == ORACLE_BUCKET) return j;
    return (int64_t)(((uint64_t)off + (uint64_t)j * pp) % (uint64_t)d);
}

int64_t oracle_position(int32_t strategy, int64_t j, int64_t d, int64_t off) {
    return oracle_position_p(strategy, j, d, off, (int64_t)ORACLE_PRIME);
}

/* k_i = min(d_i, s)   (Alg. 1 l.6, L961) */
static int64_t oracle_k(int64_t d, int64_t s) { return d < s ? d : s; }

/* Sampling rate, PAPER.md:L1290-1303 (Table sample_rate): sum_i min(d_i, s) / nnz;
 * nnz == 0 -> 1.0. */
double oracle_rate(int64_t n_rows, const int64_t* rowptr, int64_t s) {
    int64_t kept = 0, nnz = rowptr[n_rows] - rowptr[0];
    for (int64_t i = 0; i < n_rows; ++i) kept += oracle_k(rowptr[i + 1] - rowptr[i], s);
    return nnz == 0 ? 1.0 : (double)kept / (double)nnz;
}

/* Stage 1 of Alg. 1 materialised (the paper's "pre-sampled graph", L1509-1514):
 * s_rowptr[0..n_rows] = exclusive prefix of k_i; then, if s_colind != NULL, slot j of
 * row i holds (colind, val, position) of nonzero rowptr[i] + p_j, in SLOT order with
 * duplicates kept (reading R2).  row_base = global id of row 0 (for the seeded offset).
 * rowptr entries are absolute offsets into colind/val. */
void oracle_sample(int64_t n_rows, const int64_t* rowptr, const int32_t* colind,
                   const float* val, int64_t s, int32_t strategy, uint64_t seed,
                   int64_t row_base, int64_t prime, int64_t* s_rowptr, int32_t* s_colind,
                   float* s_val, int64_t* s_pos) {
    s_rowptr[0] = 0;
    for (int64_t i = 0; i < n_rows; ++i)
        s_rowptr[i + 1] = s_rowptr[i] + oracle_k(rowptr[i + 1] - rowptr[i], s);
    if (!s_colind) return;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n_rows; ++i) {
        int64_t d = rowptr[i + 1] - rowptr[i];
        int64_t k = oracle_k(d, s);
        int64_t off = strategy == ORACLE_FASTRAND ? oracle_offset(seed, row_base + i, d) : 0;
        for (int64_t j = 0; j < k; ++j) {
            int64_t p = oracle_position_p(strategy, j, d, off, prime);
            int64_t e = rowptr[i] + p;
            int64_t o = s_rowptr[i] + j;
            s_colind[o] = colind[e];
            if (s_val) s_val[o] = val ? val[e] : 1.0f;
            if (s_pos) s_pos[o] = p;
        }
    }
}

/* One output row of the sampled SpMM (Alg. 1 l.5-16 for all col_id of a row):
 *   acc[c] = sum_{j<k} val[e_j] * B[colind[e_j], c]   in fp64, slot order
 *   SUM:  C[c] = fp32(acc[c])
 *   MEAN: C[c] = fp32(acc[c]) / fp32(k)  (IEEE fp32 division), k == 0 -> 0   (R5, R8, R9)
 *         (mean_by_degree: / fp32(d) instead -- the other reading of L1571, NEXT-4) */
static void oracle_row(int64_t d, const int32_t* cols, const float* vals, const float* B,
                       int64_t F, int64_t ldb, int64_t s, int32_t strategy, int64_t off,
                       int32_t reduce, int64_t prime, int32_t mean_by_degree, double* acc,
                       float* Crow) {
    int64_t k = oracle_k(d, s);
    int64_t div = mean_by_degree ? d : k;
    for (int64_t c = 0; c < F; ++c) acc[c] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        int64_t p = oracle_position_p(strategy, j, d, off, prime);
        double a = vals ? (double)vals[p] : 1.0;
        const float* Brow = B + (int64_t)cols[p] * ldb;
        for (int64_t c = 0; c < F; ++c) acc[c] += a * (double)Brow[c];
    }
    for (int64_t c = 0; c < F; ++c) {
        float v = (float)acc[c];
        if (reduce == ORACLE_MEAN) v = div > 0 ? v / (float)div : 0.0f;
        Crow[c] = v;
    }
}

/* C[i, 0:F] for rows i in [0, n_rows) (rows == NULL), or for the n_sel rows listed in
 * rows[] (output row r of C is then global-slice row rows[r]).  Returns -1 on OOM. */
int oracle_spmm(int64_t n_rows, const int64_t* rowptr, const int32_t* colind, const float* val,
                const float* B, int64_t F, int64_t ldb, int64_t s, int32_t strategy,
                uint64_t seed, int32_t reduce, int64_t row_base, int64_t prime,
                int32_t mean_by_degree, const int64_t* rows, int64_t n_sel, float* C, int64_t ldc) {
    int64_t n_out = rows ? n_sel : n_rows;
    int bad = 0;
#pragma omp parallel
    {
        double* acc = (double*)malloc(sizeof(double) * (size_t)(F > 0 ? F : 1));
        if (!acc) {
#pragma omp atomic write
            bad = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < n_out; ++r) {
            if (!acc) continue;
            int64_t i = rows ? rows[r] : r;
            int64_t d = rowptr[i + 1] - rowptr[i];
            int64_t off = strategy == ORACLE_FASTRAND ? oracle_offset(seed, row_base + i, d) : 0;
            oracle_row(d, colind + rowptr[i], val ? val + rowptr[i] : NULL, B, F, ldb, s,
                       strategy, off, reduce, prime, mean_by_degree, acc, C + r * ldc);
        }
        free(acc);
    }
    return bad ? -1 : 0;
}

/* Backward of the sampled SpMM w.r.t. B -- the training variant the paper leaves to future
 * work (§6.2: dynamic sampling "could accelerate GNN training").
 * Over the SAME sampled slots as the forward (Alg. 1 positions, Eq. 2, R6 rotation):
 *   dB[col_ij, c] += w_ij * dC[i, c],   w_ij = val[e_ij] (SUM)  or  val[e_ij] / k_i (MEAN)
 * i.e. dB = A_s^T dC with A_s the (row-scaled for MEAN) sampled matrix.  Rows in order,
 * slots in order, fp64 accumulation, rounded once to fp32 and ADDED to dB (n_cols x ldb).
 * Single-threaded on purpose (one obvious summation order).  Returns -1 on OOM. */
int oracle_spmm_backward(int64_t n_rows, const int64_t* rowptr, const int32_t* colind,
                         const float* val, const float* dC, int64_t F, int64_t ldc, int64_t s,
                         int32_t strategy, uint64_t seed, int32_t reduce, int64_t row_base,
                         int64_t prime, int32_t mean_by_degree, int64_t n_cols, float* dB,
                         int64_t ldb) {
    double* acc = (double*)calloc((size_t)(n_cols > 0 ? n_cols : 1) * (size_t)(F > 0 ? F : 1),
                                  sizeof(double));
    if (!acc) return -1;
    for (int64_t i = 0; i < n_rows; ++i) {
        int64_t d = rowptr[i + 1] - rowptr[i];
        int64_t k = oracle_k(d, s);
        int64_t off = strategy == ORACLE_FASTRAND ? oracle_offset(seed, row_base + i, d) : 0;
        for (int64_t j = 0; j < k; ++j) {
            int64_t e = rowptr[i] + oracle_position_p(strategy, j, d, off, prime);
            double w = val ? (double)val[e] : 1.0;
            if (reduce == ORACLE_MEAN) w /= (double)(mean_by_degree ? d : k);
            double* row = acc + (int64_t)colind[e] * F;
            for (int64_t c = 0; c < F; ++c) row[c] += w * (double)dC[i * ldc + c];
        }
    }
    for (int64_t r = 0; r < n_cols; ++r)
        for (int64_t c = 0; c < F; ++c) dB[r * ldb + c] += (float)acc[r * F + c];
    free(acc);
    return 0;
}

/* fp32 TIMING MODE (SURVEY 8(d) "fp32-FMA mode for timing, like the paper's kernel"): the same
 * rows, slots and order as oracle_row, but acc[c] = fmaf(val, B, acc[c]) in fp32 -- the
 * arithmetic a straightforward CPU port of Alg. 1 performs.  Used only to time the CPU
 * baseline; parity always uses the fp64 oracle_spmm.  Pinned by tests/test_oracle_pins.py
 * (B = 1 counts exactly; within the sequential-sum bound gamma_k of oracle_spmm). */
/* compiled for the FMA instruction set (the CPU's vfmadd, not libm's software fmaf) where the host
 * has it -- oracle_spmm_f32 checks at run time and uses the portable copy otherwise */
#define ORACLE_ROW_F32_BODY                                                                        \
    int64_t k = oracle_k(d, s);                                                                    \
    for (int64_t c = 0; c < F; ++c) acc[c] = 0.0f;                                                 \
    for (int64_t j = 0; j < k; ++j) {                                                              \
        int64_t p = oracle_position_p(strategy, j, d, off, (int64_t)ORACLE_PRIME);                 \
        float a = vals ? vals[p] : 1.0f;                                                           \
        const float* Brow = B + (int64_t)cols[p] * ldb;                                            \
        for (int64_t c = 0; c < F; ++c) acc[c] = fmaf(a, Brow[c], acc[c]);                         \
    }                                                                                              \
    for (int64_t c = 0; c < F; ++c) {                                                              \
        float v = acc[c];                                                                          \
        if (reduce == ORACLE_MEAN) v = k > 0 ? v / (float)k : 0.0f;                                \
        Crow[c] = v;                                                                               \
    }
#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target("fma")))
static void oracle_row_f32_fma(int64_t d, const int32_t* cols, const float* vals, const float* B,
                               int64_t F, int64_t ldb, int64_t s, int32_t strategy, int64_t off,
                               int32_t reduce, float* acc, float* Crow) {
    ORACLE_ROW_F32_BODY
}
#endif
static void oracle_row_f32(int64_t d, const int32_t* cols, const float* vals, const float* B,
                           int64_t F, int64_t ldb, int64_t s, int32_t strategy, int64_t off,
                           int32_t reduce, float* acc, float* Crow) {
#if defined(__x86_64__) && defined(__GNUC__)
    if (__builtin_cpu_supports("fma")) {
        oracle_row_f32_fma(d, cols, vals, B, F, ldb, s, strategy, off, reduce, acc, Crow);
        return;
    }
#endif
    ORACLE_ROW_F32_BODY
}
#if 0
    int64_t k = oracle_k(d, s);
    for (int64_t c = 0; c < F; ++c) acc[c] = 0.0f;
    for (int64_t j = 0; j < k; ++j) {
        int64_t p = oracle_position_p(strategy, j, d, off, (int64_t)ORACLE_PRIME);
        float a = vals ? vals[p] : 1.0f;
        const float* Brow = B + (int64_t)cols[p] * ldb;
        for (int64_t c = 0; c < F; ++c) acc[c] = fmaf(a, Brow[c], acc[c]);
    }
    for (int64_t c = 0; c < F; ++c) {
        float v = acc[c];
        if (reduce == ORACLE_MEAN) v = k > 0 ? v / (float)k : 0.0f;
        Crow[c] = v;
    }
}
#endif

int oracle_spmm_f32(int64_t n_rows, const int64_t* rowptr, const int32_t* colind, const float* val,
                    const float* B, int64_t F, int64_t ldb, int64_t s, int32_t strategy, uint64_t seed,
                    int32_t reduce, const int64_t* rows, int64_t n_sel, float* C, int64_t ldc) {
    int64_t n_out = rows ? n_sel : n_rows;
    int bad = 0;
#pragma omp parallel
    {
        float* acc = (float*)malloc(sizeof(float) * (size_t)(F > 0 ? F : 1));
        if (!acc) {
#pragma omp atomic write
            bad = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < n_out; ++r) {
            if (!acc) continue;
            int64_t i = rows ? rows[r] : r;
            int64_t d = rowptr[i + 1] - rowptr[i];
            int64_t off = strategy == ORACLE_FASTRAND ? oracle_offset(seed, i, d) : 0;
            oracle_row_f32(d, colind + rowptr[i], val ? val + rowptr[i] : NULL, B, F, ldb, s, strategy, off,
                           reduce, acc, C + r * ldc);
        }
        free(acc);
    }
    return bad ? -1 : 0;
}

/* OpenMP threads of the calls that follow (the single-thread CPU baseline time). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
