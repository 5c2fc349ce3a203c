// es_abi.cu -- the extern "C" boundary (include/es_spmm.h): argument validation,
// kernel selection, the host-buffer pipeline and the row partitioner.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "es_internal.h"
#include "es_spmm.h"

namespace {

std::atomic<int64_t> g_launches{0};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

es_status_t check_common(int64_t n_rows, int64_t n_cols, int64_t F, int64_t ldb, int64_t ldc,
                         int32_t s, int32_t strategy, int32_t reduce) {
    if (n_rows < 0 || n_cols < 0 || F < 1 || ldb < F || ldc < F || s < 1) return ES_ERR_INVALID_VALUE;
    if (strategy != ES_BUCKET && strategy != ES_FASTRAND) return ES_ERR_INVALID_VALUE;
    if (reduce != ES_REDUCE_SUM && reduce != ES_REDUCE_MEAN) return ES_ERR_INVALID_VALUE;
    return ES_OK;
}

struct Opts {
    uint32_t prime = 577;
    int32_t mean_by_degree = 0;
    int32_t bf16 = 0;
    float* const* c_peers = nullptr;
    int32_t n_peers = 0;
    int32_t deterministic = 0;
    void* workspace = nullptr;
    int64_t workspace_bytes = 0;
    int32_t reuse_sampled = 0;
};

es_status_t read_opts(const es_spmm_options_t* o, Opts* out) {
    *out = Opts{};
    if (!o) return ES_OK;
    if (o->struct_size < (int32_t)offsetof(es_spmm_options_t, c_peers)) return ES_ERR_INVALID_VALUE;
    if (o->prime < 0) return ES_ERR_INVALID_VALUE;
    if (o->mean_divisor != ES_MEAN_BY_SAMPLED && o->mean_divisor != ES_MEAN_BY_DEGREE) return ES_ERR_INVALID_VALUE;
    if (o->b_dtype != ES_DTYPE_F32 && o->b_dtype != ES_DTYPE_BF16) return ES_ERR_INVALID_VALUE;
    out->prime = o->prime == 0 ? 577u : (uint32_t)o->prime;
    out->mean_by_degree = o->mean_divisor == ES_MEAN_BY_DEGREE;
    out->bf16 = o->b_dtype == ES_DTYPE_BF16;
    if (o->struct_size >= (int32_t)offsetof(es_spmm_options_t, deterministic)) {
        if (o->n_peers < 0 || (o->n_peers > 0 && !o->c_peers)) return ES_ERR_INVALID_VALUE;
        out->c_peers = o->c_peers;
        out->n_peers = o->n_peers;
    }
    if (o->struct_size >= (int32_t)offsetof(es_spmm_options_t, workspace)) out->deterministic = o->deterministic != 0;
    if (o->struct_size >= (int32_t)offsetof(es_spmm_options_t, reuse_sampled)) {
        if (o->workspace_bytes < 0 || (o->workspace_bytes > 0 && !o->workspace)) return ES_ERR_INVALID_VALUE;
        out->workspace = o->workspace;
        out->workspace_bytes = o->workspace_bytes;
    }
    if (o->struct_size >= (int32_t)sizeof(es_spmm_options_t)) out->reuse_sampled = o->reuse_sampled != 0;
    return ES_OK;
}

// ---- slab path (es_slab.cu): when, and the workspace layout
constexpr int64_t kSlabF = 64;                       // floats per feature slice (256-B slab rows)

int64_t env_i64(const char* name, int64_t dflt) {
    const char* e = getenv(name);
    return e ? atoll(e) : dflt;
}

// Run time (a workspace was passed): the slab path runs whenever it can -- F > 16 and a
// 64-float slab of B (n_cols x 256 B) fits L2.  ES_SPMM_SLAB=0 disables, =1 forces.
bool slab_feasible(int64_t n_cols, int64_t F) {
    const int64_t force = env_i64("ES_SPMM_SLAB", -1);
    if (force == 0 || F <= kSlabF / 4) return false;
    if (force == 1) return true;
    return n_cols * kSlabF * 4 <= (env_i64("ES_SPMM_SLAB_MAX_SLAB_MB", 80) << 20);
}

// es_spmm_workspace_bytes's choice (measured, profiles/r01.md "Slab path" and the s-sweep in
// BASELINE.md): feasible, F >= 128, and rows that sample enough slots on average -- the bound
// used is min(s, nnz / n_rows) >= 128 for F > 128 (several slices: Reddit-shaped F=602 s=128
// 5.8 -> 4.95 ms, s=256 9.8 -> 7.8 ms) and >= 192 for F <= 128 (two slices; at s=128 the fused
// two-slot ring is 1-6 % faster, at s=192 the slab path wins 1.50 -> 1.39 ms).  Below that each
// slice pass's per-row start-up outweighs the L2-resident gathers (Reddit F=602 s=16: 2.0 vs
// 4.5 TFLOP/s), and short rows (Arxiv-shaped, mean degree 14) keep the fused kernel.
bool slab_wanted(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t s) {
    if (!slab_feasible(n_cols, F)) return false;
    if (env_i64("ES_SPMM_SLAB", -1) == 1) return true;
    const int64_t mean_deg = n_rows > 0 ? nnz / n_rows : 0;
    const int64_t k_est = s < mean_deg ? s : mean_deg;
    const int64_t min_k = env_i64("ES_SPMM_SLAB_MIN_K", F > 128 ? 128 : 192);
    return F >= env_i64("ES_SPMM_SLAB_MIN_F", 128) && k_est >= min_k;
}

int64_t slab_align(int64_t x) { return (x + 255) & ~(int64_t)255; }

struct SlabLayout {
    int64_t off_rowptr, off_temp, temp_bytes, off_col, off_val, bytes_fixed;
};
SlabLayout slab_layout(int64_t n) {
    SlabLayout L{};
    L.off_rowptr = 0;
    L.off_temp = slab_align(8 * (n + 1));
    L.temp_bytes = (int64_t)es::slab_scan_temp_bytes(n);
    L.off_col = slab_align(L.off_temp + L.temp_bytes);
    L.bytes_fixed = L.off_col;
    return L;
}

// The workspace's sampled-slot arrays (es_spmm_sample layout); false if it holds no slot.
struct SlabSlots {
    int64_t* s_rowptr;
    int32_t* s_col;
    float* s_val;
    int64_t cap;
    void* temp;
    size_t temp_bytes;
};
bool slab_slots(const Opts& o, int64_t n, bool has_val, SlabSlots* out) {
    const SlabLayout L = slab_layout(n);
    const int64_t per_slot = has_val ? 8 : 4;
    const int64_t cap = (o.workspace_bytes - L.bytes_fixed - 256) / per_slot;
    if (cap < 1) return false;
    char* ws = static_cast<char*>(o.workspace);
    out->s_rowptr = reinterpret_cast<int64_t*>(ws + L.off_rowptr);
    out->s_col = reinterpret_cast<int32_t*>(ws + L.off_col);
    out->s_val = has_val ? reinterpret_cast<float*>(ws + slab_align(L.off_col + 4 * cap)) : nullptr;
    out->cap = cap;
    out->temp = ws + L.off_temp;
    out->temp_bytes = (size_t)L.temp_bytes;
    return true;
}
// a1-a3 once into the workspace: count, scan, materialise
cudaError_t slab_sample(const SlabSlots& sl, const int64_t* rowptr, int64_t nnz_base, const int32_t* colind,
                        const float* val, int64_t n, int32_t s, int32_t strategy, uint64_t seed, int64_t row_begin,
                        uint32_t prime, cudaStream_t st, int* launches) {
    cudaError_t err = es::launch_slab_count(rowptr, n, s, sl.s_rowptr, sl.temp, sl.temp_bytes, st, launches);
    if (err != cudaSuccess) return err;
    err = es::launch_sample_materialize(rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, prime,
                                        sl.s_rowptr, sl.s_col, sl.s_val, nullptr, st, sl.cap);
    ++*launches;
    return err;
}

es_status_t run_rows_impl(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, int64_t nnz_base,
                          const int32_t* colind, const float* val, const void* B, int64_t F,
                          int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                          float* C, int64_t ldc, int64_t row_begin, int64_t row_end,
                          const Opts& o, cudaStream_t st) {
    es_status_t rc = check_common(n_rows, n_cols, F, ldb, ldc, s, strategy, reduce);
    if (rc != ES_OK) return rc;
    if (row_begin < 0 || row_end < row_begin || row_end > n_rows) return ES_ERR_INVALID_VALUE;
    const int64_t n = row_end - row_begin;
    if (n == 0) return ES_OK;
    if (!rowptr || !C || (n_cols > 0 && !B)) return ES_ERR_INVALID_VALUE;
    es::SpmmParams p{};
    p.rowptr = rowptr;
    p.nnz_base = nnz_base;
    p.colind = colind;
    p.val = val;
    p.B = static_cast<const float*>(B);
    p.F = F;
    p.ldb = ldb;
    p.s = s;
    p.strategy = strategy;
    p.seed = seed;
    p.reduce = reduce;
    p.C = C;
    p.ldc = ldc;
    p.n_rows = n;
    p.row_base = row_begin;
    p.prime = o.prime;
    p.mean_by_degree = o.mean_by_degree;
    p.b_bf16 = o.bf16;
    p.c_peers = o.c_peers;
    p.n_peers = o.n_peers;
    const es::Plan plan = o.bf16 ? es::make_plan_bf16(F, ldb, ldc, B, C) : es::make_plan(F, ldb, ldc, B, C, s);
    if (plan.unsupported) return ES_ERR_UNSUPPORTED;
    const uintptr_t bu = reinterpret_cast<uintptr_t>(B), cu = reinterpret_cast<uintptr_t>(C);
    // any C layout: 16-B vector stores where C's rows allow them, scalar stores otherwise
    const bool c_vec16 = cu % 16 == 0 && ldc % 4 == 0;
    if (o.workspace && bu % 16 == 0 && ldb % (o.bf16 ? 8 : 4) == 0 && slab_feasible(n_cols, F)) {
        SlabSlots sl;
        int launches = 0;
        cudaError_t err = cudaSuccess;
        if (slab_slots(o, n, val != nullptr, &sl)) {
            // Bucket takes the first k_i entries of each row: they already lie contiguous in the
            // CSR (Alg. 1 with p_j = j), so the passes read them in place -- no sampling pass
            const bool direct = strategy == ES_BUCKET;
            if (!o.reuse_sampled && !direct)
                err = slab_sample(sl, rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, o.prime, st,
                                  &launches);
            const int stages = (int)env_i64("ES_SPMM_SLAB_STAGES", 4);
            const int lanes = (int)env_i64("ES_SPMM_SLAB_G", 8);
            // slices of 256-B slab rows: 64 fp32 or 128 bf16 elements
            const int64_t wsl = o.bf16 ? 2 * kSlabF : kSlabF;
            for (int64_t c0 = 0; err == cudaSuccess && c0 < F; c0 += wsl) {
                es::SlabParams sp{};
                sp.s_rowptr = direct ? rowptr : sl.s_rowptr;
                sp.slot_base = direct ? nnz_base : 0;
                sp.cap = direct ? INT64_MAX : sl.cap;
                sp.s_colind = direct ? colind : sl.s_col;
                sp.s_val = direct ? val : sl.s_val;
                sp.direct_s = direct ? s : 0;
                sp.rowptr = rowptr;
                sp.b_bf16 = o.bf16;
                sp.B = o.bf16 ? reinterpret_cast<const float*>(static_cast<const uint16_t*>(B) + c0)
                              : static_cast<const float*>(B) + c0;
                sp.ldb = ldb;
                sp.w = (int32_t)(F - c0 < wsl ? F - c0 : wsl);
                sp.nv = o.bf16 ? (sp.w + 7) / 8 : (sp.w + 3) / 4;
                sp.C = C + c0;
                sp.c_peers = o.c_peers;
                sp.n_peers = o.n_peers;
                sp.row_base = row_begin;
                sp.col0 = c0;
                sp.ldc = ldc;
                sp.c_vec = c_vec16 ? 1 : 0;
                sp.n_rows = n;
                sp.reduce = reduce;
                sp.mean_by_degree = o.mean_by_degree;
                err = es::launch_slab_pass(sp, lanes, stages, st);
                ++launches;
            }
            g_launches.fetch_add(launches, std::memory_order_relaxed);
            return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
        }
    }
    cudaError_t err = es::launch_spmm(p, plan, st);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

}  // namespace

extern "C" {

const char* es_status_string(es_status_t status) {
    switch (status) {
        case ES_OK: return "ES_OK";
        case ES_ERR_INVALID_VALUE: return "ES_ERR_INVALID_VALUE";
        case ES_ERR_MISALIGNED: return "ES_ERR_MISALIGNED";
        case ES_ERR_UNSUPPORTED: return "ES_ERR_UNSUPPORTED";
        case ES_ERR_CUDA: return "ES_ERR_CUDA";
    }
    return "ES_ERR_UNKNOWN";
}

int64_t es_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int64_t es_spmm_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb,
                                int32_t s, int32_t has_val) {
    if (n_rows <= 0 || n_cols < 0 || nnz < 0 || F < 1 || ldb < F || s < 1) return 0;
    if (!slab_wanted(n_rows, n_cols, nnz, F, s)) return 0;
    const SlabLayout L = slab_layout(n_rows);
    const int64_t cap = nnz < n_rows * (int64_t)s ? nnz : n_rows * (int64_t)s;
    return L.bytes_fixed + 256 + slab_align(4 * (cap > 0 ? cap : 1)) + (has_val ? 4 * (cap > 0 ? cap : 1) : 0) + 256;
}

es_status_t es_spmm_plan(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C,
                         char* buf, int32_t buf_len) {
    if (F < 1 || ldb < F || ldc < F || !buf || buf_len < 1) return ES_ERR_INVALID_VALUE;
    const es::Plan pl = es::make_plan(F, ldb, ldc, B, C);
    if (pl.tma)
        snprintf(buf, (size_t)buf_len, "es::spmm_tma<nch%d,stages%d>(rows/warp %d)%s", pl.nch, pl.stages,
                 pl.rows_per_warp, pl.c_vec ? "" : " (scalar C)");
    else if (pl.cpasync)
        snprintf(buf, (size_t)buf_len, "es::spmm_cpasync%s<stages%d>%s", pl.halfwarp ? "_hw" : "", pl.stages,
                 pl.c_vec ? "" : " (scalar C)");
    else if (pl.subwarp)
        snprintf(buf, (size_t)buf_len, "es::spmm_subwarp<vec%d,g%d>%s", pl.vec, pl.g, pl.c_vec ? "" : " (scalar C)");
    else
        snprintf(buf, (size_t)buf_len, "es::spmm_warp<vec%d,nch%d>%s", pl.vec, pl.nch, pl.c_vec ? "" : " (scalar C)");
    return ES_OK;
}

es_status_t es_spmm_sample(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                           const int32_t* colind, const float* val, int32_t s, int32_t strategy,
                           uint64_t seed, int64_t row_base, int64_t* s_rowptr, int32_t* s_colind,
                           float* s_val, int64_t* s_pos, void* stream) {
    return es_spmm_sample_ex(n_rows, n_cols, rowptr, colind, val, s, strategy, seed, row_base, s_rowptr,
                             s_colind, s_val, s_pos, nullptr, stream);
}

es_status_t es_spmm_sample_ex(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                              const int32_t* colind, const float* val, int32_t s, int32_t strategy,
                              uint64_t seed, int64_t row_base, int64_t* s_rowptr, int32_t* s_colind,
                              float* s_val, int64_t* s_pos, const es_spmm_options_t* opt, void* stream) {
    Opts o;
    if (read_opts(opt, &o) != ES_OK) return ES_ERR_INVALID_VALUE;
    if (n_rows < 0 || n_cols < 0 || s < 1 || row_base < 0) return ES_ERR_INVALID_VALUE;
    if (strategy != ES_BUCKET && strategy != ES_FASTRAND) return ES_ERR_INVALID_VALUE;
    if (!rowptr || !s_rowptr) return ES_ERR_INVALID_VALUE;
    cudaStream_t st = as_stream(stream);
    int launches = 0;
    cudaError_t err = es::launch_sample_count(rowptr, n_rows, s, s_rowptr, st, &launches);
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    if (err != cudaSuccess) return ES_ERR_CUDA;
    if (!s_colind || n_rows == 0) return ES_OK;
    // nnz_base: colind/val are indexed with the absolute rowptr entries.
    err = es::launch_sample_materialize(rowptr, 0, colind, val, n_rows, s, strategy, seed, row_base,
                                        o.prime, s_rowptr, s_colind, s_val, s_pos, st);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

es_status_t es_spmm_run(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, const int32_t* colind,
                        const float* val, const float* B, int64_t F, int64_t ldb, int32_t s,
                        int32_t strategy, uint64_t seed, int32_t reduce, float* C, int64_t ldc,
                        void* stream) {
    return run_rows_impl(n_rows, n_cols, rowptr, 0, colind, val, B, F, ldb, s, strategy, seed, reduce,
                         C, ldc, 0, n_rows, Opts{}, as_stream(stream));
}

es_status_t es_spmm_run_rows(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, int64_t nnz_base,
                             const int32_t* colind, const float* val, const float* B, int64_t F,
                             int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             float* C, int64_t ldc, int64_t row_begin, int64_t row_end, void* stream) {
    return run_rows_impl(n_rows, n_cols, rowptr, nnz_base, colind, val, B, F, ldb, s, strategy, seed,
                         reduce, C, ldc, row_begin, row_end, Opts{}, as_stream(stream));
}

es_status_t es_spmm_run_ex(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, int64_t nnz_base,
                           const int32_t* colind, const float* val, const void* B, int64_t F,
                           int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                           float* C, int64_t ldc, int64_t row_begin, int64_t row_end,
                           const es_spmm_options_t* opt, void* stream) {
    Opts o;
    if (read_opts(opt, &o) != ES_OK) return ES_ERR_INVALID_VALUE;
    return run_rows_impl(n_rows, n_cols, rowptr, nnz_base, colind, val, B, F, ldb, s, strategy, seed,
                         reduce, C, ldc, row_begin, row_end, o, as_stream(stream));
}

es_status_t es_spmm_backward(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, int64_t nnz_base,
                             const int32_t* colind, const float* val, const float* dC, int64_t F,
                             int64_t ldc, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             float* dB, int64_t ldb, int64_t row_begin, int64_t row_end, void* stream) {
    return es_spmm_backward_ex(n_rows, n_cols, rowptr, nnz_base, colind, val, dC, F, ldc, s, strategy, seed,
                               reduce, dB, ldb, row_begin, row_end, nullptr, stream);
}

es_status_t es_spmm_backward_ex(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, int64_t nnz_base,
                                const int32_t* colind, const float* val, const float* dC, int64_t F,
                                int64_t ldc, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                                float* dB, int64_t ldb, int64_t row_begin, int64_t row_end,
                                const es_spmm_options_t* opt, void* stream) {
    Opts o;
    if (read_opts(opt, &o) != ES_OK) return ES_ERR_INVALID_VALUE;
    if (o.bf16) return ES_ERR_UNSUPPORTED;
    es_status_t rc = check_common(n_rows, n_cols, F, ldb, ldc, s, strategy, reduce);
    if (rc != ES_OK) return rc;
    if (row_begin < 0 || row_end < row_begin || row_end > n_rows) return ES_ERR_INVALID_VALUE;
    const int64_t n = row_end - row_begin;
    if (n == 0) return ES_OK;
    if (!rowptr || !dC || (n_cols > 0 && !dB)) return ES_ERR_INVALID_VALUE;
    es::BwdParams p{};
    p.rowptr = rowptr;
    p.nnz_base = nnz_base;
    p.colind = colind;
    p.val = val;
    p.dC = dC;
    p.F = F;
    p.ldc = ldc;
    p.s = s;
    p.strategy = strategy;
    p.seed = seed;
    p.reduce = reduce;
    p.dB = dB;
    p.ldb = ldb;
    p.n_rows = n;
    p.row_base = row_begin;
    p.prime = o.prime;
    p.mean_by_degree = o.mean_by_degree;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dC), b = reinterpret_cast<uintptr_t>(dB);
    if (a % 16 == 0 && b % 16 == 0 && ldc % 4 == 0 && ldb % 4 == 0) p.vec = 4;
    else if (a % 8 == 0 && b % 8 == 0 && ldc % 2 == 0 && ldb % 2 == 0) p.vec = 2;
    else p.vec = 1;
    if (o.deterministic) {
        int launches = 0;
        bool too_large = false;
        cudaError_t err = es::launch_backward_deterministic(p, n_cols, as_stream(stream), &launches, &too_large);
        g_launches.fetch_add(launches, std::memory_order_relaxed);
        if (too_large) return ES_ERR_UNSUPPORTED;
        return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
    }
    // slab path (a workspace was passed): the gradient one 64-float slice at a time, the dB slab
    // L2-resident while its reductions land; the sampled slots come from the workspace
    // (reuse_sampled: the forward's) or are sampled here
    SlabSlots sl;
    if (o.workspace && p.vec == 4 && slab_feasible(n_cols, F) && slab_slots(o, n, val != nullptr, &sl)) {
        cudaStream_t st = as_stream(stream);
        int launches = 0;
        cudaError_t err = cudaSuccess;
        const bool direct = strategy == ES_BUCKET;               // first k_i entries, in place
        if (!o.reuse_sampled && !direct)
            err = slab_sample(sl, rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, o.prime, st,
                              &launches);
        for (int64_t c0 = 0; err == cudaSuccess && c0 < F; c0 += kSlabF) {
            es::SlabParams sp{};
            sp.s_rowptr = direct ? rowptr : sl.s_rowptr;
            sp.slot_base = direct ? nnz_base : 0;
            sp.cap = direct ? INT64_MAX : sl.cap;
            sp.s_colind = direct ? colind : sl.s_col;
            sp.s_val = direct ? val : sl.s_val;
            sp.direct_s = direct ? s : 0;
            sp.rowptr = rowptr;
            sp.ldb = ldb;
            sp.w = (int32_t)(F - c0 < kSlabF ? F - c0 : kSlabF);
            sp.nv = (sp.w + 3) / 4;
            sp.ldc = ldc;
            sp.n_rows = n;
            sp.reduce = reduce;
            sp.mean_by_degree = o.mean_by_degree;
            err = es::launch_slab_backward(sp, dC + c0, dB + c0, st);
            ++launches;
        }
        g_launches.fetch_add(launches, std::memory_order_relaxed);
        return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
    }
    cudaError_t err = es::launch_backward(p, as_stream(stream));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

int32_t es_ipc_handle_bytes(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

es_status_t es_ipc_alloc(int64_t bytes, void** dev_ptr_out) {
    if (bytes <= 0 || !dev_ptr_out) return ES_ERR_INVALID_VALUE;
    return cudaMalloc(dev_ptr_out, (size_t)bytes) == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

es_status_t es_ipc_free(void* dev_ptr) {
    if (!dev_ptr) return ES_ERR_INVALID_VALUE;
    return cudaFree(dev_ptr) == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

es_status_t es_ipc_export(void* dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out) return ES_ERR_INVALID_VALUE;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, dev_ptr) != cudaSuccess) return ES_ERR_CUDA;
    std::memcpy(handle_out, &h, sizeof(h));
    return ES_OK;
}

es_status_t es_ipc_import(const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return ES_ERR_INVALID_VALUE;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? ES_OK
                                                                                              : ES_ERR_CUDA;
}

es_status_t es_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return ES_ERR_INVALID_VALUE;
    return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

es_status_t es_partition_rows(const int64_t* rowptr_host, int64_t n_rows, int32_t s, int64_t F,
                              int32_t n_parts, int64_t* bounds_host) {
    if (!rowptr_host || !bounds_host || n_rows < 0 || s < 1 || F < 1 || n_parts < 1)
        return ES_ERR_INVALID_VALUE;
    // prefix[r] = sum_{i<r} w_i, w_i = k_i*(4F+8) + 4F  (exact int64 arithmetic)
    std::vector<int64_t> prefix((size_t)n_rows + 1, 0);
    for (int64_t i = 0; i < n_rows; ++i) {
        const int64_t d = rowptr_host[i + 1] - rowptr_host[i];
        const int64_t k = d < (int64_t)s ? d : (int64_t)s;
        prefix[(size_t)i + 1] = prefix[(size_t)i] + k * (4 * F + 8) + 4 * F;
    }
    const int64_t total = prefix[(size_t)n_rows];
    bounds_host[0] = 0;
    for (int32_t p = 1; p < n_parts; ++p) {
        // smallest r with prefix[r] >= ceil(total * p / P)  (128-bit to avoid overflow)
        const __int128 num = (__int128)total * p;
        const int64_t target = (int64_t)((num + n_parts - 1) / n_parts);
        int64_t r = (int64_t)(std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin());
        r = std::max(r, bounds_host[p - 1]);
        bounds_host[p] = std::min(r, n_rows);
    }
    bounds_host[n_parts] = n_rows;
    return ES_OK;
}

// ---------------------------------------------------------------- host-buffer pipeline
static inline int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

int64_t es_spmm_host_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F,
                                     int64_t ldb, int32_t has_val) {
    (void)F;
    if (n_rows < 0 || n_cols < 0 || nnz < 0 || ldb < 1) return -1;
    return align256((n_rows + 1) * 8) + align256(nnz * 4) + (has_val ? align256(nnz * 4) : 0) +
           align256(n_cols * ldb * 4) + align256(n_rows * ldb * 4);
}

es_status_t es_spmm_run_host(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                             const int32_t* colind, const float* val, const float* B, int64_t F,
                             int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             int64_t row_base, float* C, int64_t ldc, void* workspace,
                             int64_t workspace_bytes, void* stream) {
    es_status_t rc = check_common(n_rows, n_cols, F, ldb, ldc, s, strategy, reduce);
    if (rc != ES_OK) return rc;
    if (n_rows == 0) return ES_OK;
    if (!rowptr || !C || !workspace || (n_cols > 0 && !B) || row_base < 0) return ES_ERR_INVALID_VALUE;
    const int64_t base = rowptr[0];
    const int64_t nnz = rowptr[n_rows] - base;
    if (nnz > 0 && !colind) return ES_ERR_INVALID_VALUE;
    const int64_t need = es_spmm_host_workspace_bytes(n_rows, n_cols, nnz, F, ldb, val != nullptr);
    if (workspace_bytes < need) return ES_ERR_INVALID_VALUE;

    // device workspace layout; the device C uses ldc' = ldb (dense, 16 B rows when ldb % 4 == 0)
    char* w = static_cast<char*>(workspace);
    int64_t* d_rowptr = reinterpret_cast<int64_t*>(w); w += align256((n_rows + 1) * 8);
    int32_t* d_colind = reinterpret_cast<int32_t*>(w); w += align256(nnz * 4);
    float* d_val = nullptr;
    if (val) { d_val = reinterpret_cast<float*>(w); w += align256(nnz * 4); }
    float* d_B = reinterpret_cast<float*>(w); w += align256(n_cols * ldb * 4);
    float* d_C = reinterpret_cast<float*>(w);
    const int64_t dldc = ldb;

    cudaStream_t st = as_stream(stream);
    cudaStream_t s_in = nullptr, s_out = nullptr;
    const int kMaxChunks = 8;
    int n_chunks = (int)std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, n_rows / 4096));
    std::vector<cudaEvent_t> ev_in((size_t)n_chunks, nullptr), ev_done((size_t)n_chunks, nullptr);
    cudaEvent_t ev_start = nullptr, ev_out = nullptr;
    cudaError_t err = cudaSuccess;
    auto ok = [&](cudaError_t e) { if (err == cudaSuccess && e != cudaSuccess) err = e; return err == cudaSuccess; };

    if (!ok(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking)) ||
        !ok(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking)) ||
        !ok(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming)) ||
        !ok(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming))) goto cleanup;
    for (int c = 0; c < n_chunks; ++c)
        if (!ok(cudaEventCreateWithFlags(&ev_in[(size_t)c], cudaEventDisableTiming)) ||
            !ok(cudaEventCreateWithFlags(&ev_done[(size_t)c], cudaEventDisableTiming))) goto cleanup;

    // inputs may only be overwritten after earlier work on the caller's stream
    if (!ok(cudaEventRecord(ev_start, st)) || !ok(cudaStreamWaitEvent(s_in, ev_start, 0))) goto cleanup;
    if (!ok(cudaMemcpyAsync(d_rowptr, rowptr, (size_t)(n_rows + 1) * 8, cudaMemcpyHostToDevice, s_in)))
        goto cleanup;
    if (n_cols > 0 &&
        !ok(cudaMemcpyAsync(d_B, B, (size_t)(n_cols * ldb) * 4, cudaMemcpyHostToDevice, s_in))) goto cleanup;
    {
        int64_t r0 = 0;
        for (int c = 0; c < n_chunks; ++c) {
            // rows [r0, r1) hold ~nnz/n_chunks nonzeros
            int64_t r1 = n_rows;
            if (c + 1 < n_chunks) {
                const int64_t target = base + (nnz * (c + 1)) / n_chunks;
                r1 = (int64_t)(std::lower_bound(rowptr, rowptr + n_rows + 1, target) - rowptr);
                r1 = std::max(r0, std::min(r1, n_rows));
            }
            const int64_t e0 = rowptr[r0] - base, e1 = rowptr[r1] - base;
            if (e1 > e0) {
                if (!ok(cudaMemcpyAsync(d_colind + e0, colind + e0, (size_t)(e1 - e0) * 4,
                                        cudaMemcpyHostToDevice, s_in))) goto cleanup;
                if (val && !ok(cudaMemcpyAsync(d_val + e0, val + e0, (size_t)(e1 - e0) * 4,
                                               cudaMemcpyHostToDevice, s_in))) goto cleanup;
            }
            if (!ok(cudaEventRecord(ev_in[(size_t)c], s_in)) || !ok(cudaStreamWaitEvent(st, ev_in[(size_t)c], 0)))
                goto cleanup;
            rc = run_rows_impl(row_base + n_rows, n_cols, d_rowptr + r0, base, d_colind, d_val, d_B, F,
                               ldb, s, strategy, seed, reduce, d_C + r0 * dldc, dldc, row_base + r0,
                               row_base + r1, Opts{}, st);
            if (rc != ES_OK) goto cleanup;
            if (!ok(cudaEventRecord(ev_done[(size_t)c], st)) || !ok(cudaStreamWaitEvent(s_out, ev_done[(size_t)c], 0)))
                goto cleanup;
            if (r1 > r0 &&
                !ok(cudaMemcpy2DAsync(C + r0 * ldc, (size_t)ldc * 4, d_C + r0 * dldc, (size_t)dldc * 4,
                                      (size_t)F * 4, (size_t)(r1 - r0), cudaMemcpyDeviceToHost, s_out)))
                goto cleanup;
            r0 = r1;
        }
    }
    if (!ok(cudaEventRecord(ev_out, s_out)) || !ok(cudaStreamWaitEvent(st, ev_out, 0))) goto cleanup;
    ok(cudaStreamSynchronize(st));

cleanup:
    if (err != cudaSuccess) cudaStreamSynchronize(st);
    for (auto e : ev_in) if (e) cudaEventDestroy(e);
    for (auto e : ev_done) if (e) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_out) cudaEventDestroy(ev_out);
    if (s_in) { cudaStreamSynchronize(s_in); cudaStreamDestroy(s_in); }
    if (s_out) { cudaStreamSynchronize(s_out); cudaStreamDestroy(s_out); }
    if (rc != ES_OK) return rc;
    return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

}  // extern "C"
