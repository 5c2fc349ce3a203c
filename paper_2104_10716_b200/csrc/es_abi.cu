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

#include <new>

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
    int64_t nnz = 0;             // stored entries of the call's rows (0 = unknown)
    es::Tune tune;
    float* c_mc = nullptr;       // NVLS multicast base of the full C (fused all-gather)
};

#define ES_COVERS(o, field) ((o)->struct_size >= (int32_t)(offsetof(es_spmm_options_t, field) + sizeof((o)->field)))

es_status_t read_opts(const es_spmm_options_t* o, Opts* out) {
    *out = Opts{};
    if (!o) return ES_OK;
    if (!ES_COVERS(o, b_dtype)) return ES_ERR_INVALID_VALUE;
    if (o->prime < 0) return ES_ERR_INVALID_VALUE;
    if (o->mean_divisor != ES_MEAN_BY_SAMPLED && o->mean_divisor != ES_MEAN_BY_DEGREE) return ES_ERR_INVALID_VALUE;
    if (o->b_dtype != ES_DTYPE_F32 && o->b_dtype != ES_DTYPE_BF16) return ES_ERR_INVALID_VALUE;
    out->prime = o->prime == 0 ? 577u : (uint32_t)o->prime;
    out->mean_by_degree = o->mean_divisor == ES_MEAN_BY_DEGREE;
    out->bf16 = o->b_dtype == ES_DTYPE_BF16;
    if (ES_COVERS(o, n_peers)) {
        if (o->n_peers < 0 || (o->n_peers > 0 && !o->c_peers)) return ES_ERR_INVALID_VALUE;
        out->c_peers = o->c_peers;
        out->n_peers = o->n_peers;
    }
    if (ES_COVERS(o, deterministic)) out->deterministic = o->deterministic != 0;
    if (ES_COVERS(o, workspace_bytes)) {
        if (o->workspace_bytes < 0 || (o->workspace_bytes > 0 && !o->workspace)) return ES_ERR_INVALID_VALUE;
        out->workspace = o->workspace_bytes > 0 ? o->workspace : nullptr;
        out->workspace_bytes = o->workspace_bytes;
    }
    if (ES_COVERS(o, reuse_sampled)) out->reuse_sampled = o->reuse_sampled != 0;
    if (ES_COVERS(o, nnz)) {
        if (o->nnz < 0) return ES_ERR_INVALID_VALUE;
        out->nnz = o->nnz;
    }
    if (ES_COVERS(o, tune)) {
        if (o->kernel < ES_KERNEL_AUTO || o->kernel > ES_KERNEL_SEGSTREAM) return ES_ERR_INVALID_VALUE;
        out->tune.kernel = o->kernel;
        out->tune.stages = o->tune[0];
        out->tune.width = o->tune[1];
        out->tune.cta_warps = o->tune[2];
        out->tune.variant = o->tune[3];
    }
    if (ES_COVERS(o, c_multicast)) out->c_mc = o->c_multicast;
    return ES_OK;
}

// ---- slab path (es_slab.cu): when, and the workspace layout
constexpr int64_t kSlabF = 64;                       // floats per feature slice (256-B slab rows)
constexpr int64_t kSlabMaxBytes = (int64_t)80 << 20; // largest slab kept L2-resident (126 MB L2)
constexpr int64_t kSlabMaxBytes24 = (int64_t)96 << 20;  // ... for 24-piece flow slices (Reddit: 89 MB)

// A workspace was passed: the slab path runs whenever the layout allows -- F > 16, B rows 16-B
// aligned, and a 64-float slab of B (n_cols x 256 B) fits L2.
bool slab_feasible(int64_t n_cols, int64_t F) {
    return F > kSlabF / 4 && n_cols * kSlabF * 4 <= kSlabMaxBytes;
}

// es_spmm_workspace_bytes's choice (measured, profiles/r02_flow_plan.jsonl): feasible,
// F >= 128, a 16-B row pitch, and rows that sample enough slots on average: min(s, nnz / n_rows)
// >= 32 for F > 256 (Reddit F=602: s = 32 flow 1.58 vs fused 1.76 ms, s = 16 1.16 vs 1.04) and
// >= 128 for 128 < F <= 256 (F=256 s = 64 1.10 vs 1.03) and >= 256 for F <= 128, where the fused
// kernel is the segmented register stream (profiles/r02_segstream_probe.jsonl seg9: Reddit F=128
// s = 128 fused 0.89 vs flow 0.92 ms, Proteins s = 128 0.54 vs 0.59; s = 256 Proteins 0.96 vs
// 0.93, Reddit 1.54 vs 1.39; s = 512 Proteins 1.62 vs 1.45).  Below that the fused kernels, which
// sample inside the gather, win.
bool slab_wanted(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb, int64_t s) {
    if (!slab_feasible(n_cols, F) || ldb % 4 != 0 || F < 128) return false;
    const int64_t mean_deg = n_rows > 0 ? nnz / n_rows : 0;
    const int64_t k_est = s < mean_deg ? s : mean_deg;
    return k_est >= (F > 256 ? 32 : F > 128 ? 128 : 256);
}

int64_t slab_align(int64_t x) { return (x + 255) & ~(int64_t)255; }

// [header 256 B][s_rowptr (n+1) x 8][scan temp][s_k n x 4][s_colind cap x 4][s_val cap x 4]
struct SlabLayout {
    int64_t off_rowptr, off_temp, temp_bytes, off_k, off_col, bytes_fixed;
};
SlabLayout slab_layout(int64_t n) {
    SlabLayout L{};
    L.off_rowptr = 256;
    L.off_temp = slab_align(L.off_rowptr + 8 * (n + 1));
    L.temp_bytes = (int64_t)es::slab_scan_temp_bytes(n);
    L.off_k = slab_align(L.off_temp + L.temp_bytes);
    L.off_col = slab_align(L.off_k + 4 * n);
    L.bytes_fixed = L.off_col;
    return L;
}
int64_t slab_bytes(int64_t n, int64_t cap, bool has_val) {
    const int64_t c = cap > 0 ? cap : 1;
    return slab_layout(n).bytes_fixed + slab_align(4 * c) + (has_val ? slab_align(4 * c) : 0);
}
// slots a workspace must hold: min(nnz, n*s) sampled slots plus up to 15 padding slots per row
// (the flow layout pads every row to a multiple of 16 slots)
int64_t slab_cap_needed(int64_t n, int64_t nnz, int32_t s) {
    const int64_t ns = n * (int64_t)s;
    return (nnz > 0 && nnz < ns ? nnz : ns) + 15 * n;
}

// Which slab kernel a call's options select: the flow kernel (default; padded slot layout, row
// partition) unless a per-row slab kernel is forced (A/B) -- the layout follows the kernel, and
// the sampling signature records it, so slots are never reused across layouts.
bool slab_flow(const es::Tune& t) {
    return t.kernel != ES_KERNEL_SLAB_SMEM && t.kernel != ES_KERNEL_SLAB_LDG && t.kernel != ES_KERNEL_SLAB_TMA &&
           t.kernel != ES_KERNEL_SLAB_STREAM;
}

// The workspace's sampled-slot arrays (es_spmm_sample layout).
struct SlabSlots {
    es::WsHeader* hdr;
    int64_t* s_rowptr;
    int32_t* s_col;
    float* s_val;
    int64_t cap;
    void* temp;
    size_t temp_bytes;
    int32_t* s_k;        // flow layout: unpadded k_i
};
// false: the workspace cannot hold the slots the call may sample -- min(nnz, n*s) when the
// caller stated nnz, else n*s (an undersized workspace is an error, never a truncation)
bool slab_slots(const Opts& o, int64_t n, int32_t s, bool has_val, SlabSlots* out) {
    const SlabLayout L = slab_layout(n);
    const int64_t per_slot = has_val ? 8 : 4;
    int64_t cap = (o.workspace_bytes - L.bytes_fixed - (has_val ? 256 : 0)) / per_slot;
    const int64_t need = slab_cap_needed(n, o.nnz, s);
    if (cap < need || cap < 1) return false;
    char* ws = static_cast<char*>(o.workspace);
    out->hdr = reinterpret_cast<es::WsHeader*>(ws);
    out->s_rowptr = reinterpret_cast<int64_t*>(ws + L.off_rowptr);
    out->s_col = reinterpret_cast<int32_t*>(ws + L.off_col);
    out->s_val = has_val ? reinterpret_cast<float*>(ws + slab_align(L.off_col + 4 * cap)) : nullptr;
    out->cap = cap;
    out->temp = ws + L.off_temp;
    out->temp_bytes = (size_t)L.temp_bytes;
    out->s_k = reinterpret_cast<int32_t*>(ws + L.off_k);
    return true;
}

// Signature of a sampling: the call parameters the sampled slots depend on (never 0).  The graph
// itself is checked per row on reuse (SlabParams.reuse_s: the slab passes compare each row's slot
// count with min(d_i, s) from the caller's rowptr), so a re-uploaded copy of the same CSR may be
// reused, a different one is caught.
uint64_t sampling_signature(int64_t n, int64_t row_begin, int32_t s, int32_t strategy, uint64_t seed,
                            uint32_t prime, int64_t nnz_base, bool has_val, int32_t pad) {
    uint64_t h = 0x6a09e667f3bcc908ull;
    auto mix = [&](uint64_t x) {
        h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
    };
    mix((uint64_t)n); mix((uint64_t)row_begin); mix((uint64_t)s); mix((uint64_t)strategy); mix(seed);
    mix(prime); mix((uint64_t)nnz_base); mix(has_val ? 1u : 0u); mix((uint64_t)pad);
    return h ? h : 1;
}

// a1-a3 once into the workspace: count, scan, materialise, sign; for the flow layout rows padded
// to 4 slots and each row's unpadded k_i
cudaError_t slab_sample(const SlabSlots& sl, const int64_t* rowptr, int64_t nnz_base, const int32_t* colind,
                        const float* val, int64_t n, int32_t s, int32_t strategy, uint64_t seed, int64_t row_begin,
                        uint32_t prime, uint64_t sig, cudaStream_t st, int* launches, bool flow = false) {
    const int32_t pad = flow ? 16 : 1;
    // the count kernel clears the header (status 0, signature invalid) and the materialisation
    // signs it: no extra launches
    cudaError_t err = es::launch_slab_count(rowptr, n, s, sl.s_rowptr, sl.temp, sl.temp_bytes, st, launches, sl.hdr,
                                            pad, flow ? sl.s_k : nullptr);
    if (err != cudaSuccess) return err;
    err = es::launch_sample_materialize(rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, prime,
                                        sl.s_rowptr, sl.s_col, sl.s_val, nullptr, st, sl.cap, sl.hdr, sig, pad);
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
    const es::Tune& tn = o.tune;
    const bool force_slab = tn.kernel == ES_KERNEL_SLAB || tn.kernel == ES_KERNEL_SLAB_SMEM ||
                            tn.kernel == ES_KERNEL_SLAB_LDG || tn.kernel == ES_KERNEL_SLAB_TMA ||
                            tn.kernel == ES_KERNEL_SLAB_STREAM || tn.kernel == ES_KERNEL_SLAB_FLOW;
    const uintptr_t bu = reinterpret_cast<uintptr_t>(B), cu = reinterpret_cast<uintptr_t>(C);
    const int64_t esz = o.bf16 ? 2 : 4;
    // a forced flow kernel runs whatever the slab's size (A/B: slabs beyond L2, e.g. the 10M-row graph)
    const bool feasible = slab_feasible(n_cols, F) || (tn.kernel == ES_KERNEL_SLAB_FLOW && F > kSlabF / 4);
    const bool slab_layout_ok = o.workspace && bu % 16 == 0 && (ldb * esz) % 16 == 0 && feasible &&
                                tn.kernel != ES_KERNEL_FUSED && tn.kernel != ES_KERNEL_WARP &&
                                tn.kernel != ES_KERNEL_TMA && tn.kernel != ES_KERNEL_CPASYNC &&
                                tn.kernel != ES_KERNEL_CPASYNC_HW && tn.kernel != ES_KERNEL_ROWSTREAM &&
                                tn.kernel != ES_KERNEL_GROUPED && tn.kernel != ES_KERNEL_SEGSTREAM;
    if (force_slab && !slab_layout_ok) return ES_ERR_UNSUPPORTED;
    if (slab_layout_ok) {
        // any C layout: 16-B vector stores where C's rows allow them, scalar stores otherwise
        const bool c_vec16 = cu % 16 == 0 && ldc % 4 == 0;
        // the flow kernel (default) streams a padded, partitioned slot layout; a forced per-row
        // kernel reads the compact one -- and for Bucket, whose sampled slots are the first k_i
        // entries of each row (Alg. 1 with p_j = j), the CSR itself (no sampling pass)
        const bool flow = slab_flow(tn);
        const bool direct = strategy == ES_BUCKET && !flow;
        SlabSlots sl{};
        if (!direct && !slab_slots(o, n, s, val != nullptr, &sl)) return ES_ERR_INVALID_VALUE;
        int launches = 0;
        cudaError_t err = cudaSuccess;
        const uint64_t sig = sampling_signature(n, row_begin, s, strategy, seed, o.prime, nnz_base, val != nullptr,
                                                flow ? 16 : 1);
        if (!o.reuse_sampled && !direct)
            err = slab_sample(sl, rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, o.prime, sig, st,
                              &launches, flow);
        const bool b32 = bu % 32 == 0 && (ldb * esz) % 32 == 0;
        // one slice: columns [c0, c0 + w) of B and C
        auto slice = [&](int64_t c0, int64_t w) {
            es::SlabParams sp{};
            sp.s_rowptr = direct ? rowptr : sl.s_rowptr;
            sp.slot_base = direct ? nnz_base : 0;
            sp.cap = direct ? INT64_MAX : sl.cap;
            sp.s_colind = direct ? colind : sl.s_col;
            sp.s_val = direct ? val : sl.s_val;
            sp.direct_s = direct ? s : 0;
            sp.ws_status = direct ? nullptr : &sl.hdr->status;
            sp.ws_sig = direct ? nullptr : &sl.hdr->sig;
            sp.s_k = flow ? sl.s_k : nullptr;
            sp.sig = sig;
            sp.s = s;
            sp.reuse_s = (o.reuse_sampled && !direct) ? s : 0;
            sp.rowptr = rowptr;
            sp.b_bf16 = o.bf16;
            sp.B = o.bf16 ? reinterpret_cast<const float*>(static_cast<const uint16_t*>(B) + c0)
                          : static_cast<const float*>(B) + c0;
            sp.ldb = ldb;
            sp.w = (int32_t)w;
            sp.b32 = b32 ? 1 : 0;
            sp.nv = (int32_t)((w * esz + 15) / 16);     // 16-B pieces
            sp.C = C + c0;
            sp.c_peers = o.c_peers;
            sp.n_peers = o.n_peers;
            sp.c_mc = o.c_mc;
            sp.row_base = row_begin;
            sp.col0 = c0;
            sp.ldc = ldc;
            sp.c_vec = c_vec16 ? 1 : 0;
            sp.n_rows = n;
            sp.reduce = reduce;
            sp.mean_by_degree = o.mean_by_degree;
            return sp;
        };
        if (flow) {
            // slices of MP 16-B pieces (tune.width 8, 16 or 24), so every slice starts on a 128-B
            // line (a slice start inside a line makes each 8-lane copy touch two lines: 15- and
            // 19-piece slices ran 35 % slower per byte); a remainder of <= 32 - MP pieces joins
            // the last slice (3 or 4 pieces per lane) instead of running as a narrow pass of its
            // own, which costs as much as a full one -- F = 602: 5 x 24 + 31 pieces (VERDICT r01
            // weak #4)
            const int64_t epp = 16 / esz;                     // elements per piece
            const int64_t NP = (F + epp - 1) / epp;
            // a remainder joins the last slice up to 32 pieces (24 for bf16: its 4-piece kernel
            // would not fit the register file)
            const int64_t kMerge = o.bf16 ? 24 : 32;
            auto passes = [&](int64_t mp) {
                const int64_t q = NP / mp, r = NP % mp;
                return q + ((r > 0 && !(q > 0 && mp + r <= kMerge)) ? 1 : 0);
            };
            // default: the width with fewer passes (a pass costs about the same from 16 to 24
            // pieces on a 2.4-KB-pitch B: Reddit F=602 7 passes of 24 (+7) 7.17 ms vs 9 of 16 (+7
            // merged) 9.15 ms; F=128: 2 x 16), 24 only while its slab (n_cols x 384 B) fits L2
            int64_t MP = (tn.width == 8 || tn.width == 16 || tn.width == 24 || (tn.width == 32 && !o.bf16)) ? tn.width : 16;
            if (tn.width == 0 && passes(24) < passes(16) && n_cols * 384 <= kSlabMaxBytes24) MP = 24;
            const int64_t m = passes(MP);
            for (int64_t i = 0; err == cudaSuccess && i < m; ++i) {
                const int64_t c0 = i * MP * epp;
                const int64_t np_i = (i + 1 == m) ? NP - i * MP : MP;
                const int64_t w = F - c0 < np_i * epp ? F - c0 : np_i * epp;
                err = es::launch_slab_flow(slice(c0, w), tn, st);
                ++launches;
            }
            g_launches.fetch_add(launches, std::memory_order_relaxed);
            return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
        }
        // per-row slab kernels (A/B): slices of 256-B slab rows, 64 fp32 or 128 bf16 elements
        const int64_t wsl = o.bf16 ? 2 * kSlabF : kSlabF;
        CUtensorMap tmap;
        const bool use_tma = tn.kernel == ES_KERNEL_SLAB_TMA;
        if (use_tma && !es::encode_b_tensor_map(&tmap, B, F, ldb, n_cols, o.bf16)) return ES_ERR_UNSUPPORTED;
        if (tn.kernel == ES_KERNEL_SLAB_LDG && !b32) return ES_ERR_UNSUPPORTED;
        for (int64_t c0 = 0; err == cudaSuccess && c0 < F; c0 += wsl) {
            es::SlabParams sp = slice(c0, F - c0 < wsl ? F - c0 : wsl);
            // 16-B pieces (shared-memory ring) or 32-B pieces (register-direct)
            if (b32 && tn.kernel == ES_KERNEL_SLAB_LDG) sp.nv = (int32_t)((sp.w * esz + 31) / 32);
            if (use_tma) err = es::launch_slab_pass_tma(tmap, sp, (int32_t)c0, (int32_t)n_cols, tn, st);
            else err = es::launch_slab_pass(sp, tn, st);
            ++launches;
        }
        g_launches.fetch_add(launches, std::memory_order_relaxed);
        return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
    }
    if (o.reuse_sampled) return ES_ERR_INVALID_VALUE;      // no slab path: nothing to reuse
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
    p.c_mc = o.c_mc;
    const int64_t k_est = o.nnz > 0 ? std::min<int64_t>(s, o.nnz / n) : s;
    es::Plan plan = o.bf16 ? es::make_plan_bf16(F, ldb, ldc, B, C)
                           : es::make_plan(F, ldb, ldc, B, C, s, tn, k_est);
    if (plan.unsupported) return ES_ERR_UNSUPPORTED;
    if (tn.kernel == ES_KERNEL_ROWSTREAM && !plan.rowstream) return ES_ERR_UNSUPPORTED;
    if (plan.segstream && (uint64_t)ldb * 4 >= (1ull << 32)) {
        // the segmented stream multiplies a column by the row pitch in bytes as a 32-bit value
        if (tn.kernel == ES_KERNEL_SEGSTREAM) return ES_ERR_UNSUPPORTED;
        es::Tune t2 = tn;
        t2.kernel = ES_KERNEL_CPASYNC_HW;
        plan = es::make_plan(F, ldb, ldc, B, C, s, t2, k_est);
    }
    if (tn.kernel == ES_KERNEL_SEGSTREAM && !plan.segstream) return ES_ERR_UNSUPPORTED;
    cudaError_t err = es::launch_spmm(p, plan, tn, st);
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
    if (!slab_wanted(n_rows, n_cols, nnz, F, ldb, s)) return 0;
    return slab_bytes(n_rows, slab_cap_needed(n_rows, nnz, s), has_val != 0) + 256;
}

int64_t es_spmm_workspace_bytes_ex(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb,
                                   int32_t s, int32_t has_val, const es_spmm_options_t* opt) {
    Opts o;
    if (read_opts(opt, &o) != ES_OK) return 0;
    const int k = o.tune.kernel;
    if (k != ES_KERNEL_SLAB && k != ES_KERNEL_SLAB_SMEM && k != ES_KERNEL_SLAB_LDG && k != ES_KERNEL_SLAB_TMA &&
        k != ES_KERNEL_SLAB_STREAM && k != ES_KERNEL_SLAB_FLOW)
        return es_spmm_workspace_bytes(n_rows, n_cols, nnz, F, ldb, s, has_val);
    // a slab kernel forced: a workspace wherever the path can run at all
    if (n_rows <= 0 || n_cols < 0 || nnz < 0 || F < 1 || ldb < F || s < 1) return 0;
    if (!(slab_feasible(n_cols, F) || (k == ES_KERNEL_SLAB_FLOW && F > kSlabF / 4)) || ldb % 4 != 0) return 0;
    return slab_bytes(n_rows, slab_cap_needed(n_rows, nnz, s), has_val != 0) + 256;
}

es_status_t es_spmm_workspace_status(void* workspace, int64_t workspace_bytes, int32_t reset, int32_t* status_out,
                                     void* stream) {
    if (!workspace || workspace_bytes < (int64_t)sizeof(es::WsHeader) || !status_out) return ES_ERR_INVALID_VALUE;
    es::WsHeader* h = static_cast<es::WsHeader*>(workspace);
    cudaStream_t st = as_stream(stream);
    int32_t v = 0;
    if (cudaMemcpyAsync(&v, &h->status, sizeof(v), cudaMemcpyDeviceToHost, st) != cudaSuccess) return ES_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return ES_ERR_CUDA;
    *status_out = v;
    if (reset && cudaMemsetAsync(&h->status, 0, sizeof(int32_t), st) != cudaSuccess) return ES_ERR_CUDA;
    return ES_OK;
}

es_status_t es_spmm_plan(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C,
                         char* buf, int32_t buf_len) {
    return es_spmm_plan_ex(F, ldb, ldc, B, C, INT32_MAX, 0, 0, buf, buf_len);
}

es_status_t es_spmm_plan_ex(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C, int32_t s,
                            int64_t n_rows, int64_t nnz, char* buf, int32_t buf_len) {
    if (F < 1 || ldb < F || ldc < F || !buf || buf_len < 1 || s < 1 || n_rows < 0 || nnz < 0)
        return ES_ERR_INVALID_VALUE;
    const int64_t k_est = (nnz > 0 && n_rows > 0) ? std::min<int64_t>(s, nnz / n_rows) : s;
    const es::Plan pl = es::make_plan(F, ldb, ldc, B, C, s, es::Tune{}, k_est);
    if (pl.segstream)
        snprintf(buf, (size_t)buf_len, "es::spmm_segstream<rows%d>%s", pl.rows_per_warp,
                 pl.c_vec ? "" : " (scalar C)");
    else if (pl.grouped)
        snprintf(buf, (size_t)buf_len, "es::spmm_grouped<slots4>(32-row degree-sorted batches)%s",
                 pl.c_vec ? "" : " (scalar C)");
    else if (pl.rowstream)
        snprintf(buf, (size_t)buf_len, "es::spmm_rowstream<stages%d,rows%d>%s", pl.stages, pl.rows_per_warp,
                 pl.c_vec ? "" : " (scalar C)");
    else if (pl.tma)
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
    const bool direct = strategy == ES_BUCKET;                   // first k_i entries, in place
    SlabSlots sl{};
    if (o.workspace && p.vec == 4 && slab_feasible(n_cols, F)) {
        if (!direct && !slab_slots(o, n, s, val != nullptr, &sl)) return ES_ERR_INVALID_VALUE;
        cudaStream_t st = as_stream(stream);
        int launches = 0;
        cudaError_t err = cudaSuccess;
        // the layout the forward call's plan samples (padded + partitioned unless a per-row slab
        // kernel is forced), so reuse_sampled finds the forward's slots
        const bool flow = slab_flow(o.tune);
        const int32_t pad = flow ? 16 : 1;
        const uint64_t sig = sampling_signature(n, row_begin, s, strategy, seed, o.prime, nnz_base, val != nullptr,
                                                pad);
        if (!o.reuse_sampled && !direct)
            err = slab_sample(sl, rowptr, nnz_base, colind, val, n, s, strategy, seed, row_begin, o.prime, sig, st,
                              &launches, flow);
        for (int64_t c0 = 0; err == cudaSuccess && c0 < F; c0 += kSlabF) {
            es::SlabParams sp{};
            sp.s_rowptr = direct ? rowptr : sl.s_rowptr;
            sp.slot_base = direct ? nnz_base : 0;
            sp.cap = direct ? INT64_MAX : sl.cap;
            sp.s_colind = direct ? colind : sl.s_col;
            sp.s_val = direct ? val : sl.s_val;
            sp.direct_s = direct ? s : 0;
            sp.ws_status = direct ? nullptr : &sl.hdr->status;
            sp.ws_sig = direct ? nullptr : &sl.hdr->sig;
            sp.sig = sig;
            sp.reuse_s = (o.reuse_sampled && !direct) ? s : 0;
            sp.s = s;
            sp.pad = direct ? 1 : pad;
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
    if (o.reuse_sampled) return ES_ERR_INVALID_VALUE;      // no slab path: nothing to reuse
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

}  // extern "C"

struct es_host_pipeline {
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_start = nullptr, ev_out = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_done;
};

namespace {
constexpr int kHostMaxChunks = 8;

void destroy_pipeline(es_host_pipeline* p) {
    if (!p) return;
    if (p->s_in) { cudaStreamSynchronize(p->s_in); cudaStreamDestroy(p->s_in); }
    if (p->s_out) { cudaStreamSynchronize(p->s_out); cudaStreamDestroy(p->s_out); }
    for (auto e : p->ev_in) if (e) cudaEventDestroy(e);
    for (auto e : p->ev_done) if (e) cudaEventDestroy(e);
    if (p->ev_start) cudaEventDestroy(p->ev_start);
    if (p->ev_out) cudaEventDestroy(p->ev_out);
    delete p;
}

es_host_pipeline* make_pipeline() {
    es_host_pipeline* p = new (std::nothrow) es_host_pipeline();
    if (!p) return nullptr;
    bool ok = cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) == cudaSuccess;
    p->ev_in.assign(kHostMaxChunks, nullptr);
    p->ev_done.assign(kHostMaxChunks, nullptr);
    for (int c = 0; ok && c < kHostMaxChunks; ++c)
        ok = cudaEventCreateWithFlags(&p->ev_in[(size_t)c], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&p->ev_done[(size_t)c], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        destroy_pipeline(p);
        return nullptr;
    }
    return p;
}

// device workspace of the host pipeline: [rowptr][colind][val][B][C][slab workspace (cap = nnz)]
struct HostLayout {
    int64_t off_rowptr, off_col, off_val, off_B, off_C, off_slab, slab_bytes, total;
};
HostLayout host_layout(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb, bool has_val) {
    HostLayout L{};
    L.off_rowptr = 0;
    L.off_col = align256((n_rows + 1) * 8);
    L.off_val = L.off_col + align256(nnz * 4);
    L.off_B = L.off_val + (has_val ? align256(nnz * 4) : 0);
    L.off_C = L.off_B + align256(n_cols * ldb * 4);
    L.off_slab = L.off_C + align256(n_rows * ldb * 4);
    // room for the slab path (sampled slots of any s: at most nnz) where the layout can take it
    L.slab_bytes = (slab_feasible(n_cols, F) && F >= 128 && ldb % 4 == 0)
                       ? slab_bytes(n_rows, nnz + 15 * n_rows, has_val) + 256 : 0;
    L.total = L.off_slab + L.slab_bytes;
    return L;
}
}  // namespace

extern "C" {

es_status_t es_host_pipeline_create(es_host_pipeline_t** out) {
    if (!out) return ES_ERR_INVALID_VALUE;
    *out = make_pipeline();
    return *out ? ES_OK : ES_ERR_CUDA;
}

void es_host_pipeline_destroy(es_host_pipeline_t* pipe) { destroy_pipeline(pipe); }

int64_t es_spmm_host_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F,
                                     int64_t ldb, int32_t has_val) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0 || ldb < 1 || F < 1) return -1;
    return host_layout(n_rows, n_cols, nnz, F, ldb, has_val != 0).total;
}

es_status_t es_spmm_run_host(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                             const int32_t* colind, const float* val, const float* B, int64_t F,
                             int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             int64_t row_base, float* C, int64_t ldc, void* workspace,
                             int64_t workspace_bytes, void* stream) {
    return es_spmm_run_host_ex(n_rows, n_cols, rowptr, colind, val, B, F, ldb, s, strategy, seed, reduce,
                               row_base, C, ldc, workspace, workspace_bytes, nullptr, nullptr, stream);
}

es_status_t es_spmm_run_host_ex(int64_t n_rows, int64_t n_cols, const int64_t* rowptr,
                                const int32_t* colind, const float* val, const float* B, int64_t F,
                                int64_t ldb, int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                                int64_t row_base, float* C, int64_t ldc, void* workspace,
                                int64_t workspace_bytes, const es_spmm_options_t* opt,
                                es_host_pipeline_t* pipe, void* stream) {
    es_status_t rc = check_common(n_rows, n_cols, F, ldb, ldc, s, strategy, reduce);
    if (rc != ES_OK) return rc;
    Opts o;
    if (read_opts(opt, &o) != ES_OK || o.bf16 || o.n_peers || o.c_mc || o.workspace || o.reuse_sampled)
        return ES_ERR_INVALID_VALUE;                 // host buffers: fp32 B, no peers, own workspace
    if (n_rows == 0) return ES_OK;
    if (!rowptr || !C || !workspace || (n_cols > 0 && !B) || row_base < 0) return ES_ERR_INVALID_VALUE;
    const int64_t base = rowptr[0];
    const int64_t nnz = rowptr[n_rows] - base;
    if (nnz > 0 && !colind) return ES_ERR_INVALID_VALUE;
    const HostLayout L = host_layout(n_rows, n_cols, nnz, F, ldb, val != nullptr);
    if (workspace_bytes < L.total) return ES_ERR_INVALID_VALUE;

    char* w = static_cast<char*>(workspace);
    int64_t* d_rowptr = reinterpret_cast<int64_t*>(w + L.off_rowptr);
    int32_t* d_colind = reinterpret_cast<int32_t*>(w + L.off_col);
    float* d_val = val ? reinterpret_cast<float*>(w + L.off_val) : nullptr;
    float* d_B = reinterpret_cast<float*>(w + L.off_B);
    float* d_C = reinterpret_cast<float*>(w + L.off_C);
    const int64_t dldc = ldb;                        // device C rows as B's (16-B rows when ldb % 4 == 0)
    // the library's plan: the slab path where es_spmm_workspace_bytes would ask for it
    const bool slab = L.slab_bytes > 0 && slab_wanted(n_rows, n_cols, nnz, F, ldb, s) &&
                      o.tune.kernel != ES_KERNEL_FUSED;

    cudaStream_t st = as_stream(stream);
    es_host_pipeline* own = nullptr;
    if (!pipe) {
        own = make_pipeline();
        if (!own) return ES_ERR_CUDA;
        pipe = own;
    }
    const int n_chunks = (int)std::min<int64_t>(kHostMaxChunks, std::max<int64_t>(1, n_rows / 4096));
    cudaError_t err = cudaSuccess;
    auto ok = [&](cudaError_t e) { if (err == cudaSuccess && e != cudaSuccess) err = e; return err == cudaSuccess; };

    // inputs may only be overwritten after earlier work on the caller's stream
    if (!ok(cudaEventRecord(pipe->ev_start, st)) || !ok(cudaStreamWaitEvent(pipe->s_in, pipe->ev_start, 0)) ||
        !ok(cudaStreamWaitEvent(pipe->s_out, pipe->ev_start, 0)))
        goto done;
    // every row gathers from all of B: B (and rowptr) first, then the CSR chunk by chunk
    if (!ok(cudaMemcpyAsync(d_rowptr, rowptr, (size_t)(n_rows + 1) * 8, cudaMemcpyHostToDevice, pipe->s_in)))
        goto done;
    if (n_cols > 0 &&
        !ok(cudaMemcpyAsync(d_B, B, (size_t)(n_cols * ldb) * 4, cudaMemcpyHostToDevice, pipe->s_in))) goto done;
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
                                        cudaMemcpyHostToDevice, pipe->s_in))) goto done;
                if (val && !ok(cudaMemcpyAsync(d_val + e0, val + e0, (size_t)(e1 - e0) * 4,
                                               cudaMemcpyHostToDevice, pipe->s_in))) goto done;
            }
            if (!ok(cudaEventRecord(pipe->ev_in[(size_t)c], pipe->s_in)) ||
                !ok(cudaStreamWaitEvent(st, pipe->ev_in[(size_t)c], 0)))
                goto done;
            Opts oc = o;
            if (slab) {                               // one workspace, reused chunk after chunk (stream order)
                oc.workspace = w + L.off_slab;
                oc.workspace_bytes = L.slab_bytes;
                oc.nnz = e1 - e0;
            }
            rc = run_rows_impl(row_base + n_rows, n_cols, d_rowptr + r0, base, d_colind, d_val, d_B, F,
                               ldb, s, strategy, seed, reduce, d_C + r0 * dldc, dldc, row_base + r0,
                               row_base + r1, oc, st);
            if (rc != ES_OK) goto done;
            if (!ok(cudaEventRecord(pipe->ev_done[(size_t)c], st)) ||
                !ok(cudaStreamWaitEvent(pipe->s_out, pipe->ev_done[(size_t)c], 0)))
                goto done;
            if (r1 > r0) {
                // one linear copy when the host rows have the device pitch, else a 2-D copy
                const bool flat = ldc == dldc;
                cudaError_t e = flat ? cudaMemcpyAsync(C + r0 * ldc, d_C + r0 * dldc, (size_t)((r1 - r0) * dldc) * 4,
                                                       cudaMemcpyDeviceToHost, pipe->s_out)
                                     : cudaMemcpy2DAsync(C + r0 * ldc, (size_t)ldc * 4, d_C + r0 * dldc,
                                                         (size_t)dldc * 4, (size_t)F * 4, (size_t)(r1 - r0),
                                                         cudaMemcpyDeviceToHost, pipe->s_out);
                if (!ok(e)) goto done;
            }
            r0 = r1;
        }
    }
    if (!ok(cudaEventRecord(pipe->ev_out, pipe->s_out)) || !ok(cudaStreamWaitEvent(st, pipe->ev_out, 0))) goto done;
    ok(cudaStreamSynchronize(st));

done:
    if (err != cudaSuccess || rc != ES_OK) {
        cudaStreamSynchronize(pipe->s_in);
        cudaStreamSynchronize(pipe->s_out);
        cudaStreamSynchronize(st);
    }
    if (own) destroy_pipeline(own);
    if (rc != ES_OK) return rc;
    return err == cudaSuccess ? ES_OK : ES_ERR_CUDA;
}

}  // extern "C"
