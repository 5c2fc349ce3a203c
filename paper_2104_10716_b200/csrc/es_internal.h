// es_internal.h -- internal (C++) interface between the C ABI layer and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace es {

// Kernel selection / A-B knobs (es_spmm_options_t.kernel + tune[]; 0 = the measured default).
// The product path reads no environment: everything arrives through the options struct.
struct Tune {
    int kernel = 0;      // ES_KERNEL_*
    int stages = 0;      // ring depth
    int width = 0;       // lanes per slot (slab) / rows per warp (TMA)
    int cta_warps = 0;   // warps per CTA
    int variant = 0;     // kernel-specific variant bits
};

struct SpmmParams {
    const int64_t* rowptr;   // local row r uses rowptr[r], rowptr[r+1] (absolute offsets)
    int64_t nnz_base;        // subtracted from rowptr entries before indexing colind/val
    const int32_t* colind;
    const float* val;        // NULL => 1.0
    const float* B;
    int64_t F, ldb;
    int32_t s, strategy;
    uint64_t seed;
    int32_t reduce;
    int32_t c_vec;           // vector stores to C allowed
    float* C;                // row r of this launch at C + r*ldc
    int64_t ldc;
    int64_t n_rows;          // rows in this launch
    int64_t row_base;        // global id of local row 0 (seeded FastRand offset)
    uint32_t prime;          // P' (577 unless overridden, NEXT-4)
    int32_t mean_by_degree;  // MEAN divides by d_i instead of k_i (NEXT-4)
    int32_t b_bf16;          // B stored as bf16 (fp32 accumulation, NEXT-4)
    float* const* c_peers;   // fused all-gather: full-C bases of every rank (NEXT-1)
    int32_t n_peers;         // 0: plain store to C
    float* c_mc;             // fused all-gather through NVLS multicast (multimem.st), or NULL
};

struct Plan {
    int vec;        // floats per gather (4, 2, 1)
    bool subwarp;   // small-F streamed mapping
    int g;          // lanes per stream (subwarp)
    int nch;        // vectors per lane per feature tile (warp)
    bool c_vec;
    bool tma;          // TMA-ring kernel (spmm_tma)
    bool cpasync;      // cp.async ring kernel (spmm_cpasync)
    bool bf16;         // B stored as bf16 (cp.async ring only)
    bool halfwarp;     // cp.async ring, two slots per step (spmm_cpasync_hw)
    bool rowstream;    // several short rows per warp as one slot stream (spmm_rowstream)
    bool grouped;      // short rows: degree-sorted 32-row batches, a half-warp per row (spmm_grouped)
    bool segstream;    // short rows: R rows per warp as one register-direct slot stream (spmm_segstream)
    bool unsupported;  // no kernel for this layout (bf16 with misaligned rows)
    int stages;         // ring depth (tma)
    int rows_per_warp;  // consecutive rows per warp (tma)
    int minb;           // __launch_bounds__ min blocks per SM (tma register cap)
    int u;              // slots in flight per lane (warp kernel, NCH == 1: 8 or 16)
};

// Backward w.r.t. B: dB[col_ij] += w_ij * dC[i]  (w = val, or val / k_i for MEAN)
struct BwdParams {
    const int64_t* rowptr;   // local row r uses rowptr[r], rowptr[r+1] (absolute offsets)
    int64_t nnz_base;
    const int32_t* colind;
    const float* val;
    const float* dC;         // row r of this launch at dC + r*ldc
    int64_t F, ldc;
    int32_t s, strategy;
    uint64_t seed;
    int32_t reduce;
    float* dB;               // n_cols x ldb, accumulated
    int64_t ldb;
    int64_t n_rows, row_base;
    int32_t vec;             // 4, 2, 1 (alignment of dC, dB, ldc, ldb)
    uint32_t prime;
    int32_t mean_by_degree;
};

// One feature slice of the slab path (es_slab.cu): C[:, 0:w] of the slice from the compact
// sampled slots (es_spmm_sample layout) and the slice's B columns.
struct SlabParams {
    const int64_t* s_rowptr;  // local row r: slots [s_rowptr[r] - slot_base, s_rowptr[r+1] - slot_base)
    int64_t slot_base;
    int64_t cap;              // slots the workspace holds (reads are clamped to it)
    const int32_t* s_colind;
    const float* s_val;       // NULL => 1.0
    const int64_t* rowptr;    // original CSR rows (MEAN by degree only)
    const float* B;           // the slice's first column, row pitch ldb (16-B aligned)
    int64_t ldb;
    int32_t w;                // floats in the slice (<= 64)
    int32_t nv;               // 16-B pieces in the slice = ceil(w / 4) (<= 16)
    float* C;                 // the slice's first column of local row 0
    int64_t ldc;
    int32_t c_vec;
    int64_t n_rows;
    int32_t reduce;
    int32_t mean_by_degree;
    float* const* c_peers;    // fused all-gather (NEXT-1): full-C bases of every rank, or NULL
    int32_t n_peers;
    float* c_mc;              // fused all-gather through NVLS multicast (multimem.st), or NULL
    int64_t row_base;         // global id of local row 0 (peer stores)
    int64_t col0;             // the slice's first column (peer stores)
    int32_t b_bf16;           // B holds bf16 (NEXT-4 storage variant): B points at uint16_t elements
    int32_t b32;              // B base and row pitch 32-B aligned (256-bit gathers possible)
    int32_t direct_s;         // > 0 (Bucket): the slots are the CSR itself -- s_rowptr/s_colind/s_val
                              // are rowptr/colind/val, k_i = min(d_i, direct_s); no sampling pass
    // device backstops (workspace header, DESIGN.md §1 "Boundary"): a row whose slots end past
    // `cap` (overflow) or a call whose expected sampling signature differs from the one the
    // sampling pass wrote (reuse_sampled) writes NaN rows and ORs a flag into *ws_status
    int32_t* ws_status;       // NULL: no workspace (direct Bucket slots)
    const uint64_t* ws_sig;   // signature written by the sampling call (NULL: not checked)
    uint64_t sig;             // the signature this call expects
    int32_t reuse_s;          // > 0 (reuse_sampled): also check each row's slot count == min(d_i, reuse_s)
    // flow layout (spmm_slab_flow): rows padded to 4-slot multiples, k_i = min(d_i, s) from rowptr
    int32_t s;                // the sampling cap s
    const int32_t* s_k;       // flow layout: k_i = min(d_i, s) of every row (the count kernel's)
    int32_t pad;              // backward: slot padding of the layout (1 compact, 4 flow; col -1 = padding)
};

// workspace header (first 256 B of a slab workspace)
struct WsHeader {
    uint64_t sig;             // signature of the sampling call that filled the slots
    int32_t status;           // ES_WS_* flags (device-written)
    int32_t pad;
};
constexpr int kWsOverflow = 1, kWsSignature = 2;

cudaError_t launch_slab_pass(const SlabParams& p, const Tune& t, cudaStream_t st);
// Flow slab path (the default, es_slab.cu spmm_slab_flow): one slice pass over the padded slot
// layout.  Slices of up to 16 pieces run the 2-piece-per-lane kernel, up to 24 the 3-piece one.
cudaError_t launch_slab_flow(const SlabParams& p, const Tune& t, cudaStream_t st);
// TMA gather4 slab pass: tm = a 2-D tensor map over B (inner dim F elements, rows n_cols, box
// {256 B of elements, 1}), c0 = the slice's first column
cudaError_t launch_slab_pass_tma(const CUtensorMap& tm, const SlabParams& p, int32_t c0, int32_t n_cols,
                                 const Tune& t, cudaStream_t st);
// encodes that tensor map (driver entry point, no libcuda link); false if the layout is not
// expressible (pitch not a multiple of 16 B, > 2^31 rows, ...)
bool encode_b_tensor_map(CUtensorMap* tm, const void* B, int64_t F, int64_t ldb, int64_t n_cols, bool bf16);

// backward slab pass: p.C/ldc describe dC's slice (read), dB the slice of the gradient (reduced into)
cudaError_t launch_slab_backward(const SlabParams& p, const float* dC, float* dB, cudaStream_t st);
size_t slab_scan_temp_bytes(int64_t n);
// hdr (may be NULL): the workspace header, cleared by the count kernel (status 0, signature 0)
cudaError_t launch_slab_count(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr, void* temp,
                              size_t temp_bytes, cudaStream_t st, int* launches, WsHeader* hdr = nullptr,
                              int32_t pad = 1, int32_t* s_k = nullptr);
// s_k (may be NULL): k_i of every row, unpadded
cudaError_t launch_sample_count_only(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr,
                                     cudaStream_t st, WsHeader* hdr = nullptr, int32_t pad = 1,
                                     int32_t* s_k = nullptr);

cudaError_t launch_backward(const BwdParams& p, cudaStream_t st);
cudaError_t launch_backward_deterministic(const BwdParams& p, int64_t n_cols, cudaStream_t st, int* launches,
                                          bool* too_large);

// k_est: expected sampled slots per row, min(s, nnz / rows) when the caller stated nnz, else s
Plan make_plan(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C, int32_t s = INT32_MAX,
               const Tune& t = Tune{}, int64_t k_est = -1);
Plan make_plan_bf16(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C);
cudaError_t launch_spmm(SpmmParams p, const Plan& plan, const Tune& t, cudaStream_t st);
cudaError_t launch_sample_count(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr,
                                cudaStream_t st, int* launches);
cudaError_t launch_sample_materialize(const int64_t* rowptr, int64_t nnz_base, const int32_t* colind,
                                      const float* val, int64_t n, int32_t s, int32_t strategy,
                                      uint64_t seed, int64_t row_base, uint32_t prime,
                                      const int64_t* s_rowptr, int32_t* s_colind, float* s_val,
                                      int64_t* s_pos, cudaStream_t st, int64_t cap = INT64_MAX,
                                      WsHeader* hdr = nullptr, uint64_t sig = 0, int32_t pad = 1);

}  // namespace es
