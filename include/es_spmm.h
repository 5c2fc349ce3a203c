/* es_spmm.h -- C ABI of the B200-native ES-SpMM sampled SpMM (arXiv 2104.10716).
 *
 * The operation (PAPER.md Doc B):
 *   problem statement, §4.1: "Input to the kernel is a sparse matrix A in CSR
 *     format ... A dense matrix B contains the nodes' features.  The output of the kernel
 *     is a dense matrix C ...  B and C are both in row-major format."
 *   Alg. 1 "Pseudo Code of CacheSample", L952-976:
 *     S = min(row_nnz, shmem_width)                                   (l.6)
 *     for i < S: sample_idx = get_sample_index(i, row_nnz);
 *                sh_data[i], sh_cols[i] = load_A(sample_idx)          (l.7-10)
 *     acc = sum_{j<S} sh_data[j] * B[sh_cols[j], col_id];  C[row_id, col_id] = acc  (l.12-16)
 *   Bucket: first S entries, L1042-1047.  FastRand, Eq. 2:
 *     sample_idx = (shmem_idx * P') mod row_nnz,  P' = 577 (L1058).
 *   GraphSage mean / in-kernel normalisation, L1570-1575 (divides by k_i; R5).
 *   No preprocessing: sampling happens inside the kernel, L1005, L1201.
 *
 * Readings where the paper is silent are listed in DESIGN.md ("Readings R1-R11"):
 *   R1 Eq. 2 applies even when d_i <= s (whole row, permuted order);
 *   R2 duplicates (577 | d_i) are kept and multiplied again; MEAN divides by k_i slots;
 *   R6 seed != 0 rotates row i's FastRand sequence by mix64(seed + G*(i+1)) mod d_i
 *      (i = GLOBAL row id, G = 0x9E3779B97F4A7C15, mix64 = splitmix64 finalizer);
 *      seed == 0 is exactly Eq. 2;
 *   R8 fp32 storage, fp32 FMA accumulation (32-slot chunk partials), IEEE division.
 *
 * Conventions (all entry points):
 *   * Pointers marked [dev] are device pointers; [host] are host pointers.  The caller
 *     owns every buffer.  es_spmm_run / es_spmm_run_rows never allocate.
 *   * Every device call is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream) and returns without synchronising, except where noted.
 *   * Layouts: rowptr int64[n_rows+1] (absolute offsets into colind/val, rowptr[0] may be
 *     non-zero); colind int32[nnz]; val fp32[nnz] or NULL (= all 1.0, the unweighted
 *     adjacency of L615); B fp32 row-major, n_cols rows x ldb (the allocation holds
 *     n_cols*ldb floats; columns F..ldb-1 are padding and are never stored); C fp32
 *     row-major, rows x ldc (columns F..ldc-1 are left untouched).
 *   * CSR invariants (rowptr non-decreasing, 0 <= colind < n_cols) are preconditions,
 *     not checked on the hot path.  Column order within a row is taken as stored
 *     (R4: Bucket keeps the first k stored entries).
 *   * Errors: status codes only, no exceptions or aborts cross the ABI.  Host-checked:
 *     NULL required pointers, negative sizes, s < 1, F < 1, ldb < F, ldc < F, unknown
 *     strategy/reduce -> ES_ERR_INVALID_VALUE.  Misaligned B/C never fail: a narrower
 *     vector path is chosen.  Launch failures -> ES_ERR_CUDA.
 *   * Thread-safe: no mutable global state other than an atomic launch counter.
 *   * There is no CPU fallback: every step of the path runs in this library's kernels.
 */
#ifndef ES_SPMM_H
#define ES_SPMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ES_OK = 0,
    ES_ERR_INVALID_VALUE = 1,
    ES_ERR_MISALIGNED = 2,   /* reserved: misalignment is never fatal */
    ES_ERR_UNSUPPORTED = 3,
    ES_ERR_CUDA = 4
} es_status_t;

enum { ES_BUCKET = 1, ES_FASTRAND = 2 };          /* sampling strategy, §4.4 */
enum { ES_REDUCE_SUM = 0, ES_REDUCE_MEAN = 1 };   /* GCN sum (Eq. 1) / GraphSage mean (L1256) */
enum { ES_MEAN_BY_SAMPLED = 0, ES_MEAN_BY_DEGREE = 1 };
enum { ES_DTYPE_F32 = 0, ES_DTYPE_BF16 = 1 };

/* Sensitivity variants.  Zero-initialised = the defaults
 * every non-_ex entry point uses.
 *   prime        : P' of Eq. 2 (L1064-1067); 0 means 577 (L1058).  Any value >= 1 is accepted
 *                  (the bijection property needs gcd(P', d_i) = 1).
 *   mean_divisor : ES_MEAN_BY_SAMPLED divides MEAN by k_i (reading R5, default) or
 *                  ES_MEAN_BY_DEGREE by the original d_i (the other reading of L1571).
 *   b_dtype      : ES_DTYPE_F32, or ES_DTYPE_BF16: B holds bf16 values (2 bytes; rows 16-B
 *                  aligned, ldb % 8 == 0, F <= 2048, else ES_ERR_UNSUPPORTED); the arithmetic
 *                  stays fp32 (exact widening, fp32 FMA) -- only the storage of B changes. */
typedef struct {
    int32_t struct_size;   /* sizeof(es_spmm_options_t) (forward compatibility) */
    int32_t prime;
    int32_t mean_divisor;
    int32_t b_dtype;
    /* Fused all-gather of C (es_spmm_run_ex only).  n_peers > 0: c_peers [dev]
     * is an array of n_peers device pointers, each the row-0 base of one rank's FULL C
     * (n_rows x ldc; peer buffers mapped with es_ipc_import, own buffer included); the
     * epilogue stores every output row (global id) into all of them over NVLink, so after the
     * kernel plus a cross-rank barrier every rank holds the whole C.  `C` must then be this
     * rank's own full-C base (used for alignment).  (Read only when struct_size covers them.) */
    float* const* c_peers;
    int32_t n_peers;
    /* es_spmm_backward_ex only: 1 = bitwise-reproducible dB (stable radix sort of the sampled
     * slots by column, one writer per dB row; takes stream-ordered scratch and synchronises the
     * stream once to size it; K and n_cols must be < 2^31, else ES_ERR_UNSUPPORTED). */
    int32_t deterministic;
    /* Feature-sliced ("slab") path (es_spmm_run_ex; es_spmm_backward_ex: see there; DESIGN.md §5
     * "Feature-sliced path"; the reason is Alg. 1 l.13-15: C[:, c] needs only B[:, c]).  A caller-owned device
     * workspace of workspace_bytes >= es_spmm_workspace_bytes(...) bytes makes the call
     * materialise the sampled slots once (es_spmm_sample's layout) and run the gather-FMA one
     * 64-float feature slice at a time, each slice's B slab (n_cols x 256 B) L2-resident.  Pass
     * it only when es_spmm_workspace_bytes returned > 0 (that is where it was measured faster);
     * the call takes the path whenever a workspace is given and the slab fits L2.  Same C as
     * the fused kernels within the parity bound; the fused all-gather (c_peers) applies to it as
     * well, and so does bf16 storage of B (128-element slices).  NULL, or a layout the path
     * does not take (B rows not 16-B aligned, F <= 16) = the fused kernels.  The workspace must not be shared by calls in flight.
     * Launches: count + scan + sample materialisation + one per 64-float slice, all on `stream`;
     * no allocation, no synchronisation.  (Read only when struct_size covers them.) */
    void* workspace;
    int64_t workspace_bytes;
    /* Slab path only: 1 = skip the sampling stage (a1-a3) and reuse the sampled slots already in
     * `workspace` from an earlier call on the same rows with the same s, strategy, seed and P'
     * (e.g. the layers of a GNN aggregating over one sampled graph, or timing the gather passes
     * alone).  Checked on the device against the signature the sampling call wrote into the
     * workspace header (rows, s, strategy, seed, P', val presence): on a mismatch every output
     * row of the call is written as NaN and es_spmm_workspace_status reports
     * ES_WS_SIGNATURE_MISMATCH -- never a silently wrong C.  A call that cannot take the slab
     * path (layout) with reuse_sampled = 1 returns ES_ERR_INVALID_VALUE. */
    int32_t reuse_sampled;
    /* Stored entries of the call's rows, rowptr[row_end] - rowptr[row_begin] (a host value the
     * caller knows; the library never reads device memory to size anything).  Sizes the slab
     * path's capacity check: the workspace must hold min(nnz, n_rows * s) slots (0 = unknown:
     * n_rows * s slots).  An undersized workspace returns ES_ERR_INVALID_VALUE.  If the value
     * is wrong (smaller than the truth) the device backstop writes NaN rows and reports
     * ES_WS_OVERFLOW instead of truncating.  (Read only when struct_size covers it.) */
    int64_t nnz;
    /* Kernel selection for A/B measurement and the parity tests' per-family coverage:
     * ES_KERNEL_AUTO (0) = the library's measured plan, else force a family where
     * it applies (ES_ERR_UNSUPPORTED where it cannot run the layout).  tune[] = family knobs,
     * 0 = the default: tune[0] ring depth, tune[1] lanes per slot (slab) / rows per warp (TMA),
     * tune[2] warps per CTA, tune[3] variant bits.  No result changes beyond each family's
     * documented summation order.  (Read only when struct_size covers them.) */
    int32_t kernel;
    int32_t tune[4];
    /* Fused all-gather through NVLink SHARP multicast (NVLS): c_multicast [dev] is
     * the multicast address of every rank's FULL C (n_rows x ldc, e.g. the multicast_ptr of a
     * torch symmetric-memory buffer): the epilogue stores each output row ONCE with multimem.st
     * and the switch delivers it to every rank (instead of n_peers unicast stores).  Takes
     * precedence over c_peers; NULL = not used.  `C` must be this rank's own full-C base (used
     * for alignment).  (Read only when struct_size covers it.) */
    float* c_multicast;
} es_spmm_options_t;

enum {
    ES_KERNEL_AUTO = 0,
    ES_KERNEL_FUSED = 1,        /* the plan's one-launch fused kernel; never the slab path       */
    ES_KERNEL_WARP = 2,         /* LDG warp-per-row gathers                                       */
    ES_KERNEL_TMA = 3,          /* cp.async.bulk ring of whole B rows                             */
    ES_KERNEL_CPASYNC = 4,      /* per-lane cp.async ring, one slot per step                      */
    ES_KERNEL_CPASYNC_HW = 5,   /* per-lane cp.async ring, two slots per step                     */
    ES_KERNEL_SLAB = 6,         /* feature-sliced path with the plan's slab kernel (workspace)    */
    ES_KERNEL_SLAB_SMEM = 7,    /* feature-sliced path, cp.async shared-memory ring               */
    ES_KERNEL_SLAB_LDG = 8,     /* feature-sliced path, register-direct 256-bit gathers           */
    ES_KERNEL_SLAB_TMA = 9,     /* feature-sliced path, TMA tile::gather4 into a shared-memory ring */
    ES_KERNEL_ROWSTREAM = 10,   /* short rows: R rows per warp as one flat slot stream (F <= 128)   */
    ES_KERNEL_SLAB_STREAM = 11, /* feature-sliced path, R rows per warp as one padded slot stream   */
    ES_KERNEL_SLAB_FLOW = 12,   /* feature-sliced path, persistent warps streaming slot-balanced
                                   row ranges across row boundaries (the plan's slab kernel)      */
    ES_KERNEL_GROUPED = 13,     /* short rows, F <= 128: 32-row batches sorted by k_i, a half-warp
                                   per row with register-direct gathers                           */
    ES_KERNEL_SEGSTREAM = 14    /* short rows, F <= 128: R rows per warp as one slot stream, row
                                   and chunk events as lane-parallel ballots, register-direct
                                   double-buffered gathers                                       */
};

/* Status word of a slab workspace (written by the device; reading it synchronises `stream`).
 * ES_WS_OK, or the OR of: ES_WS_OVERFLOW (the sampled slots did not fit: the affected rows of
 * C were written as NaN), ES_WS_SIGNATURE_MISMATCH (reuse_sampled over slots of a different
 * sampling: the call's rows of C were written as NaN).  reset = 1 clears it afterwards. */
enum { ES_WS_OK = 0, ES_WS_OVERFLOW = 1, ES_WS_SIGNATURE_MISMATCH = 2 };
es_status_t es_spmm_workspace_status(void* workspace /*[dev]*/, int64_t workspace_bytes, int32_t reset,
                                     int32_t* status_out /*[host]*/, void* stream);

/* Bytes of workspace es_spmm_run_ex needs to take the slab path for rows holding `nnz` stored
 * entries (pass the same nnz in es_spmm_options_t.nnz; the kernels never read or write past
 * the workspace, and an undersized one is an error, never a truncation), sampling cap s,
 * feature width F, and B of n_cols rows with pitch ldb.  > 0 when the measured plan prefers the
 * slab path: F >= 128, ldb % 4 == 0, a 64-float slab of B (n_cols x 256 B) fits L2, and rows
 * sample enough slots on average.  0 otherwise: pass no workspace then.
 * has_val = 0 when val will be NULL (no slot values are stored); a workspace sized with
 * has_val = 0 is too small for a call with val (ES_ERR_INVALID_VALUE). */
int64_t es_spmm_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb,
                                int32_t s, int32_t has_val);
/* Same, honouring opt->kernel: with a slab kernel forced (ES_KERNEL_SLAB*), > 0 wherever the slab
 * path can run at all (F > 16, ldb % 4 == 0, the slab fits L2), not only where it is measured
 * faster.  opt NULL = es_spmm_workspace_bytes. */
int64_t es_spmm_workspace_bytes_ex(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t F, int64_t ldb,
                                   int32_t s, int32_t has_val, const es_spmm_options_t* opt);

/* Edge sampling materialised (stage 1 of Alg. 1; the paper's "pre-sampled graph",
 * §5.6).
 *   Phase 1 (s_colind == NULL): writes s_rowptr[0..n_rows] [dev] = exclusive prefix sum
 *     of k_i = min(d_i, s), with s_rowptr[0] = 0.  The caller reads s_rowptr[n_rows]
 *     (a D->H sync it performs itself) to size phase 2.
 *   Phase 2: additionally writes, for slot j < k_i of row i, at offset s_rowptr[i] + j:
 *     s_colind[.] = colind[rowptr[i] + p_j], s_val[.] = val[...] (1.0 if val == NULL),
 *     s_pos[.] = p_j (optional, may be NULL), in SLOT order with duplicates kept (R2).
 *     s_val may be NULL (not written).
 *   p_j = j (Bucket) or (off_i + j*577) mod d_i (FastRand, R6), i = row_base + local row.
 *   Phase 1 takes a stream-ordered scratch allocation (cudaMallocAsync) for its scan. */
es_status_t es_spmm_sample(int64_t n_rows, int64_t n_cols,
                           const int64_t* rowptr /*[dev]*/, const int32_t* colind /*[dev]*/,
                           const float* val /*[dev], NULL => 1.0f*/,
                           int32_t s, int32_t strategy, uint64_t seed, int64_t row_base,
                           int64_t* s_rowptr /*[dev] n_rows+1*/, int32_t* s_colind /*[dev]*/,
                           float* s_val /*[dev] or NULL*/, int64_t* s_pos /*[dev] or NULL*/,
                           void* stream);

/* Fused sampled SpMM (Alg. 1 stages 1+2, sampling inside the kernel):
 *   C[i, 0:F] = reduce_{j < k_i} val[e_ij] * B[colind[e_ij], 0:F],  e_ij = rowptr[i] + p_j
 * for i in [0, n_rows); reduce = SUM, or MEAN (divide by k_i; k_i == 0 gives a zero row).
 * Global row id of local row i is i (seeded FastRand offset). */
es_status_t es_spmm_run(int64_t n_rows, int64_t n_cols,
                        const int64_t* rowptr /*[dev]*/, const int32_t* colind /*[dev]*/,
                        const float* val /*[dev] or NULL*/,
                        const float* B /*[dev] n_cols x ldb*/, int64_t F, int64_t ldb,
                        int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                        float* C /*[dev] n_rows x ldc*/, int64_t ldc, void* stream);

/* Same operation restricted to global rows [row_begin, row_end) of a CSR that may be a
 * slice (the multi-GPU path):
 *   rowptr [dev] points at the entries for rows row_begin..row_end (row_end-row_begin+1
 *   values, ABSOLUTE offsets of the global CSR); colind/val [dev] are the slice's arrays
 *   already offset so that global nonzero e lives at colind[e - nnz_base];
 *   C [dev] points at the output row for row_begin.
 * n_rows is the GLOBAL row count (only used for validation); the seeded offset uses the
 * global row id, so the result is bitwise identical to the corresponding rows of
 * es_spmm_run on the full CSR. */
es_status_t es_spmm_run_rows(int64_t n_rows, int64_t n_cols,
                             const int64_t* rowptr /*[dev]*/, int64_t nnz_base,
                             const int32_t* colind /*[dev]*/, const float* val /*[dev] or NULL*/,
                             const float* B /*[dev]*/, int64_t F, int64_t ldb,
                             int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             float* C /*[dev]*/, int64_t ldc,
                             int64_t row_begin, int64_t row_end, void* stream);

/* es_spmm_run_rows with options (NULL = defaults).  B is `const void*` typed by opt->b_dtype. */
es_status_t es_spmm_run_ex(int64_t n_rows, int64_t n_cols,
                           const int64_t* rowptr /*[dev]*/, int64_t nnz_base,
                           const int32_t* colind /*[dev]*/, const float* val /*[dev] or NULL*/,
                           const void* B /*[dev]*/, int64_t F, int64_t ldb,
                           int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                           float* C /*[dev]*/, int64_t ldc, int64_t row_begin, int64_t row_end,
                           const es_spmm_options_t* opt, void* stream);

/* es_spmm_sample with options (only `prime` applies; NULL = defaults). */
es_status_t es_spmm_sample_ex(int64_t n_rows, int64_t n_cols,
                              const int64_t* rowptr, const int32_t* colind, const float* val,
                              int32_t s, int32_t strategy, uint64_t seed, int64_t row_base,
                              int64_t* s_rowptr, int32_t* s_colind, float* s_val, int64_t* s_pos,
                              const es_spmm_options_t* opt, void* stream);

/* Backward w.r.t. B of es_spmm_run_rows (training variant; the paper leaves training with
 * dynamic sampling to future work, §6.2):
 *   dB[col_ij, 0:F] += w_ij * dC[i, 0:F]  over the SAME sampled slots (same s, strategy, seed),
 *   w_ij = val[e_ij] (SUM) or val[e_ij] / k_i (MEAN), i.e. dB += A_s^T dC.
 * Arguments as es_spmm_run_rows; dC [dev] points at row row_begin's gradient (rows x ldc, the
 * allocation holds rows*ldc floats), dB [dev] is the full n_cols x ldb gradient, ACCUMULATED
 * into (the caller zeroes it; several row blocks / ranks may add into one dB).  Uses fp32
 * vector reductions (red.global.add.v4.f32): the order of additions across rows is not
 * deterministic; per-element error <= (n_c + 1) u sum|terms| for n_c contributions. */
es_status_t es_spmm_backward(int64_t n_rows, int64_t n_cols,
                             const int64_t* rowptr /*[dev]*/, int64_t nnz_base,
                             const int32_t* colind /*[dev]*/, const float* val /*[dev] or NULL*/,
                             const float* dC /*[dev]*/, int64_t F, int64_t ldc,
                             int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             float* dB /*[dev] n_cols x ldb*/, int64_t ldb,
                             int64_t row_begin, int64_t row_end, void* stream);

/* es_spmm_backward with options (prime, mean_divisor, deterministic; b_dtype must be
 * ES_DTYPE_F32).  A workspace (as for es_spmm_run_ex, dC/dB 16-B aligned, ldc/ldb % 4 == 0)
 * selects the feature-sliced backward: one pass per 64-float slice, the dB slab L2-resident while
 * its reductions land; with reuse_sampled = 1 it reuses the slots the forward call sampled into
 * that workspace (same rows, s, strategy, seed, P').  deterministic = 1 takes precedence. */
es_status_t es_spmm_backward_ex(int64_t n_rows, int64_t n_cols,
                                const int64_t* rowptr, int64_t nnz_base,
                                const int32_t* colind, const float* val,
                                const float* dC, int64_t F, int64_t ldc,
                                int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                                float* dB, int64_t ldb, int64_t row_begin, int64_t row_end,
                                const es_spmm_options_t* opt, void* stream);

/* End-to-end variant with HOST inputs and output (the call a user with host data makes):
 * copies rowptr/colind/val/B host->device, runs the library's plan on the device copies (the
 * slab path where es_spmm_workspace_bytes would ask for it, else the fused kernel) and copies C
 * back; rowptr entries are absolute offsets with colind[0] holding nonzero rowptr[0].  Pipelined
 * over up to 8 row chunks: B first, then each chunk's colind/val on an internal copy stream while
 * earlier chunks compute on `stream` and their C rows go back on a second copy stream (one linear
 * copy per chunk when ldc == ldb, the device pitch).  Host buffers should be pinned
 * (cudaHostAlloc/cudaHostRegister) for asynchronous copies.
 *   workspace [dev] of es_spmm_host_workspace_bytes(...) bytes is owned by the caller (device
 *   copies of the inputs, C, and room for the slab path's sampled slots).
 * Synchronises `stream` before returning (C is valid on return). */
int64_t es_spmm_host_workspace_bytes(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                     int64_t F, int64_t ldb, int32_t has_val);
es_status_t es_spmm_run_host(int64_t n_rows, int64_t n_cols,
                             const int64_t* rowptr /*[host]*/, const int32_t* colind /*[host]*/,
                             const float* val /*[host] or NULL*/,
                             const float* B /*[host]*/, int64_t F, int64_t ldb,
                             int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                             int64_t row_base /* global id of row 0 (seeded FastRand) */,
                             float* C /*[host]*/, int64_t ldc,
                             void* workspace /*[dev]*/, int64_t workspace_bytes, void* stream);

/* The copy streams and events of the host pipeline, created once and reused across calls
 * (es_spmm_run_host creates and destroys its own per call).  Owned by the caller; one call in
 * flight per pipeline. */
typedef struct es_host_pipeline es_host_pipeline_t;
es_status_t es_host_pipeline_create(es_host_pipeline_t** out);
void es_host_pipeline_destroy(es_host_pipeline_t* pipe);

/* es_spmm_run_host with options (prime, mean_divisor, kernel/tune; workspace, peers, bf16 and
 * reuse_sampled must be unset: ES_ERR_INVALID_VALUE) and a caller-owned pipeline (NULL = a
 * temporary one). */
es_status_t es_spmm_run_host_ex(int64_t n_rows, int64_t n_cols,
                                const int64_t* rowptr /*[host]*/, const int32_t* colind /*[host]*/,
                                const float* val /*[host] or NULL*/,
                                const float* B /*[host]*/, int64_t F, int64_t ldb,
                                int32_t s, int32_t strategy, uint64_t seed, int32_t reduce,
                                int64_t row_base, float* C /*[host]*/, int64_t ldc,
                                void* workspace /*[dev]*/, int64_t workspace_bytes,
                                const es_spmm_options_t* opt, es_host_pipeline_t* pipe, void* stream);

/* Peer-memory helpers for the fused all-gather (one process per GPU of a node).
 *   es_ipc_alloc/free: a dedicated cudaMalloc allocation (so an IPC handle maps exactly it).
 *   es_ipc_export: cudaIpcGetMemHandle of such an allocation into handle_out [host] of
 *     es_ipc_handle_bytes() bytes; es_ipc_import maps a peer's handle (cudaIpcOpenMemHandle,
 *     lazy peer access), es_ipc_close unmaps it.  Importing a handle exported by the same
 *     process is an error (use the local pointer). */
int32_t es_ipc_handle_bytes(void);
es_status_t es_ipc_alloc(int64_t bytes, void** dev_ptr_out);
es_status_t es_ipc_free(void* dev_ptr);
es_status_t es_ipc_export(void* dev_ptr, void* handle_out);
es_status_t es_ipc_import(const void* handle, void** dev_ptr_out);
es_status_t es_ipc_close(void* dev_ptr);

/* Host-side, deterministic row partition for P ranks:
 *   bounds_host[0..n_parts] with bounds[0] = 0, bounds[n_parts] = n_rows, contiguous
 *   blocks of ~equal sum_i w_i, w_i = k_i*(4F+8) + 4F (sampled bytes; reduces to
 *   "balanced by nnz" when s >= max degree).  rowptr_host [host] int64[n_rows+1]. */
es_status_t es_partition_rows(const int64_t* rowptr_host, int64_t n_rows, int32_t s, int64_t F,
                              int32_t n_parts, int64_t* bounds_host);

/* Static description of the kernel the library would launch for (F, ldb, ldc, pointers):
 * writes a short NUL-terminated name into buf (e.g. "es_spmm_warp_v4x5"). */
es_status_t es_spmm_plan(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C,
                         char* buf, int32_t buf_len);
/* Same for a call with sampling cap s over n_rows rows holding nnz stored entries (the fused
 * plan depends on min(s, nnz / n_rows): short rows take the degree-sorted half-warp kernel);
 * nnz = 0: unknown (min(s, .) = s, as es_spmm_run_rows, which states no nnz). */
es_status_t es_spmm_plan_ex(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C, int32_t s,
                            int64_t n_rows, int64_t nnz, char* buf, int32_t buf_len);

/* Number of kernels this library has launched in this process (atomic counter). */
int64_t es_launch_count(void);

const char* es_status_string(es_status_t status);

#ifdef __cplusplus
}
#endif
#endif /* ES_SPMM_H */
