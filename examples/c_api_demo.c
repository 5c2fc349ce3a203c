/* c_api_demo.c -- the ES-SpMM boundary used from plain C (no Python, no torch).
 *
 * Builds a small ragged CSR on the host, copies it to the GPU with the CUDA runtime, runs the
 * fused sampled SpMM (FastRand, s = 3, GraphSage mean) through include/es_spmm.h, and checks
 * every output element against a direct host evaluation of Alg. 1 / Eq. 2 (PAPER.md
 * L952-976, L1064-1067) -- positions (j * 577) mod d, mean over k = min(d, s).  Then the
 * feature-sliced path (es_spmm_run_ex with a caller-owned workspace sized by
 * es_spmm_workspace_bytes_ex; forced here with opt.kernel = ES_KERNEL_SLAB since the graph is tiny) on a
 * 72-wide B (a full 64-float slice + an 8-float tail), checked the same way.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2104_10716_b200 -lesspmm \
 *       -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -o /tmp/c_api_demo
 *   LD_LIBRARY_PATH=paper_2104_10716_b200 /tmp/c_api_demo        (needs a GPU)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "es_spmm.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 2; } } while (0)

/* host Alg. 1: FastRand slot j -> position (j * 577) mod d, MEAN by k */
static void host_ref(int n, const int64_t* rowptr, const int32_t* colind, const float* val, const float* B,
                     int F, int s, float* ref) {
    for (int i = 0; i < n; ++i) {
        int64_t d = rowptr[i + 1] - rowptr[i], k = d < s ? d : s;
        for (int c = 0; c < F; ++c) {
            double acc = 0.0;
            for (int64_t j = 0; j < k; ++j) {
                int64_t e = rowptr[i] + (j * 577) % d;
                acc += (double)val[e] * (double)B[colind[e] * F + c];
            }
            ref[i * F + c] = k ? (float)acc / (float)k : 0.0f;
        }
    }
}

int main(void) {
    enum { N = 6, NC = 9, F = 5, S = 3, F2 = 72 };   /* F2: 16-B row pitch for the slab path */
    const int64_t rowptr[N + 1] = {0, 4, 4, 5, 12, 13, 20};       /* row 1 empty */
    int32_t colind[20];
    float val[20], B[NC * F], C[N * F], ref[N * F];
    for (int e = 0; e < 20; ++e) { colind[e] = (e * 7 + 3) % NC; val[e] = 0.5f + 0.05f * (float)e; }
    for (int i = 0; i < NC * F; ++i) B[i] = (float)((i * 37) % 101) / 101.0f;

    host_ref(N, rowptr, colind, val, B, F, S, ref);

    int64_t* d_rowptr; int32_t* d_colind; float *d_val, *d_B, *d_C;
    CK(cudaMalloc((void**)&d_rowptr, sizeof(rowptr)));
    CK(cudaMalloc((void**)&d_colind, sizeof(colind)));
    CK(cudaMalloc((void**)&d_val, sizeof(val)));
    CK(cudaMalloc((void**)&d_B, sizeof(B)));
    CK(cudaMalloc((void**)&d_C, sizeof(C)));
    CK(cudaMemcpy(d_rowptr, rowptr, sizeof(rowptr), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_colind, colind, sizeof(colind), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_val, val, sizeof(val), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_B, B, sizeof(B), cudaMemcpyHostToDevice));

    es_status_t st = es_spmm_run(N, NC, d_rowptr, d_colind, d_val, d_B, F, F, S, ES_FASTRAND,
                                 /*seed*/ 0, ES_REDUCE_MEAN, d_C, F, /*stream*/ NULL);
    if (st != ES_OK) { fprintf(stderr, "es_spmm_run: %s\n", es_status_string(st)); return 1; }
    CK(cudaMemcpy(C, d_C, sizeof(C), cudaMemcpyDeviceToHost));

    int bad = 0;
    for (int i = 0; i < N * F; ++i)
        if (fabsf(C[i] - ref[i]) > 1e-5f * fabsf(ref[i]) + 1e-6f) ++bad;
    /* an invalid argument is reported, not fatal */
    es_status_t inv = es_spmm_run(N, NC, d_rowptr, d_colind, d_val, d_B, F, F, 0, ES_FASTRAND, 0,
                                  ES_REDUCE_MEAN, d_C, F, NULL);

    /* the slab path: workspace from es_spmm_workspace_bytes, passed through the options */
    static float B2[NC * F2], C2[N * F2], ref2[N * F2];
    for (int i = 0; i < NC * F2; ++i) B2[i] = (float)((i * 53) % 97) / 97.0f;
    host_ref(N, rowptr, colind, val, B2, F2, S, ref2);
    es_spmm_options_t opt = {0};
    opt.struct_size = (int32_t)sizeof(opt);
    opt.kernel = ES_KERNEL_SLAB;                       /* the graph is tiny: force the slab path */
    opt.nnz = 20;                                      /* stored entries of the rows (capacity check) */
    const int64_t ws_bytes = es_spmm_workspace_bytes_ex(N, NC, 20, F2, F2, S, 1, &opt);
    float *d_B2, *d_C2; void* d_ws;
    CK(cudaMalloc((void**)&d_B2, sizeof(B2)));
    CK(cudaMalloc((void**)&d_C2, sizeof(C2)));
    CK(cudaMalloc(&d_ws, (size_t)ws_bytes));
    CK(cudaMemcpy(d_B2, B2, sizeof(B2), cudaMemcpyHostToDevice));
    opt.workspace = d_ws;
    opt.workspace_bytes = ws_bytes;
    const int64_t l0 = es_launch_count();
    st = es_spmm_run_ex(N, NC, d_rowptr, 0, d_colind, d_val, d_B2, F2, F2, S, ES_FASTRAND, 0, ES_REDUCE_MEAN,
                        d_C2, F2, 0, N, &opt, NULL);
    if (st != ES_OK) { fprintf(stderr, "es_spmm_run_ex: %s\n", es_status_string(st)); return 1; }
    CK(cudaMemcpy(C2, d_C2, sizeof(C2), cudaMemcpyDeviceToHost));
    int bad2 = 0;
    for (int i = 0; i < N * F2; ++i)
        if (fabsf(C2[i] - ref2[i]) > 1e-5f * fabsf(ref2[i]) + 1e-6f) ++bad2;

    printf("c_api_demo: %d/%d elements off, s=0 -> %s; slab path (workspace %lld B, %lld launches): "
           "%d/%d off\n", bad, N * F, es_status_string(inv), (long long)ws_bytes,
           (long long)(es_launch_count() - l0), bad2, N * F2);
    cudaFree(d_rowptr); cudaFree(d_colind); cudaFree(d_val); cudaFree(d_B); cudaFree(d_C);
    cudaFree(d_B2); cudaFree(d_C2); cudaFree(d_ws);
    return (bad == 0 && bad2 == 0 && inv == ES_ERR_INVALID_VALUE && ws_bytes > 0) ? 0 : 1;
}
