// es_backward_det.cu -- deterministic backward w.r.t. B (training variant, NEXT-2).
//
// dB = A_s^T dC over the forward's sampled slots (§6.2 L1577-1586 future work),
// bitwise reproducible: the sampled matrix is transposed by a STABLE radix sort of its slots
// on the column index (cub::DeviceRadixSort, values = slot ids in row-major order), then one
// warp per B row sums that row's contributions in (row, slot) order and is the only writer
// of dB[c].  Cost: one pass writing K (col, slot, row, w) records, a sort of K keys, and a
// gather of dC rows -- versus the default atomic scatter (es_backward in es_kernels.cu).
#include <cstdint>
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "es_device.cuh"
#include "es_internal.h"

namespace es {
namespace {

constexpr int kThr = 256;
constexpr int kWpb = kThr / 32;

// one record per sampled slot (row-major slot order o = s_rowptr[r] + j)
__global__ void __launch_bounds__(kThr)
det_records(const BwdParams p, const int64_t* __restrict__ s_rowptr, int32_t* __restrict__ key,
            int32_t* __restrict__ slot, int32_t* __restrict__ slot_row, float* __restrict__ slot_w) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    RowSampler rs;
    rs.init(p.rowptr[r] - p.nnz_base, p.rowptr[r + 1] - p.nnz_base, p.s, p.strategy, p.seed,
            p.row_base + r, p.prime);
    const int64_t o0 = s_rowptr[r];
    const float div = (float)(p.mean_by_degree ? rs.d : (int64_t)rs.k);
    for (int32_t j = lane; j < rs.k; j += 32) {
        const int64_t e = rs.beg + rs.pos(j);
        const int64_t o = o0 + j;
        const float a = p.val ? p.val[e] : 1.0f;
        key[o] = p.colind[e];
        slot[o] = (int32_t)o;
        slot_row[o] = (int32_t)r;
        slot_w[o] = p.reduce == kMean ? __fdiv_rn(a, div) : a;
    }
}

// s_rowptr[i+1] = k_i (inclusive-scanned afterwards)
__global__ void det_count(const BwdParams p, int64_t* __restrict__ s_rowptr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) s_rowptr[0] = 0;
    if (i < p.n_rows) {
        const int64_t d = p.rowptr[i + 1] - p.rowptr[i];
        s_rowptr[i + 1] = d < (int64_t)p.s ? d : (int64_t)p.s;
    }
}

// col_ptr[c + 1] = number of sorted keys equal to c (run lengths; integer, order-free)
__global__ void det_col_hist(const int32_t* __restrict__ key, int64_t K, int64_t* __restrict__ col_cnt) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < K) atomicAdd(reinterpret_cast<unsigned long long*>(col_cnt + key[e] + 1), 1ull);
}

// one warp per B row c: dB[c, :] += sum over its slots, in (row, slot) order
__global__ void __launch_bounds__(kThr)
det_gather(const BwdParams p, int64_t n_cols, const int64_t* __restrict__ col_ptr,
           const int32_t* __restrict__ slot, const int32_t* __restrict__ slot_row,
           const float* __restrict__ slot_w) {
    constexpr int kPer = 8;                                   // features per lane per tile
    const int lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * kWpb + (threadIdx.x >> 5);
    if (c >= n_cols) return;
    const int64_t e0 = col_ptr[c], e1 = col_ptr[c + 1];
    if (e0 == e1) return;
    float* dBrow = p.dB + c * p.ldb;
    for (int64_t f0 = 0; f0 < p.F; f0 += 32 * kPer) {
        float acc[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) acc[q] = 0.0f;
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t o = slot[e];
            const float w = slot_w[o];
            const float* dCrow = p.dC + (int64_t)slot_row[o] * p.ldc;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int64_t f = f0 + lane + 32 * q;
                if (f < p.F) acc[q] = fmaf(w, dCrow[f], acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int64_t f = f0 + lane + 32 * q;
            if (f < p.F) dBrow[f] += acc[q];
        }
    }
}


// Stream-ordered scratch allocations released on every return path: whatever was
// allocated is freed, in stream order, when the owner goes out of scope.
struct Scratch {
    cudaStream_t st;
    void* ptrs[12] = {};
    int n = 0;
    template <typename T>
    cudaError_t get(T** out, int64_t count) {
        *out = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), (size_t)(count > 0 ? count : 1) * sizeof(T), st);
        if (e == cudaSuccess) ptrs[n++] = *out;
        return e;
    }
    cudaError_t bytes(void** out, size_t nb) {
        *out = nullptr;
        cudaError_t e = cudaMallocAsync(out, nb > 0 ? nb : 1, st);
        if (e == cudaSuccess) ptrs[n++] = *out;
        return e;
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(ptrs[i], st);
    }
};

}  // namespace

cudaError_t launch_backward_deterministic(const BwdParams& p, int64_t n_cols, cudaStream_t st,
                                          int* launches, bool* too_large) {
    *too_large = false;
    if (p.n_rows <= 0 || n_cols <= 0) return cudaSuccess;
    Scratch sc{st};
    cudaError_t err;
    int64_t* s_rowptr = nullptr;
    if ((err = sc.get(&s_rowptr, p.n_rows + 1)) != cudaSuccess) return err;
    det_count<<<(unsigned)((p.n_rows + 1 + 255) / 256), 256, 0, st>>>(p, s_rowptr);
    ++*launches;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    if ((err = cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, s_rowptr + 1, s_rowptr + 1, p.n_rows, st)) !=
            cudaSuccess ||
        (err = sc.bytes(&temp, temp_bytes)) != cudaSuccess ||
        (err = cub::DeviceScan::InclusiveSum(temp, temp_bytes, s_rowptr + 1, s_rowptr + 1, p.n_rows, st)) !=
            cudaSuccess)
        return err;
    ++*launches;
    int64_t K = 0;                                            // the one D->H sync of this mode
    if ((err = cudaMemcpyAsync(&K, s_rowptr + p.n_rows, sizeof(K), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (err = cudaStreamSynchronize(st)) != cudaSuccess)
        return err;
    if (K >= (int64_t)INT32_MAX || n_cols >= (int64_t)INT32_MAX) {
        *too_large = true;
        return cudaSuccess;
    }
    if (K == 0) return cudaSuccess;
    int32_t *key = nullptr, *key_s = nullptr, *slot = nullptr, *slot_s = nullptr, *slot_row = nullptr;
    float* slot_w = nullptr;
    int64_t* col_ptr = nullptr;
    if ((err = sc.get(&key, K)) != cudaSuccess || (err = sc.get(&key_s, K)) != cudaSuccess ||
        (err = sc.get(&slot, K)) != cudaSuccess || (err = sc.get(&slot_s, K)) != cudaSuccess ||
        (err = sc.get(&slot_row, K)) != cudaSuccess || (err = sc.get(&slot_w, K)) != cudaSuccess ||
        (err = sc.get(&col_ptr, n_cols + 1)) != cudaSuccess)
        return err;
    det_records<<<(unsigned)((p.n_rows + kWpb - 1) / kWpb), kThr, 0, st>>>(p, s_rowptr, key, slot, slot_row,
                                                                           slot_w);
    ++*launches;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    int end_bit = 1;
    while (end_bit < 31 && (1ll << end_bit) < n_cols) ++end_bit;
    temp_bytes = 0;
    void* temp2 = nullptr;
    if ((err = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, key, key_s, slot, slot_s, (int)K, 0, end_bit,
                                               st)) != cudaSuccess ||
        (err = sc.bytes(&temp2, temp_bytes)) != cudaSuccess ||
        (err = cub::DeviceRadixSort::SortPairs(temp2, temp_bytes, key, key_s, slot, slot_s, (int)K, 0, end_bit,
                                               st)) != cudaSuccess)  // stable
        return err;
    ++*launches;
    if ((err = cudaMemsetAsync(col_ptr, 0, (size_t)(n_cols + 1) * sizeof(int64_t), st)) != cudaSuccess) return err;
    det_col_hist<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(key_s, K, col_ptr);
    ++*launches;
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    temp_bytes = 0;
    void* temp3 = nullptr;
    if ((err = cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, col_ptr + 1, col_ptr + 1, n_cols, st)) !=
            cudaSuccess ||
        (err = sc.bytes(&temp3, temp_bytes)) != cudaSuccess ||
        (err = cub::DeviceScan::InclusiveSum(temp3, temp_bytes, col_ptr + 1, col_ptr + 1, n_cols, st)) != cudaSuccess)
        return err;
    ++*launches;
    det_gather<<<(unsigned)((n_cols + kWpb - 1) / kWpb), kThr, 0, st>>>(p, n_cols, col_ptr, slot_s, slot_row,
                                                                         slot_w);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace es
