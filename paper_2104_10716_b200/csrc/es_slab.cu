// es_slab.cu -- feature-sliced ("slab") path of the sampled SpMM for wide F.
//
// Why: the gather-FMA touches every B row a row of A samples.  When B does not
// fit the 126 MB L2 (Reddit-shaped, F=602: 566 MB), most gathers go to HBM although each B row
// is gathered ~170 times per call.  C[:, c] depends only on B[:, c] (Alg. 1 l.13-15 is a
// per-feature sum), so the call is split into feature slices of 64 fp32 (or 128 bf16) elements
// whose B slab (n_cols x 256 B = 60 MB for Reddit) stays L2-resident for the whole pass:
//   1. es::launch_sample_count + scan : k_i = min(d_i, s) and its prefix     (a1, Alg. 1 l.5-6)
//   2. es::launch_sample_materialize   : the sampled (col, val) of every row, slot order, compact
//                                        (a2 + a3, Alg. 1 l.7-11 / Eq. 2) -- read once per call
//   3. spmm_slab, once per slice       : a4 + a5 over the compact slots   (Alg. 1 l.12-16)
// Per element, slot j of a row is FMA'd (fp32) into the partial of lane group (j mod S); each
// group adds its partial to its total every 32 slots; the group totals are added by an xor tree
// (with S = 2 groups the order of spmm_cpasync_hw, bitwise; DESIGN.md §6 error bound).
// Also here: the feature-sliced backward (spmm_slab_bwd, NEXT-2).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include "es_device.cuh"
#include "es_internal.h"

namespace es {
namespace {

constexpr int kSlabThreads = 256;
constexpr int kSlabWarps = kSlabThreads / 32;
constexpr unsigned kAll = 0xffffffffu;

// 16-B global -> shared copy, zero-filling when src_bytes == 0 (no global read is made): the
// ring is refilled branch-free, slots past the row's end land as zeros.
// (.cg: L2 only -- the .ca form, L1-allocating, measured slower: profiles/r01.md)
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}

// A 16-B piece of a B row: 4 fp32, or 8 bf16 widened exactly to fp32 (NEXT-4 storage variant).
template <bool BF16> struct SlabPiece;
template <> struct SlabPiece<false> {
    static constexpr int kElems = 4;
    __device__ __forceinline__ static void widen(const float4& raw, float* out) {
        out[0] = raw.x; out[1] = raw.y; out[2] = raw.z; out[3] = raw.w;
    }
};
template <> struct SlabPiece<true> {
    static constexpr int kElems = 8;
    __device__ __forceinline__ static void widen(const float4& raw, float* out) {
        const uint32_t w[4] = {__float_as_uint(raw.x), __float_as_uint(raw.y), __float_as_uint(raw.z),
                               __float_as_uint(raw.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            out[2 * i] = __uint_as_float(w[i] << 16);
            out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
};

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}

// One warp per row, split into S = 32/G groups of G lanes.  Step u of a 32-slot chunk consumes
// slots S*u + e (group e = lane / G); lane `sub` = lane % G of a group owns the P 16-B pieces
// sub + G*q (q < P) of the slice (nv <= G*P <= 16 pieces), so each LDGSTS instruction of a
// group covers G*16 contiguous bytes.  A narrow last slice uses fewer lanes per slot (more
// slots per step, fewer steps).  The copy for step u + D is issued right after step u is
// consumed, into the stage it released.  Per element: group e sums slots j = e (mod S) in slot
// order (32-slot-chunk partials), then an xor tree over the groups (G = 16: spmm_cpasync_hw's
// order, bitwise).
// W warps per CTA (register cap as for MINB 256-thread CTAs per SM): small CTAs free their
// slot as soon as their few rows are done instead of waiting for the longest of 8 rows.
template <int G, int P, int D, int MINB, bool FULL, int W, bool BF16 = false>
__global__ void __launch_bounds__(32 * W, MINB * 8 / W)
spmm_slab(const SlabParams p) {
    constexpr int E = SlabPiece<BF16>::kElems;   // B elements (-> fp32 accumulators) per piece
    constexpr int S = 32 / G;            // slots per step
    constexpr int U = 32 / S;            // steps per 32-slot chunk (= G)
    static_assert((G == 2 || G == 4 || G == 8 || G == 16) && G * P <= 16, "lanes x pieces per slot");
    static_assert(D >= 2 && U % D == 0, "ring depth must divide the steps of a chunk");
    constexpr int kStage = 32 * P;                               // float4 per warp stage
    extern __shared__ __align__(16) float4 slab_ring[];          // [warps][D][S][P][G]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int e = lane / G, sub = lane % G;
    const int64_t r = (int64_t)blockIdx.x * W + warp;
    if (r >= p.n_rows) return;
    const int64_t beg = ld_stream(p.s_rowptr + r, policy_evict_first()) - p.slot_base;
    int64_t end = ld_stream(p.s_rowptr + r + 1, policy_evict_first()) - p.slot_base;
    if (end > p.cap) end = p.cap;                                // workspace bound (never read past)
    if (p.direct_s > 0 && end - beg > p.direct_s) end = beg + p.direct_s;   // Bucket: first s of the row
    const int32_t k = end > beg ? (int32_t)(end - beg) : 0;
    const uint32_t my_s = smem_u32(slab_ring + (size_t)warp * D * kStage + e * (P * G) + sub);
    const char* bl = reinterpret_cast<const char*>(p.B) + sub * 16;
    const uint32_t row_bytes = (uint32_t)(p.ldb * (BF16 ? 2 : 4));

    // FULL: all 16 pieces of the slice exist (every slice but a narrower last one)
    auto copy = [&](int stage, int32_t col, bool valid) {
        const char* src = bl + (uint64_t)(uint32_t)col * row_bytes;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const bool on = FULL ? valid : (valid && sub + G * q < p.nv);
            cp_async16_zfill(my_s + (stage * kStage + q * G) * 16, src + q * G * 16, on ? 16u : 0u);
        }
    };
    auto load_pair = [&](int64_t j, int32_t& c, float& a) {      // slot j of the row (coalesced)
        const uint64_t pol = policy_evict_first();
        c = ld_stream(p.s_colind + beg + j, pol);
        a = p.s_val ? ld_stream(p.s_val + beg + j, pol) : 1.0f;
    };

    // (col, val) of the chunk being consumed (c0, a0) and of the next one (c1, a1); slots past
    // k carry (0, 0.0f), so their (zero-filled) pieces add exactly +0.
    int32_t c0 = 0, c1 = 0;
    float a0 = 0.0f, a1 = 0.0f;
    if (lane < k) load_pair(lane, c0, a0);
    if (32 + lane < k) load_pair(32 + lane, c1, a1);
#pragma unroll
    for (int t = 0; t < D; ++t) {
        copy(t, __shfl_sync(kAll, c0, S * t + e), S * t + e < k);
        cp_async_commit();
    }
    float part[P][E], tot[P][E];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < E; ++c) { part[q][c] = 0.0f; tot[q][c] = 0.0f; }
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
#pragma unroll 1
        for (int u0 = 0; u0 < U; u0 += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {                        // step u = u0 + d, stage d
                const int u = u0 + d;
                cp_async_wait<D - 1>();                          // step u has landed
                const float av = __shfl_sync(kAll, a0, S * u + e);
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    float x[E];
                    SlabPiece<BF16>::widen(lds128(my_s + (d * kStage + q * G) * 16), x);
#pragma unroll
                    for (int c = 0; c < E; ++c) part[q][c] = fmaf(av, x[c], part[q][c]);
                }
                const int tn = u + D;                            // refill: step u + D
                const int32_t cn = __shfl_sync(kAll, tn < U ? c0 : c1, (S * tn + e) & 31);
                copy(d, cn, j0 + S * tn + e < k);
                cp_async_commit();
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
            for (int c = 0; c < E; ++c) { tot[q][c] += part[q][c]; part[q][c] = 0.0f; }
        c0 = c1;
        a0 = a1;
        c1 = 0;
        a1 = 0.0f;
        if (j0 + 64 + lane < k) load_pair(j0 + 64 + lane, c1, a1);
    }
    cp_async_wait<0>();
    const uint64_t pol_a = policy_evict_first();
    int64_t div = k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
    // xor tree over the S groups: (g0 + g1) + (g2 + g3) ...; commutative adds, so every lane of
    // every group ends with the same bits
#pragma unroll
    for (int o = G; o < 32; o <<= 1)
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
            for (int c = 0; c < E; ++c) {
                const float other = __shfl_xor_sync(kAll, tot[q][c], o);
                tot[q][c] = (lane & o) ? other + tot[q][c] : tot[q][c] + other;
            }
    if (e == 0) {
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const int piece = sub + G * q;
            if (FULL || piece < p.nv) {
#pragma unroll
                for (int h4 = 0; h4 < E / 4; ++h4) {                 // 4 output floats at a time
                    float res[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float t = tot[q][4 * h4 + c];
                        res[c] = p.reduce == kMean ? (div > 0 ? __fdiv_rn(t, (float)div) : 0.0f) : t;
                    }
                    const int col = piece * E + 4 * h4;              // first output column
                    const int rem = p.w - col;                       // valid floats from there
                    auto put = [&](float* dst) {
                        if (p.c_vec && rem >= 4) st_stream4(dst, res, pol_a);
                        else
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                if (c < rem) st_stream(dst + c, res[c], pol_a);
                    };
                    if (rem <= 0) continue;
                    if (p.n_peers == 0) {
                        put(p.C + r * p.ldc + col);
                    } else {                                     // fused all-gather: every rank's C
                        const int64_t off = (p.row_base + r) * p.ldc + p.col0 + col;
                        for (int q2 = 0; q2 < p.n_peers; ++q2) put(p.c_peers[q2] + off);
                    }
                }
            }
        }
    }
}

template <int G, int P, int D, int MINB, int W, bool BF16 = false>
cudaError_t launch_slab_w(const SlabParams& p, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + W - 1) / W;
    const size_t smem = (size_t)W * D * 32 * P * 16;
    auto k = p.nv == G * P ? spmm_slab<G, P, D, MINB, true, W, BF16> : spmm_slab<G, P, D, MINB, false, W, BF16>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

template <int G, int D, int MINB, int P = 16 / G>
cudaError_t launch_slab_k(const SlabParams& p, cudaStream_t st) {
    const char* we = getenv("ES_SPMM_SLAB_CTA_WARPS");     // tuning: warps per CTA (default 4)
    const int w = we ? atoi(we) : 4;
    if (w == 1) return launch_slab_w<G, P, D, MINB, 1>(p, st);
    if (w == 2) return launch_slab_w<G, P, D, MINB, 2>(p, st);
    if (w == 8) return launch_slab_w<G, P, D, MINB, 8>(p, st);
    return launch_slab_w<G, P, D, MINB, 4>(p, st);
}

// ---------------------------------------------------------------- backward (NEXT-2), slab path
// dB[col_ij, c0:c0+w] += w_ij * dC[i, c0:c0+w] over the compact sampled slots, one launch per
// 64-float slice, so the dB slab the reductions land in (n_cols x 256 B) stays L2-resident and
// the 16-B vector reductions (red.global.add.v4.f32) resolve in L2 instead of read-modify-
// writing HBM.  One warp per row; the row's dC slice is read once into registers (MEAN: divided
// by the row's divisor with IEEE division, as the fused backward); 4 slots per step (groups of 8
// lanes, 2 pieces each).  Addition order across rows is not deterministic (as the fused one).
template <int W>
__global__ void __launch_bounds__(32 * W, 32 / W)
spmm_slab_bwd(const SlabParams p, const float* __restrict__ dC, float* __restrict__ dB) {
    constexpr int G = 8, P = 2, S = 4;
    const int lane = threadIdx.x & 31;
    const int e = lane / G, sub = lane % G;
    const int64_t r = (int64_t)blockIdx.x * W + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    const int64_t beg = ld_stream(p.s_rowptr + r, pol_a) - p.slot_base;
    int64_t end = ld_stream(p.s_rowptr + r + 1, pol_a) - p.slot_base;
    if (end > p.cap) end = p.cap;
    if (p.direct_s > 0 && end - beg > p.direct_s) end = beg + p.direct_s;
    const int32_t k = end > beg ? (int32_t)(end - beg) : 0;
    if (k == 0) return;
    float div = (float)k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = (float)(ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a));
    float x[P][4];
#pragma unroll
    for (int q = 0; q < P; ++q) {
        const int piece = sub + G * q;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int col = piece * 4 + c;
            float v = col < p.w ? ld_stream(dC + r * p.ldc + col, pol_a) : 0.0f;
            x[q][c] = p.reduce == kMean ? __fdiv_rn(v, div) : v;
        }
    }
    const int64_t ldb = p.ldb;
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
        int32_t cj = 0;
        float aj = 0.0f;
        if (j0 + lane < k) {
            cj = ld_stream(p.s_colind + beg + j0 + lane, pol_a);
            aj = p.s_val ? ld_stream(p.s_val + beg + j0 + lane, pol_a) : 1.0f;
        }
        const int n_here = min(32, k - j0);
        for (int u = 0; u < (n_here + S - 1) / S; ++u) {
            const int slot = S * u + e;
            const int32_t cn = __shfl_sync(kAll, cj, slot);
            const float av = __shfl_sync(kAll, aj, slot);
            if (slot < n_here) {
                float* brow = dB + (int64_t)(uint32_t)cn * ldb;
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int piece = sub + G * q;
                    if (piece < p.nv) {
                        if (piece * 4 + 4 <= p.w)
                            red_add4(brow + piece * 4, av * x[q][0], av * x[q][1], av * x[q][2], av * x[q][3]);
                        else
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                if (piece * 4 + c < p.w) red_add1(brow + piece * 4 + c, av * x[q][c]);
                    }
                }
            }
        }
    }
}

}  // namespace

// Instantiations: G = 8 (default: 2 pieces per lane, 4 slots per step) or 16; D = 2, 4, 8.
// MINB = the register cap that does not spill (spilling cp.async kernels trapped on B200,
// _build.py refuses them).  Measured alternatives (register-staged LDG with every cache
// operator, cp.async.ca, 4 lanes per slot, a row-stream variant over a padded layout) were
// all slower: profiles/r01.md "Slab path".
cudaError_t launch_slab_pass(const SlabParams& p, int lanes_per_slot, int stages, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    if (p.b_bf16) {                      // bf16 B (NEXT-4): 128-element slices, 8 elements per piece
        if (p.nv <= 4) return launch_slab_w<2, 2, 2, 3, 4, true>(p, st);
        if (p.nv <= 8) return launch_slab_w<4, 2, 4, 3, 4, true>(p, st);
        return lanes_per_slot == 16 ? launch_slab_w<16, 1, 4, 4, 4, true>(p, st)
                                    : launch_slab_w<8, 2, 4, 3, 4, true>(p, st);
    }
    if (lanes_per_slot == 16) {
        switch (stages) {
            case 2: return launch_slab_k<16, 2, 5>(p, st);
            case 8: return launch_slab_k<16, 8, 4>(p, st);
            default: return launch_slab_k<16, 4, 5>(p, st);
        }
    }
    // narrow last slice: 4 lanes x 2 pieces (8 slots per step) for <= 8 pieces, 2 x 2 (16 slots
    // per step) for <= 4 -- half / a quarter of the steps of a full slice
    if (p.nv <= 4) return launch_slab_k<2, 2, 4, 2>(p, st);
    if (p.nv <= 8) return launch_slab_k<4, 4, 4, 2>(p, st);
    switch (stages) {
        case 2: return launch_slab_k<8, 2, 4>(p, st);
        case 8: return launch_slab_k<8, 8, 4>(p, st);
        default: return launch_slab_k<8, 4, 4>(p, st);
    }
}

cudaError_t launch_slab_backward(const SlabParams& p, const float* dC, float* dB, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    constexpr int W = 4;
    spmm_slab_bwd<W><<<(unsigned)((p.n_rows + W - 1) / W), 32 * W, 0, st>>>(p, dC, dB);
    return cudaGetLastError();
}

size_t slab_scan_temp_bytes(int64_t n) {
    size_t temp = 0;
    if (n > 0) cub::DeviceScan::InclusiveSum(nullptr, temp, (int64_t*)nullptr, (int64_t*)nullptr, n);
    return temp;
}

cudaError_t launch_slab_count(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr, void* temp,
                              size_t temp_bytes, cudaStream_t st, int* launches) {
    cudaError_t err = launch_sample_count_only(rowptr, n, s, s_rowptr, st);
    ++*launches;
    if (err != cudaSuccess || n == 0) return err;
    err = cub::DeviceScan::InclusiveSum(temp, temp_bytes, s_rowptr + 1, s_rowptr + 1, n, st);
    *launches += 2;                      // CUB's scan: DeviceScanInitKernel + DeviceScanKernel (ncu)
    return err;
}

}  // namespace es
