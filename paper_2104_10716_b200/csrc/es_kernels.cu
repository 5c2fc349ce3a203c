// es_kernels.cu -- sm_100a kernels of the ES-SpMM hot path (arXiv 2104.10716).
//
// One fused kernel per call does all of SURVEY 8(a) a1-a5 for a row:
//   a1  d_i, k_i = min(d_i, s)                     Alg. 1 l.5-6
//   a2  sample positions p_j (Bucket / Eq. 2)      Alg. 1 l.8, L1042-1067
//   a3  stage 1: (colind, val) of the k_i slots    Alg. 1 l.7-11 -- staged in REGISTERS,
//       one slot per lane (coalesced for Bucket), broadcast by warp shuffles, the next
//       32-slot chunk requested one chunk ahead
//   a4  stage 2: gather-FMA over B rows             Alg. 1 l.12-15 -- fp32 FMA of each slot
//       into a per-32-slot partial, partials summed in order (DESIGN.md §6 error bound)
//   a5  epilogue: SUM, or MEAN = / k_i (IEEE)      Alg. 1 l.16, L1570-1575 (R5)
//
// Kernel families (make_plan picks one from F, ldb and alignment):
//   * spmm_tma     : 512 < F <= 1024, 16-B rows: lane 0 of a one-warp CTA moves whole B rows
//                    with cp.async.bulk into a 4-stage smem ring (mbarrier expect_tx);
//   * spmm_cpasync : 64 < F <= 512, 16-B rows: every lane streams its own 16-B pieces of each
//                    B row into a private smem ring with cp.async (no synchronisation);
//   * spmm_warp    : other F/VEC > 16 (8-/4-B aligned rows, F > 1024): one warp per row,
//                    lane l owns feature vectors l + 32c, U rows in flight in registers;
//   * spmm_subwarp : F/VEC <= 16: the warp is split into E = 32/G streams of G lanes, stream e
//                    sums slots j = e (mod E), then an xor-shuffle tree.
// spmm_tma / spmm_cpasync / spmm_warp share one per-element summation order (bitwise equal).
// The order depends only on (k_i, F, vector width), never on which rows a launch covers:
// row blocks computed on different GPUs are bitwise identical.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include "es_device.cuh"
#include "es_internal.h"
#include "es_spmm.h"

namespace es {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
// the plan would take the row stream when rows sample at most this many slots on average; 0:
// never -- measured slower than the two-slot ring at every Arxiv-shaped s (profiles/r02.md)
constexpr int64_t kRowStreamMaxK = 0;
// the degree-sorted half-warp kernel (spmm_grouped): 4-warp CTAs; the plan takes it for F <= 128
// when rows sample at most this many slots on average (profiles/r02_grouped_probe.jsonl)
constexpr int kGroupedWarps = 4;
constexpr int64_t kGroupedMaxK = 0;     // never by default: measured no faster than the two-slot ring (profiles/r02_grouped_probe.jsonl)
// the segmented register stream (spmm_segstream): rows per warp, register cap (4-warp CTAs per
// SM), and the plan's threshold on the mean sampled slots per row (profiles/r02_segstream_probe.jsonl)
constexpr int kSegRows = 8;
constexpr int kSegMinB = 7;
constexpr int kSegCtaWarps = 2;         // 2-warp CTAs: Arxiv s=64 0.132 vs 0.135 ms with 4 (seg10)
constexpr int64_t kSegMaxK = INT64_MAX;

template <int VEC>
__device__ __forceinline__ void store_out(float* Crow, int64_t vidx, int64_t F, const float* r,
                                          bool c_vec, uint64_t pol) {
    const int64_t c0 = vidx * VEC;
    if (c_vec && c0 + VEC <= F) {
        if constexpr (VEC == 4) st_stream4(Crow + c0, r, pol);
        else if constexpr (VEC == 2) st_stream2(Crow + c0, r, pol);
        else st_stream(Crow + c0, r[0], pol);
    } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q)
            if (c0 + q < F) st_stream(Crow + c0 + q, r[q], pol);
    }
}

// a5 store of one VEC-wide piece of local row r: to C, or -- fused all-gather (NEXT-1) -- to
// global row row_base + r of every rank's full C over peer memory (NVLink stores).
template <int VEC>
__device__ __forceinline__ void store_c(const SpmmParams& p, int64_t r, int64_t vidx, const float* res,
                                        uint64_t pol) {
    if (p.c_mc) {                                   // NVLS multicast: one store reaches every rank
        float* row = p.c_mc + (p.row_base + r) * p.ldc;
        const int64_t c0 = vidx * VEC;
        if constexpr (VEC == 4) {
            if (p.c_vec && c0 + 4 <= p.F) { st_multicast4(row + c0, res); return; }
        }
#pragma unroll
        for (int q = 0; q < VEC; ++q)
            if (c0 + q < p.F) st_multicast(row + c0 + q, res[q]);
        return;
    }
    if (p.n_peers == 0) {
        store_out<VEC>(p.C + r * p.ldc, vidx, p.F, res, p.c_vec, pol);
        return;
    }
    const int64_t off = (p.row_base + r) * p.ldc;
    for (int q = 0; q < p.n_peers; ++q)
        store_out<VEC>(p.c_peers[q] + off, vidx, p.F, res, p.c_vec, pol);
}

// a5 epilogue: SUM, or MEAN = / div (IEEE) with div = k_i (reading R5) or d_i (NEXT-4 option)
__device__ __forceinline__ float finish(float x, int reduce, int64_t div) {
    if (reduce == kMean) return div > 0 ? __fdiv_rn(x, (float)div) : 0.0f;
    return x;
}
__device__ __forceinline__ int64_t mean_div(const SpmmParams& p, int64_t d, int32_t k) {
    return p.mean_by_degree ? d : (int64_t)k;
}

// ------------------------------------------------------------------ warp per row
template <int VEC, int NCH, int U, int MINB = 1>
__global__ void __launch_bounds__(kThreads, MINB)
spmm_warp(const SpmmParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();

    RowSampler rs;
    rs.init(ld_stream(p.rowptr + r, pol_a) - p.nnz_base, ld_stream(p.rowptr + r + 1, pol_a) - p.nnz_base,
            p.s, p.strategy, p.seed, p.row_base + r, p.prime);
    const int64_t NV = (p.F + VEC - 1) / VEC;

    for (int64_t v0 = 0; v0 < NV; v0 += 32 * NCH) {       // feature tiles (1 pass if NV <= 32*NCH)
        // part: sequential sum over the (<= 32) slots of the current chunk; tot: sum of chunk
        // partials (DESIGN.md §6 error bound: (31 + ceil(k/32)) u).
        float part[NCH][VEC], tot[NCH][VEC];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int q = 0; q < VEC; ++q) { part[c][q] = 0.0f; tot[c][q] = 0.0f; }

        // stage 1 (a2+a3): lane l samples slot j0+l and loads its (col, val); the next
        // chunk's pair is requested before this chunk's gathers (one chunk of lookahead)
        int32_t col = 0, col_n = 0;
        float a = 0.0f, a_n = 0.0f;
        if (lane < rs.k) {
            const int64_t e = rs.beg + rs.pos(lane);
            col = ld_stream(p.colind + e, pol_a);
            a = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
        }
        for (int32_t j0 = 0; j0 < rs.k; j0 += 32) {
            if (j0 + 32 + lane < rs.k) {
                const int64_t e = rs.beg + rs.pos(j0 + 32 + lane);
                col_n = ld_stream(p.colind + e, pol_a);
                a_n = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
            }
            const int n_here = min(32, rs.k - j0);
            // stage 2 (a4): U slots in flight
            for (int t = 0; t < n_here; t += U) {
                Vec<VEC> x[U][NCH];
                float au[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int src = (t + u) & 31;
                    const int32_t cu = __shfl_sync(kFull, col, src);
                    const float av = __shfl_sync(kFull, a, src);
                    const bool ok = (t + u) < n_here;
                    au[u] = ok ? av : 0.0f;
                    const float* brow = p.B + (int64_t)cu * p.ldb;
#pragma unroll
                    for (int c = 0; c < NCH; ++c) {
                        const int64_t vidx = v0 + lane + 32 * c;
                        if (ok && vidx < NV) {
                            x[u][c] = ld_gather<VEC>(brow + vidx * VEC, pol_b);
                        } else {
#pragma unroll
                            for (int q = 0; q < VEC; ++q) x[u][c].v[q] = 0.0f;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
#pragma unroll
                        for (int q = 0; q < VEC; ++q) part[c][q] = fmaf(au[u], x[u][c].v[q], part[c][q]);
            }
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int q = 0; q < VEC; ++q) { tot[c][q] += part[c][q]; part[c][q] = 0.0f; }
            col = col_n;
            a = a_n;
        }
        // a5 epilogue
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int64_t vidx = v0 + lane + 32 * c;
            if (vidx < NV) {
                float res[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) res[q] = finish(tot[c][q], p.reduce, mean_div(p, rs.d, rs.k));
                store_c<VEC>(p, r, vidx, res, pol_a);
            }
        }
    }
}

// ------------------------------------------------------------------ sub-warp streams (small F)
template <int VEC, int G, int U>
__global__ void __launch_bounds__(kThreads)
spmm_subwarp(const SpmmParams p) {
    constexpr int E = 32 / G;                // edge streams per warp
    const int lane = threadIdx.x & 31;
    const int e = lane / G, g = lane % G;
    const int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();

    RowSampler rs;
    rs.init(ld_stream(p.rowptr + r, pol_a) - p.nnz_base, ld_stream(p.rowptr + r + 1, pol_a) - p.nnz_base,
            p.s, p.strategy, p.seed, p.row_base + r, p.prime);
    const int64_t NV = (p.F + VEC - 1) / VEC;    // <= G
    float acc[VEC], part[VEC];        // acc: sum of per-chunk stream partials
#pragma unroll
    for (int q = 0; q < VEC; ++q) { acc[q] = 0.0f; part[q] = 0.0f; }

    for (int32_t j0 = 0; j0 < rs.k; j0 += 32) {
        int32_t col = 0;
        float a = 0.0f;
        if (j0 + lane < rs.k) {
            const int64_t e_ = rs.beg + rs.pos(j0 + lane);
            col = ld_stream(p.colind + e_, pol_a);
            a = p.val ? ld_stream(p.val + e_, pol_a) : 1.0f;
        }
        const int n_here = min(32, rs.k - j0);
        for (int t = 0; t < n_here; t += E * U) {
            Vec<VEC> x[U];
            float au[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int slot = t + u * E + e;
                const int32_t cu = __shfl_sync(kFull, col, slot & 31);
                const float av = __shfl_sync(kFull, a, slot & 31);
                const bool ok = slot < n_here;
                au[u] = ok ? av : 0.0f;
                if (ok && g < NV) {
                    x[u] = ld_gather<VEC>(p.B + (int64_t)cu * p.ldb + g * VEC, pol_b);
                } else {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) x[u].v[q] = 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < VEC; ++q) part[q] = fmaf(au[u], x[u].v[q], part[q]);
        }
#pragma unroll
        for (int q = 0; q < VEC; ++q) { acc[q] += part[q]; part[q] = 0.0f; }
    }
    // reduce the E streams (xor butterfly: every lane ends with the same bits)
#pragma unroll
    for (int o = G; o < 32; o <<= 1)
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] += __shfl_xor_sync(kFull, acc[q], o);
    if (e == 0 && g < NV) {
        float res[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) res[q] = finish(acc[q], p.reduce, mean_div(p, rs.d, rs.k));
        store_c<VEC>(p, r, g, res, pol_a);
    }
}

// ------------------------------------------------------------------ cp.async ring
// One warp per row; lane l owns feature vectors l + 32c, c < NCH (F <= 128*NCH).  Each lane
// streams ITS OWN 16-B pieces of every gathered B row into a private D-deep shared-memory
// ring with cp.async (SASS LDGSTS): bytes in flight live in smem, not registers (D slots per
// warp at ~40 registers/thread -> 48 warps/SM for F=128), and since a lane only ever reads
// what it copied, no warp or CTA synchronisation is needed.  Same per-element order as
// spmm_warp / spmm_tma (32-slot partials), so results are bitwise interchangeable.
template <typename TB>
struct Piece;                                   // a 16-B piece of a B row, widened to fp32
template <> struct Piece<float> {
    static constexpr int kElems = 4;
    __device__ __forceinline__ static void widen(const float4& raw, float* out) {
        out[0] = raw.x; out[1] = raw.y; out[2] = raw.z; out[3] = raw.w;
    }
};
template <> struct Piece<uint16_t> {            // bf16 storage (NEXT-4): exact widening
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

template <typename TB, int NCH, int D, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
spmm_cpasync(const SpmmParams p) {
    static_assert(D >= 1 && D <= 32, "ring depth");
    constexpr int EPP = Piece<TB>::kElems;                       // B elements per 16-B piece
    extern __shared__ __align__(16) float4 ring_smem[];          // [kWarps][D][NCH*32]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    RowSampler rs;
    rs.init(ld_stream(p.rowptr + r, pol_a) - p.nnz_base, ld_stream(p.rowptr + r + 1, pol_a) - p.nnz_base,
            p.s, p.strategy, p.seed, p.row_base + r, p.prime);
    const int NV = (int)((p.F + EPP - 1) / EPP);
    const int32_t k = rs.k;
    constexpr int kStage = NCH * 32;                             // pieces per stage
    float4* my = ring_smem + (size_t)warp * D * kStage + lane;
    const TB* bl = reinterpret_cast<const TB*>(p.B) + lane * EPP;

    auto copy_slot = [&](int stage, int32_t c) {
        const TB* src = bl + (int64_t)c * p.ldb;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            // no L2 hint on the bf16 instantiations: ptxas 12.9 placed their 64-bit policy
            // descriptor in a misaligned uniform register pair (desc[UR1]) -> illegal
            // instruction on B200 (_build.py now scans the SASS for that pattern)
            if (lane + 32 * ch < NV)
                cp_async16<sizeof(TB) == 4>(my + stage * kStage + 32 * ch, src + 32 * EPP * ch, pol_b);
    };

    // (col, val) of the chunk holding the consumer slot (c0, a0) and of the next chunk (c1, a1)
    int32_t c0 = 0, c1 = 0;
    float a0 = 0.0f, a1 = 0.0f;
    if (lane < k) {
        const int64_t e = rs.beg + rs.pos(lane);
        c0 = ld_stream(p.colind + e, pol_a);
        a0 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
    }
    if (32 + lane < k) {
        const int64_t e = rs.beg + rs.pos(32 + lane);
        c1 = ld_stream(p.colind + e, pol_a);
        a1 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
    }
    // prologue: slots 0 .. D-1 (all in chunk 0 since D <= 32)
#pragma unroll
    for (int t = 0; t < D; ++t) {
        const int32_t c = __shfl_sync(kFull, c0, t);
        if (t < k) copy_slot(t, c);
        cp_async_commit();
    }
    float part[NCH][EPP], tot[NCH][EPP];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < EPP; ++q) { part[ch][q] = 0.0f; tot[ch][q] = 0.0f; }
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
        const int n_here = min(32, k - j0);
#pragma unroll 4
        for (int u = 0; u < 32; ++u) {
            if (u >= n_here) break;
            const int st = (j0 + u) % D;
            cp_async_wait<D - 1>();                               // slot j0+u has landed
            const float av = __shfl_sync(kFull, a0, u);
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                if (lane + 32 * ch < NV) {
                    float x[EPP];
                    Piece<TB>::widen(my[st * kStage + 32 * ch], x);
#pragma unroll
                    for (int q = 0; q < EPP; ++q) part[ch][q] = fmaf(av, x[q], part[ch][q]);
                }
            }
            // refill this stage with slot j0 + u + D (current chunk or the next)
            const int tn = u + D;
            const int32_t cc = __shfl_sync(kFull, c0, tn & 31);
            const int32_t cn = __shfl_sync(kFull, c1, tn & 31);
            if (j0 + tn < k) copy_slot(st, tn < 32 ? cc : cn);
            cp_async_commit();
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < EPP; ++q) { tot[ch][q] += part[ch][q]; part[ch][q] = 0.0f; }
        // advance the chunk window; the chunk after next is requested now (used >= 32 - D slots later)
        c0 = c1;
        a0 = a1;
        c1 = 0;
        a1 = 0.0f;
        if (j0 + 64 + lane < k) {
            const int64_t e = rs.beg + rs.pos(j0 + 64 + lane);
            c1 = ld_stream(p.colind + e, pol_a);
            a1 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
        }
    }
    cp_async_wait<0>();
    // d_i re-read here (L2 hit) instead of kept live through the loop: the loop's register
    // budget decides the occupancy (and spilling cp.async kernels trapped on B200, _build.py)
    int64_t div = k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        if (lane + 32 * ch < NV) {
#pragma unroll
            for (int h = 0; h < EPP / 4; ++h) {
                float res[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) res[q] = finish(tot[ch][4 * h + q], p.reduce, div);
                store_c<4>(p, r, (int64_t)(lane + 32 * ch) * (EPP / 4) + h, res, pol_a);
            }
        }
    }
}

// ------------------------------------------------------------------ row stream (short rows)
// Degree-adaptive mapping for short rows (§4.5.1 thread management L1073-1081, §4.5.3
// load balancing L1100-1105): one warp owns R <= 32 consecutive rows (lane i holds row i's
// metadata) and walks their sampled slots as ONE flat stream t = 0 .. T-1 (T = sum k_i), so the
// cp.async ring (each lane one 16-B piece of the slot's B row, 64 < F <= 128) stays D slots
// ahead across row boundaries and the per-row costs -- the rowptr / colind latency chain, ring
// start-up, the epilogue's reductions -- are paid once per R rows instead of once per row.
// A row's result is stored when the stream passes its last slot (no cross-lane reduction:
// each lane owns its columns).  Per element: the row's slots in slot order with 32-slot chunk
// partials (chunks counted from the row's first slot) -- spmm_cpasync's order, bitwise.
__device__ __forceinline__ int64_t sample_pos(int32_t strategy, uint64_t off, int64_t d, uint32_t prime,
                                              bool narrow, int32_t j) {
    if (strategy == kBucket) return j;
    if (narrow) return (int64_t)(((uint32_t)off + (uint32_t)j * prime) % (uint32_t)d);
    return (int64_t)((off + (uint64_t)j * prime) % (uint64_t)d);
}

template <int D, int R, int W, int MINW>
__global__ void __launch_bounds__(32 * W, MINW / W)
spmm_rowstream(const SpmmParams p) {
    static_assert(D >= 2 && (D & (D - 1)) == 0 && D <= 16 && R >= 1 && R <= 32, "ring depth / rows per warp");
    extern __shared__ __align__(16) float4 ring_smem[];          // [W][D][32]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * W + warp) * R;
    if (r0 >= p.n_rows) return;
    const int nr = (int)min((int64_t)R, p.n_rows - r0);
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    // lane i < nr: row r0 + i (a1: k_i = min(d_i, s); a2: its FastRand rotation, R6)
    RowSampler rs;
    if (lane < nr)
        rs.init(ld_stream(p.rowptr + r0 + lane, pol_a) - p.nnz_base,
                ld_stream(p.rowptr + r0 + lane + 1, pol_a) - p.nnz_base, p.s, p.strategy, p.seed,
                p.row_base + r0 + lane, p.prime);
    else
        rs.init(0, 0, p.s, p.strategy, 0, 0, p.prime);
    const int32_t k_me = rs.k;
    int32_t incl = k_me;                                         // inclusive prefix of k over the rows
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
    }
    const int32_t T = __shfl_sync(kFull, incl, 31);
    const unsigned nonempty = __ballot_sync(kFull, k_me > 0);
    const int NV = (int)((p.F + 3) / 4);
    const bool active = lane < NV;                               // lane owns float4 `lane` of the row
    // rows with k_i = 0 (empty in A): a zero row (no division), stored up front
    unsigned empty = __ballot_sync(kFull, lane < nr && k_me == 0);
    while (empty) {
        const int i = __ffs(empty) - 1;
        empty &= empty - 1;
        const float z[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (active) store_c<4>(p, r0 + i, lane, z, pol_a);
    }
    if (T == 0) return;

    float4* my = ring_smem + (size_t)warp * D * 32 + lane;
    const float* bl = p.B + lane * 4;
    auto copy_slot = [&](int stage, int32_t c) {
        if (active) cp_async16<false>(my + stage * 32, bl + (int64_t)c * p.ldb, pol_b);
    };
    // (col, val) of flat slot t (lane-parallel: each lane one slot of a 32-slot chunk): its row
    // is the first i with incl_i > t, found by a binary search over the lanes' prefixes
    auto load_slot = [&](int32_t t, int32_t& c, float& a) {
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int32_t v = __shfl_sync(kFull, incl, lo + step - 1);
            if (v <= t) lo += step;
        }
        const int i = lo;                                        // row of slot t (lane i holds it)
        const int64_t beg = __shfl_sync(kFull, rs.beg, i);
        const int64_t d = __shfl_sync(kFull, rs.d, i);
        const uint64_t off = __shfl_sync(kFull, rs.off, i);
        const bool narrow = __shfl_sync(kFull, (int)rs.narrow, i) != 0;
        const int32_t j = t - (__shfl_sync(kFull, incl, i) - __shfl_sync(kFull, k_me, i));
        c = 0;
        a = 0.0f;
        if (t < T) {
            const int64_t e = beg + sample_pos(p.strategy, off, d, p.prime, narrow, j);
            c = ld_stream(p.colind + e, pol_a);
            a = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
        }
    };
    int32_t c0, c1;
    float a0, a1;
    load_slot(lane, c0, a0);
    load_slot(32 + lane, c1, a1);
#pragma unroll
    for (int t = 0; t < D; ++t) {
        const int32_t c = __shfl_sync(kFull, c0, t);
        if (t < T) copy_slot(t, c);
        cp_async_commit();
    }
    float part[4] = {0.0f, 0.0f, 0.0f, 0.0f}, tot[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int cur = __ffs(nonempty) - 1;                               // row being accumulated
    int32_t cur_end = __shfl_sync(kFull, incl, cur);
    int32_t j = 0;                                               // slot index within the row
    for (int32_t t0 = 0; t0 < T; t0 += 32) {
        const int n_here = min(32, T - t0);
#pragma unroll 4
        for (int u = 0; u < 32; ++u) {
            if (u >= n_here) break;
            const int32_t t = t0 + u;
            const int st = t & (D - 1);
            cp_async_wait<D - 1>();                               // slot t has landed
            const float av = __shfl_sync(kFull, a0, u);
            if (active) {
                const float4 x = my[st * 32];
                part[0] = fmaf(av, x.x, part[0]);
                part[1] = fmaf(av, x.y, part[1]);
                part[2] = fmaf(av, x.z, part[2]);
                part[3] = fmaf(av, x.w, part[3]);
            }
            const int tn = u + D;                                 // refill: slot t + D
            const int32_t cc = __shfl_sync(kFull, c0, tn & 31);
            const int32_t cn = __shfl_sync(kFull, c1, tn & 31);
            if (t + D < T) copy_slot(st, tn < 32 ? cc : cn);
            cp_async_commit();
            if ((j & 31) == 31) {                                 // the row's 32-slot chunk partial
#pragma unroll
                for (int q = 0; q < 4; ++q) { tot[q] += part[q]; part[q] = 0.0f; }
            }
            ++j;
            if (t + 1 == cur_end) {                               // a5: the row is complete
                const int32_t k = j;
                int64_t div = k;
                if (p.reduce == kMean && p.mean_by_degree) div = __shfl_sync(kFull, rs.d, cur);
                float res[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    res[q] = finish(tot[q] + part[q], p.reduce, div);
                    tot[q] = 0.0f;
                    part[q] = 0.0f;
                }
                if (active) store_c<4>(p, r0 + cur, lane, res, pol_a);
                const unsigned rest = nonempty & ~((2u << cur) - 1u);
                cur = rest ? __ffs(rest) - 1 : 31;
                cur_end = __shfl_sync(kFull, incl, cur);
                j = 0;
            }
        }
        c0 = c1;
        a0 = a1;
        load_slot(t0 + 64 + lane, c1, a1);
    }
    cp_async_wait<0>();
}

// ------------------------------------------------------------------ cp.async ring, two slots per step
// F <= 128 (F/4 <= 32 pieces): the two half-warps take alternate slots (even -> lanes 0-15, odd
// -> lanes 16-31), each lane copying/consuming two 16-B pieces per slot, so the per-slot
// bookkeeping (shuffles, address math, commit/wait) is paid once per two slots.  Each half
// sums its slots in order with 32-slot-chunk partials; the halves are added at the end
// (a + b in both halves, so every lane holds the same bits).  Deterministic; a different
// (interleaved) order than spmm_cpasync, inside the same error bound.
// W warps per CTA (register cap as for MINB 256-thread CTAs).
template <int D, int MINB, int W = kWarps>
__global__ void __launch_bounds__(32 * W, MINB * kWarps / W)
spmm_cpasync_hw(const SpmmParams p) {
    static_assert(D >= 1 && D <= 8, "ring depth (2D slots must fit one 32-slot chunk)");
    extern __shared__ __align__(16) float4 ring_smem[];          // [W][D][2][32]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int h = lane >> 4, sub = lane & 15;
    const int64_t r = (int64_t)blockIdx.x * W + warp;
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    RowSampler rs;
    rs.init(ld_stream(p.rowptr + r, pol_a) - p.nnz_base, ld_stream(p.rowptr + r + 1, pol_a) - p.nnz_base,
            p.s, p.strategy, p.seed, p.row_base + r, p.prime);
    const int NV = (int)((p.F + 3) / 4);                          // <= 32
    const bool act0 = sub < NV, act1 = sub + 16 < NV;
    const int32_t k = rs.k;
    float4* my = ring_smem + (size_t)warp * D * 64 + h * 32 + sub;  // + stage*64 (+16 for piece 1)
    const float* bl = p.B + sub * 4;

    auto copy_slot = [&](int stage, int32_t c) {
        const float* src = bl + (int64_t)c * p.ldb;
        if (act0) cp_async16(my + stage * 64, src, pol_b);
        if (act1) cp_async16(my + stage * 64 + 16, src + 64, pol_b);
    };

    int32_t c0 = 0, c1 = 0;
    float a0 = 0.0f, a1 = 0.0f;
    if (lane < k) {
        const int64_t e = rs.beg + rs.pos(lane);
        c0 = ld_stream(p.colind + e, pol_a);
        a0 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
    }
    if (32 + lane < k) {
        const int64_t e = rs.beg + rs.pos(32 + lane);
        c1 = ld_stream(p.colind + e, pol_a);
        a1 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
    }
    // prologue: steps 0 .. D-1 = slots 0 .. 2D-1 (chunk 0)
#pragma unroll
    for (int t = 0; t < D; ++t) {
        const int32_t c = __shfl_sync(kFull, c0, 2 * t + h);
        if (2 * t + h < k) copy_slot(t, c);
        cp_async_commit();
    }
    float part[8], tot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { part[q] = 0.0f; tot[q] = 0.0f; }
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
        const int n_steps = (min(32, k - j0) + 1) / 2;
#pragma unroll 2
        for (int u = 0; u < 16; ++u) {                           // step u: slots j0+2u (+h)
            if (u >= n_steps) break;
            const int st = (j0 / 2 + u) % D;
            cp_async_wait<D - 1>();
            const int slot = 2 * u + h;
            const float av = __shfl_sync(kFull, a0, slot);
            if (j0 + slot < k) {
                if (act0) {
                    const float4 x = my[st * 64];
                    part[0] = fmaf(av, x.x, part[0]); part[1] = fmaf(av, x.y, part[1]);
                    part[2] = fmaf(av, x.z, part[2]); part[3] = fmaf(av, x.w, part[3]);
                }
                if (act1) {
                    const float4 x = my[st * 64 + 16];
                    part[4] = fmaf(av, x.x, part[4]); part[5] = fmaf(av, x.y, part[5]);
                    part[6] = fmaf(av, x.z, part[6]); part[7] = fmaf(av, x.w, part[7]);
                }
            }
            const int tn = slot + 2 * D;                         // refill: step u + D
            const int32_t cc = __shfl_sync(kFull, c0, tn & 31);
            const int32_t cn = __shfl_sync(kFull, c1, tn & 31);
            if (j0 + tn < k) copy_slot(st, tn < 32 ? cc : cn);
            cp_async_commit();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) { tot[q] += part[q]; part[q] = 0.0f; }
        c0 = c1;
        a0 = a1;
        c1 = 0;
        a1 = 0.0f;
        if (j0 + 64 + lane < k) {
            const int64_t e = rs.beg + rs.pos(j0 + 64 + lane);
            c1 = ld_stream(p.colind + e, pol_a);
            a1 = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
        }
    }
    cp_async_wait<0>();
    int64_t div = k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
    float res[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float o = __shfl_xor_sync(kFull, tot[q], 16);
        res[q] = finish(h == 0 ? tot[q] + o : o + tot[q], p.reduce, div);
    }
    if (h == 0) {
        if (act0) store_c<4>(p, r, sub, res, pol_a);
        if (act1) store_c<4>(p, r, sub + 16, res + 4, pol_a);
    }
}

// ------------------------------------------------------------------ short rows: segmented register stream
// The row-to-warp mapping for short rows (§4.5.1 thread management L1073-1081, §4.5.3
// load balancing L1100-1105), round 2: one warp owns R consecutive rows and walks their sampled
// slots as ONE flat stream, each row padded to whole 4-slot groups, so that
//   * every per-row and per-slot decision is made LANE-PARALLEL once per 32-slot chunk: lane l
//     finds the row of padded slot t0 + l (binary search over the lanes' padded prefix), its
//     position (Eq. 2 / R6), (col, val) and the B row's float4 index; warp ballots turn "slot is
//     real", "group starts a row" and "group starts a 32-slot partial chunk of its row" into
//     uniform bit masks.  A chunk's (col, val) pairs are copied by cp.async straight into one of
//     three per-warp shared-memory slots two chunks ahead (the colind latency is hidden and costs
//     no registers), and a group reads its 4 columns / 4 values with one broadcast LDS.128 each;
//   * row ends and chunk partials fall on group boundaries: one event test per 4-slot group, no
//     per-slot bookkeeping (padding slots: predicated-off gathers and FMAs, no memory traffic);
//   * B rows are gathered register-direct (one LDG.128 per lane per slot; lane l owns float4 l of
//     the row, F <= 128), 4 slots per group, double-buffered: group g+1's loads are issued before
//     group g's FMAs, across chunk boundaries, so 4-8 gathers per warp are always in flight;
//   * the group loop is rolled (two groups per iteration, one copy of the row epilogue per
//     group site): the hot loop stays inside the ~6 KB L0 instruction cache.
// Per element: the row's slots in slot order with 32-slot chunk partials (tot += part at every
// chunk start and at the row's end) -- spmm_warp's order, bitwise.  Needs 4 ldb < 2^32 (the
// row pitch in bytes as a 32-bit multiplier; the ABI checks it).
__device__ __forceinline__ unsigned group_bits(unsigned m) {     // bits 0, 4, .., 28 -> bits 0 .. 7
    m &= 0x11111111u;
    m = (m | (m >> 3)) & 0x03030303u;
    m = (m | (m >> 6)) & 0x000F000Fu;
    return (m | (m >> 12)) & 0xFFu;
}

template <int R, int W, int MINB, bool HAS_VAL>
__global__ void __launch_bounds__(32 * W, MINB)
spmm_segstream(const SpmmParams p) {
    static_assert(R >= 1 && R <= 32, "rows per warp");
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * W + w) * R;
    if (r0 >= p.n_rows) return;
    const int nr = (int)min((int64_t)R, p.n_rows - r0);
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();
    // lane i < nr: row r0 + i (a1: k_i = min(d_i, s); a2: its FastRand rotation, R6)
    RowSampler rs;
    if (lane < nr)
        rs.init(ld_stream(p.rowptr + r0 + lane, pol_a) - p.nnz_base,
                ld_stream(p.rowptr + r0 + lane + 1, pol_a) - p.nnz_base, p.s, p.strategy, p.seed,
                p.row_base + r0 + lane, p.prime);
    else
        rs.init(0, 0, p.s, p.strategy, 0, 0, p.prime);
    const int32_t k_me = rs.k;
    const int32_t kp_me = (k_me + 3) & ~3;                       // padded to whole 4-slot groups
    int32_t incl = kp_me;                                        // inclusive prefix of the padded k
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
    }
    const int32_t T = __shfl_sync(kFull, incl, 31);              // padded slots (multiple of 4)
    const int NV = (int)((p.F + 3) / 4);
    const bool active = lane < NV;                               // lane owns float4 `lane` of the row
    // rows with k_i = 0 (empty in A): a zero row (no division), stored up front
    unsigned empty = __ballot_sync(kFull, lane < nr && k_me == 0);
    while (empty) {
        const int i = __ffs(empty) - 1;
        empty &= empty - 1;
        const float z[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (active) store_c<4>(p, r0 + i, lane, z, pol_a);
    }
    if (T == 0) return;
    unsigned rem = __ballot_sync(kFull, k_me > 0);               // rows not yet started, in order
    // the rows' sampling state (read lane-parallel by the chunk searches) and three chunk slots of
    // (col, val) + masks: chunk k is consumed from slot k % 3 while k+1 is ready and k+2 in flight
    __shared__ int64_t s_beg[W][32], s_d[W][32];
    __shared__ uint64_t s_off[W][32];
    __shared__ int32_t s_start[W][32], s_k[W][32];
    __shared__ __align__(16) int32_t s_col[W][3][32];
    __shared__ __align__(16) float s_a[W][3][32];
    __shared__ unsigned s_mask[W][3][2];                         // [slot][real, events]
    s_beg[w][lane] = rs.beg;
    s_d[w][lane] = rs.narrow ? rs.d : -rs.d;                     // sign: 64-bit position arithmetic
    s_off[w][lane] = rs.off;
    s_start[w][lane] = incl - kp_me;
    s_k[w][lane] = k_me;
    __syncwarp();

    // chunk metadata (a2 + a3, lane-parallel): padded slot t = t0 + lane.  Its (col, val) are
    // copied asynchronously into the slot (one cp.async group per chunk); the masks real (per
    // slot) and events (bits 0-7: group g starts a row, bits 8-15: group g starts a 32-slot chunk
    // of its row) are stored at once.
    auto chunk = [&](int32_t t0, int slot) {
        const int32_t t = t0 + lane;
        int lo = 0;                                              // row of slot t (< R): first i with incl_i > t
#pragma unroll
        for (int step = R > 16 ? 16 : R > 8 ? 8 : R > 4 ? 4 : R > 2 ? 2 : 1; step >= 1; step >>= 1) {
            const int32_t v = __shfl_sync(kFull, incl, lo + step - 1);
            if (v <= t) lo += step;
        }
        const int32_t j = t - s_start[w][lo];
        const bool valid = t < T && j < s_k[w][lo];
        if (valid) {
            const int64_t dd = s_d[w][lo];
            const int64_t e = s_beg[w][lo] + sample_pos(p.strategy, s_off[w][lo], dd < 0 ? -dd : dd, p.prime,
                                                        dd > 0, j);
            cp_async4(&s_col[w][slot][lane], p.colind + e);
            if constexpr (HAS_VAL) cp_async4(&s_a[w][slot][lane], p.val + e);
        }
        cp_async_commit();
        const unsigned real = __ballot_sync(kFull, valid);
        const unsigned ev = group_bits(__ballot_sync(kFull, t < T && j == 0)) |
                            (group_bits(__ballot_sync(kFull, t < T && j > 0 && (j & 31) == 0)) << 8);
        if (lane == 0) { s_mask[w][slot][0] = real; s_mask[w][slot][1] = ev; }
    };
    // the lane's piece of B row 0, held opaque (one register pair, not re-derived per gather);
    // slot address = bl + col * (4 ldb): one IMAD.WIDE.U32 per gather
    uint64_t bl;
    asm("mov.b64 %0, %1;" : "=l"(bl) : "l"(reinterpret_cast<const float4*>(p.B) + (active ? lane : 0)));
    const uint32_t ldb_bytes = (uint32_t)(p.ldb * 4);
    auto load4 = [&](float4 (&x)[4], int slot, unsigned real, int g) {
        const int4 c4 = *reinterpret_cast<const int4*>(&s_col[w][slot][4 * g]);
        const uint32_t cs[4] = {(uint32_t)c4.x, (uint32_t)c4.y, (uint32_t)c4.z, (uint32_t)c4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((real >> (4 * g + q)) & 1u) {
                uint64_t addr;
                asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(addr) : "r"(cs[q]), "r"(ldb_bytes), "l"(bl));
                const Vec<4> v = ld_gather<4>(reinterpret_cast<const float*>(addr), pol_b);
                x[q] = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
            }
        }
    };
    float part[4] = {0.0f, 0.0f, 0.0f, 0.0f}, tot[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int cur = 0;                                                 // lane (row) being accumulated
    bool open = false;
    // plain epilogue store: one 16-B store per lane (no peers / multicast, vector C, whole piece)
    const bool plain_st = !p.c_mc && p.n_peers == 0 && p.c_vec && (int64_t)lane * 4 + 4 <= p.F;
    auto flush = [&]() {                                         // a5: the current row is complete
        float res[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            tot[q] += part[q];
            res[q] = tot[q];
            tot[q] = 0.0f;
            part[q] = 0.0f;
        }
        if (p.reduce == kMean) {                                 // MEAN = / k_i (R5) or / d_i (NEXT-4)
            int64_t div = s_k[w][cur];
            if (p.mean_by_degree) {
                const int64_t dd = s_d[w][cur];
                div = dd < 0 ? -dd : dd;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) res[q] = finish(res[q], kMean, div);
        }
        if (plain_st) st_stream4(p.C + (r0 + cur) * p.ldc + lane * 4, res, pol_a);
        else if (active) store_c<4>(p, r0 + cur, lane, res, pol_a);
    };
    auto consume4 = [&](const float4 (&x)[4], int slot, unsigned real, unsigned ev, int g) {
        if ((ev >> g) & 0x101u) {                                // an event: one uniform test per group
            if ((ev >> g) & 1u) {                                // the group starts the next non-empty row
                if (open) flush();
                cur = __ffs(rem) - 1;
                rem &= rem - 1;
                open = true;
            } else {                                             // the row's next 32-slot chunk
#pragma unroll
                for (int e = 0; e < 4; ++e) { tot[e] += part[e]; part[e] = 0.0f; }
            }
        }
        float av[4] = {1.0f, 1.0f, 1.0f, 1.0f};
        if constexpr (HAS_VAL) {
            const float4 a4 = *reinterpret_cast<const float4*>(&s_a[w][slot][4 * g]);
            av[0] = a4.x; av[1] = a4.y; av[2] = a4.z; av[3] = a4.w;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((real >> (4 * g + q)) & 1u) {
                part[0] = fmaf(av[q], x[q].x, part[0]);
                part[1] = fmaf(av[q], x[q].y, part[1]);
                part[2] = fmaf(av[q], x[q].z, part[2]);
                part[3] = fmaf(av[q], x[q].w, part[3]);
            }
        }
    };

    const int n_chunks = (T + 31) >> 5;
    chunk(0, 0);
    if (n_chunks > 1) chunk(32, 1);
    if (n_chunks > 1) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncwarp();
    unsigned real = s_mask[w][0][0], ev = s_mask[w][0][1];
    float4 x0[4], x1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x0[q] = x1[q] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    load4(x0, 0, real, 0);
    int slot = 0;
    for (int k = 0; k < n_chunks; ++k) {
        const int nslot = slot == 2 ? 0 : slot + 1;
        const bool next = k + 1 < n_chunks;
        unsigned nreal = 0u, nev = 0u;
        if (next) {                                              // chunk k+1 ready (issued a chunk ago); issue k+2
            if (k + 2 < n_chunks) {
                chunk((k + 2) * 32, nslot == 2 ? 0 : nslot + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            nreal = s_mask[w][nslot][0];
            nev = s_mask[w][nslot][1];
        }
        const int ng = min(32, T - k * 32) >> 2;                 // groups in this chunk (8 unless last)
#pragma unroll 1
        for (int g = 0; g < ng; g += 2) {
            if (g + 1 < ng) load4(x1, slot, real, g + 1);
            consume4(x0, slot, real, ev, g);
            if (g + 1 >= ng) break;
            if (g + 2 < ng) load4(x0, slot, real, g + 2);
            else if (next) load4(x0, nslot, nreal, 0);           // the next chunk's first group
            consume4(x1, slot, real, ev, g + 1);
        }
        real = nreal;
        ev = nev;
        slot = nslot;
    }
    if (open) flush();
}

// ------------------------------------------------------------------ short rows: degree-sorted half-warps
// SURVEY 8(a)'s row-to-warp mapping by degree bucket (§4.5.1 L1073-1081 thread
// management, §4.5.3 L1100-1105 load balancing), for graphs whose rows sample few slots (Arxiv:
// mean k 13.7, where a warp per row spends most of its instructions on per-row work).  A warp
// takes 32 consecutive rows; lane i reads row i's (beg, d) and k_i = min(d_i, s), and the warp
// sorts the 32 rows by k_i, descending (bitonic network over shuffles; ties by row).  Then 16
// rounds: in round j the two 16-lane halves take the sorted rows 2j and 2j + 1 -- rows of adjacent
// k, so the halves' slot loops have nearly equal trip counts (an unsorted pair runs as long as its
// longer row) -- and each half streams its row's slots with register-direct 16-B gathers, U slots
// in flight per lane, no shared memory and no cross-lane reduction: lane l of a half owns pieces
// l and l + 16 of the row (F <= 128).  Positions (Eq. 2 / R6) are stepped 16 slots at a time
// (pos + 16 P' mod d), the row's (col, val) staged 16 slots per chunk in the half's lanes, two
// chunks ahead.  Per element: slot order with 32-slot-chunk partials -- spmm_warp's order, bitwise.
template <int U, int MINB>
__global__ void __launch_bounds__(32 * kGroupedWarps, MINB)
spmm_grouped(const SpmmParams p) {
    constexpr int H = 16;                                         // lanes per row
    static_assert(H % U == 0, "slots in flight must divide the chunk");
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, l = lane & 15;
    const int64_t r0 = ((int64_t)blockIdx.x * kGroupedWarps + (threadIdx.x >> 5)) * 32;
    if (r0 >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
    const int NV = (int)((p.F + 3) / 4);                          // 16-B pieces (<= 32)
    const bool act0 = l < NV, act1 = l + 16 < NV;
    // lane i: row r0 + i
    int64_t beg = 0, deg = 0;
    int32_t k = -1;                                               // -1: no row
    if (r0 + lane < p.n_rows) {
        const int64_t a = ld_stream(p.rowptr + r0 + lane, pol_a);
        const int64_t b = ld_stream(p.rowptr + r0 + lane + 1, pol_a);
        beg = a - p.nnz_base;
        deg = b - a;
        k = deg < (int64_t)p.s ? (int32_t)deg : p.s;
    }
    // bitonic sort of (k, lane), descending by k then ascending by lane (a strict order, so every
    // pair of lanes agrees on its exchange)
    int32_t sk = k, si = lane;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int32_t ok = __shfl_xor_sync(kFull, sk, stride), oi = __shfl_xor_sync(kFull, si, stride);
            const bool other_first = ok > sk || (ok == sk && oi < si);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & stride) == 0;
            if ((desc == lower) ? other_first : !other_first) { sk = ok; si = oi; }
        }
    }
    const float* bl = p.B + l * 4;
    for (int round = 0; round < 16; ++round) {
        const int32_t kmax = __shfl_sync(kFull, sk, 2 * round);  // the round's longer row (sorted)
        if (kmax < 0) break;                                      // no rows left (warp-uniform)
        const int32_t kk = __shfl_sync(kFull, sk, 2 * round + h); // this half's row (-1: none)
        const int ri = __shfl_sync(kFull, si, 2 * round + h);
        const int64_t rb = __shfl_sync(kFull, beg, ri), rd = __shfl_sync(kFull, deg, ri);
        const int64_t r = r0 + ri;
        RowSampler rs;
        rs.init(rb, rb + (kk >= 0 ? rd : 0), p.s, p.strategy, p.seed, p.row_base + r, p.prime);
        // slot j = 16m + l of this lane: its CSR position, stepped by 16 slots
        const bool step_ok = p.strategy == kBucket || (rs.narrow && rs.d < ((int64_t)1 << 31));
        const uint32_t d32 = (uint32_t)rs.d;
        const uint32_t delta = p.strategy == kBucket ? 16u : (rs.d > 0 ? (uint32_t)((16ull * rs.prime) % (uint64_t)rs.d) : 0u);
        uint32_t pos = (l < kk) ? (uint32_t)rs.pos(l) : 0u;
        auto load_chunk = [&](int32_t m, int32_t& c, float& a) {     // slot 16m + l
            const int32_t j = 16 * m + l;
            c = 0;
            a = 0.0f;
            if (j < kk) {
                const int64_t pj = step_ok ? (int64_t)pos : rs.pos(j);
                c = ld_stream(p.colind + rs.beg + pj, pol_a);
                a = p.val ? ld_stream(p.val + rs.beg + pj, pol_a) : 1.0f;
            }
            if (step_ok) {                                        // pos of slot j + 16
                pos += delta;
                if (p.strategy != kBucket && pos >= d32) pos -= d32;
            }
        };
        int32_t c0, c1, c2 = 0;
        float a0, a1, a2 = 0.0f;
        load_chunk(0, c0, a0);
        load_chunk(1, c1, a1);
        if (kmax > 32) load_chunk(2, c2, a2);
        float4 v[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        auto issue = [&](int u, int32_t j) {                      // slot j's gathers into v[u]
            const int32_t cj = __shfl_sync(kFull, (j >> 4) == 0 ? c0 : c1, (lane & 16) | (j & 15));
            if (j < kk) {
                const float* src = bl + (int64_t)cj * p.ldb;
                if (act0) { const Vec<4> x = ld_gather<4>(src, pol_b); v[u][0] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]); }
                if (act1) { const Vec<4> x = ld_gather<4>(src + 64, pol_b); v[u][1] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]); }
            }
        };
        float part[8], tot[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) { part[q] = 0.0f; tot[q] = 0.0f; }
#pragma unroll
        for (int u = 0; u < U; ++u) issue(u, u);
        for (int32_t j0 = 0; j0 < kmax; j0 += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t j = j0 + u;                          // slots j0 .. j0+U-1: one chunk
                const float av = __shfl_sync(kFull, a0, (lane & 16) | (j & 15));
                if (j < kk) {
                    part[0] = fmaf(av, v[u][0].x, part[0]); part[1] = fmaf(av, v[u][0].y, part[1]);
                    part[2] = fmaf(av, v[u][0].z, part[2]); part[3] = fmaf(av, v[u][0].w, part[3]);
                    part[4] = fmaf(av, v[u][1].x, part[4]); part[5] = fmaf(av, v[u][1].y, part[5]);
                    part[6] = fmaf(av, v[u][1].z, part[6]); part[7] = fmaf(av, v[u][1].w, part[7]);
                }
                // slot j + U: in this chunk or the next (c1); the chunk rotates below
                const int32_t jn = j + U;
                const int32_t cj = __shfl_sync(kFull, ((jn >> 4) == (j >> 4)) ? c0 : c1, (lane & 16) | (jn & 15));
                if (jn < kk) {
                    const float* src = bl + (int64_t)cj * p.ldb;
                    if (act0) { const Vec<4> x = ld_gather<4>(src, pol_b); v[u][0] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]); }
                    if (act1) { const Vec<4> x = ld_gather<4>(src + 64, pol_b); v[u][1] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]); }
                }
            }
            if (((j0 + U) & 15) == 0) {                             // chunk consumed
                if (((j0 + U) & 31) == 0) {                        // a 32-slot partial
#pragma unroll
                    for (int q = 0; q < 8; ++q) { tot[q] += part[q]; part[q] = 0.0f; }
                }
                c0 = c1; a0 = a1;
                c1 = c2; a1 = a2;
                if (j0 + U + 32 < kmax) load_chunk((j0 + U + 32) >> 4, c2, a2);
            }
        }
        if (kk < 0) continue;
#pragma unroll
        for (int q = 0; q < 8; ++q) tot[q] += part[q];
        const int64_t div = mean_div(p, rs.d, kk);
        float res[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) res[q] = finish(tot[q], p.reduce, div);
        if (act0) store_c<4>(p, r, l, res, pol_a);
        if (act1) store_c<4>(p, r, l + 16, res + 4, pol_a);
    }
}

// The same degree-sorted half-warp pairs with a cp.async ring per half instead of register-direct
// gathers (U = 0 selects it in launch_grouped): lane l of a half copies pieces l and l + 16 of each
// slot's B row into its own D-deep shared-memory ring and reads back only what it copied (no
// synchronisation), so D slots of the row are in flight without holding registers; the next
// round's first (col, val) chunk is loaded during the current round.  Per element: slot order,
// 32-slot-chunk partials -- bitwise spmm_warp / spmm_grouped.
template <int D, int MINB>
__global__ void __launch_bounds__(32 * kGroupedWarps, MINB)
spmm_grouped_ring(const SpmmParams p) {
    extern __shared__ __align__(16) float4 gring[];              // [warps][D][2 pieces][32 lanes]
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, l = lane & 15;
    const int warp = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * kGroupedWarps + warp) * 32;
    if (r0 >= p.n_rows) return;
    float4* my = gring + (size_t)warp * D * 64 + lane;            // + stage * 64 (+ 32 for piece 1)
    const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
    const int NV = (int)((p.F + 3) / 4);
    const bool act0 = l < NV, act1 = l + 16 < NV;
    int64_t beg = 0, deg = 0;
    int32_t k = -1;
    if (r0 + lane < p.n_rows) {
        const int64_t a = ld_stream(p.rowptr + r0 + lane, pol_a);
        const int64_t b = ld_stream(p.rowptr + r0 + lane + 1, pol_a);
        beg = a - p.nnz_base;
        deg = b - a;
        k = deg < (int64_t)p.s ? (int32_t)deg : p.s;
    }
    int32_t sk = k, si = lane;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int32_t ok = __shfl_xor_sync(kFull, sk, stride), oi = __shfl_xor_sync(kFull, si, stride);
            const bool other_first = ok > sk || (ok == sk && oi < si);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & stride) == 0;
            if ((desc == lower) ? other_first : !other_first) { sk = ok; si = oi; }
        }
    }
    const float* bl = p.B + l * 4;
    // a round's row for this half: sampler, stepped positions, the first (col, val) chunk
    struct RoundRow {
        RowSampler rs;
        int32_t kk;
        int64_t r;
        uint32_t pos, delta;
        bool step_ok;
    };
    auto round_row = [&](int round, RoundRow& q) {
        q.kk = __shfl_sync(kFull, sk, 2 * round + h);
        const int ri = __shfl_sync(kFull, si, 2 * round + h);
        const int64_t rb = __shfl_sync(kFull, beg, ri), rd = __shfl_sync(kFull, deg, ri);
        q.r = r0 + ri;
        q.rs.init(rb, rb + (q.kk >= 0 ? rd : 0), p.s, p.strategy, p.seed, p.row_base + q.r, p.prime);
        q.step_ok = p.strategy == kBucket || (q.rs.narrow && q.rs.d < ((int64_t)1 << 31));
        q.delta = p.strategy == kBucket ? 16u : (q.rs.d > 0 ? (uint32_t)((16ull * q.rs.prime) % (uint64_t)q.rs.d) : 0u);
        q.pos = (l < q.kk) ? (uint32_t)q.rs.pos(l) : 0u;
    };
    auto load_chunk = [&](RoundRow& q, int32_t m, int32_t& c, float& a) {   // slot 16m + l of q's row
        const int32_t j = 16 * m + l;
        c = 0;
        a = 0.0f;
        if (j < q.kk) {
            const int64_t pj = q.step_ok ? (int64_t)q.pos : q.rs.pos(j);
            c = ld_stream(p.colind + q.rs.beg + pj, pol_a);
            a = p.val ? ld_stream(p.val + q.rs.beg + pj, pol_a) : 1.0f;
        }
        if (q.step_ok) {
            q.pos += q.delta;
            if (p.strategy != kBucket && q.pos >= (uint32_t)q.rs.d) q.pos -= (uint32_t)q.rs.d;
        }
    };
    RoundRow cur, nxt;
    int32_t nc0 = 0;
    float na0 = 0.0f;
    round_row(0, cur);
    int32_t c0, c1 = 0;
    float a0, a1 = 0.0f;
    load_chunk(cur, 0, c0, a0);
    for (int round = 0; round < 16; ++round) {
        const int32_t kmax = __shfl_sync(kFull, sk, 2 * round);
        if (kmax < 0) break;
        // the next round's row and first chunk, loaded while this round streams
        const bool more = round + 1 < 16 && __shfl_sync(kFull, sk, 2 * round + 2) >= 0;
        if (more) {
            round_row(round + 1, nxt);
            load_chunk(nxt, 0, nc0, na0);
        }
        if (kmax > 16) load_chunk(cur, 1, c1, a1);
        auto copy_slot = [&](int stage, int32_t j, int32_t cj) {
            if (j < cur.kk) {
                const float* src = bl + (int64_t)cj * p.ldb;
                if (act0) cp_async16(my + stage * 64, src, pol_b);
                if (act1) cp_async16(my + stage * 64 + 32, src + 64, pol_b);
            }
        };
#pragma unroll
        for (int t = 0; t < D; ++t) {
            copy_slot(t, t, __shfl_sync(kFull, c0, (lane & 16) | t));
            cp_async_commit();
        }
        float part[8], tot[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) { part[q] = 0.0f; tot[q] = 0.0f; }
        for (int32_t j0 = 0; j0 < kmax; j0 += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int32_t j = j0 + d;                        // stage d (j0 is a multiple of D)
                cp_async_wait<D - 1>();
                const float av = __shfl_sync(kFull, a0, (lane & 16) | (j & 15));
                if (j < cur.kk) {
                    if (act0) {
                        const float4 x = my[d * 64];
                        part[0] = fmaf(av, x.x, part[0]); part[1] = fmaf(av, x.y, part[1]);
                        part[2] = fmaf(av, x.z, part[2]); part[3] = fmaf(av, x.w, part[3]);
                    }
                    if (act1) {
                        const float4 x = my[d * 64 + 32];
                        part[4] = fmaf(av, x.x, part[4]); part[5] = fmaf(av, x.y, part[5]);
                        part[6] = fmaf(av, x.z, part[6]); part[7] = fmaf(av, x.w, part[7]);
                    }
                }
                const int32_t jn = j + D;                        // refill: slot j + D
                const int32_t cn = __shfl_sync(kFull, ((jn >> 4) == (j >> 4)) ? c0 : c1, (lane & 16) | (jn & 15));
                copy_slot(d, jn, cn);
                cp_async_commit();
                if (((j + 1) & 15) == 0) {                       // chunk consumed
                    if (((j + 1) & 31) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) { tot[q] += part[q]; part[q] = 0.0f; }
                    }
                    c0 = c1; a0 = a1;
                    c1 = 0; a1 = 0.0f;
                    if (j + 17 < kmax) load_chunk(cur, ((j + 1) >> 4) + 1, c1, a1);
                }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
        if (cur.kk >= 0) {
#pragma unroll
            for (int q = 0; q < 8; ++q) tot[q] += part[q];
            const int64_t div = mean_div(p, cur.rs.d, cur.kk);
            float res[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) res[q] = finish(tot[q], p.reduce, div);
            if (act0) store_c<4>(p, cur.r, l, res, pol_a);
            if (act1) store_c<4>(p, cur.r, l + 16, res + 4, pol_a);
        }
        if (!more) break;
        cur = nxt;
        c0 = nc0; a0 = na0;
        c1 = 0; a1 = 0.0f;
    }
}

// ------------------------------------------------------------------ per-warp slot stream
// A warp owns R <= 32 consecutive rows; their sampled slots form one flat stream (row by
// row, slot order).  Row i's metadata (a1) lives in lane i; (col, val) of 32 consecutive
// slots (a2+a3) are loaded coalesced by the whole warp, one chunk ahead of use, so no row
// or chunk boundary exposes a dependent-load latency.
struct WarpStream {
    RowSampler rs;      // lane i: row i of the warp
    int32_t kk;         // lane i: k of row i (0 for lanes >= nr)
    int64_t incl;       // lane i: flat end of row i (inclusive prefix of k)
    int64_t T;          // total slots of the warp
    int nr;
    int32_t col_cur, col_nxt;
    float a_cur, a_nxt;
    int64_t chunk_cur;
    int64_t tp;         // producer cursor

    __device__ __forceinline__ void init(const SpmmParams& p, int64_t r_begin, int nrows, int lane,
                                         uint64_t pol) {
        nr = nrows;
        rs = RowSampler{};
        kk = 0;
        if (lane < nr) {
            rs.init(ld_stream(p.rowptr + r_begin + lane, pol) - p.nnz_base,
                    ld_stream(p.rowptr + r_begin + lane + 1, pol) - p.nnz_base,
                    p.s, p.strategy, p.seed, p.row_base + r_begin + lane, p.prime);
            kk = rs.k;
        }
        incl = kk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        T = __shfl_sync(kFull, incl, 31);
        chunk_cur = 0;
        tp = 0;
        load_chunk(p, 0, lane, col_cur, a_cur, pol);
        load_chunk(p, 1, lane, col_nxt, a_nxt, pol);
    }

    // (col, val) of flat slot 32c + lane
    __device__ __forceinline__ void load_chunk(const SpmmParams& p, int64_t c, int lane, int32_t& col,
                                               float& a, uint64_t pol) const {
        const int64_t t = c * 32 + lane;
        const int64_t pre = incl - kk;
        int row = 0;
        for (int i = 1; i < nr; ++i)
            if (__shfl_sync(kFull, pre, i) <= t) row = i;
        const int64_t beg = __shfl_sync(kFull, rs.beg, row);
        const int64_t d = __shfl_sync(kFull, rs.d, row);
        const uint64_t off = __shfl_sync(kFull, rs.off, row);
        const int narrow = __shfl_sync(kFull, (int)rs.narrow, row);
        const int64_t j = t - __shfl_sync(kFull, pre, row);
        col = 0;
        a = 0.0f;
        if (t < T) {
            int64_t pos;
            if (p.strategy == kBucket) pos = j;
            else if (narrow) pos = (int64_t)(((uint32_t)off + (uint32_t)j * p.prime) % (uint32_t)d);
            else pos = (int64_t)((off + (uint64_t)j * p.prime) % (uint64_t)d);
            col = ld_stream(p.colind + beg + pos, pol);
            a = p.val ? ld_stream(p.val + beg + pos, pol) : 1.0f;
        }
    }

    // Warp-collective: (col, val) of the next slot of the stream; false when exhausted.
    __device__ __forceinline__ bool next(const SpmmParams& p, int lane, int32_t& col, float& a,
                                         uint64_t pol) {
        if (tp >= T) return false;
        if ((tp >> 5) != chunk_cur) {
            col_cur = col_nxt;
            a_cur = a_nxt;
            ++chunk_cur;
            load_chunk(p, chunk_cur + 1, lane, col_nxt, a_nxt, pol);
        }
        col = __shfl_sync(kFull, col_cur, (int)(tp & 31));
        a = __shfl_sync(kFull, a_cur, (int)(tp & 31));
        ++tp;
        return true;
    }
};

// Row accumulator of spmm_tma: slot j of a row FMAs into `part`; every 32 slots part is
// added to `tot`.  spmm_warp uses the same order, so the two kernel
// families are bitwise interchangeable (tests: same_as_first in scripts/tune.py).
template <int NCH, int VEC>
struct RowAcc {
    float part[NCH][VEC], tot[NCH][VEC];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int q = 0; q < VEC; ++q) { part[c][q] = 0.0f; tot[c][q] = 0.0f; }
    }
    __device__ __forceinline__ void chunk_end() {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int q = 0; q < VEC; ++q) { tot[c][q] += part[c][q]; part[c][q] = 0.0f; }
    }
    __device__ __forceinline__ void store(const SpmmParams& p, int64_t row, int lane, int64_t NV,
                                          int64_t div, uint64_t pol) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int64_t vidx = lane + 32 * c;
            if (vidx < NV) {
                float res[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) res[q] = finish(tot[c][q] + part[c][q], p.reduce, div);
                store_c<VEC>(p, row, vidx, res, pol);
            }
        }
    }
};

// ------------------------------------------------------------------ TMA ring (wide F)
// One warp per CTA (R rows) and a ring of STAGES B-row buffers in shared memory.  The
// producer cursor of the warp's slot stream runs STAGES slots ahead of the consumer,
// across row boundaries: lane 0 issues one cp.async.bulk (a whole 16-B padded B row,
// ldb*4 bytes) per slot into the stage the consumer just released, completion tracked by
// that stage's mbarrier (expect_tx).  Bytes in flight live in the TMA engine / smem, not in
// registers (profiles/r01.md: 6.7 TB/s DRAM vs 2.4 TB/s for register-staged gathers).
template <int NCH, int STAGES, int MINB>
__global__ void __launch_bounds__(32, MINB)
spmm_tma(const SpmmParams p, int R) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const uint32_t row_bytes = (uint32_t)(p.ldb * 4);       // multiple of 16 (ldb % 4 == 0)
    const int64_t row_floats = p.ldb;
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * row_bytes);
    float* sval = reinterpret_cast<float*>(bar + STAGES);
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_b = policy_evict_last();

    const int64_t r_begin = (int64_t)blockIdx.x * R;
    if (r_begin >= p.n_rows) return;
    const int nr = (int)min((int64_t)R, p.n_rows - r_begin);

    WarpStream ws;
    ws.init(p, r_begin, nr, lane, pol_a);

    if (lane == 0) {
        for (int i = 0; i < STAGES; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();

    int64_t tp = 0;
    auto issue = [&]() {                                       // warp-collective
        int32_t c;
        float a;
        if (!ws.next(p, lane, c, a, pol_a)) return;
        if (lane == 0) {
            const int st = (int)(tp % STAGES);
            sval[st] = a;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[st], row_bytes);
            bulk_g2s(ring + (size_t)st * row_floats, p.B + (int64_t)c * p.ldb, row_bytes, &bar[st], pol_b);
        }
        ++tp;
    };

#pragma unroll 1
    for (int i = 0; i < STAGES; ++i) issue();

    const int64_t NV = (p.F + 3) / 4;
    int64_t tc = 0;                                            // consumer cursor
    RowAcc<NCH, 4> acc;
#pragma unroll 1
    for (int i = 0; i < nr; ++i) {
        const int32_t k = __shfl_sync(kFull, ws.kk, i);
        acc.zero();
#pragma unroll 1
        for (int32_t j = 0; j < k; ++j, ++tc) {
            const int st = (int)(tc % STAGES);
            mbar_wait(&bar[st], (uint32_t)((tc / STAGES) & 1));
            const float av = sval[st];
            const float* src = ring + (size_t)st * row_floats;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const int64_t vidx = lane + 32 * c;
                if (vidx < NV) {
                    const float4 x = *reinterpret_cast<const float4*>(src + vidx * 4);
                    acc.part[c][0] = fmaf(av, x.x, acc.part[c][0]);
                    acc.part[c][1] = fmaf(av, x.y, acc.part[c][1]);
                    acc.part[c][2] = fmaf(av, x.z, acc.part[c][2]);
                    acc.part[c][3] = fmaf(av, x.w, acc.part[c][3]);
                }
            }
            if ((j & 31) == 31) acc.chunk_end();
            __syncwarp();
            issue();                                           // refill the stage just released
        }
        acc.store(p, r_begin + i, lane, NV, mean_div(p, __shfl_sync(kFull, ws.rs.d, i), k), pol_a);
    }
}

// ------------------------------------------------------------------ backward w.r.t. B (NEXT-2)
// The training variant (§6.2, future work there): over the SAME sampled
// slots as the forward, dB[col_ij, :] += w_ij * dC[i, :] with w = val (SUM) or val/k_i (MEAN).
// One warp per row: the dC row is read once into registers (MEAN: divided by k_i with IEEE
// division), then every sampled slot scatters w * dC_row into its B row with 128-bit vector
// reductions (red.global.add.v4.f32).  Summation order across rows is not deterministic.
template <int VEC, int NCH>
__global__ void __launch_bounds__(kThreads)
spmm_bwd_warp(const BwdParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    const uint64_t pol_a = policy_evict_first();
    RowSampler rs;
    rs.init(ld_stream(p.rowptr + r, pol_a) - p.nnz_base, ld_stream(p.rowptr + r + 1, pol_a) - p.nnz_base,
            p.s, p.strategy, p.seed, p.row_base + r, p.prime);
    if (rs.k == 0) return;
    const int64_t NV = (p.F + VEC - 1) / VEC;
    const float* dCrow = p.dC + r * p.ldc;
    for (int64_t v0 = 0; v0 < NV; v0 += 32 * NCH) {
        float x[NCH][VEC];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int64_t vidx = v0 + lane + 32 * c;
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const int64_t col = vidx * VEC + q;
                float v = (vidx < NV && col < p.F) ? ld_stream(dCrow + col, pol_a) : 0.0f;
                x[c][q] = p.reduce == kMean ? __fdiv_rn(v, (float)(p.mean_by_degree ? rs.d : (int64_t)rs.k)) : v;
            }
        }
        for (int32_t j0 = 0; j0 < rs.k; j0 += 32) {
            int32_t colj = 0;
            float a = 0.0f;
            if (j0 + lane < rs.k) {
                const int64_t e = rs.beg + rs.pos(j0 + lane);
                colj = ld_stream(p.colind + e, pol_a);
                a = p.val ? ld_stream(p.val + e, pol_a) : 1.0f;
            }
            const int n_here = min(32, rs.k - j0);
            for (int t = 0; t < n_here; ++t) {
                const int32_t cu = __shfl_sync(kFull, colj, t);
                const float av = __shfl_sync(kFull, a, t);
                float* brow = p.dB + (int64_t)cu * p.ldb;
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const int64_t vidx = v0 + lane + 32 * c;
                    if (vidx >= NV) continue;
                    const int64_t c0 = vidx * VEC;
                    if (c0 + VEC <= p.F) {
                        if constexpr (VEC == 4) red_add4(brow + c0, av * x[c][0], av * x[c][1], av * x[c][2], av * x[c][3]);
                        else if constexpr (VEC == 2) red_add2(brow + c0, av * x[c][0], av * x[c][1]);
                        else red_add1(brow + c0, av * x[c][0]);
                    } else {
#pragma unroll
                        for (int q = 0; q < VEC; ++q)
                            if (c0 + q < p.F) red_add1(brow + c0 + q, av * x[c][q]);
                    }
                }
            }
        }
    }
}

namespace {
template <int VEC>
cudaError_t launch_bwd_vec(const BwdParams& p, cudaStream_t st) {
    const int64_t NV = (p.F + VEC - 1) / VEC;
    const int64_t nch = (NV + 31) / 32;
    const int64_t blocks = (p.n_rows + kWarps - 1) / kWarps;
    if (nch <= 1) spmm_bwd_warp<VEC, 1><<<(unsigned)blocks, kThreads, 0, st>>>(p);
    else if (nch <= 2) spmm_bwd_warp<VEC, 2><<<(unsigned)blocks, kThreads, 0, st>>>(p);
    else if (nch <= 4) spmm_bwd_warp<VEC, 4><<<(unsigned)blocks, kThreads, 0, st>>>(p);
    else spmm_bwd_warp<VEC, 8><<<(unsigned)blocks, kThreads, 0, st>>>(p);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_backward(const BwdParams& p, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    switch (p.vec) {
        case 4: return launch_bwd_vec<4>(p, st);
        case 2: return launch_bwd_vec<2>(p, st);
        default: return launch_bwd_vec<1>(p, st);
    }
}

// ------------------------------------------------------------------ sampler (es_spmm_sample)
// k_i = min(d_i, s), rounded up to a multiple of `pad` slots (pad 4: the flow slab layout, whose
// rows start on a 4-slot step; 1 elsewhere)
__global__ void sample_count(const int64_t* __restrict__ rowptr, int64_t n, int32_t s,
                             int64_t* __restrict__ s_rowptr, WsHeader* hdr, int32_t pad,
                             int32_t* __restrict__ s_k) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        s_rowptr[0] = 0;
        if (hdr) { hdr->status = 0; hdr->sig = 0; }     // a new sampling: clear the workspace header
    }
    if (i < n) {
        const int64_t d = rowptr[i + 1] - rowptr[i];
        const int64_t k = d < (int64_t)s ? d : (int64_t)s;
        s_rowptr[i + 1] = (k + pad - 1) / pad * pad;
        if (s_k) s_k[i] = (int32_t)k;
    }
}

__global__ void __launch_bounds__(kThreads)
sample_materialize(const int64_t* __restrict__ rowptr, int64_t nnz_base,
                   const int32_t* __restrict__ colind, const float* __restrict__ val, int64_t n,
                   int32_t s, int32_t strategy, uint64_t seed, int64_t row_base, uint32_t prime,
                   const int64_t* __restrict__ s_rowptr, int32_t* __restrict__ s_colind,
                   float* __restrict__ s_val, int64_t* __restrict__ s_pos, int64_t cap, WsHeader* hdr,
                   uint64_t sig, int32_t pad) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (hdr && blockIdx.x == 0 && threadIdx.x == 0) hdr->sig = sig;    // the slots' signature
    if (r >= n) return;
    RowSampler rs;
    rs.init(rowptr[r] - nnz_base, rowptr[r + 1] - nnz_base, s, strategy, seed, row_base + r, prime);
    const int64_t o0 = s_rowptr[r];
    // overflow backstop: the row's slots do not fit (the caller understated nnz); the slab
    // passes poison the row (es_slab.cu slab_row_guard) -- flagged here too
    if (hdr && lane == 0 && o0 + (rs.k + pad - 1) / pad * pad > cap) atomicOr(&hdr->status, kWsOverflow);
    for (int32_t j = lane; j < rs.k && o0 + j < cap; j += 32) {
        const int64_t pj = rs.pos(j);
        const int64_t e = rs.beg + pj;
        s_colind[o0 + j] = colind[e];
        if (s_val) s_val[o0 + j] = val ? val[e] : 1.0f;
        if (s_pos) s_pos[o0 + j] = pj;
    }
    // padding slots of the flow layout (k_i .. next multiple of pad): column -1, value 0 -- the
    // flow kernel zero-fills their pieces, so they add exactly +0
    const int32_t kp = (rs.k + pad - 1) / pad * pad;
    if (lane < kp - rs.k && o0 + rs.k + lane < cap) {
        s_colind[o0 + rs.k + lane] = -1;
        if (s_val) s_val[o0 + rs.k + lane] = 0.0f;
    }
}

// ------------------------------------------------------------------ host launchers
namespace {

template <int NCH, int D, int MINB, typename TB = float>
cudaError_t launch_cpasync_k(const SpmmParams& p, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + kWarps - 1) / kWarps;
    auto k = spmm_cpasync<TB, NCH, D, MINB>;
    const size_t smem = (size_t)kWarps * D * NCH * 32 * 16;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, kThreads, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_cpasync_bf16(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    switch (plan.nch) {
        case 1: return launch_cpasync_k<1, 4, 5, uint16_t>(p, st);
        case 2: return launch_cpasync_k<2, 4, 1, uint16_t>(p, st);
        case 3: return launch_cpasync_k<3, 4, 1, uint16_t>(p, st);
        case 4: return launch_cpasync_k<4, 4, 1, uint16_t>(p, st);
        default: return launch_cpasync_k<8, 4, 1, uint16_t>(p, st);
    }
}

template <int D, int MINB, int W>
cudaError_t launch_cpasync_hw_w(const SpmmParams& p, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + W - 1) / W;
    const size_t smem = (size_t)W * D * 64 * 16;
    auto k = spmm_cpasync_hw<D, MINB, W>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

template <int D, int MINB>
cudaError_t launch_cpasync_hw_k(const SpmmParams& p, int cta_warps, cudaStream_t st) {
    // 2-warp CTAs: a CTA's slot frees as soon as its 2 rows are done (short, unequal rows:
    // Arxiv-shaped F=128 s=64 0.177 -> 0.156 ms; Proteins s=64 -0.7 %; profiles/r01.md)
    const int w = cta_warps > 0 ? cta_warps : 2;
    if (w == 4) return launch_cpasync_hw_w<D, MINB, 4>(p, st);
    if (w == 2) return launch_cpasync_hw_w<D, MINB, 2>(p, st);
    return launch_cpasync_hw_w<D, MINB, 8>(p, st);
}

cudaError_t launch_cpasync(const SpmmParams& p, const Plan& plan, const Tune& t, cudaStream_t st) {
    if (plan.bf16) return launch_cpasync_bf16(p, plan, st);
    if (plan.halfwarp) {
        switch (plan.stages) {
            case 2: return launch_cpasync_hw_k<2, 5>(p, t.cta_warps, st);
            case 8: return launch_cpasync_hw_k<8, 5>(p, t.cta_warps, st);
            default: return launch_cpasync_hw_k<4, 5>(p, t.cta_warps, st);
        }
    }
    // Register caps that force spills made this kernel trap with cudaErrorIllegalInstruction on
    // B200 (MINB 8 for f32, 6 for bf16; profiles/r01.md) -- _build.py rejects any spilling
    // spmm_cpasync instantiation, so MINB 5 (48 registers, 40 warps/SM) is the ceiling.
    if (plan.nch == 1) {
        const bool m4 = plan.minb <= 4;
        switch (plan.stages) {
            case 2: return m4 ? launch_cpasync_k<1, 2, 4>(p, st) : launch_cpasync_k<1, 2, 5>(p, st);
            case 3: return m4 ? launch_cpasync_k<1, 3, 4>(p, st) : launch_cpasync_k<1, 3, 5>(p, st);
            case 8: return m4 ? launch_cpasync_k<1, 8, 4>(p, st) : launch_cpasync_k<1, 8, 5>(p, st);
            default: return m4 ? launch_cpasync_k<1, 4, 4>(p, st) : launch_cpasync_k<1, 4, 5>(p, st);
        }
    }
    const bool d2 = plan.stages == 2;
    if (plan.nch == 2) {
        const bool m4 = plan.minb >= 4;
        switch (plan.stages) {
            case 2: return m4 ? launch_cpasync_k<2, 2, 4>(p, st) : launch_cpasync_k<2, 2, 1>(p, st);
            case 8: return m4 ? launch_cpasync_k<2, 8, 4>(p, st) : launch_cpasync_k<2, 8, 1>(p, st);
            default: return m4 ? launch_cpasync_k<2, 4, 4>(p, st) : launch_cpasync_k<2, 4, 1>(p, st);
        }
    }
    switch (plan.nch) {
        case 3: return d2 ? launch_cpasync_k<3, 2, 1>(p, st) : launch_cpasync_k<3, 4, 1>(p, st);
        case 4: return d2 ? launch_cpasync_k<4, 2, 1>(p, st) : launch_cpasync_k<4, 4, 1>(p, st);
        case 5: return d2 ? launch_cpasync_k<5, 2, 1>(p, st) : launch_cpasync_k<5, 4, 1>(p, st);
        case 6: return d2 ? launch_cpasync_k<6, 2, 1>(p, st) : launch_cpasync_k<6, 4, 1>(p, st);
        case 7: return d2 ? launch_cpasync_k<7, 2, 1>(p, st) : launch_cpasync_k<7, 4, 1>(p, st);
        default: return d2 ? launch_cpasync_k<8, 2, 1>(p, st) : launch_cpasync_k<8, 4, 1>(p, st);
    }
}

template <int D, int R, int W, int MINW>
cudaError_t launch_rowstream_k(const SpmmParams& p, cudaStream_t st) {
    const int64_t warps = (p.n_rows + R - 1) / R;
    const int64_t blocks = (warps + W - 1) / W;
    const size_t smem = (size_t)W * D * 32 * 16;
    spmm_rowstream<D, R, W, MINW><<<(unsigned)blocks, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

// rows per warp tune.width (8, 16 or 32; default 16), ring depth tune.stages (4 default; 8)
template <int U, int MINB>
cudaError_t launch_grouped_k(const SpmmParams& p, cudaStream_t st) {
    const int64_t warps = (p.n_rows + 31) / 32;
    const int64_t blocks = (warps + kGroupedWarps - 1) / kGroupedWarps;
    spmm_grouped<U, MINB><<<(unsigned)blocks, 32 * kGroupedWarps, 0, st>>>(p);
    return cudaGetLastError();
}

template <int D, int MINB>
cudaError_t launch_grouped_ring_k(const SpmmParams& p, cudaStream_t st) {
    const int64_t warps = (p.n_rows + 31) / 32;
    const int64_t blocks = (warps + kGroupedWarps - 1) / kGroupedWarps;
    const size_t smem = (size_t)kGroupedWarps * D * 64 * 16;
    auto k = spmm_grouped_ring<D, MINB>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * kGroupedWarps, smem, st>>>(p);
    return cudaGetLastError();
}

// slots in flight per lane U = tune.stages (4 default; 2, 8); tune.variant & 1: the cp.async-ring
// form (ring depth 4, or 8 with stages 8)
cudaError_t launch_grouped(const SpmmParams& p, const Tune& t, cudaStream_t st) {
    if (t.variant & 1) return t.stages == 8 ? launch_grouped_ring_k<8, 5>(p, st) : launch_grouped_ring_k<4, 6>(p, st);
    if (t.stages == 2) return launch_grouped_k<2, 8>(p, st);
    if (t.stages == 8) return launch_grouped_k<8, 4>(p, st);
    return launch_grouped_k<4, 6>(p, st);
}

template <int R, int W, int MINB>
cudaError_t launch_segstream_k(const SpmmParams& p, cudaStream_t st) {
    const int64_t warps = (p.n_rows + R - 1) / R;
    const int64_t blocks = (warps + W - 1) / W;
    if (p.val) spmm_segstream<R, W, MINB, true><<<(unsigned)blocks, 32 * W, 0, st>>>(p);
    else spmm_segstream<R, W, MINB, false><<<(unsigned)blocks, 32 * W, 0, st>>>(p);
    return cudaGetLastError();
}

// rows per warp tune.width (8, 16 or 32, and 4 with 2-warp CTAs at the default cap; default kSegRows),
// register cap tune.stages (CTAs of 4
// warps per SM: 6 = 80 registers, 7 = 72 or 8 = 64; default kSegMinB), tune.cta_warps 2 or 4 warps
// per CTA (default kSegCtaWarps; the register caps are the same per SM)
cudaError_t launch_segstream(const SpmmParams& p, const Tune& t, cudaStream_t st) {
    const int R = t.width > 0 ? t.width : kSegRows;
    const int minb = t.stages > 0 ? t.stages : kSegMinB;
    const int ctaw = t.cta_warps > 0 ? t.cta_warps : kSegCtaWarps;
    if (ctaw == 2) {                                             // 2-warp CTAs (finer tail), same register caps
        if (minb == 6) {
            if (R <= 8) return launch_segstream_k<8, 2, 12>(p, st);
            if (R <= 16) return launch_segstream_k<16, 2, 12>(p, st);
            return launch_segstream_k<32, 2, 12>(p, st);
        }
        if (minb == 8) {
            if (R <= 8) return launch_segstream_k<8, 2, 16>(p, st);
            if (R <= 16) return launch_segstream_k<16, 2, 16>(p, st);
            return launch_segstream_k<32, 2, 16>(p, st);
        }
        if (R <= 4) return launch_segstream_k<4, 2, 14>(p, st);
        if (R <= 8) return launch_segstream_k<8, 2, 14>(p, st);
        if (R <= 16) return launch_segstream_k<16, 2, 14>(p, st);
        return launch_segstream_k<32, 2, 14>(p, st);
    }
    if (minb == 6) {
        if (R <= 8) return launch_segstream_k<8, 4, 6>(p, st);
        if (R <= 16) return launch_segstream_k<16, 4, 6>(p, st);
        return launch_segstream_k<32, 4, 6>(p, st);
    }
    if (minb == 8) {
        if (R <= 8) return launch_segstream_k<8, 4, 8>(p, st);
        if (R <= 16) return launch_segstream_k<16, 4, 8>(p, st);
        return launch_segstream_k<32, 4, 8>(p, st);
    }
    if (R <= 8) return launch_segstream_k<8, 4, 7>(p, st);
    if (R <= 16) return launch_segstream_k<16, 4, 7>(p, st);
    return launch_segstream_k<32, 4, 7>(p, st);
}

cudaError_t launch_rowstream(const SpmmParams& p, const Tune& t, cudaStream_t st) {
    const int R = t.width > 0 ? t.width : 16;
    if (t.stages == 8) {
        if (R <= 8) return launch_rowstream_k<8, 8, 4, 40>(p, st);
        if (R <= 16) return launch_rowstream_k<8, 16, 4, 40>(p, st);
        return launch_rowstream_k<8, 32, 4, 40>(p, st);
    }
    if (R <= 8) return launch_rowstream_k<4, 8, 4, 48>(p, st);
    if (R <= 16) return launch_rowstream_k<4, 16, 4, 48>(p, st);
    return launch_rowstream_k<4, 32, 4, 48>(p, st);
}

template <int VEC, int NCH>
cudaError_t launch_warp(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    constexpr int U = NCH == 1 ? 8 : (NCH == 2 ? 4 : 2);
    const int64_t blocks = (p.n_rows + kWarps - 1) / kWarps;
    if constexpr (NCH == 1 && VEC == 4) {      // tuning variants (ES_SPMM_U / ES_SPMM_MINB)
        auto k = spmm_warp<VEC, 1, 4, 4>;
        if (plan.u == 2) k = plan.minb >= 6 ? spmm_warp<VEC, 1, 2, 6> : plan.minb >= 5 ? spmm_warp<VEC, 1, 2, 5>
                                                                            : spmm_warp<VEC, 1, 2, 4>;
        else if (plan.u == 4) k = plan.minb >= 6 ? spmm_warp<VEC, 1, 4, 6> : plan.minb >= 5 ? spmm_warp<VEC, 1, 4, 5>
                                                                               : spmm_warp<VEC, 1, 4, 4>;
        else if (plan.u == 8) k = plan.minb >= 4 ? spmm_warp<VEC, 1, 8, 4> : spmm_warp<VEC, 1, 8, 3>;
        k<<<(unsigned)blocks, kThreads, 0, st>>>(p);
        return cudaGetLastError();
    } else {
        spmm_warp<VEC, NCH, U><<<(unsigned)blocks, kThreads, 0, st>>>(p);
        return cudaGetLastError();
    }
}

template <int VEC, int G>
cudaError_t launch_subwarp(const SpmmParams& p, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + kWarps - 1) / kWarps;
    spmm_subwarp<VEC, G, 4><<<(unsigned)blocks, kThreads, 0, st>>>(p);
    return cudaGetLastError();
}

template <int NCH, int STAGES>
cudaError_t launch_tma(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    const size_t smem = (size_t)STAGES * (size_t)(p.ldb * 4) + STAGES * 12;
    auto kern = plan.minb >= 24 ? spmm_tma<NCH, STAGES, 24> : spmm_tma<NCH, STAGES, 1>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int64_t blocks = (p.n_rows + plan.rows_per_warp - 1) / plan.rows_per_warp;
    kern<<<(unsigned)blocks, 32, smem, st>>>(p, plan.rows_per_warp);
    return cudaGetLastError();
}

template <int NCH>
cudaError_t dispatch_tma_stages(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    switch (plan.stages) {
        case 3: return launch_tma<NCH, 3>(p, plan, st);
        case 8: return launch_tma<NCH, 8>(p, plan, st);
        default: return launch_tma<NCH, 4>(p, plan, st);
    }
}

cudaError_t dispatch_tma(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    switch (plan.nch) {
        case 2: return dispatch_tma_stages<2>(p, plan, st);
        case 3: return dispatch_tma_stages<3>(p, plan, st);
        case 4: return dispatch_tma_stages<4>(p, plan, st);
        case 5: return dispatch_tma_stages<5>(p, plan, st);
        case 6: return dispatch_tma_stages<6>(p, plan, st);
        case 7: return dispatch_tma_stages<7>(p, plan, st);
        default: return dispatch_tma_stages<8>(p, plan, st);
    }
}

template <int VEC>
cudaError_t dispatch_vec(const SpmmParams& p, const Plan& plan, cudaStream_t st) {
    if (plan.subwarp) {
        switch (plan.g) {
            case 1: return launch_subwarp<VEC, 1>(p, st);
            case 2: return launch_subwarp<VEC, 2>(p, st);
            case 4: return launch_subwarp<VEC, 4>(p, st);
            case 8: return launch_subwarp<VEC, 8>(p, st);
            default: return launch_subwarp<VEC, 16>(p, st);
        }
    }
    switch (plan.nch) {
        case 1: return launch_warp<VEC, 1>(p, plan, st);
        case 2: return launch_warp<VEC, 2>(p, plan, st);
        case 3: return launch_warp<VEC, 3>(p, plan, st);
        case 4: return launch_warp<VEC, 4>(p, plan, st);
        case 5: return launch_warp<VEC, 5>(p, plan, st);
        case 6: return launch_warp<VEC, 6>(p, plan, st);
        case 7: return launch_warp<VEC, 7>(p, plan, st);
        default: return launch_warp<VEC, 8>(p, plan, st);
    }
}

}  // namespace

Plan make_plan_bf16(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C) {
    // bf16 B (NEXT-4): cp.async ring only -- 16-B aligned rows (ldb % 8 == 0), F <= 2048.
    Plan pl{};
    const uintptr_t b = reinterpret_cast<uintptr_t>(B), c = reinterpret_cast<uintptr_t>(C);
    const int64_t nv8 = (F + 7) / 8;
    if (b % 16 != 0 || ldb % 8 != 0 || nv8 > 32 * 8) { pl.unsupported = true; return pl; }
    pl.bf16 = true;
    pl.cpasync = true;
    pl.vec = 4;
    const int64_t nch = (nv8 + 31) / 32;
    pl.nch = nch <= 4 ? (int)nch : 8;
    pl.stages = 4;
    pl.c_vec = (c % 16 == 0) && (ldc % 4 == 0);
    return pl;
}

Plan make_plan(int64_t F, int64_t ldb, int64_t ldc, const void* B, const void* C, int32_t s, const Tune& t,
               int64_t k_est) {
    Plan pl{};
    const uintptr_t b = reinterpret_cast<uintptr_t>(B), c = reinterpret_cast<uintptr_t>(C);
    if (b % 16 == 0 && ldb % 4 == 0) pl.vec = 4;
    else if (b % 8 == 0 && ldb % 2 == 0) pl.vec = 2;
    else pl.vec = 1;
    const int64_t nv = (F + pl.vec - 1) / pl.vec;
    if (nv <= 16) {
        pl.subwarp = true;
        int g = 1;
        while (g < nv) g <<= 1;
        pl.g = g;
    } else {
        pl.subwarp = false;
        const int64_t nch = (nv + 31) / 32;
        pl.nch = (int)(nch > 8 ? 8 : nch);
    }
    pl.c_vec = (c % (4u * (unsigned)pl.vec) == 0) && (ldc % pl.vec == 0);
    pl.u = 4;
    pl.minb = 4;
    const int ov = t.kernel;
    // TMA ring: whole 16-B padded B rows as bulk copies; needs 16-B alignment and F <= 1024.
    // Measured (profiles/r01.md): TMA wins for wide rows (Reddit F=602: 9.5 vs 26.8 ms,
    // F=256: 4.8 vs 8.2 ms); for 512-B rows (F=128) the LDG warp kernel wins (2.97 vs 4.3 ms).
    const int64_t nv4 = (F + 3) / 4;
    constexpr int64_t kTmaMinRowBytes = 2048;
    const bool tma_ok = pl.vec == 4 && nv4 > 32 && nv4 <= 32 * 8;
    pl.tma = tma_ok && ov != ES_KERNEL_WARP && (ov == ES_KERNEL_TMA || ldb * 4 >= kTmaMinRowBytes);
    // cp.async ring: 16-B aligned B, 16 < F/4 <= 128 by default (profiles/r01.md: Reddit F=128
    // 1.95 vs 2.27 ms, F=256 3.13 vs 4.55 (TMA), F=512 7.23 vs 7.51 (TMA); F=602 TMA wins 9.4 vs
    // 10.4); forced up to F/4 <= 256 with ES_KERNEL_CPASYNC.
    const bool force_cp = ov == ES_KERNEL_CPASYNC || ov == ES_KERNEL_CPASYNC_HW;
    pl.cpasync = pl.vec == 4 && nv4 > 16 && nv4 <= 32 * 8 &&
                 (force_cp || ((ov == ES_KERNEL_AUTO || ov == ES_KERNEL_FUSED) && nv4 <= 32 * 4));
    if (pl.cpasync) {
        pl.tma = false;
        pl.nch = (int)((nv4 + 31) / 32);
        pl.stages = t.stages > 0 ? t.stages : 4;
        pl.minb = pl.nch == 1 ? 5 : 1;
        // two slots per step for F <= 128 (profiles/r01.md: Reddit F=128 1.88 vs 1.99 ms,
        // Proteins 1.19 vs 1.30 ms); ES_KERNEL_CPASYNC forces the one-slot ring
        pl.halfwarp = pl.nch == 1 && ov != ES_KERNEL_CPASYNC;
    }
    // row stream for short rows (64 < F <= 128): several rows per warp as one slot stream;
    // forced with ES_KERNEL_ROWSTREAM (A/B; the auto plan keeps the two-slot ring, faster on the
    // Arxiv-shaped graph, mean degree 14: profiles/r02.md)
    if (k_est < 0) k_est = s;
    const bool rs_ok = pl.vec == 4 && nv4 > 16 && nv4 <= 32;
    if (rs_ok && (ov == ES_KERNEL_ROWSTREAM ||
                  ((ov == ES_KERNEL_AUTO || ov == ES_KERNEL_FUSED) && k_est <= kRowStreamMaxK))) {
        pl.rowstream = true;
        pl.cpasync = pl.tma = pl.halfwarp = pl.subwarp = false;
        pl.stages = t.stages == 8 ? 8 : 4;
        pl.rows_per_warp = t.width > 0 ? t.width : 16;
        return pl;
    }
    // short rows (F <= 128): the segmented register stream when rows sample few slots
    if (rs_ok && (ov == ES_KERNEL_SEGSTREAM ||
                  ((ov == ES_KERNEL_AUTO || ov == ES_KERNEL_FUSED) && k_est > 0 && k_est <= kSegMaxK))) {
        pl.segstream = true;
        pl.cpasync = pl.tma = pl.halfwarp = pl.subwarp = pl.rowstream = false;
        pl.rows_per_warp = t.width > 0 ? t.width : kSegRows;
        return pl;
    }
    // short rows (F <= 128): the degree-sorted half-warp kernel when rows sample few slots
    if (rs_ok && (ov == ES_KERNEL_GROUPED ||
                  ((ov == ES_KERNEL_AUTO || ov == ES_KERNEL_FUSED) && k_est > 0 && k_est <= kGroupedMaxK))) {
        pl.grouped = true;
        pl.cpasync = pl.tma = pl.halfwarp = pl.subwarp = pl.rowstream = false;
        return pl;
    }
    if (pl.tma) {
        pl.nch = (int)((nv4 + 31) / 32);
        pl.subwarp = false;
        pl.stages = (t.stages == 3 || t.stages == 8) ? t.stages : 4;
        // rows per warp: 4 when rows are short (s <= 64: the warp's slot stream then spans
        // several rows and one CTA's start-up serves them; Reddit F=602 s=16 1.08 -> 0.94 ms,
        // bitwise identical; profiles/r01.md), else 1 (s = 256: 1 is best)
        pl.rows_per_warp = (t.width >= 1 && t.width <= 32) ? t.width : (s <= 64 ? 4 : 1);
        pl.minb = 1;
    }
    return pl;
}

cudaError_t launch_spmm(SpmmParams p, const Plan& plan, const Tune& t, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    p.c_vec = plan.c_vec ? 1 : 0;
    if (plan.segstream) return launch_segstream(p, t, st);
    if (plan.grouped) return launch_grouped(p, t, st);
    if (plan.rowstream) return launch_rowstream(p, t, st);
    if (plan.tma) return dispatch_tma(p, plan, st);
    if (plan.cpasync) return launch_cpasync(p, plan, t, st);
    switch (plan.vec) {
        case 4: return dispatch_vec<4>(p, plan, st);
        case 2: return dispatch_vec<2>(p, plan, st);
        default: return dispatch_vec<1>(p, plan, st);
    }
}

cudaError_t launch_sample_count_only(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr,
                                     cudaStream_t st, WsHeader* hdr, int32_t pad, int32_t* s_k) {
    const int64_t blocks = (n + 1 + 255) / 256;
    sample_count<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(rowptr, n, s, s_rowptr, hdr, pad, s_k);
    return cudaGetLastError();
}

cudaError_t launch_sample_count(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr,
                                cudaStream_t st, int* launches) {
    cudaError_t err = launch_sample_count_only(rowptr, n, s, s_rowptr, st);
    ++*launches;
    if (err != cudaSuccess || n == 0) return err;
    size_t temp_bytes = 0;
    err = cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, s_rowptr + 1, s_rowptr + 1, n, st);
    if (err != cudaSuccess) return err;
    void* temp = nullptr;
    err = cudaMallocAsync(&temp, temp_bytes, st);
    if (err != cudaSuccess) return err;
    err = cub::DeviceScan::InclusiveSum(temp, temp_bytes, s_rowptr + 1, s_rowptr + 1, n, st);
    *launches += 2;                      // CUB's scan: DeviceScanInitKernel + DeviceScanKernel (ncu)
    cudaError_t err2 = cudaFreeAsync(temp, st);
    return err != cudaSuccess ? err : err2;
}

cudaError_t launch_sample_materialize(const int64_t* rowptr, int64_t nnz_base, const int32_t* colind,
                                      const float* val, int64_t n, int32_t s, int32_t strategy,
                                      uint64_t seed, int64_t row_base, uint32_t prime,
                                      const int64_t* s_rowptr, int32_t* s_colind, float* s_val,
                                      int64_t* s_pos, cudaStream_t st, int64_t cap, WsHeader* hdr,
                                      uint64_t sig, int32_t pad) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + kWarps - 1) / kWarps;
    sample_materialize<<<(unsigned)blocks, kThreads, 0, st>>>(rowptr, nnz_base, colind, val, n, s,
                                                               strategy, seed, row_base, prime,
                                                               s_rowptr, s_colind, s_val, s_pos, cap, hdr, sig,
                                                               pad);
    return cudaGetLastError();
}

}  // namespace es
